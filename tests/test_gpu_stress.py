"""Seeded sweep over shapes the fixed cases do not reach: odd orders, tile
widths that do not divide n, up to 8 logical devices, several right-hand
sides, every dtype -- solution within the reference's tolerances (10 N eps
elementwise against the unblocked oracle, 100 N eps residual) and the
inverse within the same bounds; solutions bit-identical across the device
counts of each case (reference test_solvers.py:172-179)."""

import numpy as np
import pytest

bc = pytest.importorskip("paper_2601_14466_b200")
from oracle import bcmg_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
DTYPES = [np.float32, np.float64, np.complex64, np.complex128]


def _cases(count, seed):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        n = int(rng.integers(33, 700))
        t = int(rng.integers(8, min(n, 300) + 1))
        dt = DTYPES[int(rng.integers(0, 4))]
        nrhs = int(rng.integers(1, 5))
        ds = sorted({int(d) for d in rng.choice([1, 2, 3, 4, 5, 8], size=2, replace=False)})
        yield n, t, dt, nrhs, ds


@pytest.mark.parametrize("n,t,dt,nrhs,ds", list(_cases(16, 2026)))
def test_potrs_sweep(meshes, n, t, dt, nrhs, ds):
    a = O.make_matrix("random_spd", n, dt, n)
    rng = np.random.default_rng(n + t)
    b = rng.standard_normal((n, nrhs))
    if np.iscomplexobj(np.zeros(1, dt)):
        b = b + 1j * rng.standard_normal((n, nrhs))
    b = np.asfortranarray(b.astype(dt))
    xr = O.solve_unblocked(a, b)
    eps = O.eps_of(dt)
    first = None
    for d in ds:
        x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(t))
        assert np.abs(x - xr).max() <= 10 * n * eps * max(1.0, np.abs(xr).max()), (d, np.abs(x - xr).max())
        assert O.solve_residual(a, x, b) <= 100 * n * eps
        if first is None:
            first = x
        else:
            assert np.array_equal(x, first), f"bits differ between D={ds[0]} and D={d}"


@pytest.mark.parametrize("n,t,dt,nrhs,ds", list(_cases(8, 4040)))
def test_potri_sweep(meshes, n, t, dt, nrhs, ds):
    a = O.make_matrix("random_spd", n, dt, n + 1)
    eps = O.eps_of(dt)
    first = None
    for d in ds:
        inv, _ = bc.invert_positive_definite(meshes(d), a, bc.TileSpec(t))
        assert np.array_equal(inv, inv.conj().T)
        assert O.inverse_residual(a, inv) <= 100 * n * eps
        if first is None:
            first = inv
        else:
            assert np.array_equal(inv, first), f"bits differ between D={ds[0]} and D={d}"


@pytest.mark.parametrize("n,t,dt,ds", [
    (3000, 256, np.float32, [1, 3]), (2560, 512, np.complex64, [1, 2]), (2048, 384, np.float64, [1, 4]),
    (2304, 256, np.complex128, [1, 3]), (4096, 1024, np.float32, [2, 4]), (1800, 300, np.complex64, [1, 5]),
])
def test_potrs_sweep_tensor_core_sizes(meshes, n, t, dt, ds):
    """Sizes where the trailing update and panel solve take the tensor-core
    kernels (TMA + DMMA, pre-split tcgen05, complex embeddings)."""
    a = O.make_matrix("random_spd", n, dt, 5)
    b = np.asfortranarray(np.ones((n, 2), dtype=dt))
    eps = O.eps_of(dt)
    first = None
    for d in ds:
        x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(t))
        assert O.solve_residual(a, x, b) <= 100 * n * eps
        if first is None:
            xr = np.linalg.solve(a.astype(np.complex128 if np.iscomplexobj(a) else np.float64), b)
            assert np.abs(x - xr).max() <= 10 * n * eps * max(1.0, np.abs(xr).max())
            first = x
        else:
            assert np.array_equal(x, first), f"bits differ between D={ds[0]} and D={d}"
