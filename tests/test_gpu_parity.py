"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's own golden outputs.  Redistribution is bit-exact; solves and
inverses are within the reference's tolerances (10*N*eps elementwise,
100*N*eps residual, SPEC acceptance criteria); results are bit-identical
across device counts for a fixed tile width (reference test_solvers.py:172-179)."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import ALL_DTYPES, GOLDEN, numbered_columns
from oracle import bcmg_oracle as O

pytestmark = pytest.mark.gpu

bc = pytest.importorskip("paper_2601_14466_b200")


@pytest.fixture(scope="module")
def meshes(cuda):
    cache = {}

    def get(d):
        if d not in cache:
            cache[d] = bc.DeviceMesh(d, device=0)
        return cache[d]

    yield get
    for m in cache.values():
        m.close()


def _et(dtype):
    return bc.ElementType.from_dtype(np.dtype(dtype))


def _redistribute_case(mesh, n_rows, n, t, dtype):
    a = numbered_columns(n_rows, n, dtype)
    desc = bc.MatrixDescriptor(n_rows, n, _et(dtype))
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(t))
    bc.write_array(mesh, dm, a)
    cyc = bc.redistribute_in(mesh, dm)
    from paper_2601_14466_b200.solvers import device_concat

    got = device_concat(mesh, cyc)
    want = O.deal_columns(a, t, mesh.num_devices)
    back = bc.redistribute_out(mesh, cyc)
    return got, want, device_concat(mesh, back), a


# ----------------------------------------------------------------- redistribution


def test_redistribution_exhaustive_grid(meshes):
    """reference test_acceptance.py:86-135 grid (n <= 32, all T, D <= 4, f64; n=16 all dtypes)."""
    bad = []
    cases = [(n, t, d, np.float64) for n in range(1, 33) for t in range(1, n + 1) for d in range(1, 5)]
    cases += [(16, t, d, dt) for t in range(1, 17) for d in range(1, 5) for dt in ALL_DTYPES]
    for n, t, d, dt in cases:
        got, want, back, a = _redistribute_case(meshes(d), 3, n, t, dt)
        if got.tobytes(order="F") != want.tobytes(order="F"):
            bad.append(("forward", n, t, d, np.dtype(dt).name))
        if back.tobytes(order="F") != a.tobytes(order="F"):
            bad.append(("round-trip", n, t, d, np.dtype(dt).name))
    assert bad == []


def test_redistribution_matches_reference_transcript(meshes):
    """Executed order equals the reference's own execute_plan output (golden)."""
    lay = json.load(open(os.path.join(GOLDEN, "layout_golden.json")))
    for c in lay["cases"][::7]:
        n, t, d = c["n"], c["t"], c["d"]
        got, _, _, _ = _redistribute_case(meshes(d), 1, n, t, np.float64)
        assert got[0].astype(np.int64).tolist() == c["executed"], (n, t, d)


@pytest.mark.parametrize("n,t,d,rows", [(2048, 256, 2, 2048), (4096, 512, 4, 64), (1000, 37, 3, 33),
                                        (3072, 128, 8, 16)])
def test_redistribution_large_shapes(meshes, n, t, d, rows):
    rng = np.random.default_rng(n + t + d)
    a = np.asfortranarray(rng.standard_normal((rows, n)))
    desc = bc.MatrixDescriptor(rows, n, bc.ElementType.real64)
    mesh = meshes(d)
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(t))
    bc.write_array(mesh, dm, a)
    cyc = bc.redistribute_in(mesh, dm)
    from paper_2601_14466_b200.solvers import device_concat

    assert np.array_equal(device_concat(mesh, cyc), O.deal_columns(a, t, d))
    back = bc.redistribute_out(mesh, cyc)
    assert np.array_equal(device_concat(mesh, back), a)


# ----------------------------------------------------------------- potrf known answers


def _factor(mesh, a, t):
    desc = bc.MatrixDescriptor(a.shape[0], a.shape[1], _et(a.dtype), bc.Structure.positive_definite)
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(t))
    bc.write_array(mesh, dm, a)
    cyc = bc.redistribute_in(mesh, dm)
    res = bc.potrf(mesh, cyc)
    from paper_2601_14466_b200.solvers import device_concat

    return res, device_concat(mesh, res.factor)


def test_potrf_known_answers(meshes):
    """reference test_solvers.py:67-100."""
    res, f = _factor(meshes(2), np.asfortranarray(np.eye(4)), 2)
    assert res.info == 0 and np.array_equal(f, O.deal_columns(np.eye(4), 2, 2))
    res, f = _factor(meshes(1), np.asfortranarray(np.diag([1.0, 2.0, 3.0, 4.0])), 4)
    assert res.info == 0
    assert np.allclose(np.tril(f), np.diag([1.0, math.sqrt(2.0), math.sqrt(3.0), 2.0]), rtol=0, atol=1e-15)
    res, f = _factor(meshes(2), np.asfortranarray([[4.0, 2.0], [2.0, 3.0]]), 1)
    assert res.info == 0 and np.allclose(np.tril(f), [[2.0, 0.0], [1.0, math.sqrt(2.0)]], atol=1e-15)
    res, _ = _factor(meshes(2), np.asfortranarray(np.diag([1.0, -1.0])), 1)
    assert res.info == 2
    res, f = _factor(meshes(1), np.asfortranarray(np.diag([4.0, 9.0, -1.0])), 1)
    assert res.info == 3 and f[0, 0] == 2.0 and f[1, 1] == 3.0


@pytest.mark.parametrize("n,t", [(96, 64), (200, 64), (300, 128), (1100, 512)])
def test_potrf_info_inside_blocked_tile(meshes, n, t):
    """A negative pivot deep inside a recursively factored tile reports LAPACK info."""
    a = O.make_matrix("random_spd", n, np.float64, 3)
    bad = n - 7
    a[bad, bad] = -1e6
    res, _ = _factor(meshes(2), np.asfortranarray(a), t)
    _, want = O.cholesky_unblocked(a)
    assert res.info == want == bad + 1


# ----------------------------------------------------------------- potrs / potri vs reference golden


def _golden():
    meta = json.load(open(os.path.join(GOLDEN, "solver_golden.json")))
    arr = np.load(os.path.join(GOLDEN, "solver_golden.npz"))
    return meta, arr


def test_potrs_against_reference_golden(meshes):
    meta, arr = _golden()
    for c in meta["cases"]:
        if c["kind"] != "potrs":
            continue
        k = c["key"]
        a, b, xr = arr[k + "_a"], arr[k + "_b"], arr[k + "_x"]
        eps = O.eps_of(a.dtype)
        for d in (1, c["d"], 4):
            x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(c["t"]))
            err = np.abs(x - xr).max()
            assert err <= 10 * c["n"] * eps * max(1.0, np.abs(xr).max()), (k, d, err)
            assert O.solve_residual(a, x, b) <= 100 * c["n"] * eps, (k, d)


def test_potri_against_reference_golden(meshes):
    meta, arr = _golden()
    for c in meta["cases"]:
        if c["kind"] != "potri":
            continue
        k = c["key"]
        a, ir = arr[k + "_a"], arr[k + "_inv"]
        eps = O.eps_of(a.dtype)
        inv, _ = bc.invert_positive_definite(meshes(c["d"]), a, bc.TileSpec(c["t"]))
        assert np.array_equal(inv, inv.conj().T), k
        assert np.abs(inv - ir).max() <= 10 * c["n"] * eps * max(1.0, np.abs(ir).max()), k
        assert O.inverse_residual(a, inv) <= 100 * c["n"] * eps, k


@pytest.mark.parametrize("dtype", ALL_DTYPES)
@pytest.mark.parametrize("n", [64, 256])
def test_potrs_oracle_equivalence(meshes, dtype, n):
    """reference test_acceptance.py:174-196 (T=32, D in 1,2,4)."""
    a = O.make_matrix("random_spd", n, dtype, n)
    b = np.ones((n, 1), dtype=dtype, order="F")
    xr = O.solve_unblocked(a, b)
    eps = O.eps_of(dtype)
    for d in (1, 2, 4):
        x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(32))
        assert np.abs(x - xr).max() <= 10 * n * eps
        assert O.solve_residual(a, x, b) <= 100 * n * eps


def test_device_count_bit_exact(meshes):
    """reference test_solvers.py:172-179 and :221-227."""
    n = 300
    a = O.make_matrix("random_spd", n, np.complex128, 8)
    b = np.asfortranarray(np.ones((n, 2)) + 0.5j)
    base, _ = bc.solve_positive_definite(meshes(1), a, b, bc.TileSpec(40))
    for d in (2, 3, 4):
        x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(40))
        assert np.array_equal(x, base), d
    a = O.make_matrix("random_spd", 150, np.float64, 12)
    base, _ = bc.invert_positive_definite(meshes(1), a, bc.TileSpec(16))
    for d in (2, 4):
        inv, _ = bc.invert_positive_definite(meshes(d), a, bc.TileSpec(16))
        assert np.array_equal(inv, base), d
    a = O.make_matrix("random_spd", 200, np.complex128, 13)
    base, _ = bc.invert_positive_definite(meshes(1), a, bc.TileSpec(24))
    for d in (3, 4):
        inv, _ = bc.invert_positive_definite(meshes(d), a, bc.TileSpec(24))
        assert np.array_equal(inv, base), d


def test_potri_large_device_count_bit_exact(meshes):
    """potri at a size where the W-sweep GEMMs take the TMA kernel on one
    device and the cp.async kernels on two: same bits, inverse within tolerance."""
    n, t = 4096, 512
    a = O.make_matrix("random_spd", n, np.float64, 3)
    base, _ = bc.invert_positive_definite(meshes(1), a, bc.TileSpec(t))
    assert np.array_equal(base, base.T)
    assert O.inverse_residual(a, base) <= 100 * n * O.eps_of(np.float64)
    inv, _ = bc.invert_positive_definite(meshes(2), a, bc.TileSpec(t))
    assert np.array_equal(inv, base)


def test_paper_benchmark_fixture(meshes):
    """A = diag(1..N), b = ones -> x = 1/i (reference test_acceptance.py:143-166)."""
    n = 4096
    a = np.asfortranarray(np.diag(np.arange(1.0, n + 1)))
    for t in (64, 256, 1024):
        x, _ = bc.solve_positive_definite(meshes(4), a, np.ones((n, 1), order="F"), bc.TileSpec(t))
        assert np.abs(x[:, 0] - 1.0 / np.arange(1.0, n + 1)).max() <= 1e-12
    n32 = 1024
    a32 = np.asfortranarray(np.diag(np.arange(1.0, n32 + 1)).astype(np.float32))
    for t in (64, 256, 1024):
        x, _ = bc.solve_positive_definite(meshes(4), a32, np.ones((n32, 1), np.float32, order="F"), bc.TileSpec(t))
        assert np.abs(x[:, 0].astype(np.float64) - 1.0 / np.arange(1.0, n32 + 1)).max() <= 1e-4


def test_config1_matches_reference(meshes):
    """BASELINE config 1: potrs f64 N=2048, T=256, N_RHS=1, 2 devices, random_spd seed 1."""
    meta, arr = _golden()
    cfg = meta["config1"]
    a = O.make_matrix("random_spd", cfg["n"], np.float64, cfg["seed"])
    assert hashlib.sha256(a.tobytes(order="F")).hexdigest() == cfg["a_sha256"]
    b = np.ones((cfg["n"], 1), order="F")
    x, _ = bc.solve_positive_definite(meshes(cfg["d"]), a, b, bc.TileSpec(cfg["t"]))
    xr = arr["config1_x"]
    assert np.abs(x - xr).max() <= 1e-10 * np.abs(xr).max()
    assert O.solve_residual(a, x, b) <= 100 * cfg["n"] * O.eps_of(np.float64)


def test_potri_quality(meshes):
    """reference test_acceptance.py:204-215."""
    n = 256
    for dt in (np.float64, np.complex128):
        a = O.make_matrix("random_spd", n, dt, 21)
        inv, _ = bc.invert_positive_definite(meshes(2), a, bc.TileSpec(32))
        assert O.inverse_residual(a, inv) <= 100 * n * O.eps_of(dt)
    a = np.asfortranarray(np.diag(np.arange(1.0, n + 1)))
    inv, _ = bc.invert_positive_definite(meshes(2), a, bc.TileSpec(32))
    assert np.abs(inv - np.diag(1.0 / np.arange(1.0, n + 1))).max() <= 1e-12


def test_errors(meshes):
    with pytest.raises(bc.NotPositiveDefiniteError) as exc:
        bc.solve_positive_definite(meshes(2), np.asfortranarray(np.diag([1.0, -1.0])), np.ones((2, 1)),
                                   bc.TileSpec(1))
    assert exc.value.pivot == 2 and "pivot=2" in str(exc.value)
    with pytest.raises(bc.NotPositiveDefiniteError) as exc:
        bc.invert_positive_definite(meshes(2), np.asfortranarray(np.diag([1.0, -1.0])), bc.TileSpec(1))
    assert exc.value.pivot == 2
    with pytest.raises(bc.DescriptorError):
        bc.solve_positive_definite(meshes(1), np.eye(4), np.ones((3, 1)), bc.TileSpec(2))
    with pytest.raises(bc.DescriptorError) as e2:
        bc.solve_positive_definite(meshes(1), np.eye(6), np.ones((6, 1)) + 1j, bc.TileSpec(2))
    assert e2.value.kind == "type-structure"
    with pytest.raises(bc.DescriptorError):
        bc.solve_positive_definite(meshes(1), np.eye(8), np.ones((8, 1)), bc.TileSpec(16))


# ----------------------------------------------------------------- drop-in API


@pytest.mark.parametrize("dtype", ALL_DTYPES)
def test_dropin_potrs_row_sharded(meshes, dtype):
    import torch

    n, t = 512, 64
    a = O.make_matrix("random_spd", n, dtype, 5)
    rng = np.random.default_rng(1)
    b = rng.standard_normal((n, 3)).astype(dtype)
    mesh = meshes(4)
    A = torch.from_numpy(np.ascontiguousarray(a)).cuda()  # row-major, row-sharded over 4 virtual devices
    x = bc.potrs(A, torch.from_numpy(b).cuda(), T_A=t, mesh=mesh, in_specs=(bc.P("x", None), bc.P(None, None)))
    xr = O.solve_unblocked(a, b)
    eps = O.eps_of(dtype)
    assert np.abs(x.cpu().numpy() - xr).max() <= 10 * n * eps * max(1, np.abs(xr).max())
    assert np.array_equal(A.cpu().numpy(), np.ascontiguousarray(a)), "caller's A must be untouched"


@pytest.mark.parametrize("shape", [(256, 1), (256,)])
def test_dropin_potrs_leaves_b_untouched(meshes, shape):
    """Caller inputs are never mutated (reference SPEC.md:556), including a
    single right-hand side already on the device in the solve dtype."""
    import torch

    n = shape[0]
    a = O.make_matrix("random_spd", n, np.float64, 9)
    b = torch.ones(shape, dtype=torch.float64, device="cuda")
    x = bc.potrs(torch.from_numpy(np.ascontiguousarray(a)).cuda(), b, T_A=32, mesh=meshes(2))
    assert torch.equal(b, torch.ones_like(b))
    assert x.shape == b.shape and x.data_ptr() != b.data_ptr()
    xr = O.solve_unblocked(a, np.ones((n, 1)))
    assert np.abs(x.cpu().numpy().reshape(n, 1) - xr).max() <= 10 * n * O.eps_of(np.float64)


def test_dropin_potri_row_sharded(meshes):
    import torch

    n = 256
    a = O.make_matrix("random_spd", n, np.complex128, 7)
    A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    inv = bc.potri(A, T_A=32, mesh=meshes(2), in_specs=(bc.P("x", None),)).cpu().numpy()
    assert O.inverse_residual(a, inv) <= 100 * n * O.eps_of(np.complex128)


@pytest.mark.parametrize("n,t,d,rows,chunk", [(2048, 256, 2, 64, 8192), (1000, 37, 3, 33, 1 << 20),
                                              (96, 8, 4, 5, 1 << 20)])
def test_staged_redistribution_path(meshes, monkeypatch, n, t, d, rows, chunk):
    """The cross-process (pack / exchange / unpack) redistribution algorithm,
    forced on one process: bit-exact forward and round trip."""
    monkeypatch.setenv("BCMG_STAGED_REDIST", "1")
    monkeypatch.setenv("BCMG_REDIST_STAGING", str(chunk))
    rng = np.random.default_rng(n + d)
    a = np.asfortranarray(rng.standard_normal((rows, n)))
    desc = bc.MatrixDescriptor(rows, n, bc.ElementType.real64)
    mesh = meshes(d)
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(t))
    bc.write_array(mesh, dm, a)
    cyc = bc.redistribute_in(mesh, dm)
    from paper_2601_14466_b200.solvers import device_concat

    assert np.array_equal(device_concat(mesh, cyc), O.deal_columns(a, t, d))
    back = bc.redistribute_out(mesh, cyc)
    assert np.array_equal(device_concat(mesh, back), a)


@pytest.mark.parametrize("dtype,n,t", [(np.float64, 2048, 128), (np.float64, 1000, 96), (np.complex128, 768, 96),
                                       (np.float32, 1024, 128)])
def test_dropin_streamed_host_input(meshes, dtype, n, t):
    """Pinned host A on one device streams in while the factorisation starts
    (bcmg_potrs_streamed; float64: first quarter of the tiles left-looking):
    same answer as the device-resident call to rounding, reference tolerances."""
    import torch

    a = O.make_matrix("random_spd", n, dtype, 17)
    b = np.random.default_rng(4).standard_normal((n, 2)).astype(dtype)
    mesh = meshes(1)
    host = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    x = bc.potrs(host, torch.from_numpy(b), T_A=t, mesh=mesh).cpu().numpy()
    xd = bc.potrs(host.cuda(), torch.from_numpy(b), T_A=t, mesh=mesh).cpu().numpy()
    eps = O.eps_of(dtype)
    xr = O.solve_unblocked(a, b)
    assert np.abs(x - xr).max() <= 10 * n * eps * max(1.0, np.abs(xr).max())
    assert np.abs(x - xd).max() <= 10 * n * eps * max(1.0, np.abs(xd).max())
    assert O.solve_residual(a, x, b) <= 100 * n * eps
    assert np.array_equal(host.numpy(), np.ascontiguousarray(a)), "caller's host A must be untouched"


@pytest.mark.parametrize("bad", [150, 700])
def test_dropin_streamed_not_positive_definite(meshes, bad):
    """A failing pivot in the left-looking upload phase (tile 2) or in the
    right-looking phase (tile 10) raises with the LAPACK pivot."""
    import torch

    n, t = 1024, 64
    a = np.diag(np.arange(1.0, n + 1))
    a[bad, bad] = -1.0
    host = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    with pytest.raises(bc.NotPositiveDefiniteError) as ei:
        bc.potrs(host, torch.ones(n, dtype=torch.float64), T_A=t, mesh=meshes(1))
    assert ei.value.pivot == bad + 1


def test_out_of_memory_before_any_data_movement(meshes):
    """Workspace is reserved before the pipeline touches the shards: an
    impossible workspace fails with OUT_OF_MEMORY and the input is unchanged
    (reference test_solvers.py:344-352)."""
    import ctypes as C

    import torch

    from paper_2601_14466_b200 import _lib

    lib = _lib.load()
    mesh = meshes(1)
    buf = torch.arange(4096, dtype=torch.float64, device="cuda")
    before = buf.clone()
    n, t = 2_000_000, 100_000  # panels alone would need ~1.6 TB
    x = torch.zeros(16, dtype=torch.float64, device="cuda")
    info = C.c_int(0)
    rc = lib.bcmg_potrs(mesh.session, mesh.stream_handle(), 1, n, 1, t, 1, _lib.ptr_array([buf.data_ptr()]),
                        C.c_void_p(x.data_ptr()), n, 0, C.byref(info))
    assert rc == _lib.BCMG_ERR_OUT_OF_MEMORY
    torch.cuda.synchronize()
    assert torch.equal(buf, before)
    # the session is still usable afterwards
    a = O.make_matrix("random_spd", 64, np.float64, 1)
    xs, _ = bc.solve_positive_definite(mesh, a, np.ones((64, 1)), bc.TileSpec(16))
    assert O.solve_residual(a, xs, np.ones((64, 1))) <= 100 * 64 * O.eps_of(np.float64)


@pytest.mark.parametrize("dtype", ALL_DTYPES)
@pytest.mark.parametrize("nrhs", [1, 2, 3, 4, 5])
def test_potrs_narrow_rhs_sweeps(meshes, dtype, nrhs):
    """The substitution's bandwidth kernels (N_RHS <= 4, not float64) and the
    split-K path (N_RHS = 5, float64): ragged n, chunks of 512 rows crossed,
    against the unblocked oracle, and the same bits for D = 1 and 3."""
    n, t = 1100, 96
    a = O.make_matrix("random_spd", n, dtype, 30 + nrhs)
    rng = np.random.default_rng(nrhs)
    b = rng.standard_normal((n, nrhs))
    if np.iscomplexobj(np.zeros(1, dtype)):
        b = b + 1j * rng.standard_normal((n, nrhs))
    b = np.asfortranarray(b.astype(dtype))
    xr = O.solve_unblocked(a, b)
    eps = O.eps_of(dtype)
    base, _ = bc.solve_positive_definite(meshes(1), a, b, bc.TileSpec(t))
    assert np.abs(base - xr).max() <= 10 * n * eps * max(1.0, np.abs(xr).max())
    assert O.solve_residual(a, base, b) <= 100 * n * eps
    x3, _ = bc.solve_positive_definite(meshes(3), a, b, bc.TileSpec(t))
    assert np.array_equal(x3, base)


@pytest.mark.parametrize("dtype", ALL_DTYPES)
def test_potri_device_count_bit_exact_ragged(meshes, dtype):
    """potri bits do not depend on D for every dtype, with a ragged last tile
    and devices whose column counts fall under the tcgen05 tile width (found
    by tools/stress.py: float32 n=649, T_A=64, D=2)."""
    n, t = 649, 64
    a = O.make_matrix("random_spd", n, dtype, 1172)
    base, _ = bc.invert_positive_definite(meshes(1), a, bc.TileSpec(t))
    assert O.inverse_residual(a, base) <= 100 * n * O.eps_of(dtype)
    for d in (2, 3, 8):
        inv, _ = bc.invert_positive_definite(meshes(d), a, bc.TileSpec(t))
        assert np.array_equal(inv, base), d


@pytest.mark.parametrize("dtype", [np.float32, np.complex64])
def test_potrs_device_count_bit_exact_odd_n_wide_tile(meshes, dtype):
    """Odd n puts later devices' shards at 4-byte offsets of the flat buffer;
    the diagonal factor's GEMMs must not pick a different kernel for them
    (found by tools/stress.py: float32 n=1441, T_A=512, D=2)."""
    n, t = 1441, 512
    a = O.make_matrix("random_spd", n, dtype, 77)
    b = np.asfortranarray(np.ones((n, 2), dtype=dtype))
    base, _ = bc.solve_positive_definite(meshes(1), a, b, bc.TileSpec(t))
    assert O.solve_residual(a, base, b) <= 100 * n * O.eps_of(dtype)
    for d in (2, 3):
        x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(t))
        assert np.array_equal(x, base), d
