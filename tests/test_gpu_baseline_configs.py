"""GPU parity at the BASELINE.json configurations (VERDICT r1 "next" item 1).

* config 2 exactly: potrs float64 N=32768, T_A=1024, N_RHS=16 on one GPU --
  residual over the regenerated A and the analytic diag(1..N) fixture;
* config 4 at reduced N: potri complex128, T_A=512, 8 logical devices --
  inverse residual and bit-identity between 1 and 8 devices;
* config 5 at reduced N: potrs float32 / complex64, N=8192, every T_A of the
  sweep at 8 logical devices -- residual and elementwise against the oracle;
* accuracy stress: ill-conditioned SPD inputs (graded spectrum, kappa up to
  1e8; the SURVEY 8(d) shift of 1.05 x the spectral radius) against the
  oracle's tiled pipeline.

Tolerances (the reference's acceptance criteria, cli.py:113-152 and
test_acceptance.py:143-196): backward residual ||Ax-b||_F / (||A||_F ||x||_F +
||b||_F) <= 100 N eps; elementwise <= 10 N eps max|x| against the oracle on
well-conditioned input; forward error between two backward-stable solvers on
ill-conditioned input <= 2 N kappa eps (normwise, relative).
"""

import ctypes as C

import numpy as np
import pytest

from conftest import ALL_DTYPES
from oracle import bcmg_oracle as O

pytestmark = pytest.mark.gpu

bc = pytest.importorskip("paper_2601_14466_b200")
from paper_2601_14466_b200 import _lib  # noqa: E402

_TORCH = {0: "float32", 1: "float64", 2: "complex64", 3: "complex128"}


def _code(dtype):
    return bc.ElementType.from_dtype(np.dtype(dtype)).code


def _gpu_residual(A, x, b, chunk=4096):
    """||Ax-b||_F / (||A||_F ||x||_F + ||b||_F) in 64-bit on the device (checker only)."""
    import torch

    wide = torch.complex128 if A.is_complex() else torch.float64
    xw, bw = x.to(wide), b.to(wide)
    num2 = torch.zeros((), dtype=torch.float64, device=A.device)
    an2 = torch.zeros((), dtype=torch.float64, device=A.device)
    for r0 in range(0, A.shape[0], chunk):
        blk = A[r0:r0 + chunk].to(wide)
        num2 += (blk @ xw - bw[r0:r0 + chunk]).abs().square().sum()
        an2 += blk.abs().square().sum()
    return float(num2.sqrt() / (an2.sqrt() * xw.norm() + bw.norm()))


# ----------------------------------------------------------------- config 2 (exact)


def test_config2_exact_random_spd(cuda):
    """potrs f64 N=32768, T_A=1024, N_RHS=16 on one B200: A = (R+R^T)/2 + N I
    from the device generator (bench.py's input), overwrite_a=True."""
    import torch

    n, t, nrhs = 32768, 1024, 16
    lib = _lib.load()
    mesh = bc.make_mesh(1)
    A = torch.empty(n, n, dtype=torch.float64, device=cuda)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def regen():
        _lib.check(lib.bcmg_generate_spd(st, 1, n, 0, n, C.c_void_p(A.data_ptr()), n, 1, float(n)))

    regen()
    b = torch.rand(n, nrhs, dtype=torch.float64, device=cuda, generator=torch.Generator(cuda).manual_seed(3)) * 2 - 1
    x = bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)
    regen()
    res = _gpu_residual(A, x, b)
    assert res <= 100 * n * O.eps_of(np.float64), res
    # the generator is exactly symmetric and diagonally dominant
    assert torch.equal(A[:2048, :2048], A[:2048, :2048].t())
    del A
    torch.cuda.empty_cache()


def test_config2_exact_diag_analytic(cuda):
    """diag(1..N), N=32768, T_A=1024, N_RHS=16: x_i = b_i / i within 1e-12
    (the paper's fixture, reference test_acceptance.py:143-166 at config 2's size)."""
    import torch

    n, t, nrhs = 32768, 1024, 16
    A = torch.zeros(n, n, dtype=torch.float64, device=cuda)
    d = torch.arange(1, n + 1, dtype=torch.float64, device=cuda)
    A.diagonal().copy_(d)
    b = torch.ones(n, nrhs, dtype=torch.float64, device=cuda)
    b[:, 1:] *= torch.arange(2, nrhs + 1, dtype=torch.float64, device=cuda)
    x = bc.potrs(A, b, T_A=t, mesh=bc.make_mesh(1), overwrite_a=True)
    want = b / d[:, None]
    assert float((x - want).abs().max()) <= 1e-12
    del A
    torch.cuda.empty_cache()


# ----------------------------------------------------------------- config 4 (reduced N)


@pytest.mark.parametrize("n", [4096, 8192])
def test_config4_potri_c128_reduced(meshes, cuda, n):
    """potri complex128, T_A=512, 8 logical devices (config 4 at N=4096/8192):
    ||AX - I||_F / sqrt(N) <= 100 N eps, exactly Hermitian output, and the same
    bits as on one device."""
    import torch

    t = 512
    a = O.make_matrix("random_spd", n, np.complex128, 21)
    inv8, _ = bc.invert_positive_definite(meshes(8), a, bc.TileSpec(t))
    inv1, _ = bc.invert_positive_definite(meshes(1), a, bc.TileSpec(t))
    assert np.array_equal(inv8, inv1), "potri bits must not depend on the device count"
    assert np.array_equal(inv8, inv8.conj().T), "output must be exactly Hermitian"
    Ad = torch.from_numpy(a).to(cuda)
    Xd = torch.from_numpy(inv8).to(cuda)
    r = float((Ad @ Xd - torch.eye(n, dtype=torch.complex128, device=cuda)).norm() / np.sqrt(n))
    assert r <= 100 * n * O.eps_of(np.complex128), r


# ----------------------------------------------------------------- config 5 (reduced N)


@pytest.mark.parametrize("dtype", [np.float32, np.complex64])
def test_config5_sweep_reduced(meshes, dtype):
    """potrs float32 / complex64, N=8192, T_A in {128..2048}, 8 logical devices,
    b = ones (config 5 at N=8192): residual <= 100 N eps and elementwise within
    10 N eps max|x| of the oracle's tiled pipeline run in 64-bit on the same
    input."""
    n = 8192
    a = O.make_matrix("random_spd", n, dtype, 1)
    b = np.ones((n, 1), dtype=dtype, order="F")
    wide = np.complex128 if np.iscomplexobj(a) else np.float64
    xr = O.solve_pipeline(a.astype(wide), b.astype(wide), 1024)
    eps = O.eps_of(dtype)
    for t in (128, 256, 512, 1024, 2048):
        x, _ = bc.solve_positive_definite(meshes(8), a, b, bc.TileSpec(t))
        assert x.dtype == np.dtype(dtype)
        res = O.solve_residual(a, x, b)
        assert res <= 100 * n * eps, (t, res)
        err = float(np.abs(x.astype(wide) - xr).max())
        assert err <= 10 * n * eps * np.abs(xr).max(), (t, err)


# ----------------------------------------------------------------- accuracy stress


def _graded_spd(n, dtype, kappa, seed):
    """Q diag(lambda) Q^H with lambda log-spaced over [1/kappa, 1], Q the unitary
    factor of a seeded Gaussian matrix (graded and rotated spectrum)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    if np.dtype(dtype).kind == "c":
        g = g + 1j * rng.standard_normal((n, n))
    q, _ = np.linalg.qr(g)
    lam = np.logspace(0, -np.log10(kappa), n)
    a = (q * lam) @ q.conj().T
    a = (a + a.conj().T) / 2
    return np.asfortranarray(a.astype(dtype))


@pytest.mark.parametrize("dtype,kappa", [(np.float64, 1e8), (np.complex128, 1e8), (np.float32, 1e3),
                                         (np.complex64, 1e3)])
def test_ill_conditioned_against_oracle(meshes, dtype, kappa):
    n, t = 2048, 256
    a = _graded_spd(n, dtype, kappa, 11)
    rng = np.random.default_rng(12)
    b = rng.standard_normal((n, 4)).astype(dtype)
    eps = O.eps_of(dtype)
    xr = O.solve_pipeline(a, b, t)  # the reference's tiled arithmetic, same precision
    for d in (1, 2):
        x, _ = bc.solve_positive_definite(meshes(d), a, b, bc.TileSpec(t))
        res = O.solve_residual(a, x, b)
        assert res <= 100 * n * eps, (d, res)
        fwd = float(np.linalg.norm(O._wide(x) - O._wide(xr)) / np.linalg.norm(O._wide(xr)))
        assert fwd <= 2 * n * kappa * eps, (d, fwd)


@pytest.mark.parametrize("dtype", ALL_DTYPES)
def test_shifted_spectral_radius_stress(meshes, dtype):
    """SURVEY 8(d) accuracy-stress input: (R+R^H)/2 + 1.05 rho I (kappa ~ 40)."""
    n, t = 2048, 256
    rng = np.random.default_rng(5)
    r = rng.uniform(-1, 1, (n, n))
    if np.dtype(dtype).kind == "c":
        r = r + 1j * rng.uniform(-1, 1, (n, n))
    h = (r + r.conj().T) / 2
    ev = np.linalg.eigvalsh(h)
    rho = float(np.abs(ev).max())
    a = np.asfortranarray((h + 1.05 * rho * np.eye(n)).astype(dtype))
    kappa = (1.05 * rho + ev.max()) / (1.05 * rho + ev.min())
    assert 20 < kappa < 100
    b = np.ones((n, 2), dtype=dtype, order="F")
    eps = O.eps_of(dtype)
    xr = O.solve_pipeline(a, b, t)
    x, _ = bc.solve_positive_definite(meshes(4), a, b, bc.TileSpec(t))
    assert O.solve_residual(a, x, b) <= 100 * n * eps
    fwd = float(np.linalg.norm(O._wide(x) - O._wide(xr)) / np.linalg.norm(O._wide(xr)))
    assert fwd <= 2 * n * kappa * eps, fwd


# ----------------------------------------------------------------- workspace / session contracts


@pytest.mark.parametrize("dtype", ALL_DTYPES)
def test_pipelines_stay_inside_the_reservation(cuda, dtype):
    """A fresh session running bcmg_potrs / bcmg_potri holds exactly the bytes
    workspace_nbytes reports (the reservation made before any data moves covers
    every buffer the drivers use: out-of-memory cannot strike after movement)."""
    for routine, n, t, d, nrhs in (("potrs", 2048, 256, 4, 3), ("potri", 2048, 256, 4, 1),
                                   ("potrs", 4096, 1024, 2, 70), ("potri", 4096, 512, 8, 1)):
        mesh = bc.DeviceMesh(d, device=0)
        try:
            a = O.make_matrix("random_spd", n, dtype, 2)
            if routine == "potrs":
                bc.solve_positive_definite(mesh, a, np.ones((n, nrhs), dtype=dtype, order="F"), bc.TileSpec(t))
            else:
                bc.invert_positive_definite(mesh, a, bc.TileSpec(t))
            held = C.c_int64(0)
            _lib.check(_lib.load().bcmg_session_workspace_bytes(mesh.session, C.byref(held)))
            desc = bc.MatrixDescriptor(n, n, bc.ElementType.from_dtype(np.dtype(dtype)))
            plan = bc.workspace_nbytes(routine, desc, bc.TileSpec(t), d, n_rhs=nrhs)
            shards = sum(c * n * desc.element_type.width for c in bc.device_column_counts(n, bc.TileSpec(t), d))
            assert held.value == sum(plan) - shards, (routine, n, t, d, held.value, sum(plan) - shards)
        finally:
            mesh.close()


def test_potrs_rejects_a_stale_factorization(cuda):
    """The diagonal-block inverses belong to the LAST successful potrf: solving on
    an older factorization (or another shape / type) is refused with CONFIG,
    never answered with the other matrix's inverses."""
    import torch

    mesh = bc.DeviceMesh(2, device=0)
    try:
        n, t = 512, 64
        mats = []
        for seed in (1, 2):
            a = O.make_matrix("random_spd", n, np.float64, seed)
            desc = bc.MatrixDescriptor(n, n, bc.ElementType.real64, bc.Structure.positive_definite)
            dm = bc.create_distributed(mesh, desc, bc.TileSpec(t))
            bc.write_array(mesh, dm, a)
            mats.append((a, bc.redistribute_in(mesh, dm)))
        assert bc.potrf(mesh, mats[0][1]).info == 0
        assert bc.potrf(mesh, mats[1][1]).info == 0
        rhs = torch.ones(n, dtype=torch.float64, device=cuda)
        with pytest.raises(bc.DescriptorError, match="last successful potrf"):
            bc.potrs_factored(mesh, mats[0][1], [rhs], 1)
        bc.potrs_factored(mesh, mats[1][1], [rhs], 1)  # the current one is fine
        x = rhs.cpu().numpy()[:, None]
        assert O.solve_residual(mats[1][0], x, np.ones((n, 1))) <= 100 * n * O.eps_of(np.float64)
        # potri consumes the factorization (the shards become the inverse)
        bc.potri_factored(mesh, mats[1][1])
        with pytest.raises(bc.DescriptorError, match="last successful potrf"):
            bc.potrs_factored(mesh, mats[1][1], [rhs], 1)
    finally:
        mesh.close()


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_row_sharded_rhs_restored_on_error(meshes, cuda, dtype):
    """BCMG_FLAG_ROW_SHARDED conjugates a complex b for the solve; on a
    not-positive-definite A the caller's b comes back untouched."""
    import torch

    n, t = 256, 64
    a = np.asfortranarray(np.diag(np.r_[np.ones(100), -1.0, np.ones(n - 101)]).astype(dtype))
    A = torch.from_numpy(np.ascontiguousarray(a)).to(cuda)
    b = (torch.arange(n * 2, dtype=torch.float64, device=cuda).reshape(2, n) * (1 + 2j)).to(getattr(torch, _TORCH[_code(dtype)]))
    b0 = b.clone()
    mesh = meshes(2)
    counts = bc.device_column_counts(n, bc.TileSpec(t), 2)
    ptrs = _lib.ptr_array([A.data_ptr(), A.data_ptr() + counts[0] * n * A.element_size()])
    info = C.c_int(0)
    rc = _lib.load().bcmg_potrs(mesh.session, mesh.stream_handle(), _code(dtype), n, 2, t, 2, ptrs,
                                C.c_void_p(b.data_ptr()), n, _lib.BCMG_FLAG_ROW_SHARDED, C.byref(info))
    torch.cuda.synchronize()
    assert rc == _lib.BCMG_ERR_NOT_POSITIVE_DEFINITE and info.value == 101
    assert torch.equal(b, b0)
