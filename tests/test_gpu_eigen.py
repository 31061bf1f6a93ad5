"""GPU parity of the eigensolver (csrc/eigen.cu through bcmg_syevd /
bcmg_syevd_cyclic) against the reference's golden outputs and the oracle,
with the reference's own eigensolver tests (test_solvers.py:231-280,
test_acceptance.py:219-268) restated on the GPU path."""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import bcmg_oracle as O

pytestmark = pytest.mark.gpu

bc = pytest.importorskip("paper_2601_14466_b200")
G = np.load(os.path.join(GOLDEN, "eigen_golden.npz"))
CASES = sorted({k.split("__")[0] for k in G.files})


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


def _eps(dt):
    return float(np.finfo(np.float32 if np.dtype(dt) in (np.float32, np.complex64) else np.float64).eps)


def _quality(a, w, v):
    wide = np.complex128 if np.iscomplexobj(a) else np.float64
    a64, v64 = a.astype(wide), v.astype(wide)
    n = a.shape[0]
    res = np.linalg.norm(a64 @ v64 - v64 * w.astype(np.float64)) / np.linalg.norm(a64)
    orth = np.linalg.norm(v64.conj().T @ v64 - np.eye(n))
    return res, orth


@pytest.mark.parametrize("name", CASES)
def test_matches_reference_golden(meshes, name):
    a, w_ref, v_ref, cfg = (G[f"{name}__{k}"] for k in ("a", "w", "v", "cfg"))
    n = a.shape[0]
    d, t = int(cfg[0]), int(cfg[1])
    w, v, _ = bc.eigh_hermitian(meshes(d), a, bc.TileSpec(t))
    eps = _eps(a.dtype)
    assert w.dtype == w_ref.dtype and v.dtype == a.dtype and v.shape == a.shape
    assert np.all(np.diff(w) >= 0)
    scale = max(1.0, float(np.max(np.abs(w_ref))))
    assert np.max(np.abs(w.astype(np.float64) - w_ref)) <= 10 * n * eps * scale
    res, orth = _quality(a, w, v)
    assert res <= 100 * n * eps and orth <= 100 * n * eps, (res, orth)
    if name.startswith("sep") or name in ("diag3", "hand2"):
        wide = np.complex128 if np.iscomplexobj(a) else np.float64
        assert np.max(np.abs(v.astype(wide) - v_ref.astype(wide))) <= 100 * n * eps


def test_diag_is_sorted_permutation(meshes):
    """test_solvers.py:235-239"""
    w, v, _ = bc.eigh_hermitian(meshes(1), np.asfortranarray(np.diag([3.0, 1.0, 2.0])), bc.TileSpec(1))
    assert np.allclose(w, [1.0, 2.0, 3.0], atol=1e-14)
    assert np.allclose(np.abs(v), np.eye(3)[:, [1, 2, 0]], atol=1e-12)


def test_hand_2x2(meshes):
    """test_solvers.py:242-249"""
    w, v, _ = bc.eigh_hermitian(meshes(2), np.asfortranarray([[2.0, 1.0], [1.0, 2.0]]), bc.TileSpec(1))
    assert np.allclose(w, [1.0, 3.0], atol=5e-15)
    s = 1.0 / math.sqrt(2.0)
    for k, want in enumerate((np.array([s, -s]), np.array([s, s]))):
        aligned = v[:, k] if abs(v[0, k] - want[0]) < abs(-v[0, k] - want[0]) else -v[:, k]
        assert np.max(np.abs(aligned - want)) <= 5e-15


def test_identity_degenerate(meshes):
    """test_solvers.py:252-256"""
    w, v, _ = bc.eigh_hermitian(meshes(2), np.asfortranarray(np.eye(8)), bc.TileSpec(3))
    assert np.allclose(w, np.ones(8), atol=1e-14)
    assert np.linalg.norm(v.conj().T @ v - np.eye(8)) <= 1e-13


def test_deterministic_and_sign_convention(meshes):
    """test_solvers.py:273-283: two runs bit-identical; anchors real positive."""
    a = G["rand12_f64__a"]
    w1, v1, _ = bc.eigh_hermitian(meshes(2), a, bc.TileSpec(4))
    w2, v2, _ = bc.eigh_hermitian(meshes(2), a, bc.TileSpec(4))
    assert np.array_equal(w1, w2) and np.array_equal(v1, v2)
    for k in range(a.shape[0]):
        assert v1[np.argmax(np.abs(v1[:, k])), k] > 0
    ac = G["rand24_c128__a"]
    _, vc, _ = bc.eigh_hermitian(meshes(3), ac, bc.TileSpec(5))
    for k in range(ac.shape[0]):
        anchor = vc[np.argmax(np.abs(vc[:, k])), k]
        assert anchor.real > 0 and anchor.imag == 0


def test_tile_device_invariance(meshes):
    """test_acceptance.py:249-268 (eigen part): every (tile, devices) within
    10 n eps of the T=1, D=1 run after phase alignment."""
    a = G["sep32_f64__a"]
    n = a.shape[0]
    tol = 10 * n * np.finfo(np.float64).eps
    base_w, base_v, _ = bc.eigh_hermitian(meshes(1), a, bc.TileSpec(1))
    for t in (1, 7, 16, n):
        for d in (1, 2, 3, 4):
            w, v, _ = bc.eigh_hermitian(meshes(d), a, bc.TileSpec(t))
            assert np.max(np.abs(w - base_w)) <= tol * max(1.0, np.max(np.abs(base_w)))
            assert np.max(np.abs(O.phase_align(v, base_v) - base_v)) <= tol, (t, d)


@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.complex64, np.complex128])
@pytest.mark.parametrize("n,t,d", [(128, 16, 2), (257, 64, 3), (600, 128, 2)])
def test_random_against_oracle(meshes, dtype, n, t, d):
    """test_acceptance.py:223-241 bounds at larger orders, eigenvalues against the oracle."""
    et = bc.ElementType.from_dtype(np.dtype(dtype))
    a = O.make_matrix("random_spd", n, np.dtype(dtype), seed=13) if n <= 257 else None
    if a is None:
        rng = np.random.default_rng(n)
        b = rng.uniform(-1, 1, (n, n))
        if et.is_complex:
            b = b + 1j * rng.uniform(-1, 1, (n, n))
        a = np.asfortranarray(((b + b.conj().T) / 2).astype(dtype))  # indefinite Hermitian
    w, v, _ = bc.eigh_hermitian(meshes(d), a, bc.TileSpec(t))
    eps = _eps(dtype)
    res, orth = _quality(a, w, v)
    assert res <= 100 * n * eps and orth <= 100 * n * eps, (res, orth)
    w_or = np.linalg.eigvalsh(a.astype(np.complex128 if et.is_complex else np.float64))
    assert np.max(np.abs(w.astype(np.float64) - w_or)) <= 100 * n * eps * np.max(np.abs(w_or))


def test_diag_eigenvalues(meshes):
    """test_acceptance.py:237-241: diag(1..64) eigenvalues within 1e-10."""
    m = 64
    w, _, _ = bc.eigh_hermitian(meshes(2), np.asfortranarray(np.diag(np.arange(1.0, m + 1))), bc.TileSpec(16))
    assert np.max(np.abs(w - np.arange(1.0, m + 1))) <= 1e-10


def test_cyclic_building_block(meshes):
    """syevd on the block-cyclic layout (solvers.py:862-910): eigenvector j at
    cyclic column j; redistribute_out gives the pipeline's bits."""
    a = G["sep20_c128__a"]
    mesh = meshes(3)
    desc = bc.MatrixDescriptor(20, 20, bc.ElementType.complex128, bc.Structure.hermitian)
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(4))
    bc.write_array(mesh, dm, a)
    cyc = bc.redistribute_in(mesh, dm)
    w, vecs = bc.syevd_cyclic(mesh, cyc)
    out = bc.redistribute_out(mesh, vecs)
    v = bc.gather_array(mesh, out)
    w2, v2, _ = bc.eigh_hermitian(mesh, a, bc.TileSpec(4))
    assert np.array_equal(w, w2) and np.array_equal(v, v2)


def test_rejections(meshes):
    """test_solvers.py:286-289 (non-square) and the structure check (solvers.py:867-872)."""
    with pytest.raises(bc.DescriptorError):
        bc.eigh_hermitian(meshes(1), np.asfortranarray(np.ones((3, 2))), bc.TileSpec(1))
    mesh = meshes(1)
    desc = bc.MatrixDescriptor(4, 4, bc.ElementType.real64, bc.Structure.general)
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(2))
    with pytest.raises(bc.DescriptorError):
        bc.syevd_cyclic(mesh, bc.redistribute_in(mesh, dm))


@pytest.mark.parametrize("dtype", [np.float64, np.complex128, np.float32])
def test_paper_api_row_sharded(meshes, dtype):
    """jaxmg.syevd-style call on a row-major torch tensor:
    the caller's A is untouched, V[:, j] is the eigenvector of w[j]."""
    import torch

    a = G["sep20_c128__a"] if np.dtype(dtype).kind == "c" else G["sep32_f64__a"]
    a = a.astype(dtype)
    n = a.shape[0]
    At = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    keep = At.clone()
    w, V = bc.syevd(At, T_A=4, mesh=meshes(1), in_specs=(bc.P("x", None),))
    assert torch.equal(At, keep)
    w_ref, v_ref = O.syevd_dense(a, 4)
    eps = _eps(dtype)
    assert np.max(np.abs(w.cpu().numpy() - w_ref)) <= 10 * n * eps * np.max(np.abs(w_ref))
    assert np.max(np.abs(V.cpu().numpy() - v_ref)) <= 100 * n * eps
    assert torch.equal(bc.syevd(At, T_A=4, mesh=meshes(1), return_eigenvectors=False), w)


@pytest.mark.parametrize("n,t,d", [(1, 1, 1), (2, 2, 2), (3, 1, 3), (65, 64, 1), (129, 64, 5), (300, 256, 2),
                                   (97, 13, 8), (257, 128, 4)])
@pytest.mark.parametrize("dtype", [np.float32, np.float64, np.complex64, np.complex128])
def test_edge_shapes(meshes, n, t, d, dtype):
    """Orders that do not divide the tile, tiles wider than the 64-wide symv
    tile and the 256-reflector WY block edge, n = 1 and 2, up to 8 devices."""
    rng = np.random.default_rng(1000 * n + t)
    b = rng.uniform(-1, 1, (n, n))
    if np.dtype(dtype).kind == "c":
        b = b + 1j * rng.uniform(-1, 1, (n, n))
    a = np.asfortranarray(((b + b.conj().T) / 2).astype(dtype))
    w, v, _ = bc.eigh_hermitian(meshes(d), a, bc.TileSpec(t))
    eps = _eps(dtype)
    assert w.shape == (n,) and v.shape == (n, n) and np.all(np.diff(w) >= 0)
    res, orth = _quality(a, w, v)
    scale = max(1.0, n)
    assert res <= 100 * scale * eps and orth <= 100 * scale * eps, (res, orth)
    wide = np.complex128 if np.dtype(dtype).kind == "c" else np.float64
    w_ref = np.linalg.eigvalsh(a.astype(wide))
    assert np.max(np.abs(w.astype(np.float64) - w_ref)) <= 100 * scale * eps * max(1.0, np.max(np.abs(w_ref)))
