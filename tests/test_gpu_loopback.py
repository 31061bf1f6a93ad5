"""The multi-process drivers on ONE GPU: `world` sessions of this process act
as the ranks (one host thread each, own streams), joined by the in-process
loopback transport (bcmg_loopback_id) instead of NCCL.  This runs the exact
world > 1 code of solver.cu -- cross-process redistribution (pack / grouped
send+recv / unpack), per-step panel broadcasts, substitution hand-offs, potri's
W-tile broadcasts and block gathers, the info all-reduce -- on the device, and
the result must be bit-identical to the single-process run (the reference's
bit-exactness across device counts, test_solvers.py:172-179)."""

import ctypes as C
import gc
import threading

import numpy as np
import pytest


bc = pytest.importorskip("paper_2601_14466_b200")
from paper_2601_14466_b200 import _lib  # noqa: E402
from oracle import bcmg_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
CODES = {np.float32: 0, np.float64: 1, np.complex64: 2, np.complex128: 3}


def _run_ranks(world, body):
    """body(rank, session, stream) on `world` threads with loopback sessions."""
    import torch

    lib = _lib.load()
    idbuf = C.create_string_buffer(128)
    _lib.check(lib.bcmg_loopback_id(idbuf))
    sessions = []
    for r in range(world):
        s = C.c_void_p()
        _lib.check(lib.bcmg_open(torch.cuda.current_device(), r, world, idbuf.raw, C.byref(s)))
        sessions.append(s)
    results, errors = [None] * world, []

    def work(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                results[r] = body(r, sessions[r], st)
            st.synchronize()
        except Exception as exc:  # noqa: BLE001
            errors.append((r, exc))

    # Nothing may synchronise the whole context while ranks are parked on peer
    # flags (they share one GPU here): no garbage collection of other sessions
    # (their destructors synchronise the device) during the multi-rank section.
    gc.collect()
    torch.cuda.synchronize()
    gc.disable()
    try:
        threads = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
    finally:
        gc.enable()
    assert not any(t.is_alive() for t in threads), "a rank hung"
    torch.cuda.synchronize()
    for s in sessions:
        _lib.check(lib.bcmg_close(s))
    assert not errors, errors
    return results


def _local_shards(a, n, t, ndev, world, r, device):
    """This rank's logical devices' shards (contiguous layout), back to back."""
    import torch

    counts = [0] * ndev
    arr = (C.c_int64 * ndev)()
    _lib.check(_lib.load().bcmg_column_counts(n, t, ndev, arr))
    counts = list(arr)
    nloc = ndev // world
    c0 = sum(counts[: r * nloc])
    c1 = c0 + sum(counts[r * nloc:(r + 1) * nloc])
    block = torch.from_numpy(np.ascontiguousarray(a[:, c0:c1].T)).to(device)  # column-major n x (c1 - c0)
    ptrs, off = [], 0
    for d in range(r * nloc, (r + 1) * nloc):
        ptrs.append(block.data_ptr() + off * n * block.element_size())
        off += counts[d]
    return block, _lib.ptr_array(ptrs), (c0, c1)


def _potrs_ranks(a, b, n, t, ndev, world, dtype):
    """One multi-rank potrs; device inputs are prepared before the rank threads
    start, so nothing in the threads allocates while a peer waits on a flag."""
    import torch

    lib = _lib.load()
    inputs = []
    for r in range(world):
        block, ptrs, _ = _local_shards(a, n, t, ndev, world, r, "cuda")
        x = torch.from_numpy(np.ascontiguousarray(b.T)).to("cuda")  # column-major replica
        inputs.append((block, ptrs, x))
    torch.cuda.synchronize()

    def body(r, sess, st):
        _, ptrs, x = inputs[r]
        info = C.c_int(0)
        _lib.check(lib.bcmg_potrs(sess, C.c_void_p(st.cuda_stream), CODES[dtype], n, b.shape[1], t, ndev, ptrs,
                                  C.c_void_p(x.data_ptr()), n, 0, C.byref(info)))
        assert info.value == 0
        return r

    _run_ranks(world, body)
    torch.cuda.synchronize()
    return [inputs[r][2].cpu().numpy().T for r in range(world)]


@pytest.mark.parametrize("dtype,n,t,ndev,world", [
    (np.float64, 300, 32, 2, 2), (np.float64, 512, 64, 4, 2), (np.complex128, 260, 24, 4, 2),
    (np.float32, 384, 64, 4, 4), (np.complex64, 200, 40, 2, 2), (np.float64, 2048, 256, 4, 2),
    # T_A = 128: the TMA-epilogue kernel (f32) and the two-column 2-SM pair items with
    # owned columns D apart (c64, one device per rank)
    (np.float32, 2048, 128, 2, 2), (np.float32, 2048, 128, 4, 2), (np.complex64, 2048, 128, 2, 2),
    (np.complex64, 2560, 128, 4, 4),
])
@pytest.mark.parametrize("paths", ["ce+p2p", "nccl+staged"])
def test_loopback_potrs_matches_single_process(dtype, n, t, ndev, world, paths, monkeypatch):
    """The single-process bits, with either set of cross-process paths:
    ce+p2p      -- the defaults: copy-engine panel pushes into peer-mapped panel
                   buffers with stream-memory-operation flags, and the in-place
                   peer rotation of the redistribution;
    nccl+staged -- the transport's broadcast and the pack / send+recv / unpack
                   redistribution (the fallbacks)."""
    a = O.make_matrix("random_spd", n, dtype, 11)
    b = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 3)).astype(dtype))
    mesh = bc.make_mesh(ndev)
    base, _ = bc.solve_positive_definite(mesh, a, b, bc.TileSpec(t))
    mesh.close()
    monkeypatch.delenv("BCMG_P2P", raising=False)
    monkeypatch.setenv("BCMG_PANEL_BCAST", "ce" if paths == "ce+p2p" else "nccl")
    monkeypatch.setenv("BCMG_REDIST_NCCL", "0" if paths == "ce+p2p" else "1")
    xs = _potrs_ranks(a, b, n, t, ndev, world, dtype)
    for x in xs:
        assert np.array_equal(x, base), "solution differs from the single-process bits"
    assert O.solve_residual(a, xs[0], b) <= 100 * n * O.eps_of(dtype)


@pytest.mark.parametrize("dtype,n,t,ndev,world", [
    (np.float64, 256, 32, 2, 2), (np.complex128, 192, 24, 4, 2), (np.float64, 1024, 128, 4, 4),
])
@pytest.mark.parametrize("redist", ["p2p", "staged"])
def test_loopback_potri_matches_single_process(dtype, n, t, ndev, world, redist, monkeypatch):
    monkeypatch.setenv("BCMG_REDIST_NCCL", "0" if redist == "p2p" else "1")
    lib = _lib.load()
    a = O.make_matrix("random_spd", n, dtype, 12)
    base, _ = bc.invert_positive_definite(bc.make_mesh(ndev), a, bc.TileSpec(t))

    def body(r, sess, st):
        block, ptrs, cols = _local_shards(a, n, t, ndev, world, r, "cuda")
        info = C.c_int(0)
        _lib.check(lib.bcmg_potri(sess, C.c_void_p(st.cuda_stream), CODES[dtype], n, t, ndev, ptrs, 0,
                                  C.byref(info)))
        assert info.value == 0
        st.synchronize()
        return cols, block.cpu().numpy().T

    parts = _run_ranks(world, body)
    inv = np.zeros((n, n), dtype=dtype, order="F")
    for (c0, c1), blk in parts:
        inv[:, c0:c1] = blk
    assert np.array_equal(inv, base)


def test_loopback_not_positive_definite_info_on_every_rank():
    """The pivot found on one rank reaches every rank (the info all-reduce)."""
    import torch

    lib = _lib.load()
    n, t, ndev, world = 96, 16, 2, 2
    a = np.asfortranarray(np.diag(np.arange(1.0, n + 1)))
    a[70, 70] = -1.0  # tile 4 -> logical device 0 -> rank 0; the pivot is global column 71

    def body(r, sess, st):
        block, ptrs, _ = _local_shards(a, n, t, ndev, world, r, "cuda")
        x = torch.ones(n, dtype=torch.float64, device="cuda")
        info = C.c_int(0)
        rc = lib.bcmg_potrs(sess, C.c_void_p(st.cuda_stream), 1, n, 1, t, ndev, ptrs, C.c_void_p(x.data_ptr()), n,
                            0, C.byref(info))
        return rc, info.value

    for rc, info in _run_ranks(world, body):
        assert rc == _lib.BCMG_ERR_NOT_POSITIVE_DEFINITE and info == 71


@pytest.mark.parametrize("redist", ["p2p", "staged"])
@pytest.mark.parametrize("dtype,n_rows,n,t,ndev,world", [
    (np.float64, 40, 64, 8, 4, 2), (np.float64, 33, 48, 5, 4, 4), (np.complex64, 17, 30, 3, 2, 2),
    (np.float32, 64, 96, 7, 6, 3), (np.complex128, 128, 512, 64, 8, 4), (np.float64, 1024, 4096, 256, 8, 2),
])
def test_loopback_redistribution_bit_exact(dtype, n_rows, n, t, ndev, world, redist, monkeypatch):
    """Cross-process redistribution, both paths: the in-place rotation over
    peer-mapped shards (each rank rotates its lane range of every cycle) and the
    staged NCCL fallback -- bit-exact dealing (oracle deal_columns, the
    reference's execute_plan result) and an exact round trip."""
    import torch

    monkeypatch.setenv("BCMG_REDIST_NCCL", "0" if redist == "p2p" else "1")
    from conftest import numbered_columns

    lib = _lib.load()
    a = numbered_columns(n_rows, n, dtype)
    want = O.deal_columns(a, t, ndev)
    arr = (C.c_int64 * ndev)()
    _lib.check(lib.bcmg_column_counts(n, t, ndev, arr))
    counts = list(arr)
    nloc = ndev // world
    blocks, ptrs = [], []
    for r in range(world):
        c0 = sum(counts[: r * nloc])
        c1 = c0 + sum(counts[r * nloc:(r + 1) * nloc])
        blk = torch.from_numpy(np.ascontiguousarray(a[:, c0:c1].T)).to("cuda")
        p, off = [], 0
        for d in range(r * nloc, (r + 1) * nloc):
            p.append(blk.data_ptr() + off * n_rows * blk.element_size())
            off += counts[d]
        blocks.append((blk, c0, c1))
        ptrs.append(_lib.ptr_array(p))
    torch.cuda.synchronize()

    def body(r, sess, st):
        for direction in (0, 1):
            _lib.check(lib.bcmg_redistribute(sess, C.c_void_p(st.cuda_stream), CODES[dtype], n_rows, n, t, ndev,
                                             ptrs[r], direction))
            st.synchronize()
            if direction == 0:
                blk, c0, c1 = blocks[r]
                got = blk.cpu().numpy().T
                assert np.array_equal(got, want[:, c0:c1]), f"rank {r}: dealt columns differ"
        return r

    _run_ranks(world, body)
    for blk, c0, c1 in blocks:
        assert np.array_equal(blk.cpu().numpy().T, a[:, c0:c1]), "round trip differs"


@pytest.mark.parametrize("dtype,n,t,ndev,world", [
    (np.float64, 96, 8, 2, 2), (np.complex128, 80, 8, 4, 2), (np.float32, 64, 16, 4, 4), (np.complex64, 72, 12, 2, 2),
])
def test_loopback_syevd_matches_single_process(dtype, n, t, ndev, world):
    """syevd across processes (the matrix gathered on rank 0, solved there,
    eigenvector shards and eigenvalues sent back): the single-process bits on
    every rank (reference eigh_hermitian, solvers.py:1019-1043)."""
    import torch

    lib = _lib.load()
    a = O.make_matrix("random_spd", n, dtype, 5)
    w0, v0, _ = bc.eigh_hermitian(bc.make_mesh(ndev), a, bc.TileSpec(t))
    real = torch.float32 if dtype in (np.float32, np.complex64) else torch.float64
    inputs = []
    for r in range(world):
        block, ptrs, cols = _local_shards(a, n, t, ndev, world, r, "cuda")
        inputs.append((block, ptrs, cols, torch.empty(n, dtype=real, device="cuda")))
    torch.cuda.synchronize()

    def body(r, sess, st):
        _, ptrs, _, w = inputs[r]
        info = C.c_int(0)
        _lib.check(lib.bcmg_syevd(sess, C.c_void_p(st.cuda_stream), CODES[dtype], n, t, ndev, ptrs,
                                  C.c_void_p(w.data_ptr()), 0, C.byref(info)))
        assert info.value == 0
        return r

    _run_ranks(world, body)
    v = np.zeros((n, n), dtype=dtype, order="F")
    for block, _, (c0, c1), w in inputs:
        assert np.array_equal(w.cpu().numpy(), w0), "eigenvalues differ from the single-process bits"
        v[:, c0:c1] = block.cpu().numpy().T
    assert np.array_equal(v, v0), "eigenvectors differ from the single-process bits"
