"""CPU, world_size 2 (gloo): the multi-process logic of the native drivers.

`bcmg_schedule` returns exactly the per-process operation sequence the CUDA
drivers execute (solver.cu potrf/potrs/potri_schedule).  Here each rank
executes its own sequence with numpy on its logical devices' shards and real
`torch.distributed` broadcasts (gloo) in place of NCCL, and the result must
equal the oracle: this checks tile ownership, broadcast roots / sizes / order
(collectives must match across ranks or the run deadlocks), the update
ranges (no tile missed or updated twice) and the substitution hand-offs."""

import ctypes as C
import os
import socket

import numpy as np
import pytest

bc = pytest.importorskip("paper_2601_14466_b200")
from paper_2601_14466_b200 import _lib  # noqa: E402

from oracle import bcmg_oracle as O  # noqa: E402

S_FACTOR, S_BCAST, S_UPDATE, S_COPYBACK, S_STEP_END, S_FWD, S_BWD, S_SHARE = range(1, 9)
S_WFINAL, S_TILE_BCAST, S_WACC, S_PGEMM, S_PGATHER = range(9, 14)


def schedule(routine, n, t, ndev, world, rank, nrhs=1):
    lib = _lib.load()
    cnt = C.c_int64()
    _lib.check(lib.bcmg_schedule(routine, n, t, ndev, world, rank, nrhs, None, 0, C.byref(cnt)))
    buf = np.zeros((max(cnt.value, 1), 7), dtype=np.int64)
    _lib.check(lib.bcmg_schedule(routine, n, t, ndev, world, rank, nrhs, buf.ctypes.data_as(_lib._i64p),
                                 cnt.value, C.byref(cnt)))
    return [tuple(int(v) for v in row) for row in buf[: cnt.value]]


@pytest.mark.parametrize("n,t,ndev,world", [(96, 8, 2, 2), (100, 7, 4, 2), (64, 16, 4, 4), (50, 50, 2, 2)])
def test_schedule_static_properties(n, t, ndev, world):
    nt = -(-n // t)
    nloc = ndev // world
    bcasts = []
    for rank in range(world):
        ops = schedule(0, n, t, ndev, world, rank)
        owns = lambda k: rank * nloc <= k % ndev < (rank + 1) * nloc  # noqa: E731
        factored = [o[2] for o in ops if o[0] == S_FACTOR]
        assert factored == [k for k in range(nt) if owns(k)]
        updated = {}
        for kind, _, k, a, b, _, _ in ops:
            if kind == S_UPDATE:
                for m in range(a, b):
                    if owns(m):
                        updated[(k, m)] = updated.get((k, m), 0) + 1
        want = {(k, m): 1 for k in range(nt) for m in range(k + 1, nt) if owns(m) and min(n, (k + 1) * t) < n}
        assert updated == want
        # a tile is factored only after every update it needs
        pos = {("F", o[2]): i for i, o in enumerate(ops) if o[0] == S_FACTOR}
        for (k, m), _ in want.items():
            upd = max(i for i, o in enumerate(ops) if o[0] == S_UPDATE and o[2] == k and o[3] <= m < o[4])
            assert upd < pos[("F", m)]
        bcasts.append([(o[2], o[5], o[6]) for o in ops if o[0] == S_BCAST])
    assert all(b == bcasts[0] for b in bcasts), "collective sequence differs between ranks"
    if world > 1:
        assert [k for k, _, _ in bcasts[0]] == [k for k in range(nt) if min(n, (k + 1) * t) < n]
        for k, root, elems in bcasts[0]:
            s0, s1 = k * t, min(n, (k + 1) * t)
            assert root == (k % ndev) // nloc and elems == (n - s1) * (s1 - s0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, t, ndev, nrhs, dtype, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = O.make_matrix("random_spd", n, dtype, 5)
        b = np.asfortranarray(np.random.default_rng(3).standard_normal((n, nrhs)).astype(dtype))
        nt = -(-n // t)
        nloc = ndev // world
        owns = lambda k: rank * nloc <= k % ndev < (rank + 1) * nloc  # noqa: E731
        # cyclic shards of this rank's logical devices: tile k -> device k % ndev, local col (k // ndev) * t
        shards = {d: np.zeros((n, sum(min(t, n - k * t) for k in range(d, nt, ndev))), dtype=dtype, order="F")
                  for d in range(rank * nloc, (rank + 1) * nloc)}
        for k in range(nt):
            if owns(k):
                s0, s1 = k * t, min(n, (k + 1) * t)
                shards[k % ndev][:, (k // ndev) * t:(k // ndev) * t + s1 - s0] = a[:, s0:s1]

        def tile(k):
            s0, s1 = k * t, min(n, (k + 1) * t)
            loc = (k // ndev) * t
            return shards[k % ndev][:, loc:loc + s1 - s0]

        panel = [np.zeros(n * t, dtype=dtype), np.zeros(n * t, dtype=dtype)]
        xinv = {}

        def bcast(buf, elems, root):  # stands in for ncclBroadcast (bytes of `elems` elements)
            tt = torch.from_numpy(buf[:elems].view(np.float64).copy())
            dist.broadcast(tt, src=root)
            buf[:elems] = tt.numpy().view(dtype)

        for kind, _, k, lo, hi, root, elems in schedule(0, n, t, ndev, world, rank):
            s0, s1 = k * t, min(n, (k + 1) * t)
            tc = s1 - s0
            P = panel[k % 2][: (n - s1) * tc].reshape((n - s1, tc), order="F")
            if kind == S_FACTOR:
                assert owns(k)
                T_ = tile(k)
                L, info = O.cholesky_unblocked(T_[s0:s1, :])
                assert info == 0
                T_[s0:s1, :] = np.tril(L) + np.triu(T_[s0:s1, :], 1)
                X = np.linalg.inv(np.tril(L))
                xinv[k] = X
                if s1 < n:
                    P[...] = T_[s1:, :] @ X.conj().T
            elif kind == S_BCAST:
                assert elems == (n - s1) * tc
                bcast(panel[k % 2], elems, root)
            elif kind == S_UPDATE:
                for m in range(lo, hi):
                    if not owns(m):
                        continue
                    ms, me = m * t, min(n, (m + 1) * t)
                    tile(m)[ms:, :] -= P[ms - s1:, :] @ P[ms - s1:me - s1, :].conj().T
            elif kind == S_COPYBACK:
                tile(k)[s1:, :] = P
        # factor check: every local tile's lower part equals the oracle's L
        L_ref, _ = O.cholesky_unblocked(a)
        for k in range(nt):
            if owns(k):
                s0, s1 = k * t, min(n, (k + 1) * t)
                got = np.tril(tile(k), -s0)
                np.testing.assert_allclose(got, np.tril(L_ref[:, s0:s1], -s0), rtol=0,
                                           atol=1e3 * n * O.eps_of(dtype) * np.abs(L_ref).max())
        # substitution with the solution replicated on every rank
        x = np.array(b, order="F")
        xb = np.zeros(n * nrhs, dtype=dtype)
        for kind, _, k, lo, hi, root, elems in schedule(1, n, t, ndev, world, rank, nrhs):
            s0, s1 = k * t, min(n, (k + 1) * t)
            if kind == S_FWD:
                x[s0:s1] = xinv[k] @ x[s0:s1]
                if s1 < n:
                    x[s1:] -= tile(k)[s1:, :] @ x[s0:s1]
            elif kind == S_BWD:
                if s1 < n:
                    x[s0:s1] -= tile(k)[s1:, :].conj().T @ x[s1:]
                x[s0:s1] = xinv[k].conj().T @ x[s0:s1]
            elif kind == S_SHARE:
                assert elems == (hi - lo) * nrhs
                xb[:elems] = np.asfortranarray(x[lo:hi]).ravel(order="F")
                bcast(xb, elems, root)
                x[lo:hi] = xb[:elems].reshape((hi - lo, nrhs), order="F")
        xr = O.solve_unblocked(a, b)
        err = float(np.abs(x - xr).max())
        out[rank] = err

        # potri on the factored tiles (solver.cu potri_schedule): W sweep, product sweep, mirror
        def cols_below(d, s):
            return ((s - d + ndev - 1) // ndev) * t if s > d else 0

        def cols_upto(d, s):
            return cols_below(d, s) + (min(n, (s + 1) * t) - s * t if s % ndev == d else 0)

        pan = np.zeros(n * t, dtype=dtype)
        W = None
        for kind, _, s, lo, hi, root, elems in schedule(2, n, t, ndev, world, rank):
            ss, se = s * t, min(n, (s + 1) * t)
            tcs = se - ss
            if kind == S_WFINAL:
                assert owns(s)
                T_ = tile(s)
                if se < n:
                    T_[se:, :] = -(T_[se:, :] @ xinv[s])
                T_[ss:se, :] = xinv[s]
            elif kind == S_TILE_BCAST:
                assert elems == (n - ss) * tcs and root == (s % ndev) // nloc
                if owns(s):
                    pan[:elems] = np.asfortranarray(tile(s)[ss:, :]).ravel(order="F")
                bcast(pan, elems, root)
                W = pan[:elems].reshape((n - ss, tcs), order="F").copy()
            elif kind == S_WACC:
                for d in shards:
                    c = cols_below(d, s)
                    if c:
                        stage = shards[d][ss:se, :c].copy()
                        shards[d][ss:se, :c] = 0
                        shards[d][ss:, :c] += W @ stage
            elif kind == S_PGEMM:
                blocks = {}
                for d in shards:
                    c = cols_upto(d, s)
                    if c:
                        blocks[d] = W.conj().T @ shards[d][ss:, :c]
                for d, blk in blocks.items():
                    shards[d][ss:se, :blk.shape[1]] = blk
            elif kind == S_PGATHER:
                assert elems == tcs * sum(cols_upto(d, s) for d in shards)
                flat = np.concatenate([blocks[d].ravel(order="F") for d in sorted(blocks)] or
                                      [np.zeros(0, dtype=dtype)])
                assert flat.size == elems
                gathered = [None] * world
                dist.all_gather_object(gathered, {d: blocks[d] for d in blocks})  # stands in for send/recv
                if rank == root:
                    T_ = tile(s)
                    for part in gathered:
                        for d, blk in part.items():
                            for cl in range(cols_below(d, s)):
                                T_[((cl // t) * ndev + d) * t + cl % t, :] = blk[:, cl].conj()
                    B = T_[ss:se, :].copy()
                    T_[ss:se, :] = np.tril(B, -1) + np.triu(B.conj().T, 1)
                    T_[np.arange(ss, se), np.arange(tcs)] = B.diagonal().real
        inv_ref = np.linalg.inv(a)
        inv_err = 0.0
        for k in range(nt):
            if owns(k):
                s0, s1 = k * t, min(n, (k + 1) * t)
                inv_err = max(inv_err, float(np.abs(tile(k) - inv_ref[:, s0:s1]).max()))
        out[(rank, "inv")] = inv_err / float(np.abs(inv_ref).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,t,ndev,nrhs,dtype", [(96, 8, 2, 2, np.float64), (100, 7, 4, 3, np.float64),
                                                  (60, 9, 2, 1, np.complex128)])
def test_two_rank_gloo_execution_matches_oracle(n, t, ndev, nrhs, dtype):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, n, t, ndev, nrhs, dtype, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, "rank failed or deadlocked"
    for r in range(2):
        assert out[r] <= 1e3 * n * O.eps_of(dtype), out[r]
        assert out[(r, "inv")] <= 1e3 * n * O.eps_of(dtype), out[(r, "inv")]


# ----------------------------------------------------------------- cross-process redistribution


def redist_plan(n, t, ndev, world, direction):
    lib = _lib.load()
    seg, cnt = C.c_int64(), C.c_int64()
    _lib.check(lib.bcmg_redistribute_plan(n, t, ndev, world, direction, C.byref(seg), None, 0, C.byref(cnt)))
    buf = np.zeros((max(cnt.value, 1), 4), dtype=np.int64)
    _lib.check(lib.bcmg_redistribute_plan(n, t, ndev, world, direction, C.byref(seg),
                                          buf.ctypes.data_as(_lib._i64p), cnt.value, C.byref(cnt)))
    return seg.value, [tuple(int(v) for v in r) for r in buf[: cnt.value]]


def _redist_rank(rank, world, port, n_rows, n, t, ndev, chunk, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = np.asfortranarray(np.arange(n_rows * n, dtype=np.float64).reshape(n_rows, n, order="F"))
        counts = O.column_counts(n, t, ndev)
        offs = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(int)
        nloc = ndev // world
        mine = range(rank * nloc, (rank + 1) * nloc)
        shards = {d: a[:, offs[d]:offs[d] + counts[d]].copy(order="F") for d in mine}
        colb = n_rows * 8

        def run(direction):
            seg, moves = redist_plan(n, t, ndev, world, direction)
            segb = seg * colb

            def view(pos):  # byte view of segment `pos` in its (local) shard
                col = pos * seg
                d = int(np.searchsorted(offs, col, side="right") - 1)
                flat = shards[d].reshape(-1, order="F").view(np.uint8)
                return flat[(col - offs[d]) * colb:(col - offs[d]) * colb + segb]

            sends = [m for m in moves if m[2] == rank and m[3] != rank]
            locs = [m for m in moves if m[2] == rank and m[3] == rank]
            recvs = [m for m in moves if m[3] == rank and m[2] != rank]
            for o in range(0, segb, chunk):
                ln = min(chunk, segb - o)
                pack = [view(m[0])[o:o + ln].copy() for m in sends + locs]  # all reads first
                reqs = [dist.isend(torch.from_numpy(pack[j]), dst=m[3]) for j, m in enumerate(sends)]
                rbuf = [torch.empty(ln, dtype=torch.uint8) for _ in recvs]
                reqs += [dist.irecv(rbuf[j], src=m[2]) for j, m in enumerate(recvs)]
                for r in reqs:
                    r.wait()
                for j, m in enumerate(locs):
                    view(m[1])[o:o + ln] = pack[len(sends) + j]
                for j, m in enumerate(recvs):
                    view(m[1])[o:o + ln] = rbuf[j].numpy()

        def gathered():
            parts = [None] * world
            dist.all_gather_object(parts, [shards[d] for d in mine])
            return np.hstack([s for p in parts for s in p])

        run(0)
        fwd = gathered()
        run(1)
        back = gathered()
        out[rank] = (fwd.tobytes(order="F") == O.deal_columns(a, t, ndev).tobytes(order="F"),
                     back.tobytes(order="F") == a.tobytes(order="F"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_rows,n,t,ndev,chunk", [(3, 32, 4, 2, 8), (5, 40, 3, 4, 16), (2, 24, 5, 2, 1000),
                                                    (4, 64, 8, 4, 24)])
def test_two_rank_gloo_redistribution_bit_exact(n_rows, n, t, ndev, chunk):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_redist_rank, args=(r, 2, port, n_rows, n, t, ndev, chunk, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, "rank failed or deadlocked"
    assert out[0] == (True, True) and out[1] == (True, True)


def test_redistribution_plan_covers_every_moved_segment():
    for n, t, ndev, world in [(2048, 256, 2, 2), (131072, 1024, 8, 8), (100, 7, 4, 2), (10, 3, 3, 1)]:
        seg, moves = redist_plan(n, t, ndev, world, 0)
        moved = sum(len(c) for c in O.cycles_of(O.dest_positions(n, t, ndev)))
        assert len(moves) * seg == moved
        dests = [m[1] for m in moves]
        assert len(set(dests)) == len(dests) and sorted(dests) == sorted(m[0] for m in moves)
