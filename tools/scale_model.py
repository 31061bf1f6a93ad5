#!/usr/bin/env python3
"""Projection of the multi-GPU potrf schedule from MEASURED single-GPU kernel
times (no 2/4/8-GPU box was available to this build; the driver's SCALE run is
the measurement, this is the model it can be checked against).

    python tools/scale_model.py [--n 131072] [--t 1024] [--nrhs 64] [--json out.json]

1. On one B200, run the config-3 potrs pipeline once with per-kernel CUDA-event
   timing (bcmg_set_profiling + BCMG_PROFILE_DUMP): every lookahead update U(k)
   (tile k+1), bulk update B(k) (tiles >= k+2), diagonal factor D(k) and panel
   solve S(k) gets its own measured duration.
2. Replay the per-process schedule of solver.cu for W = 1, 2, 4, 8 processes
   as a discrete-event model:
     * process r owns tiles m = r (mod W); its share of B(k) takes the measured
       B(k) time scaled by its share of the update flops;
     * owner-first (this round's schedule, world > 1): the owner of k+1 runs
       U(k), D(k+1), S(k+1) on the whole GPU, then its share of B(k); panel
       k+1 reaches the others after the copy-engine push, (W-1) x panel bytes
       at 900 GB/s NVLink egress (datasheet) + 10 us;
     * round-1 schedule for comparison: the panel solve of k+1 queues behind
       the owner's persistent bulk grid and the NCCL broadcast behind every
       rank's bulk grid (kernels need SMs), i.e. panel k+1 is available at
       max_r(end of B(k) on r) + D + S + the broadcast.
   The substitution (potrs) and the redistribution are added from their
   measured single-GPU times / the NVLink ideal (15 GB per GPU at
   D=8).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NVLINK = 900e9  # bytes/s per direction per GPU (NVLink 5 datasheet)


def measure(n: int, t: int, nrhs: int) -> dict:
    import torch

    import paper_2601_14466_b200 as bc
    from paper_2601_14466_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    A = torch.empty(n, n, dtype=torch.float64, device=dev)
    st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    regen = lambda: _lib.check(lib.bcmg_generate_spd(st(), 1, n, 0, n, C.c_void_p(A.data_ptr()), n, 1, float(n)))  # noqa
    b = torch.ones(n, nrhs, dtype=torch.float64, device=dev)
    mesh = bc.make_mesh(1)
    regen()
    bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)  # warm-up
    regen()
    torch.cuda.synchronize()
    lib.bcmg_set_profiling(mesh.session, 1)
    bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)
    torch.cuda.synchronize()
    ph = (C.c_float * 4)()
    _lib.check(lib.bcmg_last_timings(mesh.session, ph))
    dump = tempfile.mktemp(suffix=".txt")
    os.environ["BCMG_PROFILE_DUMP"] = dump
    stats = (C.c_double * 4)()
    for kind in (0, 1, 2):
        _lib.check(lib.bcmg_kernel_stats(mesh.session, kind, stats))
    del os.environ["BCMG_PROFILE_DUMP"]
    rows = [ln.split() for ln in open(dump)]
    os.unlink(dump)
    per = {k: [(float(r[2]), float(r[3])) for r in rows if int(r[0]) == k] for k in (0, 1, 2)}
    return {"n": n, "t": t, "nrhs": nrhs, "trail": per[0], "trsm": per[1], "diag": per[2],
            "phase_ms": [float(v) for v in ph]}


def split_trail(meas: dict):
    """U(k) and B(k) in issue order: U(k) is tile k+1 only (flops 2 K (rows tc - tc(tc-1)/2))."""
    n, t = meas["n"], meas["t"]
    nt = -(-n // t)
    U, B = {}, {}
    it = iter(meas["trail"])
    for k in range(nt - 1):
        s1 = min(n, (k + 1) * t)
        tc = min(t, n - s1)
        U[k] = next(it)
        assert abs(U[k][1] - 2.0 * t * ((n - s1) * tc - tc * (tc - 1) / 2)) <= 1e-6 * U[k][1] + 1, (k, U[k])
        if k + 2 < nt:
            B[k] = next(it)
    return U, B


def tile_flops(n, t, k, m):
    ms = m * t
    rows, tc = n - ms, min(t, n - ms)
    return 2.0 * t * (rows * tc - tc * (tc - 1) / 2)


def simulate(meas: dict, W: int, owner_first: bool) -> dict:
    n, t, nrhs = meas["n"], meas["t"], meas["nrhs"]
    nt = -(-n // t)
    U, B = split_trail(meas)
    D = [d[0] * 1e-3 for d in meas["diag"]]
    S = [s[0] * 1e-3 for s in meas["trsm"]] + [0.0]
    # rank r's share of B(k): measured B(k) time x its share of the flops
    def bulk_share(k, r, _owner):
        if k not in B:
            return 0.0
        tot = B[k][1]  # tile k+1 is U(k)'s, on its owner
        mine = sum(tile_flops(n, t, k, m) for m in range(k + 2, nt) if m % W == r)
        return B[k][0] * 1e-3 * (mine / tot if tot else 0.0)

    def bcast(k):  # panel k from its owner to the W-1 others, copy engines
        if W == 1:
            return 0.0
        bytes_ = (n - min(n, (k + 1) * t)) * t * 8.0
        return (W - 1) * bytes_ / NVLINK + 10e-6

    free = [0.0] * W     # when each rank's stream is free
    ready = {0: None}
    # step 0 factor on owner 0
    free[0] = D[0] + S[0]
    ready[0] = free[0] + bcast(0)
    for k in range(nt - 1):
        o = (k + 1) % W
        if owner_first:
            for r in range(W):
                start = max(free[r], ready[k])
                if r == o:
                    f_done = start + U[k][0] * 1e-3 + D[k + 1] + S[k + 1]
                    ready[k + 1] = f_done + bcast(k + 1)
                    free[r] = f_done + bulk_share(k, r, True)
                else:
                    free[r] = start + bulk_share(k, r, False)
        else:
            # the owner's D(k+1) + S(k+1) wait for SMs until its bulk grid ends; the NCCL
            # ring broadcast (each link carries the panel once) until every rank's grid ends
            ends = []
            for r in range(W):
                start = max(free[r], ready[k])
                ends.append(start + bulk_share(k, r, False) + (U[k][0] * 1e-3 if r == o else 0.0))
            f_done = ends[o] + D[k + 1] + S[k + 1]
            ring = (n - min(n, (k + 2) * t)) * t * 8.0 / NVLINK + 10e-6 if W > 1 else 0.0
            ready[k + 1] = max(f_done, max(ends)) + ring
            for r in range(W):
                free[r] = ends[r] if r != o else f_done
    potrf_s = max(max(free), ready.get(nt - 1, 0.0) or 0.0)
    potrs_s = meas["phase_ms"][2] * 1e-3  # substitution measured on one GPU (latency-bound chain)
    moved = 2 * 8.0 * n * n * (1 - 1.0 / nt) if W > 1 else 0.0  # ~all tiles move
    redist_s = (moved / 2) * (W - 1) / W / W / NVLINK if W > 1 else 0.0
    total = potrf_s + potrs_s + redist_s
    flops = n ** 3 / 3 + 2.0 * n * n * nrhs
    return {"W": W, "schedule": "owner-first + copy-engine push" if owner_first else "round-1 (queued behind bulk)",
            "potrf_s": potrf_s, "potrs_s": potrs_s, "redistribute_s": redist_s, "total_s": total,
            "tflops": flops / total / 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--t", type=int, default=1024)
    ap.add_argument("--nrhs", type=int, default=64)
    ap.add_argument("--json", default="")
    ap.add_argument("--from-json", default="", help="re-run the model on a saved measurement")
    a = ap.parse_args()
    meas = json.load(open(a.from_json))["measurement"] if a.from_json else measure(a.n, a.t, a.nrhs)
    out = {"measurement": meas, "model": [simulate(meas, W, of) for W in (1, 2, 4, 8) for of in (True, False)]}
    for m in out["model"]:
        print(f"W={m['W']} {m['schedule']:36s} potrf {m['potrf_s']:.3f} s  total {m['total_s']:.3f} s  "
              f"{m['tflops']:.1f} TFLOP/s")
    if a.json:
        json.dump(out, open(a.json, "w"))


if __name__ == "__main__":
    main()
