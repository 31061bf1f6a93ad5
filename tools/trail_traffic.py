#!/usr/bin/env python3
"""One config-3 potrs (f64 N=131072, T_A=1024, one GPU) for an ncu capture of
the trailing-update launches at the bench shape, plus the algorithmic bytes
and flops of every trail_tma_kernel launch in issue order (U(k): tile k+1 on
the critical stream, then B(k): tiles k+2.. on the bulk stream).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        -k regex:trail_tma --launch-skip 20 --launch-count 4 --csv \\
        python tools/trail_traffic.py --n 131072 > launches.csv
    python tools/trail_traffic.py --n 131072 --expected   # the algorithmic side (no GPU)

Algorithmic bytes of a launch = panel rows read once + the lower trapezoid of
every updated tile read and written (8 B each); flops = 2 K (rows tc - tc(tc-1)/2)
per tile.
"""

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def expected(n: int, t: int) -> list:
    nt = -(-n // t)
    out = []

    def tiles(k, ms):
        fl = by = 0.0
        for m in ms:
            rows, tc = n - m * t, min(t, n - m * t)
            trap = rows * tc - tc * (tc - 1) / 2
            fl += 2.0 * t * trap
            by += 2 * 8.0 * trap
        s1 = min(n, (k + 1) * t)
        return fl, by + 8.0 * (n - s1) * t

    for k in range(nt - 1):
        fl, by = tiles(k, [k + 1])
        out.append({"launch": len(out), "k": k, "what": "U(k) tile k+1", "flops": fl, "bytes": by})
        if k + 2 < nt:
            fl, by = tiles(k, range(k + 2, nt))
            out.append({"launch": len(out), "k": k, "what": "B(k) tiles k+2..", "flops": fl, "bytes": by})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--t", type=int, default=1024)
    ap.add_argument("--expected", action="store_true")
    a = ap.parse_args()
    if a.expected:
        print(json.dumps(expected(a.n, a.t)))
        return
    import torch

    import paper_2601_14466_b200 as bc
    from paper_2601_14466_b200 import _lib

    lib = _lib.load()
    A = torch.empty(a.n, a.n, dtype=torch.float64, device="cuda")
    _lib.check(lib.bcmg_generate_spd(C.c_void_p(torch.cuda.current_stream().cuda_stream), 1, a.n, 0, a.n,
                                     C.c_void_p(A.data_ptr()), a.n, 1, float(a.n)))
    b = torch.ones(a.n, 64, dtype=torch.float64, device="cuda")
    bc.potrs(A, b, T_A=a.t, mesh=bc.make_mesh(1), overwrite_a=True)
    torch.cuda.synchronize()
    print("trail_traffic: done", file=sys.stderr)


if __name__ == "__main__":
    main()
