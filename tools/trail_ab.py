#!/usr/bin/env python3
"""A/B timing of the f64 trailing-update kernel variants (one process per
variant: the selection is read once).  Prints one JSON line: potrs f64 N, T=1024
on one GPU, the trailing-update launches' CUDA-event time and TF/s, the step time.

    BCMG_TRAIL_VARIANT=1 python tools/trail_ab.py --n 65536
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
lib = _lib.load()
A = torch.empty(a.n, a.n, dtype=torch.float64, device="cuda")
b = torch.ones(a.n, 64, dtype=torch.float64, device="cuda")
mesh = bc.make_mesh(1)
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
gen = lambda: _lib.check(lib.bcmg_generate_spd(st(), 1, a.n, 0, a.n, C.c_void_p(A.data_ptr()), a.n, 1, float(a.n)))  # noqa
gen()
bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)
best = None
for _ in range(a.reps):
    gen()
    torch.cuda.synchronize()
    lib.bcmg_set_profiling(mesh.session, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)
    e1.record()
    torch.cuda.synchronize()
    lib.bcmg_set_profiling(mesh.session, 0)
    s = (C.c_double * 4)()
    _lib.check(lib.bcmg_kernel_stats(mesh.session, 0, s))
    r = {"n": a.n, "t": a.t, "variant": os.environ.get("BCMG_TRAIL_VARIANT", "0"), "step_ms": e0.elapsed_time(e1),
         "trail_ms": s[1], "trail_tflops": s[2] / (s[1] * 1e-3) / 1e12,
         "step_tflops": (a.n ** 3 / 3 + 2 * a.n ** 2 * 64) / (e0.elapsed_time(e1) * 1e-3) / 1e12}
    best = r if best is None or r["step_ms"] < best["step_ms"] else best
print(json.dumps(best), flush=True)
