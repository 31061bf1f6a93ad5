#!/usr/bin/env python3
"""Per-kernel-kind time of one potrs (CUDA events around each launch on its own
stream; kinds: trailing update, panel solve, diagonal factor) for a dtype / N /
T_A on one GPU -- where a configuration's time goes.

    python tools/kernel_split.py --dtype f32 --n 65536 --t 1024
"""
import argparse, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f32")
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--t", type=int, default=1024)
a = ap.parse_args()
code, dt = {"f32": (0, torch.float32), "f64": (1, torch.float64), "c64": (2, torch.complex64),
            "c128": (3, torch.complex128)}[a.dtype]
lib = _lib.load()
A = torch.empty(a.n, a.n, dtype=dt, device="cuda")
b = torch.ones(a.n, 1, dtype=dt, device="cuda")
mesh = bc.make_mesh(1)
gen = lambda: _lib.check(lib.bcmg_generate_spd(C.c_void_p(torch.cuda.current_stream().cuda_stream), code, a.n, 0, a.n,  # noqa
                                                C.c_void_p(A.data_ptr()), a.n, 21, float(a.n)))
gen()
bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)
gen()
torch.cuda.synchronize()
lib.bcmg_set_profiling(mesh.session, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)
e1.record()
torch.cuda.synchronize()
cf = 4.0 if dt.is_complex else 1.0
out = {"dtype": a.dtype, "n": a.n, "t": a.t, "step_ms": e0.elapsed_time(e1),
       "step_tflops": cf * (a.n ** 3 / 3 + 2 * a.n ** 2) / (e0.elapsed_time(e1) * 1e-3) / 1e12}
s = (C.c_double * 4)()
for kind, name in ((0, "trailing_update"), (1, "panel_solve"), (2, "diag_factor")):
    _lib.check(lib.bcmg_kernel_stats(mesh.session, kind, s))
    out[name] = {"launches": s[0], "ms": s[1], "tflops": s[2] / (s[1] * 1e-3) / 1e12 if s[1] else None}
print(json.dumps(out), flush=True)
