#!/usr/bin/env python3
"""Per-kernel time of one potrs / potri on one GPU from the CUPTI activity
trace (torch.profiler; every stream, kernels not serialised): where a
configuration's device time goes, by kernel name.

    python tools/profile_kernels.py --routine potri --dtype c128 --n 65536 --t 512 --d 8
"""
import argparse, collections, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--routine", default="potri", choices=("potrs", "potri"))
ap.add_argument("--dtype", default="c128")
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--t", type=int, default=512)
ap.add_argument("--d", type=int, default=8)
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
code, dt = {"f32": (0, torch.float32), "f64": (1, torch.float64), "c64": (2, torch.complex64),
            "c128": (3, torch.complex128)}[a.dtype]
lib = _lib.load()
A = torch.empty(a.n, a.n, dtype=dt, device="cuda")
b = torch.ones(a.n, 1, dtype=dt, device="cuda")
mesh = bc.make_mesh(a.d)
gen = lambda: _lib.check(lib.bcmg_generate_spd(C.c_void_p(torch.cuda.current_stream().cuda_stream), code, a.n, 0, a.n,  # noqa
                                                C.c_void_p(A.data_ptr()), a.n, 21, float(a.n)))
run = (lambda: bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)) if a.routine == "potrs" else \
      (lambda: bc.potri(A, T_A=a.t, mesh=mesh, overwrite_a=True))
gen()
run()  # warm-up (workspace, tensor maps, module load)
gen()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
wall = e0.elapsed_time(e1)
agg = collections.defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        name = ev.name.split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ev.device_time_total / 1e3 if hasattr(ev, "device_time_total") else ev.cuda_time_total / 1e3
cf = 4.0 if dt.is_complex else 1.0
flops = cf * (a.n ** 3 / 3 if a.routine == "potrs" else a.n ** 3)
rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
print(json.dumps({"routine": a.routine, "dtype": a.dtype, "n": a.n, "t": a.t, "d": a.d, "ms": wall,
                  "tflops": flops / (wall * 1e-3) / 1e12,
                  "kernels": [{"name": k, "launches": v[0], "ms": round(v[1], 3)} for k, v in rows[:a.top]]}), flush=True)
mesh.close()
