#!/usr/bin/env python3
"""CUPTI timeline of one potrs on one GPU (torch.profiler, every stream): the
bulk trailing-update launches, the gaps between them (time the GPU spends
on the critical path alone) and which kernels run inside those gaps.

    python tools/timeline.py --dtype f64 --n 32768 --t 1024
"""
import argparse, collections, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f64")
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--d", type=int, default=1)
a = ap.parse_args()
code, dt = {"f32": (0, torch.float32), "f64": (1, torch.float64), "c64": (2, torch.complex64),
            "c128": (3, torch.complex128)}[a.dtype]
lib = _lib.load()
A = torch.empty(a.n, a.n, dtype=dt, device="cuda")
b = torch.ones(a.n, 16, dtype=dt, device="cuda")
mesh = bc.make_mesh(a.d)
gen = lambda: _lib.check(lib.bcmg_generate_spd(C.c_void_p(torch.cuda.current_stream().cuda_stream), code, a.n, 0, a.n,  # noqa
                                                C.c_void_p(A.data_ptr()), a.n, 21, float(a.n)))
gen()
bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)
gen()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    bc.potrs(A, b, T_A=a.t, mesh=mesh, overwrite_a=True)
    torch.cuda.synchronize()
evs = sorted([(e.time_range.start, e.time_range.end, e.name.split("(")[0]) for e in prof.events()
              if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda x: x[0])
t0, t1 = evs[0][0], max(e[1] for e in evs)
bulk = [e for e in evs if "trail" in e[2]]
# union of bulk-kernel busy intervals
busy, cur = [], None
for s, e, _ in bulk:
    if cur and s <= cur[1]:
        cur[1] = max(cur[1], e)
    else:
        if cur:
            busy.append(cur)
        cur = [s, e]
if cur:
    busy.append(cur)
gaps = [(busy[i][1], busy[i + 1][0]) for i in range(len(busy) - 1) if busy[i + 1][0] > busy[i][1]]
gaps = [(t0, busy[0][0])] + gaps + [(busy[-1][1], t1)]
in_gaps = collections.defaultdict(float)
for gs, ge in gaps:
    for s, e, n in evs:
        ov = min(e, ge) - max(s, gs)
        if ov > 0:
            in_gaps[n] += ov
gap_total = sum(ge - gs for gs, ge in gaps)
print(json.dumps({"dtype": a.dtype, "n": a.n, "t": a.t, "d": a.d, "total_us": t1 - t0,
                  "bulk_busy_us": sum(e - s for s, e in busy), "gap_us": gap_total,
                  "first_gap_us": gaps[0][1] - gaps[0][0], "last_gap_us": gaps[-1][1] - gaps[-1][0],
                  "largest_gaps_us": sorted([round(ge - gs, 1) for gs, ge in gaps], reverse=True)[:12],
                  "kernels_in_gaps_us": dict(sorted(((k[:70], round(v, 1)) for k, v in in_gaps.items()),
                                                    key=lambda kv: -kv[1])[:12])}), flush=True)
mesh.close()
