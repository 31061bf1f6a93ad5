#!/usr/bin/env python3
"""The substitution phase alone (bcmg_potrs_factored after one bcmg_potrf):
CUDA-event time and a CUPTI per-kernel split, against the HBM floor of reading
the factor twice (forward + backward sweeps).

    python tools/potrs_phase.py --dtype f32 --n 65536 --t 1024 --nrhs 1 --d 8
"""
import argparse, collections, ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="f32")
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--d", type=int, default=8)
a = ap.parse_args()
code, dt = {"f32": (0, torch.float32), "f64": (1, torch.float64), "c64": (2, torch.complex64),
            "c128": (3, torch.complex128)}[a.dtype]
lib = _lib.load()
st = torch.cuda.current_stream()
mesh = bc.make_mesh(a.d)
counts = [len(range(d * a.t, a.n, a.d * a.t)) * a.t for d in range(a.d)]  # columns per device (n % (d t) == 0 here)
counts = [sum(min(a.t, a.n - c0) for c0 in range(d * a.t, a.n, a.d * a.t)) for d in range(a.d)]
shards = [torch.empty(cnt, a.n, dtype=dt, device="cuda") for cnt in counts]  # column-major n x cnt
ptrs = (C.c_void_p * a.d)(*[s.data_ptr() for s in shards])
# cyclic shards of the SPD generator's matrix: generate the contiguous rows then redistribute in place
A = torch.empty(a.n, a.n, dtype=dt, device="cuda")
_lib.check(lib.bcmg_generate_spd(C.c_void_p(st.cuda_stream), code, a.n, 0, a.n, C.c_void_p(A.data_ptr()), a.n, 21,
                                 float(a.n)))
c0 = 0
for d in range(a.d):
    shards[d].copy_(A[c0:c0 + counts[d]])
    c0 += counts[d]
del A
_lib.check(lib.bcmg_redistribute(mesh.session, C.c_void_p(st.cuda_stream), code, a.n, a.n, a.t, a.d, ptrs, 0))
info = C.c_int(0)
_lib.check(lib.bcmg_potrf(mesh.session, C.c_void_p(st.cuda_stream), code, a.n, a.t, a.d, ptrs, C.byref(info)))
assert info.value == 0
x = torch.ones(a.nrhs, a.n, dtype=dt, device="cuda")  # column-major n x nrhs
x0 = x.clone()
def run():
    _lib.check(lib.bcmg_potrs_factored(mesh.session, C.c_void_p(st.cuda_stream), code, a.n, a.nrhs, a.t, a.d, ptrs,
                                       C.c_void_p(x.data_ptr()), a.n))
run()
times = []
for _ in range(3):
    x.copy_(x0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
x.copy_(x0)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = agg[e.name.split("(")[0][:70]]
        k[0] += 1
        k[1] += (e.time_range.end - e.time_range.start) / 1e3
esz = torch.empty(0, dtype=dt).element_size()
floor_bytes = 2 * (a.n * a.n / 2) * esz
print(json.dumps({"dtype": a.dtype, "n": a.n, "t": a.t, "nrhs": a.nrhs, "d": a.d, "ms": min(times),
                  "factor_read_floor_ms": floor_bytes / 6457e9 * 1e3,
                  "kernels": sorted([[k, v[0], round(v[1], 3)] for k, v in agg.items()], key=lambda r: -r[2])[:10]}))
mesh.close()
