#!/usr/bin/env python3
"""Time the diagonal-block factor alone: bcmg_potrf on a single tile (n = T),
device-resident, idle GPU, CUDA events, median of 20 after warm-up.

    python tools/diag_bench.py
"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import _lib  # noqa: E402

lib = _lib.load()
mesh = bc.make_mesh(1)
st = torch.cuda.current_stream()
for name, code, dt in (("f64", 1, torch.float64), ("f32", 0, torch.float32), ("c64", 2, torch.complex64),
                       ("c128", 3, torch.complex128)):
    for t in [int(v) for v in os.environ.get("DIAG_TILES", "256,512,1024,2048").split(",")]:
        A0 = torch.empty(t, t, dtype=dt, device="cuda")
        _lib.check(lib.bcmg_generate_spd(C.c_void_p(st.cuda_stream), code, t, 0, t, C.c_void_p(A0.data_ptr()), t, 3,
                                         float(t)))
        A = A0.clone()
        ptrs = (C.c_void_p * 1)(A.data_ptr())
        info = C.c_int(0)
        times = []
        for i in range(25):
            A.copy_(A0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.bcmg_potrf(mesh.session, C.c_void_p(st.cuda_stream), code, t, t, 1, ptrs, C.byref(info)))
            e1.record()
            torch.cuda.synchronize()
            if i >= 5:
                times.append(e0.elapsed_time(e1))
        times.sort()
        cf = 4 if dt.is_complex else 1
        ms = times[len(times) // 2]
        print(json.dumps({"dtype": name, "t": t, "ms_median": ms, "ms_min": times[0],
                          "gflops_potrf": cf * t ** 3 / 3 / (ms * 1e-3) / 1e9}), flush=True)
mesh.close()

if len(sys.argv) > 1 and sys.argv[1] == "--trace":  # per-kernel CUPTI trace of one f64 / c64 1024 tile
    mesh = bc.make_mesh(1)
    for name, code, dt in (("f64", 1, torch.float64), ("c64", 2, torch.complex64)):
      for t in [int(v) for v in os.environ.get("TRACE_TILES", "1024").split(",")]:
          A = torch.empty(t, t, dtype=dt, device="cuda")
          _lib.check(lib.bcmg_generate_spd(C.c_void_p(st.cuda_stream), code, t, 0, t, C.c_void_p(A.data_ptr()), t, 3,
                                           float(t)))
          A0 = A.clone()
          ptrs = (C.c_void_p * 1)(A.data_ptr())
          info = C.c_int(0)
          _lib.check(lib.bcmg_potrf(mesh.session, C.c_void_p(st.cuda_stream), code, t, t, 1, ptrs, C.byref(info)))
          A.copy_(A0)
          torch.cuda.synchronize()
          with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
              _lib.check(lib.bcmg_potrf(mesh.session, C.c_void_p(st.cuda_stream), code, t, t, 1, ptrs, C.byref(info)))
              torch.cuda.synchronize()
          evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                       key=lambda e: e.time_range.start)
          t0 = evs[0].time_range.start
          for e in evs:
              print(json.dumps({"dtype": name, "kernel": e.name.split("(")[0][:80], "start_us": e.time_range.start - t0,
                                "dur_us": e.time_range.end - e.time_range.start}))
    mesh.close()
