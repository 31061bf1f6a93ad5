"""Latency of the diagonal-tile factor (leaf and recursion) via bcmg_potrf on one tile."""
import ctypes as C, os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc
from paper_2601_14466_b200 import _lib
lib = _lib.load()
mesh = bc.make_mesh(1)
for n in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else "8,64,128,256,512,1024".split(","))]:
    A0 = torch.rand(n, n, dtype=torch.float64, device="cuda")
    A0 = A0 + A0.t() + n * torch.eye(n, dtype=torch.float64, device="cuda")
    A = A0.clone()
    ptrs = _lib.ptr_array([A.data_ptr()])
    info = C.c_int()
    st = mesh.stream_handle()
    for _ in range(3):
        A.copy_(A0); lib.bcmg_potrf(mesh.session, st, 1, n, n, 1, ptrs, C.byref(info))
    torch.cuda.synchronize()
    lib.bcmg_set_profiling(mesh.session, 1)
    reps = 50
    t0 = time.perf_counter()
    for _ in range(reps):
        A.copy_(A0); lib.bcmg_potrf(mesh.session, st, 1, n, n, 1, ptrs, C.byref(info))
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e3
    s = (C.c_double * 4)()
    lib.bcmg_kernel_stats(mesh.session, 2, s)
    lib.bcmg_set_profiling(mesh.session, 0)
    print(json.dumps({"n": n, "diag_ms_avg": round(s[1] / max(s[0], 1), 4), "wall_ms_per_call": round(wall, 4), "info": info.value}))
