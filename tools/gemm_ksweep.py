"""Per-item overhead of the TMA DMMA GEMM: fixed M=N=16384, K swept."""
import ctypes as C, sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_14466_b200 import _lib
lib = _lib.load()
m = n = 16384
for k in [256, 512, 1024, 2048, 4096]:
    A = torch.rand(k, m, dtype=torch.float64, device="cuda")
    B = torch.rand(k, n, dtype=torch.float64, device="cuda")
    Cm = torch.rand(n, m, dtype=torch.float64, device="cuda")
    f = lambda: lib.bcmg_gemm(None, 1, m, n, k, -1.0, C.c_void_p(A.data_ptr()), m, 0, C.c_void_p(B.data_ptr()), n, 1, 1.0, C.c_void_p(Cm.data_ptr()), m)
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); reps = 4
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"tile": os.environ.get("BCMG_TRAIL_TILE", "2"), "k": k, "ms": round(ms, 3), "tflops": round(2 * m * n * k / ms / 1e9, 2)}))
