"""DMMA GEMM throughput through bcmg_gemm (f64, A op N, B op C = the trailing-update shape)."""
import ctypes as C, sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_14466_b200 import _lib
lib = _lib.load()
for (m, n, k) in [(16384, 16384, 1024), (16384, 16384, 4096), (32768, 8192, 1024), (8192, 8192, 8192)]:
    A = torch.rand(k, m, dtype=torch.float64, device="cuda")   # col-major m x k
    B = torch.rand(k, n, dtype=torch.float64, device="cuda")   # col-major n x k (op C)
    Cm = torch.rand(n, m, dtype=torch.float64, device="cuda")
    f = lambda: lib.bcmg_gemm(None, 1, m, n, k, -1.0, C.c_void_p(A.data_ptr()), m, 0, C.c_void_p(B.data_ptr()), n, 1, 1.0, C.c_void_p(Cm.data_ptr()), m)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); reps = 5
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"m": m, "n": n, "k": k, "ms": round(ms, 3), "tflops": round(2 * m * n * k / ms / 1e9, 2)}))
