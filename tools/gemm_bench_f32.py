"""tcgen05 3xTF32 GEMM throughput (f32, A op N, B op C) through bcmg_gemm."""
import ctypes as C, sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_14466_b200 import _lib
lib = _lib.load()
SHAPES = [(8192, 8192, 1024), (16384, 16384, 1024), (16384, 16384, 4096)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for (m, n, k) in SHAPES:
    A = torch.rand(k, m, dtype=torch.float32, device="cuda")
    B = torch.rand(k, n, dtype=torch.float32, device="cuda")
    Cm = torch.rand(n, m, dtype=torch.float32, device="cuda")
    f = lambda: lib.bcmg_gemm(None, 0, m, n, k, -1.0, C.c_void_p(A.data_ptr()), m, 0, C.c_void_p(B.data_ptr()), n, 1, 1.0, C.c_void_p(Cm.data_ptr()), m)
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); reps = 5
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2 * m * n * k / ms / 1e9
    print(json.dumps({"m": m, "n": n, "k": k, "ms": round(ms, 3), "eff_fp32_tflops": round(tf, 1), "tf32_tensor_tflops": round(3 * tf, 1)}))
