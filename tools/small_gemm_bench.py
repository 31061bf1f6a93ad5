"""Times the non-trailing GEMM shapes of potrf/potrs (diag recursion, substitution)
through bcmg_gemm for every dtype.  Probe tool, not the bench."""
import ctypes as C, sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_14466_b200 import _lib
lib = _lib.load()
TD = {0: torch.float32, 1: torch.float64, 2: torch.complex64, 3: torch.complex128}
# (name, M, N, K, op_a, op_b): op 0 = N, 1 = C (bcmg_gemm semantics: C = alpha op(A) op(B) + beta C)
SHAPES = [
    ("fwd_diag", 1024, 16, 1024, 0, 0),
    ("fwd_off", 7168, 16, 1024, 0, 0),
    ("bwd_diag", 1024, 16, 1024, 1, 0),
    ("rec_l21", 512, 512, 512, 0, 1),
    ("rec_x21", 512, 512, 512, 0, 0),
    ("rec_l21_s", 64, 64, 64, 0, 1),
    ("rec_x21_256", 256, 256, 256, 0, 0),
]
dts = [int(a) for a in sys.argv[1:]] or [0, 1, 2, 3]
for dt in dts:
    for (name, m, n, k, oa, ob) in SHAPES:
        t = TD[dt]
        A = torch.rand(max(m, k) * max(m, k) * 2, dtype=torch.float64, device="cuda").to(t)
        B = torch.rand(max(n, k) * max(n, k) * 2, dtype=torch.float64, device="cuda").to(t)
        Cm = torch.rand(m * n, dtype=torch.float64, device="cuda").to(t)
        lda = m if oa == 0 else k
        ldb = k if ob == 0 else n
        f = lambda: lib.bcmg_gemm(None, dt, m, n, k, -1.0, C.c_void_p(A.data_ptr()), lda, oa,
                                  C.c_void_p(B.data_ptr()), ldb, ob, 1.0, C.c_void_p(Cm.data_ptr()), m)
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps): f()
        e1.record(); e1.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        cf = 4 if dt >= 2 else 1
        print(json.dumps({"dt": dt, "shape": name, "m": m, "n": n, "k": k, "us": round(us, 1),
                          "tflops": round(cf * 2 * m * n * k / us / 1e6, 2)}), flush=True)
