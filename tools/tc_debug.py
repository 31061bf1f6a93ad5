import ctypes as C, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_14466_b200 import _lib
lib = _lib.load()
out = {}
for (m, n, k) in [(128, 128, 64), (256, 128, 32), (128, 128, 96), (128, 128, 128), (128, 256, 32), (384, 128, 32)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = (torch.randint(-4, 5, (k, m), generator=g, device="cuda")).float()   # col-major m x k (small ints: exact in tf32)
    B = (torch.randint(-4, 5, (k, n), generator=g, device="cuda")).float()   # col-major n x k
    Cm = torch.zeros(n, m, device="cuda")
    rc = lib.bcmg_gemm(None, 0, m, n, k, 1.0, C.c_void_p(A.data_ptr()), m, 0, C.c_void_p(B.data_ptr()), n, 1, 0.0, C.c_void_p(Cm.data_ptr()), m)
    torch.cuda.synchronize()
    out[f"A_{m}_{n}_{k}"] = A.cpu().numpy(); out[f"B_{m}_{n}_{k}"] = B.cpu().numpy(); out[f"C_{m}_{n}_{k}"] = Cm.cpu().numpy()
    ref = (A.t().double() @ B.double())  # m x n
    got = Cm.t().double()
    print(m, n, k, rc, float((got - ref).abs().max()), float(ref.abs().max()))
np.savez("gpurun_out/tc_debug.npz", **out)
