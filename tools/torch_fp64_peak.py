"""cuBLAS DGEMM (torch.matmul float64) throughput on the box: the library reference point
for the FP64 roofline, measured like the driver measures bf16 (best of 10, CUDA events)."""
import torch, json
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1))
tf = 2 * n**3 / best / 1e9
# sustained: back-to-back for ~3 s
import time
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); cnt = 0; t = time.time()
while time.time() - t < 3:
    torch.matmul(a, b); cnt += 1
e1.record(); e1.synchronize()
sus = 2 * n**3 * cnt / e0.elapsed_time(e1) / 1e9
print(json.dumps({"cublas_dgemm_tflops_burst": round(tf, 2), "cublas_dgemm_tflops_sustained": round(sus, 2), "n": n}))
