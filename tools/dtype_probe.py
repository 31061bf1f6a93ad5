"""Throughput of potrs / potri per dtype through the drop-in API (device-resident A)."""
import argparse, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384); ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=16); ap.add_argument("--dtypes", default="f32,f64,c64,c128")
ap.add_argument("--routine", default="potrs")
a = ap.parse_args()
n, t = a.n, a.t
mesh = bc.make_mesh(1)
for name in a.dtypes.split(","):
    dt = {"f32": torch.float32, "f64": torch.float64, "c64": torch.complex64, "c128": torch.complex128}[name]
    g = torch.Generator(device="cuda").manual_seed(1)
    R = torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
    if dt.is_complex:
        R = R + 1j * (torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1)
    A0 = ((R + R.conj().t()) * 0.5)
    A0.diagonal().add_(float(n))
    A0 = A0.to(dt); del R
    b = torch.ones(n, a.nrhs, device="cuda", dtype=dt)
    A = torch.empty_like(A0)
    cf = 4.0 if dt.is_complex else 1.0
    for rep in range(2):
        A.copy_(A0); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if a.routine == "potrs":
            x = bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True); flops = cf * (n**3 / 3 + 2 * n * n * a.nrhs)
        else:
            x = bc.potri(A, T_A=t, mesh=mesh, overwrite_a=True); flops = cf * n**3
        e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    if a.routine == "potrs":
        r = float((A0.to(torch.complex128 if dt.is_complex else torch.float64) @ x.to(torch.complex128 if dt.is_complex else torch.float64) - b).norm() / (A0.double().norm() if not dt.is_complex else A0.to(torch.complex128).norm()) / x.norm())
    else:
        I = torch.eye(n, device="cuda", dtype=torch.complex128 if dt.is_complex else torch.float64)
        r = float((A0.to(I.dtype) @ x.to(I.dtype) - I).norm() / n ** 0.5)
    print(json.dumps({"routine": a.routine, "dtype": name, "n": n, "t": t, "ms": round(ms, 2), "tflops": round(flops / ms / 1e9, 2), "resid": r, "phases": bc.last_timings(mesh)}), flush=True)
    del A, A0, x
    torch.cuda.empty_cache()
