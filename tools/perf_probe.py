"""Quick GPU probe: potrs f64 at a given N/T/NRHS through the drop-in API,
device-timed, with phase split and residual. Not the bench (see bench.py)."""
import argparse, json, time
import numpy as np
import torch
import paper_2601_14466_b200 as bc

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=16)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
n, t, nrhs = args.n, args.t, args.nrhs
g = torch.Generator(device="cuda").manual_seed(1)
R = torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
A0 = (R + R.t()) * 0.5
A0.diagonal().add_(float(n))
del R
b = torch.rand(n, nrhs, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
mesh = bc.make_mesh(args.d)
A = torch.empty_like(A0)
for rep in range(args.reps):
    A.copy_(A0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x = bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    flops = n**3 / 3 + 2 * n * n * nrhs
    r = (A0 @ x - b).norm() / (A0.norm() * x.norm() + b.norm())
    print(json.dumps({"rep": rep, "ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 3),
                      "phases": {k: round(v, 3) for k, v in bc.last_timings(mesh).items()},
                      "residual": float(r)}), flush=True)
