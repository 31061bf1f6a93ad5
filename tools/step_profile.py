"""Per-launch profile of one potrs (kernel kind, ms, algorithmic work) via
bcmg_set_profiling + BCMG_PROFILE_DUMP; prints per-kind efficiency."""
import argparse, ctypes as C, os, sys, collections
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc
from paper_2601_14466_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768); ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--nrhs", type=int, default=16); ap.add_argument("--out", default="gpurun_out/step_profile.txt")
a = ap.parse_args()
n, t = a.n, a.t
g = torch.Generator(device="cuda").manual_seed(1)
A0 = torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
A0 = (A0 + A0.t()) * 0.5; A0.diagonal().add_(float(n))
b = torch.rand(n, a.nrhs, device="cuda", dtype=torch.float64, generator=g)
mesh = bc.make_mesh(1); lib = _lib.load()
A = A0.clone(); bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)
A.copy_(A0); torch.cuda.synchronize()
lib.bcmg_set_profiling(mesh.session, 1)
if os.path.exists(a.out): os.remove(a.out)
os.environ["BCMG_PROFILE_DUMP"] = a.out
bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)
st = (C.c_double * 4)()
for kind in range(4): lib.bcmg_kernel_stats(mesh.session, kind, st)
names = {0: "trail", 1: "trsm", 2: "diag", 3: "rotate"}
rows = [l.split() for l in open(a.out)]
for kind in range(4):
    r = [(int(x[1]), float(x[2]), float(x[3])) for x in rows if int(x[0]) == kind]
    if not r: continue
    ms = sum(x[1] for x in r); w = sum(x[2] for x in r)
    print(f"{names[kind]:6s} launches={len(r):4d} ms={ms:9.3f} work={w:.3e} rate={w/ms/1e9 if ms else 0:8.2f} T/s")
    if kind == 0:
        for i, msi, wi in r:
            print(f"   trail[{i:3d}] {msi:8.3f} ms {wi/msi/1e9 if msi else 0:7.2f} TF/s  ({wi:.2e} flop)")
print(bc.last_timings(mesh))
