"""Run one potrs (dtype, n, t, nrhs) for launch-list profiling."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc
dt = {"f32": torch.float32, "f64": torch.float64, "c64": torch.complex64, "c128": torch.complex128}[sys.argv[1]]
n, t, nrhs = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
R = torch.rand(n, n, device="cuda", dtype=torch.float64) - 0.5
A = (R + R.t()).to(dt); A.diagonal().add_(n); del R
b = torch.ones(n, nrhs, device="cuda", dtype=dt)
x = bc.potrs(A, b, T_A=t, mesh=bc.make_mesh(1), overwrite_a=True)
torch.cuda.synchronize(); print("ok", float(x.abs().max()))
