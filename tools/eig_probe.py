"""Time the GPU eigensolver (bcmg_syevd through eigh_hermitian) -- probe, not the bench.

    python tools/eig_probe.py --n 2048,4096 --tile 64 --dtype f64
"""
import argparse, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="2048")
ap.add_argument("--tile", type=int, default=64)
ap.add_argument("--dtype", default="f64")
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--check", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
dt = {"f32": np.float32, "f64": np.float64, "c64": np.complex64, "c128": np.complex128}[a.dtype]
mesh = bc.DeviceMesh(a.d, device=0)
for n in map(int, a.n.split(",")):
    rng = np.random.default_rng(n)
    b = rng.uniform(-1, 1, (n, n))
    if np.dtype(dt).kind == "c":
        b = b + 1j * rng.uniform(-1, 1, (n, n))
    A = np.asfortranarray(((b + b.conj().T) / 2).astype(dt))
    bc.eigh_hermitian(mesh, A[:64, :64].copy(order="F"), bc.TileSpec(min(a.tile, 64)))  # warm
    runs = []
    for _ in range(a.reps):  # the first call also allocates the session workspace
        t0 = time.perf_counter()
        w, v, tm = bc.eigh_hermitian(mesh, A, bc.TileSpec(a.tile))
        runs.append((time.perf_counter() - t0, tm.device_ms))
    t1 = 0.0
    out = {"n": n, "dtype": a.dtype, "tile": a.tile, "wall_s": [round(r[0], 3) for r in runs],
           "device_ms": [round(r[1], 1) for r in runs],
           "launches": int(bc._lib.load().bcmg_launch_count())}
    if a.check:
        import torch
        wide = torch.complex128 if np.dtype(dt).kind == "c" else torch.float64
        At = torch.from_numpy(A).to("cuda", wide)
        Vt = torch.from_numpy(np.ascontiguousarray(v)).to("cuda", wide)
        Wt = torch.from_numpy(w.astype(np.float64)).to("cuda")
        res = torch.linalg.norm(At @ Vt - Vt * Wt).item() / torch.linalg.norm(At).item()
        orth = torch.linalg.norm(Vt.conj().T @ Vt - torch.eye(n, device="cuda", dtype=wide)).item()
        wr = torch.linalg.eigvalsh(At).cpu().numpy()
        out.update(residual=res, orth=orth, max_w_err=float(np.max(np.abs(w - wr))))
    print(out, flush=True)
mesh.close()
