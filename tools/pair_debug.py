"""Locate the first tile where the paired-panel factor departs from the unpaired one."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2601_14466_b200 as bc
    from oracle import bcmg_oracle as O
    n, t, d = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    a = O.make_matrix("random_spd", n, np.float32, 1)
    mesh = bc.DeviceMesh(d)
    desc = bc.MatrixDescriptor(n, n, bc.ElementType.real32, bc.Structure.positive_definite)
    dm = bc.create_distributed(mesh, desc, bc.TileSpec(t))
    bc.write_array(mesh, dm, a)
    cyc = bc.redistribute_in(mesh, dm)
    r = bc.potrf(mesh, cyc)
    back = bc.redistribute_out(mesh, cyc)
    L = np.tril(bc.gather_array(mesh, back))
    np.save(sys.argv[5], L)
    print("info", r.info)
    sys.exit(0)
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
t = int(sys.argv[3]) if len(sys.argv) > 3 else 128
out = {}
for pp in ("0", "1"):
    env = dict(os.environ, BCMG_PAIR_PANELS=pp)
    f = f"/tmp/L_{pp}.npy"
    r = subprocess.run([sys.executable, __file__, "child", str(n), str(t), str(d), f], env=env, capture_output=True, text=True)
    print(pp, r.stdout.strip(), r.stderr[-500:])
    out[pp] = np.load(f)
diff = np.abs(out["0"].astype(np.float64) - out["1"].astype(np.float64))
for k in range(n // t):
    blk = diff[:, k * t:(k + 1) * t]
    print(k, float(blk.max()), float(np.abs(out["0"][:, k * t:(k + 1) * t]).max()))
