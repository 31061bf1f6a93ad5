"""tcgen05 CTA-pair (B multicast) trailing update vs the single-CTA one: the
factor must be bit-identical (same MMAs per element, only the CTA-to-row map and
the B delivery differ).  Runs each variant in its own process (the switch is
read once)."""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2601_14466_b200 as bc
    from oracle import bcmg_oracle as O
    n, t, d, dt = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), {"f32": np.float32, "c64": np.complex64}[sys.argv[5]]
    a = O.make_matrix("random_spd", n, dt, 3)
    b = np.ones((n, 2), dtype=dt, order="F")
    x, _ = bc.solve_positive_definite(bc.DeviceMesh(d), a, b, bc.TileSpec(t))
    np.save(sys.argv[6], x)
    print("residual", O.solve_residual(a, x, b))
    sys.exit(0)
ok = True
for n, t, d, dt in ((2048, 512, 1, "f32"), (4096, 1024, 2, "f32"), (3072, 512, 1, "c64"), (4096, 256, 4, "f32")):
    xs = []
    for cl in ("0", "1"):
        f = f"/tmp/x_{cl}.npy"
        r = subprocess.run([sys.executable, __file__, "child", str(n), str(t), str(d), dt, f],
                           env=dict(os.environ, BCMG_TCK_CLUSTER=cl), capture_output=True, text=True, timeout=300)
        print(n, t, d, dt, "cluster", cl, r.stdout.strip(), r.stderr[-300:])
        xs.append(np.load(f))
    same = np.array_equal(xs[0], xs[1])
    ok &= same
    print("bit-identical:", same)
sys.exit(0 if ok else 1)
