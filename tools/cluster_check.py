"""tcgen05 2-SM UMMA (CTA pair, BCMG_TCK_CLUSTER=2) trailing update vs the
single-CTA one: solutions within 10 N eps of each other (bit-identical if the
pair MMA sums each element in the same order).  Runs each variant in its own process (the switch is
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
    for cl in ("0", "2"):
        f = f"/tmp/x_{cl}.npy"
        r = subprocess.run([sys.executable, __file__, "child", str(n), str(t), str(d), dt, f],
                           env=dict(os.environ, BCMG_TCK_CLUSTER=cl), capture_output=True, text=True, timeout=300)
        print(n, t, d, dt, "cluster", cl, r.stdout.strip(), r.stderr[-300:])
        xs.append(np.load(f))
    same = np.array_equal(xs[0], xs[1])
    rel = float(np.abs(xs[0].astype(np.complex128) - xs[1]).max() / np.abs(xs[0]).max())
    ok &= rel <= 10 * n * 1.2e-7
    print("bit-identical:", same, "max rel diff", rel)
sys.exit(0 if ok else 1)
