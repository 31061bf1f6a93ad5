"""A/B a kernel switch (an environment variable read once per process) on the
factor/solve: each variant solves the same systems in its own process; reports
bit-identity and the max relative difference (must be within 10 N eps).

    python tools/ab_check.py BCMG_TCK_EPI 0 1
"""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASES = ((2048, 128, 1, "f32"), (4096, 128, 2, "f32"), (3072, 128, 1, "c64"), (4096, 128, 8, "f32"), (2048, 256, 4, "c64"),
         (3072, 256, 1, "f32"), (4096, 512, 2, "f32"), (4096, 1024, 1, "c64"))
if os.environ.get("AB_CASES") == "all":
    CASES = CASES + ((1500, 64, 1, "f64"), (2100, 100, 3, "c128"), (1441, 512, 2, "f64"), (777, 60, 1, "f32"),
                     (1000, 200, 1, "c64"))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2601_14466_b200 as bc
    from oracle import bcmg_oracle as O
    n, t, d, dt = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), {"f32": np.float32, "c64": np.complex64, "f64": np.float64, "c128": np.complex128}[sys.argv[5]]
    a = O.make_matrix("random_spd", n, dt, 3)
    b = np.ones((n, 2), dtype=dt, order="F")
    x, _ = bc.solve_positive_definite(bc.DeviceMesh(d), a, b, bc.TileSpec(t))
    np.save(sys.argv[6], x)
    print("residual", O.solve_residual(a, x, b))
    sys.exit(0)
var, v0, v1 = sys.argv[1], sys.argv[2], sys.argv[3]
ok = True
for n, t, d, dt in CASES:
    xs = []
    for v in (v0, v1):
        f = f"/tmp/ab_x_{(v0, v1).index(v)}.npy"
        r = subprocess.run([sys.executable, __file__, "child", str(n), str(t), str(d), dt, f],
                           env=dict(os.environ, **{var: v}), capture_output=True, text=True, timeout=300)
        print(n, t, d, dt, var, v, r.stdout.strip(), r.stderr[-300:])
        xs.append(np.load(f))
    rel = float(np.abs(xs[0].astype(np.complex128) - xs[1]).max() / np.abs(xs[0]).max())
    ok &= rel <= 10 * n * 1.2e-7
    print("bit-identical:", np.array_equal(xs[0], xs[1]), "max rel diff", rel)
sys.exit(0 if ok else 1)
