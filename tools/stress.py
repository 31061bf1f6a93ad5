#!/usr/bin/env python3
"""Randomised parity sweep on the GPU: potrs / potri over random (n, T_A, D,
dtype, N_RHS) against the unblocked oracle (elementwise 10 n eps, residual
100 n eps), plus D-invariance of the bits on every fourth case.  Prints one
JSON line per failure and a summary.

    python tools/stress.py --cases 200 --seed 1
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from oracle import bcmg_oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=200)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--dtypes", default="f32,f64,c64,c128")
ap.add_argument("--tiles", default="16,32,48,64,96,128,192,256,384,512")
ap.add_argument("--nmax", type=int, default=3000)
ap.add_argument("--dcheck", type=int, default=4, help="check D-invariance on every k-th case")
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
meshes = {}
def mesh(d):
    if d not in meshes:
        meshes[d] = bc.make_mesh(d)
    return meshes[d]
dtypes = [{"f32": np.float32, "f64": np.float64, "c64": np.complex64, "c128": np.complex128}[x]
          for x in a.dtypes.split(",")]
tiles = [int(x) for x in a.tiles.split(",")]
fails, done = 0, 0
for i in range(a.cases):
    dt = dtypes[rng.integers(len(dtypes))]
    n = int(rng.integers(65, a.nmax + 1))
    t = int(rng.choice(tiles))
    t = min(t, n)
    d = int(rng.choice([1, 2, 3, 4, 8]))
    routine = "potri" if rng.random() < 0.25 else "potrs"
    nrhs = int(rng.integers(1, 7))
    A = O.make_matrix("random_spd", n, dt, 1000 + i)
    eps = O.eps_of(dt)
    case = {"i": i, "dtype": np.dtype(dt).name, "n": n, "t": t, "d": d, "routine": routine, "nrhs": nrhs}
    try:
        if routine == "potrs":
            b = rng.standard_normal((n, nrhs))
            if np.iscomplexobj(np.zeros(1, dt)):
                b = b + 1j * rng.standard_normal((n, nrhs))
            b = np.asfortranarray(b.astype(dt))
            x, _ = bc.solve_positive_definite(mesh(d), A, b, bc.TileSpec(t))
            xr = O.solve_unblocked(A, b)
            err = float(np.abs(x - xr).max() / max(1.0, np.abs(xr).max()))
            res = float(O.solve_residual(A, x, b))
            ok = err <= 10 * n * eps and res <= 100 * n * eps
            if ok and i % a.dcheck == 0:
                x1, _ = bc.solve_positive_definite(mesh(1), A, b, bc.TileSpec(t))
                ok = np.array_equal(x1, x)
                case["d_invariant"] = bool(ok)
        else:
            inv, _ = bc.invert_positive_definite(mesh(d), A, bc.TileSpec(t))
            res = float(O.inverse_residual(A, inv))
            err = None
            ok = res <= 100 * n * eps and np.array_equal(inv, inv.conj().T)
            if ok and i % a.dcheck == 0:
                inv1, _ = bc.invert_positive_definite(mesh(1), A, bc.TileSpec(t))
                ok = np.array_equal(inv1, inv)
                case["d_invariant"] = bool(ok)
        case.update({"err": err, "res": res})
    except Exception as e:  # noqa: BLE001
        ok = False
        case["exception"] = repr(e)[:300]
    done += 1
    if not ok:
        fails += 1
        print(json.dumps(case), flush=True)
print(json.dumps({"cases": done, "failures": fails}), flush=True)
for m in meshes.values():
    m.close()
