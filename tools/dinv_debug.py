"""Where do potri bits diverge between device counts?  Factor (potrf) and
invert (potri) the same matrix at D=1 and D=2 and compare the factor and the
inverse column block by column block (float32 n=649 T_A=64 by default)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2601_14466_b200 as bc  # noqa: E402
from paper_2601_14466_b200 import solvers as S  # noqa: E402
from oracle import bcmg_oracle as O  # noqa: E402

n, t = int(os.environ.get("N", 649)), int(os.environ.get("T", 64))
dt = {"f32": np.float32, "c64": np.complex64}[os.environ.get("DT", "f32")]
a = O.make_matrix("random_spd", n, dt, 1172)
out = {}
for d in (1, 2):
    mesh = bc.make_mesh(d)
    desc = S._matrix_descriptor(a, S.Structure.positive_definite)
    dm = S.create_distributed(mesh, desc, bc.TileSpec(t))
    S.write_array(mesh, dm, a)
    dm = S.redistribute_in(mesh, dm)
    r = S.potrf(mesh, dm)
    dm = S.redistribute_out(mesh, dm)
    L = S.gather_array(mesh, dm)
    dm = S.redistribute_in(mesh, dm)
    S.potri(mesh, dm)
    dm = S.redistribute_out(mesh, dm)
    X = S.gather_array(mesh, dm)
    out[d] = (L, X)
    mesh.close()
L1, X1 = out[1]
L2, X2 = out[2]
for name, A1, A2 in (("factor", L1, L2), ("inverse", X1, X2)):
    diff = np.argwhere(A1 != A2)
    print(name, "differing elements:", len(diff))
    if len(diff):
        cols = sorted(set(int(c) // t for c in diff[:, 1]))
        rows = sorted(set(int(r) // t for r in diff[:, 0]))
        print("  tile columns:", cols[:20], " tile rows:", rows[:20], " first:", diff[:5].tolist())
