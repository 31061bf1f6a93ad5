"""complex128 potrs through the real-embedded TMA trailing update vs numpy (debug probe)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc
from oracle import bcmg_oracle as O

cases = [(12, 5, 1), (12, 5, 3), (16, 4, 1), (64, 32, 1), (64, 32, 2), (256, 64, 1), (1000, 100, 2), (2048, 256, 1)]
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in sys.argv[1].split(","))]
for n, t, d in cases:
    a = O.make_matrix("random_spd", n, np.complex128, 4)
    b = np.ones((n, 2), dtype=np.complex128, order="F")
    x, _ = bc.solve_positive_definite(bc.make_mesh(d), a, b, bc.TileSpec(t))
    xr = np.linalg.solve(a, b)
    print(n, t, d, float(np.abs(x - xr).max() / np.abs(xr).max()), flush=True)
