"""Time the REFERENCE eigensolver on this container's CPU cores (measurement
helper, test infrastructure): imports /root/reference read-only and runs its
public eigh_hermitian (solvers.py:1019-1043) beside scipy's LAPACK eigh.

    python oracle/time_reference_eigen.py
"""
import sys, time, os
import numpy as np
sys.path.insert(0, "/root/reference/pkg/src")
from bcmg import DeviceMesh, ElementType, TileSpec, cli
from bcmg.solvers import eigh_hermitian
import scipy.linalg
print(f"cpu_count={os.cpu_count()}")
for n in (256, 512, 1024):
    a = cli.make_matrix("random_spd", n, ElementType.real64, 1)
    t0 = time.perf_counter(); w, v, _ = eigh_hermitian(DeviceMesh(1), a, TileSpec(64)); t1 = time.perf_counter()
    t2 = time.perf_counter(); scipy.linalg.eigh(a); t3 = time.perf_counter()
    print(f"reference eigh_hermitian f64 n={n} T=64 D=1: {t1-t0:.2f} s; scipy.linalg.eigh (LAPACK, OpenBLAS threads): {t3-t2:.3f} s", flush=True)
