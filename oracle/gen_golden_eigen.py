"""Golden fixtures for the eigensolver from the REFERENCE itself.

    python oracle/gen_golden_eigen.py

Imports the reference package (``bcmg`` from /root/reference/pkg/src)
read-only, runs its public ``eigh_hermitian`` (solvers.py:1019-1043) on the
cases of its own tests (test_solvers.py:231-280, test_acceptance.py:219-268)
and writes tests/golden/eigen_golden.npz.  Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "eigen_golden.npz")


def main():
    sys.path.insert(0, REF_SRC)
    from bcmg import DeviceMesh, ElementType, TileSpec, cli  # reference, read-only
    from bcmg.solvers import eigh_hermitian

    cases = {}

    def add(name, a, devices, tile):
        w, v, _ = eigh_hermitian(DeviceMesh(devices), a, TileSpec(tile))
        cases[f"{name}__a"] = a
        cases[f"{name}__w"] = w
        cases[f"{name}__v"] = v
        cases[f"{name}__cfg"] = np.array([devices, tile])

    f = lambda x: np.asfortranarray(np.asarray(x, dtype=np.float64))  # noqa: E731
    add("diag3", f(np.diag([3.0, 1.0, 2.0])), 1, 1)
    add("hand2", f([[2.0, 1.0], [1.0, 2.0]]), 2, 1)
    add("eye8", f(np.eye(8)), 2, 3)
    for et, tag in ((ElementType.real32, "f32"), (ElementType.real64, "f64"), (ElementType.complex64, "c64"),
                    (ElementType.complex128, "c128")):
        add(f"rand24_{tag}", cli.make_matrix("random_spd", 24, et, 6), 3, 5)
        add(f"rand40_{tag}", cli.make_matrix("random_spd", 40, et, 13), 2, 16)
    add("rand12_f64", cli.make_matrix("random_spd", 12, ElementType.real64, 7), 2, 4)
    # separated spectrum (eigenvalues 1..n: elementwise eigenvector comparison is well posed)
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((32, 32)))
    sep = q @ np.diag(np.arange(1.0, 33.0)) @ q.T
    add("sep32_f64", f((sep + sep.T) / 2), 2, 7)
    qc, _ = np.linalg.qr(rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20)))
    sepc = qc @ np.diag(np.arange(1.0, 21.0)) @ qc.conj().T
    add("sep20_c128", np.asfortranarray((sepc + sepc.conj().T) / 2), 3, 4)
    np.savez_compressed(OUT, **cases)
    # BCMG matrix files written by the reference's own write_matrix (core.py:255-273)
    from bcmg import write_matrix
    gold = os.path.dirname(OUT)
    write_matrix(os.path.join(gold, "ref_random_spd5_c64.bcmg"), cli.make_matrix("random_spd", 5, ElementType.complex64, 2))
    write_matrix(os.path.join(gold, "ref_vector3_f32.bcmg"), np.array([1.5, -2.0, 3.25], dtype=np.float32))
    print(f"wrote {OUT}: {len(cases) // 4} cases")


if __name__ == "__main__":
    main()
