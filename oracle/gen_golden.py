"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python oracle/gen_golden.py

It imports the reference package (``bcmg`` from /root/reference/pkg/src)
read-only, runs its own public entry points, and writes small fixtures to
``tests/golden/``.  Those fixtures travel with the repo; nothing at test
time reads /root/reference.  The oracle (oracle/bcmg_oracle.py) and the
GPU path are both checked against them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _ref():
    sys.path.insert(0, REF_SRC)
    import bcmg  # noqa: F401  (reference, read-only)
    from bcmg import cli, layout, oracle, solvers
    return bcmg, cli, layout, oracle, solvers


def numbered(n_rows, n_cols, dtype):
    base = np.arange(n_rows * n_cols, dtype=np.float64).reshape(n_rows, n_cols, order="F")
    dt = np.dtype(dtype)
    if dt.kind == "c":
        return np.asfortranarray((base - 1j * (base + 0.5)).astype(dt))
    return np.asfortranarray(base.astype(dt))


def layout_fixture(bcmg, layout):
    """dest_of + cycles + inverse cycles for every n<=24, T<=n, D<=4 and the
    reference's own executed column order (execute_plan on a 1-row matrix of
    numbered columns), so the fixture pins the executed behaviour, not just
    the formula."""
    from bcmg import DeviceMesh, ElementType, MatrixDescriptor, TileSpec
    from bcmg.solvers import create_distributed, write_array

    cases = []
    for n in range(1, 25):
        for t in range(1, n + 1):
            for d in range(1, 5):
                perm = layout.build_permutation(n, TileSpec(t), d)
                plan = layout.decompose_cycles(perm)
                inv = layout.invert_plan(plan)
                mesh = DeviceMesh(d)
                a = numbered(1, n, np.float64)
                dm = create_distributed(mesh, MatrixDescriptor(1, n, ElementType.real64), TileSpec(t))
                write_array(mesh, dm, a)
                cyc = layout.execute_plan(dm, plan, mesh)
                parts = []
                for h in cyc.shards:
                    cnt = h.nbytes // 8
                    parts.append(np.array(mesh.view(h, np.float64, (1, cnt))))
                executed = np.hstack(parts)[0].astype(np.int64).tolist()
                cases.append({
                    "n": n, "t": t, "d": d,
                    "dest_of": [int(x) for x in perm.dest_of],
                    "cycles": [list(map(int, c)) for c in plan.cycles],
                    "inverse": [list(map(int, c)) for c in inv.cycles],
                    "executed": executed,
                    "counts": layout.device_column_counts(n, TileSpec(t), d),
                })
    # BASELINE shapes: the tile-level structure only (column-level plans are big)
    shapes = []
    for (n, t, d) in [(2048, 256, 2), (32768, 1024, 1), (131072, 1024, 2), (131072, 1024, 4),
                      (131072, 1024, 8), (65536, 512, 8), (65536, 128, 2), (65536, 128, 4),
                      (65536, 128, 8), (65536, 2048, 8)]:
        plan = layout.decompose_cycles(layout.build_permutation(n, TileSpec(t), d))
        lens = [len(c) for c in plan.cycles]
        h = hashlib.sha256(np.asarray([x for c in plan.cycles for x in c], dtype=np.int64).tobytes()).hexdigest()
        shapes.append({"n": n, "t": t, "d": d, "n_cycles": len(plan.cycles),
                       "moved": int(sum(lens)), "max_len": max(lens) if lens else 0,
                       "first_cycles": [list(map(int, c)) for c in plan.cycles[:3]],
                       "sha256_members": h})
    return {"cases": cases, "baseline_shapes": shapes}


def solver_fixture(bcmg, cli, solvers):
    from bcmg import DeviceMesh, ElementType, TileSpec

    arrays = {}
    meta = []
    ets = {"f32": ElementType.real32, "f64": ElementType.real64,
           "c64": ElementType.complex64, "c128": ElementType.complex128}
    # random SPD solve/inverse cases small enough to commit whole
    for name, et in ets.items():
        for (n, t, d, nrhs, seed) in [(12, 5, 3, 3, 4), (24, 5, 2, 2, 8), (64, 32, 2, 1, 64),
                                      (40, 7, 4, 4, 11)]:
            a = cli.make_matrix("random_spd", n, et, seed)
            b = np.asfortranarray(numbered(n, nrhs, et.dtype) / n)
            x, _ = solvers.solve_positive_definite(DeviceMesh(d), a, b, TileSpec(t))
            key = f"potrs_{name}_n{n}_t{t}_d{d}_r{nrhs}_s{seed}"
            arrays[key + "_a"] = a
            arrays[key + "_b"] = b
            arrays[key + "_x"] = x
            meta.append({"key": key, "kind": "potrs", "dtype": name, "n": n, "t": t, "d": d,
                         "nrhs": nrhs, "seed": seed})
        for (n, t, d, seed) in [(20, 6, 2, 3), (18, 4, 4, 12), (33, 8, 3, 5)]:
            a = cli.make_matrix("random_spd", n, et, seed)
            inv, _ = solvers.invert_positive_definite(DeviceMesh(d), a, TileSpec(t))
            key = f"potri_{name}_n{n}_t{t}_d{d}_s{seed}"
            arrays[key + "_a"] = a
            arrays[key + "_inv"] = inv
            meta.append({"key": key, "kind": "potri", "dtype": name, "n": n, "t": t, "d": d,
                         "seed": seed})
    # BASELINE config 1: potrs f64 N=2048, T=256, N_RHS=1, 2 devices, random_spd seed 1.
    # A is regenerated from its seed at test time (32 MB); its hash pins the generator.
    a = cli.make_matrix("random_spd", 2048, ElementType.real64, 1)
    b = np.ones((2048, 1), order="F")
    x, _ = solvers.solve_positive_definite(DeviceMesh(2), a, b, TileSpec(256))
    arrays["config1_x"] = x
    cfg1 = {"n": 2048, "t": 256, "d": 2, "nrhs": 1, "seed": 1,
            "a_sha256": hashlib.sha256(np.ascontiguousarray(a).tobytes(order="F")).hexdigest(),
            "residual": cli.solve_residual(a, x, b)}
    # paper benchmark fixture input (diag) through the reference at a few tiles
    for t in (64, 256):
        a = cli.make_matrix("diag", 1024, ElementType.real64, 1)
        x, _ = solvers.solve_positive_definite(DeviceMesh(4), a, np.ones((1024, 1), order="F"),
                                               TileSpec(t))
        arrays[f"diag1024_t{t}_x"] = x
    # generator pins: hashes of make_matrix at a few sizes/dtypes
    gen = []
    for name, et in ets.items():
        for n, seed in [(16, 1), (64, 64), (256, 21)]:
            a = cli.make_matrix("random_spd", n, et, seed)
            gen.append({"dtype": name, "n": n, "seed": seed,
                        "sha256": hashlib.sha256(a.tobytes(order="F")).hexdigest()})
    return arrays, {"cases": meta, "config1": cfg1, "generator": gen}


def main():
    bcmg, cli, layout, oracle, solvers = _ref()
    os.makedirs(OUT, exist_ok=True)
    lay = layout_fixture(bcmg, layout)
    with open(os.path.join(OUT, "layout_golden.json"), "w") as fh:
        json.dump(lay, fh, separators=(",", ":"))
    arrays, meta = solver_fixture(bcmg, cli, solvers)
    np.savez_compressed(os.path.join(OUT, "solver_golden.npz"), **arrays)
    with open(os.path.join(OUT, "solver_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", OUT, len(lay["cases"]), "layout cases,", len(meta["cases"]), "solver cases")


if __name__ == "__main__":
    main()
