"""`verify` / `bench` command line in the reference's schema (reference
pkg/src/bcmg/cli.py), on the B200 path.

    python -m paper_2601_14466_b200.cli verify --routine potrs --n 4096 --tile 256 --devices 1,2,4
    python -m paper_2601_14466_b200.cli bench  --routine potrs --n 8192 --tile 1024 --reps 5 --out run.csv

* verify prints one ``PASS|FAIL <check> tile=T devices=D value=V tol=TOL``
  line per check (cli.py:355-362) and exits 1 on the first failure;
* bench writes a CSV whose first columns are the reference's BENCH_COLUMNS
  (cli.py:65-68) followed by the device-side phase split and TFLOP/s;
* residuals are evaluated on the GPU at 64-bit precision (cli.py:113-125):
  the product A x (or A X) is one call of the library's own GEMM
  (bcmg_gemm) on the widened operands, the norms are device reductions;
* exit codes: 0 ok, 1 check failure / not positive definite / out of device
  memory, 2 configuration error (cli.py:462-482).

Matrix sources: ``diag`` (diag(1..n)), ``random_spd`` (B B^H + n I, B from
numpy Philox(key=seed), cli.py:81-103 -- host-generated, O(n^3)),
``device_spd`` ((R + R^H)/2 + n I generated on the GPU by bcmg_generate_spd,
for large n) and ``file:PATH`` (a BCMG matrix file, core.py:255-303; ``gen``
writes one, cli.py:449-458).  Routines: potrs, potri and syevd (eigen-residual,
orthonormality, ascending order and the diag(1..n) spectrum, cli.py:320-337).
Modes (``--mode`` or ``$BCMG_MODE``, cli.py:62-64, 242-256): ``spmd`` -- one
session with every logical device in one address space; ``mpmd`` -- one
isolated worker (own session, own shard allocation) per logical device, shards
reached only through the transport's handle exchange (isolated.py); both give
the same bits.  Out of scope: copy transcripts (``--trace``),
rejected as a configuration error.
"""

from __future__ import annotations

import argparse
import csv
import ctypes as C
import statistics
import sys

import numpy as np

from . import _lib, isolated
from .core import (ConvergenceError, DescriptorError, ElementType, MatrixFileError, NotPositiveDefiniteError,
                   OutOfDeviceMemoryError, TileSpec, read_matrix, write_matrix)
from .mesh import DeviceMesh
from .solvers import eigh_hermitian, invert_positive_definite, solve_positive_definite

ROUTINES = ("potrs", "potri", "syevd")
MATRIX_KINDS = ("diag", "random_spd", "device_spd")
BENCH_COLUMNS = ["routine", "n", "tile", "devices", "dtype", "mode", "rep", "alloc_seconds", "solve_seconds",
                 "residual"]
EXTRA_COLUMNS = ["redistribute_ms", "potrf_ms", "finish_ms", "device_ms", "tflops"]
_DTYPE_NAMES = {ElementType.real32: "f32", ElementType.real64: "f64", ElementType.complex64: "c64",
                ElementType.complex128: "c128"}


# ----------------------------------------------------------------- test problems
def make_matrix(kind: str, n: int, et: ElementType, seed: int) -> np.ndarray:
    """diag(1..n) or B B^H + n I with B ~ U[-1, 1) from Philox(key=seed),
    made exactly Hermitian (the reference generator, cli.py:81-103)."""
    dt = et.dtype
    if kind == "diag":
        return np.asfortranarray(np.diag(np.arange(1, n + 1)).astype(dt))
    if kind == "random_spd":
        gen = np.random.Generator(np.random.Philox(key=seed))
        b = gen.uniform(-1.0, 1.0, (n, n))
        if et.is_complex:
            b = b + 1j * gen.uniform(-1.0, 1.0, (n, n))
        a = b @ b.conj().T + n * np.eye(n)
        a = (a + a.conj().T) / 2
        return np.asfortranarray(a.astype(dt))
    if kind == "device_spd":
        import torch

        lib = _lib.load()
        t = torch.empty(n, n, dtype=et.torch_dtype, device="cuda")
        _lib.check(lib.bcmg_generate_spd(C.c_void_p(torch.cuda.current_stream().cuda_stream), et.code, n, 0, n,
                                         C.c_void_p(t.data_ptr()), n, seed, float(n)))
        return np.asfortranarray(t.cpu().numpy())  # row-major element (i, j) = A_ij
    raise DescriptorError("type-structure", f"--matrix must be one of {MATRIX_KINDS}, got {kind!r}")


# ----------------------------------------------------------------- GPU residuals (64-bit)
def _wide(arr: np.ndarray, device):
    """Column-major device copy at 64-bit precision (the buffer of a.T is a's columns)."""
    import torch

    wide = np.complex128 if np.iscomplexobj(arr) else np.float64
    host = np.ascontiguousarray(np.asarray(arr, dtype=wide).T)
    return torch.from_numpy(host).to(device)


def _gemm_residual(a, x, rhs, device):
    """(A X - R) as a device tensor via bcmg_gemm, R given (column-major)."""
    import torch

    cplx = np.iscomplexobj(a) or np.iscomplexobj(x) or np.iscomplexobj(rhs)
    if cplx:
        a, x, rhs = (np.asarray(v, dtype=np.complex128) for v in (a, x, rhs))
    A, X, R = _wide(a, device), _wide(x, device), _wide(rhs, device)
    n, k = a.shape[0], x.shape[1]
    code = 3 if cplx else 1
    lib = _lib.load()
    stream = C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    _lib.check(lib.bcmg_gemm(stream, code, n, k, n, 1.0, C.c_void_p(A.data_ptr()), n, 0, C.c_void_p(X.data_ptr()), n,
                             0, -1.0, C.c_void_p(R.data_ptr()), n))
    return A, X, R


def solve_residual(a: np.ndarray, x: np.ndarray, b: np.ndarray, device="cuda") -> float:
    """||A x - b||_F / (||A||_F ||x||_F + ||b||_F) at 64-bit precision (cli.py:113-118)."""
    import torch

    x2 = x.reshape(-1, 1) if x.ndim == 1 else x
    b2 = b.reshape(-1, 1) if b.ndim == 1 else b
    A, X, R = _gemm_residual(a, x2, b2, device)
    num = torch.linalg.vector_norm(R)
    den = torch.linalg.vector_norm(A) * torch.linalg.vector_norm(X) + float(np.linalg.norm(np.asarray(b2, np.complex128)))
    return float(num / den) if float(den) else float(num)


def inverse_residual(a: np.ndarray, inv: np.ndarray, device="cuda") -> float:
    """||A X - I||_F / sqrt(n) at 64-bit precision (cli.py:121-125)."""
    import torch

    n = a.shape[0]
    _, _, R = _gemm_residual(a, inv, np.eye(n), device)
    return float(torch.linalg.vector_norm(R) / np.sqrt(n))


def eigen_residual(a: np.ndarray, w: np.ndarray, v: np.ndarray, device="cuda") -> float:
    """||A V - V diag(w)||_F / ||A||_F at 64-bit precision (cli.py:128-133):
    A V through bcmg_gemm, minus V diag(w) on the device."""
    import torch

    A, V, AV = _gemm_residual(a, v, np.zeros(v.shape, dtype=np.result_type(a, v)), device)
    W = torch.from_numpy(np.asarray(w, dtype=np.float64)).to(device)
    R = AV - V * W[:, None].to(V.dtype)  # column-major buffers: row j of the .T view is column j
    den = torch.linalg.vector_norm(A)
    num = torch.linalg.vector_norm(R)
    return float(num / den) if float(den) else float(num)


def orthonormality_defect(v: np.ndarray, device="cuda") -> float:
    """||V^H V - I||_F at 64-bit precision (cli.py:136-140)."""
    import torch

    V = _wide(v, device)  # rows of V are the columns of v
    n = v.shape[1]
    G = V.conj() @ V.T
    return float(torch.linalg.vector_norm(G - torch.eye(n, dtype=G.dtype, device=device)))


def _residual_tol(et: ElementType, n: int) -> float:
    return 100.0 * n * et.eps


def _elementwise_tol(et: ElementType) -> float:
    return 1e-12 if et.eps < 1e-10 else 1e-4


def _eigen_diag_tol(et: ElementType) -> float:
    return 1e-10 if et.eps < 1e-10 else 1e-4


# ----------------------------------------------------------------- parser
def _int_list(text: str) -> list[int]:
    try:
        return [int(part) for part in text.split(",") if part]
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers: {text!r}")


def _common(p: argparse.ArgumentParser) -> None:
    p.add_argument("--tile", type=_int_list, default=None, help="tile width(s), comma list (default min(64, n))")
    p.add_argument("--devices", type=_int_list, default=[1], help="logical device count(s), comma list")
    p.add_argument("--dtype", choices=sorted(_DTYPE_NAMES.values()), default="f64")
    p.add_argument("--mode", choices=("spmd", "mpmd"), default=None)
    p.add_argument("--matrix", default="diag", metavar="SOURCE", help="diag, random_spd, device_spd or file:PATH")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--nrhs", type=int, default=1)
    p.add_argument("--trace", metavar="PATH", help="(not supported on the GPU path)")
    p.add_argument("--arena-cap", type=int, default=None, metavar="BYTES", help="(ignored: HBM is the arena)")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="bcmg-b200", description="Distributed Cholesky solves on B200.")
    sub = parser.add_subparsers(dest="command", required=True)
    v = sub.add_parser("verify", help="run a routine and check invariants")
    v.add_argument("--routine", required=True, choices=ROUTINES)
    v.add_argument("--n", type=int, default=None, help="matrix order (from the file for file:PATH)")
    v.add_argument("--rhs", metavar="PATH", help="read the right-hand side from a matrix file (potrs)")
    v.add_argument("--result-out", metavar="PATH", help="write the solution / inverse / eigenvectors")
    v.add_argument("--eigenvalues-out", metavar="PATH", help="write the eigenvalues as an n x 1 matrix (syevd)")
    v.add_argument("--tolerance", type=float, default=None)
    _common(v)
    b = sub.add_parser("bench", help="time repeated runs, CSV per rep")
    b.add_argument("--routine", required=True, choices=ROUTINES)
    b.add_argument("--n", type=int, required=True)
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--out", default="-", metavar="PATH")
    _common(b)
    g = sub.add_parser("gen", help="write a test matrix file")
    g.add_argument("--kind", required=True, choices=("diag", "random_spd", "ones"))
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--nrhs", type=int, default=1, help="columns for --kind ones")
    g.add_argument("--dtype", choices=sorted(_DTYPE_NAMES.values()), default="f64")
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True, metavar="PATH")
    return parser


MODE_ENV_VAR = "BCMG_MODE"
CLI_MODES = ("spmd", "mpmd")


def _resolve_mode(args) -> str:
    """--mode, else $BCMG_MODE, else spmd (cli.py:242-248)."""
    import os

    mode = args.mode if args.mode is not None else os.environ.get(MODE_ENV_VAR, "spmd")
    if mode not in CLI_MODES:
        raise DescriptorError("type-structure", f"{MODE_ENV_VAR}={mode!r} is not one of {CLI_MODES}")
    return mode


def _check_scope(args) -> None:
    args.mode = _resolve_mode(args)
    if args.trace:
        raise DescriptorError("type-structure", "--trace: the GPU rotation keeps no copy transcript")
    if args.matrix.startswith("file:"):
        return
    if args.matrix not in MATRIX_KINDS:
        raise DescriptorError("type-structure",
                              f"--matrix must be one of {MATRIX_KINDS} or file:PATH, got {args.matrix!r}")
    if args.n is None or args.n < 1:
        raise DescriptorError("dimension-mismatch", f"--n must be >= 1, got {args.n}")
    if any(d < 1 for d in args.devices):
        raise DescriptorError("dimension-mismatch", f"--devices must be >= 1, got {args.devices}")


def _tiles(args, n: int) -> list[int]:
    return args.tile if args.tile else [min(64, n)]


def _load_problem(args):
    """(A, element type, generator kind or None for a file) -- cli.py:263-285."""
    if args.matrix.startswith("file:"):
        a = read_matrix(args.matrix[len("file:"):])
        if a.shape[0] != a.shape[1]:
            raise DescriptorError("dimension-mismatch", f"input matrix must be square, got {a.shape[0]}x{a.shape[1]}")
        return a, ElementType.from_dtype(a.dtype), None
    et = ElementType.from_name(args.dtype)
    return make_matrix(args.matrix, args.n, et, args.seed), et, args.matrix


def _flops(routine: str, n: int, nrhs: int, et: ElementType) -> float:
    if routine == "syevd":  # tridiagonalisation 4/3 n^3 + back-transformation 2 n^3 (LAWN-41)
        return (10 * n ** 3 / 3) * (4 if et.is_complex else 1)
    f = n ** 3 / 3 + 2 * n * n * nrhs if routine == "potrs" else n ** 3
    return f * (4 if et.is_complex else 1)


# ----------------------------------------------------------------- commands
def _verify_one(args, a, et, kind, tile, devices):
    """One configuration: [(check, value, tol)] (cli.py:288-345)."""
    n = a.shape[0]
    res_tol = args.tolerance if args.tolerance is not None else _residual_tol(et, n)
    elem_tol = args.tolerance if args.tolerance is not None else _elementwise_tol(et)
    mpmd = args.mode == "mpmd"
    mesh = None if mpmd else DeviceMesh(devices)
    checks = []
    try:
        if args.routine == "potrs":
            if args.rhs:
                b = read_matrix(args.rhs)
                if ElementType.from_dtype(b.dtype) is not et:
                    raise DescriptorError("type-structure", "right-hand side element type does not match the matrix")
            else:
                b = np.ones((n, args.nrhs), dtype=et.dtype, order="F")
            x, _ = (isolated.solve_positive_definite_isolated(a, b, TileSpec(tile), devices) if mpmd else
                    solve_positive_definite(mesh, a, b, TileSpec(tile)))
            checks.append(("solve-residual", solve_residual(a, x, b), res_tol))
            if kind == "diag" and not args.rhs:
                expected = 1.0 / np.arange(1, n + 1, dtype=np.float64)
                checks.append(("diag-solution", float(np.abs(x.astype(np.complex128) - expected[:, None]).max()),
                               elem_tol))
            result = x
        elif args.routine == "potri":
            inv, _ = (isolated.invert_positive_definite_isolated(a, TileSpec(tile), devices) if mpmd else
                      invert_positive_definite(mesh, a, TileSpec(tile)))
            checks.append(("inverse-residual", inverse_residual(a, inv), res_tol))
            if kind == "diag":
                expected = np.diag(1.0 / np.arange(1, n + 1, dtype=np.float64))
                checks.append(("diag-inverse", float(np.abs(inv.astype(np.complex128) - expected).max()), elem_tol))
            result = inv
        else:
            w, v, _ = (isolated.eigh_hermitian_isolated(a, TileSpec(tile), devices) if mpmd else
                       eigh_hermitian(mesh, a, TileSpec(tile)))
            checks.append(("eigen-residual", eigen_residual(a, w, v), res_tol))
            checks.append(("orthonormal", orthonormality_defect(v), res_tol))
            ascent = float(max(0.0, np.max(w[:-1] - w[1:]))) if n > 1 else 0.0
            checks.append(("ascending", ascent, 0.0))
            if kind == "diag":
                err = float(np.max(np.abs(w.astype(np.float64) - np.arange(1, n + 1, dtype=np.float64))))
                checks.append(("diag-eigenvalues", err,
                               args.tolerance if args.tolerance is not None else _eigen_diag_tol(et)))
            if args.eigenvalues_out:
                write_matrix(args.eigenvalues_out, w.reshape(-1, 1))
            result = v
        if args.result_out:
            write_matrix(args.result_out, result)
    finally:
        if mesh is not None:
            mesh.close()
    return checks


def _cmd_verify(args) -> int:
    _check_scope(args)
    a, et, kind = _load_problem(args)
    failed = []
    for tile in _tiles(args, a.shape[0]):
        for devices in args.devices:
            for name, value, tol in _verify_one(args, a, et, kind, tile, devices):
                ok = value <= tol  # False for NaN as well
                if not ok:
                    failed.append(name)
                print(f"{'PASS' if ok else 'FAIL'} {name} tile={tile} devices={devices} value={value!r} tol={tol!r}")
    if failed:
        print(f"failed: {failed[0]}", file=sys.stderr)
        return 1
    return 0


def _cmd_gen(args) -> int:
    """Write a test matrix file (cli.py:449-458)."""
    et = ElementType.from_name(args.dtype)
    if args.n < 1:
        raise DescriptorError("dimension-mismatch", f"--n must be >= 1, got {args.n}")
    if args.kind == "ones":
        arr = np.ones((args.n, args.nrhs), dtype=et.dtype, order="F")
    else:
        arr = make_matrix(args.kind, args.n, et, args.seed)
    write_matrix(args.out, arr)
    return 0


def _cmd_bench(args) -> int:
    _check_scope(args)
    if args.reps < 1:
        raise DescriptorError("dimension-mismatch", "--reps must be >= 1")
    a, et, _ = _load_problem(args)
    n = a.shape[0]
    out = open(args.out, "w", newline="") if args.out != "-" else sys.stdout
    try:
        w = csv.writer(out, lineterminator="\n")
        w.writerow(BENCH_COLUMNS + EXTRA_COLUMNS)
        for tile in _tiles(args, n):
            for devices in args.devices:
                mpmd = args.mode == "mpmd"
                mesh = None if mpmd else DeviceMesh(devices)
                solves, allocs = [], []
                for rep in range(args.reps):
                    if args.routine == "potrs":
                        b = np.ones((n, args.nrhs), dtype=et.dtype, order="F")
                        x, tm = (isolated.solve_positive_definite_isolated(a, b, TileSpec(tile), devices) if mpmd
                                 else solve_positive_definite(mesh, a, b, TileSpec(tile)))
                        residual = solve_residual(a, x, b)
                    elif args.routine == "potri":
                        inv, tm = (isolated.invert_positive_definite_isolated(a, TileSpec(tile), devices) if mpmd
                                   else invert_positive_definite(mesh, a, TileSpec(tile)))
                        residual = inverse_residual(a, inv)
                    else:
                        ev, vecs, tm = (isolated.eigh_hermitian_isolated(a, TileSpec(tile), devices) if mpmd
                                        else eigh_hermitian(mesh, a, TileSpec(tile)))
                        residual = eigen_residual(a, ev, vecs)
                    solves.append(tm.solve_seconds)
                    allocs.append(tm.alloc_seconds)
                    tflops = _flops(args.routine, n, args.nrhs, et) / (tm.device_ms * 1e-3) / 1e12 if tm.device_ms else 0
                    w.writerow([args.routine, n, tile, devices, args.dtype, args.mode, rep, repr(tm.alloc_seconds),
                                repr(tm.solve_seconds), repr(residual), tm.redistribute_ms, tm.potrf_ms, tm.finish_ms,
                                tm.device_ms, tflops])
                if mesh is not None:
                    mesh.close()
                print(f"{args.routine} n={n} tile={tile} devices={devices} dtype={args.dtype} mode={args.mode} "
                      f"reps={args.reps}: alloc min={min(allocs):.9f} median={statistics.median(allocs):.9f} s; "
                      f"solve min={min(solves):.9f} median={statistics.median(solves):.9f} s", file=sys.stderr)
    finally:
        if out is not sys.stdout:
            out.close()
    return 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        if args.command == "gen":
            return _cmd_gen(args)
        return _cmd_verify(args) if args.command == "verify" else _cmd_bench(args)
    except MatrixFileError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except (DescriptorError, ValueError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except NotPositiveDefiniteError as exc:
        print(f"not positive definite: pivot={exc.pivot}", file=sys.stderr)
        return 1
    except OutOfDeviceMemoryError as exc:
        print(f"out of device memory: {exc}", file=sys.stderr)
        return 1
    except ConvergenceError as exc:
        print(f"did not converge: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
