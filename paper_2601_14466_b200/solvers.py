"""Distributed Cholesky solve / inverse on B200 -- the reference's solver API
(pkg/src/bcmg/solvers.py) over GPU shards and the native C ABI.

Every routine here is a thin host shim: it validates arguments exactly like
the reference, lays out device memory (torch is used only as the device
allocator) and calls ``libbcmg_b200.so``.  There is no CPU compute path; if
the library or a GPU is missing the calls fail.

Layout of a :class:`DistributedMatrix`: one flat device buffer per process
holding its logical devices' shards back to back; shard ``d`` is
``n_rows x counts[d]`` column-major (leading dimension ``n_rows``), exactly
the reference's per-device arena content (solvers.py:87-103).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, replace
from typing import Sequence

import numpy as np

from . import _lib
from .core import (
    ConvergenceError,
    DescriptorError,
    ElementType,
    MatrixDescriptor,
    NotPositiveDefiniteError,
    OutOfDeviceMemoryError,
    RhsDescriptor,
    StaleSessionError,
    Structure,
    TileSpec,
    validate_descriptor,
    validate_tile,
)
from .layout import device_column_counts
from .mesh import DeviceMesh

__all__ = [
    "DistributedMatrix",
    "FactorizationResult",
    "Timings",
    "create_distributed",
    "free_distributed",
    "write_array",
    "gather_array",
    "redistribute_in",
    "redistribute_out",
    "workspace_nbytes",
    "allocate_panel_workspace",
    "potrf",
    "potrs",
    "potri",
    "solve_positive_definite",
    "invert_positive_definite",
    "syevd",
    "eigh_hermitian",
]


@dataclass(frozen=True)
class DistributedMatrix:
    """Column tiles of a matrix over the mesh's logical devices.

    ``buffer`` is this process's flat device buffer; ``shards`` are views of
    it, one per local logical device.  ``layout`` is ``"contiguous"`` or
    ``"block_cyclic"`` (solvers.py:87-103)."""

    descriptor: MatrixDescriptor
    tile: TileSpec
    counts: tuple[int, ...]
    buffer: object  # torch.Tensor, flat
    shards: tuple  # torch.Tensor views
    layout: str = "contiguous"
    num_devices: int = 1

    def shard_ptrs(self):
        return _lib.ptr_array([s.data_ptr() for s in self.shards])


@dataclass(frozen=True)
class FactorizationResult:
    """potrf outcome with LAPACK info semantics (solvers.py:106-116)."""

    factor: DistributedMatrix
    info: int


@dataclass(frozen=True)
class Timings:
    """Wall-clock split (solvers.py:119-128) plus the device-side phase split
    measured with CUDA events inside the native pipeline."""

    alloc_seconds: float
    solve_seconds: float
    redistribute_ms: float = 0.0
    potrf_ms: float = 0.0
    finish_ms: float = 0.0
    device_ms: float = 0.0


def _torch():
    import torch

    return torch


def _raise_for(rc: int, info: int | None = None) -> None:
    if rc == _lib.BCMG_OK:
        return
    code, msg = _lib.last_error()
    if rc == _lib.BCMG_ERR_NOT_POSITIVE_DEFINITE:
        raise NotPositiveDefiniteError(int(info or 0))
    if rc == _lib.BCMG_ERR_OUT_OF_MEMORY:
        raise OutOfDeviceMemoryError(msg)
    if rc == _lib.BCMG_ERR_CONFIG:
        raise DescriptorError("dimension-mismatch", msg)
    if rc == _lib.BCMG_ERR_NO_CONVERGENCE:
        raise ConvergenceError(msg)
    if rc == _lib.BCMG_ERR_STALE_SESSION:
        raise StaleSessionError(msg)
    raise _lib.BcmgError(rc, msg)


def _require_layout(dmat: DistributedMatrix, layout: str) -> None:
    if dmat.layout != layout:
        raise ValueError(f"expected {layout} layout, matrix is {dmat.layout}")


# -- distribution ---------------------------------------------------------


def create_distributed(mesh: DeviceMesh, desc: MatrixDescriptor, tile: TileSpec) -> DistributedMatrix:
    """Allocate this process's shards (one flat device buffer)."""
    validate_descriptor(desc)
    validate_tile(tile, desc.n_cols)
    torch = _torch()
    counts = tuple(device_column_counts(desc.n_cols, tile, mesh.num_devices))
    local = [counts[d] for d in mesh.local_devices]
    n = desc.n_rows
    try:
        buf = torch.empty(n * sum(local), dtype=desc.element_type.torch_dtype, device=mesh.torch_device)
    except torch.cuda.OutOfMemoryError as exc:
        raise OutOfDeviceMemoryError(str(exc)) from None
    shards, off = [], 0
    for c in local:
        shards.append(buf[off * n:(off + c) * n])
        off += c
    return DistributedMatrix(desc, tile, counts, buf, tuple(shards), "contiguous", mesh.num_devices)


def free_distributed(mesh: DeviceMesh, dmat: DistributedMatrix) -> None:
    """Storage is reference-counted by torch; kept for API parity."""
    return None


def _local_col_range(mesh: DeviceMesh, dmat: DistributedMatrix) -> tuple[int, int]:
    first = sum(dmat.counts[: mesh.local_devices[0]])
    return first, first + sum(dmat.counts[d] for d in mesh.local_devices)


def write_array(mesh: DeviceMesh, dmat: DistributedMatrix, array) -> None:
    """Load a global host (numpy) or torch matrix into a contiguous-layout
    matrix; each process writes the columns of its logical devices
    (solvers.py:212-225)."""
    _require_layout(dmat, "contiguous")
    torch = _torch()
    desc = dmat.descriptor
    if tuple(array.shape) != desc.shape:
        raise DescriptorError("dimension-mismatch",
                              f"array shape {tuple(array.shape)} does not match descriptor {desc.shape}")
    c0, c1 = _local_col_range(mesh, dmat)
    if isinstance(array, np.ndarray):
        cols = np.asfortranarray(array[:, c0:c1], dtype=desc.element_type.dtype)
        host = torch.from_numpy(cols.ravel(order="F"))
        dmat.buffer.copy_(host.to(dmat.buffer.device, non_blocking=False))
    else:
        t = array.to(device=dmat.buffer.device, dtype=dmat.buffer.dtype)
        dmat.buffer.copy_(t[:, c0:c1].t().contiguous().reshape(-1))


def gather_array(mesh: DeviceMesh, dmat: DistributedMatrix) -> np.ndarray:
    """Contiguous-layout matrix back to the host (solvers.py:228-241)."""
    _require_layout(dmat, "contiguous")
    desc = dmat.descriptor
    flat = dmat.buffer.cpu().numpy()
    local = flat.reshape((desc.n_rows, -1), order="F")
    if mesh.world == 1:
        return np.asfortranarray(local)
    torch = _torch()
    parts = [None] * mesh.world
    torch.distributed.all_gather_object(parts, local)
    return np.asfortranarray(np.hstack(parts))


def device_concat(mesh: DeviceMesh, dmat: DistributedMatrix) -> np.ndarray:
    """Shard contents side by side in device order, whatever the layout."""
    desc = dmat.descriptor
    return np.asfortranarray(dmat.buffer.cpu().numpy().reshape((desc.n_rows, -1), order="F"))


def _redistribute(mesh: DeviceMesh, dmat: DistributedMatrix, direction: int) -> DistributedMatrix:
    desc = dmat.descriptor
    with mesh.coordinated():
        rc = _lib.load().bcmg_redistribute(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows,
                                           desc.n_cols, dmat.tile.tile_width, mesh.num_devices, dmat.shard_ptrs(),
                                           direction)
    _raise_for(rc)
    return dmat


def redistribute_in(mesh: DeviceMesh, dmat: DistributedMatrix) -> DistributedMatrix:
    """Contiguous -> block-cyclic, in place on the GPU (solvers.py:262-266)."""
    _require_layout(dmat, "contiguous")
    _redistribute(mesh, dmat, _lib.BCMG_TO_CYCLIC)
    return replace(dmat, layout="block_cyclic")


def redistribute_out(mesh: DeviceMesh, dmat: DistributedMatrix) -> DistributedMatrix:
    """Block-cyclic -> contiguous, in place (solvers.py:269-273)."""
    _require_layout(dmat, "block_cyclic")
    _redistribute(mesh, dmat, _lib.BCMG_TO_CONTIG)
    return replace(dmat, layout="contiguous")


# -- workspace ------------------------------------------------------------


def workspace_nbytes(routine: str, desc: MatrixDescriptor, tile: TileSpec, num_devices: int, n_rhs: int = 1,
                     world: int = 1) -> list[int]:
    """Device bytes per logical device incl. shards (solvers.py:279-308).

    potrs / potri: the shard plus the process's workspace, which the native
    pipelines reserve in full before moving any data (so out-of-memory leaves
    the shards untouched) and charge here to the first logical device of each
    process.  The workspace figure is the native plan itself
    (``bcmg_workspace_nbytes``, csrc/solver.cu ``workspace_plan``): two
    panels (the complex128 [P | -iP] embedding doubles them and adds a planar
    copy), tf32 hi / lo split planes for real32 / complex64, the complex
    embedding scratch, the diagonal-block inverses, split-K slabs and the
    hand-off buffer (potrs), the W-tile / gather buffers (potri)."""
    esz = desc.element_type.width
    et = desc.element_type
    n, T = desc.n_rows, tile.tile_width
    counts = device_column_counts(desc.n_cols, tile, num_devices)
    if routine in ("potrs", "potri"):
        if num_devices % world:
            raise ValueError("logical devices must be a multiple of the processes")
        nb = C.c_int64(0)
        _lib.check(_lib.load().bcmg_workspace_nbytes(1 if routine == "potrs" else 2, et.code, n, T, num_devices,
                                                     world, max(1, n_rhs), C.byref(nb)))
        per = num_devices // world
        return [c * desc.column_nbytes + (nb.value if d % per == 0 else 0) for d, c in enumerate(counts)]
    if routine == "syevd":
        # csrc/eigen.cu: dense working copy, the eigenvector matrix V (Q, then
        # Q times the QL rotations), U | W panels, symv partials, WY blocks, vectors, the rotation
        # ring -- one GPU holds it all, so it is charged to logical device 0
        cs = 16 if et.is_complex else 8
        nb = -(-n // 64)
        eig = (2 * n * n * cs + 2 * n * T * cs + 2 * nb * n * cs + 2 * 256 * 256 * cs
               + 2 * 256 * n * cs + (3 * n + 2 * T) * cs + 3 * n * 8 + n * 8 + (n // 8 + 2) * 24
               + 8 * (64 * n * 16 + 129 * 8))
        return [c * desc.column_nbytes + (eig if d == 0 else 0) for d, c in enumerate(counts)]
    raise ValueError(f"unknown routine {routine!r}")


def allocate_panel_workspace(mesh: DeviceMesh, desc: MatrixDescriptor, tile: TileSpec) -> list:
    """Panels are owned by the native session (grow-only, reused across
    calls); kept for API parity with solvers.py:311-316."""
    return []


# -- factorisation and solves ---------------------------------------------


def potrf(mesh: DeviceMesh, dmat: DistributedMatrix, panel_workspace: Sequence = ()) -> FactorizationResult:
    """Tiled right-looking Cholesky on the GPU; info is returned, not raised
    (solvers.py:341-406)."""
    _require_layout(dmat, "block_cyclic")
    desc = dmat.descriptor
    if desc.structure is not Structure.positive_definite:
        raise DescriptorError("type-structure",
                              f"potrf requires positive_definite structure, got {desc.structure.name}")
    info = C.c_int(0)
    with mesh.coordinated():
        rc = _lib.load().bcmg_potrf(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows,
                                    dmat.tile.tile_width, mesh.num_devices, dmat.shard_ptrs(), C.byref(info))
    _raise_for(rc)
    return FactorizationResult(dmat, int(info.value))


def potrs(mesh: DeviceMesh, factored: DistributedMatrix, rhs_replicas: Sequence, n_rhs: int | None = None) -> None:
    """Solve L L^H x = b on the factor; every replica (a device tensor holding
    the n x n_rhs column-major RHS) is overwritten with x (solvers.py:430-474)."""
    _require_layout(factored, "block_cyclic")
    desc = factored.descriptor
    first = rhs_replicas[0]
    n_rhs = n_rhs or first.numel() // desc.n_rows
    with mesh.coordinated():
        rc = _lib.load().bcmg_potrs_factored(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows,
                                             n_rhs, factored.tile.tile_width, mesh.num_devices, factored.shard_ptrs(),
                                             C.c_void_p(first.data_ptr()), desc.n_rows)
    _raise_for(rc)
    for r in rhs_replicas[1:]:
        r.copy_(first)


def potri(mesh: DeviceMesh, factored: DistributedMatrix, panel_workspace: Sequence = (),
          acc_workspace: Sequence = ()) -> DistributedMatrix:
    """Full Hermitian inverse from the factor, in place (solvers.py:487-594)."""
    _require_layout(factored, "block_cyclic")
    desc = factored.descriptor
    with mesh.coordinated():
        rc = _lib.load().bcmg_potri_factored(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows,
                                             factored.tile.tile_width, mesh.num_devices, factored.shard_ptrs())
    _raise_for(rc)
    return factored


# -- end-to-end pipelines ----------------------------------------------------


def _matrix_descriptor(a, structure: Structure) -> MatrixDescriptor:
    if len(a.shape) != 2:
        raise DescriptorError("dimension-mismatch", f"expected a 2-D matrix, got ndim={len(a.shape)}")
    et = ElementType.from_dtype(a.dtype)
    desc = MatrixDescriptor(int(a.shape[0]), int(a.shape[1]), et, structure)
    validate_descriptor(desc)
    return desc


def _timings(mesh: DeviceMesh, t0: float, t1: float, t2: float) -> Timings:
    ms = (C.c_float * 4)()
    _lib.check(_lib.load().bcmg_last_timings(mesh.session, ms))
    return Timings(t1 - t0, t2 - t1, float(ms[0]), float(ms[1]), float(ms[2]), float(ms[3]))


def solve_positive_definite(mesh: DeviceMesh, a: np.ndarray, b: np.ndarray, tile: TileSpec):
    """Factor A and solve A x = b; host arrays in, host array out
    (solvers.py:931-985).  Returns (x, Timings)."""
    desc = _matrix_descriptor(a, Structure.positive_definite)
    validate_tile(tile, desc.n_cols)
    if np.iscomplexobj(b) and not desc.element_type.is_complex:
        raise DescriptorError("type-structure", "complex right-hand side with a real matrix")
    b_arr = np.asfortranarray(b, dtype=desc.element_type.dtype)
    one_dim = b_arr.ndim == 1
    if one_dim:
        b_arr = b_arr.reshape(-1, 1)
    if b_arr.ndim != 2 or b_arr.shape[0] != desc.n_rows:
        raise DescriptorError("dimension-mismatch",
                              f"right-hand side shape {np.shape(b)} does not match a {desc.n_rows}-row matrix")
    n_rhs = b_arr.shape[1]
    RhsDescriptor(b_arr.shape[0], n_rhs, desc.element_type)
    torch = _torch()

    def body():
        t0 = time.perf_counter()
        dmat = create_distributed(mesh, desc, tile)
        try:
            xdev = torch.empty(desc.n_rows * n_rhs, dtype=desc.element_type.torch_dtype, device=mesh.torch_device)
        except torch.cuda.OutOfMemoryError as exc:
            raise OutOfDeviceMemoryError(str(exc)) from None
        t1 = time.perf_counter()
        write_array(mesh, dmat, a)
        xdev.copy_(torch.from_numpy(b_arr.ravel(order="F")).to(mesh.torch_device))
        info = C.c_int(0)
        rc = _lib.load().bcmg_potrs(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows, n_rhs,
                                    tile.tile_width, mesh.num_devices, dmat.shard_ptrs(), C.c_void_p(xdev.data_ptr()),
                                    desc.n_rows, 0, C.byref(info))
        _raise_for(rc, info.value)
        x = xdev.cpu().numpy().reshape((desc.n_rows, n_rhs), order="F")
        t2 = time.perf_counter()
        return np.asfortranarray(x), _timings(mesh, t0, t1, t2)

    x, timings = mesh.run_coordinated(body)
    return (x[:, 0] if one_dim else x), timings


def invert_positive_definite(mesh: DeviceMesh, a: np.ndarray, tile: TileSpec):
    """Full inverse of a positive-definite matrix, both triangles filled
    (solvers.py:988-1016).  Returns (inverse, Timings)."""
    desc = _matrix_descriptor(a, Structure.positive_definite)
    validate_tile(tile, desc.n_cols)

    def body():
        t0 = time.perf_counter()
        dmat = create_distributed(mesh, desc, tile)
        t1 = time.perf_counter()
        write_array(mesh, dmat, a)
        info = C.c_int(0)
        rc = _lib.load().bcmg_potri(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows,
                                    tile.tile_width, mesh.num_devices, dmat.shard_ptrs(), 0, C.byref(info))
        _raise_for(rc, info.value)
        inv = gather_array(mesh, dmat)
        t2 = time.perf_counter()
        return inv, _timings(mesh, t0, t1, t2)

    return mesh.run_coordinated(body)


# -- Hermitian eigendecomposition ----------------------------------------------


def _real_torch_dtype(et: ElementType):
    torch = _torch()
    return torch.float32 if et in (ElementType.real32, ElementType.complex64) else torch.float64


def _require_hermitian(desc: MatrixDescriptor) -> None:
    if desc.structure is Structure.general:
        raise DescriptorError("type-structure", "eigendecomposition requires symmetric, hermitian or "
                                                "positive_definite structure")
    if desc.n_rows != desc.n_cols:
        raise DescriptorError("dimension-mismatch", f"matrix must be square, got {desc.n_rows}x{desc.n_cols}")


def syevd(mesh: DeviceMesh, dmat: DistributedMatrix, ws: Sequence = ()) -> tuple[np.ndarray, DistributedMatrix]:
    """Eigenvalues (ascending, host array of the real type) and eigenvectors of
    a Hermitian matrix on the block-cyclic layout; the eigenvectors overwrite
    the shards, column j of the cyclic layout belonging to w[j], each scaled so
    its first largest-magnitude component is real and positive
    (solvers.py:862-910).  Across processes the matrix is gathered and solved
    on rank 0 (csrc/eigen.cu)."""
    _require_layout(dmat, "block_cyclic")
    desc = dmat.descriptor
    _require_hermitian(desc)
    torch = _torch()
    w = torch.empty(desc.n_rows, dtype=_real_torch_dtype(desc.element_type), device=mesh.device)
    with mesh.coordinated():
        rc = _lib.load().bcmg_syevd_cyclic(mesh.session, mesh.stream_handle(), desc.element_type.code, desc.n_rows,
                                           dmat.tile.tile_width, mesh.num_devices, dmat.shard_ptrs(),
                                           C.c_void_p(w.data_ptr()))
    _raise_for(rc)
    return w.cpu().numpy(), dmat


def _hermitian_structure(et: ElementType) -> Structure:
    return Structure.hermitian if et.is_complex else Structure.symmetric


def eigh_hermitian(mesh: DeviceMesh, a: np.ndarray, tile: TileSpec):
    """Ascending eigenvalues and eigenvectors of a Hermitian matrix; host
    array in, (w, v, Timings) out (solvers.py:1019-1043).  The native pipeline
    gathers the working copy straight from the contiguous shards and scatters
    the eigenvectors straight back, so redistribute_in / _out fold into it."""
    et = ElementType.from_dtype(np.asarray(a).dtype)
    desc = _matrix_descriptor(a, _hermitian_structure(et))
    _require_hermitian(desc)
    validate_tile(tile, desc.n_cols)
    torch = _torch()

    def body():
        t0 = time.perf_counter()
        dmat = create_distributed(mesh, desc, tile)
        w = torch.empty(desc.n_rows, dtype=_real_torch_dtype(et), device=mesh.device)
        t1 = time.perf_counter()
        write_array(mesh, dmat, a)
        info = C.c_int(0)
        rc = _lib.load().bcmg_syevd(mesh.session, mesh.stream_handle(), et.code, desc.n_rows, tile.tile_width,
                                    mesh.num_devices, dmat.shard_ptrs(), C.c_void_p(w.data_ptr()), 0,
                                    C.byref(info))
        _raise_for(rc, info.value)
        v = gather_array(mesh, dmat)
        wh = w.cpu().numpy()
        t2 = time.perf_counter()
        return wh, v, _timings(mesh, t0, t1, t2)

    return mesh.run_coordinated(body)
