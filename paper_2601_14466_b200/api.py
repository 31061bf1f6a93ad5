"""Drop-in frontend with JAXMg's call surface (reference PAPER.md:88-101):

    mesh = make_mesh(num_devices, ("x",))
    x = potrs(A, b, T_A=T_A, mesh=mesh, in_specs=(P("x", None), P(None, None)))
    Ainv = potri(A, T_A=T_A, mesh=mesh, in_specs=(P("x", None),))

``A`` is row-sharded over the mesh axis (JAX ``P("x", None)``): with one
process it is the whole N x N matrix (a CUDA torch tensor, or a host array
that is uploaded); with torchrun it is this rank's N/world x N row block on
its GPU.  ``b`` (N x N_RHS) is replicated.  Row blocks of a row-major matrix
are the column blocks of A^T, i.e. of A for real symmetric input and of
conj(A) for complex Hermitian input -- the native pipeline is told so
(BCMG_FLAG_ROW_SHARDED) and solves conj(A) conj(x) = conj(b).

Unlike JAX arrays torch tensors are mutable: by default A is copied before
being factored in place (``overwrite_a=False``, the reference never mutates
caller input); ``overwrite_a=True`` donates A's storage, which
is what lets N = 131072 float64 (137 GB) run on one 180 GB B200.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .core import DescriptorError, ElementType, TileSpec, validate_tile
from .layout import device_column_counts
from .mesh import DeviceMesh
from .solvers import _raise_for

__all__ = ["P", "make_mesh", "potrs", "potri", "last_timings"]


class P(tuple):
    """PartitionSpec stand-in: ``P("x", None)`` shards dim 0 over axis "x"."""

    def __new__(cls, *axes):
        return super().__new__(cls, axes)

    def __repr__(self) -> str:
        return "P(" + ", ".join(repr(a) for a in self) + ")"


ROW_SHARDED = P("x", None)
REPLICATED = P(None, None)


def make_mesh(num_devices: int | None = None, axis_names=("x",), device: int | None = None) -> DeviceMesh:
    """1D mesh of ``num_devices`` logical devices (default: one per process).
    With one process and num_devices > 1 the devices are virtual devices on
    the process's GPU."""
    if tuple(axis_names) != ("x",) and len(tuple(axis_names)) != 1:
        raise ValueError("only 1D meshes are supported (the reference has no 2D grids, SPEC.md:185)")
    mesh = DeviceMesh(num_devices, device=device)
    mesh.axis_names = tuple(axis_names)
    return mesh


def _check_specs(in_specs, mesh: DeviceMesh, n_inputs: int):
    if in_specs is None:
        return
    specs = tuple(in_specs)
    axis = getattr(mesh, "axis_names", ("x",))[0]
    if len(specs) < 1 or tuple(specs[0]) != (axis, None):
        raise DescriptorError("dimension-mismatch", f"A must be row-sharded P({axis!r}, None), got {specs[0]!r}")
    if n_inputs > 1 and len(specs) > 1 and tuple(specs[1]) != (None, None):
        raise DescriptorError("dimension-mismatch", f"b must be replicated P(None, None), got {specs[1]!r}")


def _prepare_a(A, mesh: DeviceMesh, overwrite_a: bool):
    import torch

    if isinstance(A, np.ndarray):
        A = torch.from_numpy(np.ascontiguousarray(A))
    if not isinstance(A, torch.Tensor) or A.ndim != 2:
        raise DescriptorError("dimension-mismatch", "A must be a 2-D array")
    et = ElementType.from_dtype(A.dtype)
    rows, n = int(A.shape[0]), int(A.shape[1])
    if rows * mesh.world != n:
        raise DescriptorError("dimension-mismatch",
                              f"row shard {rows}x{n} does not tile an {n}x{n} matrix over {mesh.world} processes")
    dev = mesh.torch_device
    if A.device != dev or not A.is_contiguous():
        A = A.to(dev).contiguous()  # a copy: caller storage untouched
    elif not overwrite_a:
        A = A.clone()
    return A, et, n


def _shard_ptrs(A, mesh: DeviceMesh, n: int, tile: int, esz: int):
    counts = device_column_counts(n, TileSpec(tile), mesh.num_devices)
    local = [counts[d] for d in mesh.local_devices]
    # this process's logical devices together hold exactly its row block (N / world
    # columns of the symmetric A); a mesh may put several logical devices on a process
    if mesh.world > 1 and sum(local) * mesh.world != n:
        raise DescriptorError("dimension-mismatch",
                              f"row shards of N/{mesh.world} need N % (T_A * devices) == 0 (N={n}, T_A={tile})")
    base, ptrs, off = A.data_ptr(), [], 0
    for c in local:
        ptrs.append(base + off * n * esz)
        off += c
    return _lib.ptr_array(ptrs)


def potrs(A, b, T_A: int, mesh: DeviceMesh | None = None, in_specs=None, *, overwrite_a: bool = False):
    """Solve A x = b for Hermitian positive-definite A (cusolverMgPotrs
    semantics).  Returns x shaped like b, on A's device."""
    import torch

    mesh = mesh or make_mesh()
    _check_specs(in_specs, mesh, 2)
    # pinned host A on one device: stream it in while the factorisation starts
    # (bcmg_potrs_streamed) instead of uploading it first
    host_src = None
    if (isinstance(A, torch.Tensor) and A.device.type == "cpu" and A.is_pinned() and A.is_contiguous()
            and A.ndim == 2 and mesh.num_devices == 1 and mesh.world == 1):
        host_src = A
        et = ElementType.from_dtype(A.dtype)
        n = int(A.shape[1])
        if int(A.shape[0]) != n:
            raise DescriptorError("dimension-mismatch", f"row shard {tuple(A.shape)} does not tile an {n}x{n} matrix")
        A = torch.empty((n, n), dtype=A.dtype, device=mesh.torch_device)
    else:
        A, et, n = _prepare_a(A, mesh, overwrite_a)
    validate_tile(TileSpec(int(T_A)), n)
    if isinstance(b, np.ndarray):
        b = torch.from_numpy(np.ascontiguousarray(b))
    if b.is_complex() and not et.is_complex:
        raise DescriptorError("type-structure", "complex right-hand side with a real matrix")
    one_dim = b.ndim == 1
    b2 = b.reshape(-1, 1) if one_dim else b
    if b2.ndim != 2 or int(b2.shape[0]) != n:
        raise DescriptorError("dimension-mismatch", f"right-hand side shape {tuple(b.shape)} does not match n={n}")
    nrhs = int(b2.shape[1])
    # column-major RHS on the device (n x nrhs, ld n)
    # a fresh buffer: b2.t().contiguous() would alias the caller's b when N_RHS == 1
    x = torch.empty((nrhs, n), dtype=et.torch_dtype, device=mesh.torch_device)
    x.copy_(b2.t())
    info = C.c_int(0)
    with mesh.coordinated():
        if host_src is not None:
            rc = _lib.load().bcmg_potrs_streamed(mesh.session, mesh.stream_handle(), et.code, n, nrhs, int(T_A),
                                                 C.c_void_p(A.data_ptr()), C.c_void_p(host_src.data_ptr()),
                                                 C.c_void_p(x.data_ptr()), n, _lib.BCMG_FLAG_ROW_SHARDED,
                                                 C.byref(info))
        else:
            rc = _lib.load().bcmg_potrs(mesh.session, mesh.stream_handle(), et.code, n, nrhs, int(T_A),
                                        mesh.num_devices, _shard_ptrs(A, mesh, n, int(T_A), et.width),
                                        C.c_void_p(x.data_ptr()), n, _lib.BCMG_FLAG_ROW_SHARDED, C.byref(info))
    _raise_for(rc, info.value)
    out = x.t()
    return out.reshape(-1) if one_dim else out


def potri(A, T_A: int, mesh: DeviceMesh | None = None, in_specs=None, *, overwrite_a: bool = False):
    """Inverse of a Hermitian positive-definite matrix (cusolverMgPotri),
    returned with A's row sharding."""
    mesh = mesh or make_mesh()
    _check_specs(in_specs, mesh, 1)
    A, et, n = _prepare_a(A, mesh, overwrite_a)
    validate_tile(TileSpec(int(T_A)), n)
    info = C.c_int(0)
    with mesh.coordinated():
        rc = _lib.load().bcmg_potri(mesh.session, mesh.stream_handle(), et.code, n, int(T_A), mesh.num_devices,
                                    _shard_ptrs(A, mesh, n, int(T_A), et.width), _lib.BCMG_FLAG_ROW_SHARDED,
                                    C.byref(info))
    _raise_for(rc, info.value)
    return A


def syevd(A, T_A: int, mesh: DeviceMesh | None = None, in_specs=None, *, return_eigenvectors: bool = True,
          overwrite_a: bool = False):
    """Eigenvalues (ascending) and eigenvectors of a Hermitian matrix
    (cusolverMgSyevd semantics; reference eigh_hermitian,
    solvers.py:1019-1043).  Returns (w, V) -- or w alone -- on A's device; V is
    row-major with V[:, j] the eigenvector of w[j], its first largest-magnitude
    component real and positive.  Single-process meshes.

    The row-major buffer of A is the column-major conj(A) (Hermitian), so the
    native call computes the eigenvectors of conj(A), which are conj(V) under
    the same phase convention; V is that buffer conjugate-transposed."""
    import torch

    mesh = mesh or make_mesh()
    _check_specs(in_specs, mesh, 1)
    if mesh.world != 1:  # (solvers.eigh_hermitian / bcmg_syevd run across processes: DESIGN.md §3b)
        raise DescriptorError("dimension-mismatch", "the drop-in syevd returns row-major V from one process; "
                                                    "use eigh_hermitian(mesh, a, tile) across processes")
    A, et, n = _prepare_a(A, mesh, overwrite_a)
    validate_tile(TileSpec(int(T_A)), n)
    real = torch.float32 if et in (ElementType.real32, ElementType.complex64) else torch.float64
    w = torch.empty(n, dtype=real, device=mesh.torch_device)
    info = C.c_int(0)
    with mesh.coordinated():
        rc = _lib.load().bcmg_syevd(mesh.session, mesh.stream_handle(), et.code, n, int(T_A), mesh.num_devices,
                                    _shard_ptrs(A, mesh, n, int(T_A), et.width), C.c_void_p(w.data_ptr()), 0,
                                    C.byref(info))
    _raise_for(rc, info.value)
    if not return_eigenvectors:
        return w
    V = A.t().conj() if et.is_complex else A.t()
    return w, V.contiguous().resolve_conj()


def last_timings(mesh: DeviceMesh) -> dict:
    """Device-side phase split (ms) of the last potrs/potri on ``mesh``."""
    ms = (C.c_float * 4)()
    _lib.check(_lib.load().bcmg_last_timings(mesh.session, ms))
    return {"redistribute_ms": ms[0], "potrf_ms": ms[1], "finish_ms": ms[2], "total_ms": ms[3]}
