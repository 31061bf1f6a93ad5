"""1D block-cyclic column layout: placement arithmetic and the permutation
cycle plan, computed by the native planner (csrc/planner.cpp) through the C
ABI.  Same names and semantics as the reference's layout module
(pkg/src/bcmg/layout.py:43-183); execution of a plan happens on the GPU
(:func:`paper_2601_14466_b200.solvers.redistribute_in`).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .core import TileSpec, validate_tile

__all__ = [
    "STAGING_BUFFER_COUNT",
    "ColumnPlacement",
    "ColumnPermutation",
    "RedistributionPlan",
    "device_column_counts",
    "device_column_offsets",
    "map_column",
    "build_permutation",
    "decompose_cycles",
    "invert_plan",
    "serialize_plan",
    "segment_plan_info",
]

# The reference stages one column in each of two host buffers
# (layout.py:38-40); the GPU rotation keeps its staging in registers, one
# 16-byte lane per thread, so this is kept only for API compatibility.
STAGING_BUFFER_COUNT = 2


@dataclass(frozen=True)
class ColumnPlacement:
    device_index: int
    local_column: int


@dataclass(frozen=True)
class ColumnPermutation:
    """dest_of[p] = block-cyclic position of contiguous position p."""

    size: int
    dest_of: np.ndarray

    def is_identity(self) -> bool:
        return bool(np.all(self.dest_of == np.arange(self.size)))


@dataclass(frozen=True)
class RedistributionPlan:
    """Disjoint cycles in rotation order (fixed points omitted)."""

    size: int
    cycles: tuple[tuple[int, ...], ...]
    staging_buffer_count: int = STAGING_BUFFER_COUNT
    staging_buffer_width: int = 1


def _check_grid(n_cols: int, tile: TileSpec, num_devices: int) -> None:
    if num_devices < 1:
        raise ValueError(f"need at least one device, got {num_devices}")
    validate_tile(tile, n_cols)


def device_column_counts(n_cols: int, tile: TileSpec, num_devices: int) -> list[int]:
    """Columns owned by each device (layout.py:82-95)."""
    _check_grid(n_cols, tile, num_devices)
    out = np.zeros(num_devices, dtype=np.int64)
    _lib.check(_lib.load().bcmg_column_counts(n_cols, tile.tile_width, num_devices,
                                               out.ctypes.data_as(_lib._i64p)))
    return [int(x) for x in out]


def device_column_offsets(n_cols: int, tile: TileSpec, num_devices: int) -> list[int]:
    counts = device_column_counts(n_cols, tile, num_devices)
    return [int(x) for x in np.concatenate([[0], np.cumsum(counts)[:-1]])]


def map_column(global_col: int, n_cols: int, tile: TileSpec, num_devices: int) -> ColumnPlacement:
    """Cyclic home of one global column (layout.py:107-123)."""
    _check_grid(n_cols, tile, num_devices)
    if not 0 <= global_col < n_cols:
        raise IndexError(f"column {global_col} out of range for {n_cols} columns")
    w = tile.tile_width
    t = global_col // w
    return ColumnPlacement(t % num_devices, (t // num_devices) * w + global_col % w)


def build_permutation(n_cols: int, tile: TileSpec, num_devices: int) -> ColumnPermutation:
    """Contiguous -> block-cyclic position map (layout.py:126-145)."""
    _check_grid(n_cols, tile, num_devices)
    dest = np.empty(n_cols, dtype=np.int64)
    _lib.check(_lib.load().bcmg_build_permutation(n_cols, tile.tile_width, num_devices,
                                                   dest.ctypes.data_as(_lib._i64p)))
    return ColumnPermutation(size=n_cols, dest_of=dest)


def _unpack(members: np.ndarray, offsets: np.ndarray, nc: int) -> tuple[tuple[int, ...], ...]:
    return tuple(tuple(int(x) for x in members[offsets[c]:offsets[c + 1]]) for c in range(nc))


def decompose_cycles(perm: ColumnPermutation) -> RedistributionPlan:
    """Disjoint cycles, smallest member first, ascending heads (layout.py:148-172)."""
    n = perm.size
    dest = np.ascontiguousarray(perm.dest_of, dtype=np.int64)
    if dest.shape != (n,):
        raise ValueError("dest_of is not a bijection on [0, size)")
    members = np.empty(max(n, 1), dtype=np.int64)
    offsets = np.empty(n + 1, dtype=np.int64)
    nc = C.c_int64(0)
    rc = _lib.load().bcmg_decompose_cycles(n, dest.ctypes.data_as(_lib._i64p), members.ctypes.data_as(_lib._i64p),
                                           offsets.ctypes.data_as(_lib._i64p), C.byref(nc))
    if rc == _lib.BCMG_ERR_CONFIG:
        raise ValueError("dest_of is not a bijection on [0, size)")
    _lib.check(rc)
    return RedistributionPlan(size=n, cycles=_unpack(members, offsets, nc.value))


def invert_plan(plan: RedistributionPlan) -> RedistributionPlan:
    """Inverse permutation: head kept, tail reversed (layout.py:175-183)."""
    lens = [len(c) for c in plan.cycles]
    offsets = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    members = np.array([x for c in plan.cycles for x in c] or [0], dtype=np.int64)
    _lib.check(_lib.load().bcmg_invert_cycles(len(lens), offsets.ctypes.data_as(_lib._i64p),
                                               members.ctypes.data_as(_lib._i64p)))
    return replace(plan, cycles=_unpack(members, offsets, len(lens)))


def serialize_plan(plan: RedistributionPlan) -> str:
    """One cycle per line, comma-separated positions (layout.py:186-188)."""
    return "".join(",".join(str(p) for p in c) + "\n" for c in plan.cycles)


def segment_plan_info(n_cols: int, tile: TileSpec, num_devices: int) -> dict:
    """Segment width S, cycle count and moved columns of the device plan."""
    _check_grid(n_cols, tile, num_devices)
    s, nc, mv = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(_lib.load().bcmg_segment_plan_info(n_cols, tile.tile_width, num_devices, C.byref(s), C.byref(nc),
                                                   C.byref(mv)))
    return {"segment_width": s.value, "n_cycles": nc.value, "moved_columns": mv.value}
