"""B200-native (sm_100a) multi-GPU Cholesky solve path of JAXMg (arXiv 2601.14466).

Public surface, mirroring the reference package ``bcmg`` (pkg/src/bcmg/__init__.py)
for the hot path plus JAXMg's drop-in call:

* ``potrs(A, b, T_A=, mesh=, in_specs=)`` / ``potri(A, T_A=, mesh=, in_specs=)``
* ``solve_positive_definite`` / ``invert_positive_definite`` (host arrays)
* ``potrf`` / ``potrs_factored`` (``solvers.potrs``) / ``solvers.potri`` on
  ``DistributedMatrix`` shards, ``redistribute_in`` / ``redistribute_out``
* layout planning: ``build_permutation``, ``decompose_cycles``, ``invert_plan``...

All compute runs in ``lib/libbcmg_b200.so`` (hand-written CUDA for sm_100a).
"""

from .core import (
    ConcurrentCallError,
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
from .layout import (
    STAGING_BUFFER_COUNT,
    ColumnPermutation,
    ColumnPlacement,
    RedistributionPlan,
    build_permutation,
    decompose_cycles,
    device_column_counts,
    device_column_offsets,
    invert_plan,
    map_column,
    segment_plan_info,
    serialize_plan,
)
from .mesh import DeviceMesh
from .solvers import (
    DistributedMatrix,
    FactorizationResult,
    Timings,
    create_distributed,
    eigh_hermitian,
    gather_array,
    invert_positive_definite,
    potrf,
    redistribute_in,
    redistribute_out,
    solve_positive_definite,
    workspace_nbytes,
    write_array,
)
from .solvers import potri as potri_factored
from .solvers import potrs as potrs_factored
from .solvers import syevd as syevd_cyclic
from .api import P, last_timings, make_mesh, potri, potrs, syevd

__all__ = [
    "ConcurrentCallError", "ConvergenceError", "DescriptorError", "ElementType", "MatrixDescriptor", "NotPositiveDefiniteError",
    "OutOfDeviceMemoryError", "RhsDescriptor", "StaleSessionError", "Structure", "TileSpec",
    "validate_descriptor", "validate_tile",
    "STAGING_BUFFER_COUNT", "ColumnPermutation", "ColumnPlacement", "RedistributionPlan", "build_permutation",
    "decompose_cycles", "device_column_counts", "device_column_offsets", "invert_plan", "map_column",
    "segment_plan_info", "serialize_plan",
    "DeviceMesh", "DistributedMatrix", "FactorizationResult", "Timings", "create_distributed", "gather_array",
    "invert_positive_definite", "potrf", "potrs_factored", "potri_factored", "redistribute_in", "redistribute_out",
    "solve_positive_definite", "syevd_cyclic", "eigh_hermitian", "workspace_nbytes", "write_array",
    "P", "make_mesh", "potrs", "potri", "syevd", "last_timings",
]
