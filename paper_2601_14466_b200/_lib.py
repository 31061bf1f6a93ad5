"""ctypes binding of libbcmg_b200.so (the C ABI declared in include/bcmg_b200.h).

The library is built in-tree (``__graft_entry__.build()`` ->
``paper_2601_14466_b200/csrc/Makefile``).  There is no fallback: if the
shared object is missing or a symbol is absent, importing the solvers fails
loudly with :class:`LibraryMissingError`.
"""

from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("BCMG_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                           "libbcmg_b200.so")

# Stable error codes (reference pkg/frontend/src/errors.ts:9-23) + CUDA.
BCMG_OK = 0
BCMG_ERR_NOT_POSITIVE_DEFINITE = 1
BCMG_ERR_CONFIG = 2
BCMG_ERR_NO_CONVERGENCE = 3
BCMG_ERR_OUT_OF_MEMORY = 4
BCMG_ERR_CHECK_FAILED = 5
BCMG_ERR_STALE_SESSION = 6
BCMG_ERR_IO = 7
BCMG_ERR_CUDA = 8

BCMG_TO_CYCLIC = 0
BCMG_TO_CONTIG = 1
BCMG_FLAG_ROW_SHARDED = 1

_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p
_vpp = C.POINTER(C.c_void_p)
_ip = C.POINTER(C.c_int)

# symbol -> (restype, argtypes); must match include/bcmg_b200.h exactly
SIGNATURES = {
    "bcmg_version": (C.c_int, []),
    "bcmg_last_error": (C.c_int, []),
    "bcmg_last_error_message": (C.c_char_p, []),
    "bcmg_column_counts": (C.c_int, [_i64, _i64, C.c_int, _i64p]),
    "bcmg_build_permutation": (C.c_int, [_i64, _i64, C.c_int, _i64p]),
    "bcmg_decompose_cycles": (C.c_int, [_i64, _i64p, _i64p, _i64p, _i64p]),
    "bcmg_invert_cycles": (C.c_int, [_i64, _i64p, _i64p]),
    "bcmg_segment_plan_info": (C.c_int, [_i64, _i64, C.c_int, _i64p, _i64p, _i64p]),
    "bcmg_schedule": (C.c_int, [C.c_int, _i64, _i64, C.c_int, C.c_int, C.c_int, _i64, _i64p, _i64, _i64p]),
    "bcmg_redistribute_plan": (C.c_int, [_i64, _i64, C.c_int, C.c_int, C.c_int, _i64p, _i64p, _i64, _i64p]),
    "bcmg_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "bcmg_open": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
    "bcmg_close": (C.c_int, [_vp]),
    "bcmg_potrs": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, _i64, C.c_int, _vpp, _vp, _i64, C.c_int, _ip]),
    "bcmg_potri": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, C.c_int, _vpp, C.c_int, _ip]),
    "bcmg_syevd": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, C.c_int, _vpp, _vp, C.c_int, _ip]),
    "bcmg_syevd_cyclic": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, C.c_int, _vpp, _vp]),
    "bcmg_potrs_streamed": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _i64, C.c_int, _ip]),
    "bcmg_redistribute": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, _i64, C.c_int, _vpp, C.c_int]),
    "bcmg_potrf": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, C.c_int, _vpp, _ip]),
    "bcmg_potrs_factored": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, _i64, C.c_int, _vpp, _vp, _i64]),
    "bcmg_potri_factored": (C.c_int, [_vp, _vp, C.c_int, _i64, _i64, C.c_int, _vpp]),
    "bcmg_gemm": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, C.c_double, _vp, _i64, C.c_int, _vp, _i64, C.c_int,
                            C.c_double, _vp, _i64]),
    "bcmg_last_timings": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "bcmg_last_moved_bytes": (C.c_int64, [_vp]),
    "bcmg_workspace_nbytes": (C.c_int, [C.c_int, C.c_int, _i64, _i64, C.c_int, C.c_int, _i64, _i64p]),
    "bcmg_session_workspace_bytes": (C.c_int, [_vp, _i64p]),
    "bcmg_ipc_export": (C.c_int, [_vp, C.c_char_p]),
    "bcmg_ipc_open": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "bcmg_ipc_close_all": (C.c_int, []),
    "bcmg_stream_write_flag": (C.c_int, [_vp, _vp, C.c_uint]),
    "bcmg_stream_wait_flag": (C.c_int, [_vp, _vp, C.c_uint]),
    "bcmg_set_profiling": (C.c_int, [_vp, C.c_int]),
    "bcmg_kernel_stats": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double)]),
    "bcmg_launch_count": (C.c_int64, []),
    "bcmg_measure_fp64_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "bcmg_loopback_id": (C.c_int, [C.c_char_p]),
    "bcmg_generate_spd": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, _i64, C.c_uint64, C.c_double]),
}

KERNEL_KINDS = {"trailing_update": 0, "panel_trsm": 1, "diag_factor": 2, "rotate": 3}


class LibraryMissingError(ImportError):
    """libbcmg_b200.so is absent or incomplete: run __graft_entry__.build()."""


class BcmgError(RuntimeError):
    """A non-zero return code from the C ABI; ``code`` follows errors.ts."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[bcmg code {code}] {message}")
        self.code = code
        self.message = message


_lib = None


def load() -> C.CDLL:
    """Load the in-tree library once, binding every declared signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissingError(
            f"{LIB_PATH} not found; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError as exc:
            raise LibraryMissingError(f"{LIB_PATH} does not export {name}") from exc
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> tuple[int, str]:
    lib = load()
    return int(lib.bcmg_last_error()), lib.bcmg_last_error_message().decode(errors="replace")


def check(rc: int) -> None:
    """Raise BcmgError for a non-zero return code."""
    if rc != BCMG_OK:
        code, msg = last_error()
        raise BcmgError(rc, msg or f"error {rc}")


def ptr_array(ptrs) -> C.Array:
    arr = (C.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = int(p)
    return arr
