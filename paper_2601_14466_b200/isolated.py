"""MPMD ("isolated") execution of the pipelines on one GPU (reference
runtime.py:405-466 run_workers / run_coordinated in ``isolated`` mode, the CLI's
``--mode mpmd``, cli.py:62-64, 242-256).

Every logical device is a worker with its own native session (rank d of a
world of D, joined by the in-process loopback transport) and its own shard
allocation; a worker sees the other workers' shards only through the
transport's pointer exchange -- the handle publication of the reference's
HandleRegistry -- and the world > 1 drivers move data between them exactly as
between processes (in-place peer rotation of the redistribution, copy-engine
panel hand-offs, substitution hand-offs).  Across GPUs the same drivers run one
process per GPU under torchrun (NCCL + CUDA IPC tokens, see ipc.py).  Results
are bit-identical to the shared-address (spmd) run.
"""

from __future__ import annotations

import ctypes as C
import gc
import threading
import time

import numpy as np

from . import _lib
from .core import DescriptorError, ElementType, NotPositiveDefiniteError, Structure, TileSpec, validate_tile
from .layout import device_column_counts
from .solvers import Timings, _matrix_descriptor, _raise_for


def _run_workers(devices: int, device: int, body):
    """body(rank, session, stream) on one thread per logical device."""
    import torch

    lib = _lib.load()
    idbuf = C.create_string_buffer(128)
    _lib.check(lib.bcmg_loopback_id(idbuf))
    sessions = []
    try:
        for r in range(devices):
            s = C.c_void_p()
            _lib.check(lib.bcmg_open(device, r, devices, idbuf.raw, C.byref(s)))
            sessions.append(s)
        results, errors = [None] * devices, []

        def work(r):
            try:
                with torch.cuda.device(device):
                    st = torch.cuda.Stream()
                    with torch.cuda.stream(st):
                        results[r] = body(r, sessions[r], st)
                    st.synchronize()
            except BaseException as exc:  # noqa: BLE001 - reported to the caller
                errors.append((r, exc))

        # nothing may synchronise the whole device while a worker's stream is
        # parked on a peer flag: no collection of other sessions meanwhile
        gc.collect()
        torch.cuda.synchronize(device)
        gc.disable()
        try:
            threads = [threading.Thread(target=work, args=(r,), name=f"device-worker-{r}") for r in range(devices)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
        finally:
            gc.enable()
        if errors:  # the lowest device's exception, as the reference (runtime.py:441-444)
            raise min(errors, key=lambda e: e[0])[1]
        return results
    finally:
        for s in sessions:
            lib.bcmg_close(s)


def _worker_shards(a: np.ndarray, tile: int, devices: int, device: int):
    """Each worker's own allocation: its logical device's columns (contiguous layout)."""
    import torch

    n = a.shape[1]
    counts = device_column_counts(n, TileSpec(tile), devices)
    out, c0 = [], 0
    for d in range(devices):
        blk = torch.from_numpy(np.ascontiguousarray(a[:, c0:c0 + counts[d]].T)).to(f"cuda:{device}")
        out.append((blk, c0, c0 + counts[d]))
        c0 += counts[d]
    return out


def solve_positive_definite_isolated(a: np.ndarray, b: np.ndarray, tile: TileSpec, devices: int, device: int = 0):
    """solve_positive_definite (solvers.py:931-985) with one isolated worker per device."""
    import torch

    desc = _matrix_descriptor(a, Structure.positive_definite)
    validate_tile(tile, desc.n_cols)
    et = desc.element_type
    n, t = desc.n_rows, tile.tile_width
    b2 = np.asarray(b)
    one = b2.ndim == 1
    b2 = b2.reshape(n, -1) if one else b2
    if b2.shape[0] != n:
        raise DescriptorError("dimension-mismatch", f"right-hand side shape {b.shape} does not match n={n}")
    if np.iscomplexobj(b2) and not et.is_complex:
        raise DescriptorError("type-structure", "complex right-hand side with a real matrix")
    t0 = time.perf_counter()
    shards = _worker_shards(np.asarray(a, dtype=et.dtype), t, devices, device)
    xs = [torch.from_numpy(np.ascontiguousarray(b2.astype(et.dtype).T)).to(f"cuda:{device}") for _ in range(devices)]
    torch.cuda.synchronize(device)
    t1 = time.perf_counter()
    lib = _lib.load()
    infos = [C.c_int(0) for _ in range(devices)]

    def body(r, sess, st):
        ptrs = _lib.ptr_array([shards[r][0].data_ptr()])
        rc = lib.bcmg_potrs(sess, C.c_void_p(st.cuda_stream), et.code, n, b2.shape[1], t, devices, ptrs,
                            C.c_void_p(xs[r].data_ptr()), n, 0, C.byref(infos[r]))
        if rc != _lib.BCMG_OK:
            _raise_for(rc, infos[r].value)
        ms = (C.c_float * 4)()
        _lib.check(lib.bcmg_last_timings(sess, ms))
        return [float(v) for v in ms]

    phases = _run_workers(devices, device, body)
    x = xs[0].cpu().numpy().T
    t2 = time.perf_counter()
    ph = [max(p[i] for p in phases) for i in range(4)]
    out = np.asfortranarray(x[:, 0] if one else x)
    return out, Timings(t1 - t0, t2 - t1, ph[0], ph[1], ph[2], ph[3])


def invert_positive_definite_isolated(a: np.ndarray, tile: TileSpec, devices: int, device: int = 0):
    """invert_positive_definite (solvers.py:988-1016) with one isolated worker per device."""
    desc = _matrix_descriptor(a, Structure.positive_definite)
    validate_tile(tile, desc.n_cols)
    et = desc.element_type
    n, t = desc.n_rows, tile.tile_width
    t0 = time.perf_counter()
    shards = _worker_shards(np.asarray(a, dtype=et.dtype), t, devices, device)
    t1 = time.perf_counter()
    lib = _lib.load()
    infos = [C.c_int(0) for _ in range(devices)]

    def body(r, sess, st):
        ptrs = _lib.ptr_array([shards[r][0].data_ptr()])
        rc = lib.bcmg_potri(sess, C.c_void_p(st.cuda_stream), et.code, n, t, devices, ptrs, 0, C.byref(infos[r]))
        if rc != _lib.BCMG_OK:
            _raise_for(rc, infos[r].value)
        ms = (C.c_float * 4)()
        _lib.check(lib.bcmg_last_timings(sess, ms))
        return [float(v) for v in ms]

    phases = _run_workers(devices, device, body)
    inv = np.empty((n, n), dtype=et.dtype, order="F")
    for blk, c0, c1 in shards:
        inv[:, c0:c1] = blk.cpu().numpy().T
    t2 = time.perf_counter()
    ph = [max(p[i] for p in phases) for i in range(4)]
    return inv, Timings(t1 - t0, t2 - t1, ph[0], ph[1], ph[2], ph[3])


def eigh_hermitian_isolated(a: np.ndarray, tile: TileSpec, devices: int, device: int = 0):
    """eigh_hermitian with worker-owned shards published to the coordinator
    (run_workers + HandleRegistry + run_coordinated, runtime.py:191-233): the
    workers allocate and fill their shards, the coordinator collects the
    published addresses and runs the eigensolver on them."""
    import torch

    from .ipc import HandleRegistry
    from .solvers import _hermitian_structure, _require_hermitian

    desc = _matrix_descriptor(a, _hermitian_structure(ElementType.from_dtype(np.asarray(a).dtype)))
    _require_hermitian(desc)
    validate_tile(tile, desc.n_cols)
    et = desc.element_type
    n, t = desc.n_rows, tile.tile_width
    t0 = time.perf_counter()
    shards = _worker_shards(np.asarray(a, dtype=et.dtype), t, devices, device)
    reg = HandleRegistry(devices, mode="shared_address")  # one process: publication is the address itself
    for d, (blk, _, _) in enumerate(shards):
        reg.publish(d, blk)
    handles = reg.coordinator_handles()
    torch.cuda.synchronize(device)
    t1 = time.perf_counter()
    lib = _lib.load()
    sess = C.c_void_p()
    _lib.check(lib.bcmg_open(device, 0, 1, None, C.byref(sess)))
    try:
        real = torch.float32 if et in (ElementType.real32, ElementType.complex64) else torch.float64
        w = torch.empty(n, dtype=real, device=f"cuda:{device}")
        info = C.c_int(0)
        st = torch.cuda.current_stream(device)
        rc = lib.bcmg_syevd(sess, C.c_void_p(st.cuda_stream), et.code, n, t, devices,
                            _lib.ptr_array([h.data_ptr() for h in handles]), C.c_void_p(w.data_ptr()), 0,
                            C.byref(info))
        _raise_for(rc, info.value)
        st.synchronize()
        ms = (C.c_float * 4)()
        _lib.check(lib.bcmg_last_timings(sess, ms))
    finally:
        lib.bcmg_close(sess)
    v = np.empty((n, n), dtype=et.dtype, order="F")
    for blk, c0, c1 in shards:
        v[:, c0:c1] = blk.cpu().numpy().T
    t2 = time.perf_counter()
    return w.cpu().numpy(), v, Timings(t1 - t0, t2 - t1, float(ms[0]), float(ms[1]), float(ms[2]), float(ms[3]))


__all__ = ["solve_positive_definite_isolated", "invert_positive_definite_isolated", "eigh_hermitian_isolated",
           "NotPositiveDefiniteError"]
