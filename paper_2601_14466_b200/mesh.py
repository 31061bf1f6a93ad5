"""Device mesh: the set of logical devices a distributed matrix is dealt over,
and the native session (streams, workspaces, NCCL communicator) that drives
them.

The reference's DeviceMesh (pkg/src/bcmg/runtime.py:255-499) simulates D
devices in one process and forces a single coordinating caller
(run_coordinated, runtime.py:449-466).  Here:

* one process per GPU (torchrun); ``num_devices`` logical devices are split
  evenly over the ``world`` processes of ``torch.distributed``;
* with one process all logical devices are *virtual devices* on the same GPU
  (the multi-device arithmetic of the reference, runnable on one B200);
* the single-caller contract is kept: concurrent entry raises
  :class:`ConcurrentCallError`, both here and inside the C ABI.
"""

from __future__ import annotations

import ctypes as C
import threading
from contextlib import contextmanager

from . import _lib
from .core import ConcurrentCallError, StaleSessionError

__all__ = ["DeviceMesh"]


class DeviceMesh:
    """``num_devices`` logical devices over this job's processes.

    Parameters
    ----------
    num_devices: total logical devices (the reference's D); default = world size.
    device: CUDA device index of this process (default: LOCAL_RANK or current).
    distributed: use torch.distributed's world (rank/world) and NCCL between
        processes; default True when torch.distributed is initialised with
        more than one rank.
    """

    def __init__(self, num_devices: int | None = None, device: int | None = None, distributed: bool | None = None):
        import torch

        dist_ok = torch.distributed.is_available() and torch.distributed.is_initialized()
        if distributed is None:
            distributed = dist_ok and torch.distributed.get_world_size() > 1
        if distributed and not dist_ok:
            raise RuntimeError("distributed=True needs torch.distributed to be initialised")
        self.rank = torch.distributed.get_rank() if distributed else 0
        self.world = torch.distributed.get_world_size() if distributed else 1
        if num_devices is None:
            num_devices = self.world
        if num_devices < 1:
            raise ValueError(f"need at least one device, got {num_devices}")
        if num_devices % self.world:
            raise ValueError(f"num_devices={num_devices} is not a multiple of the {self.world} processes")
        self.num_devices = int(num_devices)
        self.local_count = self.num_devices // self.world
        self.local_devices = list(range(self.rank * self.local_count, (self.rank + 1) * self.local_count))
        if device is None:
            import os

            device = int(os.environ.get("LOCAL_RANK", torch.cuda.current_device() if torch.cuda.is_available() else 0))
        self.device = int(device)
        self._session = None
        self._closed = False
        self._lock = threading.Lock()

    # -- native session ------------------------------------------------------
    @property
    def session(self) -> C.c_void_p:
        if self._closed:
            raise StaleSessionError("mesh is closed")
        if self._session is None:
            lib = _lib.load()
            nccl_id = None
            if self.world > 1:
                import torch

                buf = C.create_string_buffer(128)
                if self.rank == 0:
                    _lib.check(lib.bcmg_nccl_unique_id(buf))
                obj = [bytes(buf.raw) if self.rank == 0 else None]
                torch.distributed.broadcast_object_list(obj, src=0)
                nccl_id = obj[0]
            h = C.c_void_p()
            _lib.check(lib.bcmg_open(self.device, self.rank, self.world, nccl_id, C.byref(h)))
            self._session = h
        return self._session

    def close(self) -> None:
        if self._session is not None:
            _lib.check(_lib.load().bcmg_close(self._session))
            self._session = None
        self._closed = True

    def __del__(self):
        try:
            if self._session is not None:
                _lib.load().bcmg_close(self._session)
        except Exception:
            pass

    @property
    def torch_device(self):
        import torch

        return torch.device("cuda", self.device)

    def stream_handle(self):
        import torch

        return C.c_void_p(torch.cuda.current_stream(self.torch_device).cuda_stream)

    # -- single-caller contract (runtime.py:449-466) --------------------------
    @contextmanager
    def coordinated(self):
        if not self._lock.acquire(blocking=False):
            raise ConcurrentCallError("another caller is already driving this mesh")
        try:
            yield self
        finally:
            self._lock.release()

    def run_coordinated(self, fn):
        with self.coordinated():
            return fn()

    def owner_of_tile(self, k: int) -> int:
        return k % self.num_devices

    def __repr__(self) -> str:
        return (f"DeviceMesh(num_devices={self.num_devices}, world={self.world}, rank={self.rank}, "
                f"device=cuda:{self.device})")
