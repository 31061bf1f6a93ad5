"""MPMD / isolated-namespace handle exchange (reference runtime.py:170-233,
390-406: ``_TokenChannel``, ``HandleRegistry``, ``publish_handle`` /
``open_handle``).

In the reference, workers of an *isolated* mesh allocate their shards in their
own namespaces and publish handles; the coordinator collects one handle per
device and opens them in its own namespace.  On a B200 node the namespaces are
processes and the handles are CUDA IPC tokens: ``publish_handle`` exports any
device tensor of this process as a 72-byte token (the IPC handle of its
allocation plus the offset inside it, ``bcmg_ipc_export``); ``open_handle``
maps a token from another process into this one (``bcmg_ipc_open``; NVLink peer
memory when the exporter sits on another GPU) and returns a tensor view of it.
The drivers use the same tokens internally for the in-place peer
redistribution and the copy-engine panel broadcast (csrc/comm.cpp).
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

from . import _lib

TOKEN_BYTES = 72


class RegistryError(RuntimeError):
    """Handle registry misuse: double publish or incomplete registry (runtime.py:67-68)."""


class HandleDomainError(RuntimeError):
    """A token used in the namespace (process) that exported it (runtime.py:55-56)."""


@dataclass(frozen=True)
class HandleToken:
    """Opaque cross-process ticket produced by ``publish_handle`` (runtime.py:82-87)."""

    token: bytes
    device_index: int
    nbytes: int
    dtype: str
    shape: tuple


def publish_handle(tensor, device_index: int = 0) -> HandleToken:
    """Export a CUDA tensor of this process (runtime.py:392-397)."""
    if not getattr(tensor, "is_cuda", False):
        raise ValueError("publish_handle needs a CUDA tensor")
    if not tensor.is_contiguous():
        raise ValueError("publish_handle needs a contiguous tensor")
    buf = C.create_string_buffer(TOKEN_BYTES)
    _lib.check(_lib.load().bcmg_ipc_export(C.c_void_p(tensor.data_ptr()), buf))
    dtype = str(tensor.dtype).replace("torch.", "")
    return HandleToken(buf.raw, int(device_index), int(tensor.numel() * tensor.element_size()), dtype,
                       tuple(int(x) for x in tensor.shape))


class _CudaArray:
    """__cuda_array_interface__ wrapper of an opened (peer) device address."""

    _TYPESTR = {"float32": "<f4", "float64": "<f8", "complex64": "<c8", "complex128": "<c16", "int32": "<i4"}

    def __init__(self, ptr: int, token: HandleToken):
        self.__cuda_array_interface__ = {"shape": token.shape, "typestr": self._TYPESTR[token.dtype],
                                         "data": (int(ptr), False), "version": 3, "strides": None, "stream": None}


def open_handle(token: HandleToken, device=None):
    """Map a token from another process into this one (runtime.py:399-406);
    returns a tensor view of the exporter's memory (not a copy)."""
    import torch

    ptr = C.c_void_p()
    rc = _lib.load().bcmg_ipc_open(token.token, C.byref(ptr))
    if rc != _lib.BCMG_OK:
        code, msg = _lib.last_error()
        raise HandleDomainError(msg)
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        return torch.as_tensor(_CudaArray(ptr.value, token), device="cuda")


def close_all() -> None:
    """Unmap every opened token of this process."""
    _lib.check(_lib.load().bcmg_ipc_close_all())


class HandleRegistry:
    """Per-device handle slots filled by workers and read by the coordinator
    (runtime.py:191-233): each device publishes exactly once; the coordinator
    may collect only when every slot is filled; in isolated mode collection
    opens the tokens in the coordinator's process."""

    def __init__(self, num_devices: int, mode: str = "isolated"):
        if mode not in ("isolated", "shared_address"):
            raise ValueError(f"unknown mode {mode!r}")
        self.mode = mode
        self._slots: list = [None] * int(num_devices)
        self._lock = threading.Lock()

    def publish(self, device_index: int, entry) -> None:
        """``entry``: a HandleToken (isolated) or a tensor (shared_address)."""
        if not 0 <= device_index < len(self._slots):
            raise ValueError(f"no slot for device {device_index}")
        if self.mode == "isolated" and not isinstance(entry, HandleToken):
            entry = publish_handle(entry, device_index)
        with self._lock:
            if self._slots[device_index] is not None:
                raise RegistryError(f"device {device_index} already published")
            self._slots[device_index] = entry

    @property
    def missing(self) -> list[int]:
        return [d for d, slot in enumerate(self._slots) if slot is None]

    @property
    def complete(self) -> bool:
        return not self.missing

    def coordinator_handles(self) -> list:
        if not self.complete:
            raise RegistryError(f"incomplete registry: missing devices {self.missing}")
        if self.mode == "isolated":
            return [open_handle(t) for t in self._slots]
        return list(self._slots)
