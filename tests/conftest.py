"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else
runs on CPU (oracle vs golden vectors, planner, host logic, ABI exports)."""

import os

# Several loopback ranks share one GPU in tests/test_gpu_loopback.py; with more
# streams than hardware work queues, a stream parked on a peer flag can hold up
# an unrelated stream that aliases its queue.  Read at CUDA context creation.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built libbcmg_b200.so")


def numbered_columns(n_rows, n_cols, dtype):
    """Every element distinct, complex lanes distinct (reference conftest.py:23-34)."""
    base = np.arange(n_rows * n_cols, dtype=np.float64).reshape(n_rows, n_cols, order="F")
    dt = np.dtype(dtype)
    if dt.kind == "c":
        return np.asfortranarray((base - 1j * (base + 0.5)).astype(dt))
    return np.asfortranarray(base.astype(dt))


ALL_DTYPES = [np.float32, np.float64, np.complex64, np.complex128]


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


@pytest.fixture(scope="module")
def meshes(cuda):
    """Cached DeviceMesh per logical-device count (virtual devices on GPU 0)."""
    import paper_2601_14466_b200 as bc

    cache = {}

    def get(d):
        if d not in cache:
            cache[d] = bc.DeviceMesh(d, device=0)
        return cache[d]

    yield get
    for m in cache.values():
        m.close()
