"""GPU: the DMMA GEMM (every contraction of the path) against a plain PyTorch
float64 / complex128 reference of the same op, through the C ABI `bcmg_gemm`.
Tolerance: |C - C_ref| <= 8 * K * eps * (|A| |B|) elementwise bound (FP64
accumulation in a different order)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
bc = pytest.importorskip("paper_2601_14466_b200")
from paper_2601_14466_b200 import _lib  # noqa: E402


def _run(torch, dt, m, n, k, op_a, op_b, alpha, beta, lda_pad=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    tdt = {0: torch.float32, 1: torch.float64, 2: torch.complex64, 3: torch.complex128}[dt]
    wide = torch.complex128 if tdt.is_complex else torch.float64

    def rand(r, c):
        x = torch.rand(r, c, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        if tdt.is_complex:
            x = x + 1j * (torch.rand(r, c, device="cuda", dtype=torch.float64, generator=g) * 2 - 1)
        return x.to(tdt)

    ar, ac = (m, k) if op_a == 0 else (k, m)
    br, bc_ = (k, n) if op_b == 0 else (n, k)
    lda = ar + lda_pad
    A = rand(lda, ac)  # column-major storage = transposed torch tensor
    B = rand(br, bc_)
    Cm = rand(m, n)
    Acm = A.t().contiguous()  # (ac, lda) row-major == (lda, ac) col-major
    Bcm = B.t().contiguous()
    Ccm = Cm.t().contiguous()
    opA = A[:ar].to(wide) if op_a == 0 else A[:ar].to(wide).conj().t()
    opB = B.to(wide) if op_b == 0 else B.to(wide).conj().t()
    ref = alpha * (opA @ opB) + beta * Cm.to(wide)
    rc = _lib.load().bcmg_gemm(None, dt, m, n, k, alpha, C.c_void_p(Acm.data_ptr()), lda, op_a,
                               C.c_void_p(Bcm.data_ptr()), br, op_b, beta, C.c_void_p(Ccm.data_ptr()), m)
    _lib.check(rc)
    torch.cuda.synchronize()
    got = Ccm.t().to(wide)
    bound = (opA.abs() @ opB.abs()) * abs(alpha) + abs(beta) * Cm.to(wide).abs()
    eps = 2.0 ** -52 if tdt in (torch.float64, torch.complex128) else 2.0 ** -23
    err = (got - ref).abs() - 8 * (k + 2) * eps * bound - 1e-300
    return float(err.max())


@pytest.mark.parametrize("dt", [0, 1, 2, 3])
@pytest.mark.parametrize("op_a,op_b", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (37, 19, 23), (130, 16, 70), (257, 129, 65), (64, 200, 300)])
def test_gemm_matches_torch(cuda, dt, op_a, op_b, m, n, k):
    import torch

    assert _run(torch, dt, m, n, k, op_a, op_b, -1.0, 1.0) <= 0
    assert _run(torch, dt, m, n, k, op_a, op_b, 1.0, 0.0, lda_pad=3, seed=1) <= 0


@pytest.mark.parametrize("m,n,k", [(4096, 2048, 1024), (2100, 1500, 333)])
def test_gemm_large_tma_path(cuda, m, n, k):
    """Shapes large enough for the TMA + mbarrier persistent kernel."""
    import torch

    for op_b in (0, 1):
        assert _run(torch, 1, m, n, k, 0, op_b, -1.0, 1.0) <= 0


@pytest.mark.parametrize("m,n,k", [(512, 256, 96), (4096, 2048, 1024), (1000, 300, 77), (256, 64, 32)])
def test_gemm_f32_tcgen05_3xtf32(cuda, m, n, k):
    """float32 natural-layout shapes take the tcgen05 kind::tf32 3xTF32 kernel
    (TMEM accumulators); FP32-level accuracy against a float64 torch reference."""
    import torch

    pad = (-m) % 4
    assert _run(torch, 0, m, n, k, 0, 1, -1.0, 1.0, lda_pad=pad) <= 0
    assert _run(torch, 0, m, n, k, 0, 1, 1.0, 0.0, lda_pad=pad, seed=3) <= 0


@pytest.mark.parametrize("m,n,k", [(2100, 1500, 333), (1030, 2050, 517), (4096, 1024, 512)])
def test_gemm_c128_real_embedding(cuda, m, n, k):
    """complex128 shapes large enough for the real embedding on the FP64 TMA
    kernel: op_b = N reads B in place (k-contiguous operand, interleaved A
    embedding), op_b = C takes the planar gather; odd K and padded lda."""
    import torch

    for op_a in (0, 1):
        for op_b in (0, 1):
            assert _run(torch, 3, m, n, k, op_a, op_b, -1.0, 1.0) <= 0
            assert _run(torch, 3, m, n, k, op_a, op_b, 1.0, 0.0, lda_pad=3, seed=2) <= 0
