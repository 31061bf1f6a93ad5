#!/usr/bin/env python3
"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck), one
path per invocation, checked against the oracle so a silent corruption also
fails:

    compute-sanitizer --tool memcheck python tools/sanitize_probe.py redist
    compute-sanitizer --tool racecheck python tools/sanitize_probe.py f64

redist  bulk-copy cycle rotation (rotate_bulk_kernel, cp.async.bulk + mbarrier)
        and the lane rotation, 4 virtual devices, both directions
f64     potrs f64 N=1536, T=256: trail_tma_kernel / gemm_tma_kernel (TMA + DMMA),
        diagonal factor, substitution
f32     potrs f32 N=1536, T=256: tck_trail_kernel / tck_gemm_kernel (tcgen05)
c64     potrs c64 N=1024, T=256: the complex64 embedding on tcgen05
loop    2 loopback ranks: in-place peer redistribution + copy-engine panel hand-off
"""

import ctypes as C
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2601_14466_b200 as bc  # noqa: E402
from oracle import bcmg_oracle as O  # noqa: E402  (checker only)
from paper_2601_14466_b200 import _lib  # noqa: E402


def redist():
    from paper_2601_14466_b200.solvers import device_concat

    mesh = bc.DeviceMesh(4)
    for n_rows, n, t, dt in ((512, 1024, 64, np.float64), (64, 200, 7, np.float32), (256, 512, 32, np.complex128)):
        a = (np.arange(n_rows * n, dtype=np.float64).reshape(n_rows, n, order="F")).astype(dt)
        dm = bc.create_distributed(mesh, bc.MatrixDescriptor(n_rows, n, bc.ElementType.from_dtype(np.dtype(dt))),
                                   bc.TileSpec(t))
        bc.write_array(mesh, dm, np.asfortranarray(a))
        cyc = bc.redistribute_in(mesh, dm)
        assert np.array_equal(device_concat(mesh, cyc), O.deal_columns(np.asfortranarray(a), t, 4))
        back = bc.redistribute_out(mesh, cyc)
        assert np.array_equal(device_concat(mesh, back), a)
    mesh.close()


def solve(dt, n, t):
    a = O.make_matrix("random_spd", n, dt, 3)
    b = np.ones((n, 2), dtype=dt, order="F")
    mesh = bc.DeviceMesh(1)
    x, _ = bc.solve_positive_definite(mesh, a, b, bc.TileSpec(t))
    mesh.close()
    assert O.solve_residual(a, x, b) <= 100 * n * O.eps_of(dt)


def gemm_tma():
    """bcmg_gemm large enough for the persistent TMA kernel (gemm_tma_kernel, >= 148 blocks)."""
    import torch

    m, nn, k = 2048, 1280, 256
    rng = np.random.default_rng(1)
    a = torch.from_numpy(rng.standard_normal((k, m))).cuda()   # column-major m x k
    b = torch.from_numpy(rng.standard_normal((k, nn))).cuda()  # op C: B stored n x k column-major
    c = torch.zeros(nn, m, dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.load().bcmg_gemm(st, 1, m, nn, k, 1.0, C.c_void_p(a.data_ptr()), m, 0, C.c_void_p(b.data_ptr()),
                                     nn, 1, 0.0, C.c_void_p(c.data_ptr()), m))
    torch.cuda.synchronize()
    want = (a.t() @ b).t()  # C(i, j) = sum_k A(i, k) B(j, k)
    assert float((c - want).abs().max()) <= 1e-9 * float(want.abs().max())


def loop():
    import torch

    lib = _lib.load()
    n, t, ndev, world = 512, 64, 4, 2
    a = O.make_matrix("random_spd", n, np.float64, 4)
    idbuf = C.create_string_buffer(128)
    _lib.check(lib.bcmg_loopback_id(idbuf))
    sess = []
    for r in range(world):
        s = C.c_void_p()
        _lib.check(lib.bcmg_open(0, r, world, idbuf.raw, C.byref(s)))
        sess.append(s)
    half = n // world
    blocks = [torch.from_numpy(np.ascontiguousarray(a[:, r * half:(r + 1) * half].T)).cuda() for r in range(world)]
    xs = [torch.ones(n, dtype=torch.float64, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    errs = []

    def work(r):
        try:
            st = torch.cuda.Stream()
            p = _lib.ptr_array([blocks[r].data_ptr(), blocks[r].data_ptr() + (half // 2) * n * 8])
            info = C.c_int(0)
            _lib.check(lib.bcmg_potrs(sess[r], C.c_void_p(st.cuda_stream), 1, n, 1, t, ndev, p,
                                      C.c_void_p(xs[r].data_ptr()), n, 0, C.byref(info)))
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for s in sess:
        lib.bcmg_close(s)
    assert O.solve_residual(a, xs[0].cpu().numpy()[:, None], np.ones((n, 1))) <= 100 * n * O.eps_of(np.float64)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "f64"
    {"redist": redist, "f64": lambda: (solve(np.float64, 1536, 256), gemm_tma()), "f32": lambda: solve(np.float32, 1536, 256),
     "c64": lambda: solve(np.complex64, 1024, 256), "loop": loop}[what]()
    print(f"sanitize probe {what}: ok")
