"""BASELINE configs 4 and 5 on one GPU (probe, not the bench):

  --config 4 : potri complex128 N=65536, T_A=512 (D logical devices on this GPU)
  --config 5 : potrs float32 / complex64 N=65536, T_A in {128..2048}: potrs TFLOP/s
               and redistribution GB/s with D virtual devices

A is generated on the device (bcmg_generate_spd) and factored in place."""
import argparse, ctypes as C, json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc
from paper_2601_14466_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--n", type=int, default=65536)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--tiles", default="128,256,512,1024,2048")
ap.add_argument("--dtypes", default="f32,c64")
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
lib = _lib.load()
CODES = {"f32": (0, torch.float32), "f64": (1, torch.float64), "c64": (2, torch.complex64), "c128": (3, torch.complex128)}
stream = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731


def gen(A, code, n):
    _lib.check(lib.bcmg_generate_spd(stream(), code, n, 0, n, C.c_void_p(A.data_ptr()), n, 21, float(n)))


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    e1.synchronize()
    return out, e0.elapsed_time(e1)


n = a.n
mesh = bc.make_mesh(a.d)
if a.config == 4:
    code, dt = CODES["c128"]
    t = 512
    A = torch.empty(n, n, dtype=dt, device="cuda")
    for rep in range(a.reps):
        gen(A, code, n)
        _, ms = timed(lambda: bc.potri(A, T_A=t, mesh=mesh, overwrite_a=True))
        ph = bc.last_timings(mesh)
        flops = 4.0 * n ** 3  # potrf + trtri + lauum, complex (x4)
        # residual on a column sample: ||A X[:, cols] - I[:, cols]|| / sqrt(cols)
        X = A  # the inverse, in A's storage
        cols = torch.arange(0, n, n // 64, device="cuda")
        Xs = X[:, cols].clone()
        gen(A, code, n)
        R = A @ Xs
        R[cols, torch.arange(len(cols), device="cuda")] -= 1
        res = float(R.norm() / len(cols) ** 0.5)
        print(json.dumps({"config": 4, "routine": "potri", "dtype": "c128", "n": n, "t": t, "d": a.d, "ms": ms,
                          "tflops": flops / ms / 1e9, "phases": ph, "inverse_residual_sample": res}), flush=True)
elif a.config == 5:
    for name in a.dtypes.split(","):
        code, dt = CODES[name]
        A = torch.empty(n, n, dtype=dt, device="cuda")
        b = torch.ones(n, a.nrhs, dtype=dt, device="cuda")
        for t in [int(x) for x in a.tiles.split(",")]:
            best = None
            for rep in range(a.reps):
                gen(A, code, n)
                x, ms = timed(lambda: bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True))
                best = ms if best is None else min(best, ms)
            ph = bc.last_timings(mesh)
            cf = 4.0 if dt.is_complex else 1.0
            flops = cf * (n ** 3 / 3 + 2 * n * n * a.nrhs)
            gen(A, code, n)
            r = float((A @ x).sub(b).norm() / (A.norm() * x.norm() + b.norm()))
            # redistribution GB/s with 8 virtual devices (in place, both directions)
            vm = bc.make_mesh(8)
            esz = A.element_size()
            ptrs = _lib.ptr_array([A.data_ptr() + i * (n // 8) * n * esz for i in range(8)])
            lib.bcmg_set_profiling(vm.session, 1)
            for direction in (0, 1, 0, 1):
                _lib.check(lib.bcmg_redistribute(vm.session, vm.stream_handle(), code, n, n, t, 8, ptrs, direction))
            torch.cuda.synchronize()
            st = (C.c_double * 4)()
            _lib.check(lib.bcmg_kernel_stats(vm.session, 3, st))
            vm.close()
            print(json.dumps({"config": 5, "routine": "potrs", "dtype": name, "n": n, "t": t, "d": a.d, "ms": best,
                              "tflops": flops / best / 1e9, "phases": ph, "residual": r,
                              "redistribute_gbs_8dev": st[2] / (st[1] * 1e-3) / 1e9 if st[1] else None}),
                  flush=True)
        del A
        torch.cuda.empty_cache()
