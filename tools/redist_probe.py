"""Redistribution (in-place cycle rotation) GB/s with D virtual devices on one GPU."""
import ctypes as C, sys, os, json, argparse
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_14466_b200 as bc
from paper_2601_14466_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384); ap.add_argument("--t", type=int, default=1024)
ap.add_argument("--d", type=int, default=8); ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n, t, d = a.n, a.t, a.d
lib = _lib.load()
A = torch.arange(n * n, dtype=torch.float64, device="cuda").reshape(n, n)
ref = A.clone()
vm = bc.make_mesh(d)
ptrs = _lib.ptr_array([A.data_ptr() + i * (n // d) * n * 8 for i in range(d)])
st = (C.c_double * 4)()
for rep in range(a.reps):
    lib.bcmg_set_profiling(vm.session, 1)
    for direction in (0, 1):
        _lib.check(lib.bcmg_redistribute(vm.session, vm.stream_handle(), 1, n, n, t, d, ptrs, direction))
    torch.cuda.synchronize()
    _lib.check(lib.bcmg_kernel_stats(vm.session, 3, st))
    print(json.dumps({"n": n, "t": t, "d": d, "launches": st[0], "ms": st[1], "bytes": st[2],
                      "gbs": st[2] / (st[1] * 1e-3) / 1e9}), flush=True)
print("roundtrip_exact", bool(torch.equal(A, ref)))
