#!/usr/bin/env python3
"""Benchmark of the B200 Cholesky solve path (BASELINE.json metric:
"potrs TFLOP/s fp64 N=131072 at 1/2/4/8 B200; block-cyclic redistribute GB/s").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload at every GPU count: BASELINE config 3 -- potrs float64 N=131072,
T_A=1024, N_RHS=64, A row-sharded over the N GPUs (P("x", None)); at N=1 the
whole 137 GB matrix sits on one 180 GB B200 and is factored in place
(overwrite_a=True).  Total work is fixed as N grows ("scaling": "strong").

A step is one potrs pipeline on a synthetic SPD matrix already resident in
HBM: regenerate A in place (potrf destroys it; a write-only device kernel,
bcmg_generate_spd, kept inside the timed region -- it only makes the number
conservative), contiguous -> block-cyclic redistribution, tiled potrf, tiled
substitution.  `value` = algorithmic TFLOP/s (N^3/3 + 2 N^2 N_RHS per step)
over the max-over-ranks device time of the K timed steps.  `e2e` = the same
metric through the public drop-in call `potrs(A_host, b_host, T_A, mesh)`
with A's row block and b in pinned HOST memory and x read back to the host.
`--impl reference` times the reference's CPU algorithm (the oracle port of
pkg/src/bcmg/solvers.py on numpy/scipy-openblas) on a bounded sample.
`--n/--t/--nrhs` override the shape (probe runs only).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "potrs TFLOP/s fp64 N=131072 at 1/2/4/8 B200; block-cyclic redistribute GB/s"
UNIT = "TFLOP/s"
SEED = 1


def potrs_flops(n: int, nrhs: int) -> float:
    return n ** 3 / 3.0 + 2.0 * n * n * nrhs


def workload(world: int, args) -> dict:
    if args.n:
        return {"n": args.n, "t": args.t or 1024, "nrhs": args.nrhs or 64,
                "workload": f"potrs f64 N={args.n} T_A={args.t or 1024} N_RHS={args.nrhs or 64} "
                            f"row-sharded over {world}xB200 (probe shape)"}
    return {"n": 131072, "t": 1024, "nrhs": 64,
            "workload": f"BASELINE config 3: potrs float64 N=131072, T_A=1024, N_RHS=64 row-sharded over "
                        f"{world}xB200"}


# ---------------------------------------------------------------- CPU baseline (oracle port)
def cpu_baseline(seconds: float = 12.0, n: int = 4096, t: int = 1024, nrhs: int = 64, full_n: int = 131072) -> dict:
    """The reference's tiled algorithm (oracle/bcmg_oracle.py, a restatement of
    pkg/src/bcmg/solvers.py potrf/potrs on numpy + scipy-openblas) on host cores."""
    import numpy as np

    from oracle import bcmg_oracle as O

    try:
        from threadpoolctl import threadpool_info

        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1])
    except Exception:
        cores = os.cpu_count() or 1
    a = O.make_matrix("random_spd", n, np.float64, 1)
    b = np.ones((n, nrhs), order="F")
    t0 = time.perf_counter()
    reps = 0
    while True:
        x = O.solve_pipeline(a, b, t)
        reps += 1
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    res = O.solve_residual(a, x, b)
    return {"value": potrs_flops(n, nrhs) * reps / dt / 1e12, "unit": UNIT, "cores": int(cores), "kind": "port",
            "sample": f"oracle port of the reference tiled potrf+potrs (solvers.py:341-474), f64 N={n} T_A={t} "
                      f"N_RHS={nrhs}, {reps} solves in {dt:.1f}s, residual {res:.2e}; N^3 extrapolation to "
                      f"N={full_n} = {dt / reps * (full_n / n) ** 3 / 3600:.1f} h/solve"}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    k, w = max(1, args.steps), max(0, args.warmup)
    per = 6.0  # seconds of CPU work per timed step (bounded sample)
    for _ in range(min(w, 1)):
        cpu_baseline(seconds=1.0)
    vals = [cpu_baseline(seconds=per) for _ in range(k)]
    v = sum(x["value"] for x in vals) / len(vals)
    cfg = workload(world, args)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": k,
            "warmup": w, "ms_per_step": per * 1000.0, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "reference_sample": vals[0]["sample"]},
            "cpu_baseline": {**vals[0], "value": v},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        import statistics

        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        loaded = [x for x in sm if x > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- GPU arm
def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2601_14466_b200 as bc
    from paper_2601_14466_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = workload(world, args)
    n, t, nrhs = cfg["n"], cfg["t"], cfg["nrhs"]
    rows = n // world
    lib = _lib.load()
    stream = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # this rank's row block of A (row-major rows x n == columns rank*rows.. of the symmetric A)
    A = torch.empty(rows, n, dtype=torch.float64, device=dev)

    def regen(dst):
        _lib.check(lib.bcmg_generate_spd(stream(), 1, n, rank * rows, rows, C.c_void_p(dst.data_ptr()), n, SEED,
                                         float(n)))

    gb = torch.Generator(device=dev).manual_seed(7)
    b = torch.rand(n, nrhs, dtype=torch.float64, device=dev, generator=gb) * 2 - 1
    mesh = bc.make_mesh(world)
    peak = C.c_double(0)
    _lib.check(lib.bcmg_measure_fp64_peak(local_rank, C.byref(peak)))

    def step():
        regen(A)
        return bc.potrs(A, b, T_A=t, mesh=mesh, overwrite_a=True)

    warm = max(3, args.warmup)
    for _ in range(warm):
        x = step()
    sync_all()

    # accuracy of the last warm-up solve: ||Ax - b||_F / (||A||_F ||x||_F + ||b||_F) on a fresh A
    regen(A)
    ax = torch.empty(rows, nrhs, dtype=torch.float64, device=dev)
    anorm2 = torch.zeros((), dtype=torch.float64, device=dev)
    for r0 in range(0, rows, 4096):
        blk = A[r0:r0 + 4096]
        torch.matmul(blk, x, out=ax[r0:r0 + 4096])
        anorm2 += (blk * blk).sum()
    if world > 1:
        full = [torch.empty_like(ax) for _ in range(world)]
        dist.all_gather(full, ax)
        ax = torch.cat(full)
        dist.all_reduce(anorm2)
    resid = float((ax - b).norm() / (anorm2.sqrt() * x.norm() + b.norm()))
    del ax, blk  # blk is a view: it would keep A's storage alive past `del A` below

    lib.bcmg_set_profiling(mesh.session, 1)
    launches0 = lib.bcmg_launch_count()
    sync_all()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        e0.record()
        for _ in range(args.steps):
            x = step()
        e1.record()
        torch.cuda.synchronize()
    sync_all()
    # library kernels + the per-step generator launch (bcmg_generate_spd is ours too)
    launches = lib.bcmg_launch_count() - launches0
    ms = e0.elapsed_time(e1)
    lib.bcmg_set_profiling(mesh.session, 0)
    st = (C.c_double * 4)()
    _lib.check(lib.bcmg_kernel_stats(mesh.session, 0, st))
    trail = {"launches": st[0], "ms": st[1], "flops": st[2]}
    other = {}
    for kind, name in ((1, "panel_trsm"), (2, "diag_factor"), (3, "rotate")):
        _lib.check(lib.bcmg_kernel_stats(mesh.session, kind, st))
        other[name] = {"launches": st[0], "ms": st[1]}
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t)
    flops = potrs_flops(n, nrhs)
    value = flops * args.steps / (ms * 1e-3) / 1e12

    # redistribution GB/s: the same matrix as 8 virtual devices on this GPU (D=1 itself is the identity)
    redist = None
    if world == 1 and n % (8 * t) == 0:
        vm = bc.make_mesh(8)
        regen(A)
        ptrs = _lib.ptr_array([A.data_ptr() + d * (n // 8) * n * 8 for d in range(8)])
        lib.bcmg_set_profiling(vm.session, 1)
        for _ in range(2):
            for direction in (0, 1):
                _lib.check(lib.bcmg_redistribute(vm.session, vm.stream_handle(), 1, n, n, t, 8, ptrs, direction))
        torch.cuda.synchronize()
        _lib.check(lib.bcmg_kernel_stats(vm.session, 3, st))
        rot_gbs = st[2] / (st[1] * 1e-3) / 1e9
        redist = {"value": rot_gbs, "unit": "GB/s", "config": f"f64 N={n} T_A={t} 8 virtual devices on 1 GPU",
                  "bytes_per_launch": st[2] / max(st[0], 1), "launches": st[0],
                  "roofline": {"bound": "hbm", "achieved": rot_gbs, "peak": _hbm_peak(), "unit": "GB/s",
                               "frac": rot_gbs / _hbm_peak()}}
        vm.close()

    # e2e through the public call with host buffers: A's row block and b in pinned host
    # memory, x read back; A's device block is released first (the call uploads its own copy)
    regen(A)
    Ah = torch.empty(rows, n, dtype=torch.float64, pin_memory=True)
    Ah.copy_(A)
    bh = b.cpu().pin_memory()
    del A  # stays in torch's cache: the call's upload reuses the block
    sync_all()
    ke = 1
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(ke):
        xh = bc.potrs(Ah, bh, T_A=t, mesh=mesh).cpu()
    t1.record()
    torch.cuda.synchronize()
    ems = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ems, op=dist.ReduceOp.MAX)
    e2e = {"value": flops * ke / (float(ems) * 1e-3) / 1e12, "unit": UNIT,
           "h2d_bytes_per_step": int(Ah.numel() * 8 + bh.numel() * 8),
           "d2h_bytes_per_step": int(xh.numel() * 8), "steps": ke,
           "path": "paper_2601_14466_b200.potrs(A_row_block_host_pinned, b_host, T_A, mesh) -> x.cpu()"}
    e2e_ok = bool(torch.allclose(xh, x.cpu(), rtol=0, atol=1e-12))
    del Ah

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    achieved = trail["flops"] / (trail["ms"] * 1e-3) / 1e12 if trail["ms"] else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": warm, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": n, "tile": t, "n_rhs": nrhs, "logical_devices": world,
                   "parallelism": f"1D block-cyclic columns over {world} GPU(s)",
                   "l2": "inputs (A: %.1f GB per GPU) exceed L2 (126 MB)" % (rows * n * 8 / 1e9),
                   "input": "A = (R+R^T)/2 + N I, R ~ U[-1,1) hashed per unordered (i,j) (bcmg_generate_spd, "
                            "seed 1); b ~ U[-1,1)",
                   "step": "regenerate A in place (inside the timed region) + redistribute_in + potrf + potrs",
                   "residual": resid, "e2e_matches_device_x": e2e_ok},
        "roofline": {"bound": "tensor", "kernel": "trail_tma_kernel (TMA + DMMA trailing update)",
                     "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                     "frac": achieved / peak.value if peak.value else None,
                     "peak_source": "measured live: bcmg_measure_fp64_peak (register-resident mma.sync.m8n8k4.f64 "
                                    "loop on all SMs); MEASURED_PEAKS.json has no FP64 entry",
                     "traffic": _profile_traffic(), "launches": trail["launches"],
                     "flops_per_launch": trail["flops"] / max(trail["launches"], 1),
                     "ms_per_launch": trail["ms"] / max(trail["launches"], 1),
                     "share_of_step": trail["ms"] / ms if ms else None,
                     "step_fraction_of_peak": value / peak.value if peak.value else None},
        "kernels": other,
        "clocks": clocks.summary(),
        "gpu_launches": int(launches),
        "e2e": e2e,
        "redistribute": redist,
        "cpu_baseline": cpu_baseline() if world == 1 and not args.no_cpu else None,  # rank 0 at N=1 only
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _hbm_peak() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def _profile_traffic():
    """dram bytes per trail_tma_kernel launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "trail_kernel_traffic.json")
    try:
        return json.load(open(p))["dram_bytes_per_launch"]
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--t", type=int, default=0)
    ap.add_argument("--nrhs", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
