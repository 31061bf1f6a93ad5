#!/usr/bin/env python3
"""Benchmark of the B200 Cholesky solve path (BASELINE.json metric:
"potrs TFLOP/s fp64 N=131072 at 1/2/4/8 B200; block-cyclic redistribute GB/s").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dry-run]

Workload at every GPU count: BASELINE config 3 -- potrs float64 N=131072,
T_A=1024, N_RHS=64, A row-sharded over the N GPUs (P("x", None)); at N=1 the
whole 137 GB matrix sits on one 180 GB B200 and is factored in place
(overwrite_a=True).  Total work is fixed as N grows ("scaling": "strong").

Process model: one process per GPU.  The driver launches N > 1 with
torch.distributed.run; `python bench.py --gpus N` without a torchrun
environment launches the N ranks itself the same way (127.0.0.1 rendezvous,
NCCL_DEBUG=INFO into a per-rank file whose communicator lines rank 0 quotes).

A step is one potrs pipeline on a synthetic SPD matrix already resident in
HBM: regenerate A in place (potrf destroys it; a write-only device kernel,
bcmg_generate_spd, kept inside the timed region -- it only makes the number
conservative), contiguous -> block-cyclic redistribution (NVLink peer copies
between GPUs), tiled potrf, tiled substitution.  `value` = algorithmic TFLOP/s
(N^3/3 + 2 N^2 N_RHS per step) over the max-over-ranks device time of the K
timed steps.  `e2e` = the same metric through the public drop-in call
`potrs(A_host, b_host, T_A, mesh)` with A's row block and b in pinned HOST
memory and x read back to the host.

`--impl reference` times the reference itself (pkg/src/bcmg, installed
unmodified into baseline/_ref by `pip install --target`) through its own
public `solve_positive_definite` on the host cores: each timed step one solve
at N=4096 with config 3's T_A=1024, 8 devices and N_RHS=64, plus config 1
exactly and an N ladder with the N^3 extrapolation to N=131072 (labelled).
Without baseline/_ref it falls back to the oracle port (kind "port").
`--dry-run` runs the multi-rank host logic on CPU with gloo (no GPU).
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


# ---------------------------------------------------------------- CPU baseline (the reference itself)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _host_cores() -> int:
    try:
        from threadpoolctl import threadpool_info

        return int(max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1]))
    except Exception:
        return int(os.cpu_count() or 1)


def _import_reference():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "bcmg")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import bcmg  # noqa: F401
        from bcmg import cli as ref_cli  # noqa: F401

        return bcmg
    except Exception:
        return None


def _ref_solve(bcmg, n: int, t: int, d: int, nrhs: int, seed: int = 1):
    """One reference solve_positive_definite (solvers.py:931-985) on host arrays;
    returns (seconds, residual)."""
    import numpy as np
    from bcmg import cli as ref_cli

    a = ref_cli.make_matrix("random_spd", n, bcmg.ElementType.real64, seed)
    b = np.ones((n, nrhs))
    mesh = bcmg.DeviceMesh(d)
    t0 = time.perf_counter()
    x, _ = bcmg.solve_positive_definite(mesh, a, b, bcmg.TileSpec(t))
    dt = time.perf_counter() - t0
    res = float(ref_cli.solve_residual(a, x, b)) if hasattr(ref_cli, "solve_residual") else None
    return dt, res


def _port_solve(n: int, t: int, nrhs: int):
    """The oracle port (oracle/bcmg_oracle.py restates solvers.py:341-474 on numpy/scipy)."""
    import numpy as np

    from oracle import bcmg_oracle as O

    a = O.make_matrix("random_spd", n, np.float64, 1)
    b = np.ones((n, nrhs), order="F")
    t0 = time.perf_counter()
    x = O.solve_pipeline(a, b, t)
    return time.perf_counter() - t0, O.solve_residual(a, x, b)


SAMPLE = {"n": 4096, "t": 1024, "d": 8, "nrhs": 64}


def cpu_baseline(seconds: float = 12.0, full_n: int = 131072) -> dict:
    """Bounded sample of the workload on the host cores: reference solves at
    N=4096 (config 3's T_A, device count and N_RHS) for >= `seconds`."""
    bcmg = _import_reference()
    n, t, d, nrhs = SAMPLE["n"], SAMPLE["t"], SAMPLE["d"], SAMPLE["nrhs"]
    tot, reps, res = 0.0, 0, None
    while tot < seconds or reps == 0:
        dt, res = _ref_solve(bcmg, n, t, d, nrhs) if bcmg else _port_solve(n, t, nrhs)
        tot += dt
        reps += 1
    per = tot / reps
    kind = "reference" if bcmg else "port"
    what = ("reference bcmg.solve_positive_definite (baseline/_ref, unmodified pkg/src/bcmg)" if bcmg else
            "oracle port of the reference tiled potrf+potrs (solvers.py:341-474)")
    return {"value": potrs_flops(n, nrhs) / per / 1e12, "unit": UNIT, "cores": _host_cores(), "kind": kind,
            "sample": f"{what}, f64 N={n} T_A={t} D={d} N_RHS={nrhs}, random_spd seed 1, b = ones; {reps} solves "
                      f"in {tot:.1f}s ({per:.2f} s/solve, residual {res if res is None else f'{res:.2e}'}); N^3 "
                      f"extrapolation to N={full_n}: {per * (full_n / n) ** 3 / 3600:.1f} h/solve"}


def reference_ladder(bcmg) -> dict:
    """Config 1 exactly (min / median of 3) and an N ladder at config 3's T_A / D /
    N_RHS, fitted to N^3 and extrapolated (labelled) to N=32768 and 131072."""
    import numpy as np

    out = {}
    c1 = [_ref_solve(bcmg, 2048, 256, 2, 1) for _ in range(3)]
    ts = sorted(x[0] for x in c1)
    out["config1"] = {"what": "potrs f64 N=2048, T_A=256, N_RHS=1, DeviceMesh(2), random_spd seed 1, b = ones",
                      "min_s": ts[0], "median_s": ts[1], "residual": c1[0][1],
                      "tflops": potrs_flops(2048, 1) / ts[0] / 1e12}
    pts = []
    for n in (2048, 4096, 8192):
        dt, res = _ref_solve(bcmg, n, 1024, 8, 64)
        pts.append((n, dt))
        out[f"n{n}"] = {"s": dt, "tflops": potrs_flops(n, 64) / dt / 1e12, "residual": res}
    # t = c N^3 with c averaged over the two largest points
    c = float(np.mean([dt / n ** 3 for n, dt in pts[1:]]))
    out["extrapolated_N3"] = {"n32768_s": c * 32768 ** 3, "n131072_s": c * 131072 ** 3,
                              "n131072_tflops": potrs_flops(131072, 64) / (c * 131072 ** 3) / 1e12,
                              "label": "EXTRAPOLATED proportional to N^3 from the N=4096/8192 points, not measured"}
    # secondary comparator: LAPACK potrf + potrs through scipy on the same cores
    try:
        import scipy.linalg as sl
        from bcmg import cli as ref_cli

        lap = {}
        for n in (4096, 8192):
            a = ref_cli.make_matrix("random_spd", n, bcmg.ElementType.real64, 1)
            b = np.ones((n, 64))
            t0 = time.perf_counter()
            x = sl.cho_solve(sl.cho_factor(a, lower=True, check_finite=False), b, check_finite=False)
            dt = time.perf_counter() - t0
            lap[f"n{n}"] = {"s": dt, "tflops": potrs_flops(n, 64) / dt / 1e12,
                            "residual": float(ref_cli.solve_residual(a, x, b))}
        try:
            from threadpoolctl import threadpool_info

            lap["blas"] = [{k: i.get(k) for k in ("internal_api", "version", "num_threads")} for i in threadpool_info()]
        except Exception:
            pass
        out["lapack_cho_solve"] = lap
    except Exception as e:  # the comparator is optional
        out["lapack_cho_solve"] = {"unavailable": str(e)[:200]}
    return out


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    k, w = max(1, args.steps), max(0, args.warmup)
    bcmg = _import_reference()
    n, t, d, nrhs = SAMPLE["n"], SAMPLE["t"], SAMPLE["d"], SAMPLE["nrhs"]
    solve = (lambda: _ref_solve(bcmg, n, t, d, nrhs)) if bcmg else (lambda: _port_solve(n, t, nrhs))
    for _ in range(min(w, 1)):
        solve()
    times, res = [], None
    for _ in range(k):
        dt, res = solve()
        times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    v = potrs_flops(n, nrhs) * len(times) / sum(times) / 1e12
    cfg = workload(world, args)
    kind = "reference" if bcmg else "port"
    ladder = reference_ladder(bcmg) if bcmg and not args.no_ladder else None
    sample = (f"{'reference bcmg.solve_positive_definite (baseline/_ref)' if bcmg else 'oracle port'} f64 N={n} "
              f"T_A={t} D={d} N_RHS={nrhs} per step (config 3 scaled to a bounded CPU sample), residual {res:.2e}")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": k,
            "warmup": w, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "reference_sample": sample, "ladder": ladder},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": _host_cores(), "kind": kind, "sample": sample},
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
        # communicator evidence (nranks, NVLS) into a per-rank file, not stdout: rank 0
        # quotes it in its JSON line (also when the driver launches torchrun itself)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        os.environ.setdefault("NCCL_DEBUG_FILE", NCCL_LOG)
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
    # per-phase split of the last timed step (CUDA events inside the pipeline), max over ranks
    ph = (C.c_float * 4)()
    _lib.check(lib.bcmg_last_timings(mesh.session, ph))
    ph_t = torch.tensor([float(v) for v in ph], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ph_t, op=dist.ReduceOp.MAX)
    phases = {"redistribute_ms": float(ph_t[0]), "potrf_ms": float(ph_t[1]), "potrs_ms": float(ph_t[2]),
              "pipeline_ms": float(ph_t[3]), "of": "last timed step, max over ranks"}
    redist_x = None
    if world > 1:  # the cross-GPU redistribution of the last step: NVLink peer moves between the ranks
        moved = float(lib.bcmg_last_moved_bytes(mesh.session))
        egress, ingress = _nvlink_bytes(lib, n, t, world, rank)
        eg = torch.tensor([egress, ingress], dtype=torch.float64, device=dev)
        dist.all_reduce(eg, op=dist.ReduceOp.MAX)
        sec = max(phases["redistribute_ms"], 1e-6) * 1e-3
        redist_x = {"value": moved / sec / 1e9, "unit": "GB/s", "bytes": moved,
                    "what": "algorithmic bytes (2 s N x moved columns, whole job) / redistribute phase time",
                    "nvlink_bytes_per_gpu_max": float(eg[0]), "nvlink_in_bytes_per_gpu_max": float(eg[1]),
                    "nvlink_gbs_per_gpu": float(eg[0]) / sec / 1e9, "nvlink_peak_gbs": 900.0,
                    "nvlink_peak_source": "NVLink 5 datasheet, 900 GB/s per direction per GPU (not measured here)",
                    "path": os.environ.get("BCMG_REDIST_NCCL") and "nccl pack/send/recv" or "in-place P2P rotation"}

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
                     "traffic": (_profile_traffic() or {}).get("dram_bytes_per_launch"),
                     "traffic_detail": _profile_traffic(), "launches": trail["launches"],
                     "flops_per_launch": trail["flops"] / max(trail["launches"], 1),
                     "ms_per_launch": trail["ms"] / max(trail["launches"], 1),
                     "share_of_step": trail["ms"] / ms if ms else None,
                     "step_fraction_of_peak": value / peak.value if peak.value else None},
        "kernels": {**other, "note": "CUDA-event brackets on each kind's launching stream over the timed steps; "
                                     "the diagonal factor and panel solve run on the critical stream next to the "
                                     "persistent bulk grid, so their times include waiting for SMs (not kernel "
                                     "durations; tools/kernel_split.py, tools/scale_model.py with "
                                     "CUDA_LAUNCH_BLOCKING=1 give those)"},
        "clocks": clocks.summary(),
        "nccl": _nccl_summary() if world > 1 else None,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "redistribute": redist if world == 1 else redist_x,
        "phases": phases,
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
    """ncu DRAM bytes (read + write) per bulk trail_tma_kernel launch at the bench shape
    (profiles/r02_trail_traffic_n131072.json, tools/trail_traffic.py), with the same
    launches' algorithmic bytes."""
    p = os.path.join(ROOT, "profiles", "r02_trail_traffic_n131072.json")
    try:
        d = json.load(open(p))
        return {"dram_bytes_per_launch": d["bulk_launch_traffic_mean"],
                "algorithmic_bytes_per_launch": d["bulk_launch_algorithmic_mean"],
                "ratio": d["bulk_ratio_mean"], "source": "profiles/r02_trail_traffic_n131072.json"}
    except Exception:
        return None


def _nvlink_bytes(lib, n: int, t: int, world: int, rank: int) -> tuple:
    """Bytes this rank sends / receives over NVLink in the redistribution (moves whose
    source and destination segments live on different processes)."""
    import ctypes as C

    seg, cnt = C.c_int64(0), C.c_int64(0)
    lib.bcmg_redistribute_plan(n, t, world, world, 0, C.byref(seg), None, 0, C.byref(cnt))
    mv = (C.c_int64 * (4 * max(cnt.value, 1)))()
    lib.bcmg_redistribute_plan(n, t, world, world, 0, C.byref(seg), mv, cnt.value, C.byref(cnt))
    seg_bytes = seg.value * n * 8
    out = sum(seg_bytes for i in range(cnt.value) if mv[4 * i + 2] == rank and mv[4 * i + 3] != rank)
    inn = sum(seg_bytes for i in range(cnt.value) if mv[4 * i + 3] == rank and mv[4 * i + 2] != rank)
    return float(out), float(inn)


NCCL_LOG = "/tmp/bcmg_nccl_debug.%h.%p.log"
_T_START = time.time()


def _nccl_summary():
    """Communicator facts from the NCCL_DEBUG=INFO file(s) of this host (self-launched runs)."""
    import glob
    import re

    lines = []
    files = [f for f in glob.glob(NCCL_LOG.replace("%h", "*").replace("%p", "*"))
             if os.path.getmtime(f) >= _T_START - 5]  # this job's ranks only (stale /tmp files skipped)
    for f in sorted(files)[:16]:
        try:
            for ln in open(f, errors="replace"):
                if re.search(r"nranks|NVLS|Init COMPLETE|comm 0x", ln):
                    lines.append(ln.strip()[:200])
        except OSError:
            pass
    return {"debug_file": NCCL_LOG, "lines": lines[:24]} if lines else None


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1) without a torchrun environment: launch the N
    ranks exactly as the driver does (torch.distributed.run, 127.0.0.1 rendezvous)."""
    env = dict(os.environ)
    if not args.dry_run:
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        env.setdefault("NCCL_DEBUG_FILE", NCCL_LOG)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def run_dry(args, rank: int, world: int) -> None:
    """Multi-rank host logic on CPU (gloo, no GPU): every rank builds its potrf /
    potrs schedules and its share of the redistribution plan at the workload
    shape; the per-rank time is reduced with MAX and rank 0 prints one line."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2601_14466_b200 import _lib

    if world > 1:
        dist.init_process_group("gloo")
    cfg = workload(world, args)
    n, t, nrhs = cfg["n"], cfg["t"], cfg["nrhs"]
    lib = _lib.load()
    t0 = time.perf_counter()
    counts = {}
    for routine, name in ((0, "potrf"), (1, "potrs")):
        cnt = C.c_int64(0)
        _lib.check(lib.bcmg_schedule(routine, n, t, world, world, rank, nrhs, None, 0, C.byref(cnt)))
        ops = (C.c_int64 * (7 * cnt.value))()
        _lib.check(lib.bcmg_schedule(routine, n, t, world, world, rank, nrhs, ops, cnt.value, C.byref(cnt)))
        counts[name] = {"ops": cnt.value,
                        "bcast_bytes": 8 * sum(ops[7 * i + 6] for i in range(cnt.value) if ops[7 * i] in (2, 8))}
    egress, ingress = _nvlink_bytes(lib, n, t, world, rank)
    ms = (time.perf_counter() - t0) * 1e3
    red = torch.tensor([ms, egress, ingress], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
    if rank == 0:
        line = {"metric": METRIC, "value": 0.0, "unit": UNIT, "n_gpus": world, "steps": 0, "warmup": 0,
                "ms_per_step": float(red[0]), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "dry_run": True,
                "config": {"workload": cfg["workload"], "n": n, "tile": t, "n_rhs": nrhs, "backend": "gloo (CPU)"},
                "schedule_rank0": counts, "nvlink_bytes_per_gpu_max": float(red[1]),
                "nvlink_in_bytes_per_gpu_max": float(red[2])}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    ap.add_argument("--no-ladder", action="store_true", help="reference arm: skip the config 1 / N ladder")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank host logic on CPU (gloo), no GPU")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.dry_run:
        return run_dry(args, rank, world)
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
