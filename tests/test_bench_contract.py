"""bench.py's JSON-line contracts that run on CPU: the reference arm (the
reference package itself from baseline/_ref on host cores, else the oracle
port) and the multi-rank launcher in gloo dry-run mode."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                           "--no-ladder"],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)


def test_reference_arm_prints_one_contract_line():
    r = _run({})
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1
    assert d["unit"] == "TFLOP/s" and d["higher_is_better"] is True and d["value"] > 0
    ref_installed = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "bcmg"))
    assert d["cpu_baseline"]["kind"] == ("reference" if ref_installed else "port")
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["ms_per_step"] > 0 and abs(d["ms_per_step"] - 6000.0) > 1e-9  # measured, not a constant
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "config 3" in d["config"]["workload"]


def test_reference_arm_non_zero_rank_is_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_gpus_2_self_launches_ranks_dry_run():
    """`bench.py --gpus 2` without a torchrun environment launches 2 ranks itself
    (torch.distributed.run, 127.0.0.1); in --dry-run they run the host logic on
    gloo, reduce their times with MAX and rank 0 alone prints the line."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] is True and d["n_gpus"] == 2 and d["scaling"] == "strong"
    # N=131072, T=1024, 2 GPUs: tiles alternate, so half of the moved columns cross NVLink
    assert d["nvlink_bytes_per_gpu_max"] == d["nvlink_in_bytes_per_gpu_max"] > 0
    assert d["schedule_rank0"]["potrf"]["bcast_bytes"] > 0
