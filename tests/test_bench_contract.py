"""The driver contract of bench.py (one JSON line with fixed keys): the reference arm on the
CPU here, our arm on the GPU (small step counts, no secondary measurements)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout, env=None):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "steps/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("cfg2")


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--no-secondary", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["metric"] == "SMC verify+resample steps/s; achieved HBM GB/s vs B200 peak"
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] == 3 * d["steps"]                 # K1 + K2 + one reindex per step
    assert d["e2e"]["h2d_bytes_per_step"] > 60e6 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["config"]["workload"].startswith("cfg2")


def test_gpus_n_self_launches_ranks():
    """`bench.py --gpus 2` with no torchrun wrapper launches 2 ranks itself (the reference arm:
    CPU only, gloo plumbing); rank 0 prints the one line with n_gpus = 2."""
    d = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"], 600)
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["value"] > 0


def test_world_size_mismatch_is_an_error():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "4", "--steps", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=120, env={**os.environ, "WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


@pytest.mark.gpu
def test_our_arm_two_ranks_self_launched():
    """Our arm at --gpus 2 without a wrapper; on a 1-GPU box the ranks share cuda:0 over gloo
    (SMCSD_BENCH_BACKEND=gloo: a functional check, not a bench value)."""
    env = {} if torch_gpus() >= 2 else {"SMCSD_BENCH_BACKEND": "gloo"}
    d = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--no-secondary", "--no-cpu-baseline"],
             900, env=env)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"] == "dp2 (prompts)"


def torch_gpus():
    import torch
    return torch.cuda.device_count()
