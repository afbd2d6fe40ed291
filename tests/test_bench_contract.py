"""bench.py's JSON-line contract (the driver parses it): the keys and their
types for the reference arm (the fp64 oracle on the host cores, CPU test) and
for our arm on the GPU (value, roofline, cpu_baseline, e2e, clocks,
gpu_launches, sustained)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, timeout=900):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "20", "--warmup", "3"], timeout=300)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "Gpts/s" and d["higher_is_better"] is True
    assert d["steps"] == 20 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["config"]["workload"] == "C1" and d["dtype"] == "f64"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "Gpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "40", "--warmup", "3", "--cpu-budget", "1", "--sustained", "0.2"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["metric"].startswith("grid-point updates/s") and d["unit"] == "Gpts/s"
    assert d["value"] > 50 and d["steps"] == 40 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["scaling"] == "weak" and d["vs_baseline"] is None and d["dtype"] == "f32"
    assert d["config"]["workload"] == "C3" and d["config"]["order"] == 2
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.3 < r["frac"] < 1.3
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["algorithmic_bytes_per_point"] == 10.0 and r["kernel"] == "tb2ws_step_kernel"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    e = d["e2e"]
    assert 0 < e["value"] < d["value"] * 1.05 and e["unit"] == "Gpts/s"
    assert e["h2d_bytes_per_step"] >= 512 ** 3 * 4 / 40 and e["d2h_bytes_per_step"] >= 512 ** 3 * 4 / 40
    assert d["gpu_launches"] >= 20                       # 40 steps, two per launch (+ graph counters)
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    s = d["sustained"]
    assert s["value"] > 0 and s["steps"] >= 40
    r = d["repetitions"]
    assert r["n"] == 5 and len(r["ms"]) == 5 and r["value_min"] <= d["value"] <= r["value_max"]
    assert abs(d["ms_per_step"] - r["ms_per_step_median"]) < 1e-12
    assert isinstance(d["gpu_launches"], int) and d["config"]["graph_steps"] > 0


def test_gpus_flag_spawns_ranks_launch_check():
    """`bench.py --gpus 2` without torchrun's environment starts two ranks
    itself (torch.distributed.run on 127.0.0.1) and rank 0 reports n_gpus 2
    (FD_BENCH_SHARE_GPU=1: no GPU count check; gloo, no GPU work)."""
    env = {**os.environ, "FD_BENCH_SHARE_GPU": "1"}
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["gpus_requested"] == 2 and sorted(r[0] for r in d["ranks"]) == [0, 1]


def test_gpus_flag_refuses_without_enough_gpus():
    """Without the test hook, --gpus N on a node with fewer GPUs fails loudly
    instead of silently measuring one GPU."""
    env = {k: v for k, v in os.environ.items() if k not in ("FD_BENCH_SHARE_GPU", "WORLD_SIZE")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 2 and "needs 2 GPUs" in p.stderr


def test_world_size_must_match_gpus_flag():
    env = {**os.environ, "WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--launch-check"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 2 and "WORLD_SIZE=1" in p.stderr
