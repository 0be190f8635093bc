"""bench.py keeps the driver's JSON contract: the reference arm on CPU (a
small N so it runs in seconds) and, on the GPU, our arm on a reduced system."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--n", "512", "--steps", "2", "--warmup", "1"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["higher_is_better"] is True and d["value"] > 0 and d["unit"] == d["e2e"]["unit"]
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] == "port" and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the reference arm runs only the oracle (no library of this repo mapped),
    # times attempts of the real solve prefix, and names the same config as ours
    assert d["native_libs"] == ["oracle/liborc.so"], d["native_libs"]
    assert d["prefix"]["evals"] >= 3 * d["steps"]
    import bench
    assert d["config"] == bench.workload_config(512, "f32", 1)


def test_reference_arm_other_ranks_exit_without_work():
    """Under torchrun only rank 0 runs and prints the reference arm; the other
    ranks exit 0 at once with no output."""
    env = dict(os.environ, RANK="1", LOCAL_RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--n", "512",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")], r.stdout


@pytest.mark.gpu
def test_our_arm_contract(gpu):
    d = _run(["--n", "4096", "--steps", "1", "--warmup", "1", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    rf = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(rf) and rf["bound"] == "hbm"
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["config"]["workload"]
    import bench
    assert d["config"] == bench.workload_config(4096, "f32", 1)
    # the launch count is the library's own device counter, not a formula
    assert d["gpu_launches"] >= 3 * d["accepted_steps_per_solve"]
