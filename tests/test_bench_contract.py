"""bench.py keeps the driver's JSON contract (one line, the required keys):
the reference arm on CPU, and a small run of our arm on the GPU."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import has_gpu

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--size", "256", "--iters", "4", "--steps", "2", "--warmup", "1",
              "--cpu-budget", "0.3"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] in ("port", "reference")
    assert d["value"] > 0 and d["config"]["workload"].startswith("hotspot")


def test_gpus_n_spawns_ranks():
    """`--gpus 2` without a launcher re-execs under torchrun: two ranks run
    (the reference arm prints once, from rank 0, with n_gpus = the world)."""
    d = _run(["--impl", "reference", "--gpus", "2", "--size", "128", "--iters", "2", "--steps", "1",
              "--warmup", "0", "--cpu-budget", "0.1"], timeout=300)
    assert d["impl"] == "reference" and d["n_gpus"] == 2


def test_gpus_n_fails_loudly_without_gpus():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough GPUs here")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert r.returncode != 0 and "requested but only" in r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.gpu
def test_our_arm_contract_small():
    if not has_gpu():
        pytest.skip("no CUDA device")
    d = _run(["--size", "1024", "--iters", "10", "--steps", "3", "--warmup", "3", "--no-kernels",
              "--cpu-budget", "0.5"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["gpu_launches"] == 30 and d["value"] > 0 and 0 < d["roofline"]["frac"] < 1.5
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert d["e2e"]["checked"] is True
    assert d["launch_latency"]["launch_sync_us"] > 0
