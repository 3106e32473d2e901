"""bench.py's one-line JSON contract (the driver parses it): a reduced run on
the GPU prints every required key with sane values, on the tensor-core path
with its roofline and the CUDA-core path beside it."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks")


def test_bench_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--scans", "64", "--steps", "3", "--warmup", "3", "--no-cpu",
                          "--cpu-seconds", "1"],
                         cwd=REPO, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"].startswith("BASELINE configs[3]")
    r = d["roofline"]
    assert r["bound"] in ("tensor", "smem") and 0 < r["frac"] <= 1.0 and r["achieved"] > 0 and r["peak"] > 0
    assert d["tensor_cores"] and r["bound"] == "tensor"
    core = d["cuda_core_path"]
    assert core["roofline"]["bound"] == "smem" and 0 < core["roofline"]["frac"] <= 1.0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * 5  # per step: Gram, fp16 planes, step plan, A operands, the W = 32 TC kernel
    assert "sm_mhz" in d["clocks"]
