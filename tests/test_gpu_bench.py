"""The bench.py JSON-line contract (the driver parses it): one short run of the headline
configuration on the GPU, every required key present and consistent."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _run(*extra):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *extra],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_json_line_contract():
    d = _run("--steps", "5", "--warmup", "3", "--cpu-seconds", "1")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert abs(d["value"] * d["ms_per_step"] * 1e-3 - 1.0) < 1e-6  # one GPU: passes/s
    assert "workload" in d["config"]
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] <= 1 and abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-9
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 5 * d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_cfg4_batch_split_line():
    """BASELINE.json cfg4 ("batch 64 split by batch across 1/2/4/8 GPUs"): strong scaling,
    per-image draws; at one GPU the rank holds all 64 images."""
    d = _run("--config", "cfg4", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
             "--no-e2e", "--gpus", "1")
    assert d["scaling"] == "strong" and d["n_gpus"] == 1
    assert d["config"]["images_per_gpu"] == 64 and "720→180" in d["metric"]
    assert abs(d["value"] * d["ms_per_step"] * 1e-3 - 1.0) < 1e-6
    assert d["windows"]["n"] == 3 and d["windows"]["min"] <= d["windows"]["median"] <= d["windows"]["max"]
