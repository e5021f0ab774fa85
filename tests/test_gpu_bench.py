"""The bench.py contract on a GPU (the driver parses these lines): one JSON
line with the required keys for each config mode, on small configs so the
test stays short, and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("mode", ["full", "digest", "query"])
def test_bench_line_c1(mode):
    extra = ["--queries", "20000"] if mode == "query" else []
    j = _run("--config", "c1_er", "--mode", mode, "--steps", "3", "--warmup", "3", "--ref-sample", "4", *extra)
    assert KEYS <= set(j), KEYS - set(j)
    assert j["value"] > 0 and j["n_gpus"] == 1 and j["steps"] == 3 and j["gpu_launches"] > 0
    assert j["config"]["workload"] == "c1_er" and j["config"]["mode"] == mode
    r = j["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and 0 < r["frac"] < 1.5 and r["unit"] == "GB/s"
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in j["clocks"]
    if mode == "digest":
        assert j["parity"] is None or j["parity"]["match"]


def test_bench_reference_arm():
    j = _run("--impl", "reference", "--config", "c1_er", "--steps", "1", "--warmup", "0", "--ref-sample", "4")
    assert j["impl"] == "reference" and j["value"] > 0 and j["cpu_baseline"]["kind"] == "oracle"
    assert j["e2e"]["h2d_bytes_per_step"] == 0
