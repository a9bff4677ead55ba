"""bench.py's JSON line (the driver's contract): the reference arm runs on CPU
here (tiny deterministic sample); the GPU arm on a tiny C5 point."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout          # one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--nb", "64", "--D", "8", "--steps", "2", "--warmup", "1",
              "--ref-budget", "20000"], 600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["metric"] == "dp_cells_per_sec"
    assert d["value"] > 0 and d["unit"] == "visits/s" and d["higher_is_better"] is True
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and len(cb["per_step"]) == 2
    assert "nb=64" in d["config"]["workload"] and d["config"]["calls"] == 56


@pytest.mark.gpu
def test_gpu_arm_line(gpu):
    d = _run(["--nb", "256", "--D", "64", "--steps", "2", "--warmup", "1", "--no-sweep",
              "--no-latency", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["dtype"] == "f64" and d["data"] == "synthetic"
    rl = d["roofline"]
    assert rl["bound"] == "issue" and rl["peak"] > 0 and rl["kernel"] == "k_dp_level"
    assert rl["fp64_algorithmic"]["dadd_peak"] > 0
    assert set(d["breakdown_ms"]) >= {"flatten_ms", "upload_ms", "span_ms", "dp_ms", "post_ms",
                                      "exchange_ms", "decide_ms"}
    assert d["plan"] is not None and d["clocks"] is not None
