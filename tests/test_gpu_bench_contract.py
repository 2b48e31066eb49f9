"""bench.py prints the driver's JSON line (one line, the keys the contract names) on a GPU box."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_bench_line_contract(cuda):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline", "--no-traffic", "--no-other-configs"],
                         capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
                "gpu_launches", "roofline", "clocks"):
        assert key in d, key
    assert d["unit"] == "steps/s" and d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["vs_baseline"] is None  # BASELINE.md publishes no number for this metric
    assert "workload" in d["config"] and "cfg4" in d["config"]["workload"]
    assert d["value"] > 10.0 and abs(d["value"] * d["ms_per_step"] / 1e3 - 1.0) < 1e-6
    e = d["e2e"]
    assert e["value"] > 10.0 and e["h2d_bytes_per_step"] == 8 * 2047 * 2047 == e["d2h_bytes_per_step"]
    assert d["gpu_launches"] > 1000
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0.05 < r["frac"] < 1.0 and 0.05 < r["fp64"]["frac"] < 1.0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert all(it in (10, 11, 12, 13) for it in d["iterations_per_step"])
