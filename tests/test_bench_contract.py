"""bench.py's output contract (the driver parses these lines).

* -m "not gpu": `--impl reference` (the FP64 oracle timed as the reference arm) prints one JSON line
  with the keys the driver reads, on a bounded sample;
* -m gpu: the default GPU arm at a few steps prints one JSON line with value, ms_per_step,
  roofline, cpu_baseline-less run, e2e with copy bytes, gpu_launches and clocks, consistent with
  its own timing.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=600)
    assert d["impl"] == "reference" and KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "images/s" and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run(["--steps", "4", "--warmup", "3", "--no-cpu-baseline"], timeout=900)
    assert KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] >= 3 and d["scaling"] == "weak"
    assert abs(d["value"] - 256 * 1000.0 / d["ms_per_step"]) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1.2 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 256 * 3 * 227 * 227 + 256 * 4 and e["d2h_bytes_per_step"] == 4
    assert d["gpu_launches"] > 4 * 30
    assert d["clocks"] is None or d["clocks"]["sm_mhz"] > 0
