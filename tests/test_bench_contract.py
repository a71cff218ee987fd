"""bench.py's JSON-line contract (the driver parses these keys): the
reference arm on the CPU, our arm on the GPU, both at BASELINE configs[0]."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _line(args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--config", "0", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # whole oracle steps at configs[1]'s grid: the timed region is what ran
    assert d["config"]["workload"].startswith("256x256")
    assert d["ms_per_step"] * d["steps"] < 60e3


def test_default_run_is_the_declared_workload():
    """No flags = BASELINE configs[3] for its declared 20 steps after 5 warm-up."""
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse_args([])
    assert (a.config, a.steps, a.warmup, a.gpus) == (3, 20, 5, 1)
    assert bench.CONFIGS[a.config]["name"] == "4096x4096_20steps"
    assert bench.parse_args(["--config", "2"]).steps == 50


@pytest.mark.gpu
def test_our_arm_line():
    d = _line(["--config", "0", "--steps", "2", "--warmup", "3", "--no-cpu",
               "--matvec-sizes", "256", "512"])
    assert BASE_KEYS <= set(d), set(d) ^ BASE_KEYS
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert 0 < r["frac"] < 1.5 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    mv = d["matvec_sweep"]["records"]
    assert {(r["op"], r["n"]) for r in mv} == {(o, n) for o in ("ch", "poisson") for n in (256, 512)}
    assert all(r["GBps"] > 0 for r in mv)
