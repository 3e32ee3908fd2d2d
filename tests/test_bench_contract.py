"""The bench.py output contract (one JSON line; keys the driver reads), for both arms.

The reference arm runs the reference engine built from its sources (oracle/_ref/tt_tier2) on
host cores, so it is checked on CPU; the GPU arm is checked on a small workload (C1)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _bench(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "tt_tier2")):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    d = _bench("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["config"]["workload"] == "c2"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _bench("--workload", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"] == "c1" and "l2" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 256 * 256 * 4 and e["d2h_bytes_per_step"] > 0
    assert d["e2e_matches_device_result"] is True
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    t = r["tex_gather"]  # the sampling stage's roofline (measured TLD4 peak)
    assert 0 < t["frac"] < 1 and t["gathers_per_launch"] == 180 * 256 * 256
    assert d["gpu_launches"] == 3  # one fused trace launch per step (C1 has no circus stage)
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
