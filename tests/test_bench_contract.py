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
    d = _bench("--impl", "reference", "--steps", "1", "--warmup", "3", "--workload", "c2")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["config"]["workload"] == "c2"
    # the same work as the GPU line (T0..T5 + circus), extrapolated from launch-only emulator seconds
    assert d["same_config"] is True and d["config"]["functionals"] == "T0-T5 + P1-P3 circus"
    assert d["cpu_baseline"]["extrapolated"] is True and d["cpu_baseline"]["cpu_model"]
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
    # the sampling pipe (one TLD4 per distinct sampled tap, measured TLD4 peak), FP32 model beside it
    assert r["bound"] == "tex" and r["unit"] == "gathers/s"
    assert r["achieved"] * r["kernel_ms"] / 1e3 == pytest.approx(180 * 256 * 256, rel=1e-9)
    f = r["fp32_model"]
    assert 0 < f["frac"] < 1 and "26 executed flop" in f["work"]
    assert d["gpu_launches"] == 3  # one fused trace launch per step (C1 has no circus stage)
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=120, env=env)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


def test_spawn_ranks_launches_a_gloo_world(tmp_path):
    """bench.spawn_ranks (plain `python bench.py --gpus N`) runs N ranks under torch.distributed.run
    with 127.0.0.1 rendezvous; exercised with a gloo all_reduce on CPU."""
    sys.path.insert(0, ROOT)
    import bench

    script = tmp_path / "w.py"
    out = tmp_path / "out"
    script.write_text(
        "import os, sys, torch, torch.distributed as dist\n"
        "dist.init_process_group('gloo')\n"
        "t = torch.tensor([dist.get_rank() + 1.0])\n"
        "dist.all_reduce(t)\n"
        "if dist.get_rank() == 0:\n"
        "    open(sys.argv[1], 'w').write(f\"{dist.get_world_size()} {int(t.item())} {os.environ['MASTER_ADDR']}\")\n"
        "dist.destroy_process_group()\n")
    assert bench.spawn_ranks(str(script), [str(out)], 2) == 0
    assert out.read_text() == "2 3 127.0.0.1"
