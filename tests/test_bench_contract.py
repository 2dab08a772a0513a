"""bench.py keeps the driver's JSON contract (one line, the BASELINE.json
metric, roofline / cpu_baseline / e2e / clocks / gpu_launches keys) on both
arms."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRIC = "60-ch GSVD-MUSIC SSL blocks/sec; GSVD latency per block (us); x real-time"


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
def test_b200_arm_line():
    d = run_bench("--steps", "2", "--warmup", "3", "--batch", "4", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["metric"] == METRIC and d["unit"] == "blocks/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("fp64", "hbm", "tensor") and 0 < r["frac"] <= 1.0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0


def test_reference_arm_line():
    import oracle

    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "1")
    if "unavailable" in d:
        assert not oracle.ref_available()
        return
    assert d["impl"] == "reference" and d["metric"] == METRIC and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_flag_launches_the_ranks_itself():
    """`python bench.py --gpus 2` outside torchrun starts two ranks itself
    (torch.distributed.run, 127.0.0.1 rendezvous); --dry-run exercises that
    launcher and the barrier / max-over-ranks plumbing with gloo, no GPU."""
    d = run_bench("--gpus", "2", "--dry-run", "--steps", "2", "--warmup", "0")
    assert d["n_gpus"] == 2 and sorted(d["ranks"]) == [0, 1] and d["dry_run"] is True
