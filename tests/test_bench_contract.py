"""CPU check of bench.py's reference arm (the driver runs `bench.py --impl
reference` beside our own arm): it must run the reference's own step on the
host cores and print one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"] == "particle current deposits/sec" and d["unit"] == "deposits/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("C2")
    # same-config, one-core reference
    assert d["same_config"] is True and d["cpu_baseline"]["cores"] == 1
    assert "128x128x128 x 16 ppc" in d["cpu_baseline"]["sample"] and "1 core" in d["cpu_baseline"]["sample"]
    assert d["cpu_detail"]["order"] == 3 and d["cpu_detail"]["nproc"] >= 1 and d["cpu_detail"]["model"]


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_prints_the_contract_line():
    """The GPU arm on C1 (fast): every contract key, a self-check that passed,
    per-order entries, the roofline with its measured traffic, and the
    one-core same-config CPU baseline."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "3",
                        "--warmup", "3", "--e2e-steps", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "orders", "selfcheck"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["selfcheck"]["ok"]
    assert set(d["orders"]) == {"1", "2", "3"}
    assert d["roofline"]["frac"] > 0 and d["roofline"]["traffic"] is not None
    assert d["cpu_baseline"]["cores"] == 1 and d["cpu_baseline"]["same_config"] is True
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
