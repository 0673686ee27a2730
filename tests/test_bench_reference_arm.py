"""The reference arm of bench.py (--impl reference) runs on the host cores only: check its JSON
line against the bench contract on a small time budget (no GPU needed)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-budget", "1.0", "--config", "c2"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "cost+gradient evals/sec" and line["unit"] == "evals/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["config"]["workload"] == "c2"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_default_workload_is_c4_with_the_same_config_object():
    """Default workload = c4 (largest single-GPU config); its `config` equals the GPU arm's."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2304_06200_b200 import models

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--ref-budget", "0.5"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    case = models.build_case("c4", n_steps=4)
    want = bench.workload_config(case, 1, "single")
    want["n_steps"] = 4000
    assert line["config"] == want
    assert "trajectories" in line["cpu_baseline"]["sample"] and line["value"] > 0
