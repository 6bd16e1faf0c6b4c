"""bench.py's JSON contract on the CPU: the reference arm (the reference's own CPU path,
oracle/_ref or the port) prints one line with the driver's keys; the FLOP accounting matches
SURVEY 8d."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_algorithmic_flops_match_survey():
    import bench
    w = bench.WORKLOADS["llama7b-4k"]
    assert abs(bench.algorithmic_flops(w, 4096) / 1e12 - 39.58349234176) < 1e-9  # 3.958e13
    w16 = bench.WORKLOADS["llama7b-16k"]
    assert abs(bench.algorithmic_flops(w16, 16384) / 2.111e14 - 1) < 1e-3
    wf = bench.WORKLOADS["falcon7b-8k"]
    assert abs(bench.algorithmic_flops(wf, 8192) / 8.478e13 - 1) < 1e-3


@pytest.mark.timeout(600)
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "tiny",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
