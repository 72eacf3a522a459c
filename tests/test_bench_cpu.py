"""CPU checks of bench.py's contract that need no GPU: the reference arm (the float64 oracle on a
bounded sample, `--impl reference`) prints exactly one JSON line with the required keys, and the
roofline helpers read the committed ncu summaries."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in j, k
    assert j["impl"] == "reference" and j["value"] > 0 and j["warmup"] >= 3
    assert j["cpu_baseline"]["kind"] == "oracle" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]
    assert "workload" in j["config"]


def test_roofline_inputs():
    import bench
    # F_c = 2nd + n(n+1) + 4n; config 2: 49,000 flops per candidate
    assert bench.flops_per_candidate(200, 20) == 2 * 200 * 20 + 200 * 201 + 800
    tr = bench.profiled_traffic("score_tc", 2)
    assert tr is not None and tr[0] >= 2 ** 20 * 80  # at least the candidate bytes
    peaks = bench.load_peaks()
    assert peaks["bf16_sus"] > 0 and peaks["hbm"] > 0
