"""bench.py pieces that run without a GPU: the reference arm (the oracle port
timed on the host cores) and the algorithmic byte / LUP accounting."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _last_json(out: str) -> dict:
    return json.loads([ln for ln in out.strip().splitlines() if ln.startswith("{")][-1])


def test_bench_reference_arm():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "c1",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _last_json(out.stdout)
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["cores"] >= 1


def test_algorithmic_bytes_match_survey():
    """C4 17,129,537,600 B / launch, C2 2,134,900,800, C3 3,220,176,960."""
    assert bench.bytes_per_iter(bench.WORKLOADS["c4"]) == 17_129_537_600
    assert bench.bytes_per_iter(bench.WORKLOADS["c2"]) == 2_134_900_800
    assert bench.bytes_per_iter(bench.WORKLOADS["c3"]) == 3_220_176_960
    assert bench.lup_per_iter(bench.WORKLOADS["c4"]) == 1022 ** 3
    # a temporal chain of 2 sweeps reads A once and writes A once; B only in
    # the last of the run's 50 chains
    m = 1022
    assert bench.bytes_per_launch(bench.WORKLOADS["c4"], ("tb", 2)) == int(
        8 * ((m ** 3 + 6 * m ** 2) + m ** 3) + 8 * m ** 3 / 50)
