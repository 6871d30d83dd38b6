"""bench.py contract on the GPU: the default single-GPU line and the N>1
torchrun launch (2 ranks share the one visible B200 here; on an 8-GPU box each
rank binds GPU LOCAL_RANK) both print one JSON line with the required keys."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"}


def _last_json(out: str) -> dict:
    return json.loads([ln for ln in out.strip().splitlines() if ln.startswith("{")][-1])


def test_bench_single_gpu_c1():
    out = subprocess.run([sys.executable, "bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _last_json(out.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["gpu_launches"] > 0 and d["roofline"]["unit"] == "GB/s"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_torchrun_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29571", "bench.py", "--gpus", "2",
           "--workload", "c1", "--steps", "3", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _last_json(out.stdout)
    assert KEYS <= set(d) and d["n_gpus"] == 2 and d["value"] > 0
