"""Parity at the exact benchmarked configurations.

Every test here drives the GPU through the same objects bench.py times —
`bench.build_job` (the workload's setup program on a GpuJob) and
`bench.step_dag` (one step = 100 iterations as W_BATCH DAG bytes, executed by
`GpuJob.run_bytes`, repeated steps replayed from a CUDA graph) — at the benchmark's
full size, and compares EVERY array with the strict-order C oracle
(oracle/strict_eval.c, all host cores) run over the same DAGs:

* C4 — 3-D 7-point Jacobi 1024^3 fp64: bench steps until one is a CUDA-graph replay (4 steps, 400 iterations) with
  the default kernels (the 2-sweep temporal chain est_tb, B stored only by a
  run's last chain); plus the
  same geometry with 64 seeded sub-box fills per array (tests/util.py:55-64
  convention) so the interior is not dominated by exact zeros.
* C2 — 3-D 7-point heat 512^3 fp64 with the survey's parity variant: 64
  seeded sub-box fills per array (random.Random(251219851), uniform(-4, 4)
  rounded to 3 decimals), two bench steps of 100 iterations.
* C3 — 2-D acoustic wave r=2 16384^2 fp32: one bench step (100 wave steps)
  against the fp32 strict route; bar: bit-equal (and within the north star's
  1e-5 relative tolerance, asserted separately so a failure says which).
* lap16k — the paper's 2-D Laplace per-GPU shape, 16384^2 fp64 (est_tc
  ping-pong chains), bench steps up to a CUDA-graph replay.

Bar for fp64: bit-exact (NaNs compared as a class). Arrays are fetched and
compared one at a time to bound host memory (C4: 3 x 8.6 GB resident).
"""

import gc
import os
import sys

import numpy as np
import pytest

from oracle.oracle import bits_equal, strict_execute_dag

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402  (the benchmark's own job/step builders)


def _threads() -> int:
    return len(os.sched_getaffinity(0))


def _oracle(setup_prog, blob: bytes, steps: int) -> dict:
    """Strict oracle over the setup program then `steps` copies of the step DAG."""
    from paper_2512_19851_b200.wire import decode_dag

    arrays = strict_execute_dag(setup_prog.dag, setup_prog.shapes, setup_prog.dtypes, threads=_threads())
    step = decode_dag(blob)
    for _ in range(steps):
        strict_execute_dag(step, setup_prog.shapes, setup_prog.dtypes, arrays=arrays, threads=_threads())
    return arrays


def _job_with_fills(w, fills: int):
    """bench.build_job's job, but the setup program seeds `fills` sub-box fills per array."""
    from paper_2512_19851_b200.programs import DagProgram, heat3d_setup
    from paper_2512_19851_b200.session import GpuJob

    job = GpuJob(workers=1)
    prog = DagProgram()
    arrays = heat3d_setup(prog, w["n"], seed_fills=fills)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    job.run(prog.dag)
    return job, prog, arrays


def _compare_all(job, want: dict, rtol: float | None = None) -> None:
    for aid in sorted(want):
        got = job.fetch(aid)
        exp = want[aid]
        if rtol is not None:
            np.testing.assert_allclose(got, exp, rtol=rtol, atol=0)
        assert bits_equal(got, exp), (aid, float(np.nanmax(np.abs(got.astype(np.float64) - exp))))
        del got
        gc.collect()


def test_c4_bench_steps_bit_exact_with_graph_replay():
    """C4 exactly as bench.py runs it: est_tb chains, steps up to the first graph replay."""
    w = bench.WORKLOADS["c4"]
    job, prog, arrays = bench.build_job(w, 1, 0)
    try:
        blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
        ex = job.executors[0]
        job.run_bytes(blob)
        assert ex._scratch, "the default C4 path did not run the temporal chain (est_tb)"
        steps = 1
        while ex.replays == 0 and steps < 5:   # recorded, captured, then replayed (bench warm-up >= 3)
            job.run_bytes(blob)
            steps += 1
        job.sync()
        assert ex.replays == 1, "the repeated bench step was not replayed from a CUDA graph"
        want = _oracle(prog, blob, steps)
        _compare_all(job, want)
    finally:
        job.close()


def test_c4_geometry_seeded_fills_bit_exact():
    """The C4 kernel geometry (1024^3, default chain config) on a non-trivial interior."""
    w = bench.WORKLOADS["c4"]
    job, prog, arrays = _job_with_fills(w, 64)
    try:
        blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
        job.run_bytes(blob)
        assert job.executors[0]._scratch, "the temporal chain did not run"
        want = _oracle(prog, blob, 1)
        _compare_all(job, want)
    finally:
        job.close()


def test_c2_512_seeded_fills_bit_exact():
    """C2 parity variant: 512^3, 64 seeded fills per array, 100 iterations."""
    w = bench.WORKLOADS["c2"]
    job, prog, arrays = _job_with_fills(w, 64)
    try:
        blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
        job.run_bytes(blob)
        job.run_bytes(blob)             # second step: graph capture / replay path
        want = _oracle(prog, blob, 2)
        _compare_all(job, want)
    finally:
        job.close()


def test_c3_16384_fp32_wave():
    """C3 at its bench size: 16384^2 fp32, one bench step of 100 wave steps."""
    w = bench.WORKLOADS["c3"]
    job, prog, arrays = bench.build_job(w, 1, 0)
    try:
        blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
        job.run_bytes(blob)
        want = _oracle(prog, blob, 1)
        _compare_all(job, want, rtol=1e-5)
    finally:
        job.close()


def test_lap16k_bench_steps_bit_exact_with_graph_replay():
    """The paper's 2-D Laplace shape (16384^2 fp64, bench workload `lap16k`)
    as bench.py runs it: two-sweep rank-2 chains (est_tc, B stored only by a
    run's last chain), steps up to the first CUDA-graph replay."""
    w = bench.WORKLOADS["lap16k"]
    job, prog, arrays = bench.build_job(w, 1, 0)
    try:
        blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
        ex = job.executors[0]
        job.run_bytes(blob)
        assert ex._scratch, "the default lap16k path did not run the rank-2 chain (est_tc)"
        steps = 1
        while ex.replays == 0 and steps < 5:
            job.run_bytes(blob)
            steps += 1
        job.sync()
        assert ex.replays == 1
        want = _oracle(prog, blob, steps)
        _compare_all(job, want)
    finally:
        job.close()
