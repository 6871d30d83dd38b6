"""GPU parity of the rank-2 two-sweep chain skeleton temporal2d.py ("tc"):
ping-pong runs (2-D Jacobi, arity 1) and rotation runs (the acoustic wave
u2 = f(u1, u0), arity 2), bit-identical to the oracle (fp64; fp32 within the
north star's 1e-5, in fact bit-identical because the plan order is kept).

Cases: partial x tiles and y chunks, output slices that are not the full
interior and start off the 16-byte vector grid, radius 1 and 2, odd step
counts (a leftover node on the single-sweep kernels), runs that end with
arrays in their twin buffers (copied back), several batches with CUDA-graph
replay, and that the fused kernel really ran."""

import random

import numpy as np
import pytest

from oracle.oracle import bits_equal, reference_execute_dag, strict_execute_dag
from paper_2512_19851_b200.ir import add, cst, mul, ref, sub
from paper_2512_19851_b200.programs import DagProgram, wave2d_setup, wave2d_steps
from paper_2512_19851_b200.session import GpuJob, run_program
from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64, encode_dag

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "vec16"])
def chains_at_test_sizes(request, monkeypatch):
    """Every case runs with the default layout (8-byte vectors for fp32
    rotations) and with 16-byte vectors everywhere."""
    import dataclasses

    from paper_2512_19851_b200 import resident, temporal2d
    if request.param == "vec16":
        monkeypatch.setattr(temporal2d, "DEFAULT", dataclasses.replace(temporal2d.DEFAULT, vec=16))
    monkeypatch.setattr(temporal2d, "ENABLED", True)
    monkeypatch.setattr(temporal2d, "MIN_POINTS", 0)
    monkeypatch.setattr(temporal2d, "ROTATIONS", True)  # opt-in by default (measured slower at C3)
    monkeypatch.setattr(resident, "SMEM_ENABLED", False)  # the small-grid chain has its own suite


def _fills(prog, arrays, n, count, seed, dtype=DTYPE_F64):
    """Seeded sub-box constant fills (the SURVEY §8(d) parity variant, tests/util.py:55-64)."""
    rng = random.Random(seed)
    for a in arrays:
        for _ in range(count):
            y0, x0 = rng.randrange(0, n - 2), rng.randrange(0, n - 2)
            y1, x1 = rng.randrange(y0 + 1, min(n, y0 + n // 3) + 1), rng.randrange(x0 + 1, min(n, x0 + n // 3) + 1)
            prog.assign(a, (slice(y0, y1), slice(x0, x1)), cst(round(rng.uniform(-4, 4), 3)))


def _star2(u, box, radius=1):
    def sh(axis, d):
        return ref(u, tuple(slice(lo + (d if k == axis else 0), hi + (d if k == axis else 0))
                            for k, (lo, hi) in enumerate(box)))
    s = None
    for ax in (0, 1):
        for d in range(1, radius + 1):
            for dd in (-d, d):
                s = sh(ax, dd) if s is None else add(s, sh(ax, dd))
    return mul(cst(0.125), sub(s, ref(u, tuple(slice(lo, hi) for lo, hi in box))))


def _ran(job) -> bool:
    return bool(job.executors[0]._scratch)


@pytest.mark.parametrize("n,iters,box,radius", [
    (64, 8, ((1, 63), (1, 63)), 1),
    (300, 6, ((1, 299), (1, 299)), 1),      # partial x tile, several y chunks
    (517, 10, ((3, 511), (5, 509)), 1),     # S off the vector grid
    (260, 8, ((2, 258), (2, 258)), 2),      # radius 2
    (200, 9, ((2, 197), (3, 197)), 2),      # odd sweep count: a leftover node
])
def test_pingpong_chains_bit_exact(n, iters, box, radius):
    prog = DagProgram()
    u1, u2 = prog.create_array((n, n)), prog.create_array((n, n))
    _fills(prog, (u1, u2), n, 16, seed=n * 7 + iters)
    for _ in range(iters):
        prog.assign(u2, box, _star2(u1, box, radius))
        u1, u2 = u2, u1
    want = strict_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog)
    try:
        assert _ran(job), "the tc chain did not run"
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), (n, iters, aid)
    finally:
        job.close()


@pytest.mark.parametrize("n,steps,dtype", [
    (64, 6, DTYPE_F32), (256, 7, DTYPE_F32), (517, 12, DTYPE_F32), (1000, 9, DTYPE_F32),
    (300, 8, DTYPE_F64), (130, 5, DTYPE_F64),
])
def test_wave_rotation_chains_bit_exact(n, steps, dtype):
    prog = DagProgram()
    u0, u1, u2 = wave2d_setup(prog, n, dtype)
    _fills(prog, (u0, u1), n, 12, seed=steps * 31 + n, dtype=dtype)
    wave2d_steps(prog, u0, u1, u2, steps)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        assert _ran(job)
        for aid in prog.shapes:
            got = job.fetch(aid)
            if dtype == DTYPE_F32:
                np.testing.assert_allclose(got, want[aid], rtol=1e-5, atol=1e-5 * max(1.0, np.abs(want[aid]).max()))
            assert bits_equal(got, want[aid]), (n, steps, aid)
    finally:
        job.close()


def test_wave_off_grid_slice_bit_exact():
    """A rotation whose output slice is not [2:-2, 2:-2] (S off the vector grid)."""
    n = 333
    box = ((3, 325), (5, 330))
    prog = DagProgram()
    u = [prog.create_array((n, n), DTYPE_F32) for _ in range(3)]
    _fills(prog, u, n, 10, seed=5, dtype=DTYPE_F32)

    def at(a, dy, dx):
        return ref(a, tuple(slice(lo + d, hi + d) for (lo, hi), d in zip(box, (dy, dx))))
    for _ in range(8):
        lap = add(add(at(u[1], -2, 0), at(u[1], 1, 0)), add(at(u[1], 0, -1), at(u[1], 0, 2)))
        e = add(sub(mul(cst(2.0), at(u[1], 0, 0)), at(u[0], 0, 0)), mul(cst(0.05), lap))
        prog.assign(u[2], box, e)
        u = [u[1], u[2], u[0]]
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        assert _ran(job)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


@pytest.mark.parametrize("steps_per_batch", [10, 9])
def test_wave_batches_graph_replay_bit_exact(steps_per_batch):
    """Steady-state wave batches replay a captured CUDA graph holding the tc
    kernels. The rotation's roles shift by steps mod 3 between batches, so
    the DAG bytes repeat every third batch: captured at the second sighting,
    replayed from the third."""
    n, batches = 384, 8
    setup = DagProgram()
    u0, u1, u2 = wave2d_setup(setup, n, DTYPE_F32)
    full = DagProgram()
    f0, f1, f2 = wave2d_setup(full, n, DTYPE_F32)
    wave2d_steps(full, f0, f1, f2, steps_per_batch * batches)
    want = reference_execute_dag(full.dag, full.shapes, full.dtypes)
    with GpuJob() as job:
        for aid in sorted(setup.shapes):
            job.create_array(setup.shapes[aid], DTYPE_F32)
        job.run(setup.dag)
        roles = (u0, u1, u2)
        for _ in range(batches):
            step = DagProgram()
            for a in sorted(setup.shapes):
                step.builder.declare_array(a, setup.shapes[a])
            out = wave2d_steps(step, *roles, steps_per_batch)
            roles = (out["prev"], out["u"], out["next"])
            job.run_bytes(encode_dag(step.dag))
        assert _ran(job)
        assert job.executors[0].replays >= 1
        for aid in setup.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid


def test_chain_disabled_equals_enabled():
    n = 400
    prog = DagProgram()
    u0, u1, u2 = wave2d_setup(prog, n, DTYPE_F32)
    _fills(prog, (u0, u1), n, 8, seed=11, dtype=DTYPE_F32)
    wave2d_steps(prog, u0, u1, u2, 11)
    outs = []
    for on in (True, False):
        job = GpuJob()
        try:
            for aid in sorted(prog.shapes):
                job.create_array(prog.shapes[aid], DTYPE_F32)
            job.executors[0].temporal = on
            job.run(prog.dag)
            outs.append([job.fetch(a) for a in sorted(prog.shapes)])
            assert _ran(job) == on
        finally:
            job.close()
    for x, y in zip(*outs):
        assert bits_equal(x, y)
