"""GPU parity of the resident-smem skeleton (resident.py): a small rank-2
ping-pong run held in shared memory, KM sweeps per pair of grid barriers with
an overlapped ghost zone. Bit-identical to the strict oracle in fp64 and fp32.

Cases: BASELINE C1 (Laplace 1024² x 100), partial tiles and grids smaller than
one tile, an output slice S that is not the interior (so border cells of the
two arrays differ and must come from the array each sweep reads), radius 2,
asymmetric and diagonal offsets, sweep counts that leave a short last block,
several KM / rows-per-thread settings, and CUDA-graph replay across batches."""

import random

import numpy as np
import pytest

from oracle.oracle import bits_equal, strict_execute_dag
from paper_2512_19851_b200.ir import add, cst, mul, ref, sub
from paper_2512_19851_b200.programs import DagProgram
from paper_2512_19851_b200.session import GpuJob, run_program
from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64, encode_dag

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def only_rsm(monkeypatch):
    from paper_2512_19851_b200 import resident, temporal
    monkeypatch.setattr(resident, "SMEM_ENABLED", True)
    monkeypatch.setattr(temporal, "ENABLED", False)


def _ran(job) -> bool:
    return bool(job.executors[0]._bar)


def _fills(prog, arrays, shape, rng, n_fills):
    for u in arrays:
        for _ in range(n_fills):
            lo = [rng.randrange(0, e) for e in shape]
            hi = [rng.randrange(l + 1, e + 1) for l, e in zip(lo, shape)]
            prog.assign(u, tuple(slice(l, h) for l, h in zip(lo, hi)), cst(round(rng.uniform(-4, 4), 3)))


def _star2d(u, box, radius=1, diag=False):
    def at(dy, dx):
        return ref(u, ((box[0][0] + dy, box[0][1] + dy), (box[1][0] + dx, box[1][1] + dx)))
    s = None
    for d in range(1, radius + 1):
        for off in ((-d, 0), (d, 0), (0, -d), (0, d)) + (((-d, d), (d, -d)) if diag else ()):
            s = at(*off) if s is None else add(s, at(*off))
    return mul(cst(0.125), sub(s, at(0, 0)))


def _program(shape, box, iters, radius=1, diag=False, dtype=DTYPE_F64, seed=0, fills=10):
    prog = DagProgram()
    u1 = prog.create_array(shape, dtype)
    u2 = prog.create_array(shape, dtype)
    _fills(prog, (u1, u2), shape, random.Random(seed), fills)
    sl = tuple(slice(lo, hi) for lo, hi in box)
    a, b = u1, u2
    for _ in range(iters):
        prog.assign(b, sl, _star2d(a, box, radius, diag))
        a, b = b, a
    return prog


def _check(prog, expect_ran=True):
    want = strict_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        assert _ran(job) == expect_ran
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


def test_c1_laplace_1024_x100():
    from oracle.oracle import laplace_reference
    from paper_2512_19851_b200.programs import laplace_program
    prog = DagProgram()
    names = laplace_program(prog, 1024, 100)
    job, stats = run_program(prog, fused=True)
    try:
        assert _ran(job)
        assert bits_equal(job.fetch(names["u"]), laplace_reference(1024, 100))
    finally:
        job.close()


@pytest.mark.parametrize("shape,box,iters", [
    ((64, 64), ((1, 63), (1, 63)), 9),         # grid smaller than one tile per SM needs
    ((200, 333), ((1, 199), (1, 332)), 17),    # ragged tiles, short last block
    ((130, 70), ((5, 120), (3, 60)), 8),       # S off the interior: borders differ per array
    ((1000, 777), ((2, 998), (1, 776)), 2),    # shortest chain
    ((40, 1500), ((1, 39), (1, 1499)), 11),
])
def test_shapes_bit_exact(shape, box, iters):
    _check(_program(shape, box, iters, seed=len(shape) + iters))


@pytest.mark.parametrize("radius,diag", [(2, False), (1, True), (2, True)])
def test_radius_and_diagonals(radius, diag):
    r = radius
    _check(_program((150, 260), ((r, 150 - r), (r, 260 - r)), 10, radius, diag, seed=7))


def test_asymmetric_offsets():
    prog = DagProgram()
    shape = (96, 160)
    u1, u2 = prog.create_array(shape), prog.create_array(shape)
    _fills(prog, (u1, u2), shape, random.Random(3), 8)
    box = ((0, 94), (2, 160))
    at = lambda u, dy, dx: ref(u, ((box[0][0] + dy, box[0][1] + dy), (box[1][0] + dx, box[1][1] + dx)))
    a, b = u1, u2
    for _ in range(12):
        prog.assign(b, tuple(slice(*x) for x in box), add(mul(cst(0.5), at(a, 2, -2)), mul(cst(0.25), at(a, 1, 0))))
        a, b = b, a
    _check(prog)


def test_fp32():
    prog = _program((300, 300), ((1, 299), (1, 299)), 13, dtype=DTYPE_F32, seed=11)
    _check(prog)


@pytest.mark.parametrize("km,rpt", [(1, 8), (2, 4), (3, 1), (16, 8), (5, 2)])
def test_block_and_rows_settings(km, rpt, monkeypatch):
    from paper_2512_19851_b200 import resident
    monkeypatch.setattr(resident, "SMEM_KM", km)
    monkeypatch.setattr(resident, "SMEM_RPT", rpt)
    _check(_program((257, 190), ((1, 256), (1, 189)), 19, seed=km * 10 + rpt))


def test_too_large_grid_runs_node_by_node():
    # 2 x 4096^2 f64 does not fit one tile per SM in shared memory
    prog = _program((4096, 4096), ((1, 4095), (1, 4095)), 3, fills=4)
    _check(prog, expect_ran=False)


def test_graph_replay_batches():
    shape, box, per, batches = (512, 512), ((1, 511), (1, 511)), 10, 5
    setup = DagProgram()
    u1, u2 = setup.create_array(shape), setup.create_array(shape)
    _fills(setup, (u1, u2), shape, random.Random(5), 12)
    step = DagProgram()
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    sl = tuple(slice(*x) for x in box)
    a, b = u1, u2
    for _ in range(per):
        step.assign(b, sl, _star2d(a, box))
        a, b = b, a
    full = DagProgram()
    f1, f2 = full.create_array(shape), full.create_array(shape)
    _fills(full, (f1, f2), shape, random.Random(5), 12)
    a, b = f1, f2
    for _ in range(per * batches):
        full.assign(b, sl, _star2d(a, box))
        a, b = b, a
    want = strict_execute_dag(full.dag, full.shapes)
    blob = encode_dag(step.dag)
    with GpuJob() as job:
        for aid in sorted(setup.shapes):
            job.create_array(setup.shapes[aid])
        job.run(setup.dag)
        stats = [job.run_bytes(blob) for _ in range(batches)]
        assert job.executors[0].replays >= 2
        assert stats[1][0].gpu_launches == 1
        for aid in setup.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid


@pytest.mark.parametrize("seed", range(24))
def test_random_chains(seed):
    """Random ping-pong chains: shape, output box, offsets (radius <= 3 per
    axis, any sign, cross terms), constants, dtype and sweep count."""
    rng = random.Random(9000 + seed)
    ny, nx = rng.randrange(12, 320), rng.randrange(12, 320)
    r = (rng.randrange(0, 4), rng.randrange(0, 4))
    lo = (rng.randrange(r[0], r[0] + 4), rng.randrange(r[1], r[1] + 4))
    hi = (ny - rng.randrange(r[0], r[0] + 4), nx - rng.randrange(r[1], r[1] + 4))
    if hi[0] <= lo[0] or hi[1] <= lo[1]:
        pytest.skip("empty box")
    box = (lo, hi)
    dtype = rng.choice((DTYPE_F32, DTYPE_F64))
    prog = DagProgram()
    u1, u2 = prog.create_array((ny, nx), dtype), prog.create_array((ny, nx), dtype)
    _fills(prog, (u1, u2), (ny, nx), rng, 8)
    offs = {(0, 0)} | {(rng.randrange(-r[0], r[0] + 1), rng.randrange(-r[1], r[1] + 1)) for _ in range(5)}
    offs = sorted(offs)
    consts = [round(rng.uniform(-1, 1), 4) for _ in offs]
    signs = [rng.random() < 0.7 for _ in offs]

    def tree(u):
        s = None
        for (dy, dx), c, plus in zip(offs, consts, signs):
            t = mul(cst(c), ref(u, ((lo[0] + dy, hi[0] + dy), (lo[1] + dx, hi[1] + dx))))
            s = t if s is None else (add(s, t) if plus else sub(s, t))
        return s

    a, b = u1, u2
    sl = (slice(lo[0], hi[0]), slice(lo[1], hi[1]))
    for _ in range(rng.randrange(2, 26)):
        prog.assign(b, sl, tree(a))
        a, b = b, a
    want = strict_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        assert _ran(job)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), (seed, aid)
    finally:
        job.close()
