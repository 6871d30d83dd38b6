"""GPU parity of the fused-chain skeleton temporal.py (K fused ping-pong
sweeps with a twin buffer): bit-identical to the oracle (fp64; fp32 within the
north star's 1e-5, in fact bit-identical because the plan order is kept).
Every test runs with the default K = 2 chain and with a K = 4 chain (smaller
tiles so its three intermediate plane rings fit shared memory).

Cases cover partial tiles, output slices that are not the full interior, a
radius-2 and an asymmetric stencil, odd iteration counts (a leftover sweep on
the node-by-node kernel), several batches with CUDA-graph replay, and that the
fused kernel really ran (launch counts)."""

import numpy as np
import pytest

from oracle.oracle import bits_equal, reference_execute_dag, strict_execute_dag
from paper_2512_19851_b200.ir import add, cst, mul, ref, sub
from paper_2512_19851_b200.programs import DagProgram, heat3d_program, heat3d_setup, heat3d_tree
from paper_2512_19851_b200.session import GpuJob, run_program
from paper_2512_19851_b200.wire import DTYPE_F32, encode_dag

pytestmark = pytest.mark.gpu

K4 = dict(k=4, bx=32, by=32)


@pytest.fixture(autouse=True, params=["k2", "k4"])
def mode(request, monkeypatch):
    import dataclasses

    from paper_2512_19851_b200 import resident, temporal
    monkeypatch.setattr(temporal, "ENABLED", True)
    monkeypatch.setattr(resident, "SMEM_ENABLED", False)  # tests/test_gpu_resident_smem.py
    monkeypatch.setattr(temporal, "MIN_POINTS", 0)  # chains at test sizes
    if request.param == "k4":
        monkeypatch.setattr(temporal, "DEFAULT", dataclasses.replace(temporal.DEFAULT, **K4))
    return request.param


def _ran(job, mode) -> bool:
    return bool(job.executors[0]._scratch)


def _chains(mode, sweeps: int) -> bool:
    """A run of `sweeps` ping-pong nodes holds an even number (>= 2) of K-chains."""
    return sweeps >= 2 * (4 if mode == "k4" else 2)


def _fits(prog, mode) -> bool:
    """The chain kernel accepts the program's last statement (radius / shared memory)."""
    from paper_2512_19851_b200 import codegen, temporal
    from paper_2512_19851_b200.analysis import compile_plan
    st = compile_plan(prog.dag.nodes[-1], prog.dag.ast_table).statements[0]
    out = prog.dag.nodes[-1].statements[0].output
    ok = temporal.eligible(codegen.stmt_sig(st, 3), prog.dtypes.get(out, 0))
    assert ok or mode == "k4", "every K = 2 case here must be chainable"
    return ok


def _tb_launches(stats) -> int:
    return sum(s.gpu_launches for b in stats for s in b)


@pytest.mark.parametrize("n,iters", [(24, 4), (40, 8), (67, 6), (64, 13), (130, 4)])
def test_heat3d_chains_bit_exact(n, iters, mode):
    prog = DagProgram()
    heat3d_program(prog, n, iters, seed_fills=12)
    want = strict_execute_dag(prog.dag, prog.shapes)
    job, stats = run_program(prog, fused=True)
    try:
        assert _ran(job, mode) == _chains(mode, iters), "fused chain did not run"
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), (n, iters, aid)
    finally:
        job.close()


def _star(u, box, radius=1, axes=(0, 1, 2)):
    """Ordered sum of the +/- radius neighbours along `axes`, times a constant."""
    def sh(axis, d):
        return ref(u, tuple(slice(lo + (d if k == axis else 0), hi + (d if k == axis else 0))
                            for k, (lo, hi) in enumerate(box)))
    s = None
    for ax in axes:
        for d in range(1, radius + 1):
            for dd in (-d, d):
                term = sh(ax, dd)
                s = term if s is None else add(s, term)
    return mul(cst(0.0625), sub(s, ref(u, tuple(slice(lo, hi) for lo, hi in box))))


@pytest.mark.parametrize("box,radius", [
    (((2, 37), (1, 38), (3, 36)), 1),     # S off-centre, partial tiles in x and y
    (((2, 38), (2, 38), (2, 38)), 2),     # radius-2 star (depth 2)
    (((3, 30), (5, 33), (2, 38)), 2),
])
def test_subbox_chains_bit_exact(box, radius, mode):
    n = 40
    prog = DagProgram()
    u1, u2 = heat3d_setup(prog, n, seed_fills=10)
    for _ in range(8):
        prog.assign(u2, box, _star(u1, box, radius))
        u1, u2 = u2, u1
    want = reference_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog)
    try:
        assert _ran(job, mode) == _fits(prog, mode)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), (box, radius, aid)
    finally:
        job.close()


def test_asymmetric_offsets_bit_exact(mode):
    """Asymmetric z-star stencil (dz in {-2, 1}, in-plane (1,-1) and (-1,0))."""
    n = 36
    prog = DagProgram()
    u1, u2 = heat3d_setup(prog, n, seed_fills=8)
    box = ((2, 34), (1, 35), (2, 35))

    def at(u, dz, dy, dx):
        return ref(u, tuple(slice(lo + d, hi + d) for (lo, hi), d in zip(box, (dz, dy, dx))))
    for _ in range(8):
        e = add(mul(cst(0.5), at(u1, -2, 0, 0)), mul(cst(0.25), at(u1, 0, 1, -1)))
        e = sub(e, mul(cst(0.125), at(u1, 1, 0, 0)))
        e = add(e, at(u1, 0, -1, 0))
        prog.assign(u2, box, e)
        u1, u2 = u2, u1
    want = reference_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog)
    try:
        assert _ran(job, mode) == _fits(prog, mode)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


def test_heat3d_fp32_chains(mode):
    prog = DagProgram()
    heat3d_program(prog, 48, 8, seed_fills=10, dtype=DTYPE_F32)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        assert _ran(job, mode)
        for aid in prog.shapes:
            got = job.fetch(aid)
            assert got.dtype == np.float32
            np.testing.assert_allclose(got, want[aid], rtol=1e-5, atol=1e-5 * np.abs(want[aid]).max())
            assert bits_equal(got, want[aid])
    finally:
        job.close()


def test_repeated_batches_graph_replay_bit_exact(mode):
    """Steady-state batches replay a captured CUDA graph holding the chain kernels."""
    n, per, batches = 48, 10, 5
    setup = DagProgram()
    u1, u2 = heat3d_setup(setup, n, seed_fills=10)
    step = DagProgram()
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    uu1, uu2 = u1, u2
    for _ in range(per):
        step.assign(uu2, (slice(1, -1),) * 3, heat3d_tree(uu1))
        uu1, uu2 = uu2, uu1
    full = DagProgram()
    a1, a2 = heat3d_setup(full, n, seed_fills=10)
    for _ in range(per * batches):
        full.assign(a2, (slice(1, -1),) * 3, heat3d_tree(a1))
        a1, a2 = a2, a1
    want = strict_execute_dag(full.dag, full.shapes)
    blob = encode_dag(step.dag)
    with GpuJob() as job:
        for aid in sorted(setup.shapes):
            job.create_array(setup.shapes[aid])
        job.run(setup.dag)
        stats = [job.run_bytes(blob) for _ in range(batches)]
        assert job.executors[0].replays >= 2
        # 10 sweeps = 4 chains of 2 (K = 2; chain count kept even) or 2 chains of 4
        # + 2 single sweeps + the complement copy
        assert stats[1][0].gpu_launches == {"k2": 4 + 2 + 1, "k4": 2 + 2 + 1}[mode]
        for aid in setup.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid


def test_chain_disabled_equals_enabled(mode):
    prog = DagProgram()
    heat3d_program(prog, 56, 8, seed_fills=12)
    outs = []
    for on in (True, False):
        job = GpuJob()
        job_stats = None
        try:
            for aid in sorted(prog.shapes):
                job.create_array(prog.shapes[aid])
            job.executors[0].temporal = on
            job_stats = job.run(prog.dag)
            outs.append([job.fetch(a) for a in sorted(prog.shapes)])
            assert _ran(job, mode) == on
        finally:
            job.close()
        assert job_stats[0].kernel_launches == len(prog.dag.nodes)
    for x, y in zip(*outs):
        assert bits_equal(x, y)


def test_non_z_star_chain(mode):
    """A diagonal (dz, dx) load is not chainable (z-star only): node by node, bit-exact."""
    n = 32
    prog = DagProgram()
    u1, u2 = heat3d_setup(prog, n, seed_fills=6)
    box = ((1, 31), (1, 31), (1, 31))

    def at(u, dz, dy, dx):
        return ref(u, tuple(slice(lo + d, hi + d) for (lo, hi), d in zip(box, (dz, dy, dx))))
    for _ in range(4):
        prog.assign(u2, box, add(at(u1, -1, 0, 1), mul(cst(0.5), at(u1, 1, 0, 0))))
        u1, u2 = u2, u1
    want = reference_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog)
    try:
        assert not _ran(job, mode)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


def test_wave_is_not_a_chain(mode):
    """The fp32 wave (three rotating arrays) is not a ping-pong chain: node by node."""
    from paper_2512_19851_b200.programs import wave2d_program
    prog = DagProgram()
    names = wave2d_program(prog, 128, 12, dtype=DTYPE_F32)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        assert not _ran(job, mode)
        assert bits_equal(job.fetch(names["u"]), want[names["u"]])
    finally:
        job.close()


def test_default_chain_at_full_scheduling_size(mode, monkeypatch):
    """The default path (tb from MIN_POINTS output points) at a size where it is
    actually scheduled: 648^3 (646^3 = 269.6 M outputs), 8 iterations = 4 / 2
    chains, seeded fills; every array bit-identical to the strict oracle."""
    from paper_2512_19851_b200 import temporal
    monkeypatch.setattr(temporal, "MIN_POINTS", int(temporal.os.environ.get("EST_TB_MIN_POINTS", 1 << 26)))
    prog = DagProgram()
    heat3d_program(prog, 648, 8, seed_fills=12)
    want = strict_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog)
    try:
        assert _ran(job, mode)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


@pytest.mark.parametrize("seed", range(12))
def test_random_z_star_chains(seed, mode):
    """Random 3-D ping-pong chains the tb skeleton accepts (in-plane offsets
    of radius <= 2 in y/x, pure z offsets of radius 1-2, any signs), random
    boxes, constants, dtypes and even sweep counts."""
    import random as _r
    rng = _r.Random(7700 + seed)
    n = (rng.randrange(12, 60), rng.randrange(12, 90), rng.randrange(12, 90))
    rz, ry, rx = rng.randrange(1, 3), rng.randrange(0, 3), rng.randrange(0, 3)
    lo = (rz + rng.randrange(0, 3), ry + rng.randrange(0, 3), rx + rng.randrange(0, 3))
    hi = (n[0] - rz - rng.randrange(0, 3), n[1] - ry - rng.randrange(0, 3), n[2] - rx - rng.randrange(0, 3))
    from paper_2512_19851_b200.wire import DTYPE_F64
    dtype = rng.choice((DTYPE_F32, DTYPE_F64))
    prog = DagProgram()
    u1, u2 = prog.create_array(n, dtype), prog.create_array(n, dtype)
    for u in (u1, u2):
        for _ in range(6):
            a = [rng.randrange(0, e) for e in n]
            b = [rng.randrange(x + 1, e + 1) for x, e in zip(a, n)]
            prog.assign(u, tuple(slice(x, y) for x, y in zip(a, b)), cst(round(rng.uniform(-4, 4), 3)))
    offs = {(0, 0, 0), (rz, 0, 0), (-rng.randrange(1, rz + 1), 0, 0)}
    offs |= {(0, rng.randrange(-ry, ry + 1), rng.randrange(-rx, rx + 1)) for _ in range(4)}
    offs = sorted(offs)
    consts = [round(rng.uniform(-1, 1), 4) for _ in offs]
    signs = [rng.random() < 0.7 for _ in offs]

    def tree(u):
        s = None
        for (dz, dy, dx), c, plus in zip(offs, consts, signs):
            t = mul(cst(c), ref(u, tuple((l + d, h + d) for l, h, d in zip(lo, hi, (dz, dy, dx)))))
            s = t if s is None else (add(s, t) if plus else sub(s, t))
        return s

    a, b = u1, u2
    box = tuple(slice(l, h) for l, h in zip(lo, hi))
    sweeps = 2 * rng.randrange(2, 7)  # >= 4 sweeps: chains come in pairs
    for _ in range(sweeps):
        prog.assign(b, box, tree(a))
        a, b = b, a
    want = strict_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    from paper_2512_19851_b200 import codegen, temporal
    from paper_2512_19851_b200.analysis import compile_plan
    sig = codegen.stmt_sig(compile_plan(prog.dag.nodes[-1], prog.dag.ast_table).statements[0], 3)
    fits = temporal.eligible(sig, dtype)
    job, _ = run_program(prog)
    try:
        assert _ran(job, mode) == (fits and _chains(mode, sweeps))
        assert fits or mode == "k4", "every random K = 2 case must be chainable"
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), (seed, aid)
    finally:
        job.close()


@pytest.mark.parametrize("n,iters,odf,batch", [(32, 8, 2, None), (48, 12, 4, None), (40, 9, 2, 7),
                                               (64, 16, 4, 10)])
def test_slab_chains_bit_exact(n, iters, odf, batch, mode):
    """Several z-slabs in one process: every slab runs the chain on its own
    K*rz-deep halo of A; the intermediate array's ghost planes are computed
    in-chain (virtual rounds). Bit-identical to the oracle, with the
    reference's round counts."""
    from oracle.oracle import EpochSimulator
    from paper_2512_19851_b200.analysis import analyze_dag
    from paper_2512_19851_b200.ir import Dag, DagNode, compute_edges

    prog = DagProgram()
    heat3d_program(prog, n, iters, seed_fills=10)
    want = strict_execute_dag(prog.dag, prog.shapes)
    job, stats = run_program(prog, workers=1, odf=odf, batch=batch)
    try:
        if batch is None and mode == "k2":  # multi-tile chains are K = 2 only (executor._slab_chains_ok)
            assert job.executors[0].store.twins, "slab chains did not run"
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), (n, iters, odf, aid)
        sim = EpochSimulator()
        nodes = prog.dag.nodes
        for k in range(0, len(nodes), batch or len(nodes)):
            part = [DagNode(i, x.statements) for i, x in enumerate(nodes[k:k + (batch or len(nodes))])]
            d = Dag(part, compute_edges(part), prog.dag.ast_table)
            sim.simulate_batch(d, analyze_dag(d, prog.shapes))
        assert job.rounds_by_array() == sim.rounds
    finally:
        job.close()
