"""GPU parity: the generated sm_100a kernels (through libest.so) against the
pinned oracle / the reference's own stored outputs. Bit-exact for float64
(NaNs compared as a class), 1e-5 relative for float32 (north star)."""

import random

import numpy as np
import pytest

from golden_cases import case_names, get_case
from oracle.oracle import (
    bits_equal, heat3d_reference, laplace_reference, reference_execute_dag, strict_execute_dag)
from paper_2512_19851_b200.errors import MalformedDag, OffsetExceedsTileWidth
from paper_2512_19851_b200.ir import Dag, DagNode, add, compute_edges, cst, mul, ref, sub
from paper_2512_19851_b200.programs import (
    DagProgram, heat3d_program, laplace_program, wave2d_program)
from paper_2512_19851_b200.session import GpuJob, run_program
from paper_2512_19851_b200.wire import DTYPE_F32, decode_dag
from progs import random_program_2d, random_program_3d

pytestmark = pytest.mark.gpu

F32_RTOL = 1e-5


class _Prog:
    def __init__(self, dag, shapes, dtypes=None):
        self.dag, self.shapes, self.dtypes = dag, shapes, dtypes or {}


def _fits(shapes, workers, odf, depth=2):
    from paper_2512_19851_b200.tiles import decompose
    shape = next(iter(shapes.values()))
    try:
        d = decompose(shape, workers, odf)
        ext = d.tile_extents(shape)
    except Exception:
        return False
    return min(ext if len(shape) == 2 else ext[:1]) > depth


@pytest.mark.parametrize("name", case_names())
def test_golden_case_single_gpu(name):
    _, blob, shapes, expected, rounds, batch = get_case(name)
    prog = _Prog(decode_dag(blob), shapes)
    job, _ = run_program(prog, batch=batch)
    try:
        for aid, want in expected.items():
            assert bits_equal(job.fetch(aid), want), (name, aid)
        assert job.rounds_by_array() == rounds
    finally:
        job.close()


@pytest.mark.parametrize("name", [n for n in case_names() if n.startswith(("laplace", "cavity", "rand2d_00", "heat3d", "rank1", "rand3d_00"))])
@pytest.mark.parametrize("workers,odf", [(1, 4), (2, 1), (4, 1), (2, 2)])
def test_golden_case_multi_tile(name, workers, odf):
    """Co-located strips (odf > 1) and peer pulls between in-process workers."""
    _, blob, shapes, expected, rounds, batch = get_case(name)
    if not _fits(shapes, workers, odf):
        pytest.skip("tiles narrower than the stencil radius")
    prog = _Prog(decode_dag(blob), shapes)
    job, stats = run_program(prog, workers=workers, odf=odf, batch=batch)
    try:
        for aid, want in expected.items():
            assert bits_equal(job.fetch(aid), want), (name, aid, workers, odf)
        assert job.rounds_by_array() == rounds
        if workers == 1:
            assert all(s.net_messages == 0 for batch_stats in stats for s in batch_stats)
    finally:
        job.close()


def test_laplace_1024x100_bit_exact():
    prog = DagProgram()
    names = laplace_program(prog, 1024, 100)
    job, stats = run_program(prog, fused=True)
    try:
        assert bits_equal(job.fetch(names["u"]), laplace_reference(1024, 100))
    finally:
        job.close()


@pytest.mark.parametrize("n", [64, 128])
def test_heat3d_bit_exact(n):
    prog = DagProgram()
    names = heat3d_program(prog, n, 12, seed_fills=16)
    want = strict_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog, fused=True)
    try:
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


def test_heat3d_matches_handwritten_solver():
    prog = DagProgram()
    names = heat3d_program(prog, 48, 9)
    job, _ = run_program(prog)
    try:
        assert bits_equal(job.fetch(names["u"]), heat3d_reference(48, 9))
    finally:
        job.close()


def test_random_programs_200():
    rng = random.Random(20251219)
    for k in range(200):
        prog = random_program_2d(rng) if k % 2 == 0 else random_program_3d(rng)
        want = reference_execute_dag(prog.dag, prog.shapes)
        job, _ = run_program(prog, fused=bool(k % 3 == 0))
        try:
            for aid in prog.shapes:
                assert bits_equal(job.fetch(aid), want[aid]), (k, aid)
        finally:
            job.close()


def test_wave2d_fp32_within_tolerance():
    prog = DagProgram()
    names = wave2d_program(prog, 256, 40, dtype=DTYPE_F32)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        got = job.fetch(names["u"])
        ref_ = want[names["u"]]
        assert got.dtype == np.float32
        scale = np.abs(ref_).max()
        assert scale > 0
        np.testing.assert_allclose(got, ref_, rtol=F32_RTOL, atol=F32_RTOL * scale)
        # the plan order is preserved, so float32 is in fact bit-identical
        assert bits_equal(got, ref_)
    finally:
        job.close()


def test_depth_growth_across_batches_multi_worker():
    prog = DagProgram()
    a = prog.create_array((16, 16))
    b = prog.create_array((16, 16))
    c = prog.create_array((16, 16))
    prog.assign(a, ((0, 16), (0, 5)), cst(9.0))
    prog.assign(b, (slice(1, -1), slice(1, -1)), ref(a, (slice(0, 14), slice(1, -1))))
    cut = len(prog.dag.nodes)
    prog.assign(c, (slice(2, -2), slice(2, -2)), ref(a, (slice(0, 12), slice(2, -2))))
    first = Dag(prog.dag.nodes[:cut], compute_edges(prog.dag.nodes[:cut]), prog.dag.ast_table)
    rest = [DagNode(i, n.statements) for i, n in enumerate(prog.dag.nodes[cut:])]
    second = Dag(rest, compute_edges(rest), prog.dag.ast_table)
    want = reference_execute_dag(prog.dag, prog.shapes)
    with GpuJob(workers=4) as job:
        for aid in sorted(prog.shapes):
            job.create_array(prog.shapes[aid])
        job.run(first)
        job.run(second)
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid])
        assert job.rounds_by_array()[a] == 2


def test_offset_exceeding_tile_width_rejected():
    prog = DagProgram()
    a = prog.create_array((8, 8))
    b = prog.create_array((8, 8))
    prog.assign(b, (slice(2, None), slice(None)), ref(a, (slice(None, -2), slice(None))))
    with GpuJob(workers=1, odf=16) as job:
        for aid in sorted(prog.shapes):
            job.create_array(prog.shapes[aid])
        with pytest.raises(OffsetExceedsTileWidth):
            job.run(prog.dag)


def test_dependent_statements_in_one_node_rejected():
    prog = DagProgram()
    a = prog.create_array((8, 8))
    b = prog.create_array((8, 8))
    c = prog.create_array((8, 8))
    prog.assign(b, (slice(None), slice(None)), ref(a, (slice(None), slice(None))))
    prog.assign(c, (slice(None), slice(None)), ref(b, (slice(None), slice(None))))
    nodes = prog.dag.nodes
    merged = DagNode(0, [s for n in nodes[3:] for s in n.statements])
    dag = Dag([*[DagNode(i, n.statements) for i, n in enumerate(nodes[:3])],
               DagNode(3, merged.statements)], set(), prog.dag.ast_table)
    dag.edges = compute_edges(dag.nodes)
    with GpuJob() as job:
        for aid in sorted(prog.shapes):
            job.create_array(prog.shapes[aid])
        with pytest.raises(MalformedDag):
            job.run(dag)


def test_empty_dag():
    with GpuJob(workers=2) as job:
        job.create_array((8, 8))
        stats = job.run(Dag([], set(), []))
        assert all(s.nodes_executed == 0 for s in stats)


@pytest.mark.parametrize("radii", [((0, 0, 0), (2, 1, 1)), ((2, 2, 2), (0, 1, 0)), ((1, 1, 1), (3, 0, 2))])
def test_stream_multi_slot_mixed_radius(radii):
    """Two-input 3-D statements whose slots have different z-radii (the TMA
    producer must issue planes in consumption order, not slot order)."""
    from paper_2512_19851_b200.ir import add, mul
    n = 40
    prog = DagProgram()
    a = prog.create_array((n, n, n))
    b = prog.create_array((n, n, n))
    c = prog.create_array((n, n, n))
    prog.assign(a, ((3, 30), (5, 33), (2, 37)), cst(1.25))
    prog.assign(b, ((6, 38), (1, 20), (4, 31)), cst(-0.5))
    m = 4
    box = (slice(m, n - m),) * 3

    def shifted(arr, off):
        return ref(arr, tuple(slice(m + o, n - m + o) for o in off))
    (ra, rb) = radii
    expr = add(mul(shifted(a, (-ra[0], ra[1], -ra[2])), shifted(b, (rb[0], -rb[1], rb[2]))),
               add(shifted(a, (ra[0], -ra[1], ra[2])), shifted(b, (-rb[0], rb[1], -rb[2]))))
    prog.assign(c, box, expr)
    want = reference_execute_dag(prog.dag, prog.shapes)
    job, _ = run_program(prog)
    try:
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


def test_large_2d_tiles_bit_exact():
    """Rank-2 boxes of >= stream.SMALL_2D_POINTS points run the tall-tile
    configuration (128 x 48, 12 consecutive rows per thread)."""
    from paper_2512_19851_b200 import stream
    n = 3072
    assert (n - 4) ** 2 >= stream.SMALL_2D_POINTS
    prog = DagProgram()
    names = wave2d_program(prog, n, 6, dtype=DTYPE_F32)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog)
    try:
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()
    prog = DagProgram()
    names = laplace_program(prog, 3000, 5)
    job, _ = run_program(prog, fused=True)
    try:
        assert bits_equal(job.fetch(names["u"]), laplace_reference(3000, 5))
    finally:
        job.close()


def test_fused_cavity_split_into_stream_launches():
    """Fused nodes whose independent statements are large run one stream launch
    per statement (plus one point launch for the small rest); bit-exact."""
    from paper_2512_19851_b200.programs import cavity_program
    prog = DagProgram()
    names = cavity_program(prog, 512, 2)
    want = reference_execute_dag(prog.dag, prog.shapes)
    job, stats = run_program(prog, fused=True)
    try:
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
        # kernel_launches keeps the reference definition (one per node per tile)
        assert sum(s.kernel_launches for b in stats for s in b) == sum(s.nodes_executed for b in stats for s in b)
    finally:
        job.close()


@pytest.mark.parametrize("shape", [(40, 40, 40), (96, 80), (500,)])
def test_ieee_specials_propagate(shape):
    """inf / NaN / signed zero flow through the generated kernels exactly as
    through numpy (executor.py:130, oracle.py:81): 1/0, 0/0, sqrt of a
    negative, neg / abs of -0.0 and NaN, then a stencil over the result."""
    from paper_2512_19851_b200.ir import div, neg, una
    rank = len(shape)
    prog = DagProgram()
    a, b, c = (prog.create_array(shape) for _ in range(3))
    q = [n // 4 for n in shape]
    prog.assign(a, tuple((k, 2 * k) for k in q), cst(-2.0))
    prog.assign(a, tuple((2 * k, 3 * k) for k in q), cst(-0.0))
    full = tuple(slice(None) for _ in shape)
    prog.assign(b, full, div(cst(1.0), ref(a, full)))                       # +-inf, -0.5
    prog.assign(c, full, add(div(ref(a, full), ref(a, full)),              # NaN where a == 0
                             una("abs", neg(una("sqrt", ref(a, full))))))   # NaN for negatives
    inner = tuple(slice(1, -1) for _ in shape)
    terms = None
    for ax in range(rank):
        for d in (-1, 1):
            sl = tuple(slice(1 + (d if k == ax else 0), n - 1 + (d if k == ax else 0)) for k, n in enumerate(shape))
            t = ref(b, sl)
            terms = t if terms is None else add(terms, t)
    prog.assign(a, inner, sub(mul(cst(0.5), terms), ref(c, inner)))
    want = reference_execute_dag(prog.dag, prog.shapes)
    assert np.isnan(want[a]).any() and np.isinf(want[b]).any()
    job, _ = run_program(prog)
    try:
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


def test_fused_node_mixing_ranks_and_dtypes():
    """fuse() may merge independent statements on arrays of different rank or
    element type into one node; each kind gets its own launch."""
    from paper_2512_19851_b200.ir import fuse
    prog = DagProgram()
    a2, b2 = prog.create_array((16, 16)), prog.create_array((16, 16))
    a3, b3 = prog.create_array((16, 16, 16)), prog.create_array((16, 16, 16))
    f2, g2 = prog.create_array((16, 16), DTYPE_F32), prog.create_array((16, 16), DTYPE_F32)
    prog.assign(a2, ((2, 9), (3, 12)), cst(1.5))
    prog.assign(a3, ((2, 9), (3, 12), (1, 14)), cst(-2.25))
    prog.assign(f2, ((4, 13), (1, 8)), cst(0.125))
    i2, i3 = (slice(1, -1),) * 2, (slice(1, -1),) * 3
    prog.assign(b2, i2, add(ref(a2, (slice(0, -2), slice(1, -1))), ref(a2, (slice(2, None), slice(1, -1)))))
    prog.assign(b3, i3, add(ref(a3, (slice(0, -2), slice(1, -1), slice(1, -1))), ref(a3, i3)))
    prog.assign(g2, i2, mul(cst(3.0), ref(f2, (slice(1, -1), slice(2, None)))))
    fused = fuse(prog.dag)
    assert any(len(n.statements) > 1 for n in fused.nodes)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog, fused=True)
    try:
        for aid in prog.shapes:
            assert bits_equal(job.fetch(aid), want[aid]), aid
    finally:
        job.close()


@pytest.mark.parametrize("workers,odf", [(2, 1), (1, 4), (2, 2), (4, 1)])
def test_wave2d_fp32_multi_tile(workers, odf):
    """fp32 halo strips (4-byte copies) between co-located tiles and peers."""
    prog = DagProgram()
    names = wave2d_program(prog, 128, 16, dtype=DTYPE_F32)
    want = reference_execute_dag(prog.dag, prog.shapes, prog.dtypes)
    job, _ = run_program(prog, workers=workers, odf=odf)
    try:
        for aid in prog.shapes:
            got = job.fetch(aid)
            assert got.dtype == np.float32 and bits_equal(got, want[aid]), (aid, workers, odf)
    finally:
        job.close()
