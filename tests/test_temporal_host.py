"""Temporal chains (temporal.py) on the host side, CPU with the device test
double: which nodes fuse, that per-node bookkeeping (epochs, rounds, launch
counts) equals unfused execution, the twin buffer and its complement copy,
and the generated kernel's shape."""

import pytest

from fakedev import FakeDevice
from paper_2512_19851_b200 import codegen, temporal
from paper_2512_19851_b200.analysis import compile_plan
from paper_2512_19851_b200.exchange import GpuExchangeManager
from paper_2512_19851_b200.executor import GpuExecutor
from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, heat3d_setup, heat3d_tree
from paper_2512_19851_b200.tiles import ArrayInfo, GpuTileStore, decompose
from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64


@pytest.fixture(autouse=True)
def _small_grids_chain(monkeypatch):
    monkeypatch.setattr(temporal, "MIN_POINTS", 0)  # chains at test sizes (default: large grids only)


def _executor(shapes, workers=1, odf=1, temporal_on=True, rsm_on=False):
    dev = FakeDevice()
    shape = next(iter(shapes.values()))
    decomp = decompose(shape, workers, odf)
    owned = [c for c in decomp.all_coords() if decomp.owner_map(workers)[c] == 0]
    store = GpuTileStore(dev, decomp, owned)
    for a in sorted(shapes):
        store.create_array(ArrayInfo(a, shapes[a]))
    mgr = GpuExchangeManager(store, 0, decomp.owner_map(workers))
    ex = GpuExecutor(store, mgr)
    ex.temporal = temporal_on
    ex.resident_smem = rsm_on
    return ex, store, mgr, dev


def _heat(iters, n=16):
    setup, step = DagProgram(), DagProgram()
    u1, u2 = heat3d_setup(setup, n)
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    heat3d_iterations(step, u1, u2, iters)
    return setup, step


def _names(dev):
    return [e[2] for e in dev.log if e[0] == "launch"]


@pytest.mark.parametrize("iters,fused", [(4, 4), (5, 4), (7, 4), (8, 8), (3, 0), (100, 100), (10, 8)])
def test_chain_cut(iters, fused):
    setup, step = _heat(iters)
    ex, store, mgr, dev = _executor(setup.shapes)
    ex.execute_batch(setup.dag)
    plans = [compile_plan(n, step.dag.ast_table) for n in step.dag.nodes]
    sched = ex.temporal_schedule(step.dag, plans)
    K = ex.tb_cfg.k
    leads = [nid for nid, v in sched.items() if v[0] == "lead"]
    assert len(sched) == fused
    assert len(leads) == fused // K
    dev.log.clear()
    stats = ex.execute_batch(step.dag)
    names = _names(dev)
    assert names.count("est_tb") == fused // K
    assert names.count("est_stream") == iters - fused
    assert stats.kernel_launches == iters  # reference definition: one per node per tile
    assert stats.gpu_launches == len(names) + (1 if fused else 0)  # + complement copy


def test_bookkeeping_matches_unfused():
    for iters in (4, 6, 9):
        setup, step = _heat(iters)
        res = []
        for on in (True, False):
            ex, store, mgr, dev = _executor(setup.shapes, temporal_on=on)
            ex.execute_batch(setup.dag)
            st = [ex.execute_batch(step.dag, b"k") for _ in range(4)]
            res.append(({a: (store.local_epoch(a), store.ghost_epoch(a)) for a in store.arrays},
                        dict(mgr.rounds_started),
                        [(s.nodes_executed, s.kernel_launches, s.rounds, s.net_messages) for s in st]))
        assert res[0] == res[1], iters


def test_twin_buffer_and_complement_copy():
    setup, step = _heat(4, n=16)
    ex, store, mgr, dev = _executor(setup.shapes)
    ex.execute_batch(setup.dag)
    dev.copies.clear()
    ex.execute_batch(step.dag)
    a = step.dag.nodes[0].statements[0].inputs[0]
    coords = next(iter(store.tiles))
    twin = store.twins[(coords, a)]
    home = store.tiles[coords].buffers[a]
    assert (twin.py, twin.pz, twin.xoff, twin.nbytes) == (home.py, home.pz, home.xoff, home.nbytes)
    strips = [c for c in dev.copies if c[0] == "strip"]
    # padded box 18^3 minus S = [1,17)^3 in padded coords ([2,16) after depth 1) -> 6 boxes
    assert len(strips) == 6
    total = sum(c[3] * c[4] * c[5] for c in strips)
    assert total == 18 ** 3 - 14 ** 3
    assert all(c[2] - twin.ptr == c[1] - home.ptr for c in strips)
    ex.release_scratch()
    assert twin.ptr == 0


def test_slab_chains_keep_reference_bookkeeping():
    """Several z-slabs in one process (odf 2 / 4): chains run per slab on a
    2-deep halo of A (physical ghost frame K*rz, logical depth 1 as in the
    reference), the intermediate array's rounds are virtual, and epochs,
    ghost generations, rounds, net messages and launch counts equal the
    unfused execution batch for batch."""
    K = temporal.DEFAULT.k
    for odf in (2, 4):
        setup, step = _heat(8, n=16)
        res = []
        for on in (True, False):
            ex, store, mgr, dev = _executor(setup.shapes, 1, odf, temporal_on=on)
            ex.execute_batch(setup.dag)
            st = [ex.execute_batch(step.dag, b"k") for _ in range(3)]
            if on:
                assert _names(dev).count("est_tb") == 3 * odf * 8 // K  # every slab, every chain
                assert all(store.phys_depth[a] == (K, 1, 1) for a in store.arrays)
                assert all(t.depths[a] == (1, 1, 1) for t in store.tiles.values() for a in store.arrays)
                assert all(b.depth == (K, 1, 1) for t in store.tiles.values() for b in t.buffers.values())
                assert len(store.twins) == odf  # one twin per slab for the chains' input array
            res.append(({a: (store.local_epoch(a), store.ghost_epoch(a)) for a in store.arrays},
                        dict(mgr.rounds_started),
                        [(s.nodes_executed, s.kernel_launches, s.rounds, s.net_messages) for s in st]))
        assert res[0] == res[1], odf


def test_slab_chain_rounds_alternate_home_and_twin():
    """Mid-run, A lives in the twins: the halo round before an odd chain moves
    strips between twins (2 planes = the physical frame), before an even one
    between the home buffers."""
    setup, step = _heat(8, n=16)
    ex, store, mgr, dev = _executor(setup.shapes, 1, 2)
    ex.execute_batch(setup.dag)
    ex.execute_batch(step.dag)
    dev.copies.clear()
    ex.execute_batch(step.dag)
    a = step.dag.nodes[0].statements[0].inputs[0]
    homes = {t.buffers[a].ptr: t.buffers[a] for t in store.tiles.values()}
    twins = {store.twins[(c, a)].ptr: store.twins[(c, a)] for c in store.tiles}

    def owner(addr, table):
        return any(p <= addr < p + b.nbytes for p, b in table.items())

    strips = [c for c in dev.copies if c[0] == "strip" and c[3:] == (16, 16, temporal.DEFAULT.k)]  # halo planes
    in_twin = [owner(c[2], twins) for c in strips]
    assert in_twin and any(in_twin) and not all(in_twin)
    assert all(owner(c[1], twins) == t for c, t in zip(strips, in_twin))
    assert all(owner(c[2], homes) != t for c, t in zip(strips, in_twin))


def test_no_chains_between_in_process_peer_workers():
    from paper_2512_19851_b200.transport import LocalPeerGroup, LocalPeerTransport

    setup, step = _heat(8, n=16)
    ex, store, mgr, dev = _executor(setup.shapes, 2, 1)
    ex.transport = LocalPeerTransport(LocalPeerGroup([store, store]), 0)
    plans = [compile_plan(n, step.dag.ast_table) for n in step.dag.nodes]
    assert ex.temporal_schedule(step.dag, plans, phys={0: (2, 1, 1), 1: (2, 1, 1)}) == {}


def test_chain_requires_same_statement_and_ping_pong():
    prog = DagProgram()
    u1, u2 = heat3d_setup(prog, 16)
    u3 = prog.create_array((16, 16, 16))
    interior = (slice(1, -1),) * 3
    prog.assign(u2, interior, heat3d_tree(u1))
    prog.assign(u1, interior, heat3d_tree(u2))
    prog.assign(u3, interior, heat3d_tree(u1))   # breaks the ping-pong
    prog.assign(u1, interior, heat3d_tree(u3))
    ex, store, mgr, dev = _executor(prog.shapes)
    plans = [compile_plan(n, prog.dag.ast_table) for n in prog.dag.nodes]
    sched = ex.temporal_schedule(prog.dag, plans)
    assert sched == {}


def test_generated_kernel_shape():
    prog = DagProgram()
    heat3d_setup(prog, 32)
    a, b = 0, 1
    prog.assign(b, (slice(1, -1),) * 3, heat3d_tree(a))
    plan = compile_plan(prog.dag.nodes[-1], prog.dag.ast_table)
    sig = codegen.stmt_sig(plan.statements[0], 3)
    for dt in (DTYPE_F64, DTYPE_F32):
        assert temporal.eligible(sig, dt)
        src, name, block, smem, lay = temporal.source(sig, dt)
        assert name == "est_tb" and block[0] == lay["nt"] + 32 and lay["min_blocks"] >= 1
        assert smem <= temporal.SMEM_BUDGET
        assert "cp.async.bulk.tensor.3d" in src and "mbarrier.arrive" in src
        assert "__dadd_rn" in src if dt == DTYPE_F64 else "__fadd_rn" in src


def test_z_star_required():
    """Loads off the centre plane must be pure z offsets (register columns)."""
    prog = DagProgram()
    a, b = heat3d_setup(prog, 16)
    box = (slice(1, -1),) * 3
    from paper_2512_19851_b200.ir import add
    from paper_2512_19851_b200.ir import ref as r_
    diag = add(r_(a, (slice(0, -2), slice(1, -1), slice(2, None))), r_(a, (slice(2, None), slice(1, -1), slice(1, -1))))
    prog.assign(b, box, diag)
    plan = compile_plan(prog.dag.nodes[-1], prog.dag.ast_table)
    assert not temporal.eligible(codegen.stmt_sig(plan.statements[0], 3), DTYPE_F64)
    prog.assign(b, box, heat3d_tree(a))
    plan = compile_plan(prog.dag.nodes[-1], prog.dag.ast_table)
    assert temporal.eligible(codegen.stmt_sig(plan.statements[0], 3), DTYPE_F64)


# ---------------------------------------------------------------------------
# resident-smem chains (resident.py): small rank-2 runs held in shared memory

def _laplace(n, iters):
    from paper_2512_19851_b200.programs import laplace_iteration_statements, laplace_program
    setup, step = DagProgram(), DagProgram()
    names = laplace_program(setup, n, 0)
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    laplace_iteration_statements(step, names["u"], names["scratch"], iters)
    return setup, step


@pytest.mark.parametrize("iters", [2, 9, 100])
def test_resident_smem_run_is_one_launch(iters):
    setup, step = _laplace(64, iters)
    ex, store, mgr, dev = _executor(setup.shapes, temporal_on=False, rsm_on=True)
    ex.execute_batch(setup.dag)
    dev.log.clear()
    stats = ex.execute_batch(step.dag)
    assert _names(dev) == ["est_resident_smem"]
    assert stats.kernel_launches == iters and stats.nodes_executed == iters


def test_resident_smem_bookkeeping_matches_node_by_node():
    setup, step = _laplace(64, 9)
    res = []
    for on in (True, False):
        ex, store, mgr, dev = _executor(setup.shapes, temporal_on=False, rsm_on=on)
        ex.execute_batch(setup.dag)
        st = [ex.execute_batch(step.dag, b"k") for _ in range(4)]
        res.append(({a: (store.local_epoch(a), store.ghost_epoch(a)) for a in store.arrays},
                    dict(mgr.rounds_started),
                    [(s.nodes_executed, s.kernel_launches, s.rounds, s.net_messages) for s in st]))
    assert res[0] == res[1]


def test_resident_smem_scope():
    """Rank 2 only, one tile, and only when one tile per SM fits shared memory."""
    setup, step = _laplace(64, 6)
    plans = [compile_plan(n, step.dag.ast_table) for n in step.dag.nodes]
    ex, *_ = _executor(setup.shapes, temporal_on=False, rsm_on=True)
    assert ex.temporal_schedule(step.dag, plans)[step.dag.nodes[0].node_id] == ("rsm", 6)
    ex, *_ = _executor(setup.shapes, 1, 2, temporal_on=False, rsm_on=True)
    assert ex.temporal_schedule(step.dag, plans) == {}
    big, bstep = _laplace(4096, 2)   # 2 x 128 MiB: no one-tile-per-SM fit
    bplans = [compile_plan(n, bstep.dag.ast_table) for n in bstep.dag.nodes]
    ex, *_ = _executor(big.shapes, temporal_on=False, rsm_on=True)
    assert ex.temporal_schedule(bstep.dag, bplans) == {}
    h, hstep = _heat(4)              # rank 3 is not a resident-smem chain
    hplans = [compile_plan(n, hstep.dag.ast_table) for n in hstep.dag.nodes]
    ex, *_ = _executor(h.shapes, temporal_on=False, rsm_on=True)
    assert ex.temporal_schedule(hstep.dag, hplans) == {}


@pytest.mark.parametrize("ny,nx,rad,dtype", [(1022, 1022, (0, 1, 1), DTYPE_F64), (1022, 1022, (0, 1, 1), DTYPE_F32),
                                             (60, 200, (0, 2, 2), DTYPE_F64), (1, 1000, (0, 1, 1), DTYPE_F64),
                                             (1500, 1500, (0, 1, 1), DTYPE_F32)])
def test_resident_smem_geometry_covers_s(ny, nx, rad, dtype):
    from paper_2512_19851_b200 import resident
    g = resident.smem_geometry(ny, nx, rad, dtype, 148)
    assert g is not None
    assert g.ntx * g.nty <= 148 and g.ntx * g.tx >= nx and g.nty * g.ty >= ny
    assert (g.ntx - 1) * g.tx < nx and (g.nty - 1) * g.ty < ny
    assert g.smem(rad, dtype) <= resident.SMEM_BUDGET


def test_resident_smem_kernel_source():
    from paper_2512_19851_b200 import resident
    setup, step = _laplace(32, 1)
    plan = compile_plan(step.dag.nodes[-1], step.dag.ast_table)
    sig = codegen.stmt_sig(plan.statements[0], 2)
    assert resident.smem_eligible(sig, DTYPE_F64, 2) and not resident.smem_eligible(sig, DTYPE_F64, 3)
    geo = resident.smem_geometry(30, 30, (0, 1, 1), DTYPE_F64, 148)
    src, name, block, smem = resident.smem_source(sig, DTYPE_F64, geo)
    assert name == "est_resident_smem" and block == (geo.threads, 1, 1) and smem == geo.smem((0, 1, 1), DTYPE_F64)
    assert src.count("grid_sync(bar,") == 3 and "__dadd_rn" in src and "__stcg" in src


def test_tb_only_for_large_grids(monkeypatch):
    monkeypatch.setattr(temporal, "MIN_POINTS", 1 << 28)
    setup, step = _heat(4)
    plans = [compile_plan(n, step.dag.ast_table) for n in step.dag.nodes]
    ex, *_ = _executor(setup.shapes)
    assert ex.temporal_schedule(step.dag, plans) == {}
    monkeypatch.setattr(temporal, "MIN_POINTS", 14 ** 3)
    ex, *_ = _executor(setup.shapes)
    assert [v[0] for v in ex.temporal_schedule(step.dag, plans).values()] == ["lead", "member", "lead", "member"]


def test_b_written_only_by_the_last_chain_of_a_run():
    """B's stores are skipped in every chain but the run's last (the next
    chain rewrites B before anything reads it); the Params flag sits after
    the tensor map, five 64-bit fields and fourteen ints."""
    import struct
    setup, step = _heat(8)
    ex, store, mgr, dev = _executor(setup.shapes)
    ex.execute_batch(setup.dag)
    dev.params.clear()
    dev.log.clear()
    ex.execute_batch(step.dag)
    tb = [p for e, p in zip(dev.log, dev.params) if e[2] == "est_tb"]
    assert len(tb) == 4
    assert [struct.unpack_from("<i", p, 128 + 24 + 14 * 4)[0] for p in tb] == [0, 0, 0, 1]


def test_self_dependent_statement_is_rejected_before_any_launch():
    """the in-process API has no coordinator validating the DAG;
    A[S] = f(A[S + o]) must raise SelfDependency (ir.py:354-357) instead of
    being scheduled as a chain whose two arrays share one buffer."""
    from paper_2512_19851_b200.errors import SelfDependency
    from paper_2512_19851_b200.ir import Dag, DagNode, Statement, compute_edges

    setup, step = _heat(4)
    ex, store, mgr, dev = _executor(setup.shapes)
    ex.execute_batch(setup.dag)
    good = step.dag.nodes[0]
    st = good.statements[0]
    bad_st = Statement(st.ast_id, st.output, st.output_slice, tuple(st.output for _ in st.inputs))
    nodes = [DagNode(0, [bad_st]), DagNode(1, [bad_st])]
    dag = Dag(nodes, compute_edges(nodes), step.dag.ast_table)
    dev.log.clear()
    with pytest.raises(SelfDependency):
        ex.execute_batch(dag)
    assert not [e for e in dev.log if e[0] == "launch"]
    assert ex._chain_candidate(compile_plan(nodes[0], dag.ast_table)) is None
