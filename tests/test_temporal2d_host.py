"""Rank-2 two-sweep chains (temporal2d.py) on the host side, CPU with the
device test double: which nodes fuse (ping-pong and wave rotation runs), that
the per-node bookkeeping (epochs, rounds, launch counts) equals unfused
execution, the twins / complement copies / end-of-run copy-back, and that the
generated kernel compiles for sm_100a (NVRTC, no GPU needed)."""

import pytest

from fakedev import FakeDevice
from paper_2512_19851_b200 import codegen, temporal2d
from paper_2512_19851_b200.analysis import compile_plan
from paper_2512_19851_b200.exchange import GpuExchangeManager
from paper_2512_19851_b200.executor import GpuExecutor
from paper_2512_19851_b200.ir import add, cst, mul, ref, sub
from paper_2512_19851_b200.programs import DagProgram, laplace_iteration_statements, wave2d_setup, wave2d_steps
from paper_2512_19851_b200.tiles import ArrayInfo, GpuTileStore, decompose
from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64


@pytest.fixture(autouse=True)
def _small_grids_chain(monkeypatch):
    monkeypatch.setattr(temporal2d, "MIN_POINTS", 0)
    monkeypatch.setattr(temporal2d, "ROTATIONS", True)  # opt-in by default (measured slower at C3)


def _executor(shapes, dtypes=None, temporal_on=True):
    dev = FakeDevice()
    shape = next(iter(shapes.values()))
    decomp = decompose(shape, 1, 1)
    store = GpuTileStore(dev, decomp, list(decomp.all_coords()))
    for a in sorted(shapes):
        store.create_array(ArrayInfo(a, shapes[a], (dtypes or {}).get(a, DTYPE_F64)))
    mgr = GpuExchangeManager(store, 0, decomp.owner_map(1))
    ex = GpuExecutor(store, mgr)
    ex.temporal = temporal_on
    ex.resident_smem = False
    return ex, store, mgr, dev


def _wave(steps, n=64):
    setup, step = DagProgram(), DagProgram()
    u = wave2d_setup(setup, n, DTYPE_F32)
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    wave2d_steps(step, *u, steps)
    return setup, step


def _laplace(iters, n=64):
    setup, step = DagProgram(), DagProgram()
    u1, u2 = setup.create_array((n, n)), setup.create_array((n, n))
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    laplace_iteration_statements(step, u1, u2, iters)
    return setup, step


def _names(dev):
    return [e[2] for e in dev.log if e[0] == "launch"]


@pytest.mark.parametrize("steps,chains", [(2, 0), (3, 1), (7, 3), (10, 5), (1, 0)])
def test_wave_rotation_schedule(steps, chains):
    """Chains need one buffer layout for the rotation's three arrays: in a
    2-step batch u0 is read at the centre only (ghost depth 0), so that batch
    runs node by node; from 3 steps on every array is a stencil input once."""
    setup, step = _wave(steps)
    ex, store, mgr, dev = _executor(setup.shapes, setup.dtypes)
    ex.execute_batch(setup.dag)
    dev.log.clear()
    stats = ex.execute_batch(step.dag)
    names = _names(dev)
    assert names.count("est_tc") == chains
    assert stats.kernel_launches == steps  # reference definition: one per node per tile
    assert not any(ex._in_twin.values()), "every array is home after the run"
    plans = [compile_plan(n, step.dag.ast_table) for n in step.dag.nodes]
    sched = ex.temporal_schedule(step.dag, plans)
    leads = [v for v in sched.values() if v[0] == "tc"]
    if chains:
        assert len(leads) == chains and len(sched) == 2 * chains
        assert all(len(v[3]) == 3 for v in leads)  # every array of the rotation gets a twin
        assert leads[-1][2] and not any(v[2] for v in leads[:-1])


@pytest.mark.parametrize("iters,chains", [(4, 2), (5, 2), (7, 2), (8, 4), (3, 0)])
def test_pingpong_schedule_even_chains(iters, chains):
    setup, step = _laplace(iters)
    ex, store, mgr, dev = _executor(setup.shapes)
    ex.execute_batch(setup.dag)
    dev.log.clear()
    stats = ex.execute_batch(step.dag)
    assert _names(dev).count("est_tc") == chains
    assert stats.kernel_launches == iters
    assert not any(ex._in_twin.values())


def test_bookkeeping_matches_unfused():
    for build, n in ((_wave, 7), (_wave, 12), (_laplace, 6), (_laplace, 9)):
        setup, step = build(n)
        res = []
        for on in (True, False):
            ex, store, mgr, dev = _executor(setup.shapes, setup.dtypes, temporal_on=on)
            ex.execute_batch(setup.dag)
            st = [ex.execute_batch(step.dag, b"k") for _ in range(4)]
            res.append(({a: (store.local_epoch(a), store.ghost_epoch(a)) for a in store.arrays},
                        dict(mgr.rounds_started),
                        [(s.nodes_executed, s.kernel_launches, s.rounds, s.net_messages) for s in st]))
        assert res[0] == res[1], (build.__name__, n)


def test_rotation_twins_complement_and_copy_back():
    """3 chains of a rotation: each array is the step-2 output once, so all
    three end the run in their twins and are copied back (S only); the run's
    first chain fills every twin's complement of S."""
    setup, step = _wave(6, n=40)
    ex, store, mgr, dev = _executor(setup.shapes, setup.dtypes)
    ex.execute_batch(setup.dag)
    dev.copies.clear()
    ex.execute_batch(step.dag)
    coords = next(iter(store.tiles))
    assert sorted(a for c, a in store.twins) == sorted(setup.shapes)
    strips = [c for c in dev.copies if c[0] == "strip"]
    home = store.tiles[coords].buffers[0]
    npy, npx = home.pz // home.py, home.ext[2] + 2 * home.depth[2]
    s = 36  # S = [2:-2, 2:-2] of 40
    complement = npy * npx - s * s
    comp = [c for c in strips if c[3] * c[4] * c[5] != s * s]
    back = [c for c in strips if c[3] * c[4] * c[5] == s * s]
    assert sum(c[3] * c[4] * c[5] for c in comp) == 3 * complement
    assert len(back) == 3  # every array ends in its twin after 3 chains


@pytest.mark.parametrize("dtype", [DTYPE_F32, DTYPE_F64])
def test_sources_compile_for_sm100a(dtype):
    """The wave (rotation, radius 2) and a radius-1 ping-pong compile with NVRTC
    for sm_100a (offline; cached in-tree like the prebuilt kernels)."""
    from paper_2512_19851_b200.build import precompile_sources

    srcs = []
    for build in (_wave, _laplace):
        _setup, step = build(2)
        st = compile_plan(step.dag.nodes[0], step.dag.ast_table).statements[0]
        sig = codegen.stmt_sig(st, 2)
        assert temporal2d.eligible(sig, dtype)
        src, name, block, smem, lay = temporal2d.source(sig, dtype)
        assert name == "est_tc" and lay["w0"] <= 256 and smem <= 200 * 1024
        assert "cp.async.bulk.tensor.3d" in src and "bar.sync 1," in src
        srcs.append(src)
    new, cached = precompile_sources(srcs)
    assert new + cached == 2


def test_roles_reject_unchainable():
    """Diagonal stencils, a second input read off-centre, or no y-offset are not tc statements."""
    n = 32
    prog = DagProgram()
    a, b, c = (prog.create_array((n, n)) for _ in range(3))
    box = ((2, 30), (2, 30))

    def at(u, dy, dx):
        return ref(u, tuple(slice(lo + d, hi + d) for (lo, hi), d in zip(box, (dy, dx))))
    cases = [
        mul(cst(0.5), add(at(a, 1, 1), at(a, -1, 0))),          # diagonal
        add(at(a, 1, 0), at(b, 0, 1)),                           # second input off-centre
        add(at(a, 0, 1), at(a, 0, -1)),                          # no y offset (ry = 0)
        sub(at(a, 1, 0), at(a, -1, 0)),                          # fine: y-star
        add(at(a, 1, 0), at(b, 0, 0)),                           # fine: rotation
    ]
    want = [False, False, False, True, True]
    for expr, ok in zip(cases, want):
        p = DagProgram()
        for x in (a, b, c):
            p.builder.declare_array(x, (n, n))
        p.assign(c, box, expr)
        st = compile_plan(p.dag.nodes[0], p.dag.ast_table).statements[0]
        assert (temporal2d.roles(codegen.stmt_sig(st, 2)) is not None) == ok


@pytest.mark.parametrize("world", [1, 2])
def test_chain_runs_in_worker_job_with_transport(world):
    """The GPU worker process runs batches through an IPC job (a transport
    exists even at world 1): a single-tile 2-D job still chains, and a rank
    without the tile keeps the same epochs without launching."""
    from mp_workers import single_tile_chain_rank
    from paper_2512_19851_b200.ipc import spawn_local_job

    res = spawn_local_job(world, single_tile_chain_rank, "laplace", timeout=300)
    owner = [r for r in res if r["tiles"]]
    assert len(owner) == 1 and owner[0]["names"].count("est_tc") == 4
    assert len({tuple(sorted(r["epochs"].items())) for r in res}) == 1
    assert all(not r["names"] for r in res if not r["tiles"])


def test_resident_run_in_worker_job_with_transport():
    """The same for a small grid: the whole 8-sweep run is one
    shared-memory-resident launch in the worker's job (the reference-facing
    seam path of C1)."""
    from mp_workers import single_tile_chain_rank
    from paper_2512_19851_b200.ipc import spawn_local_job

    (res,) = spawn_local_job(1, single_tile_chain_rank, "laplace", True, timeout=300)
    assert res["names"].count("est_resident_smem") == 1 and "est_tc" not in res["names"]


def test_one_worker_job_replays_graphs():
    """A one-worker job behind the worker seam (a transport, no peers)
    captures repeated batches into a CUDA graph and replays them, with the
    same per-batch bookkeeping; a two-worker job never does."""
    from mp_workers import replay_rank
    from paper_2512_19851_b200.ipc import spawn_local_job

    (one,) = spawn_local_job(1, replay_rank, timeout=300)
    assert one["replays"] >= 2 and one["graph_launches"] >= 2
    two = spawn_local_job(2, replay_rank, timeout=300)
    assert all(r["replays"] == 0 for r in two)
    assert one["epochs"] == two[0]["epochs"] and one["rounds"] == two[0]["rounds"]
