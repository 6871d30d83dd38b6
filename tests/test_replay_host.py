"""Batch replay cache (CUDA-graph host path): the epoch / round bookkeeping
applied on replay equals a fresh execution of the same batches (CPU, device
test double)."""

from fakedev import FakeDevice
from paper_2512_19851_b200.exchange import GpuExchangeManager
from paper_2512_19851_b200.executor import GpuExecutor
from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, heat3d_setup, laplace_iteration_statements, laplace_program
from paper_2512_19851_b200.tiles import ArrayInfo, GpuTileStore, decompose


def _executor(shapes, odf=1):
    dev = FakeDevice()
    shape = next(iter(shapes.values()))
    decomp = decompose(shape, 1, odf)
    store = GpuTileStore(dev, decomp, decomp.all_coords())
    for a in sorted(shapes):
        store.create_array(ArrayInfo(a, shapes[a]))
    mgr = GpuExchangeManager(store, 0, decomp.owner_map(1))
    return GpuExecutor(store, mgr), store, mgr


def _state(ex, store, mgr):
    return ({a: (store.local_epoch(a), store.ghost_epoch(a), mgr.ghost_generation(a)) for a in store.arrays},
            dict(mgr.rounds_started), mgr.net_messages)


def _run(batches, use_key, odf):
    setup, step = batches
    ex, store, mgr = _executor(setup.shapes, odf)
    ex.execute_batch(setup.dag)
    stats = []
    for _ in range(5):
        stats.append(ex.execute_batch(step.dag, b"k" if use_key else None))
    return ex, _state(ex, store, mgr), stats


def _programs(kind):
    setup = DagProgram()
    step = DagProgram()
    if kind == "laplace":
        names = laplace_program(setup, 32, 0)
        u1, u2 = names["u"], names["scratch"]
        for a in sorted(setup.shapes):
            step.builder.declare_array(a, setup.shapes[a])
        laplace_iteration_statements(step, u1, u2, 6)
    else:
        u1, u2 = heat3d_setup(setup, 16)
        for a in sorted(setup.shapes):
            step.builder.declare_array(a, setup.shapes[a])
        heat3d_iterations(step, u1, u2, 4)
    return setup, step


def test_replay_bookkeeping_equals_fresh_execution():
    for kind, odf in (("laplace", 1), ("laplace", 4), ("heat3d", 1), ("heat3d", 2)):
        progs = _programs(kind)
        ex_a, fresh, stats_a = _run(progs, False, odf)
        ex_b, replayed, stats_b = _run(progs, True, odf)
        assert fresh == replayed, kind
        # batch 1 grows the ghost frame (not steady state), 2 is recorded, 3 captured,
        # 4 and 5 replay the graph
        assert ex_b.replays == 2
        for a, b in zip(stats_a, stats_b):
            assert (a.nodes_executed, a.kernel_launches, a.rounds, a.net_messages) == \
                   (b.nodes_executed, b.kernel_launches, b.rounds, b.net_messages)


def test_replay_cache_is_bounded_and_drops_stale_layouts(monkeypatch):
    """the replay cache (and the CUDA graphs it owns) is capped,
    and entries of an older buffer layout are released."""
    from paper_2512_19851_b200.executor import GpuExecutor

    closed = []

    class G:
        def close(self):
            closed.append(self)

    ex = GpuExecutor.__new__(GpuExecutor)
    ex._replay = {}
    monkeypatch.setattr(GpuExecutor, "REPLAY_CAP", 4)
    for k in range(10):
        ex._remember((bytes([k]), (1, ())), {"graph": G()})
    assert len(ex._replay) == 4 and len(closed) == 6
    ex._remember((b"new", (2, ())), {"graph": G()})
    assert list(ex._replay) == [(b"new", (2, ()))] and len(closed) == 10
