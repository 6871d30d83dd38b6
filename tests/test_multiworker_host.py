"""Multi-process (gloo, world_size 2-3) tests of the N>1 HOST path on CPU:
owner maps, push plan, round sequencing and the IPC transport handshake run
for real across processes; the device is a recording test double."""

import pytest

from oracle.oracle import EpochSimulator
from paper_2512_19851_b200.analysis import analyze_dag
from paper_2512_19851_b200.ipc import spawn_local_job
from mp_workers import _program, _split, host_logic_rank


def expected_rounds(kind, batch):
    prog, _ = _program(kind)
    sim = EpochSimulator()
    for part in _split(prog.dag, batch):
        sim.simulate_batch(part, analyze_dag(part, prog.shapes))
    return sim.rounds


@pytest.mark.parametrize("kind,world,odf,batch", [
    ("laplace", 2, 1, 7), ("laplace", 4, 1, 50), ("laplace", 2, 2, 13), ("heat3d", 2, 1, 5),
    ("heat3d", 4, 1, 100)])
def test_rounds_and_handshake_across_processes(kind, world, odf, batch):
    res = spawn_local_job(world, host_logic_rank, kind, odf, batch, timeout=300)
    want = expected_rounds(kind, batch)
    for r in res:
        assert r["rounds"] == want
    # every rank took part in every round, in the same order
    assert len({r["seq"] for r in res if r["tiles"]}) == 1
    # net strips are symmetric: what ranks pulled equals what they counted
    assert sum(r["net"] for r in res) > 0
    # rank-3 slabs: halo pulls overlap the interior planes on the copy lane
    if kind == "heat3d":
        assert all(r["copy_lane_pulls"] > 0 for r in res if r["tiles"])
    tiles = sorted(t for r in res for t in r["tiles"])
    assert len(tiles) == len(set(tiles)) == world * odf


@pytest.mark.parametrize("world,odf,batch", [(2, 1, 8), (2, 2, 20), (4, 1, 12)])
def test_slab_chains_across_processes(world, odf, batch):
    """Temporal chains on z-slabs of a multi-process job: every rank runs the
    chain kernel on its slabs, rounds are sequenced identically everywhere
    and equal the reference EpochSimulator's counts (the intermediate array's
    rounds are virtual). Halo planes travel through the owners' halo windows
    (exported from home or twin, whichever holds the array): no rank maps a
    neighbour's tile or twin buffer."""
    res = spawn_local_job(world, host_logic_rank, "heat3d", odf, batch, True, timeout=300)
    want = expected_rounds("heat3d", batch)
    for r in res:
        assert r["rounds"] == want
        assert r["tb_launches"] > 0 and r["twins"] == odf
        assert r["flag_waits"] > 0
    assert len({r["seq"] for r in res}) == 1
    assert all(r["peer_windows"] > 0 and r["peer_tile_maps"] == 0 and r["exports"] > 0 for r in res)


@pytest.mark.parametrize("kind,world,shrink_to", [("heat3d", 4, 2), ("laplace", 4, 2), ("heat3d", 4, 1)])
def test_migration_keeps_tileless_workers_in_sequence(kind, world, shrink_to):
    """After a shrink-by-migration some workers own no tile; they still count
    epochs and take part in every round, so after migrating back the round
    sequence is aligned on every worker (a misalignment deadlocks the IPC
    handshake and fails this test by timeout)."""
    from mp_workers import migrate_rank

    res = spawn_local_job(world, migrate_rank, kind, shrink_to, timeout=300)
    assert len({tuple(r["seqs"]) for r in res}) == 1, [r["seqs"] for r in res]
    assert len({tuple(sorted(r["epochs"].items())) for r in res}) == 1
    assert sum(1 for r in res if not r["tiles_shrunk"]) == world - shrink_to


def test_chain_launch_waits_for_peers_pulled():
    """Every slab-chain launch is directly preceded by a wait on the peers'
    PULLED flag: the chain overwrites A, and the peers must be done reading
    the round of A it consumed (write-after-read)."""
    from mp_workers import chain_wait_rank

    res = spawn_local_job(2, chain_wait_rank, timeout=300)
    for seqs in res:
        assert seqs and all(s == "flag_wait" for s in seqs), seqs


def test_isolated_arenas_are_reused():
    """Isolated allocations (tiles an expand's load-balance stage moves) get
    an arena of their own; once freed, the idle arena serves the next
    isolated request of the same size instead of a new cudaMalloc."""
    from fakedev import FakeDevice
    from paper_2512_19851_b200.pool import DevicePool

    dev = FakeDevice()
    pool = DevicePool(dev, arena_min=1 << 20)
    a = pool.alloc(3 << 20, isolated=True)
    b = pool.alloc(3 << 20, isolated=True)
    assert len(pool.arenas) == 2 and pool.locate(a)[0] != pool.locate(b)[0]
    pool.free(a)
    c = pool.alloc(3 << 20, isolated=True)
    assert len(pool.arenas) == 2 and c == a
    assert all(ar.size == 3 << 20 for ar in pool.arenas)  # exactly the buffer: a peer maps nothing else
