"""Multi-PROCESS GPU workers (CUDA IPC transport) on one GPU: each rank is a
separate process with its own CUDA context; halos are pulled out of the peer
process's HBM buffers through IPC handles, ordered by device-side flag words
(stream write / wait on 32-bit values in the peers' exported arenas)."""

import pytest

from mp_workers import gpu_rank
from paper_2512_19851_b200.ipc import spawn_local_job
from test_multiworker_host import expected_rounds

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,world,odf,batch", [
    ("laplace", 2, 1, 9), ("laplace", 4, 1, 100), ("laplace", 2, 2, 13),
    ("heat3d", 2, 1, 7), ("heat3d", 4, 1, 100)])
def test_ipc_workers_bit_exact(kind, world, odf, batch):
    res = spawn_local_job(world, gpu_rank, kind, odf, batch, timeout=600)
    want = expected_rounds(kind, batch)
    for r in res:
        assert all(r["ok"].values()), r["ok"]
        assert r["rounds"] == want


@pytest.mark.parametrize("world,odf,batch", [(2, 1, 8), (2, 2, 20), (4, 1, 12)])
def test_ipc_slab_chains_bit_exact(world, odf, batch):
    """Temporal chains on the z-slabs of a multi-process job: each rank's
    chain reads A's 2-plane halo pulled out of its neighbours' buffers (home
    or twin, alternating per chain), bit-exact with the reference round counts."""
    res = spawn_local_job(world, gpu_rank, "heat3d", odf, batch, True, timeout=600)
    want = expected_rounds("heat3d", batch)
    for r in res:
        assert all(r["ok"].values()), r["ok"]
        assert r["rounds"] == want
        assert r["twins"] == odf, "the slab chains did not run"
