"""Multi-PROCESS GPU workers (CUDA IPC transport) on one GPU: each rank is a
separate process with its own CUDA context; halos are pulled out of the peer
process's HBM buffers through IPC handles, ordered by IPC events."""

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
