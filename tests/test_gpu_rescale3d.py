"""C5's code path at test size: a rank-3 job on GPU worker processes under the
reference Coordinator class (session3d.Rank3Job), rescaled 2 -> 1 -> 2 mid-run
through the coordinator's unmodified four-stage rescale (load balance,
checkpoint into the GPU memory daemons, worker-process restart, restore;
expand: checkpoint, restart, restore, load balance; coordinator.py:501-607).
Both arrays must be bit-identical to the strict oracle of the unrescaled
program, fetched over W_FETCH and through the W_HASH whole-array hash."""

import numpy as np
import pytest

from oracle.oracle import bits_equal, content_hash, strict_execute_dag
from paper_2512_19851_b200.launcher import reference_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="reference not installed in baseline/_ref")]


def _programs(n, iters, fills):
    from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, heat3d_setup

    setup = DagProgram()
    u1, u2 = heat3d_setup(setup, n, seed_fills=fills)
    step = DagProgram()
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    heat3d_iterations(step, u1, u2, iters)
    return setup, step


def test_rank3_rescale_four_stages_bit_exact():
    from paper_2512_19851_b200.session3d import Rank3Job
    from paper_2512_19851_b200.wire import encode_dag

    n, per = 48, 10
    setup, step = _programs(n, per, 16)
    want = strict_execute_dag(setup.dag, setup.shapes)
    for _ in range(3):
        strict_execute_dag(step.dag, setup.shapes, arrays=want)
    blob = encode_dag(step.dag)
    with Rank3Job(2) as job:
        for a in sorted(setup.shapes):
            job.create_array(setup.shapes[a])
        job.submit(encode_dag(setup.dag))
        job.submit(blob)
        shrink = job.rescale(1)
        job.submit(blob)
        expand = job.rescale(2)
        job.submit(blob)
        got = {a: job.fetch(a) for a in sorted(setup.shapes)}
        hashes = {a: job.hash(a) for a in sorted(setup.shapes)}
        stats = job.stats()
    for t in (shrink, expand):
        assert {"lb_ms", "checkpoint_ms", "restart_ms", "restore_ms", "total_ms"} <= set(t)
        assert t["restart_ms"] > 0 and t["total_ms"] >= t["restart_ms"]
    for a in sorted(setup.shapes):
        assert bits_equal(got[a], want[a]), a
        assert hashes[a] == content_hash(want[a]), a
    # at least one halo round per iteration (restore bumps local epochs,
    # elastic.py:154-157, which may add re-exchanges after a rescale)
    assert sum(stats["rounds"].values()) >= 3 * per
