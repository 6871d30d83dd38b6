"""End-to-end drop-in check: the UNCHANGED reference coordinator and client
(installed into baseline/_ref from the reference package) drive GPU worker
processes and GPU memory daemons through the frozen wire protocol.

Skipped when the reference package is not installed next to the repo."""

import os
import sys

import numpy as np
import pytest

from oracle.oracle import bits_equal, laplace_reference
from paper_2512_19851_b200.launcher import DEFAULT_REF, GpuLauncher, reference_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="reference not installed in baseline/_ref")]


@pytest.fixture(scope="module")
def ref():
    if DEFAULT_REF not in sys.path:
        sys.path.insert(0, DEFAULT_REF)
    import elastencil.client as client
    import elastencil.programs as programs

    return client, programs


def test_laplace_over_the_wire(ref):
    client, programs = ref
    with GpuLauncher(workers=2, odf=2) as job:
        sess = client.Session(job.client_endpoint)
        bs = client.BatchingSession(sess, flush_depth=40)
        try:
            names = programs.laplace_program(bs, 64, 60)
            bs.sync()
            got = bs.fetch(names["u"])
            stats = bs.stats()
        finally:
            sess.shutdown()
    assert bits_equal(np.asarray(got), laplace_reference(64, 60))
    assert sum(stats["rounds"].values()) == 60
    assert stats["net_messages"] > 0


def test_rescale_shrink_then_expand_bit_equal(ref):
    client, programs = ref
    with GpuLauncher(workers=2, max_workers=2, odf=1) as job:
        sess = client.Session(job.client_endpoint)
        bs = client.BatchingSession(sess, flush_depth=25)
        try:
            b = programs.laplace_program(bs, 64, 20)
            shrink = bs.rescale(1)
            b = programs.laplace_iteration_statements(bs, b["u"], b["scratch"], 20)
            expand = bs.rescale(2)
            b = programs.laplace_iteration_statements(bs, b["u"], b["scratch"], 20)
            got = bs.fetch(b["u"])
            stats = bs.stats()
        finally:
            sess.shutdown()
    assert bits_equal(np.asarray(got), laplace_reference(64, 60))
    assert shrink.restart_ms > 0 and expand.restart_ms > 0
    assert len(stats["rescales"]) == 2


def test_rescale_hands_over_to_warm_spares(ref):
    """The restart stage gives worker ids to standby processes that already
    hold a CUDA context (launcher.GpuLauncher spares): the stage is much
    shorter than a cold respawn, results stay bit-exact, and the pool refills."""
    client, programs = ref
    with GpuLauncher(workers=2, max_workers=2, odf=1) as job:
        assert job.wait_spares(180), "standby pool did not fill"
        sess = client.Session(job.client_endpoint)
        bs = client.BatchingSession(sess, flush_depth=25)
        try:
            b = programs.laplace_program(bs, 64, 20)
            shrink = bs.rescale(1)
            b = programs.laplace_iteration_statements(bs, b["u"], b["scratch"], 20)
            assert job.wait_spares(180)
            expand = bs.rescale(2)
            b = programs.laplace_iteration_statements(bs, b["u"], b["scratch"], 20)
            got = bs.fetch(b["u"])
        finally:
            sess.shutdown()
        assert job.restart_log == [{"warm": 1, "cold": 0}, {"warm": 2, "cold": 0}]
    assert bits_equal(np.asarray(got), laplace_reference(64, 60))
    print(f"warm restart ms: shrink {shrink.restart_ms:.1f}, expand {expand.restart_ms:.1f}")
    assert shrink.restart_ms < 500 and expand.restart_ms < 500


# ---------------------------------------------------------------------------
# the reference runtime's behaviours (pkg/tests/test_runtime.py), re-checked
# with GPU workers and GPU memory daemons behind the unchanged coordinator

def _session(client, job, flush=10):
    s = client.Session(job.client_endpoint)
    return s, client.BatchingSession(s, flush_depth=flush)


def test_fetch_windows_and_rank1(ref):
    client, _programs = ref
    from elastencil.ir import cst, ref as aref
    with GpuLauncher(workers=2, odf=2) as job:
        s, session = _session(client, job)
        try:
            a = session.create_array((32, 32))
            session.assign(a, (slice(None), slice(None)), cst(7.5))
            session.assign(a, (slice(4, 12), slice(16, 24)), cst(-1.0))
            full = np.asarray(session.fetch(a))
            one = np.asarray(session.fetch(a, (5, 17)))
            window = np.asarray(session.fetch(a, (slice(8, 24), slice(8, 24))))
            assert full.shape == (32, 32) and one.shape == (1, 1) and one[0, 0] == -1.0
            assert np.array_equal(window, full[8:24, 8:24])
            x = session.create_array((64,))
            y = session.create_array((64,))
            session.assign(x, ((0, 40),), cst(2.0))
            session.assign(y, ((1, 63),), aref(x, ((0, 62),)))
            want = np.zeros(64)
            want[1:41] = 2.0
            assert np.array_equal(np.asarray(session.fetch(y)), want)
        finally:
            s.shutdown()


def test_batch_error_poisons_session(ref):
    client, _programs = ref
    from elastencil.errors import OffsetExceedsTileWidth, SessionFailed
    from elastencil.ir import ref as aref
    with GpuLauncher(workers=2, odf=2) as job:
        s, session = _session(client, job)
        try:
            a = session.create_array((8, 8))
            b = session.create_array((8, 8))
            session.assign(b, (slice(4, None), slice(None)), aref(a, (slice(None, -4), slice(None))))
            with pytest.raises(OffsetExceedsTileWidth):
                session.sync()
            with pytest.raises(SessionFailed):
                session.fetch(a)
        finally:
            s.close()


def test_rescale_identity_empty_and_above_initial_count(ref):
    client, programs = ref
    from elastencil.ir import cst
    with GpuLauncher(workers=2, max_workers=4) as job:
        s, session = _session(client, job, flush=25)
        try:
            assert session.rescale(2).restart_ms > 0          # no arrays yet: stages still run
            a = session.create_array((16, 16))
            session.assign(a, (slice(None), slice(None)), cst(3.25))
            assert session.rescale(2).restart_ms > 0          # identity with data
            assert (np.asarray(session.fetch(a)) == 3.25).all()
            names = programs.laplace_program(session, 32, 10)
            assert session.rescale(4).restart_ms > 0          # beyond the initial tile owners
            names = programs.laplace_iteration_statements(session, names["u"], names["scratch"], 10)
            assert bits_equal(np.asarray(session.fetch(names["u"])), laplace_reference(32, 20))
        finally:
            s.shutdown()


def test_expand_then_immediate_shrink_and_process_census(ref):
    client, programs = ref
    job = GpuLauncher(workers=2, max_workers=4, odf=2)
    job.start()
    try:
        s, session = _session(client, job, flush=25)
        names = programs.laplace_program(session, 32, 7)
        session.rescale(4)
        session.rescale(2)
        names = programs.laplace_iteration_statements(session, names["u"], names["scratch"], 7)
        assert bits_equal(np.asarray(session.fetch(names["u"])), laplace_reference(32, 14))
        job.wait_spares(180)
        pids = job.all_pids() + job.spare_pids()  # the standby pool goes down with the job
        s.shutdown()
    finally:
        job.shutdown()
    import time
    deadline = time.time() + 20
    alive = list(pids)
    while alive and time.time() < deadline:
        alive = [p for p in alive if os.path.exists(f"/proc/{p}") and
                 open(f"/proc/{p}/stat").read().split()[2] != "Z"]
        time.sleep(0.2)
    assert not alive, f"processes left behind: {alive}"
