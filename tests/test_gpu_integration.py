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
