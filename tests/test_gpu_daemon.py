"""The GPU memory daemon (daemon.GpuMemoryDaemon) on its own, as a separate
PROCESS the way the launcher runs it (one per GPU slot).

* reference kinds (STORE / RETRIEVE / FREE / PING / STATS, daemon.py:29-143)
  keep their semantics: RETRIEVE frees, unknown ids are typed errors;
* device allocations (DEV_ALLOC / DEV_OPEN / DEV_FREE): first-fit carving of
  exported arenas, freed ranges are reused, concurrent clients never receive
  overlapping ranges, DEV_OPEN returns the allocation's metadata;
* the checkpoint / restore data path through it: a worker-side job copies
  its tiles D2D into daemon HBM (elastic.checkpoint_tiles), a fresh job in
  another process restores them (elastic.restore_tiles) - whole-array
  content hashes equal, and the daemon holds nothing afterwards.
"""

import os
import subprocess
import sys
import threading

import pytest

from paper_2512_19851_b200.daemon import DaemonClient
from paper_2512_19851_b200.errors import UnknownAllocation

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture
def daemon():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, env.get("PYTHONPATH", "")])
    proc = subprocess.Popen([sys.executable, "-m", "paper_2512_19851_b200.daemon", "--id", "0", "--device", "0"],
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, env=env, cwd=ROOT)
    try:
        line = proc.stdout.readline().decode().split()
        assert line and line[0] == "DAEMON", proc.stderr.read().decode()[-2000:]
        yield line[1]
    finally:
        proc.kill()
        proc.wait(timeout=30)


def test_reference_kinds(daemon):
    c = DaemonClient(daemon)
    try:
        assert c.ping() == {"gpu": 0}
        a = c.store(b"x" * 1000)
        b = c.store(b"")
        assert c.stats() == (2, 1000)
        assert c.retrieve_and_free(a) == b"x" * 1000
        with pytest.raises(UnknownAllocation):
            c.retrieve_and_free(a)      # RETRIEVE frees (daemon.py:61-68)
        c.free(b)
        with pytest.raises(UnknownAllocation):
            c.free(b)
        assert c.stats() == (0, 0)
    finally:
        c.close()


def test_device_allocations_carve_and_reuse(daemon):
    c = DaemonClient(daemon)
    try:
        i1, h1, off1, s1 = c.dev_alloc(3 << 20, {"k": 1})
        i2, h2, off2, s2 = c.dev_alloc(5 << 20, {"k": 2})
        assert s1 == s2 and h1 == h2  # carved out of one exported arena
        assert off2 >= off1 + (3 << 20)
        assert c.stats() == (2, 8 << 20)
        hd, offd, sd, meta = c.dev_open(i2)
        assert (hd, offd, sd, meta) == (h2, off2, s2, {"k": 2})
        c.dev_free(i1)
        i3, _h3, off3, s3 = c.dev_alloc(1 << 20, {})
        assert (s3, off3) == (s1, off1)  # first fit reuses the freed range
        for bad in (i1, 10 ** 9):
            with pytest.raises(UnknownAllocation):
                c.dev_open(bad)
            with pytest.raises(UnknownAllocation):
                c.dev_free(bad)
        c.dev_free(i2)
        c.dev_free(i3)
        assert c.stats() == (0, 0)
    finally:
        c.close()


def test_concurrent_clients_get_disjoint_ranges(daemon):
    got, errors = [], []

    def work(k):
        cl = DaemonClient(daemon)
        try:
            for j in range(8):
                i, _h, off, serial = cl.dev_alloc((k + 1) * (1 << 20) + j * 4096, {"k": k})
                got.append((serial, off, (k + 1) * (1 << 20) + j * 4096, i))
        except Exception as exc:  # surfaced below
            errors.append(exc)
        finally:
            cl.close()

    threads = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors
    assert len({g[3] for g in got}) == len(got) == 48
    by_arena = {}
    for serial, off, n, _i in got:
        by_arena.setdefault(serial, []).append((off, n))
    for ranges in by_arena.values():
        ranges.sort()
        for (o1, n1), (o2, _n2) in zip(ranges, ranges[1:]):
            assert o1 + n1 <= o2, "overlapping device allocations"
    c = DaemonClient(daemon)
    try:
        for g in got:
            c.dev_free(g[3])
        assert c.stats() == (0, 0)
    finally:
        c.close()


def test_checkpoint_restore_through_daemon_hbm(daemon, tmp_path):
    from mp_workers import checkpoint_rank, restore_rank
    from paper_2512_19851_b200.ipc import spawn_local_job

    path = str(tmp_path / "manifest.json")
    (ck,) = spawn_local_job(1, checkpoint_rank, daemon, path, timeout=600)
    assert ck["records"] == 2
    c = DaemonClient(daemon)
    try:
        n, total = c.stats()
        assert (n, total) == (2, 2 * 48 ** 3 * 8)  # one device allocation per (tile, array) payload
    finally:
        c.close()
    (rs,) = spawn_local_job(1, restore_rank, path, timeout=600)
    assert rs["hashes"] == ck["hashes"]
    assert rs["stats"]["bytes"] == 2 * 48 ** 3 * 8
    c = DaemonClient(daemon)
    try:
        assert c.stats() == (0, 0)  # the restore freed every allocation
    finally:
        c.close()
