"""Rank-3 jobs on GPU worker processes through the reference coordinator's
own worker control plane.

The frozen client protocol has no rank-3 arrays: the reference client, its
slice codec and its coordinator reject them (client.py:89, proto.py:147,
coordinator.py:383-384), while BASELINE configs C2/C4/C5 are 3-D. `Rank3Job`
therefore drives the UNCHANGED reference `Coordinator` class in-process
(imported from the reference package installed in baseline/_ref) below its
client seam: its registration, INIT, W_* request/reply matching
(`WorkerConn.request`), batch barrier and statistics (coordinator.py:75-118,
228-262, 431-446), and — the point of it — its rescale path unmodified:
`_cmd_rescale` -> `_rescale_shrink` / `_rescale_expand` with the four stages
(load balance, checkpoint into the memory daemons, worker-process restart
through the launcher, restore; coordinator.py:501-607, launcher.py:154-169).
Only the three client-side steps that are rank-limited in the reference are
done here instead: W_CREATE with the shape and decomposition (as
`_cmd_create` sends it), W_BATCH with DAG bytes from this package's rank-3
superset codec (as `_cmd_batch` sends them), and W_FETCH / W_HASH reads.

Workers are `paper_2512_19851_b200.worker` processes and daemons are
`paper_2512_19851_b200.daemon` processes spawned by `launcher.GpuLauncher`,
worker slot i on GPU i mod the visible GPUs.
"""

from __future__ import annotations

import os
import sys
import time
from types import SimpleNamespace

import numpy as np

from .launcher import DEFAULT_REF, GpuLauncher
from .wire import DTYPE_F64, W_BATCH, W_CREATE, W_FETCH, W_HASH

NP = {0: np.float64, 1: np.float32}


class Rank3Job:
    def __init__(self, workers: int, max_workers: int | None = None, odf: int = 1,
                 ref_path: str = DEFAULT_REF, scratch: str | None = None, spares: int | None = None):
        if ref_path not in sys.path:
            sys.path.insert(0, ref_path)
        from elastencil.coordinator import Coordinator  # the reference, unmodified

        self.workers = workers
        self.max_workers = max_workers or workers
        self.odf = odf
        self.scratch = scratch or f"/tmp/est-r3-{os.getpid()}-{int(time.time() * 1000)}"
        os.makedirs(self.scratch, exist_ok=True)
        self.coord = Coordinator("127.0.0.1:0", workers, self.max_workers, odf, self.scratch)
        self.launcher = GpuLauncher(workers, self.max_workers, odf, scratch=self.scratch,
                                    coordinator_pythonpath=ref_path,
                                    control_endpoint=self.coord.control_endpoint, spares=spares)
        self.shapes: dict = {}
        self.dtypes: dict = {}
        self._seq = 0

    # -- lifecycle (coordinator.serve_forever's start-up, coordinator.py:281-289)
    def start(self) -> "Rank3Job":
        self.launcher.start()
        c = self.coord
        c.wait_daemons(self.max_workers, timeout=180)
        c.wait_workers(self.workers, timeout=180)
        c.init_workers()
        c.notify_launcher_ready()
        self.launcher.wait_ready()
        return self

    def close(self) -> None:
        try:
            self.coord._do_shutdown()
        finally:
            self.launcher.shutdown()
            for s in (self.coord.client_sock, self.coord.control_sock):
                try:
                    s.close()
                except OSError:
                    pass

    def __enter__(self) -> "Rank3Job":
        return self.start()

    def __exit__(self, *exc) -> None:
        self.close()

    # -- client-side steps the reference limits to rank 1/2 ---------------------
    def create_array(self, shape, dtype: int = DTYPE_F64) -> int:
        """W_CREATE exactly as coordinator._cmd_create sends it (coordinator.py:381-404)."""
        from elastencil.grid import Decomposition, most_square_factors

        from .tiles import Decomposition as SlabCheck

        c = self.coord
        shape = tuple(int(e) for e in shape)
        if c.decomp is None:
            # the reference decomposition object (tile grid = most-square
            # factors of odf*W, grid.py:105-117; owner maps, migration plans
            # and manifests come from it); the workers split rank-3 arrays into
            # z-slabs in its linear tile order (tiles.Decomposition), so the
            # divisibility rule checked is theirs
            grid = most_square_factors(c.odf * c.initial_workers)
            SlabCheck(grid, c.odf, c.initial_workers).check_divisible(shape)
            c.decomp = Decomposition(grid, c.odf, c.initial_workers)
        aid = c.next_array_id
        meta = {"array": aid, "shape": list(shape), "dtype": int(dtype),
                "decomp": {"tile_grid": list(c.decomp.tile_grid), "odf": c.decomp.odf,
                           "initial_workers": c.decomp.initial_workers}}
        c._await_ok([w.request(W_CREATE, meta) for w in c._live_workers()])
        c.next_array_id += 1
        c.arrays[aid] = shape
        self.shapes[aid] = shape
        self.dtypes[aid] = dtype
        return aid

    def submit(self, dag_bytes: bytes) -> None:
        """W_BATCH to every live worker, replies collected at the next barrier
        (coordinator._cmd_batch, coordinator.py:406-429)."""
        c = self.coord
        batch_id = c.stats.batches + len(c.pending_batches)
        c.pending_batches.append((batch_id, [w.request(W_BATCH, {"batch": batch_id}, dag_bytes)
                                             for w in c._live_workers()]))

    def barrier(self) -> None:
        self.coord._barrier()
        self.coord._raise_session_error()

    def sync(self) -> None:
        """Barrier + a synchronising command on every worker (a one-element
        fetch: workers drain their streams before answering W_FETCH)."""
        a = next(iter(self.shapes))
        self.fetch(a, tuple((0, 1) for _ in self.shapes[a]))

    def fetch(self, array: int, bounds=None) -> np.ndarray:
        """coordinator._cmd_fetch's gather (coordinator.py:466-496), dtype-aware."""
        self.barrier()
        c = self.coord
        shape = self.shapes[array]
        bounds = tuple(tuple(b) for b in bounds) if bounds is not None else tuple((0, e) for e in shape)
        replies = c._await_ok([w.request(W_FETCH, {"array": array, "bounds": [list(b) for b in bounds]})
                               for w in c._live_workers()])
        dt = np.dtype(NP[self.dtypes[array]])
        out = np.zeros([b - a for a, b in bounds], dtype=dt)
        for pending in replies:
            off = 0
            for piece in pending.meta["pieces"]:
                ext = [b - a for a, b in piece]
                n = int(np.prod(ext)) * dt.itemsize
                block = np.frombuffer(pending.blob[off:off + n], dtype=dt).reshape(ext)
                off += n
                out[tuple(slice(a - lo, b - lo) for (a, b), (lo, _) in zip(piece, bounds))] = block
        return out

    def hash(self, array: int) -> int:
        """Whole-array content hash: the sum of every worker's W_HASH partial
        (est_hash_box over its tiles), equal for equal arrays under any
        decomposition."""
        self.barrier()
        c = self.coord
        replies = c._await_ok([w.request(W_HASH, {"array": array}) for w in c._live_workers()])
        return sum(int(p.meta["hash"]) for p in replies) % (1 << 64)

    # -- the reference rescale, unmodified ---------------------------------------
    def rescale(self, count: int) -> dict:
        """coordinator._cmd_rescale (coordinator.py:501-518): barrier, then the
        shrink (lb -> ckpt -> restart -> restore) or expand (ckpt -> restart ->
        restore -> lb) stages; -> the four StageTimings and the wall total."""
        self._seq += 1
        t0 = time.perf_counter()
        self.coord._cmd_rescale(SimpleNamespace(count=count, seq=self._seq))  # raises on failure
        total = (time.perf_counter() - t0) * 1e3
        out = dict(self.coord.stats.rescales[-1])
        out["total_ms"] = total
        return out

    def stats(self) -> dict:
        self.barrier()
        return self.coord.stats.snapshot()
