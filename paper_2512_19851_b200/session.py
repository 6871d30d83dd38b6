"""In-process job driver: W GPU workers behind one Python object.

The reference's in-process harness (pkg/tests/mesh.py:23-122, `LocalMesh`)
wires N TileStore+Executor pairs together; `GpuJob` does the same for the GPU
backend: each worker owns a `Device` (its own compute/copy streams), a
`GpuTileStore`, a `GpuExchangeManager` and a `GpuExecutor`. With one worker
there is no transport; with several, `transport.LocalPeerTransport` moves the
halo strips between the workers' HBM buffers with stream/event ordering, the
same protocol the multi-process IPC transport runs over CUDA IPC.

The production path (the reference coordinator driving GPU worker processes)
is `worker.py`; `GpuJob` is the API used by bench.py, smoke() and the parity
tests, and by users who want the backend without the socket control plane.
"""

from __future__ import annotations

import threading

import numpy as np

from .device import Device, PinnedBuffer
from .exchange import GpuExchangeManager
from .executor import GpuExecutor
from .tiles import ArrayInfo, GpuTileStore, decompose
from .wire import DTYPE_F64


class GpuJob:
    def __init__(self, workers: int = 1, odf: int = 1, devices=None, skeleton: str = "auto"):
        self.workers = workers
        self.odf = odf
        devices = list(devices) if devices is not None else [0] * workers
        self.devs = [Device(d) for d in devices]
        self.skeleton = skeleton
        self.decomp = None
        self.stores, self.managers, self.executors = [], [], []
        self.transports = []
        self._next = 0
        self.shapes: dict = {}
        self.dtypes: dict = {}
        self._stage = None
        from .wire import DagCache

        self._decoded = DagCache()

    def _build(self, shape) -> None:
        self.decomp = decompose(shape, self.workers, self.odf)
        owners = self.decomp.owner_map(self.workers)
        for w in range(self.workers):
            owned = [c for c, o in owners.items() if o == w]
            self.stores.append(GpuTileStore(self.devs[w], self.decomp, owned))
        if self.workers > 1:
            from .transport import LocalPeerTransport, LocalPeerGroup

            group = LocalPeerGroup(self.stores)
            self.transports = [LocalPeerTransport(group, w) for w in range(self.workers)]
        for w in range(self.workers):
            tr = self.transports[w] if self.transports else None
            mgr = GpuExchangeManager(self.stores[w], w, owners, tr)
            self.managers.append(mgr)
            ex = GpuExecutor(self.stores[w], mgr, self.skeleton)
            if tr is not None:
                ex.transport = tr
            self.executors.append(ex)

    def create_array(self, shape, dtype: int = DTYPE_F64) -> int:
        shape = tuple(int(e) for e in shape)
        if self.decomp is None:
            self._build(shape)
        aid = self._next
        for st in self.stores:
            st.create_array(ArrayInfo(aid, shape, dtype))
        self._next += 1
        self.shapes[aid] = shape
        self.dtypes[aid] = dtype
        return aid

    def run_bytes(self, blob: bytes) -> list:
        """Execute a batch given as DAG bytes (the W_BATCH payload).

        Repeated batches skip decode and, on a single worker, replay a captured
        CUDA graph (executor.GpuExecutor.execute_batch `key`)."""
        key, dag = self._decoded.get(blob)
        return self.run(dag, key)

    def run(self, dag, key: bytes | None = None) -> list:
        if self.workers == 1:
            return [self.executors[0].execute_batch(dag, key)]
        results = [None] * self.workers
        errors = []

        def work(w):
            try:
                results[w] = self.executors[w].execute_batch(dag)
            except BaseException as exc:  # surfaced after join
                errors.append(exc)
                for t in self.transports:
                    t.abort(exc)

        threads = [threading.Thread(target=work, args=(w,)) for w in range(self.workers)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return results

    def sync(self) -> None:
        for d in self.devs:
            d.sync()

    def fetch(self, array: int, bounds=None) -> np.ndarray:
        self.sync()
        shape = self.shapes[array]
        bounds = tuple(bounds) if bounds is not None else tuple((0, e) for e in shape)
        out = None
        nbytes = int(np.prod([b - a for a, b in bounds])) * 8
        if self._stage is None or self._stage.nbytes < nbytes:
            if self._stage is not None:
                self._stage.close()
            self._stage = PinnedBuffer(max(nbytes, 1 << 20))
        for st in self.stores:
            if not st.tiles:
                continue
            part = st.gather_slice_pieces(array, bounds, self._stage)
            if out is None:
                out = np.zeros([b - a for a, b in bounds], dtype=st.fetch_dtype(array))
            for piece, block in part:
                out[tuple(slice(a - lo, b - lo) for (a, b), (lo, _) in zip(piece, bounds))] = block
        return out

    def hash(self, array: int) -> int:
        """Whole-array position-keyed content hash (est_hash_box), summed over
        every worker's tiles: a decomposition-independent fingerprint."""
        self.sync()
        return sum(st.hash(array) for st in self.stores if st.tiles) % (1 << 64)

    def rounds_by_array(self) -> dict:
        counts = [m.snapshot_stats()["rounds"] for m in self.managers if m.store.tiles]
        for c in counts[1:]:
            assert c == counts[0], "workers disagree on round counts"
        return counts[0] if counts else {}

    def close(self) -> None:
        for ex in self.executors:
            ex.drop_replays()
        if self._stage is not None:
            self._stage.close()
            self._stage = None
        for t in self.transports:
            t.close()
        for st in self.stores:
            st.release()
        for d in self.devs:
            d.close()
        self.stores.clear()
        self.devs.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def run_program(prog, workers: int = 1, odf: int = 1, fused: bool = False, skeleton: str = "auto",
                job: GpuJob | None = None, batch: int | None = None):
    """Create the program's arrays on a GpuJob and run its DAG (optionally in batches)."""
    from .ir import Dag, DagNode, compute_edges, fuse

    job = job or GpuJob(workers, odf, skeleton=skeleton)
    for aid in sorted(prog.shapes):
        got = job.create_array(prog.shapes[aid], getattr(prog, "dtypes", {}).get(aid, DTYPE_F64))
        assert got == aid
    dag = fuse(prog.dag) if fused else prog.dag
    stats = []
    if batch:
        for k in range(0, len(dag.nodes), batch):
            nodes = [DagNode(i, n.statements) for i, n in enumerate(dag.nodes[k:k + batch])]
            part = Dag(nodes, compute_edges(nodes), dag.ast_table)
            stats.append(job.run(part))
    else:
        stats.append(job.run(dag))
    return job, stats
