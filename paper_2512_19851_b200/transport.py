"""Peer halo transport between GPU workers: pull over peer memory, event-gated.

Replaces the reference's TCP strip path (exchange.py:169-234 send/receive,
worker.py:61-248 PeerHub + busy-poll). For every round (array, epoch) — a
sequence all tile-owning workers derive identically from the DAG — worker w:

  1. records its READY event (slot r mod K) on its compute stream, right after
     whatever last wrote the array, and publishes ready_seq[w] = r;
  2. issues its co-located strip copies;
  3. for each remote neighbour p: waits on the host until ready_seq[p] >= r
     (so p's READY slot holds a record of round >= r), makes its own compute
     stream wait on that event, then pulls the strips straight from p's HBM
     tile buffer into its own ghost regions (one batched copy kernel; over
     NVLink when p lives on another GPU);
  4. records PULLED (slot r mod K) and publishes pulled_seq[w] = r.

Before a later node overwrites that array, the worker makes its stream wait on
the PULLED events of the peers that read from it in that round
(`before_write`) — the write-after-read edge the reference gets for free from
copying strips into messages. Waiting on a slot re-recorded by a LATER round is
only over-synchronisation: every record depends solely on work enqueued before
it was published, so no cycle can form.

`LocalPeerTransport` runs this between workers of one process (threads; the
reference LocalMesh analogue, usable on a single GPU). `ipc.IpcPeerTransport`
runs the same round protocol across processes entirely on the device: CUDA IPC
buffers plus READY / PULLED flag words written and waited on by the streams
themselves (stream memory operations), so no host thread waits on a peer.
"""

from __future__ import annotations

import threading

from .codegen import ELEM
from .device import COMPUTE, COPY
from .exchange import strip_copy

RING = 16


class TransportAborted(RuntimeError):
    pass


class LocalPeerGroup:
    """Shared host state of the in-process peers."""

    def __init__(self, stores):
        self.stores = stores
        self.n = len(stores)
        self.cond = threading.Condition()
        self.ready_seq = [-1] * self.n
        self.pulled_seq = [-1] * self.n
        self.transports: list = [None] * self.n
        self.error = None
        self._bar_count = 0
        self._bar_gen = 0

    def wait_for(self, pred, what: str) -> None:
        with self.cond:
            while not pred():
                if self.error is not None:
                    raise TransportAborted(f"peer failed while waiting for {what}: {self.error!r}")
                self.cond.wait(0.5)

    def publish(self, table: list, w: int, r: int) -> None:
        with self.cond:
            table[w] = r
            self.cond.notify_all()

    def barrier(self) -> None:
        with self.cond:
            gen = self._bar_gen
            self._bar_count += 1
            if self._bar_count == self.n:
                self._bar_count = 0
                self._bar_gen += 1
                self.cond.notify_all()
                return
            while gen == self._bar_gen:
                if self.error is not None:
                    raise TransportAborted(f"peer failed in barrier: {self.error!r}")
                self.cond.wait(0.5)

    def abort(self, exc) -> None:
        with self.cond:
            if self.error is None:
                self.error = exc
            self.cond.notify_all()


class LocalPeerTransport:
    def __init__(self, group: LocalPeerGroup, worker: int):
        self.group = group
        self.w = worker
        self.store = group.stores[worker]
        self.dev = self.store.dev
        self.seq = 0
        self.ready = [self.dev.event() for _ in range(RING)]
        self.pulled = [self.dev.event() for _ in range(RING)]
        self.readers: dict = {}
        self.pull_launches = 0
        self.peer_version = 0
        self._pulls: dict = {}
        group.transports[worker] = self

    # -- peer views (overridden by the IPC transport) -------------------------
    def peer_buffer(self, owner: int, coords, array: int):
        """(TileBuffer describing the layout, address to read from)."""
        buf = self.group.stores[owner].tiles[coords].buffers[array]
        return buf, buf.ptr

    def peer_event(self, owner: int, kind: str, slot: int):
        return getattr(self.group.transports[owner], kind)[slot]

    def wait_seq(self, owner: int, kind: str, r: int) -> None:
        table = self.group.ready_seq if kind == "ready" else self.group.pulled_seq
        self.group.wait_for(lambda: table[owner] >= r, f"{kind}[{owner}] >= {r}")

    def publish(self, kind: str, r: int) -> None:
        table = self.group.ready_seq if kind == "ready" else self.group.pulled_seq
        self.group.publish(table, self.w, r)

    # -- protocol -------------------------------------------------------------
    chains_ok = False  # the in-process peers do not share the temporal chains' twin buffers

    def exchange(self, array: int, epoch: int, remote, local_boxes, twin: bool = False) -> None:
        self.finish(self.post(array, epoch, remote, local_boxes, twin), overlap=False)

    def post(self, array: int, epoch: int, remote, local_boxes, twin: bool = False):
        """Steps 1-2: READY record + co-located copies; the peer pull is left
        to `finish`, which the executor may defer past the next node's
        interior launch (halo/compute overlap)."""
        r = self.seq
        self.seq += 1
        slot = r % RING
        elem = ELEM[self.store.arrays[array].dtype]
        self.ready[slot].record(COMPUTE)
        self.publish("ready", r)
        if local_boxes:
            self.dev.copy_boxes(local_boxes, elem)
        return (array, r, remote, elem, twin)

    def finish(self, token, overlap: bool = False) -> None:
        """Steps 3-4. With `overlap` the pull runs on the COPY stream (after
        this worker's own READY, so the previous readers of the ghost are
        done) and the compute stream only joins it before the boundary work
        (`join_copy`)."""
        array, r, remote, elem, twin = token
        slot = r % RING
        lane = COMPUTE
        if overlap and remote:
            lane = COPY
            self.ready[slot].wait(COPY)
        peers = sorted({owner for _, _, _, owner in remote})
        for p in peers:
            self.wait_seq(p, "ready", r)
            self.peer_event(p, "ready", slot).wait(lane)
        if remote:
            self.dev.copy_boxes(self._pull_boxes(array, remote, twin), elem, lane)
            self.pull_launches += 1
        self.pulled[slot].record(lane)
        self.publish("pulled", r)
        if peers:
            self.readers[array] = (r, peers)

    def _pull_boxes(self, array: int, remote, twin: bool = False) -> list:
        """Copy descriptors of one round's remote strips (cached per layout);
        `twin`: between the temporal chains' twin buffers (mid-run)."""
        ck = (array, self.store.version, self.peer_version, id(remote), twin)
        boxes = self._pulls.get(ck)
        if boxes is None:
            boxes = []
            for coords, d, nb, owner in remote:
                src_buf, src_addr = self.peer_buffer(owner, nb, ("twin", array) if twin else array)
                dst_buf = self.store.twins[(coords, array)] if twin else self.store.tiles[coords].buffers[array]
                boxes.append(strip_copy(src_buf, dst_buf, d, src_addr_override=src_addr))
            if len(self._pulls) > 1024:
                self._pulls.clear()
            self._pulls[ck] = boxes
        return boxes

    def join_copy(self, r: int) -> None:
        """Compute stream waits for the overlapped pull of round r."""
        self.pulled[r % RING].wait(COMPUTE)

    def before_write(self, array: int) -> None:
        ent = self.readers.pop(array, None)
        if ent is None:
            return
        r, peers = ent
        for p in peers:
            self.wait_seq(p, "pulled", r)
            self.peer_event(p, "pulled", r % RING).wait(COMPUTE)

    def before_realloc(self) -> None:
        """All peers idle and past every pull of the old buffers."""
        self.dev.sync()
        self.group.barrier()
        self.readers.clear()

    def after_realloc(self) -> None:
        self.peer_version += 1
        self.group.barrier()

    def abort(self, exc) -> None:
        self.group.abort(exc)

    def close(self) -> None:
        for ev in self.ready + self.pulled:
            ev.close()
