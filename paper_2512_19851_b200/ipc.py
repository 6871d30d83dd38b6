"""Multi-process GPU workers: one process per GPU, halos over CUDA IPC.

`IpcGpuJob(rank, world, device)` is one worker of an SPMD job (launched by
torchrun, the driver's bench launcher, or `spawn_local_job` in tests). Every
rank decodes and executes the same DAG; the block owner map decides which
tiles each rank owns (grid.py:63-76). torch.distributed (gloo) is used only as
plumbing: rendezvous, exchanging IPC handles, barriers and host gathers.

The data path never touches the host:

* each rank exports a CUDA IPC memory handle per (tile, array) HBM buffer and
  IPC event handles for its READY / PULLED event rings (transport.py);
* halo strips are pulled by the receiver's copy kernel straight out of the
  owner's mapped buffer (NVLink P2P between GPUs; also works between processes
  sharing one GPU, which is how the 1-GPU test box exercises this path);
* round signalling is DEVICE-side: every rank owns two 32-bit flag words
  (READY, PULLED) in its exported arena; a round's READY is a stream write
  (`est_flag_write`, release) behind the array's last writer, the receiver's
  copy stream waits on the owner's flag word (`est_flag_wait`, a front-end
  semaphore acquire over NVLink) before its pull, and PULLED gates the owner's
  next overwrite. The host never waits on a peer inside a batch: no per-round
  host handshake, no IPC event waits (24 us each on the host, profiles/
  r2_ipc_host_profile.txt). A /dev/shm page keeps only the abort flags, which
  `sync` polls so a dead peer raises instead of hanging the stream.
"""

from __future__ import annotations

import mmap
import os
import time
import uuid

import numpy as np

from .device import Device, PinnedBuffer
from .exchange import GpuExchangeManager
from .executor import GpuExecutor
from .tiles import ArrayInfo, GpuTileStore, TileBuffer, decompose
from .codegen import ELEM
from .device import COMPUTE, COPY
from .transport import RING, LocalPeerTransport, TransportAborted
from .wire import DTYPE_F64


class SharedCounters:
    """int64 [3, world] in /dev/shm: ready_seq, pulled_seq, abort flag."""

    def __init__(self, path: str, world: int, create: bool):
        self.path = path
        size = 3 * world * 8
        if create:
            with open(path, "wb") as fh:
                fh.write(b"\xff" * size)  # -1 everywhere
        self.fh = open(path, "r+b")
        self.mm = mmap.mmap(self.fh.fileno(), size)
        self.arr = np.ndarray((3, world), dtype=np.int64, buffer=self.mm)
        if create:
            self.arr[2, :] = 0

    def close(self) -> None:
        try:
            del self.arr
            self.mm.close()
            self.fh.close()
        except Exception:
            pass


READY_OFF, PULLED_OFF = 0, 128  # byte offsets of the two flag words (separate 128-B lines)
FLAGS_KEY = (("flags",), -1)     # buffer-table key of a rank's flag block
# the halo arena: flags + halo windows, the only memory a halo neighbour maps
HALO_ARENA = int(os.environ.get("EST_HALO_ARENA_BYTES", 64 << 20))
WINDOWS = os.environ.get("EST_HALO_WINDOWS", "1") == "1"


class IpcPeerTransport(LocalPeerTransport):
    """transport.py round protocol across processes: CUDA IPC buffers and
    device-side flag words (see the module docstring).

    Per round r (sequence shared by all ranks, value r + 1 on the wire):
      post      READY := r+1 on the compute stream (behind the array's writer)
      finish    per remote owner p: lane waits READY[p] >= r+1, pulls the
                strips, then PULLED := r+1 on the lane
      before_write  (the next overwrite of the array) compute waits
                PULLED[p] >= r+1 for every peer that read from us in round r
    Monotonic values make a later round's write only over-synchronise. PULLED
    is written from the copy lane for overlapped rounds and from the compute
    stream otherwise; the executor joins the copy lane into the compute
    stream (`join_copy`) before any later compute-stream write, so the word
    never goes backwards."""

    def __init__(self, job: "IpcGpuJob"):
        from .pool import DevicePool

        self.job = job
        self.w = job.rank
        self.store = job.store
        self.dev = job.dev
        self.seq = 0
        # flags and the rank-3 halo windows live in their own small exported
        # arena: halo neighbours map only that, never the GiB-sized tile arenas
        self.hpool = DevicePool(self.dev, HALO_ARENA, grow=2)
        self.flags = self.hpool.alloc(256)  # [READY_OFF] ready, [PULLED_OFF] pulled; zeroed
        self.windows: dict = {}  # (coords, array) -> (ptr, signature): the slab's boundary planes
        self.window_maps: set = set()  # peers' windows this rank has pulled from (introspection)
        self._exports: dict = {}
        self.ready = [self.dev.event() for _ in range(RING)]   # intra-process: copy lane after compute
        self.pulled = [self.dev.event() for _ in range(RING)]  # intra-process: compute after copy lane
        self.peer_flag_base: dict = {}
        self.readers: dict = {}
        self.pull_launches = 0
        self.peer_events: dict = {}
        self.peer_maps: dict = {}      # (owner, coords, array) -> (layout TileBuffer, addr, identity)
        self.peer_tables: dict = {}    # (owner, coords, array) -> buffer_table entry
        self.arena_maps: dict = {}     # (owner, arena serial) -> mapped base
        self.peer_event_handles: dict = {}
        self.spin_s = 0.0
        self.peer_version = 0
        self._pulls: dict = {}

    # -- handle exchange ---------------------------------------------------------
    def event_handles(self) -> dict:
        return {}  # rounds are signalled through device flags (no IPC events)

    def open_peer_events(self, table: dict) -> None:
        self.peer_event_handles = {}

    def buffer_table(self) -> dict:
        """(coords, array) -> (arena serial, arena IPC handle, offset, extents,
        depth, dtype, buffer serial): buffers live in the worker's arenas
        (pool.py), so a peer maps each arena once."""
        out = {}
        pool = self.dev.pool
        for coords, tile in self.store.tiles.items():
            for array, buf in tile.buffers.items():
                serial, handle, off = pool.locate(buf.ptr)
                out[(tuple(coords), array)] = (serial, handle, off, buf.ext[3 - buf.rank:],
                                               buf.depth[3 - buf.rank:], buf.dtype, buf.serial)
        for (coords, array), buf in self.store.twins.items():
            serial, handle, off = pool.locate(buf.ptr)
            out[(tuple(coords), ("twin", array))] = (serial, handle, off, buf.ext[3 - buf.rank:],
                                                      buf.depth[3 - buf.rank:], buf.dtype, buf.serial)
        self._ensure_windows()
        for (coords, array), (ptr, _sig) in self.windows.items():
            serial, handle, off = self.hpool.locate(ptr)
            out[(tuple(coords), ("win", array))] = (serial, handle, off, (), (), 0, ptr)
        serial, handle, off = self.hpool.locate(self.flags)
        out[FLAGS_KEY] = (serial, handle, off, (), (), 0, 0)
        return out

    # -- halo windows (rank-3 slabs) -----------------------------------------------
    # A slab's neighbours read only its pd boundary planes on each side (pd =
    # the array's physical z ghost depth). Before READY the owner copies those
    # planes (from whichever buffer holds the array: home, or the temporal
    # chain's twin mid-run) into a small window [lo: pd planes | hi: pd
    # planes] in the halo arena, and the neighbours pull from the window. A
    # restarted or re-mapped worker then maps a few MiB per neighbour instead
    # of the neighbour's whole tile arena (~65 ms per GiB mapped,
    # profiles/r2_c5_stage_split.md). The copy costs 2*pd planes per round
    # (C4 on 8 GPUs: 32 MiB, ~10 us, against ~0.5 ms of chain compute).

    @staticmethod
    def _window_sig(buf) -> tuple:
        return (buf.py, buf.pz, buf.xoff, tuple(buf.depth), tuple(buf.ext), buf.elem)

    def _ensure_windows(self) -> None:
        want = {}
        if WINDOWS:
            for coords, tile in self.store.tiles.items():
                for a, buf in tile.buffers.items():
                    if buf.rank == 3 and buf.depth[0] > 0:
                        want[(tuple(coords), a)] = buf
        for key in list(self.windows):
            ptr, sig = self.windows[key]
            if key not in want or sig != self._window_sig(want[key]):
                self.hpool.free(ptr)
                del self.windows[key]
        for key, buf in sorted(want.items()):
            if key not in self.windows:
                nbytes = 2 * buf.depth[0] * buf.pz * buf.elem
                self.windows[key] = (self.hpool.alloc(nbytes), self._window_sig(buf))
        self._exports.clear()

    def _window_box(self, buf, win: int, side: str, export: bool, dst_buf=None):
        """Copy descriptor between a slab's boundary planes and a window
        region: `side` "lo" = the first pd interior planes, "hi" = the last
        pd. export: slab -> own window; else window (a peer's, mapped at
        `win`) -> the ghost planes of `dst_buf` on the side facing it."""
        from ._lib import EstBox

        pd = buf.depth[0]
        ez, ey, ex = buf.ext
        inplane = (buf.xoff + buf.depth[1] * buf.py + buf.depth[2]) * buf.elem
        region = win + (0 if side == "lo" else pd * buf.pz * buf.elem) + inplane
        if export:
            src = buf.interior_addr((0 if side == "lo" else ez - pd, 0, 0))
            return EstBox(src, region, buf.py, buf.pz, buf.py, buf.pz, ex, ey, pd)
        # the peer's lo planes fill our high ghost planes (it is our E
        # neighbour), its hi planes our low ghost planes
        gz = pd + ez if side == "lo" else 0
        return EstBox(region, dst_buf.addr(gz, dst_buf.depth[1], dst_buf.depth[2]), buf.py, buf.pz,
                      dst_buf.py, dst_buf.pz, ex, ey, pd)

    def _export_boxes(self, array: int, twin: bool) -> list:
        from .exchange import E, W, neighbour

        ck = (array, self.store.version, id(self.job.owner_map), twin)
        boxes = self._exports.get(ck)
        if boxes is None:
            boxes = []
            owners = self.job.owner_map or {}
            info = self.store.arrays[array]
            for coords in sorted(self.store.tiles):
                if (tuple(coords), array) not in self.windows:
                    continue
                buf = self.store.twins[(coords, array)] if twin else self.store.tiles[coords].buffers[array]
                win = self.windows[(tuple(coords), array)][0]
                for d, side in ((W, "lo"), (E, "hi")):
                    nb = neighbour(self.store.decomp, info.rank, coords, d)
                    if nb is not None and owners.get(nb, self.w) != self.w:
                        boxes.append(self._window_box(buf, win, side, True))
            if len(self._exports) > 256:
                self._exports.clear()
            self._exports[ck] = boxes
        return boxes

    def peer_window(self, owner: int, coords, array: int) -> int:
        """Mapped address of `owner`'s halo window of (coords, array)."""
        aserial, handle, off = self.peer_tables[(owner, tuple(coords), ("win", array))][:3]
        self.window_maps.add((owner, tuple(coords), array))
        base = self.arena_maps.get((owner, aserial))
        if base is None:
            base = self.arena_maps[(owner, aserial)] = self.dev.ipc_open(handle)
        return base + off

    def _uses_windows(self, array: int) -> bool:
        return WINDOWS and self.store.arrays[array].rank == 3

    def _pull_boxes(self, array: int, remote, twin: bool = False) -> list:
        if not self._uses_windows(array):
            return super()._pull_boxes(array, remote, twin)
        from .exchange import E

        ck = (array, self.store.version, self.peer_version, id(remote), twin, "win")
        boxes = self._pulls.get(ck)
        if boxes is None:
            boxes = []
            for coords, d, nb, owner in remote:
                dst = self.store.twins[(coords, array)] if twin else self.store.tiles[coords].buffers[array]
                win = self.peer_window(owner, nb, array)
                boxes.append(self._window_box(dst, win, "lo" if d == E else "hi", False, dst))
            if len(self._pulls) > 1024:
                self._pulls.clear()
            self._pulls[ck] = boxes
        return boxes

    def open_peer_buffers(self, tables: list) -> None:
        """Install the peers' buffer handle tables. Mappings are opened lazily
        (`peer_buffer`): a worker maps only the tiles it actually reads
        (halo neighbours, migration sources). A mapping whose handle is
        unchanged survives; changed / departed buffers are unmapped."""
        self.peer_version += 1
        wanted = {}
        for owner, table in enumerate(tables):
            if owner == self.w:
                continue
            for (coords, array), entry in table.items():
                wanted[(owner, tuple(coords), array)] = entry
        for key, (_layout, _addr, ident) in list(self.peer_maps.items()):
            ent = wanted.get(key)
            if ent is None or (ent[0], ent[2], ent[6]) != ident:
                del self.peer_maps[key]  # the arena mapping itself stays (arenas live with the job)
        self.peer_tables = wanted

    def map_neighbours(self) -> int:
        """Open, now, the mappings / events halo rounds will use: every array
        of every remote tile adjacent to an owned tile (a bounded set, unlike
        the full table). Returns the number of mappings opened."""
        from .exchange import N, E, W, neighbour

        before = len(self.peer_maps)
        owners = self.job.owner_map or {}
        peers = set()
        for coords in self.store.tiles:
            for a, info in self.store.arrays.items():
                dirs = (E, W) if info.rank != 2 else range(N, N + 8)
                for d in dirs:
                    nb = neighbour(self.store.decomp, info.rank, coords, d)
                    if nb is None or owners.get(nb, self.w) == self.w:
                        continue
                    if self._uses_windows(a):
                        if (owners[nb], tuple(nb), ("win", a)) in self.peer_tables:
                            self.peer_window(owners[nb], nb, a)
                            peers.add(owners[nb])
                        continue
                    for arr in (a, ("twin", a)):
                        key = (owners[nb], tuple(nb), arr)
                        if key in self.peer_tables:
                            self.peer_buffer(*key)
                            peers.add(owners[nb])
        for p in peers:
            self.peer_flags(p)
        return len(self.peer_maps) - before

    def close_peer_buffers(self) -> None:
        """Forget the per-buffer views (a realloc or migration republishes
        the tables); the peers' arena mappings are kept until close()."""
        self.peer_maps.clear()
        self.peer_tables = {}

    def close_arenas(self) -> None:
        for base in self.arena_maps.values():
            try:
                self.dev.ipc_close(base)
            except Exception:
                pass
        self.arena_maps.clear()

    # -- protocol hooks ----------------------------------------------------------
    def peer_buffer(self, owner: int, coords, array: int):
        key = (owner, tuple(coords), array)
        hit = self.peer_maps.get(key)
        if hit is None:
            aserial, handle, off, ext, depth, dtype, serial = self.peer_tables[key]
            base = self.arena_maps.get((owner, aserial))
            if base is None:
                base = self.arena_maps[(owner, aserial)] = self.dev.ipc_open(handle)
            addr = base + off
            layout = TileBuffer(self.dev, ext, depth, dtype, ptr=addr)
            hit = self.peer_maps[key] = (layout, addr, (aserial, off, serial))
        return hit[0], hit[1]

    def peer_event(self, owner: int, kind: str, slot: int):
        evs = self.peer_events.setdefault(owner, {})
        lst = evs.get(kind)
        if lst is None:
            lst = evs[kind] = [None] * len(self.peer_event_handles[owner][kind])
        ev = lst[slot]
        if ev is None:
            ev = lst[slot] = self.dev.open_event(self.peer_event_handles[owner][kind][slot])
        return ev

    def peer_flags(self, owner: int) -> int:
        """Device address of `owner`'s flag block (its arena, mapped once)."""
        base = self.peer_flag_base.get(owner)
        if base is None:
            aserial, handle, off = self.peer_tables[(owner,) + FLAGS_KEY][:3]
            arena = self.arena_maps.get((owner, aserial))
            if arena is None:
                arena = self.arena_maps[(owner, aserial)] = self.dev.ipc_open(handle)
            base = self.peer_flag_base[owner] = arena + off
        return base

    # -- the round protocol on device flags ---------------------------------------
    chains_ok = True  # halo planes go through the owners' windows (home or twin), so slabs chain

    def graph_safe(self) -> bool:
        """Batches may be captured into CUDA graphs and replayed when no peer
        exists (a one-worker job: the GPU worker process behind a one-worker
        coordinator). A replay re-writes this rank's READY / PULLED flags with
        the captured values and does not advance `seq`; with peers those
        words must grow monotonically, so multi-worker batches run
        uncaptured. A later change of the worker count goes through a
        restart (fresh transports) in the reference rescale."""
        return self.job.world == 1

    def post(self, array: int, epoch: int, remote, local_boxes, twin: bool = False):
        r = self.seq
        self.seq += 1
        elem = ELEM[self.store.arrays[array].dtype]
        if self._uses_windows(array):
            exports = self._export_boxes(array, twin)
            if exports:
                self.dev.copy_boxes(exports, elem)
        self.dev.flag_write(self.flags + READY_OFF, r + 1, COMPUTE)
        if local_boxes:
            self.dev.copy_boxes(local_boxes, elem)
        return (array, r, remote, elem, twin)

    def finish(self, token, overlap: bool = False) -> None:
        array, r, remote, elem, twin = token
        slot = r % RING
        lane = COMPUTE
        if overlap and remote:
            lane = COPY
            self.ready[slot].record(COMPUTE)  # previous readers of the ghost are done
            self.ready[slot].wait(COPY)
        peers = sorted({owner for _, _, _, owner in remote})
        for p in peers:
            self.dev.flag_wait(self.peer_flags(p) + READY_OFF, r + 1, lane)
        if remote:
            self.dev.copy_boxes(self._pull_boxes(array, remote, twin), elem, lane)
            self.pull_launches += 1
        self.dev.flag_write(self.flags + PULLED_OFF, r + 1, lane)
        if lane != COMPUTE:
            self.pulled[slot].record(lane)
        if peers:
            self.readers[array] = (r, peers)

    def join_copy(self, r: int) -> None:
        self.pulled[r % RING].wait(COMPUTE)

    def before_write(self, array: int) -> None:
        ent = self.readers.pop(array, None)
        if ent is None:
            return
        r, peers = ent
        for p in peers:
            self.dev.flag_wait(self.peer_flags(p) + PULLED_OFF, r + 1, COMPUTE)

    def before_realloc(self) -> None:
        self.job.sync()
        self.job.barrier()
        self.readers.clear()
        self.close_peer_buffers()

    def after_realloc(self) -> None:
        self.job.exchange_buffers()

    def abort(self, exc) -> None:
        self.job.counters.arr[2, self.w] = 1

    def close(self) -> None:
        self.close_peer_buffers()
        self.peer_flag_base.clear()
        self.close_arenas()
        for e in self.ready + self.pulled:
            e.close()
        self.windows.clear()
        self.hpool.release()


class IpcGpuJob:
    """One rank of a multi-process GPU job (same API as session.GpuJob).

    `group` is the host plumbing (hostgroup.GlooGroup by default, or the
    worker's PeerGroup); `decomp` may be imposed (the coordinator's fixed
    decomposition, grid.py:43-117) instead of derived from the first shape.
    """

    def __init__(self, rank: int, world: int, device: int = 0, odf: int = 1,
                 skeleton: str = "auto", group=None, timeout_s: float = 600.0,
                 decomp=None, owner_map: dict | None = None, dev: Device | None = None):
        if group is None:
            import torch.distributed as dist

            if not dist.is_initialized():
                dist.init_process_group("gloo", rank=rank, world_size=world)
            from .hostgroup import GlooGroup

            group = GlooGroup()
        self.group = group
        self.rank, self.world, self.odf = rank, world, odf
        self.timeout_s = timeout_s
        self.dev = dev if dev is not None else Device(device)  # a worker may pre-create it
        from .pool import DevicePool

        self.dev.pool = DevicePool(self.dev)  # tile buffers in exported arenas, mapped once per peer
        self.devs = [self.dev]
        self.skeleton = skeleton
        self.decomp = decomp
        self.owner_map = owner_map
        self.store = None
        self.manager = None
        self.executor = None
        self.transport = None
        self.shapes: dict = {}
        self.dtypes: dict = {}
        self._next = 0
        self._stage = None
        from .wire import DagCache

        self._decoded = DagCache()
        self.counters = None
        self._open_counters()
        if decomp is not None:
            self._build(None)

    def _open_counters(self) -> None:
        name = f"/dev/shm/est-{uuid.uuid4().hex}" if self.rank == 0 else None
        if self.rank == 0:
            self.counters = SharedCounters(name, self.world, create=True)
        name = self.group.allgather(name)[0]
        if self.rank != 0:
            self.counters = SharedCounters(name, self.world, create=False)
        self.group.barrier()
        if self.rank == 0:
            try:
                os.unlink(name)  # mappings stay valid; nothing is left behind
            except OSError:
                pass

    # -- plumbing ----------------------------------------------------------------
    def barrier(self) -> None:
        self.group.barrier()

    def _all_gather(self, obj) -> list:
        return self.group.allgather(obj)

    def exchange_buffers(self) -> None:
        self.sync()
        tables = self._all_gather(self.transport.buffer_table())
        self.transport.open_peer_buffers(tables)
        self.transport.map_neighbours()
        self.barrier()

    @property
    def executors(self) -> list:
        return [self.executor]

    @property
    def managers(self) -> list:
        return [self.manager]

    # -- job API -------------------------------------------------------------
    def _build(self, shape) -> None:
        if self.decomp is None:
            self.decomp = decompose(shape, self.world, self.odf)
        owners = self.owner_map or self.decomp.owner_map(self.world)
        self.owner_map = owners
        owned = [c for c, o in owners.items() if o == self.rank]
        self.store = GpuTileStore(self.dev, self.decomp, owned)
        self.transport = IpcPeerTransport(self)
        ev = self._all_gather(self.transport.event_handles())
        self.transport.open_peer_events(dict(enumerate(ev)))
        self.manager = GpuExchangeManager(self.store, self.rank, owners, self.transport)
        self.executor = GpuExecutor(self.store, self.manager, self.skeleton)
        self.executor.transport = self.transport

    def set_owner_map(self, owners: dict) -> None:
        """Swap the tile -> worker map after a migration (worker.py:374-377)."""
        self.owner_map = dict(owners)
        self.manager.owner_map = self.owner_map

    def create_array(self, shape, dtype: int = DTYPE_F64, array: int | None = None) -> int:
        shape = tuple(int(e) for e in shape)
        if self.store is None:
            self._build(shape)
        aid = self._next if array is None else int(array)
        self.store.create_array(ArrayInfo(aid, shape, dtype))
        self._next = max(self._next, aid + 1)
        self.shapes[aid] = shape
        self.dtypes[aid] = dtype
        self.exchange_buffers()
        return aid

    def run_bytes(self, blob: bytes) -> list:
        key, dag = self._decoded.get(blob)
        return self.run(dag, key)

    def run(self, dag, key: bytes | None = None) -> list:
        try:
            return [self.executor.execute_batch(dag, key)]
        except BaseException as exc:
            if self.transport is not None:
                self.transport.abort(exc)
            raise

    def sync(self) -> None:
        """Drain both streams. They may be parked on a peer's flag word, so
        this polls (instead of blocking in the driver) and raises
        TransportAborted if a peer flagged an abort or the wait outlives
        `timeout_s` - a dead peer must not hang the worker."""
        from .device import COMPUTE, COPY

        evs = [self.dev.event(), self.dev.event()]
        evs[0].record(COMPUTE)
        evs[1].record(COPY)
        t0 = time.perf_counter()
        nap = 2e-5
        try:
            while not all(e.done() for e in evs):
                if self.counters is not None and self.counters.arr[2].any():
                    raise TransportAborted("a peer aborted while this worker's streams were waiting on it")
                if time.perf_counter() - t0 > self.timeout_s:
                    raise TransportAborted(f"device work did not drain within {self.timeout_s:.0f} s")
                time.sleep(nap)
                nap = min(nap * 2, 1e-3)
        finally:
            for e in evs:
                e.close()
        self.dev.sync()

    def fetch_local(self, array: int, bounds=None) -> list:
        self.sync()
        shape = self.shapes[array]
        bounds = tuple(bounds) if bounds is not None else tuple((0, e) for e in shape)
        nbytes = int(np.prod([b - a for a, b in bounds])) * 8
        if self._stage is None or self._stage.nbytes < nbytes:
            if self._stage is not None:
                self._stage.close()
            self._stage = PinnedBuffer(max(nbytes, 1 << 20))
        if self.store is None or not self.store.tiles:
            return []
        return self.store.gather_slice_pieces(array, bounds, self._stage)

    def fetch(self, array: int, bounds=None) -> np.ndarray:
        """Collective: every rank returns the assembled slice."""
        shape = self.shapes[array]
        bounds = tuple(bounds) if bounds is not None else tuple((0, e) for e in shape)
        parts = self._all_gather(self.fetch_local(array, bounds))
        out = np.zeros([b - a for a, b in bounds], dtype=self.store.fetch_dtype(array))
        for part in parts:
            for piece, block in part:
                out[tuple(slice(a - lo, b - lo) for (a, b), (lo, _) in zip(piece, bounds))] = block
        return out

    def hash_local(self, array: int) -> int:
        """This rank's partial of the whole-array content hash (its tiles)."""
        self.sync()
        return self.store.hash(array) if self.store is not None and self.store.tiles else 0

    def hash(self, array: int) -> int:
        """Collective: the whole array's position-keyed content hash."""
        return sum(self._all_gather(self.hash_local(array))) % (1 << 64)

    def rounds_by_array(self) -> dict:
        mine = self.manager.snapshot_stats()["rounds"] if self.store.tiles else None
        allr = [r for r in self._all_gather(mine) if r is not None]
        for r in allr[1:]:
            assert r == allr[0], "ranks disagree on round counts"
        return allr[0] if allr else {}

    def close(self) -> None:
        try:
            self.dev.sync()
            self.barrier()
        except Exception:
            pass
        if self.executor is not None:
            self.executor.drop_replays()  # captured graphs (one-worker jobs) and chain twins
        if self.transport is not None:
            self.transport.close()
        try:
            self.barrier()
        except Exception:
            pass
        if self.store is not None:
            self.store.release()
        if getattr(self.dev, "pool", None) is not None:
            self.dev.pool.release()
            self.dev.pool = None
        if self._stage is not None:
            self._stage.close()
        if self.counters is not None:
            self.counters.close()
        self.dev.close()


def _spawn_entry(rank, world, port, fn, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist

    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        res = fn(rank, world, *args)
        q.put((rank, "ok", res))
    except BaseException as exc:  # report to the parent
        import traceback

        q.put((rank, "err", traceback.format_exc()))
    finally:
        try:
            dist.destroy_process_group()
        except Exception:
            pass


def spawn_local_job(world: int, fn, *args, timeout: float = 600.0) -> list:
    """Run fn(rank, world, *args) in `world` spawned processes; return per-rank results."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_spawn_entry, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    results: dict = {}
    errors = []
    deadline = time.time() + timeout
    while len(results) + len(errors) < world and time.time() < deadline:
        try:
            rank, status, payload = q.get(timeout=1.0)
        except Exception:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
            continue
        (results.__setitem__(rank, payload) if status == "ok" else errors.append(payload))
    for p in procs:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    if errors:
        raise RuntimeError("worker failed:\n" + errors[0])
    if len(results) < world:
        raise RuntimeError(f"only {len(results)}/{world} workers finished")
    return [results[r] for r in range(world)]
