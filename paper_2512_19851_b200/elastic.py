"""Elastic N -> M rescale data path on GPUs (no host round trip).

Reference stages (coordinator.py:501-607, worker.py:341-422, elastic.py:46-169):
shrink = load-balance (migrate) -> checkpoint -> restart -> restore; expand =
checkpoint -> restart -> restore at the old owners -> migrate. The four stage
timings and the manifest JSON are unchanged; the bytes move differently:

* migrate (`migrate_tiles`): the NEW owner pulls each departing tile's interior
  straight out of the old owner's IPC-mapped HBM buffer (NVLink P2P across
  GPUs) instead of TILE_DATA frames over TCP (worker.py:362-369). Epoch rule as
  the reference: every local generation is bumped and ghost = local - 1
  (worker.py:384-387), so ghosts are re-exchanged under fresh round keys.
* checkpoint (`checkpoint_tiles`): per (tile, array) one device allocation in
  the GPU memory daemon (daemon.py DEV_ALLOC); the interior is copied D2D into
  the IPC-mapped allocation; the blob header (grid.py:236 layout, PROTOCOL.md
  "Checkpoint payload blob") travels as allocation metadata, `nbytes` keeps the
  reference's header+payload size. Ghost frames are not checkpointed.
* restore (`restore_tiles`): the restarted worker maps each allocation it owns
  per the manifest, copies D2D into fresh tile buffers, frees it, and bumps the
  local epochs (elastic.py:154-157).
"""

from __future__ import annotations

import json

import numpy as np

from ._lib import EstBox
from .daemon import DaemonClient
from .device import COMPUTE
from .tiles import (
    ArrayInfo,
    Decomposition,
    GpuTile,
    TileBuffer,
    blob_header,
    parse_blob_header,
)

MANIFEST_VERSION = 1


def _interior_box(buf, dst: int, to_dev_contig: bool) -> EstBox:
    n = buf.ext
    if to_dev_contig:
        return EstBox(buf.interior_addr((0,) * buf.rank), dst, buf.py, buf.pz, n[2], n[1] * n[2],
                      n[2], n[1], n[0])
    return EstBox(dst, buf.interior_addr((0,) * buf.rank), n[2], n[1] * n[2], buf.py, buf.pz,
                  n[2], n[1], n[0])


# --------------------------------------------------------------------------
# load balance (W_MIGRATE)

def migrate_tiles(job, plan: dict) -> dict:
    """plan {coords: (old_owner, new_owner)}; collective over every live worker.

    Returns stats {tiles_in, tiles_out, bytes_in}.
    """
    import time

    t0 = time.perf_counter()
    store, dev = job.store, job.dev
    job.sync()  # guarded: the streams may wait on peers' round flags
    # temporal-chain twins belong to the current tile set: every worker drops
    # them, the next chain batch re-creates them inside its realloc window
    for ex in job.executors:
        ex.release_scratch()
    # every worker learns the uniform local epochs (a tile-less worker has none)
    epochs = {a: store.local_epoch(a) for a in store.arrays} if store.tiles else None
    known = [e for e in job._all_gather(epochs) if e is not None]
    epochs = known[0] if known else {}
    job.barrier()
    t_agree = time.perf_counter()
    t_alloc = 0.0
    incoming = sorted(c for c, (old, new) in plan.items() if new == job.rank and old != job.rank)
    outgoing = sorted(c for c, (old, new) in plan.items() if old == job.rank and new != job.rank)
    depths = job.executor.depths
    nbytes = 0
    for coords in incoming:
        old = plan[coords][0]
        tile = store.tiles.setdefault(coords, GpuTile(coords))
        for a in sorted(store.arrays):
            info = store.arrays[a]
            ext = store.decomp.tile_extents(info.shape)
            depth = depths.get(a, (0,) * info.rank)
            frame = tuple(max(x, y) for x, y in zip(depth, store.phys_depth.get(a, depth)))
            ta = time.perf_counter()
            buf = TileBuffer(dev, ext, frame, info.dtype)
            t_alloc += time.perf_counter() - ta
            src_layout, src_addr = job.transport.peer_buffer(old, coords, a)
            # src_layout describes the peer buffer; its ptr is the mapped address
            src = src_layout.interior_addr((0,) * info.rank)
            n = buf.ext
            dev.copy_box(EstBox(src, buf.interior_addr((0,) * info.rank), src_layout.py,
                                src_layout.pz, buf.py, buf.pz, n[2], n[1], n[0]), buf.elem, COMPUTE)
            nbytes += int(np.prod(n)) * buf.elem
            tile.buffers[a] = buf
            tile.depths[a] = tuple(depth)
            tile.local_epoch[a] = epochs.get(a, 0)
            tile.ghost_epoch[a] = epochs.get(a, 0)
    dev.sync()
    t1 = time.perf_counter()
    job.barrier()  # every pull has completed before anyone frees a departed tile
    for coords in outgoing:
        tile = store.tiles.pop(coords)
        for buf in tile.buffers.values():
            buf.free()
    store.version += 1  # buffers were added / dropped
    new_map = {c: new for c, (_old, new) in plan.items()}
    job.set_owner_map(new_map)
    for a in sorted(store.arrays):
        # every worker, tile-less or not, continues from the job-wide epoch
        store.set_epochs(a, epochs.get(a, 0), epochs.get(a, 0))
        store.bump_local_epoch(a)
        store.set_ghost_epoch(a, store.local_epoch(a) - 1)
    t2 = time.perf_counter()
    job.exchange_buffers()
    return {"tiles_in": len(incoming), "tiles_out": len(outgoing), "bytes_in": nbytes,
            "pull_ms": round((t1 - t0) * 1e3, 1), "barrier_free_ms": round((t2 - t1) * 1e3, 1),
            "agree_ms": round((t_agree - t0) * 1e3, 1), "alloc_ms": round(t_alloc * 1e3, 1),
            "peer_maps_ms": round((time.perf_counter() - t2) * 1e3, 1)}


# --------------------------------------------------------------------------
# checkpoint / restore (W_CHECKPOINT / W_RESTORE)

def checkpoint_tiles(job, client: DaemonClient, owner: int) -> tuple:
    """Copy every owned (tile, array) interior into daemon HBM; records + meta."""
    store, dev = job.store, job.dev
    job.sync()
    records = []
    if store is None:
        return records, {}
    # allocate every blob, one batch of D2D copies, ONE sync; each daemon
    # arena is mapped once
    arenas: dict = {}
    for coords in sorted(store.tiles):
        tile = store.tiles[coords]
        for a in sorted(store.arrays):
            buf = tile.buffers[a]
            ext = buf.ext[3 - buf.rank:]
            depth = tile.depths[a]
            header = blob_header(a, coords, ext, depth, tile.local_epoch[a])
            payload = int(np.prod(ext)) * buf.elem
            meta = {"header": header.hex(), "dtype": buf.dtype}
            alloc_id, handle, off, serial = client.dev_alloc(payload, meta)
            base = arenas.get(serial)
            if base is None:
                base = arenas[serial] = dev.ipc_open(handle)
            dev.copy_box(_interior_box(buf, base + off, True), buf.elem, COMPUTE)
            records.append({"array": a, "tile": list(coords), "owner": owner,
                            "daemon": client.address, "alloc_id": alloc_id,
                            "nbytes": len(header) + payload})
    dev.sync()
    for base in arenas.values():
        dev.ipc_close(base)
    arrays_meta = {}
    for a, info in store.arrays.items():
        depth = next((list(t.depths[a]) for t in store.tiles.values()), None)
        arrays_meta[str(a)] = {
            "shape": list(info.shape),
            "depth": depth or list(job.executor.depths.get(a, (0,) * info.rank)),
            "local_epoch": store.local_epoch(a),
            "ghost_epoch": store.ghost_epoch(a),
            "dtype": info.dtype,
        }
    return records, arrays_meta


def build_manifest(session_seq: int, worker_count: int, decomp, arrays_meta: dict,
                   records: list) -> dict:
    m = {"version": MANIFEST_VERSION, "session_seq": session_seq, "worker_count": worker_count,
         "decomp": None, "arrays": arrays_meta, "allocations": records}
    if decomp is not None:
        m["decomp"] = {"tile_grid": list(decomp.tile_grid), "odf": decomp.odf,
                       "initial_workers": decomp.initial_workers}
    return m


def read_manifest(path: str) -> dict:
    with open(path) as fh:
        m = json.load(fh)
    if m.get("version") != MANIFEST_VERSION:
        raise ValueError(f"unsupported manifest version {m.get('version')}")
    return m


def decomp_from_manifest(m: dict):
    spec = m.get("decomp")
    if spec is None:
        return None
    return Decomposition(tuple(spec["tile_grid"]), spec["odf"], spec["initial_workers"])


def owner_map_from_manifest(m: dict) -> dict:
    owners = {tuple(r["tile"]): r["owner"] for r in m["allocations"]}
    d = decomp_from_manifest(m)
    if d is not None and not owners:
        owners = d.owner_map(m["worker_count"])
    return owners


def restore_tiles(job, manifest: dict, stats: dict | None = None, next_owners: dict | None = None) -> dict:
    """Install this worker's tiles from the daemons; returns {array: depth}.
    `stats` (optional) receives the split: daemon requests, tile-buffer
    allocation, daemon-arena IPC mapping, copies + sync, frees (ms).
    `next_owners` (optional): the owner map the following load-balance stage
    moves to (an expand restores at the old owners, then migrates to
    decomp.owner_map(new count), coordinator.py:520-528, 599-607); tiles that
    will leave get arenas of their own so their new owner maps only them."""
    import time

    store, dev = job.store, job.dev
    st = {"daemon_ms": 0.0, "alloc_ms": 0.0, "map_ms": 0.0, "copy_ms": 0.0, "free_ms": 0.0, "bytes": 0}
    depths = {}
    for key, meta in manifest["arrays"].items():
        a = int(key)
        store.arrays[a] = ArrayInfo(a, tuple(meta["shape"]), int(meta.get("dtype", 0)))
        depths[a] = tuple(meta["depth"])
        # the job-wide epochs, so workers restored without tiles keep the round
        # sequence aligned (tiles, if any, carry the same values in their blobs)
        store.set_epochs(a, int(meta.get("local_epoch", 0)), int(meta.get("local_epoch", 0)))
    clients: dict = {}
    opened = []   # (client, alloc id): all copies in flight, ONE sync
    arenas: dict = {}  # (daemon, arena serial) -> mapped base, each mapped once
    try:
        for rec in manifest["allocations"]:
            if rec["owner"] != job.rank:
                continue
            t0 = time.perf_counter()
            cl = clients.get(rec["daemon"])
            if cl is None:
                cl = clients[rec["daemon"]] = DaemonClient(rec["daemon"])
            handle, off, serial, meta = cl.dev_open(rec["alloc_id"])
            st["daemon_ms"] += (time.perf_counter() - t0) * 1e3
            header = bytes.fromhex(meta["header"])
            a, coords, ext, depth, epoch, _hs = parse_blob_header(header)
            payload = int(np.prod(ext)) * (8 if int(meta.get("dtype", 0)) == 0 else 4)
            if len(header) + payload != rec["nbytes"]:
                raise ValueError(f"allocation {rec['alloc_id']} size mismatch")
            tile = store.tiles.setdefault(tuple(coords), GpuTile(tuple(coords)))
            t0 = time.perf_counter()
            leaving = next_owners is not None and next_owners.get(tuple(coords), job.rank) != job.rank
            buf = TileBuffer(dev, ext, depth, int(meta.get("dtype", 0)), isolated=leaving)
            t1 = time.perf_counter()
            base = arenas.get((rec["daemon"], serial))
            if base is None:
                base = arenas[(rec["daemon"], serial)] = dev.ipc_open(handle)
            t2 = time.perf_counter()
            st["alloc_ms"] += (t1 - t0) * 1e3
            st["map_ms"] += (t2 - t1) * 1e3
            st["bytes"] += payload
            opened.append((cl, rec["alloc_id"]))
            dev.copy_box(_interior_box(buf, base + off, False), buf.elem, COMPUTE)
            tile.buffers[a] = buf
            tile.depths[a] = tuple(depth)
            tile.local_epoch[a] = epoch
            tile.ghost_epoch[a] = epoch
        t0 = time.perf_counter()
        dev.sync()
        t1 = time.perf_counter()
        for base in arenas.values():
            dev.ipc_close(base)
        for cl, alloc_id in opened:
            cl.dev_free(alloc_id)
        st["copy_ms"] += (t1 - t0) * 1e3
        st["free_ms"] += (time.perf_counter() - t1) * 1e3
    finally:
        for cl in clients.values():
            cl.close()
    for a in sorted(store.arrays):
        store.bump_local_epoch(a)
    if stats is not None:
        stats.update({k: (round(v, 1) if isinstance(v, float) else v) for k, v in st.items()})
    return depths
