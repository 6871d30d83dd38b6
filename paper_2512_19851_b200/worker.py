"""GPU worker process: the drop-in for pkg/src/elastencil/worker.py.

Speaks the reference's internal control protocol unchanged (REGISTER 200,
INIT 201, W_CREATE 202, W_BATCH 203, W_FETCH 204, W_MIGRATE 206,
W_CHECKPOINT 207, W_RESTORE 208, W_EXIT 209; one REPLY_OK / REPLY_ERR per
request, worker.py:252-294), so the unchanged reference Coordinator
(coordinator.py) drives it. One additive kind, W_HASH 210 (this worker's
partial of a whole-array content hash, est_hash_box), lets a driver compare
16 GiB arrays across rescales without fetching them. Differences behind the seam:

* tiles live in HBM of GPU `gpu_for_slot(id)` and batches run as generated
  sm_100a kernels (executor.GpuExecutor); W_BATCH is answered as soon as the
  batch is ENQUEUED (the coordinator only reads batch replies at its barrier,
  coordinator.py:431-446), so host-side decode/analyze of batch k+1 overlaps
  device execution of batch k. Device faults surface at the next synchronising
  command (FETCH / MIGRATE / CHECKPOINT) as REPLY_ERR, which poisons the
  session exactly like a failed batch (PROTOCOL.md:51-54);
* halo exchange is the IPC peer transport (transport.py / ipc.py) instead of
  TCP strips; peer sockets only carry host collectives (hostgroup.PeerGroup);
* checkpoint / restore / migration move tile payloads device-to-device through
  the GPU memory daemon and peer IPC mappings (elastic.py).
"""

from __future__ import annotations

import json
import logging
import os
import socket
import sys
import threading
import time

from .daemon import DaemonClient, gpu_for_slot
from .errors import StencilError
from .tiles import Decomposition
from .wire import (
    INIT, PEER_HELLO, REGISTER, REPLY_ERR, REPLY_OK, W_BATCH, W_CHECKPOINT, W_CREATE, W_EXIT,
    W_FETCH, W_HASH, W_MIGRATE, W_RESTORE, parse_json, recv_frame, send_json)

log = logging.getLogger("elastencil.gpu_worker")


class GpuWorker:
    def __init__(self, worker_id: int, coordinator: str, scratch: str, device: int | None = None,
                 dev=None):
        self.id = worker_id
        self.scratch = scratch
        self.device = gpu_for_slot(worker_id) if device is None else device
        os.makedirs(os.path.join(scratch, "logs"), exist_ok=True)
        h = logging.FileHandler(os.path.join(scratch, "logs", f"gpu-worker-{worker_id}.log"))
        h.setFormatter(logging.Formatter("%(asctime)s %(message)s"))
        log.addHandler(h)
        log.setLevel(logging.INFO)
        self.listener = socket.socket()
        self.listener.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        self.listener.bind(("127.0.0.1", 0))
        self.listener.listen(64)
        self.address = "127.0.0.1:%d" % self.listener.getsockname()[1]
        host, port = coordinator.rsplit(":", 1)
        # CUDA context + libest BEFORE registering: a (re)spawned worker is
        # device-ready when the coordinator's restart stage sees it
        # (coordinator.py:562-579), so W_RESTORE is pure data movement
        # (a standby spare created its device before it was given an id: `dev`)
        self._dev = dev
        self._dev_err = None
        self._dev_thread = threading.Thread(target=self._make_device if dev is None else (lambda: None),
                                            daemon=True)
        self._dev_thread.start()
        self._dev_thread.join()
        self.coord = socket.create_connection((host, int(port)))
        self.coord.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
        send_json(self.coord, REGISTER, {"role": "worker", "id": self.id, "address": self.address})
        self.peer_dir: dict = {}
        self.worker_count = 0
        self.daemon_addr = None
        self.group = None
        self.job = None
        self._pending_socks: list = []
        self._lock = threading.Lock()
        self._running = True
        threading.Thread(target=self._accept_loop, daemon=True).start()

    # -- peer plumbing ---------------------------------------------------------
    def _accept_loop(self) -> None:
        while self._running:
            try:
                conn, _ = self.listener.accept()
                kind, _body = recv_frame(conn)
            except (OSError, ConnectionError):
                if not self._running:
                    return
                continue
            if kind != PEER_HELLO:
                conn.close()
                continue
            with self._lock:
                if self.group is not None:
                    self.group.adopt(conn)
                else:
                    self._pending_socks.append(conn)

    def _ensure_group(self):
        from .hostgroup import PeerGroup

        if self.group is None:
            self.group = PeerGroup(self.id, self.peer_dir, self.listener)
            with self._lock:
                for s in self._pending_socks:
                    self.group.adopt(s)
                self._pending_socks.clear()
        return self.group

    def _make_device(self) -> None:
        try:
            from .device import Device

            self._dev = Device(self.device)
        except BaseException as exc:  # surfaced by the first command that needs it
            self._dev_err = exc

    def _device(self):
        self._dev_thread.join()
        if self._dev_err is not None:
            raise self._dev_err
        dev, self._dev = self._dev, None  # handed to the job, which owns and closes it
        dev.sync()  # makes the device current on THIS thread too (ctx-less calls: IPC, pinned memory)
        return dev

    def _new_job(self, decomp, owners):
        from .ipc import IpcGpuJob

        dev = self._device() if self._dev is not None or self._dev_err else None
        return IpcGpuJob(self.id, len(self.peer_dir), device=self.device, group=self._ensure_group(),
                         decomp=decomp, owner_map=owners, dev=dev)

    # -- control loop (worker.py:252-294) ----------------------------------------
    def run(self) -> None:
        while self._running:
            try:
                kind, body = recv_frame(self.coord)
            except (ConnectionError, OSError):
                break
            meta, blob = parse_json(body)
            try:
                self._dispatch(kind, meta, blob)
            except StencilError as exc:
                send_json(self.coord, REPLY_ERR, {"code": exc.code, "message": str(exc)})
            except Exception as exc:  # report, never wedge the coordinator
                log.exception("worker %d failed handling %s", self.id, kind)
                send_json(self.coord, REPLY_ERR, {"code": 1, "message": repr(exc)})
        self._running = False
        self.shutdown()

    def _dispatch(self, kind: int, meta: dict, blob: bytes) -> None:
        if kind == INIT:
            self.peer_dir = {int(k): v for k, v in meta["peers"].items()}
            self.worker_count = meta["worker_count"]
            self.daemon_addr = meta.get("daemon")
            send_json(self.coord, REPLY_OK, {})
        elif kind == W_CREATE:
            self._handle_create(meta)
        elif kind == W_BATCH:
            self._handle_batch(meta, blob)
        elif kind == W_FETCH:
            self._handle_fetch(meta)
        elif kind == W_MIGRATE:
            self._handle_migrate(meta)
        elif kind == W_CHECKPOINT:
            self._handle_checkpoint(meta)
        elif kind == W_RESTORE:
            self._handle_restore(meta)
        elif kind == W_HASH:
            h = self.job.hash_local(meta["array"]) if self.job is not None else 0
            send_json(self.coord, REPLY_OK, {"hash": str(h)})
        elif kind == W_EXIT:
            self._running = False
        else:
            send_json(self.coord, REPLY_ERR, {"code": 1, "message": f"unknown control kind {kind}"})

    def _handle_create(self, meta: dict) -> None:
        if self.job is None:
            spec = meta["decomp"]
            decomp = Decomposition(tuple(spec["tile_grid"]), spec["odf"], spec["initial_workers"])
            self.job = self._new_job(decomp, decomp.owner_map(self.worker_count))
        self.job.create_array(tuple(meta["shape"]), int(meta.get("dtype", 0)), array=meta["array"])
        send_json(self.coord, REPLY_OK, {})

    def _handle_batch(self, meta: dict, blob: bytes) -> None:
        # DAG-bytes cache: a repeated batch skips decode / analysis / codegen
        # (and replays a CUDA graph on a single worker) - SURVEY.md §8f row 1
        stats = self.job.run_bytes(blob)[0] if self.job is not None else None
        rec = {
            "batch": meta["batch"],
            "nodes": stats.nodes_executed if stats else 0,
            "launches": stats.kernel_launches if stats else 0,
            "rounds": {str(k): v for k, v in (stats.rounds if stats else {}).items()},
            "net_messages": stats.net_messages if stats else 0,
            "wall_ms": stats.wall_ms if stats else 0.0,
            "compute_ms": round(stats.compute_ms, 3) if stats else 0.0,
            "wait_ms": round(stats.wait_ms, 3) if stats else 0.0,
            "prepare_ms": round(stats.prepare_ms, 3) if stats else 0.0,
            "gpu_launches": stats.gpu_launches if stats else 0,
        }
        log.info("batch %s", json.dumps(rec, separators=(",", ":")))
        send_json(self.coord, REPLY_OK, rec)

    def _handle_fetch(self, meta: dict) -> None:
        array = meta["array"]
        bounds = tuple(tuple(b) for b in meta["bounds"])
        pieces, payload = [], bytearray()
        if self.job is not None and self.job.store is not None and array in self.job.store.arrays:
            for piece, block in self.job.fetch_local(array, bounds):
                pieces.append([list(b) for b in piece])
                payload += block.tobytes()
        send_json(self.coord, REPLY_OK, {"pieces": pieces}, bytes(payload))

    def _handle_migrate(self, meta: dict) -> None:
        from .elastic import migrate_tiles

        plan = {tuple(int(x) for x in k.split(",")): (v[0], v[1]) for k, v in meta["plan"].items()}
        self.worker_count = meta["worker_count"]
        if self.job is not None:
            t0 = time.perf_counter()
            res = migrate_tiles(self.job, plan)
            log.info("migrate %s in %.1f ms", res, (time.perf_counter() - t0) * 1e3)
        send_json(self.coord, REPLY_OK, {})

    def _handle_checkpoint(self, meta: dict) -> None:
        from .elastic import checkpoint_tiles

        if self.job is None or self.job.store is None:
            send_json(self.coord, REPLY_OK, {"records": [], "arrays": {}, "has_tiles": False})
            return
        client = DaemonClient(self.daemon_addr)
        try:
            records, arrays_meta = checkpoint_tiles(self.job, client, self.id)
        finally:
            client.close()
        send_json(self.coord, REPLY_OK, {"records": records, "arrays": arrays_meta,
                                         "has_tiles": len(self.job.store.tiles) > 0})

    def _handle_restore(self, meta: dict) -> None:
        from .elastic import decomp_from_manifest, owner_map_from_manifest, read_manifest, restore_tiles

        t0 = time.perf_counter()
        manifest = read_manifest(meta["path"])
        self.worker_count = meta["worker_count"]
        decomp = decomp_from_manifest(manifest)
        if decomp is None:
            self.job = None
            send_json(self.coord, REPLY_OK, {})
            return
        self.job = self._new_job(decomp, owner_map_from_manifest(manifest))
        t1 = time.perf_counter()
        rst: dict = {}
        # an expand's load-balance stage follows and moves tiles to the new
        # count's owner map; those tiles are restored into arenas of their own
        depths = restore_tiles(self.job, manifest, rst, next_owners=decomp.owner_map(self.worker_count))
        t2 = time.perf_counter()
        self.job.executor.depths = depths
        for a, info in self.job.store.arrays.items():
            self.job.shapes[a] = info.shape
            self.job.dtypes[a] = info.dtype
            self.job._next = max(self.job._next, a + 1)
        self.job.exchange_buffers()
        log.info("restore: job %.1f ms, tiles %.1f ms %s, peer maps %.1f ms", (t1 - t0) * 1e3,
                 (t2 - t1) * 1e3, json.dumps(rst), (time.perf_counter() - t2) * 1e3)
        send_json(self.coord, REPLY_OK, {})

    def shutdown(self) -> None:
        try:
            if self.job is not None:
                self.job.dev.sync()
        except Exception:
            pass
        try:
            self.listener.close()
        except OSError:
            pass
        if self.group is not None:
            self.group.close()


def standby(device: int):
    """A warm spare (launcher.GpuLauncher): interpreter, package, libest and
    the CUDA context on `device` are brought up BEFORE the process has a
    worker id; it reports READY on stdout and blocks until the launcher's
    restart stage hands it an id on stdin ("ID <n>"). Context creation
    (0.6-0.9 s alone, several seconds when eight processes create theirs on
    one GPU at once; profiles/r1s2_worker_startup.txt) thus leaves the
    reference rescale's restart stage (coordinator.py:562-579)."""
    from . import elastic, executor, ipc  # noqa: F401  (warm imports)
    from .device import Device

    dev = Device(device)
    dev.sync()
    sys.stdout.write("READY\n")
    sys.stdout.flush()
    line = sys.stdin.readline().split()
    null = os.open(os.devnull, os.O_WRONLY)  # nobody drains the READY pipe from here on
    os.dup2(null, 1)
    os.close(null)
    if len(line) != 2 or line[0] != "ID":
        dev.close()
        return None, None
    return int(line[1]), dev


def worker_main(argv=None) -> int:
    """`python -m paper_2512_19851_b200.worker --id I --coordinator HOST:PORT --scratch DIR`
    (or `--standby --device G ...`: a warm spare that waits for its id)."""
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--id", type=int, default=None)
    ap.add_argument("--coordinator", required=True)
    ap.add_argument("--scratch", required=True)
    ap.add_argument("--device", type=int, default=None)
    ap.add_argument("--standby", action="store_true")
    args = ap.parse_args(argv)
    if os.environ.get("EST_WORKER_LOG"):  # stage splits of batches / migrate / restore on stderr
        logging.basicConfig(level=logging.INFO, stream=sys.stderr,
                            format="%(asctime)s %(name)s %(message)s")
    dev = None
    if args.standby:
        args.id, dev = standby(args.device or 0)
        if args.id is None:
            return 0
    elif args.id is None:
        ap.error("--id is required")
    GpuWorker(args.id, args.coordinator, args.scratch, args.device, dev=dev).run()
    return 0


if __name__ == "__main__":
    sys.exit(worker_main())
