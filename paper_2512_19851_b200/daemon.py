"""GPU memory daemon: keeps tile payloads in HBM across worker restarts.

The reference daemon (pkg/src/elastencil/daemon.py:29-143) is a TCP store of
host blobs that workers push to before a restart and pull from after. The paper
keeps the data on the GPU (a CUDA context cannot outlive its
process, so a long-lived per-GPU daemon owns the memory). This daemon:

* speaks the reference daemon protocol unchanged (STORE 250 / RETRIEVE 251 /
  FREE 252 / PING 253 / STATS 254, replies D_OK 255 / D_ERR 256), so host
  blobs still work;
* adds device allocations (additive kinds): DEV_ALLOC 257 {nbytes, meta} ->
  u64 id + 64-byte CUDA IPC handle of the ARENA holding it + u64 offset + u64
  arena serial; DEV_OPEN 258 id -> the same + meta; DEV_FREE 259 id. A worker
  checkpoints by copying its tile interiors device-to-device into the
  IPC-mapped arena (no host round trip); the restarted worker maps the arena
  once and copies back, then frees. Allocations are carved out of a few large
  arenas (first fit, coalescing free list) that live as long as the daemon,
  so a rescale pays one cudaMalloc / cudaIpcOpenMemHandle per arena instead
  of one per (tile, array).

One daemon per GPU slot, registered with the coordinator as role "daemon".
"""

from __future__ import annotations

import json
import os
import socket
import socketserver
import struct
import sys
import threading

from .errors import DaemonUnreachable, UnknownAllocation
from .wire import REGISTER, recv_frame, send_frame, send_json

D_STORE, D_RETRIEVE, D_FREE, D_PING, D_STATS, D_OK, D_ERR = 250, 251, 252, 253, 254, 255, 256
D_DEV_ALLOC, D_DEV_OPEN, D_DEV_FREE = 257, 258, 259
_U64 = struct.Struct("<Q")
ARENA_MIN = int(os.environ.get("EST_DAEMON_ARENA_BYTES", 2 << 30))
ARENA_ALIGN = 1 << 16


class _Arena:
    """One exported device allocation; sub-allocations by offset."""

    serials = iter(range(1, 1 << 62))

    def __init__(self, dev, size: int):
        self.ptr = dev.alloc(size)
        dev.sync()
        self.size = size
        self.handle = dev.ipc_handle(self.ptr)
        self.serial = next(_Arena.serials)
        self.free = [(0, size)]  # sorted (offset, size)

    def take(self, n: int):
        for k, (off, sz) in enumerate(self.free):
            if sz >= n:
                if sz == n:
                    del self.free[k]
                else:
                    self.free[k] = (off + n, sz - n)
                return off
        return None

    def give(self, off: int, n: int) -> None:
        self.free.append((off, n))
        self.free.sort()
        merged = []
        for o, z in self.free:
            if merged and merged[-1][0] + merged[-1][1] == o:
                merged[-1] = (merged[-1][0], merged[-1][1] + z)
            else:
                merged.append((o, z))
        self.free = merged


class GpuMemoryDaemon:
    def __init__(self, device: int = 0, host: str = "127.0.0.1", port: int = 0):
        from .device import Device

        self.dev = Device(device)
        self.device = device
        self._lock = threading.Lock()
        self._next = 1
        self._blobs: dict = {}
        self._dev: dict = {}  # id -> (arena, offset, reserved bytes, nbytes, meta)
        self._arenas: list = []
        daemon = self

        class Handler(socketserver.BaseRequestHandler):
            def handle(self):
                try:
                    while True:
                        kind, body = recv_frame(self.request)
                        daemon._dispatch(self.request, kind, body)
                except (ConnectionError, OSError):
                    return

        class Server(socketserver.ThreadingTCPServer):
            allow_reuse_address = True
            daemon_threads = True

        self._server = Server((host, port), Handler)
        self.address = "%s:%d" % self._server.server_address

    def _new_id(self) -> int:
        with self._lock:
            i = self._next
            self._next += 1
            return i

    def _dispatch(self, sock, kind: int, body: bytes) -> None:
        if kind == D_STORE:
            i = self._new_id()
            with self._lock:
                self._blobs[i] = body
            send_frame(sock, D_OK, _U64.pack(i))
        elif kind in (D_RETRIEVE, D_FREE):
            (i,) = _U64.unpack(body)
            with self._lock:
                blob = self._blobs.pop(i, None)
            if blob is None:
                send_frame(sock, D_ERR, b"unknown allocation")
            else:
                send_frame(sock, D_OK, blob if kind == D_RETRIEVE else b"")
        elif kind == D_PING:
            send_frame(sock, D_OK, json.dumps({"gpu": self.device}).encode())
        elif kind == D_STATS:
            with self._lock:
                n = len(self._blobs) + len(self._dev)
                total = sum(len(b) for b in self._blobs.values()) + sum(v[3] for v in self._dev.values())
            send_frame(sock, D_OK, struct.pack("<QQ", n, total))
        elif kind == D_DEV_ALLOC:
            req = json.loads(body.decode())
            nbytes = int(req["nbytes"])
            need = -(-max(1, nbytes) // ARENA_ALIGN) * ARENA_ALIGN
            try:
                with self._lock:
                    for arena in self._arenas:
                        off = arena.take(need)
                        if off is not None:
                            break
                    else:
                        arena = _Arena(self.dev, max(need, ARENA_MIN))
                        self._arenas.append(arena)
                        off = arena.take(need)
                    i = self._next
                    self._next += 1
                    self._dev[i] = (arena, off, need, nbytes, req.get("meta", {}))
            except Exception as exc:
                send_frame(sock, D_ERR, f"device allocation failed: {exc}".encode())
                return
            send_frame(sock, D_OK, _U64.pack(i) + arena.handle + _U64.pack(off) + _U64.pack(arena.serial))
        elif kind == D_DEV_OPEN:
            (i,) = _U64.unpack(body)
            with self._lock:
                ent = self._dev.get(i)
            if ent is None:
                send_frame(sock, D_ERR, b"unknown allocation")
            else:
                arena, off = ent[0], ent[1]
                send_frame(sock, D_OK, arena.handle + _U64.pack(off) + _U64.pack(arena.serial)
                           + json.dumps(ent[4]).encode())
        elif kind == D_DEV_FREE:
            (i,) = _U64.unpack(body)
            with self._lock:
                ent = self._dev.pop(i, None)
                if ent is not None:
                    ent[0].give(ent[1], ent[2])
            if ent is None:
                send_frame(sock, D_ERR, b"unknown allocation")
                return
            send_frame(sock, D_OK, b"")
        else:
            send_frame(sock, D_ERR, b"bad request")

    def serve_forever(self) -> None:
        self._server.serve_forever(poll_interval=0.2)

    def serve_in_thread(self) -> threading.Thread:
        t = threading.Thread(target=self.serve_forever, daemon=True)
        t.start()
        return t

    def shutdown(self) -> None:
        self._server.shutdown()
        self._server.server_close()
        with self._lock:
            for arena in self._arenas:
                try:
                    self.dev.free(arena.ptr)
                except Exception:
                    pass
            self._arenas.clear()
            self._dev.clear()
        self.dev.close()


class DaemonClient:
    """One connection to a memory daemon (reference API + device extensions)."""

    def __init__(self, address: str):
        self.address = address
        host, port = address.rsplit(":", 1)
        try:
            self._sock = socket.create_connection((host, int(port)), timeout=30)
            self._sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            self._sock.settimeout(600)
        except OSError as exc:
            raise DaemonUnreachable(f"cannot reach daemon at {address}: {exc}")

    def _call(self, kind: int, body: bytes) -> bytes:
        try:
            send_frame(self._sock, kind, body)
            rk, reply = recv_frame(self._sock)
        except (OSError, ConnectionError) as exc:
            raise DaemonUnreachable(f"daemon {self.address} failed: {exc}")
        if rk == D_ERR:
            raise UnknownAllocation(reply.decode(errors="replace"))
        return reply

    def store(self, payload: bytes) -> int:
        return _U64.unpack(self._call(D_STORE, payload))[0]

    def retrieve_and_free(self, alloc_id: int) -> bytes:
        return self._call(D_RETRIEVE, _U64.pack(alloc_id))

    def free(self, alloc_id: int) -> None:
        self._call(D_FREE, _U64.pack(alloc_id))

    def ping(self) -> dict:
        body = self._call(D_PING, b"")
        try:
            return json.loads(body.decode()) if body else {}
        except ValueError:
            return {}

    def stats(self) -> tuple:
        return struct.unpack("<QQ", self._call(D_STATS, b""))

    def dev_alloc(self, nbytes: int, meta: dict) -> tuple:
        """-> (allocation id, arena IPC handle, offset in the arena, arena serial)."""
        reply = self._call(D_DEV_ALLOC, json.dumps({"nbytes": int(nbytes), "meta": meta}).encode())
        return (_U64.unpack_from(reply, 0)[0], reply[8:72], _U64.unpack_from(reply, 72)[0],
                _U64.unpack_from(reply, 80)[0])

    def dev_open(self, alloc_id: int) -> tuple:
        """-> (arena IPC handle, offset, arena serial, meta)."""
        reply = self._call(D_DEV_OPEN, _U64.pack(alloc_id))
        return (reply[:64], _U64.unpack_from(reply, 64)[0], _U64.unpack_from(reply, 72)[0],
                json.loads(reply[80:].decode()))

    def dev_free(self, alloc_id: int) -> None:
        self._call(D_DEV_FREE, _U64.pack(alloc_id))

    def close(self) -> None:
        self._sock.close()


def daemon_main(argv=None) -> int:
    """`python -m paper_2512_19851_b200.daemon --id I --coordinator HOST:PORT [--device D]`"""
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--id", type=int, required=True)
    ap.add_argument("--coordinator", default=None)
    ap.add_argument("--device", type=int, default=None)
    args = ap.parse_args(argv)
    device = args.device if args.device is not None else gpu_for_slot(args.id)
    d = GpuMemoryDaemon(device)
    reg = None
    if args.coordinator:
        host, port = args.coordinator.rsplit(":", 1)
        reg = socket.create_connection((host, int(port)), timeout=30)
        send_json(reg, REGISTER, {"role": "daemon", "id": args.id, "address": d.address})
    print(f"DAEMON {d.address}", flush=True)
    try:
        d.serve_forever()
    except KeyboardInterrupt:
        pass
    finally:
        if reg is not None:
            reg.close()
    return 0


def gpu_for_slot(slot: int) -> int:
    """Worker / daemon slot i lives on GPU i mod the visible GPU count."""
    n = int(os.environ.get("EST_GPUS", "0"))
    if n <= 0:
        from .device import device_count

        n = max(1, device_count())
    return slot % n


if __name__ == "__main__":
    sys.exit(daemon_main())
