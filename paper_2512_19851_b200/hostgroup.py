"""Host-side collectives between GPU worker processes (plumbing only).

The data path never uses these: they carry IPC handle tables, barriers around
buffer reallocation / migration, and fetch gathers. Two implementations of one
tiny interface (`rank`, `world`, `allgather(obj)`, `barrier()`):

* `GlooGroup`  — torch.distributed (gloo), for torchrun-launched SPMD jobs
  (bench.py at N>1, tests);
* `PeerGroup`  — the worker's own peer sockets (the reference's peer channel,
  pkg/src/elastencil/worker.py:61-139, PROTOCOL.md "Halo messages"), used when
  the unchanged reference coordinator drives GPU worker processes and there is
  no torch rendezvous. Messages are frames of kind PEER_CTL (243, additive)
  carrying a JSON header {tag, src} and a pickled body.
"""

from __future__ import annotations

import json
import pickle
import socket
import struct
import threading
import time

from .wire import PEER_HELLO, recv_frame, send_frame, send_json

PEER_CTL = 243


class GlooGroup:
    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def allgather(self, obj) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def barrier(self) -> None:
        self.dist.barrier()


class PeerGroup:
    """Collectives over TCP between the ranks listed in `peers` {rank: "host:port"}.

    Every rank calls the collectives in the same order (they follow the
    coordinator's strictly ordered control stream), so a per-call sequence
    number is the matching tag.
    """

    def __init__(self, rank: int, peers: dict, listener: socket.socket, timeout: float = 600.0):
        self.rank = rank
        self.world = len(peers)
        self.peers = {int(k): v for k, v in peers.items()}
        self.timeout = timeout
        self.seq = 0
        self.cond = threading.Condition()
        self.inbox: dict = {}
        self.out: dict = {}
        self.listener = listener
        self.closed = False
        self._threads = []

    # inbound sockets are handed over by the worker's accept loop
    def adopt(self, sock: socket.socket) -> None:
        t = threading.Thread(target=self._reader, args=(sock,), daemon=True)
        t.start()
        self._threads.append(t)

    def _reader(self, sock) -> None:
        try:
            while True:
                kind, body = recv_frame(sock)
                if kind != PEER_CTL:
                    continue
                (n,) = struct.unpack_from("<I", body, 0)
                meta = json.loads(body[4:4 + n].decode())
                obj = pickle.loads(body[4 + n:])
                with self.cond:
                    self.inbox[(meta["tag"], meta["src"])] = obj
                    self.cond.notify_all()
        except (ConnectionError, OSError):
            return

    def _sock(self, dest: int) -> socket.socket:
        s = self.out.get(dest)
        if s is None:
            host, port = self.peers[dest].rsplit(":", 1)
            s = socket.create_connection((host, int(port)), timeout=30)
            s.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            s.settimeout(None)
            send_json(s, PEER_HELLO, {"id": self.rank, "ctl": True})
            self.out[dest] = s
        return s

    def allgather(self, obj) -> list:
        tag = self.seq
        self.seq += 1
        payload = pickle.dumps(obj)
        meta = json.dumps({"tag": tag, "src": self.rank}).encode()
        body = struct.pack("<I", len(meta)) + meta + payload
        for dest in sorted(self.peers):
            if dest != self.rank:
                send_frame(self._sock(dest), PEER_CTL, body)
        res = [None] * self.world
        res[self.rank] = obj
        deadline = time.time() + self.timeout
        with self.cond:
            for src in sorted(self.peers):
                if src == self.rank:
                    continue
                while (tag, src) not in self.inbox:
                    left = deadline - time.time()
                    if left <= 0:
                        raise TimeoutError(f"peer {src} missed collective {tag}")
                    self.cond.wait(min(left, 0.5))
                res[src] = self.inbox.pop((tag, src))
        return res

    def barrier(self) -> None:
        self.allgather(None)

    def close(self) -> None:
        for s in self.out.values():
            try:
                s.close()
            except OSError:
                pass
        self.out.clear()
