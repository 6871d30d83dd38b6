"""TEST DOUBLE of device.Device for CPU-only tests of the multi-worker HOST logic
(prepare/push plan, round sequencing, IPC handshake, realloc barriers).

It performs no computation: allocations are fake addresses, launches and copy
descriptors are recorded. It lives under tests/ and is injected only by tests;
the product package has no CPU execution path.
"""

from __future__ import annotations

import itertools


class FakeEvent:
    def __init__(self, dev, name):
        self.dev, self.name = dev, name

    def record(self, stream=0):
        self.dev.log.append(("record", self.name))

    def wait(self, stream=0):
        self.dev.log.append(("wait", self.name))

    def sync(self):
        pass

    def done(self):
        return True

    def elapsed_ms(self, end):
        return 0.0

    def ipc_handle(self):
        return self.name.encode().ljust(64, b"\0")

    def close(self):
        pass


class FakeKernel:
    def __init__(self, name, block, smem):
        self.fn, self.name, self.block, self.smem = 1, name, tuple(block), smem


class FakeDevice:
    _ids = itertools.count(1)

    def __init__(self, index=0, tag="w"):
        self.index = index
        self.tag = tag
        self.launches = 0
        self.sm_count = 148
        self.log: list = []
        self.params: list = []
        self.copies: list = []
        self._next = 1 << 40
        self.allocated: dict = {}
        self.opened: list = []
        self.lane_copies: dict = {}

    def alloc(self, n):
        p = self._next
        self._next += ((n + 4095) // 4096 + 1) * 4096
        self.allocated[p] = n
        return p

    def free(self, p):
        self.allocated.pop(p)

    def memset_zero(self, *a, **k):
        pass

    def copy_box(self, box, elem, stream=0):
        self.copies.append(("box", box.src, box.dst, box.nx, box.ny, box.nz))

    def copy_boxes(self, boxes, elem, stream=0):
        self.launches += 1
        self.lane_copies[stream] = self.lane_copies.get(stream, 0) + 1
        for b in boxes:
            self.copies.append(("strip", b.src, b.dst, b.nx, b.ny, b.nz))

    def sync(self):
        pass

    def stream_sync(self, s):
        pass

    def flag_write(self, addr, value, stream=0):
        self.log.append(("flag_write", addr, value, stream))

    def flag_wait(self, addr, value, stream=0):
        self.log.append(("flag_wait", addr, value, stream))

    def event(self, interprocess=False):
        return FakeEvent(self, f"{self.tag}-ev{next(self._ids)}")

    def open_event(self, handle):
        return FakeEvent(self, handle.rstrip(b"\0").decode())

    def kernel(self, src, name, block, smem=0):
        return FakeKernel(name, block, smem)

    def occupancy(self, k):
        return 8

    def launch(self, k, grid, params, stream=0, pdl=True, cooperative=False):
        self.launches += 1
        self.log.append(("launch", grid[0], getattr(k, "name", "")))
        self.params.append(params)

    def tmap_3d(self, base, elem, dims, strides, box, l2_promotion=3):
        return base.to_bytes(8, "little").ljust(128, b"\0")

    def ipc_handle(self, ptr):
        return ptr.to_bytes(8, "little") + self.tag.encode().ljust(56, b"\0")

    def ipc_open(self, h):
        addr = int.from_bytes(h[:8], "little") | (1 << 60)
        self.opened.append(addr)
        return addr

    def ipc_close(self, p):
        self.opened.remove(p)

    def close(self):
        pass


class FakeGraph:
    def __init__(self, dev):
        self.dev = dev
        self.kernels = 0
        self.launched = 0

    def launch(self, stream=0):
        self.launched += 1
        self.dev.launches += self.kernels
        self.dev.log.append(("graph_launch", self.kernels, ""))

    def close(self):
        pass


def _graph_begin(self, stream=0):
    self.capturing = True


def _graph_end(self, stream=0):
    self.capturing = False
    return FakeGraph(self)


FakeDevice.graph_begin = _graph_begin
FakeDevice.graph_end = _graph_end
