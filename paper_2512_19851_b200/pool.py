"""Per-worker device arenas for IPC-shared tile buffers.

A multi-process job shares every tile buffer with its halo neighbours and,
during a rescale, with the workers that take tiles over (CUDA IPC). Mapping a
peer allocation (cudaIpcOpenMemHandle) costs ~50-150 ms per GiB-sized buffer
and a fresh cudaMalloc per moved or regrown tile adds more, so a worker's tile
buffers are carved out of a few large exported arenas instead: peers map each
arena once and address buffers by offset (the reference moves tiles as
TILE_DATA frames over TCP, worker.py:341-388; here they move device to device
and the mappings are reused across migrations and ghost regrowth).

First-fit with coalescing free lists; sub-allocations are 4 KiB aligned and
zero-filled like est_alloc's; freeing synchronises the device first (as
est_free does) so a range is never reused under in-flight work.
"""

from __future__ import annotations

import itertools
import os

ARENA_MIN = int(os.environ.get("EST_POOL_ARENA_BYTES", 256 << 20))
ALIGN = 4096
GROW = int(os.environ.get("EST_POOL_GROW", 4))


class _Arena:
    serials = itertools.count(1)

    def __init__(self, dev, size: int):
        self.base = dev.alloc(size)
        self.size = size
        self.serial = next(_Arena.serials)
        self.handle = None
        self.free = [(0, size)]

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
        merged = []
        for o, z in sorted(self.free + [(off, n)]):
            if merged and merged[-1][0] + merged[-1][1] == o:
                merged[-1] = (merged[-1][0], merged[-1][1] + z)
            else:
                merged.append((o, z))
        self.free = merged


class DevicePool:
    def __init__(self, dev, arena_min: int = ARENA_MIN, grow: int = GROW):
        self.dev = dev
        self.arena_min = arena_min
        self.grow = grow
        self.arenas: list = []
        self.live: dict = {}  # ptr -> (arena, offset, reserved bytes)

    def alloc(self, nbytes: int, isolated: bool = False) -> int:
        """`isolated`: an arena of its own, exactly this size - for a buffer
        that another worker is about to map (a tile an expand's load-balance
        stage will move): the peer then maps only that buffer, not the whole
        shared arena (cudaIpcOpenMemHandle costs ~50-65 ms per GiB)."""
        from .device import COMPUTE

        need = -(-max(1, int(nbytes)) // ALIGN) * ALIGN
        if isolated:
            # an idle arena of this size (an earlier isolated buffer that has
            # been freed) is reused; otherwise a new one
            arena = next((a for a in self.arenas if a.size == need and a.free == [(0, need)]), None)
            if arena is None:
                arena = _Arena(self.dev, need)
                self.arenas.append(arena)
            off = arena.take(need)
        else:
            for arena in self.arenas:
                off = arena.take(need)
                if off is not None:
                    break
            else:
                # room for three more buffers of this size: a shrink that doubles the
                # tiles per worker then needs no cudaMalloc and no new peer mapping
                arena = _Arena(self.dev, max(self.grow * need, self.arena_min))
                self.arenas.append(arena)
                off = arena.take(need)
        ptr = arena.base + off
        self.dev.memset_zero(ptr, need, COMPUTE)
        self.dev.stream_sync(COMPUTE)
        self.live[ptr] = (arena, off, need)
        return ptr

    def owns(self, ptr: int) -> bool:
        return ptr in self.live

    def free(self, ptr: int) -> None:
        arena, off, need = self.live.pop(ptr)
        self.dev.sync()
        arena.give(off, need)

    def locate(self, ptr: int) -> tuple:
        """-> (arena serial, arena IPC handle, offset) of a live sub-allocation."""
        arena, off, _need = self.live[ptr]
        if arena.handle is None:
            arena.handle = self.dev.ipc_handle(arena.base)
        return arena.serial, arena.handle, off

    def release(self) -> None:
        for arena in self.arenas:
            try:
                self.dev.free(arena.base)
            except Exception:
                pass
        self.arenas.clear()
        self.live.clear()


def device_alloc(dev, nbytes: int, isolated: bool = False) -> int:
    pool = getattr(dev, "pool", None)
    return pool.alloc(nbytes, isolated) if pool is not None else dev.alloc(nbytes)


def device_free(dev, ptr: int) -> None:
    pool = getattr(dev, "pool", None)
    if pool is not None and pool.owns(ptr):
        pool.free(ptr)
    else:
        dev.free(ptr)
