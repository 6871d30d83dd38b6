"""One GPU as seen by a worker: a libest context (compute + copy streams),
device memory, box copies, events and the kernel module cache.

Replaces the numpy/ScratchPool execution state of the reference worker
(pkg/src/elastencil/executor.py:65-83, 179-191); see include/est.h.
"""

from __future__ import annotations

import ctypes as C
import os

from . import _lib
from ._lib import EstBox, check

COMPUTE, COPY = 0, 1

DEFAULT_CACHE = os.environ.get(
    "EST_KERNEL_CACHE", os.path.join(os.path.dirname(os.path.abspath(__file__)), "kernel_cache"))

NVRTC_OPTS = (
    "--fmad=false",       # no contraction: a*b+c stays two rounded ops (bit parity)
    "-prec-div=true",
    "-prec-sqrt=true",
    "-ftz=false",
    "--std=c++17",
    "-default-device",
    "-lineinfo",
)


def device_count() -> int:
    n = C.c_int(0)
    lib = _lib.load()
    if lib.est_device_count(C.byref(n)) != 0:
        return 0
    return n.value


class Event:
    def __init__(self, dev: "Device", interprocess: bool = False, handle: bytes | None = None):
        self.dev = dev
        self.ptr = C.c_void_p()
        lib = _lib.load()
        if handle is not None:
            buf = (C.c_uint8 * 64).from_buffer_copy(handle)
            check(lib.est_ipc_event_open(buf, C.byref(self.ptr)))
        else:
            check(lib.est_event_create(dev.ctx, int(interprocess), C.byref(self.ptr)))

    def record(self, stream: int = COMPUTE) -> None:
        check(_lib.load().est_event_record(self.dev.ctx, self.ptr, stream))

    def wait(self, stream: int = COMPUTE) -> None:
        check(_lib.load().est_event_wait(self.dev.ctx, self.ptr, stream))

    def sync(self) -> None:
        check(_lib.load().est_event_sync(self.ptr))

    def done(self) -> bool:
        rc = _lib.load().est_event_query(self.ptr)
        if rc == 600:
            return False
        check(rc)
        return True

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float(0)
        check(_lib.load().est_event_elapsed_ms(self.ptr, end.ptr, C.byref(ms)))
        return float(ms.value)

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        check(_lib.load().est_ipc_event_handle(self.ptr, buf))
        return bytes(buf)

    def close(self) -> None:
        if self.ptr:
            _lib.load().est_event_destroy(self.ptr)
            self.ptr = C.c_void_p()


class Graph:
    """An instantiated CUDA graph (one batch's launches), replayable."""

    def __init__(self, dev: "Device", ptr):
        self.dev, self.ptr = dev, ptr
        self.kernels = 0

    def launch(self, stream: int = COMPUTE) -> None:
        check(_lib.load().est_graph_launch(self.dev.ctx, self.ptr, stream))
        self.dev.launches += self.kernels

    def close(self) -> None:
        if self.ptr:
            _lib.load().est_graph_destroy(self.ptr)
            self.ptr = C.c_void_p()


# programmatic dependent launch for kernels that wait on their predecessor
# themselves (griddepcontrol.wait in the generated source)
PDL = os.environ.get("EST_PDL", "1") == "1"


class Kernel:
    __slots__ = ("fn", "name", "block", "smem", "pdl")

    def __init__(self, fn: int, name: str, block, smem: int, pdl: bool = False):
        self.fn, self.name, self.block, self.smem = fn, name, tuple(block), smem
        self.pdl = pdl


class Device:
    """A libest context bound to one CUDA device."""

    def __init__(self, index: int = 0, cache_dir: str | None = DEFAULT_CACHE):
        self.lib = _lib.load()
        self.index = index
        self.ctx = C.c_void_p()
        check(self.lib.est_ctx_create(index, C.byref(self.ctx)))
        self.cache_dir = cache_dir
        self._modules: dict = {}
        self._kernels: dict = {}
        self.launches = 0          # every kernel this process launched (gpu_launches)
        self.compiles = 0
        self.cache_hits = 0
        sm, tot, free, ma, mi = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_int(), C.c_int()
        check(self.lib.est_device_info(self.ctx, C.byref(sm), C.byref(tot), C.byref(free),
                                       C.byref(ma), C.byref(mi)))
        self.sm_count, self.total_mem, self.cc = sm.value, tot.value, (ma.value, mi.value)

    # -- memory ---------------------------------------------------------------
    def alloc(self, nbytes: int) -> int:
        p = C.c_uint64()
        check(self.lib.est_alloc(self.ctx, int(nbytes), C.byref(p)))
        return p.value

    def free(self, ptr: int) -> None:
        check(self.lib.est_free(self.ctx, int(ptr)))

    def memset_zero(self, ptr: int, nbytes: int, stream: int = COMPUTE) -> None:
        check(self.lib.est_memset_zero(self.ctx, int(ptr), int(nbytes), stream))

    def copy_box(self, box: EstBox, elem: int, stream: int = COMPUTE) -> None:
        check(self.lib.est_copy_box(self.ctx, C.byref(box), elem, stream))

    def copy_boxes(self, boxes, elem: int, stream: int = COMPUTE) -> None:
        if not boxes:
            return
        arr = (EstBox * len(boxes))(*boxes)
        check(self.lib.est_copy_boxes(self.ctx, arr, len(boxes), elem, stream))
        self.launches += (len(boxes) + 47) // 48

    def hash_box(self, box, origin, gdims, elem: int) -> int:
        """Position-keyed content hash of `box`'s source side (est_hash_box)."""
        out = C.c_uint64(0)
        check(self.lib.est_hash_box(self.ctx, C.byref(box), (C.c_int64 * 3)(*origin),
                                    (C.c_int64 * 3)(*gdims), elem, C.byref(out)))
        self.launches += 1
        return out.value

    # -- sync / events ------------------------------------------------------
    def sync(self) -> None:
        check(self.lib.est_ctx_sync(self.ctx))

    def stream_sync(self, stream: int) -> None:
        check(self.lib.est_stream_sync(self.ctx, stream))

    def join(self, waiter: int, signaller: int) -> None:
        check(self.lib.est_stream_join(self.ctx, waiter, signaller))

    def flag_write(self, addr: int, value: int, stream: int = COMPUTE) -> None:
        """After all prior work on `stream`: *(uint32*)addr = value (release)."""
        check(self.lib.est_flag_write(self.ctx, int(addr), int(value) & 0xFFFFFFFF, stream))

    def flag_wait(self, addr: int, value: int, stream: int = COMPUTE) -> None:
        """`stream` waits until *(uint32*)addr >= value (wrap-safe), no host wait."""
        check(self.lib.est_flag_wait(self.ctx, int(addr), int(value) & 0xFFFFFFFF, stream))

    def event(self, interprocess: bool = False) -> Event:
        return Event(self, interprocess)

    def open_event(self, handle: bytes) -> Event:
        """Open a peer process's interprocess event (IPC handle)."""
        return Event(self, handle=handle)

    # -- kernels ------------------------------------------------------------
    def kernel(self, source: str, name: str, block, smem: int = 0) -> Kernel:
        key = (source, name)
        k = self._kernels.get(key)
        if k is not None:
            return k
        mod = self._modules.get(source)
        if mod is None:
            mod = C.c_void_p()
            opts = (C.c_char_p * len(NVRTC_OPTS))(*[o.encode() for o in NVRTC_OPTS])
            hit = C.c_int(0)
            cache = self.cache_dir.encode() if self.cache_dir else None
            check(self.lib.est_module_compile(self.ctx, source.encode(), opts, len(NVRTC_OPTS),
                                              cache, C.byref(mod), C.byref(hit)))
            self.cache_hits += hit.value
            self.compiles += 1 - hit.value
            self._modules[source] = mod
        fn = C.c_uint64()
        check(self.lib.est_module_kernel(mod, name.encode(), C.byref(fn)))
        if smem > 48 * 1024:
            check(self.lib.est_kernel_set_smem(fn.value, smem))
        k = Kernel(fn.value, name, block, smem, pdl=PDL and "griddepcontrol.wait" in source)
        self._kernels[key] = k
        return k

    def occupancy(self, k: Kernel) -> int:
        """Co-resident CTAs per SM for k's block shape and shared memory."""
        n = C.c_int(0)
        check(self.lib.est_kernel_occupancy(k.fn, int(k.block[0] * k.block[1] * k.block[2]), k.smem,
                                            C.byref(n)))
        return n.value

    def launch(self, k: Kernel, grid, params: bytes, stream: int = COMPUTE, pdl: bool = True,
               cooperative: bool = False) -> None:
        """`pdl`: the caller allows programmatic dependent launch here (no
        cross-stream / cross-process event waits interleaved with the
        predecessor kernel). `cooperative`: grid-barrier kernels; the driver
        guarantees co-residency or fails the launch."""
        g = (C.c_uint32 * 3)(*grid)
        b = (C.c_uint32 * 3)(*k.block)
        flags = (1 if (pdl and k.pdl) else 0) | (2 if cooperative else 0)
        if flags:
            check(self.lib.est_launch_ex(self.ctx, k.fn, g, b, k.smem, params, len(params), stream, flags))
        else:
            check(self.lib.est_launch(self.ctx, k.fn, g, b, k.smem, params, len(params), stream))
        self.launches += 1

    # -- CUDA graphs ----------------------------------------------------------
    def graph_begin(self, stream: int = COMPUTE) -> None:
        check(self.lib.est_graph_begin(self.ctx, stream))

    def graph_end(self, stream: int = COMPUTE) -> "Graph":
        g = C.c_void_p()
        check(self.lib.est_graph_end(self.ctx, stream, C.byref(g)))
        return Graph(self, g)

    def tmap_3d(self, base: int, elem: int, dims, strides_bytes, box, l2_promotion: int = 3) -> bytes:
        """128-byte CUtensorMap for a rank-3 buffer (innermost dimension first)."""
        out = (C.c_uint8 * 128)()
        check(self.lib.est_tmap_encode_3d(int(base), elem, (C.c_uint64 * 3)(*dims),
                                          (C.c_uint64 * 2)(*strides_bytes),
                                          (C.c_uint32 * 3)(*box), int(l2_promotion), out))
        return bytes(out)

    # -- ipc ----------------------------------------------------------------
    def ipc_handle(self, ptr: int) -> bytes:
        buf = (C.c_uint8 * 64)()
        check(self.lib.est_ipc_mem_handle(int(ptr), buf))
        return bytes(buf)

    def ipc_open(self, handle: bytes) -> int:
        p = C.c_uint64()
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        check(self.lib.est_ipc_mem_open(self.ctx, buf, C.byref(p)))
        return p.value

    def ipc_close(self, ptr: int) -> None:
        check(self.lib.est_ipc_mem_close(int(ptr)))

    def close(self) -> None:
        if self.ctx:
            for mod in self._modules.values():
                self.lib.est_module_destroy(mod)
            self._modules.clear()
            self._kernels.clear()
            self.lib.est_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()


class PinnedBuffer:
    """Page-locked host staging (D2H fetch / checkpoint payloads)."""

    def __init__(self, nbytes: int):
        self.lib = _lib.load()
        p = C.c_uint64()
        check(self.lib.est_host_alloc(int(nbytes), C.byref(p)))
        self.ptr, self.nbytes = p.value, int(nbytes)

    def view(self, dtype, count: int):
        import numpy as np

        buf = (C.c_char * (count * np.dtype(dtype).itemsize)).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dtype, count=count)

    def close(self) -> None:
        if self.ptr:
            self.lib.est_host_free(self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
