"""ctypes binding of libest.so (include/est.h).

There is deliberately no fallback: if the shared library is missing or cannot
be loaded this raises, and every GPU entry point of the package fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import from_code

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libest.so")
ABI_VERSION = 7

u64, i64, i32, u32 = C.c_uint64, C.c_int64, C.c_int, C.c_uint32
vp = C.c_void_p
P = C.POINTER


class EstBox(C.Structure):
    _fields_ = [("src", u64), ("dst", u64),
                ("src_py", i64), ("src_pz", i64), ("dst_py", i64), ("dst_pz", i64),
                ("nx", i64), ("ny", i64), ("nz", i64)]


_SIGS = {
    "est_last_error": (C.c_char_p, []),
    "est_abi_version": (i32, []),
    "est_device_count": (i32, [P(i32)]),
    "est_ctx_create": (i32, [i32, P(vp)]),
    "est_ctx_destroy": (i32, [vp]),
    "est_ctx_sync": (i32, [vp]),
    "est_stream_sync": (i32, [vp, i32]),
    "est_device_info": (i32, [vp, P(i32), P(u64), P(u64), P(i32), P(i32)]),
    "est_alloc": (i32, [vp, u64, P(u64)]),
    "est_free": (i32, [vp, u64]),
    "est_memset_zero": (i32, [vp, u64, u64, i32]),
    "est_host_alloc": (i32, [u64, P(u64)]),
    "est_host_free": (i32, [u64]),
    "est_copy_box": (i32, [vp, P(EstBox), i32, i32]),
    "est_copy_boxes": (i32, [vp, P(EstBox), i32, i32, i32]),
    "est_hash_box": (i32, [vp, P(EstBox), P(i64), P(i64), i32, P(u64)]),
    "est_module_compile": (i32, [vp, C.c_char_p, P(C.c_char_p), i32, C.c_char_p, P(vp), P(i32)]),
    "est_module_precompile": (i32, [C.c_char_p, P(C.c_char_p), i32, C.c_char_p, P(i32)]),
    "est_module_load_cubin": (i32, [vp, vp, P(vp)]),
    "est_module_kernel": (i32, [vp, C.c_char_p, P(u64)]),
    "est_module_destroy": (i32, [vp]),
    "est_kernel_set_smem": (i32, [u64, i32]),
    "est_kernel_occupancy": (i32, [u64, i32, i32, C.POINTER(C.c_int)]),
    "est_launch": (i32, [vp, u64, P(u32), P(u32), u32, vp, u32, i32]),
    "est_launch_ex": (i32, [vp, u64, P(u32), P(u32), u32, vp, u32, i32, i32]),
    "est_graph_begin": (i32, [vp, i32]),
    "est_graph_end": (i32, [vp, i32, P(vp)]),
    "est_graph_launch": (i32, [vp, vp, i32]),
    "est_graph_destroy": (i32, [vp]),
    "est_tmap_encode_3d": (i32, [u64, i32, P(u64), P(u64), P(u32), i32, vp]),
    "est_nvrtc_compile":(i32, [C.c_char_p, P(C.c_char_p), i32, C.c_char_p, P(vp), P(u64)]),
    "est_buffer_free": (None, [vp]),
    "est_event_create": (i32, [vp, i32, P(vp)]),
    "est_event_destroy": (i32, [vp]),
    "est_event_record": (i32, [vp, vp, i32]),
    "est_event_wait": (i32, [vp, vp, i32]),
    "est_event_sync": (i32, [vp]),
    "est_event_query": (i32, [vp]),
    "est_event_elapsed_ms": (i32, [vp, vp, P(C.c_float)]),
    "est_stream_join": (i32, [vp, i32, i32]),
    "est_flag_write": (i32, [vp, u64, C.c_uint32, i32]),
    "est_flag_wait": (i32, [vp, u64, C.c_uint32, i32]),
    "est_ipc_mem_handle": (i32, [u64, P(C.c_uint8)]),
    "est_ipc_mem_open": (i32, [vp, P(C.c_uint8), P(u64)]),
    "est_ipc_mem_close": (i32, [u64]),
    "est_ipc_event_handle": (i32, [vp, P(C.c_uint8)]),
    "est_ipc_event_open": (i32, [P(C.c_uint8), P(vp)]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load():
    """Load and type libest.so; raises OSError/RuntimeError, never falls back."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA backend is not built "
                "(run __graft_entry__.build()); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.est_abi_version() != ABI_VERSION:
            raise RuntimeError(f"libest.so ABI {lib.est_abi_version()} != {ABI_VERSION}; rebuild")
        _lib = lib
        return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().est_last_error()
        raise from_code(rc, msg.decode(errors="replace") if msg else f"libest error {rc}")
