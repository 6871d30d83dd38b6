"""The C-ABI library loads without a GPU and exports every symbol est.h declares."""

import ctypes
import os
import re

from paper_2512_19851_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "est.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(est_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.est_abi_version() == _lib.ABI_VERSION


def test_no_gpu_reports_error_not_crash():
    lib = _lib.load()
    n = ctypes.c_int(-1)
    rc = lib.est_device_count(ctypes.byref(n))
    # no driver in the build container: a clean error code, zero devices
    assert rc in (0, 1) and n.value >= 0
