"""Build recipe: libest.so (nvcc, sm_100a), the oracle's C evaluator, and an
offline NVRTC prebuild of the kernels the bench / smoke / tests instantiate
(so a fresh GPU box loads cubins from the in-tree cache instead of compiling).
Runs without a GPU."""

from __future__ import annotations

import ctypes as C
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
HOST_CC = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def build_libest(verbose: bool = False) -> str:
    src = os.path.join(HERE, "csrc", "est.cu")
    out = os.path.join(HERE, "libest.so")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
           "-ccbin", HOST_CC, "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-o", out, src, "-lnvrtc",
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return out


def build_oracle() -> str:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    return os.path.join(ROOT, "oracle", "liboracle.so")


def precompile_sources(sources) -> tuple:
    """NVRTC-compile kernel sources into the in-tree cache (no GPU needed)."""
    from . import _lib
    from .device import DEFAULT_CACHE, NVRTC_OPTS

    lib = _lib.load()
    opts = (C.c_char_p * len(NVRTC_OPTS))(*[o.encode() for o in NVRTC_OPTS])
    new = cached = 0
    for src in sources:
        was = C.c_int(0)
        _lib.check(lib.est_module_precompile(src.encode(), opts, len(NVRTC_OPTS),
                                             DEFAULT_CACHE.encode(), C.byref(was)))
        cached += was.value
        new += 1 - was.value
    return new, cached


def standard_sources() -> list:
    """Kernel sources for the bench workloads, smoke and the parity suites."""
    from .analysis import compile_plan
    from .codegen import kernel_source_for
    from .ir import fuse
    from .programs import (DagProgram, cavity_program, heat3d_program, laplace_program,
                           wave2d_program)
    from .wire import DTYPE_F32

    progs = []
    p = DagProgram(); laplace_program(p, 64, 2); progs.append(p)
    p = DagProgram(); heat3d_program(p, 16, 2, seed_fills=2); progs.append(p)
    p = DagProgram(); wave2d_program(p, 64, 2, dtype=DTYPE_F32); progs.append(p)
    p = DagProgram(); cavity_program(p, 16, 1, pressure_iters=1); progs.append(p)
    srcs = set()
    for p in progs:
        for dag in (p.dag, fuse(p.dag)):
            for node in dag.nodes:
                out = node.statements[0].output
                rank, dt = len(p.shapes[out]), p.dtypes.get(out, 0)
                plan = compile_plan(node, dag.ast_table)
                for skel in ("auto", "point"):
                    srcs.add(kernel_source_for(plan, rank, dt, skel)[0])
                if rank == 2:
                    srcs.add(kernel_source_for(plan, rank, dt, "auto", small=True)[0])
                if rank in (2, 3) and len(plan.statements) == 1:
                    from . import resident
                    from .codegen import stmt_sig as _ss
                    rs = _ss(plan.statements[0], rank)
                    if resident.smem_eligible(rs, dt, rank):  # C1: 1022^2 outputs on 148 SMs
                        g = resident.smem_geometry(1022, 1022, resident.slot_radius(rs)[0], dt, 148)
                        if g is not None:
                            srcs.add(resident.smem_source(rs, dt, g)[0])
                if rank == 3 and len(plan.statements) == 1:
                    from . import temporal
                    from .codegen import stmt_sig
                    sig = stmt_sig(plan.statements[0], 3)
                    if temporal.eligible(sig, dt):
                        from .tiles import TileBuffer
                        for n in (1024, 512):  # the C4 / C2 bench layouts (depth 1)
                            xoff, py, pz = TileBuffer.pitches((n, n, n), (1, 1, 1), dt)
                            srcs.add(temporal.source(sig, dt, py=py, pz=pz, xoff=xoff)[0])
                if rank == 2 and len(plan.statements) == 1:
                    from . import temporal2d
                    from .codegen import stmt_sig
                    from .tiles import TileBuffer
                    sig = stmt_sig(plan.statements[0], 2)
                    if temporal2d.eligible(sig, dt):
                        for n, d in ((16384, 2), (16384, 1)):  # the C3 wave / paper-shape Laplace layouts
                            xoff, py, _pz = TileBuffer.pitches((n, n), (d, d), dt)
                            srcs.add(temporal2d.source(sig, dt, py=py, xoff=xoff)[0])
    return sorted(srcs)


def install_reference(src: str = "/root/reference/pkg") -> str | None:
    """Best effort: the unmodified reference into baseline/_ref (git-ignored;
    used by the integration tests and the C5 rescale bench). Offline pip from
    a copy, since /root/reference is read-only."""
    import shutil
    import tempfile

    dst = os.path.join(ROOT, "baseline", "_ref")
    tests = os.path.join(dst, "ref_tests")
    if os.path.isdir(os.path.join(src, "tests")) and not os.path.isdir(tests) and os.path.isdir(dst):
        # the reference's own runtime / daemon / acceptance suites, run against
        # the GPU workers by tests/test_gpu_reference_suites.py (git-ignored like
        # the install itself; travels to the GPU box with baseline/_ref)
        shutil.copytree(os.path.join(src, "tests"), tests)
    if os.path.isdir(os.path.join(dst, "elastencil")) or not os.path.isdir(src):
        return dst if os.path.isdir(dst) else None
    tmp = tempfile.mkdtemp(prefix="refpkg-")
    try:
        shutil.copytree(src, os.path.join(tmp, "pkg"))
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                        "--no-deps", "--target", dst, os.path.join(tmp, "pkg")],
                       check=True, capture_output=True)
        shutil.copytree(os.path.join(src, "tests"), tests)
        return dst
    except (OSError, subprocess.CalledProcessError) as exc:
        print(f"[build] reference install skipped: {exc}", file=sys.stderr)
        return None
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def build_all(prebuild: bool = True) -> None:
    build_libest()
    build_oracle()
    install_reference()
    if prebuild:
        new, cached = precompile_sources(standard_sources())
        print(f"[build] kernel cache: {new} compiled, {cached} already cached", file=sys.stderr)


if __name__ == "__main__":
    build_all()
