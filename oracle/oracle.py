"""CPU oracle for the stencil backend — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline /
reference arm may import this module, and only as the checker or the timed CPU
baseline. The product package never imports it; the GPU path fails loudly when
its CUDA library is missing instead of falling back here.

Two independent routes, both restating the reference (pkg/src/elastencil/):

* `reference_execute[_dag]` — whole-array recursive numpy evaluation in program
  order (oracle.py:46-95). Constants are typed scalars of the array dtype so
  IEEE semantics (inf/nan propagation, correct rounding) hold; float32 arrays
  evaluate with numpy float32 constants (SURVEY.md §7 "Hard parts").
* `strict_execute_dag` — the C evaluator in `strict_eval.c` (compiled with
  `-ffp-contract=off`, OpenMP over rows) that interprets the postorder plan
  row by row exactly like executor.py:86-176 does per tile. Fast enough for the
  BASELINE sizes and used as the timed CPU baseline.

Parity is PINNED: `tests/golden/gen_golden.py` (run in the container that has
the reference mounted) stores the reference's own outputs, DAG bytes, round
counts and text dumps; `tests/test_oracle_pinned.py` checks both routes against
them. The float32 path has no reference counterpart (SPEC.md:104 is fp64-only),
so fp32 results are checked within the north star's 1e-5 relative tolerance.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2512_19851_b200.analysis import OP_CONST, OP_LOAD, compile_plan
from paper_2512_19851_b200.ir import Binary, Const, SlotRef, Unary
from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64

NP_DTYPE = {DTYPE_F64: np.float64, DTYPE_F32: np.float32}

_UNARY = {"neg": np.negative, "abs": np.abs, "sqrt": np.sqrt}
_BINARY = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide}


# --------------------------------------------------------------------------
# route 1: recursive numpy (oracle.py:46-95)

def _eval(expr, stmt, arrays, scalar):
    if isinstance(expr, Const):
        return scalar(expr.value)
    if isinstance(expr, SlotRef):
        return arrays[stmt.inputs[expr.slot]][tuple(slice(a, b) for a, b in expr.slice.bounds)]
    if isinstance(expr, Unary):
        return _UNARY[expr.op](_eval(expr.child, stmt, arrays, scalar))
    if isinstance(expr, Binary):
        lhs = _eval(expr.left, stmt, arrays, scalar)
        rhs = _eval(expr.right, stmt, arrays, scalar)
        return _BINARY[expr.op](lhs, rhs)
    raise TypeError(f"unknown expression {expr!r}")


def reference_execute(statements, ast_table, shapes, dtypes=None, arrays=None) -> dict:
    dtypes = dtypes or {}
    arrays = {} if arrays is None else arrays
    for aid, shape in shapes.items():
        arrays.setdefault(aid, np.zeros(shape, dtype=NP_DTYPE[dtypes.get(aid, DTYPE_F64)]))
    with np.errstate(all="ignore"):
        for st in statements:
            out = arrays[st.output]
            val = _eval(ast_table[st.ast_id].root, st, arrays, out.dtype.type)
            out[tuple(slice(a, b) for a, b in st.output_slice.bounds)] = val
    return arrays


def reference_execute_dag(dag, shapes, dtypes=None, arrays=None) -> dict:
    stmts = [s for n in dag.nodes for s in n.statements]
    return reference_execute(stmts, dag.ast_table, shapes, dtypes, arrays)


# --------------------------------------------------------------------------
# epoch / round simulation (oracle.py:141-189)

class EpochSimulator:
    def __init__(self):
        self.local: dict = {}
        self.ghost: dict = {}
        self.depth: dict = {}
        self.rounds: dict = {}

    def simulate_batch(self, dag, metas) -> None:
        need: dict = {}
        for m in metas:
            for a, off in m.array_max_offset.items():
                need[a] = off if a not in need else tuple(map(max, need[a], off))
        for a, off in sorted(need.items()):
            old = self.depth.get(a, (0,) * len(off))
            new = tuple(map(max, old, off))
            if new != old:
                self.local[a] = self.local.get(a, 0) + 1
            self.depth[a] = new
        for m in metas:
            for a in sorted(m.array_max_offset):
                if not m.needs_exchange(a):
                    continue
                loc = self.local.get(a, 0)
                if loc and self.ghost.get(a, 0) != loc:
                    self.rounds[a] = self.rounds.get(a, 0) + 1
                    self.ghost[a] = loc
            for a in m.written_arrays:
                self.local[a] = self.local.get(a, 0) + 1


def epoch_simulate(dag, metas) -> dict:
    sim = EpochSimulator()
    sim.simulate_batch(dag, metas)
    return sim.rounds


# --------------------------------------------------------------------------
# hand-written solvers (oracle.py:196-314 and the new 3-D / wave workloads)

def laplace_reference(n: int, iters: int) -> np.ndarray:
    a = np.zeros((n, n))
    b = np.zeros((n, n))
    for u in (a, b):
        u[0, :] = u[-1, :] = u[:, 0] = u[:, -1] = 1.0
    for _ in range(iters):
        b[1:-1, 1:-1] = 0.25 * (a[:-2, 1:-1] + a[2:, 1:-1] + a[1:-1, :-2] + a[1:-1, 2:])
        a, b = b, a
    return a


def heat3d_reference(n: int, iters: int) -> np.ndarray:
    """Face-Dirichlet 7-point Jacobi, same association order as heat3d_tree."""
    a = np.zeros((n, n, n))
    b = np.zeros((n, n, n))
    for u in (a, b):
        u[0], u[-1] = 1.0, 1.0
        u[:, 0], u[:, -1] = 1.0, 1.0
        u[:, :, 0], u[:, :, -1] = 1.0, 1.0
    m = slice(1, -1)
    for _ in range(iters):
        s = a[:-2, m, m] + a[2:, m, m]
        s = s + a[m, :-2, m]
        s = s + a[m, 2:, m]
        s = s + a[m, m, :-2]
        s = s + a[m, m, 2:]
        b[m, m, m] = (1.0 / 6.0) * s
        a, b = b, a
    return a


def cavity_reference(n: int, iters: int, pressure_iters: int = 10):
    from paper_2512_19851_b200.programs import cavity_constants

    c = cavity_constants(n)
    u, v, p, un, vn, pn, b = (np.zeros((n, n)) for _ in range(7))
    u[-1, :] = 1.0
    un[-1, :] = 1.0
    I = slice(1, -1)
    for _ in range(iters):
        un, u = u, un
        vn, v = v, vn
        dudx = (un[I, 2:] - un[I, :-2]) * c["inv2dx"]
        dvdy = (vn[2:, I] - vn[:-2, I]) * c["inv2dy"]
        dudy = (un[2:, I] - un[:-2, I]) * c["inv2dy"]
        dvdx = (vn[I, 2:] - vn[I, :-2]) * c["inv2dx"]
        b[I, I] = c["rho"] * (c["inv_dt"] * (dudx + dvdy) - dudx * dudx
                              - 2.0 * (dudy * dvdx) - dvdy * dvdy)
        for _ in range(pressure_iters):
            pn, p = p, pn
            p[I, I] = ((pn[I, 2:] + pn[I, :-2]) * c["dy2"]
                       + (pn[2:, I] + pn[:-2, I]) * c["dx2"]) * c["pois_den"] \
                - c["pois_b_coeff"] * b[I, I]
            p[:, -1:] = pn[:, -2:-1]
            p[0:1, :] = pn[1:2, :]
            p[:, 0:1] = pn[:, 1:2]
            p[-1:, :] = 0.0
        for a_, an, gname, gsl in ((u, un, "pgrad_x", 1), (v, vn, "pgrad_y", 0)):
            if gsl == 1:
                grad = c[gname] * (p[I, 2:] - p[I, :-2])
            else:
                grad = c[gname] * (p[2:, I] - p[:-2, I])
            a_[I, I] = (an[I, I]
                        - un[I, I] * c["dtdx"] * (an[I, I] - an[I, :-2])
                        - vn[I, I] * c["dtdy"] * (an[I, I] - an[:-2, I])
                        - grad
                        + c["visc_x"] * (an[I, 2:] - 2.0 * an[I, I] + an[I, :-2])
                        + c["visc_y"] * (an[2:, I] - 2.0 * an[I, I] + an[:-2, I]))
        u[0, :] = 0.0
        u[:, 0] = 0.0
        u[:, -1] = 0.0
        u[-1, :] = 1.0
        v[0, :] = 0.0
        v[-1, :] = 0.0
        v[:, 0] = 0.0
        v[:, -1] = 0.0
    return u, v, p


# --------------------------------------------------------------------------
# route 2: strict-order C evaluator (strict_eval.c)

_OPC = {("unary", "neg"): 2, ("unary", "abs"): 3, ("unary", "sqrt"): 4,
        ("binary", "add"): 5, ("binary", "sub"): 6, ("binary", "mul"): 7,
        ("binary", "div"): 8}
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.oracle_eval_statement.restype = ctypes.c_int
        _LIB = lib
    return _LIB


def _as3(shape):
    return (1,) * (3 - len(shape)) + tuple(shape)


def encode_plan(plan_stmt, rank: int):
    """Plan tuples -> flat arrays (op code, f64 constant, slot, 3-D offset)."""
    ops, consts, slots, offs = [], [], [], []
    for ins in plan_stmt.instructions:
        code, val, slot, off = 0, 0.0, 0, (0, 0, 0)
        if ins[0] == OP_CONST:
            val = ins[1]
        elif ins[0] == OP_LOAD:
            code, slot, off = 1, ins[1], (0,) * (3 - rank) + tuple(ins[2])
        else:
            code = _OPC[(ins[0], ins[1])]
        ops.append(code)
        consts.append(val)
        slots.append(slot)
        offs += off
    return (np.asarray(ops, np.int32), np.asarray(consts, np.float64),
            np.asarray(slots, np.int32), np.asarray(offs, np.int64))


def strict_eval_statement(plan_stmt, arrays: dict, threads: int = 0) -> None:
    out = arrays[plan_stmt.output]
    rank = out.ndim
    pad = (3 - rank)
    shape3 = np.asarray(_as3(out.shape), np.int64)
    lo = np.asarray((0,) * pad + tuple(a for a, _ in plan_stmt.output_slice_bounds), np.int64)
    ext = np.asarray((1,) * pad + tuple(b - a for a, b in plan_stmt.output_slice_bounds), np.int64)
    ops, consts, slots, offs = encode_plan(plan_stmt, rank)
    ins = [arrays[a] for a in plan_stmt.inputs]
    for x in ins + [out]:
        assert x.flags.c_contiguous and x.dtype == out.dtype
    ptrs = (ctypes.c_void_p * max(1, len(ins)))(*[x.ctypes.data for x in ins])
    dt = 1 if out.dtype == np.float32 else 0
    P = ctypes.c_void_p
    rc = _lib().oracle_eval_statement(
        ctypes.c_int(dt), P(shape3.ctypes.data), P(out.ctypes.data), P(lo.ctypes.data),
        P(ext.ctypes.data), ptrs, ctypes.c_int(len(ins)), P(ops.ctypes.data),
        P(consts.ctypes.data), P(slots.ctypes.data), P(offs.ctypes.data),
        ctypes.c_int(len(ops)), ctypes.c_int(threads))
    if rc != 0:
        raise RuntimeError(f"oracle_eval_statement failed rc={rc}")


def strict_execute_dag(dag, shapes, dtypes=None, arrays=None, threads: int = 0) -> dict:
    dtypes = dtypes or {}
    arrays = {} if arrays is None else arrays
    for aid, shape in shapes.items():
        arrays.setdefault(aid, np.zeros(shape, dtype=NP_DTYPE[dtypes.get(aid, DTYPE_F64)]))
    for node in dag.nodes:
        for st in compile_plan(node, dag.ast_table).statements:
            strict_eval_statement(st, arrays, threads)
    return arrays


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Bitwise equality with every NaN treated as equal (payloads are not IEEE-specified)."""
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    iv = np.uint64 if a.dtype == np.float64 else np.uint32
    return bool(np.array_equal(a.view(iv)[~na], b.view(iv)[~nb]))


# --------------------------------------------------------------------------
# position-keyed content hash (restates include/est.h est_hash_box for tests)

def content_hash(arr: np.ndarray, threads: int = 0) -> int:
    """sum_i mix64(bits_i + 0x9e3779b97f4a7c15 * (i + 1)) mod 2^64 over the
    C-order elements of `arr` (float64 bits, or float32 bits zero-extended);
    strict_eval.c oracle_content_hash (OpenMP)."""
    a = np.ascontiguousarray(arr)
    lib = _lib()
    lib.oracle_content_hash.restype = ctypes.c_uint64
    return int(lib.oracle_content_hash(ctypes.c_void_p(a.ctypes.data), ctypes.c_int64(a.size),
                                       ctypes.c_int(a.dtype.itemsize), ctypes.c_int(threads)))


def content_hash_numpy(arr: np.ndarray, chunk: int = 1 << 24) -> int:
    """The same hash in numpy (pins the C route in tests/test_oracle_pinned.py)."""
    a = np.ascontiguousarray(arr)
    flat = (a.view(np.uint64) if a.dtype == np.float64 else a.view(np.uint32)).ravel()
    total = 0
    with np.errstate(over="ignore"):
        for lo in range(0, flat.size, chunk):
            bits = flat[lo:lo + chunk].astype(np.uint64)
            x = bits + np.uint64(0x9E3779B97F4A7C15) * (np.arange(lo, lo + bits.size, dtype=np.uint64)
                                                        + np.uint64(1))
            x ^= x >> np.uint64(30)
            x *= np.uint64(0xBF58476D1CE4E5B9)
            x ^= x >> np.uint64(27)
            x *= np.uint64(0x94D049BB133111EB)
            x ^= x >> np.uint64(31)
            total = (total + int(np.sum(x, dtype=np.uint64))) % (1 << 64)
    return total
