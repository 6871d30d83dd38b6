"""Workload builders written against the reference's "sink" surface.

A sink offers ``create_array(shape[, dtype]) -> id`` and ``assign(array,
raw_slice, expr)`` (pkg/src/elastencil/programs.py:1-42). `DagProgram` collects
a whole program into one DAG (creation = a `const 0.0` full-slice statement,
PROTOCOL.md:95-96). The Laplace and cavity builders follow the reference
expression for expression (programs.py:57-267) so results compare bitwise; the
3-D heat and 2-D wave builders are the BASELINE.json C2/C4/C5 and C3 workloads
as specified in SURVEY.md §8(d).
"""

from __future__ import annotations

import random

import numpy as np

from .ir import Const, DagBuilder, StencilAst, add, cst, full_slice, mul, ref, sub
from .wire import DTYPE_F32, DTYPE_F64

_ZERO = StencilAst.create(Const(0.0))


class DagProgram:
    """Local sink collecting one DAG plus the array shapes and dtypes."""

    def __init__(self):
        self.builder = DagBuilder()
        self.dtypes: dict = {}
        self._next = 0

    def create_array(self, shape, dtype: int = DTYPE_F64) -> int:
        aid = self._next
        self._next += 1
        shape = tuple(int(e) for e in shape)
        self.builder.declare_array(aid, shape)
        self.dtypes[aid] = dtype
        self.builder.add_statement(self.builder.build_statement(_ZERO, aid, full_slice(shape), []))
        return aid

    def assign(self, array: int, raw_slice, expr) -> None:
        self.builder.add(expr, array, raw_slice)

    @property
    def dag(self):
        return self.builder.dag

    @property
    def shapes(self):
        return self.builder.shapes


def _jacobi2d(u, interior_src=None):
    a, b = slice(None, -2), slice(2, None)
    m = slice(1, -1)
    return mul(cst(0.25), add(add(add(ref(u, (a, m)), ref(u, (b, m))), ref(u, (m, a))), ref(u, (m, b))))


def laplace_iteration_statements(sink, u1: int, u2: int, iters: int) -> dict:
    """Jacobi sweeps only (programs.py:89-111)."""
    interior = (slice(1, -1), slice(1, -1))
    for _ in range(iters):
        sink.assign(u2, interior, _jacobi2d(u1))
        u1, u2 = u2, u1
    return {"u": u1, "scratch": u2}


def laplace_program(sink, n: int, iters: int) -> dict:
    """2-D 5-point Jacobi with unit Dirichlet boundaries (programs.py:57-86)."""
    u1 = sink.create_array((n, n))
    u2 = sink.create_array((n, n))
    for u in (u1, u2):
        for side in ((0, slice(None)), (-1, slice(None)), (slice(None), 0), (slice(None), -1)):
            sink.assign(u, side, cst(1.0))
    return laplace_iteration_statements(sink, u1, u2, iters)


# --------------------------------------------------------------------------
# 3-D 7-point heat / Jacobi (BASELINE configs C2, C4, C5)

SIXTH = 1.0 / 6.0


def heat3d_tree(u):
    """(1/6)*(((((zm+zp)+ym)+yp)+xm)+xp), axis 0 = z (slowest)."""
    lo, hi, m = slice(None, -2), slice(2, None), slice(1, -1)
    s = add(ref(u, (lo, m, m)), ref(u, (hi, m, m)))
    s = add(s, ref(u, (m, lo, m)))
    s = add(s, ref(u, (m, hi, m)))
    s = add(s, ref(u, (m, m, lo)))
    s = add(s, ref(u, (m, m, hi)))
    return mul(cst(SIXTH), s)


HEAT3D_FACES = (
    (0, slice(None), slice(None)), (-1, slice(None), slice(None)),
    (slice(None), 0, slice(None)), (slice(None), -1, slice(None)),
    (slice(None), slice(None), 0), (slice(None), slice(None), -1),
)


def heat3d_setup(sink, n: int, seed_fills: int = 0, seed: int = 251219851,
                 shape=None, dtype: int = DTYPE_F64) -> tuple:
    """Two arrays, all six faces 1.0; optional random sub-box constant fills.

    The random fills (values uniform(-4, 4) rounded to 3 decimals, the
    reference's random_program convention, pkg/tests/util.py:55-64) make the
    interior non-trivial so parity checks are not dominated by exact zeros.
    """
    shape = tuple(shape) if shape is not None else (n, n, n)
    u1 = sink.create_array(shape, dtype) if dtype != DTYPE_F64 else sink.create_array(shape)
    u2 = sink.create_array(shape, dtype) if dtype != DTYPE_F64 else sink.create_array(shape)
    rng = random.Random(seed)
    for u in (u1, u2):
        for face in HEAT3D_FACES:
            sink.assign(u, face, cst(1.0))
        for _ in range(seed_fills):
            box = []
            for e in shape:
                lo = rng.randint(1, max(1, e - 3))
                hi = rng.randint(lo + 1, e - 1) if lo + 1 <= e - 1 else lo + 1
                box.append((lo, hi))
            sink.assign(u, tuple(box), cst(round(rng.uniform(-4.0, 4.0), 3)))
    return u1, u2


def heat3d_iterations(sink, u1: int, u2: int, iters: int) -> dict:
    interior = (slice(1, -1),) * 3
    for _ in range(iters):
        sink.assign(u2, interior, heat3d_tree(u1))
        u1, u2 = u2, u1
    return {"u": u1, "scratch": u2}


def heat3d_program(sink, n: int, iters: int, seed_fills: int = 0, shape=None,
                   dtype: int = DTYPE_F64) -> dict:
    u1, u2 = heat3d_setup(sink, n, seed_fills, shape=shape, dtype=dtype)
    return heat3d_iterations(sink, u1, u2, iters)


# --------------------------------------------------------------------------
# 2-D acoustic wave, 2nd order in time, 4th order in space (config C3)

WAVE_C0 = float(np.float32(-5.0 / 2.0))
WAVE_C1 = float(np.float32(4.0 / 3.0))
WAVE_C2 = float(np.float32(-1.0 / 12.0))
WAVE_R = float(np.float32(0.1))


def wave2d_tree(u0, u1):
    """u2 = (2*u1 - u0) + R*((lapx + lapy) + (2*C0)*u1) on [2:-2, 2:-2]."""
    c = slice(2, -2)
    m2, m1, p1, p2 = slice(0, -4), slice(1, -3), slice(3, -1), slice(4, None)
    centre = ref(u1, (c, c))
    lapx = add(mul(cst(WAVE_C2), add(ref(u1, (c, m2)), ref(u1, (c, p2)))),
               mul(cst(WAVE_C1), add(ref(u1, (c, m1)), ref(u1, (c, p1)))))
    lapy = add(mul(cst(WAVE_C2), add(ref(u1, (m2, c)), ref(u1, (p2, c)))),
               mul(cst(WAVE_C1), add(ref(u1, (m1, c)), ref(u1, (p1, c)))))
    return add(sub(mul(cst(2.0), centre), ref(u0, (c, c))),
               mul(cst(WAVE_R), add(add(lapx, lapy), mul(cst(float(np.float32(2.0 * WAVE_C0))), centre))))


def wave2d_setup(sink, n: int, dtype: int = DTYPE_F32) -> tuple:
    arrays = tuple(sink.create_array((n, n), dtype) if dtype != DTYPE_F64
                   else sink.create_array((n, n)) for _ in range(3))
    h = n // 2
    pulse = (slice(h - 4, h + 4), slice(h - 4, h + 4))
    sink.assign(arrays[0], pulse, cst(1.0))
    sink.assign(arrays[1], pulse, cst(1.0))
    return arrays


def wave2d_steps(sink, u0: int, u1: int, u2: int, steps: int) -> dict:
    inner = (slice(2, -2), slice(2, -2))
    for _ in range(steps):
        sink.assign(u2, inner, wave2d_tree(u0, u1))
        u0, u1, u2 = u1, u2, u0
    return {"u": u1, "prev": u0, "next": u2}


def wave2d_program(sink, n: int, steps: int, dtype: int = DTYPE_F32) -> dict:
    u0, u1, u2 = wave2d_setup(sink, n, dtype)
    return wave2d_steps(sink, u0, u1, u2, steps)


# --------------------------------------------------------------------------
# lid-driven cavity (programs.py:114-267; constants oracle.py:213-243)

def cavity_constants(n: int) -> dict:
    rho, nu, dt = 1.0, 0.1, 0.001
    dx = dy = 2.0 / (n - 1)
    den = 1.0 / (2.0 * (dx * dx + dy * dy))
    return {
        "rho": rho, "nu": nu, "dt": dt, "dx": dx, "dy": dy,
        "dtdx": dt / dx, "dtdy": dt / dy,
        "inv2dx": 1.0 / (2.0 * dx), "inv2dy": 1.0 / (2.0 * dy),
        "dx2": dx * dx, "dy2": dy * dy,
        "pois_den": den,
        "pois_b_coeff": (dx * dx) * (dy * dy) * (1.0 / (2.0 * (dx * dx + dy * dy))),
        "pgrad_x": dt / (2.0 * rho * dx), "pgrad_y": dt / (2.0 * rho * dy),
        "visc_x": nu * dt / (dx * dx), "visc_y": nu * dt / (dy * dy),
        "inv_dt": 1.0 / dt,
    }


def cavity_program(sink, n: int, iters: int, pressure_iters: int = 10) -> dict:
    c = cavity_constants(n)
    u, v, p, un, vn, pn, b = (sink.create_array((n, n)) for _ in range(7))
    sink.assign(u, (-1, slice(None)), cst(1.0))
    sink.assign(un, (-1, slice(None)), cst(1.0))
    I = slice(1, -1)
    II = (I, I)
    E, W_ = slice(2, None), slice(None, -2)

    def ddx(a):
        return mul(sub(ref(a, (I, E)), ref(a, (I, W_))), cst(c["inv2dx"]))

    def ddy(a):
        return mul(sub(ref(a, (E, I)), ref(a, (W_, I))), cst(c["inv2dy"]))

    for _ in range(iters):
        un, u = u, un
        vn, v = v, vn
        dudx, dvdy, dudy, dvdx = ddx(un), ddy(vn), ddy(un), ddx(vn)
        rhs = sub(sub(sub(mul(cst(c["inv_dt"]), add(dudx, dvdy)), mul(dudx, dudx)),
                      mul(cst(2.0), mul(dudy, dvdx))), mul(dvdy, dvdy))
        sink.assign(b, II, mul(cst(c["rho"]), rhs))
        for _ in range(pressure_iters):
            pn, p = p, pn
            lap = add(mul(add(ref(pn, (I, E)), ref(pn, (I, W_))), cst(c["dy2"])),
                      mul(add(ref(pn, (E, I)), ref(pn, (W_, I))), cst(c["dx2"])))
            sink.assign(p, II, sub(mul(lap, cst(c["pois_den"])),
                                   mul(cst(c["pois_b_coeff"]), ref(b, II))))
            sink.assign(p, (slice(None), slice(-1, None)), ref(pn, (slice(None), slice(-2, -1))))
            sink.assign(p, (slice(0, 1), slice(None)), ref(pn, (slice(1, 2), slice(None))))
            sink.assign(p, (slice(None), slice(0, 1)), ref(pn, (slice(None), slice(1, 2))))
            sink.assign(p, (slice(-1, None), slice(None)), cst(0.0))

        def advect(an, grad):
            adv = sub(sub(sub(ref(an, II),
                              mul(mul(ref(un, II), cst(c["dtdx"])), sub(ref(an, II), ref(an, (I, W_))))),
                          mul(mul(ref(vn, II), cst(c["dtdy"])), sub(ref(an, II), ref(an, (W_, I))))),
                      grad)
            vx = mul(cst(c["visc_x"]), add(sub(ref(an, (I, E)), mul(cst(2.0), ref(an, II))), ref(an, (I, W_))))
            vy = mul(cst(c["visc_y"]), add(sub(ref(an, (E, I)), mul(cst(2.0), ref(an, II))), ref(an, (W_, I))))
            return add(add(adv, vx), vy)

        gx = mul(cst(c["pgrad_x"]), sub(ref(p, (I, E)), ref(p, (I, W_))))
        sink.assign(u, II, advect(un, gx))
        gy = mul(cst(c["pgrad_y"]), sub(ref(p, (E, I)), ref(p, (W_, I))))
        sink.assign(v, II, advect(vn, gy))
        for arr, side, val in ((u, (0, slice(None)), 0.0), (u, (slice(None), 0), 0.0),
                               (u, (slice(None), -1), 0.0), (u, (-1, slice(None)), 1.0),
                               (v, (0, slice(None)), 0.0), (v, (-1, slice(None)), 0.0),
                               (v, (slice(None), 0), 0.0), (v, (slice(None), -1), 0.0)):
            sink.assign(arr, side, cst(val))
    return {"u": u, "v": v, "p": p, "b": b}
