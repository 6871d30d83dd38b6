"""Random program generators for parity tests.

`random_program_2d` follows the reference generator pkg/tests/util.py:20-87
(constant sub-box fills with values uniform(-4,4) rounded to 3 decimals,
offsets up to +/-max_offset, sqrt guarded by abs, div by abs(x)+1.5).
`random_program_3d` is the same recipe for rank-3 grids (the reference runtime
is rank<=2, but its oracle is rank-agnostic, SURVEY.md §0 gap 1).
"""

from __future__ import annotations

import random

from paper_2512_19851_b200.ir import BoundBinary, BoundUnary, cst, ref
from paper_2512_19851_b200.programs import DagProgram
from paper_2512_19851_b200.wire import DTYPE_F64

_BIN = ["add", "sub", "mul", "div"]
_UN = ["neg", "abs", "sqrt"]


def _tame(rng):
    return round(rng.uniform(-4.0, 4.0), 3)


def _subbox(rng, shape):
    out = []
    for n in shape:
        lo = rng.randint(0, n - 2)
        out.append((lo, rng.randint(lo + 1, n)))
    return tuple(out)


def _expr(rng, inputs, box, max_off, depth):
    if depth >= 3 or (depth > 0 and rng.random() < 0.35):
        if rng.random() < 0.25:
            return cst(_tame(rng))
        arr = rng.choice(inputs)
        sl = []
        for lo, hi in box:
            d = rng.randint(-max_off, max_off)
            sl.append((lo + d, hi + d))
        return ref(arr, tuple(sl))
    if rng.random() < 0.25:
        op = rng.choice(_UN)
        child = _expr(rng, inputs, box, max_off, depth + 1)
        if op == "sqrt":
            child = BoundUnary("abs", child)
        return BoundUnary(op, child)
    op = rng.choice(_BIN)
    lhs = _expr(rng, inputs, box, max_off, depth + 1)
    rhs = _expr(rng, inputs, box, max_off, depth + 1)
    if op == "div":
        rhs = BoundBinary("add", BoundUnary("abs", rhs), cst(1.5))
    return BoundBinary(op, lhs, rhs)


def random_program_nd(rng: random.Random, rank: int, sizes, n_arrays=4, n_statements=8,
                      max_offset=2, dtype=DTYPE_F64) -> DagProgram:
    n = rng.choice(list(sizes))
    shape = (n,) * rank
    prog = DagProgram()
    arrays = [prog.create_array(shape, dtype) for _ in range(n_arrays)]
    for a in arrays:
        for _ in range(rng.randint(1, 3)):
            prog.assign(a, _subbox(rng, shape), cst(_tame(rng)))
    for _ in range(n_statements):
        out = rng.choice(arrays)
        ins = [a for a in arrays if a != out]
        rng.shuffle(ins)
        ins = ins[: rng.randint(1, min(2, len(ins)))]
        box = []
        for _d in range(rank):
            lo = rng.randint(max_offset, max_offset + 1)
            box.append((lo, n - rng.randint(max_offset, max_offset + 1)))
        box = tuple(box)
        prog.assign(out, box, _expr(rng, ins, box, max_offset, 0))
    return prog


def random_program_2d(rng, max_size=16, **kw) -> DagProgram:
    return random_program_nd(rng, 2, [s for s in range(8, max_size + 1) if s % 4 == 0], **kw)


def random_program_3d(rng, **kw) -> DagProgram:
    return random_program_nd(rng, 3, (8, 12, 16), **kw)
