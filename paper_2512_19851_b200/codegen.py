"""DAG node -> sm_100a CUDA source (NVRTC-instantiated stencil skeletons).

A node's kernel is determined by its *signature*: element type, and for every
statement the postorder plan of analysis.compile_plan (offsets padded to 3-D).
Array bindings, tile pointers, pitches and output boxes are runtime parameters,
so the Laplace ping-pong (u1->u2, u2->u1), every tile of every worker and every
batch reuse one cubin.

Bit parity with the numpy reference (executor.py:86-176 / oracle.py:46-95):
every plan instruction becomes exactly one correctly rounded IEEE operation in
the plan's order (`__dadd_rn`, `__dmul_rn`, `__ddiv_rn`, `__dsqrt_rn`, ...; the
`_rn` intrinsics are never contracted into FMA and NVRTC additionally runs with
--fmad=false), constants are emitted as exact bit patterns (ir.py:151-157), neg
is a sign flip and abs clears the sign (np.negative / np.abs).

Skeletons
---------
* ``point``  — one thread per output element of a (statement, tile) box; 3-D
  boxes march ZPT planes per thread with all loads of the unrolled z-run issued
  up front (ILP), x fastest inside a warp for coalescing. Any rank / offsets /
  multi-statement node (fused statements = separate work items of ONE launch).
* ``stream`` — rank-3 single-statement nodes whose loads fit a small radius:
  2.5-D streaming (stream.py): each CTA owns an (BY x BX) column and
  walks z, staging each input plane (+ halo) in a shared-memory ring so every
  input element is fetched from L2/HBM once per CTA, with the next plane's
  loads issued before the current plane is computed.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .analysis import OP_BINARY, OP_CONST, OP_LOAD, OP_UNARY, plan_key
from .wire import DTYPE_F32, DTYPE_F64

CTYPE = {DTYPE_F64: "double", DTYPE_F32: "float"}
ELEM = {DTYPE_F64: 8, DTYPE_F32: 4}

_BIN = {
    DTYPE_F64: {"add": "__dadd_rn", "sub": "__dsub_rn", "mul": "__dmul_rn", "div": "__ddiv_rn"},
    DTYPE_F32: {"add": "__fadd_rn", "sub": "__fsub_rn", "mul": "__fmul_rn", "div": "__fdiv_rn"},
}
_SQRT = {DTYPE_F64: "__dsqrt_rn", DTYPE_F32: "__fsqrt_rn"}
_ABS = {DTYPE_F64: "fabs", DTYPE_F32: "fabsf"}


def const_literal(value: float, dtype: int) -> str:
    if dtype == DTYPE_F64:
        (bits,) = struct.unpack("<Q", struct.pack("<d", float(value)))
        return f"__longlong_as_double(0x{bits:016x}ULL)"
    (bits,) = struct.unpack("<I", np.float32(value).tobytes())
    return f"__int_as_float(0x{bits:08x})"


@dataclass(frozen=True)
class StmtSig:
    instructions: tuple  # postorder; loads carry 3-D offsets
    arity: int


@dataclass(frozen=True)
class NodeSig:
    dtype: int
    stmts: tuple
    skeleton: str = "point"

    @property
    def max_in(self) -> int:
        return max([1] + [s.arity for s in self.stmts])


def stmt_sig(plan_stmt, rank: int) -> StmtSig:
    pad = (0,) * (3 - rank)
    ins = []
    for i in plan_stmt.instructions:
        ins.append((OP_LOAD, i[1], pad + tuple(i[2])) if i[0] == OP_LOAD else i)
    return StmtSig(tuple(ins), len(plan_stmt.inputs))


def slot_radius(sig: StmtSig) -> dict:
    """slot -> per-axis max |offset| (z, y, x) over the statement's loads."""
    rad: dict = {}
    for i in sig.instructions:
        if i[0] == OP_LOAD:
            r = rad.get(i[1], (0, 0, 0))
            rad[i[1]] = tuple(max(a, abs(b)) for a, b in zip(r, i[2]))
    return rad


# --------------------------------------------------------------------------
# expression emission

def _emit_expr(sig: StmtSig, dtype: int, load) -> tuple:
    """SSA lines for the plan; `load(slot, (dz,dy,dx))` renders one operand."""
    T = CTYPE[dtype]
    lines, stack, n = [], [], 0
    for ins in sig.instructions:
        name = f"t{n}"
        n += 1
        if ins[0] == OP_CONST:
            rhs = const_literal(ins[1], dtype)
        elif ins[0] == OP_LOAD:
            rhs = load(ins[1], ins[2])
        elif ins[0] == OP_UNARY:
            a = stack.pop()
            rhs = {"neg": f"(-{a})", "abs": f"{_ABS[dtype]}({a})", "sqrt": f"{_SQRT[dtype]}({a})"}[ins[1]]
        elif ins[0] == OP_BINARY:
            b = stack.pop()
            a = stack.pop()
            rhs = f"{_BIN[dtype][ins[1]]}({a}, {b})"
        else:
            raise ValueError(ins)
        lines.append(f"const {T} {name} = {rhs};")
        stack.append(name)
    assert len(stack) == 1
    return lines, stack[0]


# --------------------------------------------------------------------------
# parameter block (all 8-byte fields; layout mirrored by pack_items)

ITEM_SCALARS = ("out", "opy", "opz", "nx", "ny", "nz", "bxn", "byn", "stmt", "blk0")


def items_per_launch(max_in: int) -> int:
    per = 8 * (len(ITEM_SCALARS) + 3 * max_in)
    return max(1, min(16, (4000 - 8) // per))


def _param_decls(max_in: int, n_items: int) -> str:
    return (
        "struct Item {\n"
        "  unsigned long long out; long long opy, opz, nx, ny, nz, bxn, byn, stmt, blk0;\n"
        f"  unsigned long long in[{max_in}]; long long ipy[{max_in}], ipz[{max_in}];\n"
        "};\n"
        f"struct Params {{ long long n; Item it[{n_items}]; }};\n"
    )


def pack_items(items: list, max_in: int, n_items: int) -> bytes:
    """items: dicts with ITEM_SCALARS keys + 'in','ipy','ipz' lists."""
    out = bytearray(struct.pack("<q", len(items)))
    for it in items:
        out += struct.pack("<Qqqqqqqqqq", *(int(it[k]) for k in ITEM_SCALARS))
        ins = list(it["in"]) + [0] * (max_in - len(it["in"]))
        ipy = list(it["ipy"]) + [0] * (max_in - len(it["ipy"]))
        ipz = list(it["ipz"]) + [0] * (max_in - len(it["ipz"]))
        out += struct.pack(f"<{max_in}Q", *ins) + struct.pack(f"<{max_in}q", *ipy)
        out += struct.pack(f"<{max_in}q", *ipz)
    pad = n_items - len(items)
    out += b"\0" * (pad * 8 * (len(ITEM_SCALARS) + 3 * max_in))
    return bytes(out)


# --------------------------------------------------------------------------
# "point" skeleton

POINT_BLOCK_3D = (32, 8, 1)
POINT_BLOCK_1D = (256, 1, 1)
POINT_ZPT = 4


def point_geometry(rank: int):
    block = POINT_BLOCK_1D if rank == 1 else POINT_BLOCK_3D
    zpt = POINT_ZPT if rank == 3 else 1
    return block, zpt


def point_source(sig: NodeSig, rank: int) -> tuple:
    T = CTYPE[sig.dtype]
    block, zpt = point_geometry(rank)
    max_in = sig.max_in
    n_items = items_per_launch(max_in)
    cases = []
    for si, st in enumerate(sig.stmts):
        body = [f"    case {si}: {{"]
        for s in range(st.arity):
            body.append(f"      const {T}* __restrict__ s{s} = reinterpret_cast<const {T}*>(I.in[{s}])"
                        f" + (z * I.ipz[{s}] + y * I.ipy[{s}] + x);")
            body.append(f"      const long long py{s} = I.ipy[{s}], pz{s} = I.ipz[{s}]; (void)py{s}; (void)pz{s};")

        def load(slot, off):
            dz, dy, dx = off
            terms = [t for t in (f"({dz})*pz{slot}" if dz else "", f"({dy})*py{slot}" if dy else "",
                                 f"({dx})" if dx else "") if t]
            return f"__ldg(s{slot} + ({' + '.join(terms) or '0'}))"

        lines, res = _emit_expr(st, sig.dtype, load)
        body += ["      " + ln for ln in lines]
        body.append(f"      o[z * I.opz + y * I.opy + x] = {res};")
        body.append("    } break;")
        cases.append("\n".join(body))
    src = f"""// generated by paper_2512_19851_b200/codegen.py — skeleton "point"
typedef {T} T;
{_param_decls(max_in, n_items)}
extern "C" __global__ void __launch_bounds__({block[0] * block[1]})
est_node(const __grid_constant__ Params p) {{
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch: predecessor complete
  long long b = blockIdx.x;
  int k = 0;
  while (k + 1 < p.n && b >= p.it[k + 1].blk0) ++k;
  const Item& I = p.it[k];
  b -= I.blk0;
  const long long bx = b % I.bxn, rest = b / I.bxn;
  const long long by = rest % I.byn, bz = rest / I.byn;  // z-blocks: ceil(nz / ZPT)
  const long long x = bx * {block[0]} + threadIdx.x;
  const long long y = by * {block[1]} + threadIdx.y;
  if (x >= I.nx || y >= I.ny) return;
  T* __restrict__ o = reinterpret_cast<T*>(I.out);
  const long long z0 = bz * {zpt};
  #pragma unroll
  for (int dzi = 0; dzi < {zpt}; ++dzi) {{
    const long long z = z0 + dzi;
    if (z >= I.nz) break;
    switch ((int)I.stmt) {{
{chr(10).join(cases)}
    default: break;
    }}
  }}
}}
"""
    return src, "est_node", block, 0, n_items, zpt


# --------------------------------------------------------------------------
# "stream" skeleton (2.5-D, TMA): see stream.py

def stream_eligible(stmts, rank: int, dtype: int = DTYPE_F64, cfg=None) -> bool:
    from . import stream

    return stream.eligible(stmts, rank, dtype, cfg)


def stream_source(sig: NodeSig, rank: int, cfg=None) -> tuple:
    from . import stream

    return stream.source(sig, rank, cfg)


# --------------------------------------------------------------------------
# skeleton selection

_SRC_CACHE: dict = {}


def kernel_source_for(plan, rank: int, dtype: int, skeleton: str = "auto", small: bool = False) -> tuple:
    """-> (source, kernel name, block, smem, items per launch, geometry, NodeSig).

    `small`: the node's boxes are small (stream.SMALL_2D_POINTS) - rank-2
    stream nodes then use shorter tiles. Memoised on the plan instructions,
    so repeated nodes cost a dict lookup.
    """
    from . import stream

    cfg = stream.cfg_for(rank, small, dtype)
    key = (tuple(plan_key(p.instructions) for p in plan.statements), rank, dtype, skeleton, cfg)
    hit = _SRC_CACHE.get(key)
    if hit is not None:
        return hit
    stmts = tuple(stmt_sig(p, rank) for p in plan.statements)
    skel = "point"
    if skeleton in ("auto", "stream"):
        for c in stream.fallback_cfgs(rank, small, dtype):
            if stream_eligible(stmts, rank, dtype, c):
                skel, cfg = "stream", c
                break
    sig = NodeSig(dtype, stmts, skel)
    res = (*(stream_source(sig, rank, cfg) if skel == "stream" else point_source(sig, rank)), sig)
    _SRC_CACHE[key] = res
    return res
