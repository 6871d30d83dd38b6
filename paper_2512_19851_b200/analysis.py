"""Per-node access analysis and the evaluation-order contract.

`analyze` records the per-slot / per-array maximum absolute index offsets that
size ghost frames and decide halo exchanges (analysis.py:30-109 of the
reference). `compile_plan` produces the deterministic left-to-right postorder
instruction list (analysis.py:137-174); it is the operation-order contract the
generated CUDA follows instruction for instruction, which is what makes the
device results bit-identical to the numpy reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .errors import UnsupportedOp
from .ir import Binary, Const, SlotRef, Unary, walk_expr

OP_CONST = "const"
OP_LOAD = "load"
OP_UNARY = "unary"
OP_BINARY = "binary"


def _vmax(a, b):
    return b if a is None else tuple(x if x >= y else y for x, y in zip(a, b))


@dataclass
class KernelMeta:
    node_id: int
    output_extent: tuple
    slot_max_offset: dict = field(default_factory=dict)   # (stmt idx, slot) -> offset
    array_max_offset: dict = field(default_factory=dict)  # array -> offset
    written_arrays: set = field(default_factory=set)

    def needs_exchange(self, array: int) -> bool:
        off = self.array_max_offset.get(array)
        return off is not None and max(off, default=0) > 0


def analyze(node, ast_table, shapes) -> KernelMeta:
    meta = KernelMeta(node.node_id, node.output_extent)
    for si, st in enumerate(node.statements):
        base = st.output_slice.starts
        st.output_slice.validate_against(shapes[st.output])
        meta.written_arrays.add(st.output)
        for leaf in walk_expr(ast_table[st.ast_id].root):
            if not isinstance(leaf, SlotRef):
                continue
            arr = st.inputs[leaf.slot]
            leaf.slice.validate_against(shapes[arr])
            off = tuple(abs(i - o) for i, o in zip(leaf.slice.starts, base))
            meta.slot_max_offset[(si, leaf.slot)] = _vmax(meta.slot_max_offset.get((si, leaf.slot)), off)
            meta.array_max_offset[arr] = _vmax(meta.array_max_offset.get(arr), off)
    return meta


def analyze_dag(dag, shapes) -> list:
    return [analyze(n, dag.ast_table, shapes) for n in dag.nodes]


def ghost_depth(array: int, metas) -> tuple | None:
    depth = None
    for m in metas:
        if array in m.array_max_offset:
            depth = _vmax(depth, m.array_max_offset[array])
    return depth


@dataclass(frozen=True)
class StatementPlan:
    instructions: tuple
    output: int
    output_slice_bounds: tuple
    inputs: tuple
    ast_id: int = -1


@dataclass(frozen=True)
class KernelPlan:
    node_id: int
    statements: tuple


def postorder(root, out_start) -> tuple:
    """Left-to-right postorder instruction tuples for one expression tree."""
    seq: list = []

    def visit(e) -> None:
        if isinstance(e, Const):
            seq.append((OP_CONST, e.value))
        elif isinstance(e, SlotRef):
            seq.append((OP_LOAD, e.slot, tuple(i - o for i, o in zip(e.slice.starts, out_start))))
        elif isinstance(e, Unary):
            visit(e.child)
            seq.append((OP_UNARY, e.op))
        elif isinstance(e, Binary):
            visit(e.left)
            visit(e.right)
            seq.append((OP_BINARY, e.op))
        else:
            raise UnsupportedOp(f"cannot compile {e!r}")

    visit(root)
    return tuple(seq)


def plan_key(instructions) -> tuple:
    """Hashable identity of a postorder plan with constants as exact bit
    patterns: as Python floats -0.0 == 0.0 (and NaN != NaN), so plans that
    differ only in a signed zero would otherwise share cache entries."""
    import struct

    return tuple((i[0], struct.pack("<d", i[1])) if i[0] == OP_CONST else i for i in instructions)


def compile_plan(node, ast_table) -> KernelPlan:
    plans = tuple(
        StatementPlan(postorder(ast_table[st.ast_id].root, st.output_slice.starts),
                      st.output, st.output_slice.bounds, st.inputs, st.ast_id)
        for st in node.statements)
    return KernelPlan(node.node_id, plans)


def dump_meta(meta: KernelMeta) -> str:
    stmts = {si for si, _ in meta.slot_max_offset} | {0}
    lines = []
    for (si, slot), off in sorted(meta.slot_max_offset.items()):
        head = f"stmt{si} " if len(stmts) > 1 else ""
        tag = " ghost-candidate" if any(off) else ""
        lines.append(f"{head}slot{slot}: maxoff=({','.join(map(str, off))}){tag}")
    return "".join(line + "\n" for line in lines)
