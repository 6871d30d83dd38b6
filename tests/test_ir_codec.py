"""Input-contract parity: the restated IR / codec / analysis reproduce the
reference's golden bytes, dumps and plans (CPU only)."""

import os
import random
import struct

import pytest

from golden_cases import HERE, cases, meta_dumps
from paper_2512_19851_b200 import errors
from paper_2512_19851_b200.analysis import (
    OP_BINARY, OP_CONST, OP_LOAD, analyze, analyze_dag, compile_plan, dump_meta, ghost_depth)
from paper_2512_19851_b200.ir import (
    DagBuilder, SliceSpec, compute_edges, cst, dump_text, fuse, normalize_slice, ref, validate_dag)
from paper_2512_19851_b200.programs import DagProgram, laplace_program
from paper_2512_19851_b200.wire import (
    CREATE_ARRAY_TYPED, FETCH, Command, decode_command, decode_dag, decode_slice, encode_command,
    encode_dag, encode_slice)
from progs import random_program_2d, random_program_3d


def test_example1_dag_bytes_golden():
    prog = DagProgram()
    laplace_program(prog, 64, 10)
    assert encode_dag(prog.dag) == open(os.path.join(HERE, "example1.dag"), "rb").read()


def test_laplace16_dump_golden():
    prog = DagProgram()
    laplace_program(prog, 16, 10)
    assert dump_text(prog.dag) == open(os.path.join(HERE, "laplace16_dump.txt")).read()


def test_meta_dumps_and_plans_golden():
    prog = DagProgram()
    laplace_program(prog, 16, 10)
    metas = analyze_dag(prog.dag, prog.shapes)
    gold = meta_dumps()
    assert [dump_meta(m) for m in metas] == gold["laplace16"]
    assert {str(a): list(ghost_depth(a, metas) or []) for a in prog.shapes} == gold["laplace16_ghost"]
    plans = [[list(map(repr, p.instructions)) for p in compile_plan(n, prog.dag.ast_table).statements]
             for n in prog.dag.nodes]
    assert plans == gold["laplace16_plans"]


def test_all_golden_dags_roundtrip_canonically():
    for name, blob, shapes, _exp, _r, _b in cases():
        dag = decode_dag(blob)
        assert encode_dag(dag) == blob, name
        validate_dag(dag, shapes)


def test_jacobi_plan_shape():
    b = DagBuilder({0: (16, 16), 1: (16, 16)})
    m = slice(1, -1)
    b.add(cst(0.25), 1, (m, m))
    prog = DagProgram()
    laplace_program(prog, 16, 1)
    node = prog.dag.nodes[-1]
    plan = compile_plan(node, prog.dag.ast_table).statements[0]
    ops = [i[0] for i in plan.instructions]
    assert ops.count(OP_LOAD) == 4 and ops.count(OP_BINARY) == 4 and ops.count(OP_CONST) == 1
    assert sorted(i[2] for i in plan.instructions if i[0] == OP_LOAD) == [(-1, 0), (0, -1), (0, 1), (1, 0)]
    meta = analyze(node, prog.dag.ast_table, prog.shapes)
    assert dump_meta(meta) == "slot0: maxoff=(1,1) ghost-candidate\n"


def test_normalize_slice_rules():
    assert normalize_slice((0, slice(None)), (8, 8)).bounds == ((0, 1), (0, 8))
    assert normalize_slice((-1, slice(1, -1)), (8, 8)).bounds == ((7, 8), (1, 7))
    assert normalize_slice((slice(-3, None),), (8,)).bounds == ((5, 8),)
    with pytest.raises(errors.StridedSlice):
        normalize_slice((slice(0, 4, 2),), (8,))
    with pytest.raises(errors.InvalidSlice):
        normalize_slice((slice(4, 4),), (8,))
    with pytest.raises(errors.ShapeMismatch):
        normalize_slice((0, 0), (8,))


def test_self_dependency_and_shape_checks():
    b = DagBuilder({0: (8, 8), 1: (8, 8), 2: (4, 4)})
    with pytest.raises(errors.SelfDependency):
        b.add(ref(0, (slice(None), slice(None))), 0, (slice(None), slice(None)))
    with pytest.raises(errors.ShapeMismatch):
        b.add(ref(2, (slice(None), slice(None))), 1, (slice(0, 4), slice(0, 4)))


def test_random_roundtrips_rank2_and_rank3():
    rng = random.Random(3)
    for _ in range(10):
        for prog in (random_program_2d(rng), random_program_3d(rng)):
            dag = decode_dag(encode_dag(prog.dag))
            assert dag.nodes == prog.dag.nodes and dag.edges == prog.dag.edges
            fused = fuse(prog.dag)
            assert compute_edges(fused.nodes) == fused.edges
            validate_dag(fused, prog.shapes)


def test_decode_rejects_garbage_and_truncation():
    with pytest.raises(errors.ProtocolError):
        decode_dag(b"\x01\x02\x03")
    prog = DagProgram()
    laplace_program(prog, 16, 2)
    blob = encode_dag(prog.dag)
    for bad in (blob[:-3], blob + b"\x00"):
        with pytest.raises(errors.ProtocolError):
            decode_dag(bad)


def test_slice_and_command_codecs():
    spec = SliceSpec(((1, 15), (0, 8), (2, 3)))
    got, end = decode_slice(encode_slice(spec), 0)
    assert got == spec and end == 1 + 3 * 16
    with pytest.raises(errors.ProtocolError):
        decode_slice(struct.pack("<B", 4) + b"\x00" * 64, 0)
    cmd = Command(7, CREATE_ARRAY_TYPED, shape=(64, 64), dtype=1)
    assert decode_command(*encode_command(cmd)) == cmd
    cmd = Command(3, FETCH, array=2, slice=SliceSpec(((0, 4), (1, 2))))
    assert decode_command(*encode_command(cmd)) == cmd


def test_kernel_cache_distinguishes_signed_zero():
    """-0.0 == 0.0 as Python floats: generated kernels must still differ."""
    from paper_2512_19851_b200.analysis import compile_plan, plan_key
    from paper_2512_19851_b200.codegen import kernel_source_for
    from paper_2512_19851_b200.ir import cst
    from paper_2512_19851_b200.programs import DagProgram

    prog = DagProgram()
    a = prog.create_array((8, 8))
    prog.assign(a, (slice(0, 4), slice(None)), cst(0.0))
    prog.assign(a, (slice(0, 4), slice(None)), cst(-0.0))
    p0, p1 = (compile_plan(n, prog.dag.ast_table) for n in prog.dag.nodes[-2:])
    assert plan_key(p0.statements[0].instructions) != plan_key(p1.statements[0].instructions)
    s0, s1 = kernel_source_for(p0, 2, 0)[0], kernel_source_for(p1, 2, 0)[0]
    assert "0x8000000000000000" in s1 and "0x8000000000000000" not in s0
