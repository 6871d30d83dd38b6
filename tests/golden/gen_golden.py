"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests:/root/repo \
        python tests/golden/gen_golden.py

It imports `elastencil` (the reference, pkg/src/elastencil) and writes, next to
this script:

* example1.dag        — encode_dag(laplace_program(DagProgram(), 64, 10)), the
                         fixture pkg/tests/test_proto.py:150-156 expects but the
                         reference does not ship (SURVEY.md §0 gap 4)
* laplace16_dump.txt  — reference dump_text of laplace_program(16, 10)
* meta_dumps.json     — reference dump_meta / ghost depths / plan shapes
* cases.npz + cases.json — per-case DAG bytes, shapes, the reference oracle's
                         outputs (reference_execute_dag, oracle.py:89-95) and the
                         reference EpochSimulator round counts (oracle.py:141-189)

Rank-3 and wave programs are built with this repo's builders and converted to
the reference's IR objects, because the reference evaluator is rank-agnostic
but its builders/codec stop at rank 2. Nothing here is needed at test time:
the tests only read the generated files.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

import elastencil.ir as rir  # reference
from elastencil import oracle as rora
from elastencil import proto as rproto
from elastencil.analysis import analyze_dag as r_analyze_dag, compile_plan as r_compile_plan
from elastencil.analysis import dump_meta as r_dump_meta, ghost_depth as r_ghost_depth
from elastencil.programs import DagProgram as RDagProgram
from elastencil.programs import cavity_program as r_cavity_program
from elastencil.programs import laplace_program as r_laplace_program
from util import random_program as r_random_program  # reference tests/util.py

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2512_19851_b200 import ir as mir  # noqa: E402
from paper_2512_19851_b200 import programs as mprog  # noqa: E402
from paper_2512_19851_b200 import wire as mwire  # noqa: E402
from progs import random_program_3d  # noqa: E402


def to_ref_expr(e):
    if isinstance(e, mir.Const):
        return rir.Const(e.value)
    if isinstance(e, mir.SlotRef):
        return rir.SlotRef(e.slot, rir.SliceSpec(tuple(tuple(b) for b in e.slice.bounds)))
    if isinstance(e, mir.Unary):
        return rir.Unary(e.op, to_ref_expr(e.child))
    return rir.Binary(e.op, to_ref_expr(e.left), to_ref_expr(e.right))


def to_ref_dag(dag):
    table = [rir.StencilAst.create(to_ref_expr(a.root)) for a in dag.ast_table]
    nodes = [rir.DagNode(n.node_id, [rir.Statement(s.ast_id, s.output,
                                                    rir.SliceSpec(tuple(tuple(b) for b in s.output_slice.bounds)),
                                                    tuple(s.inputs)) for s in n.statements])
             for n in dag.nodes]
    return rir.Dag(nodes, set(dag.edges), table)


def split_batches(dag, size):
    out = []
    for k in range(0, len(dag.nodes), size):
        nodes = [rir.DagNode(i, n.statements) for i, n in enumerate(dag.nodes[k:k + size])]
        out.append(rir.Dag(nodes, rir.compute_edges(nodes), dag.ast_table))
    return out


def ref_rounds(rdag, shapes, batch=None):
    sim = rora.EpochSimulator()
    for part in (split_batches(rdag, batch) if batch else [rdag]):
        sim.simulate_batch(part, r_analyze_dag(part, shapes))
    return {str(k): v for k, v in sorted(sim.rounds.items())}


CASES: list = []
ARRAYS: dict = {}


def add_case(name, my_dag_bytes, rdag, shapes, batch=None, extra=None):
    expected = rora.reference_execute_dag(rdag, shapes)
    meta = {
        "name": name,
        "shapes": {str(k): list(v) for k, v in shapes.items()},
        "rounds": ref_rounds(rdag, shapes, batch),
        "batch": batch,
        "arrays": sorted(shapes),
    }
    if extra:
        meta.update(extra)
    ARRAYS[f"{name}__dag"] = np.frombuffer(my_dag_bytes, dtype=np.uint8)
    for aid, val in expected.items():
        ARRAYS[f"{name}__a{aid}"] = val
    CASES.append(meta)


def main():
    # ---- codec goldens ----------------------------------------------------
    rp = RDagProgram()
    r_laplace_program(rp, 64, 10)
    ex1 = rproto.encode_dag(rp.dag)
    mp = mprog.DagProgram()
    mprog.laplace_program(mp, 64, 10)
    assert mwire.encode_dag(mp.dag) == ex1, "restated codec diverges from the reference"
    open(os.path.join(HERE, "example1.dag"), "wb").write(ex1)

    rp16 = RDagProgram()
    r_laplace_program(rp16, 16, 10)
    open(os.path.join(HERE, "laplace16_dump.txt"), "w").write(rir.dump_text(rp16.dag))

    metas = r_analyze_dag(rp16.dag, rp16.shapes)
    meta_dump = {
        "laplace16": [r_dump_meta(m) for m in metas],
        "laplace16_ghost": {str(a): list(r_ghost_depth(a, metas) or []) for a in rp16.shapes},
        "laplace16_plans": [[list(map(repr, p.instructions)) for p in r_compile_plan(n, rp16.dag.ast_table).statements]
                            for n in rp16.dag.nodes],
        "example1_sha256": hashlib.sha256(ex1).hexdigest(),
    }

    # ---- value goldens ----------------------------------------------------
    rp = RDagProgram()
    r_laplace_program(rp, 32, 10)
    add_case("laplace32x10", rproto.encode_dag(rp.dag), rp.dag, rp.shapes)

    rp = RDagProgram()
    r_cavity_program(rp, 16, 4, pressure_iters=4)
    add_case("cavity16x4", rproto.encode_dag(rp.dag), rp.dag, rp.shapes)
    add_case("cavity16x4_fused", rproto.encode_dag(rir.fuse(rp.dag)), rir.fuse(rp.dag), rp.shapes)

    rng = random.Random(20251219)
    for k in range(60):
        prog = r_random_program(rng)
        blob = rproto.encode_dag(prog.dag)
        add_case(f"rand2d_{k:03d}", blob, prog.dag, prog.shapes)
        if k % 3 == 0:
            fused = rir.fuse(prog.dag)
            add_case(f"rand2d_{k:03d}_fused", rproto.encode_dag(fused), fused, prog.shapes)

    # rank-1 (pkg/tests/test_executor.py:303-311)
    rp = RDagProgram()
    a = rp.create_array((64,))
    b = rp.create_array((64,))
    rp.assign(a, ((0, 32),), rir.cst(3.0))
    rp.assign(b, ((2, 62),), rir.ref(a, ((0, 60),)))
    rp.assign(a, ((2, 62),), rir.ref(b, ((4, 64),)))
    add_case("rank1", rproto.encode_dag(rp.dag), rp.dag, rp.shapes)

    # rank-3: this repo's builders, converted to reference objects
    for n, iters, fills in ((12, 6, 8), (16, 25, 0)):
        mp = mprog.DagProgram()
        mprog.heat3d_program(mp, n, iters, seed_fills=fills)
        add_case(f"heat3d_{n}x{iters}", mwire.encode_dag(mp.dag), to_ref_dag(mp.dag),
                 dict(mp.shapes), batch=10)
    rng = random.Random(3119851)
    for k in range(30):
        mp = random_program_3d(rng)
        add_case(f"rand3d_{k:03d}", mwire.encode_dag(mp.dag), to_ref_dag(mp.dag), dict(mp.shapes))
        if k % 3 == 0:
            fused = mir.fuse(mp.dag)
            add_case(f"rand3d_{k:03d}_fused", mwire.encode_dag(fused), to_ref_dag(fused), dict(mp.shapes))

    # wave (config C3 tree) in float64 through the reference evaluator
    mp = mprog.DagProgram()
    mprog.wave2d_program(mp, 32, 7, dtype=mwire.DTYPE_F64)
    add_case("wave2d_32x7_f64", mwire.encode_dag(mp.dag), to_ref_dag(mp.dag), dict(mp.shapes))

    np.savez_compressed(os.path.join(HERE, "cases.npz"), **ARRAYS)
    json.dump({"cases": CASES, "meta": meta_dump}, open(os.path.join(HERE, "cases.json"), "w"),
              indent=1, sort_keys=True)
    print(f"wrote {len(CASES)} cases; example1.dag sha256 {meta_dump['example1_sha256']}")


if __name__ == "__main__":
    main()
