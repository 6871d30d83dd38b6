"""SASS listings of the shipped hot kernels (no GPU needed): NVRTC-compile the
exact sources the bench workloads instantiate, `cuobjdump -sass` each cubin into
profiles/sass/<name>.sass and count the instructions that prove the data path
(UTMALDG = TMA tensor loads, SYNCS = mbarrier ops, STG.E.128 / LDS.128 =
128-bit global stores / shared loads) into profiles/sass/summary.json."""
import collections
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def hot_sources() -> dict:
    from paper_2512_19851_b200 import resident, stream, temporal
    from paper_2512_19851_b200.analysis import compile_plan
    from paper_2512_19851_b200.codegen import kernel_source_for, stmt_sig
    from paper_2512_19851_b200.programs import DagProgram, heat3d_program, laplace_program, wave2d_program
    from paper_2512_19851_b200.tiles import TileBuffer
    from paper_2512_19851_b200.wire import DTYPE_F32

    out = {}
    p = DagProgram()
    heat3d_program(p, 16, 2)
    plan = compile_plan(p.dag.nodes[-1], p.dag.ast_table)
    sig = stmt_sig(plan.statements[0], 3)
    for n, tag in ((1024, "c4"), (512, "c2")):
        xoff, py, pz = TileBuffer.pitches((n, n, n), (1, 1, 1), 0)
        out[f"{tag}_est_tb"] = temporal.source(sig, 0, py=py, pz=pz, xoff=xoff)[0]
    out["c4_est_stream_ws2"] = kernel_source_for(plan, 3, 0, "auto")[0]
    p = DagProgram()
    wave2d_program(p, 64, 2, dtype=DTYPE_F32)
    plan = compile_plan(p.dag.nodes[-1], p.dag.ast_table)
    out["c3_est_stream_ws2_f32"] = kernel_source_for(plan, 2, DTYPE_F32, "auto")[0]
    p = DagProgram()
    laplace_program(p, 64, 2)
    plan = compile_plan(p.dag.nodes[-1], p.dag.ast_table)
    rs = stmt_sig(plan.statements[0], 2)
    g = resident.smem_geometry(1022, 1022, resident.slot_radius(rs)[0], 0, 148)
    out["c1_est_resident_smem"] = resident.smem_source(rs, 0, g)[0]
    from paper_2512_19851_b200 import temporal2d
    xoff, py, _pz = TileBuffer.pitches((16384, 16384), (1, 1), 0)
    out["lap16k_est_tc"] = temporal2d.source(rs, 0, py=py, xoff=xoff)[0]
    p = DagProgram()
    wave2d_program(p, 64, 2, dtype=DTYPE_F32)
    plan = compile_plan(p.dag.nodes[-1], p.dag.ast_table)
    xoff, py, _pz = TileBuffer.pitches((16384, 16384), (2, 2), DTYPE_F32)
    out["c3_est_tc_rotation_f32"] = temporal2d.source(stmt_sig(plan.statements[0], 2), DTYPE_F32, py=py, xoff=xoff)[0]
    return out


def main() -> None:
    from paper_2512_19851_b200.build import precompile_sources

    dst = os.path.join(ROOT, "profiles", "sass")
    os.makedirs(dst, exist_ok=True)
    summary = {}
    for name, src in hot_sources().items():
        with tempfile.TemporaryDirectory() as tmp:
            os.environ["EST_KERNEL_CACHE"] = tmp
            import paper_2512_19851_b200.device as device
            device.DEFAULT_CACHE = tmp
            precompile_sources([src])
            (cubin,) = [os.path.join(tmp, f) for f in os.listdir(tmp)]
            sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True, check=True).stdout
            res = subprocess.run(["cuobjdump", "-res-usage", cubin], capture_output=True, text=True).stdout
        open(os.path.join(dst, name + ".sass"), "w").write(sass)
        ops = collections.Counter()
        for ln in sass.splitlines():
            m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
            if m:
                ops[m.group(1)] += 1
        pick = lambda pre: sum(v for k, v in ops.items() if k.startswith(pre))
        summary[name] = {
            "static_instructions": sum(ops.values()),
            "UTMALDG": pick("UTMALDG"), "SYNCS": pick("SYNCS"),
            "STG.E.128": pick("STG.E.128"), "STG.E.64": ops.get("STG.E.64", 0), "STG.E": ops.get("STG.E", 0),
            "LDS.128": pick("LDS.128"), "LDS.64": ops.get("LDS.64", 0), "LDS": ops.get("LDS", 0),
            "DADD": ops.get("DADD", 0), "DMUL": ops.get("DMUL", 0), "DFMA": ops.get("DFMA", 0),
            "FADD": ops.get("FADD", 0), "FMUL": ops.get("FMUL", 0), "FFMA": ops.get("FFMA", 0),
            "resource_usage": " ".join(res.split())[-200:],
        }
    json.dump(summary, open(os.path.join(dst, "summary.json"), "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
