"""Sweep stream-skeleton configurations on the C4 node (1024^3 fp64 7-point).

Times only the node kernel (CUDA events around each launch) for every config;
with --ncu, run each config once so an outer `ncu --metrics ...` attributes
DRAM bytes per config (launch order = config order, after WARM launches).
Results: one JSON line per config on stdout.
"""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_19851_b200 import codegen, stream  # noqa: E402
from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, heat3d_setup  # noqa: E402
from paper_2512_19851_b200.session import GpuJob  # noqa: E402
from paper_2512_19851_b200.stream import StreamCfg  # noqa: E402

N = int(os.environ.get("SWEEP_N", 1024))
CFGS = {
    "A_np_16x8_p4_l2_256": StreamCfg(),
    "B_np_16x8_p4_l2_none": StreamCfg(l2promo=0),
    "C_np_16x8_p4_l2_128": StreamCfg(l2promo=2),
    "D_np_32x8_p2_l2_128": StreamCfg(by=32, prefetch=2, l2promo=2),
    "E_p_16x16_p4_l2_128": StreamCfg(ty=16, persistent=True, l2promo=2),
    "F_np_bx128_16x4_p2_l2_128": StreamCfg(bx=128, ty=4, prefetch=2, l2promo=2),
    "G_np_16x16_p4_l2_256": StreamCfg(ty=16),
    "H_np_8x8_p4_l2_128": StreamCfg(by=8, l2promo=2),
    "I_np_16x8_p4_z64": StreamCfg(zchunk=64),
    "J_np_16x8_p4_z256": StreamCfg(zchunk=256),
    "K_np_32x16_p2_l2_256": StreamCfg(by=32, ty=16, prefetch=2),
    "L_np_16x8_p6_l2_256": StreamCfg(prefetch=6),
}


def main():
    ncu = "--ncu" in sys.argv
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    job = GpuJob()
    prog = DagProgram()
    u1, u2 = heat3d_setup(prog, N)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    job.run(prog.dag)
    job.sync()
    it = DagProgram()
    for aid in sorted(prog.shapes):
        it.builder.declare_array(aid, prog.shapes[aid])
    heat3d_iterations(it, u1, u2, 2)
    ex = job.executors[0]
    lups = (N - 2) ** 3
    algo = 8 * (2 * (N - 2) ** 3 + 6 * (N - 2) ** 2)
    for name, cfg in CFGS.items():
        if only and name.split("_")[0] not in only:
            continue
        stream.DEFAULT = cfg
        codegen._SRC_CACHE.clear()
        ex._tmaps.clear()
        try:
            job.run(it.dag)  # compile + warm
            job.sync()
            reps = 1 if ncu else 8
            ex.time_kernels = True
            ex.kernel_events.clear()
            for _ in range(reps):
                job.run(it.dag)
            job.sync()
            ts = [a.elapsed_ms(b) for a, b in ex.kernel_events]
            ex.time_kernels = False
            ms = statistics.median(ts)
            print(json.dumps({"cfg": name, "kernel_ms": ms, "glups": lups / ms / 1e6,
                              "gbs": algo / ms / 1e6, "launches": len(ts)}), flush=True)
        except Exception as exc:  # report and continue with the next config
            print(json.dumps({"cfg": name, "error": repr(exc)[:300]}), flush=True)
            break
    job.close()


if __name__ == "__main__":
    main()
