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
B = StreamCfg(bx=128, by=8, ty=4, prefetch=3, zchunk=128, l2promo=2, ws=True, zreg=True)
R = dict(zchunk=128, l2promo=2, ws=True, zreg=True)
CFGS = {
    "T0_S8": B,
    "T1_p4": StreamCfg(bx=128, by=8, ty=4, prefetch=4, **R),
    "T2_p2": StreamCfg(bx=128, by=8, ty=4, prefetch=2, **R),
    "T3_z64": StreamCfg(bx=128, by=8, ty=4, prefetch=3, **(R | {"zchunk": 64})),
    "T4_128x8x2": StreamCfg(bx=128, by=8, ty=2, prefetch=3, **R),
    "T5_128x16x4": StreamCfg(bx=128, by=16, ty=4, prefetch=3, **R),
    "T6_64x16x4": StreamCfg(bx=64, by=16, ty=4, prefetch=3, **R),
    "T7_l2_256": StreamCfg(bx=128, by=8, ty=4, prefetch=3, **(R | {"l2promo": 3})),
    "T8_192x8x4": StreamCfg(bx=192, by=8, ty=4, prefetch=3, **R),
    "T9_128x4x4": StreamCfg(bx=128, by=4, ty=4, prefetch=3, **R),
    "T10_128x12x4": StreamCfg(bx=128, by=12, ty=4, prefetch=3, **R),
    "T11_nozreg": StreamCfg(bx=128, by=8, ty=4, prefetch=3, **(R | {"zreg": False})),
    "T12_H2_nonws": StreamCfg(bx=64, by=8, ty=8, prefetch=3, zchunk=128, l2promo=2),
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
            sustained = "--sustained" in sys.argv
            if sustained:  # emulate the bench: heat up to the power cap first
                for _ in range(200):
                    job.run(it.dag)
            reps = 1 if ncu else (40 if sustained else 8)
            ex.time_kernels = True
            ex.kernel_events.clear()
            for _ in range(reps):
                job.run(it.dag)
            job.sync()
            ts = [a.elapsed_ms(b) for a, b, _t in ex.kernel_events]
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
