"""The paper's own benchmark shapes on one B200: 2-D Laplace
at its weak-scaling per-GPU size (16384^2 fp64) and lid-driven cavity flow
(programs.cavity_program, 10 pressure sub-iterations), as repeated DAG-bytes
batches (CUDA-graph replay), device time with CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_19851_b200.ir import fuse  # noqa: E402
from paper_2512_19851_b200.programs import (DagProgram, cavity_program, laplace_iteration_statements,  # noqa: E402
                                            laplace_program)
from paper_2512_19851_b200.session import GpuJob  # noqa: E402
from paper_2512_19851_b200.wire import encode_dag  # noqa: E402


def timed(setup, step, reps=5, fused=False):
    blob = encode_dag(fuse(step.dag) if fused else step.dag)
    with GpuJob() as job:
        for a in sorted(setup.shapes):
            job.create_array(setup.shapes[a])
        job.run(setup.dag)
        for _ in range(3):
            job.run_bytes(blob)
        job.sync()
        dev = job.devs[0]
        e0, e1 = dev.event(), dev.event()
        l0 = dev.launches
        e0.record()
        for _ in range(reps):
            job.run_bytes(blob)
        e1.record()
        e1.sync()
        return e0.elapsed_ms(e1) / reps, (dev.launches - l0) // reps


out = {}
n, it = 16384, 100
setup = DagProgram()
names = laplace_program(setup, n, 0)
step = DagProgram()
for a in sorted(setup.shapes):
    step.builder.declare_array(a, setup.shapes[a])
laplace_iteration_statements(step, names["u"], names["scratch"], it)
ms, launches = timed(setup, step)
out["laplace_16384sq_f64"] = {"ms_per_100_iters": ms, "glups": (n - 2) ** 2 * it / ms / 1e6,
                              "launches_per_batch": launches}
class DeclOnly(DagProgram):
    """Sink whose create_array only declares (the arrays already exist)."""

    def create_array(self, shape, dtype=0):
        aid = self._next
        self._next += 1
        self.builder.declare_array(aid, tuple(int(e) for e in shape))
        self.dtypes[aid] = dtype
        return aid


for n in (1024, 4096, 8192):
    setup = DagProgram()
    cavity_program(setup, n, 0)
    step = DeclOnly()
    cavity_program(step, n, 1)
    for fused in (False, True):
        ms, launches = timed(setup, step, fused=fused)
        out[f"cavity_{n}sq_f64" + ("_fused" if fused else "")] = {
            "ms_per_iteration": ms, "glups": (n - 2) ** 2 / ms / 1e6,
            "launches_per_iteration": launches,
            "nodes_per_iteration": len((fuse(step.dag) if fused else step.dag).nodes)}
print(json.dumps(out, indent=1))
