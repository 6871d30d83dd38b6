"""Per-sweep device time of Laplace chains: resident (one launch per batch)
vs node by node (CUDA-graph replay), at several grid sizes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_19851_b200.programs import DagProgram, laplace_iteration_statements, laplace_program  # noqa: E402
from paper_2512_19851_b200.session import GpuJob  # noqa: E402
from paper_2512_19851_b200.wire import encode_dag  # noqa: E402

ITERS = 100
for n in (64, 128, 256, 512, 1024, 2048):
    row = {"n": n}
    for mode in ("resident", "graphs"):
        setup = DagProgram()
        names = laplace_program(setup, n, 0)
        step = DagProgram()
        for a in sorted(setup.shapes):
            step.builder.declare_array(a, setup.shapes[a])
        laplace_iteration_statements(step, names["u"], names["scratch"], ITERS)
        blob = encode_dag(step.dag)
        with GpuJob() as job:
            for a in sorted(setup.shapes):
                job.create_array(setup.shapes[a])
            job.executors[0].resident = mode == "resident"
            job.run(setup.dag)
            for _ in range(4):
                job.run_bytes(blob)
            job.sync()
            dev = job.devs[0]
            e0, e1 = dev.event(), dev.event()
            e0.record()
            for _ in range(10):
                job.run_bytes(blob)
            e1.record()
            e1.sync()
            row[mode + "_us_per_sweep"] = round(e0.elapsed_ms(e1) * 1e3 / (10 * ITERS), 3)
    print(json.dumps(row), flush=True)
