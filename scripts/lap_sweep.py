"""Laplace 16384^2 fp64 (rank-2 stream kernel) GLUP/s for the current env config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_19851_b200.programs import DagProgram, laplace_iteration_statements, laplace_program  # noqa: E402
from paper_2512_19851_b200.session import GpuJob  # noqa: E402
from paper_2512_19851_b200.wire import encode_dag  # noqa: E402

n, it = 16384, 50
setup = DagProgram()
names = laplace_program(setup, n, 0)
step = DagProgram()
for a in sorted(setup.shapes):
    step.builder.declare_array(a, setup.shapes[a])
laplace_iteration_statements(step, names["u"], names["scratch"], it)
blob = encode_dag(step.dag)
with GpuJob() as job:
    for a in sorted(setup.shapes):
        job.create_array(setup.shapes[a])
    job.run(setup.dag)
    for _ in range(2):
        job.run_bytes(blob)
    job.sync()
    dev = job.devs[0]
    e0, e1 = dev.event(), dev.event()
    e0.record()
    for _ in range(4):
        job.run_bytes(blob)
    e1.record()
    e1.sync()
    ms = e0.elapsed_ms(e1) / (4 * it)
print(" ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("EST_STREAM2D")),
      f"ms/iter {ms:.4f} GLUP/s {(n - 2) ** 2 / ms / 1e6:.1f} frac {16.0 * (n - 2) ** 2 / ms / 1e6 / 6540.5:.3f}")
