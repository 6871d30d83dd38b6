"""Where the time goes on the e2e seam path (bench.seam_e2e): C4 through the
reference Coordinator + one GPU worker process. Per step, times submit (W_BATCH
enqueue), the barrier + 1-element W_FETCH (device drain), and a one-plane
W_FETCH separately."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_19851_b200.programs import DagProgram, heat3d_setup  # noqa: E402
from paper_2512_19851_b200.session3d import Rank3Job  # noqa: E402
from paper_2512_19851_b200.wire import encode_dag  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
prog = DagProgram()
arrays = heat3d_setup(prog, w["n"])
shape = prog.shapes[arrays[0]]
plane = ((shape[0] // 2, shape[0] // 2 + 1),) + tuple((0, e) for e in shape[1:])
with Rank3Job(1, spares=0) as job:
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    job.submit(encode_dag(prog.dag))
    job.sync()
    blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
    for _ in range(3):
        job.submit(blob)
    job.sync()
    rows = []
    for _ in range(5):
        t0 = time.perf_counter()
        job.submit(blob)
        t1 = time.perf_counter()
        job.sync()
        t2 = time.perf_counter()
        job.fetch(arrays[0], plane)
        t3 = time.perf_counter()
        rows.append((t1 - t0, t2 - t1, t3 - t2))
    for r in rows:
        print("submit %.1f ms  drain %.1f ms  plane fetch %.1f ms" % tuple(x * 1e3 for x in r))
    st = job.stats()
    print("worker batch wall ms (last 5):", [round(x[1], 1) for x in st.get("batch_timeline", [])[-5:]])
