"""Where the time goes in the reference's acceptance criterion 5 loop
(test_acceptance.py:233-263) on GPU workers: Laplace 64^2 x 2000 iterations on
2 GPU worker processes under the unchanged reference coordinator and client,
flush thresholds 1 and 100. Prints the client-observed wall per threshold and
the workers' own per-batch wall (W_BATCH replies, coordinator batch_timeline)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_19851_b200.launcher import DEFAULT_REF, GpuLauncher  # noqa: E402

sys.path.insert(0, DEFAULT_REF)
import elastencil.client as client  # noqa: E402
import elastencil.programs as programs  # noqa: E402

out = {}
for threshold in [int(t) for t in (sys.argv[1:] or ["1", "100"])]:
    with GpuLauncher(workers=2) as job:
        s = client.Session(job.client_endpoint)
        b = client.BatchingSession(s, flush_depth=threshold)
        names = programs.laplace_program(b, 64, 0)
        b.sync()
        t0 = time.perf_counter()
        names = programs.laplace_iteration_statements(b, names["u"], names["scratch"], 2000)
        t_submit = time.perf_counter() - t0
        b.sync()
        wall = time.perf_counter() - t0
        st = b.stats()
        s.shutdown()
    tl = st.get("batch_timeline", [])
    out[threshold] = {"wall_s": wall, "submit_s": t_submit, "batches": len(tl),
                      "worker_wall_ms_sum": sum(w for _, w in tl),
                      "worker_wall_ms_max": max((w for _, w in tl), default=0)}
    print(threshold, json.dumps(out[threshold]), flush=True)
