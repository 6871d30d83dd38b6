"""C5-style elastic rescale benchmark through the UNCHANGED reference control plane.

The reference coordinator + client (installed in baseline/_ref) drive GPU
worker processes and GPU memory daemons (GpuLauncher). Program: 2-D Laplace
(the reference coordinator rejects rank-3 arrays, coordinator.py:383-384, so
the C5 byte volume is carried by two N x N float64 arrays; N = 32768 gives the
same 16 GiB payload as two 1024^3 arrays). Timeline: ITERS iterations on W
workers -> rescale(W/2) -> ITERS -> rescale(W) -> ITERS, then sample rows are
fetched and compared bit-for-bit with an unrescaled in-process GpuJob run of
the same 3*ITERS iterations.

Prints one JSON line: the four reference stage timings per rescale, the
client-observed rescale wall time, and the GLUP/s of each phase.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(argv=None):
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--flush", type=int, default=100)
    args = ap.parse_args(argv)

    import numpy as np

    from paper_2512_19851_b200.launcher import DEFAULT_REF, GpuLauncher, reference_available

    if not reference_available():
        print(json.dumps({"workload": "c5", "unavailable": "reference not installed in baseline/_ref"}))
        return 0
    sys.path.insert(0, DEFAULT_REF)
    import elastencil.client as client
    import elastencil.programs as programs

    n, it, w = args.n, args.iters, args.workers
    lups = (n - 2) ** 2 * it
    rows = sorted({1, n // 4 - 1, n // 4, n // 2 - 1, n // 2, n // 2 + 1, 3 * n // 4, n - 2})
    phases, rescales = {}, []
    with GpuLauncher(workers=w, max_workers=w, odf=1, scratch=os.environ.get("EST_SCRATCH")) as job:
        sess = client.Session(job.client_endpoint, timeout=1800)
        bs = client.BatchingSession(sess, flush_depth=args.flush)
        try:
            b = programs.laplace_program(bs, n, 0)
            bs.sync()
            for label, count in (("initial", None), ("shrunk", w // 2), ("restored", w)):
                if count is not None:
                    t0 = time.perf_counter()
                    st = bs.rescale(count)
                    wall = (time.perf_counter() - t0) * 1e3
                    rescales.append({"to": count, **st.as_dict(), "client_ms": wall})
                t0 = time.perf_counter()
                b = programs.laplace_iteration_statements(bs, b["u"], b["scratch"], it)
                bs.sync()
                phases[label] = lups / (time.perf_counter() - t0) / 1e9
            got = {r: np.asarray(bs.fetch(b["u"], (r, slice(None)))) for r in rows}
        finally:
            sess.shutdown()

    # unrescaled reference run of the same program on one in-process worker
    from paper_2512_19851_b200.programs import DagProgram, laplace_iteration_statements, laplace_program
    from paper_2512_19851_b200.session import GpuJob

    prog = DagProgram()
    names = laplace_program(prog, n, 0)
    with GpuJob() as ref:
        for aid in sorted(prog.shapes):
            ref.create_array(prog.shapes[aid])
        ref.run(prog.dag)
        u1, u2 = names["u"], names["scratch"]
        for _ in range(3):
            step = DagProgram()
            for aid in sorted(prog.shapes):
                step.builder.declare_array(aid, prog.shapes[aid])
            res = laplace_iteration_statements(step, u1, u2, it)
            ref.run(step.dag)
            u1, u2 = res["u"], res["scratch"]
        same = all(np.array_equal(got[r].reshape(-1).view(np.uint64),
                                  ref.fetch(u1, ((r, r + 1), (0, n))).reshape(-1).view(np.uint64))
                   for r in rows)
    line = {"workload": "c5", "metric": "rescale ms (8->4->8 workers, 1 B200)",
            "value": sum(r["client_ms"] for r in rescales), "unit": "ms", "higher_is_better": False,
            "config": {"grid": [n, n], "arrays": 2, "payload_gib": 2 * n * n * 8 / 2 ** 30,
                       "iterations_per_phase": it, "workers": [w, w // 2, w],
                       "placement": "all workers + daemons on the visible GPU(s), slot i -> GPU i mod n"},
            "rescales": rescales, "phase_glups": phases, "bit_equal_to_unrescaled": same,
            "sample_rows": rows}
    print(json.dumps(line), flush=True)
    return 0 if same else 1


if __name__ == "__main__":
    sys.exit(main())
