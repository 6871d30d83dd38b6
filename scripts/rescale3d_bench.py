"""C5 in its BASELINE shape: 3-D heat 1024^3 fp64 (2 arrays, 16 GiB) on 8 worker
processes -> redistribute to 4 -> back to 8, mid-run.

The reference coordinator rejects rank-3 arrays (coordinator.py:383-384), so
this drives the rescale's data path directly: one IpcGpuJob per process
(spawn_local_job; all processes share the visible GPU(s), rank i -> GPU i mod
n), `elastic.migrate_tiles` for the load-balance stage (D2D peer pulls of the
departing slabs, epoch rule of worker.py:384-387), ITERS iterations per phase.
Prints the redistribution ms of both directions, the GLUP/s of each phase and
whether sampled planes are bit-identical to an unrescaled single-process run
of the same 3*ITERS iterations.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _programs(n: int, iters: int):
    from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, heat3d_setup

    setup = DagProgram()
    u1, u2 = heat3d_setup(setup, n, seed_fills=8)
    step = DagProgram()
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    heat3d_iterations(step, u1, u2, iters)
    return setup, step, u1


def rank_body(rank, world, n, iters, planes):
    import numpy as np

    from paper_2512_19851_b200.device import device_count
    from paper_2512_19851_b200.elastic import migrate_tiles
    from paper_2512_19851_b200.ipc import IpcGpuJob
    from paper_2512_19851_b200.wire import encode_dag

    setup, step, u = _programs(n, iters)
    job = IpcGpuJob(rank, world, device=rank % max(1, device_count()))
    for a in sorted(setup.shapes):
        job.create_array(setup.shapes[a])
    job.run(setup.dag)
    blob = encode_dag(step.dag)
    lups = (n - 2) ** 3 * iters

    def phase():
        job.sync()
        job.barrier()
        t0 = time.perf_counter()
        job.run_bytes(blob)
        job.sync()
        job.barrier()
        return lups / (time.perf_counter() - t0) / 1e9

    def redistribute(workers):
        old = dict(job.owner_map)
        new = job.decomp.owner_map(workers)
        plan = {c: (old[c], new[c]) for c in old}
        job.sync()
        job.barrier()
        t0 = time.perf_counter()
        stats = migrate_tiles(job, plan)
        job.sync()
        job.barrier()
        return (time.perf_counter() - t0) * 1e3, stats

    out = {"glups": {}, "redistribute_ms": {}, "moved_bytes": {}, "stages": {}}
    job.run_bytes(blob)  # warm: kernels, graphs of the analysis cache, peer maps
    out["glups"]["initial_8"] = phase()
    ms, st = redistribute(world // 2)
    out["redistribute_ms"]["8->4"], out["moved_bytes"]["8->4"] = ms, st["bytes_in"]
    out["stages"]["8->4"] = {k: st[k] for k in ("pull_ms", "barrier_free_ms", "peer_maps_ms", "agree_ms", "alloc_ms")}
    out["glups"]["shrunk_4"] = phase()
    ms, st = redistribute(world)
    out["redistribute_ms"]["4->8"], out["moved_bytes"]["4->8"] = ms, st["bytes_in"]
    out["stages"]["4->8"] = {k: st[k] for k in ("pull_ms", "barrier_free_ms", "peer_maps_ms", "agree_ms", "alloc_ms")}
    out["glups"]["restored_8"] = phase()
    sample = {p: job.fetch(u, ((p, p + 1), (0, n), (0, n))) for p in planes}
    job.close()
    return out, ({p: np.ascontiguousarray(v).tobytes() for p, v in sample.items()} if rank == 0 else None)


def main():
    import argparse

    import numpy as np

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--workers", type=int, default=8)
    args = ap.parse_args()
    n, it, w = args.n, args.iters, args.workers
    planes = sorted({1, n // 8, n // 4, n // 2 - 1, n // 2, 3 * n // 4 + 1, n - 2})

    from paper_2512_19851_b200.ipc import spawn_local_job

    res = spawn_local_job(w, rank_body, n, it, planes, timeout=3000)
    per_rank = [r[0] for r in res]
    sample = res[0][1]
    # every rank measured the same collective phases; take the slowest
    glups = {k: min(r["glups"][k] for r in per_rank) for k in per_rank[0]["glups"]}
    redist = {k: max(r["redistribute_ms"][k] for r in per_rank) for k in per_rank[0]["redistribute_ms"]}
    moved = {k: sum(r["moved_bytes"][k] for r in per_rank) for k in per_rank[0]["moved_bytes"]}

    # unrescaled reference: one process, 3 * ITERS iterations
    from paper_2512_19851_b200.session import GpuJob
    from paper_2512_19851_b200.wire import encode_dag

    setup, step, u = _programs(n, it)
    with GpuJob() as ref:
        for a in sorted(setup.shapes):
            ref.create_array(setup.shapes[a])
        ref.run(setup.dag)
        blob = encode_dag(step.dag)
        for _ in range(4):  # the warm batch + 3 phases
            ref.run_bytes(blob)
        same = all(np.ascontiguousarray(ref.fetch(u, ((p, p + 1), (0, n), (0, n)))).tobytes() == sample[p]
                   for p in planes)
    line = {"workload": "c5-3d", "metric": "redistribution ms + GLUP/s per phase (8->4->8 workers)",
            "config": {"grid": [n, n, n], "dtype": "f64", "arrays": 2, "payload_gib": 2 * n ** 3 * 8 / 2 ** 30,
                       "iterations_per_phase": it, "workers": [w, w // 2, w],
                       "placement": "worker i on GPU i mod visible GPUs"},
            "redistribute_ms": redist, "moved_gib": {k: v / 2 ** 30 for k, v in moved.items()},
            "glups": glups, "bit_equal_to_unrescaled": same, "sample_planes": planes,
            "stage_ms_max_over_ranks": {d: {k: max(r["stages"][d][k] for r in per_rank)
                                            for k in per_rank[0]["stages"][d]} for d in per_rank[0]["stages"]}}
    print(json.dumps(line), flush=True)
    return 0 if same else 1


if __name__ == "__main__":
    sys.exit(main())
