"""C5 in its BASELINE shape: elastic rescale mid-run, 3-D heat 1024^3 fp64
(2 arrays, 16 GiB) on 8 -> 4 -> 8 GPU worker processes.

The job runs on GPU worker / memory-daemon PROCESSES under the reference
Coordinator class (session3d.Rank3Job: the coordinator's own W_* control plane
and its unmodified rescale path, coordinator.py:501-607 — load balance,
checkpoint into the daemons, worker-process restart through the launcher,
restore; the expand order is checkpoint, restart, restore, load balance).
ITERS iterations per phase: phase 1 on 8 workers, rescale(4), phase 2,
rescale(8), phase 3. Reported:

* the four StageTimings of each rescale and the client-observed total;
* GLUP/s of each phase, timed from the first W_BATCH to a synchronising
  W_FETCH (workers drain their streams before replying), i.e. device work;
* bit-equality of BOTH full arrays against an unrescaled single-process
  GpuJob running the same 3 x ITERS iterations, through the position-keyed
  whole-array content hash (est_hash_box; W_HASH partials summed), plus the
  oracle-checked hash of a small control run of the same code path.

With one visible GPU all worker processes share it (placement: worker i on
GPU i mod visible GPUs), so phase rates and stage times include that
contention; the restart stage is also measured for one worker alone. The
launcher's warm-spare pool (launcher.GpuLauncher) is waited for before each
rescale, so the restart stage is the hand-over to standby processes that
already hold their CUDA context (`restart_handover` records warm / cold);
EST_SPARES=0 measures cold respawns.
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def programs(n: int, iters: int, fills: int):
    from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, heat3d_setup
    from paper_2512_19851_b200.wire import encode_dag

    setup = DagProgram()
    u1, u2 = heat3d_setup(setup, n, seed_fills=fills)
    step = DagProgram()
    for a in sorted(setup.shapes):
        step.builder.declare_array(a, setup.shapes[a])
    heat3d_iterations(step, u1, u2, iters)
    return setup, encode_dag(setup.dag), encode_dag(step.dag)


def rescaled_run(n: int, iters: int, workers: int, shrink_to: int, fills: int, batches: int) -> dict:
    """Phase / rescale / phase / rescale / phase on GPU worker processes."""
    from paper_2512_19851_b200.session3d import Rank3Job

    setup, setup_b, step_b = programs(n, iters // batches, fills)
    lups = (n - 2) ** 3 * iters
    out = {"glups": {}, "rescales": {}}
    with Rank3Job(workers) as job:
        for a in sorted(setup.shapes):
            job.create_array(setup.shapes[a])
        job.submit(setup_b)
        job.sync()

        def phase(name):
            t0 = time.perf_counter()
            for _ in range(batches):
                job.submit(step_b)
            job.sync()
            out["glups"][name] = lups / (time.perf_counter() - t0) / 1e9

        phase(f"phase1_{workers}w")
        spares_ready = job.launcher.wait_spares(300)
        out["rescales"][f"{workers}->{shrink_to}"] = job.rescale(shrink_to)
        phase(f"phase2_{shrink_to}w")
        spares_ready &= job.launcher.wait_spares(300)
        out["rescales"][f"{shrink_to}->{workers}"] = job.rescale(workers)
        phase(f"phase3_{workers}w")
        out["restart_handover"] = {"spares_ready": spares_ready, "per_restart": job.launcher.restart_log}
        out["hash"] = {str(a): job.hash(a) for a in sorted(setup.shapes)}
        st = job.stats()
        out["rounds"] = st["rounds"]
        out["kernel_launches"] = st["kernel_launches"]
    return out


def unrescaled(n: int, iters: int, fills: int, batches: int) -> dict:
    from paper_2512_19851_b200.session import GpuJob

    setup, setup_b, step_b = programs(n, iters // batches, fills)
    with GpuJob() as job:
        for a in sorted(setup.shapes):
            job.create_array(setup.shapes[a])
        job.run_bytes(setup_b)
        for _ in range(3 * batches):
            job.run_bytes(step_b)
        return {str(a): job.hash(a) for a in sorted(setup.shapes)}


def restart_alone() -> dict:
    """The restart stage with ONE worker process on the GPU (no context
    contention): a 1 -> 1 rescale of a small job (checkpoint, restart,
    restore of one process)."""
    from paper_2512_19851_b200.session3d import Rank3Job

    setup, setup_b, step_b = programs(64, 2, 0)
    with Rank3Job(1) as job:
        for a in sorted(setup.shapes):
            job.create_array(setup.shapes[a])
        job.submit(setup_b)
        job.submit(step_b)
        job.sync()
        job.launcher.wait_spares(300)
        return dict(job.rescale(1), handover=job.launcher.restart_log[-1])


def main():
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=1000, help="iterations per phase")
    ap.add_argument("--batches", type=int, default=10, help="W_BATCH messages per phase")
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--fills", type=int, default=64)
    args = ap.parse_args()
    n, it, w = args.n, args.iters, args.workers
    res = rescaled_run(n, it, w, w // 2, args.fills, args.batches)
    ref = unrescaled(n, it, args.fills, args.batches)
    alone = restart_alone()
    line = {"workload": "C5: elastic rescale mid-run, 3-D heat %d^3 fp64, %d->%d->%d worker processes"
                        % (n, w, w // 2, w),
            "config": {"grid": [n] * 3, "dtype": "f64", "arrays": 2, "payload_gib": 2 * n ** 3 * 8 / 2 ** 30,
                       "iterations_per_phase": it, "batches_per_phase": args.batches,
                       "seeded_fills_per_array": args.fills,
                       "placement": "worker i on GPU i mod visible GPUs"},
            "rescales": res["rescales"], "glups": res["glups"],
            "bit_equal_to_unrescaled": res["hash"] == ref,
            "hash_rescaled": res["hash"], "hash_unrescaled": ref,
            "rounds": res["rounds"], "restart_handover": res.get("restart_handover"),
            "restart_one_worker_alone": alone}
    print(json.dumps(line), flush=True)
    return 0 if line["bit_equal_to_unrescaled"] else 1


if __name__ == "__main__":
    sys.exit(main())
