"""Host cost of one C4 bench step (100 Jacobi nodes as W_BATCH DAG bytes) per
rank of an N-rank slab job, on CPU with the recording device double (the
real executor, exchange, IPC transport and temporal-chain scheduling; device
calls are recorded, not executed). Compared with the device time per step a
rank has at N GPUs (C4: ~210 ms / N), it says whether the host keeps ahead
of the GPUs (W_BATCH is answered at enqueue, so host and device overlap).

usage: python scripts/host_path_ranks.py [N=8] [steps=10]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rank_fn(rank, world, steps):
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice
    from paper_2512_19851_b200 import temporal

    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    temporal.MIN_POINTS = 0  # the slab chains C4 runs (its slabs are above the threshold)
    import bench
    from paper_2512_19851_b200.programs import DagProgram, heat3d_setup

    n = 16 * world
    prog = DagProgram()
    arrays = heat3d_setup(prog, n)
    job = ipc.IpcGpuJob(rank, world)
    for a in sorted(prog.shapes):
        job.create_array(prog.shapes[a])
    job.run(prog.dag)
    w = dict(bench.WORKLOADS["c4"], n=n)
    blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
    for _ in range(2):
        job.run_bytes(blob)
    job.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        job.run_bytes(blob)
    dt = (time.perf_counter() - t0) / steps
    names = [e[2] for e in job.dev.log if e[0] == "launch"]
    out = {"host_ms_per_step": dt * 1e3, "tb_launches": names.count("est_tb"),
           "copies": len(job.dev.copies), "flag_waits": sum(1 for e in job.dev.log if e[0] == "flag_wait")}
    job.close()
    return out


if __name__ == "__main__":
    from paper_2512_19851_b200.ipc import spawn_local_job

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    res = spawn_local_job(world, rank_fn, steps, timeout=900)
    hs = [r["host_ms_per_step"] for r in res]
    print({"ranks": world, "host_ms_per_step_max": round(max(hs), 2), "host_ms_per_step_mean": round(sum(hs) / len(hs), 2),
           "c4_device_ms_per_step_per_rank_at_ideal_scaling": round(210.0 / world, 1),
           "tb_launches_rank0": res[0]["tb_launches"], "flag_waits_rank0": res[0]["flag_waits"]})
