"""Host cost per statement of the multi-process (IPC) path on the real device:
2 ranks, Laplace 64^2, 100-statement batches as DAG bytes (the worker path:
DAG cache, recorded launches). Prints us/statement, the handshake spin share
and a cProfile of rank 0 (tottime order)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rank_fn(rank, world, n, iters, batch):
    import cProfile
    import io
    import pstats

    from mp_workers import _split
    from paper_2512_19851_b200.ipc import IpcGpuJob
    from paper_2512_19851_b200.programs import DagProgram, laplace_program
    from paper_2512_19851_b200.wire import encode_dag

    prog = DagProgram()
    laplace_program(prog, n, iters)
    job = IpcGpuJob(rank, world, device=0)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    blobs = [encode_dag(p) for p in _split(prog.dag, batch)]
    job.run_bytes(blobs[0])
    job.run_bytes(blobs[1])
    job.sync()
    job.barrier()
    pr = cProfile.Profile() if rank == 0 else None
    spin0 = job.transport.spin_s
    t0 = time.perf_counter()
    if pr:
        pr.enable()
    for b in blobs[2:]:
        job.run_bytes(b)
    if pr:
        pr.disable()
    host = time.perf_counter() - t0
    job.sync()
    total = time.perf_counter() - t0
    nodes = sum(1 for _ in range(len(blobs) - 2)) * batch
    s = io.StringIO()
    if pr:
        pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(20)
    out = {"host_us_per_stmt": host / nodes * 1e6, "total_us_per_stmt": total / nodes * 1e6,
           "spin_us_per_stmt": (job.transport.spin_s - spin0) / nodes * 1e6, "prof": s.getvalue()}
    job.close()
    return out


if __name__ == "__main__":
    from paper_2512_19851_b200.ipc import spawn_local_job

    res = spawn_local_job(2, rank_fn, 64, 2200, 100, timeout=600)
    for r in res:
        print({k: round(v, 1) for k, v in r.items() if k != "prof"})
    print(res[0]["prof"][:5000])
