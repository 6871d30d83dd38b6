import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from paper_2512_19851_b200.ipc import spawn_local_job

def body(rank, world):
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice
    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    from paper_2512_19851_b200.programs import DagProgram, heat3d_setup, heat3d_iterations
    from paper_2512_19851_b200.wire import encode_dag
    import cProfile, pstats, io
    prog = DagProgram(); u1, u2 = heat3d_setup(prog, 64)
    job = ipc.IpcGpuJob(rank, world)
    for a in sorted(prog.shapes): job.create_array(prog.shapes[a])
    job.run(prog.dag)
    it = DagProgram()
    for a in sorted(prog.shapes): it.builder.declare_array(a, prog.shapes[a])
    heat3d_iterations(it, u1, u2, 100)
    blob = encode_dag(it.dag)
    job.run_bytes(blob)
    t0 = time.perf_counter()
    pr = cProfile.Profile() if rank == 0 else None
    if pr: pr.enable()
    for _ in range(5): job.run_bytes(blob)
    if pr: pr.disable()
    dt = (time.perf_counter() - t0) / 500
    s = io.StringIO()
    if pr: pstats.Stats(pr, stream=s).sort_stats('cumulative').print_stats(18)
    job.close()
    return dt * 1e6, s.getvalue()

if __name__ == "__main__":
    res = spawn_local_job(2, body)
    print("us per node:", [r[0] for r in res])
    print(res[0][1][:5000])
