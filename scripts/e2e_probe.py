"""Where the e2e step time goes: per iteration of the bench's e2e loop (one
step + the whole-array hash), host enqueue, device drain, hash, whether the
step was a graph replay, and the launches it issued."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 16
job, prog, arrays = bench.build_job(w, 1, 0)
blob = bench.step_dag(w, prog.shapes, prog.dtypes, arrays)
ex, dev = job.executors[0], job.devs[0]
for _ in range(3):
    job.run_bytes(blob)
job.sync()
rows = []
for _ in range(n_it):
    r0, l0 = ex.replays, dev.launches
    t0 = time.perf_counter(); job.run_bytes(blob); t1 = time.perf_counter()
    job.sync(); t2 = time.perf_counter()
    job.hash(arrays[0]); t3 = time.perf_counter()
    rows.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 1), round((t3 - t2) * 1e3, 2),
                 ex.replays - r0, dev.launches - l0))
print("(enqueue ms, drain ms, hash ms, replayed, launches) per iteration:")
for r in rows:
    print(r)
