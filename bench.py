"""Benchmark: grid-point updates per second of the fused stencil path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c2|c3|c1]
                    [--impl ours|reference]

Workload (default c4 = BASELINE.json configs[3], the config the north-star
"GLUP/s at 1/2/4/8 B200" metric and its >=80 %-of-HBM target are quoted on):
3-D 7-point Jacobi on a 1024^3 float64 grid, unit Dirichlet faces. One STEP is
one batch of 100 Jacobi iterations (the reference client's default flush
depth, pkg/src/elastencil/client.py:168) submitted as DAG bytes through the
worker seam and executed by the generated sm_100a kernels. Arrays (2 x 8.6 GB)
are far larger than L2 (126 MB), so no L2 flush is needed between steps; a
workload whose arrays fit L2 (c1) gets a 512 MB write between steps, outside
per-step event pairs.

`value`  : device time (CUDA events on the compute stream), max over ranks.
`e2e`    : host wall clock per step through the reference-facing seam (N=1:
           the reference Coordinator + a GPU worker process, W_BATCH frame in,
           the result array's device-computed content hash (8 B) out;
           `e2e.in_process` = the same through
           the in-process API GpuJob.run_bytes; N>1: the in-process API on
           every rank), max over ranks.
`roofline`: the dominant kernel kind, achieved = algorithmic bytes per launch /
           its average launch duration in the timed region (device time x its
           share of kernel time from a 2-step event-pair pass / its launches),
           against MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline`: the strict-order C oracle (oracle/strict_eval.c) on all host
           cores over a bounded z-slab sample of the same grid (rank 0, N=1),
           with the reference's own numpy evaluator (baseline/_ref
           executor.evaluate_statement) on one core beside it
           (`reference_1core`) and the host CPU model.
--impl reference: the reference's own CPU path on the host cores, rank 0
           only: C1 through the reference runtime (Launcher + BatchingSession,
           worker processes); C2/C4 through the reference's evaluate_statement
           in min(8, cores) processes on z-slabs (the runtime itself rejects
           rank 3); C3 (fp32, which the reference lacks) the oracle port.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "c4": dict(kind="heat3d", n=1024, iters_per_step=100, dtype="f64",
               label="C4: 3-D 7-point Jacobi 1024^3 fp64 (BASELINE configs[3])"),
    "c2": dict(kind="heat3d", n=512, iters_per_step=100, dtype="f64",
               label="C2: 3-D 7-point heat 512^3 fp64 (BASELINE configs[1])"),
    "c3": dict(kind="wave2d", n=16384, iters_per_step=100, dtype="f32",
               label="C3: 2-D acoustic wave r=2 16384^2 fp32 (BASELINE configs[2])"),
    "c1": dict(kind="laplace", n=1024, iters_per_step=100, dtype="f64", steps=2000,  # >= 0.5 s timed (clock samples)
               label="C1: 2-D 5-point Jacobi 1024^2 fp64 (BASELINE configs[0])"),
    # not a BASELINE config: the paper's 2-D Laplace weak-scaling per-GPU size
    "lap16k": dict(kind="laplace", n=16384, iters_per_step=100, dtype="f64",
                   label="paper shape: 2-D 5-point Jacobi 16384^2 fp64 per GPU"),
}
METRIC = "GLUP/s (grid-point updates/s)"
L2_BYTES = 126 << 20        # B200 L2
L2_FLUSH_BYTES = 512 << 20


def lup_per_iter(w) -> int:
    n = w["n"]
    if w["kind"] == "heat3d":
        return (n - 2) ** 3
    if w["kind"] == "wave2d":
        return (n - 4) ** 2
    return (n - 2) ** 2


def bytes_per_iter(w) -> int:
    """Algorithmic HBM bytes of one iteration."""
    n = w["n"]
    if w["kind"] == "heat3d":
        m = n - 2
        return 8 * (m ** 3 + 6 * m ** 2 + m ** 3)
    if w["kind"] == "wave2d":
        m = n - 4
        return 4 * ((m * m + 8 * m) + m * m + m * m)
    m = n - 2
    return 8 * (m * m + 4 * m + m * m)


def bytes_per_launch(w, tag) -> int:
    """Algorithmic HBM bytes of one launch of kernel kind `tag` = (kind, sweeps).

    A plain node kernel is one sweep (bytes_per_iter). A temporal chain of K
    sweeps (temporal.py) reads the input array once and writes A once; B is
    written only by the last chain of a run (temporal.SKIP_MID_B), so per
    launch: elem * (N_in + N_out) + elem * N_out / chains per run."""
    kind, sweeps = tag
    if kind in ("res", "rsm"):  # resident chains: every sweep counts as a full pass (data in L2 / smem)
        return bytes_per_iter(w) * sweeps
    if kind == "tc":
        # rank-2 two-sweep chain (temporal2d.py). Wave rotation: u1 read once
        # (with its halo), u0 read once, u2 and the new u0 written once;
        # ping-pong: A read and written once, B once per run
        from paper_2512_19851_b200 import temporal
        m = w["n"] - (4 if w["kind"] == "wave2d" else 2)
        if w["kind"] == "wave2d":
            return 4 * ((m * m + 8 * m) + 3 * m * m)
        chains = w["iters_per_step"] // 2
        chains -= chains % 2
        b_writes = 8 * m * m if not temporal.SKIP_MID_B else 8 * m * m / max(1, chains)
        return int(8 * ((m * m + 4 * m) + m * m) + b_writes)
    if kind != "tb":
        return bytes_per_iter(w)
    from paper_2512_19851_b200 import temporal
    n = w["n"]
    m = n - 2
    chains = w["iters_per_step"] // sweeps
    chains -= chains % 2
    b_writes = 8 * m ** 3 if not temporal.SKIP_MID_B else 8 * m ** 3 / max(1, chains)
    return int(8 * ((m ** 3 + 6 * m ** 2) + m ** 3) + b_writes)


def load_peaks() -> tuple:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None
            return self
        # the timed region starts once nvidia-smi is sampling; earlier lines are dropped
        t0 = time.time()
        while not self.lines and self.proc.poll() is None and time.time() - t0 < 5:
            time.sleep(0.01)
        self.skip = len(self.lines)
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines[getattr(self, "skip", 0):]:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port, test infrastructure)

def host_threads() -> int:
    """Every core this process may run on (torchrun exports OMP_NUM_THREADS=1
    to its ranks, so OpenMP's own default is not used)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample(w, iters: int = 2, planes: int = 34, threads: int = 0) -> dict:
    """Strict-order C oracle on a bounded sample of the workload, all host cores."""
    threads = threads or host_threads()
    from oracle.oracle import _lib as olib, strict_eval_statement
    from paper_2512_19851_b200.analysis import compile_plan
    from paper_2512_19851_b200.programs import DagProgram, heat3d_program, laplace_program
    from paper_2512_19851_b200.wire import DTYPE_F32

    n = w["n"]
    prog = DagProgram()
    if w["kind"] == "heat3d":
        shape = (planes, n, n)
        heat3d_program(prog, n, 1, shape=shape)
        sample = f"{iters} Jacobi iterations over a {planes}x{n}x{n} z-slab of the {n}^3 grid"
    elif w["kind"] == "wave2d":
        rows = max(planes * 16, 64)
        shape = (rows, n)
        from paper_2512_19851_b200.programs import wave2d_tree
        u = [prog.create_array(shape, DTYPE_F32) for _ in range(3)]
        prog.assign(u[2], (slice(2, -2), slice(2, -2)), wave2d_tree(u[0], u[1]))
        sample = f"{iters} wave steps over a {rows}x{n} row-slab of the {n}^2 grid"
    elif n <= 2048:
        shape = (n, n)
        laplace_program(prog, n, 1)
        sample = f"{iters} Jacobi iterations over the full {n}^2 grid"
    else:
        from paper_2512_19851_b200.programs import laplace_iteration_statements
        shape = (max(planes * 16, 64), n)
        u = [prog.create_array(shape) for _ in range(2)]
        laplace_iteration_statements(prog, u[0], u[1], 1)
        sample = f"{iters} Jacobi iterations over a {shape[0]}x{n} row-slab of the {n}^2 grid"
    node = prog.dag.nodes[-1]
    plan = compile_plan(node, prog.dag.ast_table).statements[0]
    dt = np.float32 if w["dtype"] == "f32" else np.float64
    rng = np.random.default_rng(0)
    arrays = {a: rng.random(shape).astype(dt) for a in prog.shapes}
    strict_eval_statement(plan, arrays, threads)  # warm (page faults, thread pool)
    cores = threads or olib().oracle_max_threads()
    t0 = time.perf_counter()
    for _ in range(iters):
        strict_eval_statement(plan, arrays, threads)
    dt_s = time.perf_counter() - t0
    lups = int(np.prod([b - a for a, b in plan.output_slice_bounds])) * iters
    return {"value": lups / dt_s / 1e9, "unit": "GLUP/s", "cores": int(cores), "kind": "port",
            "sample": sample + " (oracle/strict_eval.c, -ffp-contract=off, OpenMP)",
            "seconds": dt_s}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_evaluator_sample(w, planes: int = 34, iters: int = 1) -> dict | None:
    """The reference's OWN hot-path function on one core: baseline/_ref
    `elastencil.executor.evaluate_statement` (executor.py:86-176, numpy
    ufuncs + its ScratchPool) over a z-slab (3-D) / row-slab (2-D) of the
    workload, the statement decoded by the reference's own wire codec and
    compiled by its own `analysis.compile_plan`. The reference runtime rejects
    rank-3 arrays at its client / coordinator (SURVEY.md §8d "CPU side"), so a
    one-tile store adapter stands in for its 2-D TileStore. None when the
    reference is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "elastencil")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from types import SimpleNamespace

    import elastencil.ir as ref_ir
    from elastencil.analysis import compile_plan as ref_compile_plan  # the reference, unmodified
    from elastencil.executor import ScratchPool, evaluate_statement
    from elastencil.programs import DagProgram as RefDagProgram

    import paper_2512_19851_b200.programs as P

    n = w["n"]
    # the workload's statement built by the REFERENCE's DagBuilder / expression
    # constructors (this package's program builders are sink-agnostic; their
    # ref/cst/add/mul are swapped for the reference's while building)
    saved = {k: getattr(P, k) for k in ("ref", "cst", "add", "mul", "sub")}
    prog = RefDagProgram()
    try:
        for k in saved:
            setattr(P, k, getattr(ref_ir, k))
        if w["kind"] == "heat3d":
            shape = (planes, n, n)
            P.heat3d_program(prog, n, 1, shape=shape)
            sample = f"{iters} Jacobi iteration(s) over a {planes}x{n}x{n} z-slab of the {n}^3 grid"
        elif w["kind"] == "wave2d":
            shape = (max(planes * 16, 64), n)
            u = [prog.create_array(shape) for _ in range(3)]  # the reference evaluates in float64 only
            prog.assign(u[2], (slice(2, -2), slice(2, -2)), P.wave2d_tree(u[0], u[1]))
            sample = (f"{iters} wave step(s) over a {shape[0]}x{n} row-slab of the {n}^2 grid "
                      "(float64: the reference has no fp32 path)")
        elif n <= 2048:
            shape = (n, n)
            P.laplace_program(prog, n, 1)
            sample = f"{iters} Jacobi iteration(s) over the full {n}^2 grid"
        else:  # the paper shape: a row-slab (a full 16384^2 pair per process would not fit host memory x 8)
            shape = (max(planes * 16, 64), n)
            u = [prog.create_array(shape) for _ in range(2)]
            P.laplace_iteration_statements(prog, u[0], u[1], 1)
            sample = f"{iters} Jacobi iteration(s) over a {shape[0]}x{n} row-slab of the {n}^2 grid"
    finally:
        for k, v in saved.items():
            setattr(P, k, v)
    dag = prog.dag
    plan = ref_compile_plan(dag.nodes[-1], dag.ast_table).statements[0]
    depth = tuple(2 if w["kind"] == "wave2d" else 1 for _ in shape)
    rng = np.random.default_rng(0)
    bufs = {a: rng.random(tuple(e + 2 * d for e, d in zip(shape, depth))) for a in prog.shapes}
    arrays = {a: SimpleNamespace(shape=shape) for a in prog.shapes}
    zero = (0,) * len(shape)
    decomp = SimpleNamespace(tile_origin=lambda s, c: zero, tile_extents=lambda s: tuple(s))

    def interior_view(tile, a):  # grid.py:186-190
        return tile.buffers[a][tuple(slice(d, e - d) for d, e in zip(tile.depths[a], tile.buffers[a].shape))]

    store = SimpleNamespace(arrays=arrays, decomp=decomp, interior_view=interior_view)
    tile = SimpleNamespace(coords=zero, buffers=bufs, depths={a: depth for a in prog.shapes})
    pool = ScratchPool()
    evaluate_statement(plan, store, tile, pool)  # warm: scratch blocks, page faults
    t0 = time.perf_counter()
    for _ in range(iters):
        evaluate_statement(plan, store, tile, pool)
    dt_s = time.perf_counter() - t0
    lups = int(np.prod([b - a for a, b in plan.output_slice_bounds])) * iters
    return {"value": lups / dt_s / 1e9, "unit": "GLUP/s", "cores": 1, "kind": "reference",
            "sample": sample + " through baseline/_ref elastencil.executor.evaluate_statement",
            "seconds": dt_s}


def _ref_eval_proc(w, planes, iters, barrier, q):
    barrier.wait()
    q.put(reference_evaluator_sample(w, planes, iters))


def reference_evaluator_parallel(w, procs: int, planes: int = 8, iters: int = 1) -> dict | None:
    """`reference_evaluator_sample` in `procs` concurrent processes, each on
    its own slab - the way the reference runtime spreads tiles over one worker
    process per core (worker.py:428-431; its bench caps workers at 8).
    Aggregate GLUP/s = all processes' points / the slowest one's time."""
    import multiprocessing as mp

    if reference_evaluator_sample is None or not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "elastencil")):
        return None
    ctx = mp.get_context("fork")
    bar, q = ctx.Barrier(procs), ctx.Queue()
    ps = [ctx.Process(target=_ref_eval_proc, args=(w, planes, iters, bar, q)) for _ in range(procs)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join()
    slow = max(r["seconds"] for r in res)
    total = sum(r["value"] * r["seconds"] for r in res)  # GLUP
    return {"value": total / slow, "unit": "GLUP/s", "cores": procs, "kind": "reference",
            "sample": f"{procs} processes, each: " + res[0]["sample"], "seconds": slow}


def reference_runtime_sample(w, workers: int) -> dict | None:
    """C1 through the reference's OWN runtime and public API (BASELINE.md §3:
    Launcher + BatchingSession, flush 100, as pkg/src/elastencil/bench.py
    does), installed in baseline/_ref; None if it is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if w["kind"] != "laplace" or not os.path.isdir(os.path.join(ref, "elastencil")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    os.environ["PYTHONPATH"] = ref + os.pathsep + os.environ.get("PYTHONPATH", "")  # spawned workers
    from elastencil.bench import bench as ref_bench  # the reference, unmodified

    r = ref_bench("laplace", w["n"], w["iters_per_step"], workers=workers)
    lups = (w["n"] - 2) ** 2 * w["iters_per_step"]
    return {"value": lups / r["wall_s"] / 1e9, "seconds": r["wall_s"], "oracle_ok": r["oracle_ok"]}


def run_reference_arm(args, w):
    """The reference's CPU path on the host cores, rank 0 only: for C1 the
    reference runtime itself (baseline/_ref), otherwise the oracle port."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if w["kind"] == "laplace" and w["n"] <= 2048:  # the reference runtime at C1 size (lap16k: minutes per step)
        workers = 1
        while workers * 2 <= min(8, host_threads()):
            workers *= 2
        if reference_runtime_sample(w, workers) is not None:  # warm-up (spawn, imports)
            vals = []
            t0 = time.perf_counter()
            for _ in range(args.steps):
                vals.append(reference_runtime_sample(w, workers)["value"])
            wall = time.perf_counter() - t0
            value = statistics.median(vals)
            sample = (f"each step: the reference runtime (baseline/_ref elastencil, Launcher + "
                      f"BatchingSession flush 100, {workers} worker processes) running Laplace "
                      f"{w['n']}^2 x {w['iters_per_step']} end to end, verified against laplace_reference")
            line = {
                "impl": "reference", "metric": METRIC, "value": value, "unit": "GLUP/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": 1,
                "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
                "config": {"workload": w["label"], "grid": [w["n"]] * 2},
                "cpu_baseline": {"value": value, "unit": "GLUP/s", "cores": workers, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": value, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            }
            print(json.dumps(line), flush=True)
            return
    procs = min(8, host_threads())
    if w["kind"] != "wave2d" and reference_evaluator_parallel(w, procs, planes=34, iters=1) is not None:
        # rank 3 (and the 2-D fallback): the reference's own evaluate_statement
        vals = []
        t0 = time.perf_counter()
        last = None
        for _ in range(args.steps):
            last = reference_evaluator_parallel(w, procs, planes=34, iters=2)
            vals.append(last["value"])
        wall = time.perf_counter() - t0
        value = statistics.median(vals)
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": "GLUP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": 1,
            "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
            "config": {"workload": w["label"], "grid": [w["n"]] * (3 if w["kind"] == "heat3d" else 2)},
            "cpu_baseline": {"value": value, "unit": "GLUP/s", "cores": procs, "kind": "reference",
                             "sample": "each step: " + last["sample"], "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return
    planes = 34 if w["kind"] == "heat3d" else 8
    for _ in range(args.warmup):
        cpu_sample(w, iters=1, planes=planes)
    vals = []
    t0 = time.perf_counter()
    last = None
    for _ in range(args.steps):
        last = cpu_sample(w, iters=1, planes=planes)
        vals.append(last["value"])
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GLUP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
        "config": {"workload": w["label"], "grid": [w["n"]] * (3 if w["kind"] == "heat3d" else 2)},
        "cpu_baseline": {"value": value, "unit": "GLUP/s", "cores": last["cores"], "kind": "port",
                         "sample": "each step: " + last["sample"]},
        "e2e": {"value": value, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# GPU arm

def parity_check(w, skeleton: str = "auto") -> dict:
    """The benchmarked path validated at the benchmarked size: a fresh job
    runs the setup and ONE bench step (the same DAG bytes, kernels and chain
    schedule as the timed steps) and the whole-array content hash of every
    array (est_hash_box) is compared with the strict C oracle
    (oracle/strict_eval.c, all host cores) run over the same DAGs — i.e.
    bit-equality of every element. Test infrastructure: only the checker
    reads the oracle."""
    from oracle.oracle import content_hash, strict_execute_dag
    from paper_2512_19851_b200.wire import decode_dag

    t0 = time.perf_counter()
    job, prog, arrays = build_job(w, 1, 0, skeleton)
    try:
        blob = step_dag(w, prog.shapes, prog.dtypes, arrays)
        job.run_bytes(blob)
        got = {a: job.hash(a) for a in sorted(prog.shapes)}
        kinds = "tb chains" if job.executors[0]._scratch else "node kernels"
    finally:
        job.close()
    want = strict_execute_dag(prog.dag, prog.shapes, prog.dtypes, threads=host_threads())
    strict_execute_dag(decode_dag(blob), prog.shapes, prog.dtypes, arrays=want, threads=host_threads())
    ok = all(got[a] == content_hash(want[a]) for a in got)
    return {"ok": ok, "method": "setup + 1 bench step (%d iterations, %s) on a fresh job; whole-array "
                                "content hash of every array vs the strict C oracle (bit-equality)"
                                % (w["iters_per_step"], kinds),
            "arrays": len(got), "seconds": round(time.perf_counter() - t0, 1)}


def build_job(w, world: int, rank: int, skeleton: str = "auto"):
    from paper_2512_19851_b200.programs import DagProgram, heat3d_setup, laplace_program, wave2d_setup
    from paper_2512_19851_b200.session import GpuJob
    from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64

    if world > 1:
        from paper_2512_19851_b200.ipc import IpcGpuJob

        from paper_2512_19851_b200.device import device_count

        local = int(os.environ.get("LOCAL_RANK", rank))
        job = IpcGpuJob(rank, world, device=local % max(1, device_count()), skeleton=skeleton)
    else:
        job = GpuJob(workers=1, skeleton=skeleton)
    prog = DagProgram()
    n = w["n"]
    if w["kind"] == "heat3d":
        arrays = heat3d_setup(prog, n)
    elif w["kind"] == "wave2d":
        arrays = wave2d_setup(prog, n, DTYPE_F32)
    else:
        laplace_program(prog, n, 0)
        arrays = (0, 1)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid], prog.dtypes.get(aid, DTYPE_F64))
    job.run(prog.dag)
    job.sync()
    return job, prog, arrays


def step_dag(w, prog_shapes, dtypes, arrays):
    """DAG bytes of one step (iters_per_step iterations; roles return to start)."""
    from paper_2512_19851_b200.programs import DagProgram, heat3d_iterations, laplace_iteration_statements, wave2d_steps
    from paper_2512_19851_b200.wire import encode_dag

    prog = DagProgram()
    for aid in sorted(prog_shapes):
        prog.builder.declare_array(aid, prog_shapes[aid])
    k = w["iters_per_step"]
    if w["kind"] == "heat3d":
        heat3d_iterations(prog, arrays[0], arrays[1], k)
    elif w["kind"] == "wave2d":
        wave2d_steps(prog, *arrays, k)
    else:
        laplace_iteration_statements(prog, arrays[0], arrays[1], k)
    return encode_dag(prog.dag)


def seam_e2e(w, steps: int, warmup: int) -> dict | None:
    """The headline end-to-end number, through the reference-facing seam: the
    UNCHANGED reference Coordinator (baseline/_ref, driven in-process by
    session3d.Rank3Job) and one GPU worker PROCESS behind its W_* control
    protocol. Per step: the W_BATCH frame (the step's DAG
    bytes) goes host -> worker over the wire, the worker enqueues the kernels,
    and a W_HASH (the worker drains its stream and returns the updated array's
    64-bit content hash, reduced on the device) closes the step. None when the reference
    is not installed."""
    from paper_2512_19851_b200.launcher import reference_available

    if not reference_available():
        return None
    from paper_2512_19851_b200.programs import DagProgram, heat3d_setup, laplace_program, wave2d_setup
    from paper_2512_19851_b200.session3d import Rank3Job
    from paper_2512_19851_b200.wire import DTYPE_F32, DTYPE_F64, encode_dag

    prog = DagProgram()
    n = w["n"]
    if w["kind"] == "heat3d":
        arrays = heat3d_setup(prog, n)
    elif w["kind"] == "wave2d":
        arrays = wave2d_setup(prog, n, DTYPE_F32)
    else:
        laplace_program(prog, n, 0)
        arrays = (0, 1)
    with Rank3Job(1, spares=0) as job:
        for aid in sorted(prog.shapes):
            job.create_array(prog.shapes[aid], prog.dtypes.get(aid, DTYPE_F64))
        job.submit(encode_dag(prog.dag))
        job.sync()
        blob = step_dag(w, prog.shapes, prog.dtypes, arrays)
        for _ in range(max(2, warmup)):
            job.submit(blob)
        job.hash(arrays[0])
        t0 = time.perf_counter()
        for _ in range(steps):
            job.submit(blob)
            job.hash(arrays[0])
        dt = time.perf_counter() - t0
    return {"value": lup_per_iter(w) * w["iters_per_step"] * steps / dt / 1e9, "unit": "GLUP/s",
            "h2d_bytes_per_step": len(blob), "d2h_bytes_per_step": 8,
            "path": "reference Coordinator (baseline/_ref) -> W_BATCH frame (the step's DAG bytes) -> GPU "
                    "worker process -> W_HASH: the worker drains its stream and returns the updated array's "
                    "device-computed 64-bit content hash (8 bytes D2H), per step"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default 10 (c1: 2000, so the clocks are sampled)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skeleton", default="auto", choices=["auto", "point", "stream"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-seam", action="store_true", help="skip the e2e leg through the worker seam")
    ap.add_argument("--no-check", action="store_true",
                    help="skip the parity check of one bench step against the strict C oracle")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        args.steps = args.steps or 10
        run_reference_arm(args, w)
        return
    args.steps = args.steps or w.get("steps", 10)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # plumbing only: barrier + max-over-ranks
        dist.init_process_group("gloo")

    job, prog, arrays = build_job(w, world, rank, args.skeleton)
    blob = step_dag(w, prog.shapes, prog.dtypes, arrays)
    ex = job.executors[0]
    dev = job.devs[0]

    def one_step():
        return job.run_bytes(blob)

    # the timed region runs exactly what a user runs (CUDA-graph replay, no
    # per-kernel events); the roofline's per-kernel times come from a separate
    # 2-step pass right after it, with an event pair around every kernel
    inline_timing = w.get("inline_kernel_timing", False)

    for _ in range(args.warmup):
        one_step()
    job.sync()

    # ---- device-timed region ------------------------------------------------
    # a working set that fits L2 (C1) gets an L2 flush between steps, outside
    # the per-step event pairs; larger ones stream from HBM anyway
    work_bytes = sum(int(np.prod(prog.shapes[a])) * (4 if w["dtype"] == "f32" else 8) for a in arrays)
    flush_ptr = dev.alloc(L2_FLUSH_BYTES) if work_bytes < L2_BYTES else None
    if dist:
        dist.barrier()
    job.sync()
    clocks = ClockSampler(dev.index).start()
    ex.time_kernels = inline_timing
    ex.kernel_events.clear()
    launches0 = dev.launches
    if flush_ptr is None:
        ev0, ev1 = dev.event(), dev.event()
        ev0.record()
        for _ in range(args.steps):
            one_step()
        ev1.record()
        ev1.sync()
        job.sync()
        dev_ms = ev0.elapsed_ms(ev1)
    else:
        pairs = []
        for _ in range(args.steps):
            dev.memset_zero(flush_ptr, L2_FLUSH_BYTES)
            a, b = dev.event(), dev.event()
            a.record()
            one_step()
            b.record()
            pairs.append((a, b))
        job.sync()
        dev_ms = sum(a.elapsed_ms(b) for a, b in pairs)
        for a, b in pairs:
            a.close(), b.close()
        dev.free(flush_ptr)
    clock = clocks.stop()
    gpu_launches = dev.launches - launches0
    if not inline_timing:
        ex.time_kernels = True
        for _ in range(2):
            one_step()
        job.sync()
    by_tag: dict = {}
    for a, b, tag in ex.kernel_events:
        by_tag.setdefault(tag, []).append(a.elapsed_ms(b))
    ex.time_kernels = False
    for a, b, _tag in ex.kernel_events:
        a.close(), b.close()
    ex.kernel_events.clear()
    # dominant kernel = the kind with the largest total device time
    dom = max(by_tag, key=lambda t: sum(by_tag[t])) if by_tag else ("node", 1)
    kt = by_tag.get(dom, [])
    ev_total = sum(sum(v) for v in by_tag.values())
    share = (sum(kt) / ev_total) if ev_total > 0 else 1.0
    if dist:
        import torch
        t = torch.tensor([dev_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())

    lups_step = lup_per_iter(w) * w["iters_per_step"]
    value = lups_step * args.steps / (dev_ms / 1e3) / 1e9

    # ---- end-to-end through the public API ------------------------------------
    # the step's result read back to the host: the updated array's 64-bit
    # position-keyed content hash (est_hash_box over every element on the
    # device, 8 bytes D2H) - a scalar summary of the whole result, like a loss
    shape = prog.shapes[arrays[0]]
    d2h = 8

    def fetch_result():
        return job.hash_local(arrays[0]) if hasattr(job, "hash_local") else job.hash(arrays[0])

    one_step()        # untimed: first fetch allocates the pinned staging buffer
    fetch_result()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
        fetch_result()
    e2e_s = time.perf_counter() - t0
    if dist:
        import torch
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = lups_step * args.steps / e2e_s / 1e9

    # ---- roofline ------------------------------------------------------------
    peak, peak_src = load_peaks()
    # work done by the dominant kind = the sweeps it covered in the timed
    # steps (a node may be split into interior/boundary launches, a temporal
    # chain covers K nodes), so achieved = covered bytes / summed kernel time
    sweeps = dom[1]
    ev_steps = args.steps if inline_timing else 2
    tb_sweeps = sum(len(v) * k for (kind, k), v in by_tag.items() if kind in ("tb", "tc", "res", "rsm"))
    covered = len(kt) * sweeps if dom[0] in ("tb", "tc", "res", "rsm") else ev_steps * w["iters_per_step"] - tb_sweeps
    logical_launches = max(1, covered // sweeps)
    bytes_launch = bytes_per_launch(w, dom)
    if world > 1:
        bytes_launch //= world
    mean_iso = (sum(kt) / logical_launches) if kt else dev_ms / max(1, args.steps * w["iters_per_step"])
    # average launch duration inside the timed region: its device time x the
    # kind's share of kernel time / the logical launches it made there (the
    # isolated event-pair pass overstates launch-bound kernels: each pair
    # waits on the host's launch of the kernel it brackets)
    timed_launches = max(1, covered * args.steps // (ev_steps * sweeps))
    mean_k = dev_ms * share / timed_launches
    achieved = bytes_launch / (mean_k / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            pkey = args.workload + {"tb": "_tb%d" % sweeps, "tc": "_tc%d" % sweeps,
                                    "rsm": "_rsm%d" % sweeps}.get(dom[0], "")
            traffic = json.load(open(prof)).get(pkey, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": "GLUP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic",
        "config": {"workload": w["label"], "grid": list(shape),
                   "iterations_per_step": w["iters_per_step"],
                   "parallelism": f"slabs over {world} GPU(s)" if world > 1 else "1 GPU, 1 tile",
                   "l2": ("inputs larger than L2 (%d arrays, %.1f GB), no flush" % (len(arrays), work_bytes / 1e9)
                          if flush_ptr is None else
                          "working set %.1f MB fits L2: %d MB buffer written between steps, outside the "
                          "per-step event pairs" % (work_bytes / 1e6, L2_FLUSH_BYTES >> 20)),
                   "skeleton": args.skeleton,
                   "kernel_timing": "inline" if inline_timing else "separate 2-step pass (graphs in timed region)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": {"tb": "est_tb (K=%d fused sweeps)" % sweeps,
                                "tc": "est_tc (%d fused sweeps, rank 2)" % sweeps,
                                "res": "est_resident (%d sweeps)" % sweeps,
                                "rsm": "est_resident_smem (%d sweeps)" % sweeps}.get(dom[0], "est_stream/est_node (1 sweep)"),
                     "sweeps_per_launch": sweeps,
                     "kernel_ms": mean_k, "kernel_share_of_step": share,
                     "kernel_ms_isolated": mean_iso, "bytes_per_launch": bytes_launch,
                     "kernel_ms_basis": "timed-region device time x kernel share / launches in it",
                     "peak_source": peak_src,
                     "frac_of_8TBs": achieved / 8000.0,
                     **({"note": "the chain keeps the grid in shared memory (resident.py resident-smem); "
                                 "achieved counts each sweep's algorithmic bytes as if streamed from HBM, "
                                 "so frac compares against the single-sweep HBM bound it replaces"}
                        if dom[0] == "rsm" else {}),
                     **({"note": "achieved counts the bytes a 2-sweep chain must move (A read once, A written "
                                 "once, B once per run); sweep_equivalent counts what the same sweeps move as "
                                 "single sweeps, i.e. the HBM bandwidth a non-fused kernel would need for this rate",
                         "sweep_equivalent": {
                             "achieved": bytes_per_iter(w) // max(1, world) * sweeps / (mean_k / 1e3) / 1e9,
                             "frac": bytes_per_iter(w) // max(1, world) * sweeps / (mean_k / 1e3) / 1e9 / peak}}
                        if dom[0] in ("tb", "tc") else {})},
        "e2e": {"value": e2e_val, "unit": "GLUP/s",
                "h2d_bytes_per_step": len(blob), "d2h_bytes_per_step": d2h,
                "note": ("per step: the W_BATCH payload (DAG bytes) from host memory -> decode/analysis cache -> "
                         "kernel launches (the protocol has no array upload, PROTOCOL.md:37), then the result "
                         "array's device-computed 64-bit content hash copied D2H")},
        "gpu_launches": gpu_launches,
        "clocks": clock,
    }
    job.close()
    if world == 1 and not args.no_check:
        line["check"] = parity_check(w, args.skeleton)
    if world == 1 and not args.no_seam:
        seam = seam_e2e(w, args.steps, args.warmup)
        if seam is not None:  # the headline e2e is the seam's; the in-process API number stays beside it
            inproc = line["e2e"]
            line["e2e"] = dict(seam, in_process={k: inproc[k] for k in ("value", "h2d_bytes_per_step",
                                                                       "d2h_bytes_per_step", "note")})
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample(w)
        line["cpu_baseline"].pop("seconds", None)
        line["cpu_baseline"]["cpu_model"] = cpu_model()
        ref1 = reference_evaluator_sample(w, planes=34 if w["kind"] == "heat3d" else 8, iters=3)
        if ref1 is not None:  # the reference's own numpy evaluator, one core (SURVEY.md §8d CPU side)
            ref1.pop("seconds", None)
            line["cpu_baseline"]["reference_1core"] = ref1
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
