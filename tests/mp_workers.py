"""Per-rank bodies for the multi-process tests (importable by spawned children)."""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def _program(kind: str):
    from paper_2512_19851_b200.programs import DagProgram, heat3d_program, laplace_program

    prog = DagProgram()
    if kind == "laplace":
        names = laplace_program(prog, 32, 10)
    elif kind == "heat3d":
        names = heat3d_program(prog, 16, 9, seed_fills=4)
    else:
        raise ValueError(kind)
    return prog, names


def _split(dag, size):
    from paper_2512_19851_b200.ir import Dag, DagNode, compute_edges

    out = []
    for k in range(0, len(dag.nodes), size):
        nodes = [DagNode(i, n.statements) for i, n in enumerate(dag.nodes[k:k + size])]
        out.append(Dag(nodes, compute_edges(nodes), dag.ast_table))
    return out


def host_logic_rank(rank, world, kind, odf, batch, chains=False):
    """CPU: fake device, real executor / exchange / IPC transport host logic.
    `chains`: temporal chains at test sizes (slab chains across processes)."""
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice

    if chains:
        from paper_2512_19851_b200 import temporal

        temporal.MIN_POINTS = 0

    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    prog, _ = _program(kind)
    job = ipc.IpcGpuJob(rank, world, odf=odf)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    stats = []
    for part in _split(prog.dag, batch):
        stats += job.run(part)
    rounds = job.rounds_by_array()
    strips = [c for c in job.dev.copies if c[0] == "strip"]
    out = {"rounds": rounds, "net": sum(s.net_messages for s in stats),
           "launches": sum(s.kernel_launches for s in stats),
           "strips": len(strips), "seq": job.transport.seq,
           "copy_lane_pulls": job.dev.lane_copies.get(1, 0),
           "tiles": sorted(job.store.tiles),
           "tb_launches": sum(1 for e in job.dev.log if e[0] == "launch" and e[2] == "est_tb"),
           "twins": len(job.store.twins),
           "peer_windows": len(job.transport.window_maps),
           "peer_tile_maps": len(job.transport.peer_maps),
           "exports": sum(1 for c in job.dev.copies if c[0] == "strip" and
                          any(p <= c[2] < p + 2 * sig[3][0] * sig[1] * sig[5]
                              for p, sig in job.transport.windows.values())),
           "flag_waits": sum(1 for e in job.dev.log if e[0] == "flag_wait")}
    job.close()
    return out


def gpu_rank(rank, world, kind, odf, batch, chains=False):
    """GPU: real IPC job; several processes may share cuda:0. `chains`:
    temporal chains at test sizes (slab chains across processes)."""
    from oracle.oracle import bits_equal, reference_execute_dag
    from paper_2512_19851_b200.ipc import IpcGpuJob

    if chains:
        from paper_2512_19851_b200 import temporal

        temporal.MIN_POINTS = 0
    prog, names = _program(kind)
    job = IpcGpuJob(rank, world, device=0, odf=odf)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    for part in _split(prog.dag, batch):
        job.run(part)
    want = reference_execute_dag(prog.dag, prog.shapes)
    ok = {aid: bits_equal(job.fetch(aid), want[aid]) for aid in prog.shapes}
    rounds = job.rounds_by_array()
    twins = len(job.store.twins)
    job.close()
    return {"ok": ok, "rounds": rounds, "twins": twins}


def migrate_rank(rank, world, kind, shrink_to):
    """CPU: fake device; run, migrate every tile onto `shrink_to` workers (the
    rest own nothing), run, migrate back, run. Rounds must stay globally
    sequenced (tile-less workers keep counting epochs)."""
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice

    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    from paper_2512_19851_b200.elastic import migrate_tiles

    prog, _ = _program(kind)
    parts = _split(prog.dag, max(1, len(prog.dag.nodes) // 3))
    job = ipc.IpcGpuJob(rank, world, timeout_s=60.0)
    for aid in sorted(prog.shapes):
        job.create_array(prog.shapes[aid])
    seqs = []

    def move(workers):
        old = dict(job.owner_map)
        new = job.decomp.owner_map(workers)
        migrate_tiles(job, {c: (old[c], new[c]) for c in old})

    job.run(parts[0])
    seqs.append(job.transport.seq)
    move(shrink_to)
    tiles_shrunk = sorted(job.store.tiles)
    for part in parts[1:-1]:
        job.run(part)
    seqs.append(job.transport.seq)
    move(world)
    job.run(parts[-1])
    seqs.append(job.transport.seq)
    out = {"seqs": seqs, "tiles_shrunk": tiles_shrunk,
           "epochs": {a: job.store.local_epoch(a) for a in prog.shapes}}
    job.close()
    return out


def single_tile_chain_rank(rank, world, kind, rsm=False):
    """A single-tile 2-D job whose worker owns a transport (the GPU worker
    process, world 1 or a job whose other ranks own no tile): the rank-2
    chain kernel (est_tc) runs there too, or with `rsm` the small-grid
    shared-memory-resident run. Returns the kernels launched by one step and
    the arrays' final epochs."""
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice
    from paper_2512_19851_b200 import temporal2d
    from paper_2512_19851_b200.programs import DagProgram, laplace_iteration_statements, laplace_program
    from paper_2512_19851_b200.tiles import decompose
    from paper_2512_19851_b200.wire import encode_dag

    temporal2d.MIN_POINTS = 0
    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    prog = DagProgram()
    laplace_program(prog, 64, 0)
    decomp = decompose((64, 64), 1, 1)   # one tile, owned by rank 0
    job = ipc.IpcGpuJob(rank, world, decomp=decomp, owner_map={c: 0 for c in decomp.all_coords()})
    try:
        job.executor.resident_smem = rsm
        for a in sorted(prog.shapes):
            job.create_array(prog.shapes[a])
        job.run(prog.dag)
        step = DagProgram()
        for a in sorted(prog.shapes):
            step.builder.declare_array(a, prog.shapes[a])
        laplace_iteration_statements(step, 0, 1, 8)
        job.dev.log.clear()
        job.run_bytes(encode_dag(step.dag))
        names = [e[2] for e in job.dev.log if e[0] == "launch"]
        return {"names": names, "epochs": {a: job.store.local_epoch(a) for a in sorted(prog.shapes)},
                "tiles": len(job.store.tiles)}
    finally:
        job.close()


def checkpoint_rank(rank, world, address, manifest_path):
    """A one-worker job fills a 3-D array, checkpoints into the daemon and
    writes the manifest; returns the arrays' content hashes."""
    import json

    from paper_2512_19851_b200.daemon import DaemonClient
    from paper_2512_19851_b200.elastic import build_manifest, checkpoint_tiles
    from paper_2512_19851_b200.ipc import IpcGpuJob
    from paper_2512_19851_b200.programs import DagProgram, heat3d_program

    prog = DagProgram()
    heat3d_program(prog, 48, 6, seed_fills=10)
    job = IpcGpuJob(rank, world, device=0)
    try:
        for aid in sorted(prog.shapes):
            job.create_array(prog.shapes[aid])
        job.run(prog.dag)
        hashes = {a: job.hash(a) for a in sorted(prog.shapes)}
        c = DaemonClient(address)
        try:
            records, meta = checkpoint_tiles(job, c, rank)
        finally:
            c.close()
        with open(manifest_path, "w") as fh:
            json.dump(build_manifest(1, world, job.store.decomp, meta, records), fh)
        return {"hashes": hashes, "records": len(records)}
    finally:
        job.close()


def restore_rank(rank, world, manifest_path):
    from paper_2512_19851_b200.elastic import (decomp_from_manifest, owner_map_from_manifest, read_manifest,
                                               restore_tiles)
    from paper_2512_19851_b200.ipc import IpcGpuJob

    m = read_manifest(manifest_path)
    job = IpcGpuJob(rank, world, device=0, decomp=decomp_from_manifest(m), owner_map=owner_map_from_manifest(m))
    try:
        stats = {}
        depths = restore_tiles(job, m, stats)
        job.executor.depths = depths
        for a, info in job.store.arrays.items():
            job.shapes[a] = info.shape
        job.exchange_buffers()
        return {"hashes": {a: job.hash(a) for a in sorted(job.store.arrays)}, "stats": stats}
    finally:
        job.close()


def replay_rank(rank, world):
    """Repeated 2-D Laplace batches (DAG bytes) on an IPC job with the device
    double: replay counters, graph launches, final epochs and rounds."""
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice
    from paper_2512_19851_b200.programs import DagProgram, laplace_iteration_statements, laplace_program
    from paper_2512_19851_b200.wire import encode_dag

    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    prog = DagProgram()
    laplace_program(prog, 64, 0)
    job = ipc.IpcGpuJob(rank, world)
    try:
        for a in sorted(prog.shapes):
            job.create_array(prog.shapes[a])
        job.run(prog.dag)
        step = DagProgram()
        for a in sorted(prog.shapes):
            step.builder.declare_array(a, prog.shapes[a])
        laplace_iteration_statements(step, 0, 1, 10)
        blob = encode_dag(step.dag)
        for _ in range(5):
            job.run_bytes(blob)
        return {"replays": job.executor.replays,
                "graph_launches": sum(1 for e in job.dev.log if e[0] == "graph_launch"),
                "epochs": {a: job.store.local_epoch(a) for a in sorted(prog.shapes)},
                "rounds": dict(job.manager.rounds_started)}
    finally:
        job.close()


def chain_wait_rank(rank, world):
    """The flag operations around the est_tb launches of a 2-slab chain run
    (device double): a chain overwrites A, so right before its launch the
    stream must wait for the peers' PULLED of the round of A it just read."""
    import paper_2512_19851_b200.ipc as ipc
    from fakedev import FakeDevice
    from paper_2512_19851_b200 import temporal

    temporal.MIN_POINTS = 0
    ipc.Device = lambda device=0: FakeDevice(device, tag=f"r{rank}")
    prog, _ = _program("heat3d")
    job = ipc.IpcGpuJob(rank, world)
    try:
        for aid in sorted(prog.shapes):
            job.create_array(prog.shapes[aid])
        seqs = []
        for part in _split(prog.dag, 8):
            job.dev.log.clear()
            job.run(part)
            log = [e for e in job.dev.log if e[0] in ("launch", "flag_write", "flag_wait")]
            for k, e in enumerate(log):
                if e[0] == "launch" and e[2] == "est_tb":
                    seqs.append(log[k - 1][0] if k else None)
        return seqs
    finally:
        job.close()
