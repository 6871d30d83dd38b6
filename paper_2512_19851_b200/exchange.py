"""Generation-epoch-gated halo exchange on device memory.

Round semantics follow pkg/src/elastencil/exchange.py:106-293 exactly: a round
is keyed (array, epoch), derived identically on every worker from the shared
DAG; every owned tile receives the depth-wide strip from each existing
neighbour (8 directions with corners for rank 2, E/W in linear tile order for
ranks 1 and 3); the receiving side writes the ghost region on the side the
strip came from. Round / net-message accounting matches the reference
(`rounds_started`, `net_messages` = strips crossing a worker boundary).

Data movement is B200-native instead of pack -> bytes -> TCP -> unpack:

* co-located neighbours (odf > 1, or several tiles after a shrink): every
  strip of the round is one descriptor of ONE batched device copy kernel
  (interior strip of the neighbour -> ghost region of this tile), on the
  compute stream, so it is ordered after the producing node and before the
  consumer without any host synchronisation;
* remote neighbours: the `transport` (transport.py) pulls the neighbour's
  strip straight out of its IPC-mapped HBM buffer (NVLink P2P on a multi-GPU
  box) into the ghost region, gated by the neighbour's ready event.

Because the copies are stream-ordered, a round is complete for the host as
soon as it is enqueued; `round_complete` / `ghost_generation` keep the
reference API for the executor.
"""

from __future__ import annotations

from ._lib import EstBox
from .codegen import ELEM

N, NE, E, SE, S, SW, W, NW = range(8)
VEC_2D = {N: (-1, 0), NE: (-1, 1), E: (0, 1), SE: (1, 1),
          S: (1, 0), SW: (1, -1), W: (0, -1), NW: (-1, -1)}
_OPP = {N: S, S: N, E: W, W: E, NE: SW, SW: NE, NW: SE, SE: NW}


def opposite(direction: int) -> int:
    return _OPP[direction]


def linear_split(rank: int) -> bool:
    return rank != 2


def directions_for(depth) -> list:
    """Directions carrying a non-empty strip (exchange.py:42-50; rank 3 = slabs)."""
    if linear_split(len(depth)):
        return [E, W] if depth[0] > 0 else []
    return sorted(c for c, v in VEC_2D.items() if all(depth[a] > 0 for a in range(2) if v[a]))


def direction_vec(rank: int, direction: int) -> tuple:
    if linear_split(rank):
        step = 1 if direction == E else -1
        return (step,) + (0,) * (rank - 1)
    return VEC_2D[direction]


def strip_box(ext, depth, vec) -> tuple:
    """Interior-coordinate box of the border strip facing `vec` (_pack_sel)."""
    lo, hi = [], []
    for e, d, v in zip(ext, depth, vec):
        lo.append(0 if v <= 0 else e - d)
        hi.append(d if v < 0 else e)
    return tuple(lo), tuple(hi)


def ghost_box(ext, depth, vec) -> tuple:
    """Padded-coordinate box of the ghost region on side `vec` (_ghost_sel)."""
    lo, hi = [], []
    for e, d, v in zip(ext, depth, vec):
        if v < 0:
            lo.append(0), hi.append(d)
        elif v > 0:
            lo.append(d + e), hi.append(2 * d + e)
        else:
            lo.append(d), hi.append(d + e)
    return tuple(lo), tuple(hi)


def neighbour(decomp, rank: int, coords, direction: int):
    if linear_split(rank):
        k = decomp.linear(coords) + direction_vec(rank, direction)[0]
        return decomp.coords_of(k) if 0 <= k < decomp.n_tiles else None
    vi, vj = VEC_2D[direction]
    i, j = coords[0] + vi, coords[1] + vj
    tr, tc = decomp.tile_grid
    return (i, j) if 0 <= i < tr and 0 <= j < tc else None


def strip_copy(src_buf, dst_buf, direction: int, src_addr_override: int | None = None) -> EstBox:
    """Descriptor moving the neighbour's facing strip into dst's ghost side `direction`.

    `direction` points from the destination tile towards the source tile.
    """
    rank = dst_buf.rank
    ext = dst_buf.ext[3 - rank:]
    depth = dst_buf.depth[3 - rank:]
    vec = direction_vec(rank, direction)
    opp = tuple(-v for v in vec)
    s_lo, s_hi = strip_box(ext, depth, opp)
    g_lo, _ = ghost_box(ext, depth, vec)
    from .tiles import pad3

    n = pad3([b - a for a, b in zip(s_lo, s_hi)], 1)
    if src_addr_override is None:
        src = src_buf.interior_addr(s_lo)
    else:  # peer-mapped copy of src_buf's layout
        z, y, x = pad3(s_lo, 0)
        dz, dy, dx = src_buf.depth
        src = src_addr_override + (src_buf.xoff + (z + dz) * src_buf.pz + (y + dy) * src_buf.py
                                   + (x + dx)) * src_buf.elem
    dst = dst_buf.addr(*pad3(g_lo, 0))
    return EstBox(src, dst, src_buf.py, src_buf.pz, dst_buf.py, dst_buf.pz, n[2], n[1], n[0])


class GpuExchangeManager:
    """Per-worker round bookkeeping + device strip movement."""

    def __init__(self, store, worker_id: int, owner_map: dict, transport=None):
        self.store = store
        self.worker_id = worker_id
        self.owner_map = owner_map
        self.transport = transport
        self.completed: dict = {}
        self.rounds_started: dict = {}
        self.net_messages = 0
        self.active: dict = {}
        self.buffered: dict = {}
        self.stale_dropped = 0
        self.copy_launches = 0
        self._geometry: dict = {}  # (array, layout version, owner map) -> boxes
        self.pending: dict = {}    # array -> posted-but-unpulled round token

    def _round_geometry(self, array: int, rank: int, twin: bool = False) -> tuple:
        """Co-located strip copies and remote (tile, dir, neighbour, owner) list.
        `twin`: the array's values live in the temporal chains' twin buffers
        (mid-run), so the strips move between twins."""
        depth = self._depth(array)
        local_boxes, remote = [], []

        def buf(c):
            return self.store.twins[(c, array)] if twin else self.store.tiles[c].buffers[array]

        if depth is not None:
            for coords in sorted(self.store.tiles):
                for d in directions_for(depth):
                    nb = neighbour(self.store.decomp, rank, coords, d)
                    if nb is None:
                        continue
                    owner = self.owner_map[nb]
                    if owner == self.worker_id:
                        local_boxes.append(strip_copy(buf(nb), buf(coords), d))
                    else:
                        remote.append((coords, d, nb, owner))
        return local_boxes, remote

    def _depth(self, array: int):
        for tile in self.store.tiles.values():
            return tile.depths[array]
        return None

    def finish_pending(self, array: int | None = None, overlap: bool = False) -> list:
        """Enqueue deferred peer pulls (all, or one array's); returns their round ids."""
        done = []
        for a in ([array] if array is not None else sorted(self.pending)):
            token = self.pending.pop(a, None)
            if token is not None:
                self.transport.finish(token, overlap=overlap)
                done.append(token[1])
        return done

    def ensure_round(self, array: int, epoch: int, defer: bool = False, twin: bool = False,
                     virtual: bool = False, refresh: bool = False) -> bool:
        """Start round (array, epoch); returns True (completion is stream-ordered).

        With `defer` (multi-worker, push-plan rounds) the peer pull is posted
        but not enqueued; the executor finishes it right before / overlapped
        with the next node that reads the array (`finish_pending`).
        `virtual`: the round's ghosts are produced inside a temporal chain
        (nothing moves; counted exactly as the reference counts the round).
        `refresh`: re-run the data movement of an already counted (virtual)
        round, uncounted. Every worker makes the same choice for every round
        (they derive from the DAG), so transport sequences stay aligned."""
        if not refresh and self.completed.get(array, -1) >= epoch:
            return True
        if self.pending:
            self.finish_pending()  # keep at most one round in flight on the host
        info = self.store.arrays[array]
        ck = (array, self.store.version, id(self.owner_map), twin)
        hit = self._geometry.get(ck)
        if hit is None:
            hit = self._round_geometry(array, info.rank, twin)
            if len(self._geometry) > 1024:
                self._geometry.clear()
            self._geometry[ck] = hit
        local_boxes, remote = hit
        if remote:
            if self.transport is None:
                raise RuntimeError("remote neighbours but no transport configured")
            if not refresh:
                self.net_messages += len(remote)
        if virtual:
            pass
        elif self.transport is not None:
            # every worker takes part in every round, owning tiles or not, so the
            # transport's per-round sequencing stays globally aligned
            if defer:
                self.pending[array] = self.transport.post(array, epoch, remote, local_boxes, twin)
            else:
                self.transport.exchange(array, epoch, remote, local_boxes, twin)
        elif local_boxes:
            self.store.dev.copy_boxes(local_boxes, ELEM[info.dtype])
            self.copy_launches += 1
        if not refresh:
            self.rounds_started[array] = self.rounds_started.get(array, 0) + 1
        self.completed[array] = epoch
        self.store.set_ghost_epoch(array, epoch)
        return True

    def round_complete(self, array: int, epoch: int) -> bool:
        return self.completed.get(array, -1) >= epoch

    def ghost_generation(self, array: int) -> int:
        return self.completed.get(array, 0)

    def snapshot_stats(self) -> dict:
        return {"rounds": dict(self.rounds_started), "net_messages": self.net_messages,
                "stale_dropped": self.stale_dropped}
