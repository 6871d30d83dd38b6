"""Tile decomposition and device-resident tile storage.

Decomposition (pkg/src/elastencil/grid.py:24-117): a job has ONE fixed set of
odf x initial_workers tiles on the most-square 2-D tile grid, mapped block-wise
row-major to workers. Rank-2 arrays split by that grid; rank-1 arrays split the
same tile count in linear tile order. Rank-3 arrays (new) split into slabs along
axis 0 in the same linear order: z-faces are contiguous, the
owner map / epochs / E-W halo directions carry over unchanged.

GpuTileStore mirrors TileStore (grid.py:130-230): per (tile, array) ONE padded
device buffer = interior + symmetric ghost frame of the array's current depth,
plus local/ghost generation epochs. HBM layout per buffer (C order, padded to
rank 3 as (1,1,n) / (1,ny,nx)):

    element (z, y, x) of the padded box lives at  base + xoff + z*pz + y*py + x

with xoff chosen so the first INTERIOR element of every row is 128-byte
aligned and py (row pitch) a multiple of 128 bytes; pz = py * (ny + 2*dy).
Ghost cells outside the global domain stay zero and are never read
(SPEC.md:202); growth reallocates, zero-fills and copies the interior on the
device (grid.py:164-184).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .pool import device_alloc, device_free
from ._lib import EstBox
from .device import COMPUTE, Device, PinnedBuffer
from .errors import IndivisibleShape, InvalidShape, OffsetExceedsTileWidth
from .wire import DTYPE_F32, DTYPE_F64

NP_DTYPE = {DTYPE_F64: np.float64, DTYPE_F32: np.float32}
ALIGN_BYTES = 128


def most_square_factors(n: int) -> tuple:
    r = max(d for d in range(1, int(n ** 0.5) + 1) if n % d == 0)
    return r, n // r


@dataclass(frozen=True)
class ArrayInfo:
    array: int
    shape: tuple
    dtype: int = DTYPE_F64

    @property
    def rank(self) -> int:
        return len(self.shape)


@dataclass(frozen=True)
class Decomposition:
    tile_grid: tuple
    odf: int
    initial_workers: int

    @property
    def n_tiles(self) -> int:
        return self.tile_grid[0] * self.tile_grid[1]

    def all_coords(self) -> list:
        return [divmod(k, self.tile_grid[1]) for k in range(self.n_tiles)]

    def linear(self, coords) -> int:
        return coords[0] * self.tile_grid[1] + coords[1]

    def coords_of(self, k: int) -> tuple:
        return divmod(k, self.tile_grid[1])

    def owner_map(self, workers: int) -> dict:
        """Contiguous row-major runs; leading workers take the extra tile."""
        n = self.n_tiles
        return {self.coords_of(k): w for w in range(workers)
                for k in range(w * n // workers, (w + 1) * n // workers)}

    def _linear_split(self, shape) -> bool:
        return len(shape) != 2

    def check_divisible(self, shape) -> None:
        if self._linear_split(shape):
            if shape[0] % self.n_tiles:
                raise IndivisibleShape(f"extent {shape[0]} not divisible by {self.n_tiles} tiles")
            return
        for e, c in zip(shape, self.tile_grid):
            if e % c:
                raise IndivisibleShape(f"extent {e} not divisible by {c} tiles")

    def tile_extents(self, shape) -> tuple:
        self.check_divisible(shape)
        if self._linear_split(shape):
            return (shape[0] // self.n_tiles,) + tuple(shape[1:])
        return (shape[0] // self.tile_grid[0], shape[1] // self.tile_grid[1])

    def tile_origin(self, shape, coords) -> tuple:
        ext = self.tile_extents(shape)
        if self._linear_split(shape):
            return (self.linear(coords) * ext[0],) + (0,) * (len(shape) - 1)
        return (coords[0] * ext[0], coords[1] * ext[1])


def decompose(shape, workers: int, odf: int) -> Decomposition:
    if workers < 1 or odf < 1:
        raise InvalidShape("workers and odf must be >= 1")
    d = Decomposition(most_square_factors(odf * workers), odf, workers)
    d.check_divisible(tuple(shape))
    return d


def pad3(t, fill=0) -> tuple:
    return (fill,) * (3 - len(t)) + tuple(t)


class TileBuffer:
    """One padded device buffer (see module docstring for the layout)."""

    __slots__ = ("dev", "ptr", "rank", "dtype", "elem", "ext", "depth", "xoff", "py", "pz",
                 "nz", "nbytes", "owned", "serial")
    _serials = __import__("itertools").count(1)

    def __init__(self, dev: Device, ext, depth, dtype: int, ptr: int | None = None, isolated: bool = False):
        self.dev = dev
        self.rank = len(ext)
        self.dtype = dtype
        self.elem = np.dtype(NP_DTYPE[dtype]).itemsize
        self.ext, self.depth = pad3(ext, 1), pad3(depth, 0)
        align = ALIGN_BYTES // self.elem
        dz, dy, dx = self.depth
        self.xoff = (align - dx % align) % align
        self.py = -(-(self.xoff + self.ext[2] + 2 * dx) // align) * align
        self.pz = self.py * (self.ext[1] + 2 * dy)
        self.nz = self.ext[0] + 2 * dz
        self.nbytes = self.pz * self.nz * self.elem
        self.owned = ptr is None
        self.ptr = device_alloc(dev, self.nbytes, isolated) if ptr is None else ptr
        self.serial = next(TileBuffer._serials)  # identifies this allocation in peer tables

    @staticmethod
    def pitches(ext, depth, dtype: int) -> tuple:
        """(xoff, py, pz) in elements of a buffer with this extent / depth."""
        elem = np.dtype(NP_DTYPE[dtype]).itemsize
        align = ALIGN_BYTES // elem
        e, d = pad3(ext, 1), pad3(depth, 0)
        xoff = (align - d[2] % align) % align
        py = -(-(xoff + e[2] + 2 * d[2]) // align) * align
        return xoff, py, py * (e[1] + 2 * d[1])

    @staticmethod
    def layout_bytes(ext, depth, dtype: int) -> int:
        elem = np.dtype(NP_DTYPE[dtype]).itemsize
        align = ALIGN_BYTES // elem
        e, d = pad3(ext, 1), pad3(depth, 0)
        xoff = (align - d[2] % align) % align
        py = -(-(xoff + e[2] + 2 * d[2]) // align) * align
        return py * (e[1] + 2 * d[1]) * (e[0] + 2 * d[0]) * elem

    def addr(self, z: int, y: int, x: int) -> int:
        """Address of padded-box element (z, y, x)."""
        return self.ptr + (self.xoff + z * self.pz + y * self.py + x) * self.elem

    def interior_addr(self, local) -> int:
        """Address of interior element `local` (rank-length, tile-local)."""
        z, y, x = pad3(local, 0)
        dz, dy, dx = self.depth
        return self.addr(z + dz, y + dy, x + dx)

    def box_to(self, dst_addr: int, dst_py: int, dst_pz: int, lo, hi, padded: bool = False) -> EstBox:
        """Copy descriptor for the box [lo, hi) (interior coords unless padded)."""
        lo3, hi3 = pad3(lo, 0), pad3(hi, 1)
        src = self.addr(*lo3) if padded else self.interior_addr(lo3)
        n = [b - a for a, b in zip(lo3, hi3)]
        return EstBox(src, dst_addr, self.py, self.pz, dst_py, dst_pz, n[2], n[1], n[0])

    def free(self) -> None:
        if self.ptr and self.owned:
            device_free(self.dev, self.ptr)
        self.ptr = 0


@dataclass
class GpuTile:
    coords: tuple
    buffers: dict = field(default_factory=dict)
    depths: dict = field(default_factory=dict)
    local_epoch: dict = field(default_factory=dict)
    ghost_epoch: dict = field(default_factory=dict)


class GpuTileStore:
    """All tiles one worker owns, resident in HBM (mirrors grid.py:130-230)."""

    def __init__(self, dev: Device, decomp: Decomposition, owned):
        self.dev = dev
        self.decomp = decomp
        self.tiles: dict = {c: GpuTile(c) for c in owned}
        self.arrays: dict = {}
        self.version = 0  # bumped whenever any buffer is (re)allocated or dropped
        self._epochs: dict = {}  # array -> local epoch (also valid with no tiles)
        self._ghosts: dict = {}
        self.phys_depth: dict = {}  # array -> allocated ghost frame (>= logical; also with no tiles)
        self.logical_depth: dict = {}  # array -> job-wide logical ghost depth (also with no tiles)
        self.twins: dict = {}       # (coords, array) -> twin TileBuffer of a temporal chain's input
        self.twin_sig: dict = {}    # array -> (info, frame, store version) the twins were made for

    # -- creation / capacity ------------------------------------------------
    def create_array(self, info: ArrayInfo) -> None:
        if info.rank not in (1, 2, 3) or any(e <= 0 for e in info.shape):
            raise InvalidShape(f"bad shape {info.shape}")
        if info.dtype not in NP_DTYPE:
            raise InvalidShape(f"bad dtype {info.dtype}")
        self.decomp.check_divisible(info.shape)
        self.arrays[info.array] = info
        self.version += 1
        self._epochs[info.array] = 0
        self._ghosts[info.array] = 0
        ext = self.decomp.tile_extents(info.shape)
        zero = (0,) * info.rank
        for tile in self.tiles.values():
            tile.buffers[info.array] = TileBuffer(self.dev, ext, zero, info.dtype)
            tile.depths[info.array] = zero
            tile.local_epoch[info.array] = 0
            tile.ghost_epoch[info.array] = 0

    def check_depth_fits(self, array: int, depth) -> None:
        ext = self.decomp.tile_extents(self.arrays[array].shape)
        for d, e in zip(depth, ext):
            if d >= e:
                raise OffsetExceedsTileWidth(f"ghost depth {d} >= tile width {e} for array {array}")

    def ensure_ghost_capacity(self, array: int, depth, phys=None) -> bool:
        """Grow (never shrink) the ghost frame on the device; True if the
        LOGICAL depth (the reference's, grid.py:164-184) grew on any tile.

        `phys` (>= depth) is the frame actually allocated: rank-3 slabs of a
        multi-tile job keep K*rz planes of ghost so a K-sweep temporal chain
        can run on one halo round (executor.temporal_schedule). A purely
        physical growth keeps the ghost contents (the whole old padded box is
        copied), so no epoch changes; a logical growth copies the interior and
        the caller bumps the local epoch as the reference does."""
        self.check_depth_fits(array, depth)
        rank = self.arrays[array].rank
        # the job-wide logical depth: a worker that owns no tile sees the same
        # growth (and bumps its epochs with everyone else)
        old_logical = self.logical_depth.get(array, (0,) * rank)
        self.logical_depth[array] = tuple(max(a, b) for a, b in zip(old_logical, depth))
        phys = tuple(max(a, b) for a, b in zip(depth, phys if phys is not None else depth))
        self.phys_depth[array] = tuple(max(a, b) for a, b in zip(self.phys_depth.get(array, phys), phys))
        grew = grew_buf = False
        for tile in self.tiles.values():
            old = tile.depths[array]
            new = tuple(max(a, b) for a, b in zip(old, depth))
            src = tile.buffers[array]
            have = src.depth[3 - rank:]
            want = tuple(max(a, b) for a, b in zip(have, phys))
            if new == old and want == tuple(have):
                continue
            ext = src.ext[3 - src.rank:]
            dst = TileBuffer(self.dev, ext, want, src.dtype)
            if new == old:
                # physical only: carry the valid ghost frame along
                lo = tuple(h - o for h, o in zip(want, have))
                whole = tuple(e + 2 * o for e, o in zip(ext, have))
                self.dev.copy_box(src.box_to(dst.addr(*pad3(lo, 0)), dst.py, dst.pz,
                                             (0,) * src.rank, whole, padded=True), src.elem, COMPUTE)
            else:
                self.dev.copy_box(src.box_to(dst.interior_addr((0,) * src.rank), dst.py, dst.pz,
                                             (0,) * src.rank, ext), src.elem, COMPUTE)
                grew = True
            src.free()  # est_free synchronises the lanes before releasing
            tile.buffers[array] = dst
            tile.depths[array] = new
            grew_buf = True
        if grew_buf:
            self.version += 1
        if not self.tiles:
            return self.logical_depth[array] != old_logical
        return grew

    def fetch_dtype(self, array: int):
        return NP_DTYPE[self.arrays[array].dtype]

    # -- epochs (grid.py:192-206) -------------------------------------------
    # Epochs are uniform over a worker's tiles; the store also keeps them per
    # array so a worker that owns no tile (after a shrink-by-migration, or
    # expanded past the initial owners) keeps counting with everyone else and
    # takes part in every halo round - the transport sequences rounds globally.
    def bump_local_epoch(self, array: int, by: int = 1) -> None:
        for tile in self.tiles.values():
            tile.local_epoch[array] += by
        self._epochs[array] = self._epochs.get(array, 0) + by

    def set_epochs(self, array: int, local: int, ghost: int) -> None:
        for tile in self.tiles.values():
            tile.local_epoch[array] = local
            tile.ghost_epoch[array] = ghost
        self._epochs[array] = local
        self._ghosts[array] = ghost

    def set_ghost_epoch(self, array: int, ghost: int) -> None:
        for tile in self.tiles.values():
            tile.ghost_epoch[array] = ghost
        self._ghosts[array] = ghost

    def _uniform(self, attr: str, array: int) -> int:
        vals = {getattr(t, attr)[array] for t in self.tiles.values()}
        if len(vals) > 1:
            raise AssertionError(f"non-uniform {attr} for array {array}")
        if vals:
            return vals.pop()
        return (self._epochs if attr == "local_epoch" else self._ghosts).get(array, 0)

    def local_epoch(self, array: int) -> int:
        return self._uniform("local_epoch", array)

    def ghost_epoch(self, array: int) -> int:
        return self._uniform("ghost_epoch", array)

    # -- host <-> device ----------------------------------------------------
    def _pieces(self, array: int, bounds):
        info = self.arrays[array]
        ext = self.decomp.tile_extents(info.shape)
        for coords in sorted(self.tiles):
            origin = self.decomp.tile_origin(info.shape, coords)
            piece = []
            for (lo, hi), o, e in zip(bounds, origin, ext):
                a, b = max(lo, o), min(hi, o + e)
                if a >= b:
                    piece = None
                    break
                piece.append((a, b))
            if piece is not None:
                yield coords, origin, tuple(piece)

    def gather_slice_pieces(self, array: int, bounds, pinned: PinnedBuffer | None = None):
        """(global piece bounds, C-order block) per owned tile (grid.py:208-230).

        One pitched D2H copy per piece into pinned staging, then a host view.
        """
        info = self.arrays[array]
        dt = NP_DTYPE[info.dtype]
        pieces = list(self._pieces(array, bounds))
        total = sum(int(np.prod([b - a for a, b in p])) for _, _, p in pieces)
        if not pieces:
            return []
        own = pinned is None or pinned.nbytes < total * np.dtype(dt).itemsize
        stage = PinnedBuffer(max(1, total) * np.dtype(dt).itemsize) if own else pinned
        off = 0
        out = []
        for coords, origin, piece in pieces:
            buf = self.tiles[coords].buffers[array]
            n = [b - a for a, b in piece]
            lo = [a - o for (a, _), o in zip(piece, origin)]
            hi = [l + k for l, k in zip(lo, n)]
            n3 = pad3(n, 1)
            self.dev.copy_box(buf.box_to(stage.ptr + off * buf.elem, n3[2], n3[1] * n3[2], lo, hi),
                              buf.elem, COMPUTE)
            out.append((piece, off, n))
            off += int(np.prod(n))
        self.dev.stream_sync(COMPUTE)
        flat = stage.view(dt, total).copy()
        if own:
            stage.close()
        return [(piece, flat[o:o + int(np.prod(n))].reshape(n)) for piece, o, n in out]

    def fetch(self, array: int, bounds=None) -> np.ndarray:
        info = self.arrays[array]
        bounds = tuple(bounds) if bounds is not None else tuple((0, e) for e in info.shape)
        res = np.zeros([b - a for a, b in bounds], dtype=NP_DTYPE[info.dtype])
        for piece, block in self.gather_slice_pieces(array, bounds):
            res[tuple(slice(a - lo, b - lo) for (a, b), (lo, _) in zip(piece, bounds))] = block
        return res

    def upload_interior(self, coords, array: int, data: np.ndarray) -> None:
        """Host -> interior of one tile (used by restore/adopt and tests)."""
        buf = self.tiles[coords].buffers[array]
        data = np.ascontiguousarray(data, dtype=NP_DTYPE[buf.dtype])
        n3 = pad3(data.shape, 1)
        stage = PinnedBuffer(max(1, data.nbytes))
        stage.view(data.dtype, data.size)[:] = data.reshape(-1)
        box = EstBox(stage.ptr, buf.interior_addr((0,) * buf.rank), n3[2], n3[1] * n3[2],
                     buf.py, buf.pz, n3[2], n3[1], n3[0])
        self.dev.copy_box(box, buf.elem, COMPUTE)
        self.dev.stream_sync(COMPUTE)
        stage.close()

    # -- checkpoint blobs (grid.py:236-277) ------------------------------------
    def checkpoint_blob(self, coords, array: int) -> bytes:
        """checkpoint_blob (grid.py:239-250): header + the tile interior, little
        endian, ghost frame dropped; D2H through pinned staging. Byte-identical
        to the reference for float64 (tests/golden/blobs.json)."""
        info = self.arrays[array]
        tile = self.tiles[tuple(coords)]
        origin = self.decomp.tile_origin(info.shape, tuple(coords))
        ext = self.decomp.tile_extents(info.shape)
        pieces = self.gather_slice_pieces(array, tuple((o, o + e) for o, e in zip(origin, ext)))
        (piece, block), = [pb for pb in pieces if tuple(a for a, _ in pb[0]) == tuple(origin)]
        header = blob_header(array, tuple(coords), ext, tile.depths[array], tile.local_epoch[array])
        return header + np.ascontiguousarray(block).astype(block.dtype.newbyteorder("<"), copy=False).tobytes()

    def hash(self, array: int) -> int:
        """Sum mod 2^64 of the position-keyed hashes of every owned tile's
        interior (est_hash_box): equal for equal arrays under ANY
        decomposition, so the partial sums of all workers add up to the
        whole array's hash."""
        info = self.arrays[array]
        g3 = pad3(info.shape, 1)
        total = 0
        for coords in sorted(self.tiles):
            buf = self.tiles[coords].buffers[array]
            ext = self.decomp.tile_extents(info.shape)
            box = buf.box_to(0, 0, 0, (0,) * info.rank, ext)
            org = pad3(self.decomp.tile_origin(info.shape, coords), 0)
            total = (total + self.dev.hash_box(box, org, g3, buf.elem)) % (1 << 64)
        return total

    def adopt_blob(self, blob: bytes) -> tuple:
        """adopt_blob (grid.py:264-277): install a checkpointed tile payload.

        As in the reference the tile is created if this worker does not own it
        yet (`tiles.setdefault`), its buffer is (re)allocated zeroed at the
        BLOB's ghost depth, and the tile's epochs come from the blob; the
        store-level epoch counters follow (every blob of one checkpoint carries
        the same epoch; the adopting path bumps them uniformly afterwards).
        -> (array, coords, epoch)."""
        array, coords, ext, depth, epoch, hs = parse_blob_header(blob)
        info = self.arrays[array]
        if tuple(ext) != tuple(self.decomp.tile_extents(info.shape)):
            raise InvalidShape(f"blob extent {ext} does not match array {array}'s tiles")
        self.check_depth_fits(array, depth)
        coords = tuple(coords)
        tile = self.tiles.setdefault(coords, GpuTile(coords))
        old = tile.buffers.get(array)
        if old is None or tuple(old.depth[3 - old.rank:]) != tuple(depth):
            if old is not None:
                old.free()
            tile.buffers[array] = TileBuffer(self.dev, ext, depth, info.dtype)
            self.version += 1
        buf = tile.buffers[array]
        self.dev.memset_zero(buf.ptr, buf.nbytes, COMPUTE)
        tile.depths[array] = tuple(depth)
        data = np.frombuffer(blob, dtype=np.dtype(NP_DTYPE[info.dtype]).newbyteorder("<"),
                             offset=hs).reshape(ext)
        self.upload_interior(coords, array, data)
        tile.local_epoch[array] = tile.ghost_epoch[array] = epoch
        self._epochs[array] = self._ghosts[array] = epoch
        return array, coords, epoch

    def release(self) -> None:
        for tile in self.tiles.values():
            for buf in tile.buffers.values():
                buf.free()
            tile.buffers.clear()
        for buf in self.twins.values():
            buf.free()
        self.twins.clear()


# --------------------------------------------------------------------------
# checkpoint blob header (grid.py:236-277; PROTOCOL.md "Checkpoint payload blob")
# rank-3 tiles use the additive 3-D header tag (rank byte = 3, extra extent/depth)

BLOB_HEADER = struct.Struct("<IHHBQQQQQ")
BLOB_HEADER3 = struct.Struct("<IHHBQQQQQQQ")


def blob_header(array: int, coords, ext, depth, epoch: int) -> bytes:
    if len(ext) == 3:
        return BLOB_HEADER3.pack(array, coords[0], coords[1], 3, ext[0], ext[1], depth[0],
                                 depth[1], epoch, ext[2], depth[2])
    e1 = ext[1] if len(ext) > 1 else 0
    d1 = depth[1] if len(depth) > 1 else 0
    return BLOB_HEADER.pack(array, coords[0], coords[1], len(ext), ext[0], e1, depth[0], d1, epoch)


def parse_blob_header(blob: bytes):
    """-> (array, coords, ext, depth, epoch, header size)."""
    array, tr, tc, rank, e0, e1, d0, d1, epoch = BLOB_HEADER.unpack_from(blob, 0)
    if rank == 3:
        _, _, _, _, e0, e1, d0, d1, epoch, e2, d2 = BLOB_HEADER3.unpack_from(blob, 0)
        return array, (tr, tc), (e0, e1, e2), (d0, d1, d2), epoch, BLOB_HEADER3.size
    ext = (e0,) if rank == 1 else (e0, e1)
    depth = (d0,) if rank == 1 else (d0, d1)
    return array, (tr, tc), ext, depth, epoch, BLOB_HEADER.size
