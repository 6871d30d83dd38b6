"""The "stream" skeleton: 2.5-D streaming with TMA-staged shared-memory rings.

For rank-3 single-statement nodes (the 3-D heat/Jacobi sweeps that dominate
the BASELINE configs) every input element must cross HBM once and every
output once (16 B per update in fp64). Rank-2 nodes run the same pipeline on
a (1, Y, X) view with one tile per work item. The generated kernel (ws2):

* work item = a BX x BY column of the output box over ZCHUNK planes (rank 2:
  one tile); non-persistent grid for rank 3, persistent for rank 2;
* a dedicated producer warp streams each input slot's planes (tile + halo)
  with ONE `cp.async.bulk.tensor.3d` (TMA) per plane into a ring of
  2*rz+1+PREFETCH shared-memory stages, gated by FULL (expect_tx) / EMPTY
  (one arrive per compute warp) mbarriers. The TMA box starts at a 16-byte
  aligned x coordinate (a hardware requirement found with
  scripts/probes/tma_probe.cu; the sub-16 B shift goes into the shared-memory
  column index);
* each compute thread owns BY/TY CONSECUTIVE output rows of one column: its
  column of every slot with pure-z / centre operands lives in registers
  (2rz+1 planes, rotated by unrolling the plane loop), in-plane (dy, 0)
  operands of its own rows come from those registers, everything else from
  the ring; the postorder plan is emitted by codegen._emit_expr (one rounded
  IEEE op per plan instruction) and stored with coalesced st.global;
* ring stages and phases are counters; fill counters run across items, so
  mbarrier phases never need re-initialisation.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

from .codegen import CTYPE, ELEM, NodeSig, StmtSig, _emit_expr, slot_radius
from .wire import DTYPE_F64

MIN_ZCHUNK = 32
STORE_HINT = os.environ.get("EST_STREAM_STHINT", "0") == "1"  # evict_first L2 policy on output stores
MAX_RADIUS = 4
SMEM_BUDGET = 220 * 1024
SMEM_PER_SM = 228 * 1024


@dataclass(frozen=True)
class StreamCfg:
    """Tile / pipeline shape. Defaults = best of the measured sweeps
    (profiles/r1_stream_sweep.md): 128x16 tiles, 4 consecutive rows per
    thread (source_ws2), warp-specialised TMA producer, register z-columns."""

    bx: int = 128           # output columns per CTA
    by: int = 16            # output rows per CTA
    ty: int = 4             # thread rows; each thread computes by // ty rows
    prefetch: int = 3       # planes in flight beyond the stencil's z window
    persistent: bool = False
    zchunk: int = 128       # planes per item when not persistent
    l2promo: int = 2        # TMA L2 promotion: 0 none, 1 64B, 2 128B, 3 256B
    ws: bool = True         # warp-specialised: dedicated TMA producer warp, full/empty mbarriers
    zreg: bool = True       # (ws only) pure-z offsets of the thread's own column from registers
    v2: bool = True         # (ws only) source_ws2: consecutive rows, register y-neighbours, unrolled z


def _env_cfg() -> StreamCfg:
    e = os.environ.get
    d = StreamCfg()
    return StreamCfg(bx=int(e("EST_STREAM_BX", d.bx)), by=int(e("EST_STREAM_BY", d.by)),
                     ty=int(e("EST_STREAM_TY", d.ty)), prefetch=int(e("EST_STREAM_PREFETCH", d.prefetch)),
                     persistent=e("EST_STREAM_PERSISTENT", "0") == "1",
                     zchunk=int(e("EST_STREAM_ZCHUNK", d.zchunk)),
                     l2promo=int(e("EST_STREAM_L2PROMO", d.l2promo)),
                     ws=e("EST_STREAM_WS", "1" if d.ws else "0") == "1",
                     zreg=e("EST_STREAM_ZREG", "1" if d.zreg else "0") == "1",
                     v2=e("EST_STREAM_V2", "1" if d.v2 else "0") == "1")


DEFAULT = _env_cfg()
DEFAULT_2D = StreamCfg(bx=int(os.environ.get("EST_STREAM2D_BX", 128)),
                       by=int(os.environ.get("EST_STREAM2D_BY", 48)),
                       ty=int(os.environ.get("EST_STREAM2D_TY", 4)),
                       prefetch=int(os.environ.get("EST_STREAM2D_PREFETCH", 2)),
                       persistent=True, ws=True, zreg=False, l2promo=2,
                       v2=os.environ.get("EST_STREAM2D_V2", "1") == "1")


def layout(st: StmtSig, dtype: int, cfg: StreamCfg):
    """Per slot: ((rz, ry, rx), (w, h), stages, plane_bytes, offset); data bytes; total."""
    elem = ELEM[dtype]
    q = 16 // elem
    rad = slot_radius(st)
    slots, off = [], 0
    for s in range(st.arity):
        rz, ry, rx = rad.get(s, (0, 0, 0))
        w = -(-(cfg.bx + 2 * rx + q - 1) // q) * q   # room for the 16-byte alignment shift
        h = cfg.by + 2 * ry
        stages = 2 * rz + 1 + cfg.prefetch
        plane = -(-(w * h * elem) // 1024) * 1024
        slots.append(((rz, ry, rx), (w, h), stages, plane, off))
        off += stages * plane
    n_bars = sum(s[2] for s in slots) * (2 if cfg.ws else 1)
    return slots, off, off + 8 * n_bars + 1024


# rank-2 boxes below this many points (e.g. the 1024^2 C1 grid) use smaller
# tiles so the grid still covers every SM (64x16, 8 rows per thread: C1 sweep,
# profiles/r1s2_c1_small_tiles.txt)
SMALL_2D_POINTS = 8 << 20
DEFAULT_2D_SMALL = StreamCfg(bx=int(os.environ.get("EST_STREAM2DS_BX", 64)),
                             by=int(os.environ.get("EST_STREAM2DS_BY", 16)),
                             ty=int(os.environ.get("EST_STREAM2DS_TY", 2)),
                             prefetch=int(os.environ.get("EST_STREAM2DS_PREFETCH", 2)),
                             persistent=os.environ.get("EST_STREAM2DS_PERSISTENT", "1") == "1",
                             ws=True, zreg=False, l2promo=2, v2=True)


def fallback_cfgs(rank: int, small: bool = False, dtype: int = DTYPE_F64) -> list:
    """Configurations to try in order: the default, then shorter tiles, so
    multi-input statements whose rings do not fit the default tile's shared
    memory (e.g. cavity flow's 3-input momentum updates) still stream."""
    first = cfg_for(rank, small, dtype)
    out = [first]
    for by in (16, 8, 4):
        if by < first.by:
            out.append(StreamCfg(bx=first.bx, by=by, ty=min(first.ty, by), prefetch=min(first.prefetch, 2),
                                 persistent=first.persistent, zchunk=first.zchunk, l2promo=first.l2promo,
                                 ws=True, zreg=first.zreg, v2=first.v2))
    return out


# fp64 rank-2 tiles: 24 rows per thread (ty 2) beats the fp32 wave's 12
# (Laplace 16384^2 fp64: 0.80 -> 0.90 of measured HBM; the fp32 wave falls
# from 0.99 to 0.76 with ty 2 - profiles/r1s2_laplace16k_f64_sweep.txt)
DEFAULT_2D_F64 = StreamCfg(bx=DEFAULT_2D.bx, by=DEFAULT_2D.by,
                           ty=int(os.environ.get("EST_STREAM2D_TY_F64", 2)),
                           prefetch=DEFAULT_2D.prefetch, persistent=True, ws=True, zreg=False,
                           l2promo=2, v2=DEFAULT_2D.v2)


def cfg_for(rank: int, small: bool = False, dtype: int = DTYPE_F64) -> StreamCfg:
    """Rank-3 nodes stream along z; rank-2 nodes run the same warp-specialised
    TMA pipeline on a (1, Y, X) view: every item is one (BY+2ry) x (BX+2rx)
    tile, and the persistent grid lets the producer prefetch the NEXT items'
    tiles while the current one is computed."""
    if rank == 3:
        return DEFAULT
    if small:
        return DEFAULT_2D_SMALL
    return DEFAULT_2D_F64 if dtype == DTYPE_F64 else DEFAULT_2D


def eligible(stmts, rank: int, dtype: int = DTYPE_F64, cfg: StreamCfg | None = None) -> bool:
    cfg = cfg or cfg_for(rank, False, dtype)
    if rank not in (2, 3) or len(stmts) != 1 or stmts[0].arity == 0:
        return False
    if rank == 2 and not cfg.ws:
        return False
    rad = slot_radius(stmts[0]).values()
    if any(max(r) > MAX_RADIUS for r in rad):
        return False
    if any((cfg.bx + 2 * r[2] + 2) > 256 or (cfg.by + 2 * r[1]) > 256 for r in rad):
        return False  # TMA box extents are limited to 256 elements
    return layout(stmts[0], dtype, cfg)[2] <= SMEM_BUDGET


def threads_per_cta(cfg: StreamCfg) -> int:
    return cfg.bx * cfg.ty + (32 if cfg.ws else 0)


def blocks_per_sm(smem: int, cfg: StreamCfg) -> int:
    return max(1, min(SMEM_PER_SM // (smem + 1024), 2048 // threads_per_cta(cfg)))


_PTX_HELPERS = r"""
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n)); }
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  // bounded wait: a pipeline bug must fault (trap -> error at the next sync)
  // instead of hanging the GPU
  long long t0 = 0;
  #pragma unroll 1
  for (int spin = 0;; ++spin) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    if (ok) return;
    if (spin == 4096) t0 = clock64();
    else if (spin > 4096 && (spin & 4095) == 0 && clock64() - t0 > 40000000000LL) __trap();
  }
}
__device__ __forceinline__ void tma_load3(void* dst, const void* tm, int x, int y, int z,
                                          unsigned long long* b) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(smem_u32(dst)), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b))
               : "memory"); }
"""


def source(sig: NodeSig, rank: int, cfg: StreamCfg | None = None) -> tuple:
    """-> (source, kernel name, block, smem, items per launch, geometry).

    Only the warp-specialised ws2 pipeline is generated; the earlier
    variants (CTA-barrier rings, one row per thread, lockstep persistent
    grids) are recorded with their measurements in profiles/r1_stream_sweep.md."""
    cfg = cfg or cfg_for(rank, False, sig.dtype)
    if not (cfg.ws and cfg.v2):
        raise ValueError("only the warp-specialised ws2 stream skeleton is generated")
    return source_ws2(sig, rank, cfg)


def source_ws2(sig: NodeSig, rank: int, cfg: StreamCfg) -> tuple:
    """Lower-instruction warp-specialised variant (same TMA rings, barriers
    and work items as source_ws):

    * each thread owns RPT = BY/TY CONSECUTIVE output rows of one column, so
      in-plane (dy, 0) operands of its own rows come from registers;
    * the thread's column of every slot with pure-z / centre operands lives in
      registers (2rz+1 planes) and the plane loop is unrolled 2rz+1 times so
      the window rotates by renaming instead of moves;
    * ring stages / phases are counters, output rows are advanced pointers.
    Parity: the expression is emitted by codegen._emit_expr exactly as in the
    other skeletons (one rounded IEEE op per plan instruction)."""
    BX, BY, TY = cfg.bx, cfg.by, cfg.ty
    st = sig.stmts[0]
    T = CTYPE[sig.dtype]
    elem = ELEM[sig.dtype]
    q = 16 // elem
    slots, data_bytes, smem = layout(st, sig.dtype, cfg)
    n_in = st.arity
    RPT = BY // TY
    CT = BX * TY
    NW = CT // 32
    assert CT % 32 == 0 and BY % TY == 0
    loads = [ins for ins in st.instructions if ins[0] == "load"]
    regs = {s for s in range(n_in) if any(i[1] == s and i[2][1] == 0 and i[2][2] == 0 for i in loads)}
    Z = {s: 2 * slots[s][0][0] + 1 for s in range(n_in)}
    U = 1
    for s in regs:
        U = U * Z[s] // __import__("math").gcd(U, Z[s])
    L = []
    a = L.append
    a(f'// generated by paper_2512_19851_b200/stream.py — skeleton "stream" (TMA 2.5-D, ws2) {cfg}')
    a(f"typedef {T} T;")
    a("struct __align__(64) Tmap { unsigned long long w[16]; };")
    a(f"struct __align__(64) Params {{ Tmap tm[{n_in}];")
    a("  unsigned long long out; long long opy, opz, nx, ny, nz, zc, nbx, nby, nzc;")
    a(f"  long long cx0[{n_in}], cy0[{n_in}], cz0[{n_in}]; }};")
    L.append(_PTX_HELPERS)
    a("__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {")
    a("  asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(smem_u32(b)) : \"memory\"); }")
    a("__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {")
    a("  unsigned ok; asm volatile(\"{\\n .reg .pred p;\\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\\n\"")
    a("  \" selp.u32 %0, 1, 0, p;\\n}\" : \"=r\"(ok) : \"r\"(smem_u32(b)), \"r\"(parity) : \"memory\"); return ok; }")
    a("__device__ __forceinline__ void mbar_wait2(unsigned long long* b, unsigned parity) {")
    a("  if (!mbar_try(b, parity)) mbar_wait(b, parity); }  // fast first probe, bounded slow path")
    a(f'extern "C" __global__ void __launch_bounds__({CT + 32})')
    a("est_stream(const __grid_constant__ Params p) {")
    a("  extern __shared__ __align__(1024) unsigned char smem[];")
    a(f"  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + {data_bytes});")
    a("  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;")
    a("  const int nbx = (int)p.nbx, nby = (int)p.nby;")
    a("  const int n_items = nbx * nby * (int)p.nzc;")
    nb = 0
    for s_, (_r, _wh, stages, _pl, off) in enumerate(slots):
        a(f"  unsigned long long* full{s_} = bars + {nb};")
        a(f"  unsigned long long* empty{s_} = bars + {nb + stages};")
        nb += 2 * stages
    a("  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");  // next node may be scheduled")
    a("  if (tid == 0) {")
    for s_, (_r, _wh, stages, _pl, _off) in enumerate(slots):
        a(f"    for (int i = 0; i < {stages}; ++i) {{ mbar_init(full{s_} + i, 1); mbar_init(empty{s_} + i, {NW}); }}")
    a("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");")
    a("  }")
    a("  __syncthreads();")
    a("  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");  // previous node's writes visible, its reads done")
    # ---------------- producer warp (identical issue order to source_ws)
    a(f"  if (warp == {NW}) {{")
    a("    if (lane != 0) return;")
    for s_ in range(n_in):
        a(f"    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&p.tm[{s_}]) : \"memory\");")
    for s_ in range(n_in):
        a(f"    int fill{s_} = 0;")
    a("    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
    a("      const int bx = item % nbx, rest = item / nbx;")
    a("      const int by = rest % nby, bzc = rest / nby;")
    a(f"      const int x0 = bx * {BX}, y0 = by * {BY};")
    a("      const int zs = bzc * (int)p.zc;")
    a("      const int nzl = ((zs + (int)p.zc) < (int)p.nz ? (int)p.zc : (int)p.nz - zs);")
    a("      for (int t = 0; t < nzl; ++t) {")
    for s_, ((rz, ry, rx), (w, h), stages, plane, off) in enumerate(slots):
        a(f"        for (int k = (t == 0 ? 0 : t + {2 * rz}); k <= t + {2 * rz}; ++k) {{")
        a(f"          const int g = fill{s_} + k, stg = g % {stages};")
        a(f"          if (g >= {stages}) mbar_wait(empty{s_} + stg, ((g / {stages}) - 1) & 1);")
        a(f"          const int xs = (int)p.cx0[{s_}] + x0 - {rx};")
        a(f"          mbar_expect(full{s_} + stg, {w * h * elem});")
        a(f"          tma_load3(smem + {off} + stg * {plane}, &p.tm[{s_}], xs - (xs & {q - 1}),"
          f" (int)p.cy0[{s_}] + y0 - {ry}, (int)p.cz0[{s_}] + zs + k - {rz}, full{s_} + stg);")
        a("        }")
    a("      }")
    for s_, ((rz, _ry, _rx), _wh, _stg, _pl, _off) in enumerate(slots):
        a(f"      fill{s_} += nzl + {2 * rz};")
    a("    }")
    a("    return;")
    a("  }")
    # ---------------- compute warps
    a(f"  const int tx = tid % {BX}, ty = tid / {BX};")
    for s_ in range(n_in):
        a(f"  int fill{s_} = 0;")
    for s_ in sorted(regs):
        a(f"  T {', '.join(f'c{s_}_{r}_{k}' for r in range(RPT) for k in range(Z[s_]))};")
    a("  const long long opy = p.opy, opz = p.opz;")
    if STORE_HINT:
        a("  unsigned long long st_pol;  // outputs are not re-read by this launch: evict them first from L2")
        a("  asm volatile(\"createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\" : \"=l\"(st_pol));")
    a("  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
    a("    const int bx = item % nbx, rest = item / nbx;")
    a("    const int by = rest % nby, bzc = rest / nby;")
    a(f"    const int x0 = bx * {BX}, y0 = by * {BY};")
    a("    const int zs = bzc * (int)p.zc;")
    a("    const int nzl = ((zs + (int)p.zc) < (int)p.nz ? (int)p.zc : (int)p.nz - zs);")
    a(f"    const int yr = y0 + ty * {RPT};")
    a(f"    T* __restrict__ orow = reinterpret_cast<T*>(p.out) + (long long)zs * opz + (long long)yr * opy + (x0 + tx);")
    a("    const bool colok = (x0 + tx) < (int)p.nx;")
    for r in range(RPT):
        a(f"    const bool ok{r} = colok && (yr + {r}) < (int)p.ny;")
    for s_, ((rz, ry, rx), (w, h), stages, plane, off) in enumerate(slots):
        a(f"    const T* base{s_} = reinterpret_cast<const T*>(smem + {off}) + ((((int)p.cx0[{s_}] + x0 - {rx}) & {q - 1})"
          f" + (ty * {RPT} + {ry}) * {w} + tx + {rx});  // (row 0, dx 0) of this thread, stage 0")
        a(f"    int st{s_} = fill{s_} % {stages}, ph{s_} = (fill{s_} / {stages}) & 1;  // stage/phase of plane z")
    a(f"    for (int z0 = 0; z0 < nzl; z0 += {U}) {{")
    for m in range(U):
        def col(s_, r, k, m=m):
            return f"c{s_}_{r}_{(k + m) % Z[s_]}"
        a(f"      if (z0 + {m} < nzl) {{  // output plane z = z0 + {m}")
        for s_, ((rz, ry, rx), (w, h), stages, plane, off) in enumerate(slots):
            pe = plane // elem
            # stage of plane index z + d (d = 0 .. 2rz): st + d wrapped
            a(f"        {{ int sn = st{s_} + {2 * rz}, pn = ph{s_}; if (sn >= {stages}) {{ sn -= {stages}; pn ^= 1; }}")
            if m == 0:
                a(f"          if (z0 == 0) {{  // first plane of the item: the whole window")
                a(f"            for (int d = 0; d < {2 * rz}; ++d) {{ int sd = st{s_} + d, pd = ph{s_};"
                  f" if (sd >= {stages}) {{ sd -= {stages}; pd ^= 1; }} mbar_wait2(full{s_} + sd, pd); }}")
                if s_ in regs:
                    for d in range(2 * rz):
                        a(f"            {{ int sd = st{s_} + {d}; if (sd >= {stages}) sd -= {stages};")
                        for r in range(RPT):
                            a(f"              {col(s_, r, d)} = base{s_}[sd * {pe} + {r * w}];")
                        a("            }")
                a("          }")
            a(f"          mbar_wait2(full{s_} + sn, pn);")
            if s_ in regs:
                for r in range(RPT):
                    a(f"          {col(s_, r, 2 * rz)} = base{s_}[sn * {pe} + {r * w}];")
            a("        }")
        need = {}
        for ins in loads:
            s_, (dz, dy, dx) = ins[1], ins[2]
            if s_ in regs and dy == 0 and dx == 0:
                continue
            need.setdefault(s_, set()).add(dz)
        for s_, dzs in sorted(need.items()):
            (rz, ry, rx), (w, h), stages, plane, off = slots[s_]
            for dz in sorted(dzs):
                nm = f"P{s_}_{'m' if dz < 0 else 'p'}{abs(dz)}"
                a(f"        const T* {nm}; {{ int sd = st{s_} + {rz + dz}; if (sd >= {stages}) sd -= {stages}; {nm} = base{s_} + sd * {plane // elem}; }}")
        for r in range(RPT):
            def load(slot, off3, r=r):
                dz, dy, dx = off3
                (rz, ry, rx), (w, h), _stg, _pl, _o = slots[slot]
                if slot in regs and dy == 0 and dx == 0:
                    return col(slot, r, rz + dz)
                if slot in regs and dz == 0 and dx == 0 and 0 <= r + dy < RPT:
                    return col(slot, r + dy, rz)
                nm = f"P{slot}_{'m' if dz < 0 else 'p'}{abs(dz)}"
                return f"{nm}[{(r + dy) * w + dx}]"
            lines, res = _emit_expr(st, sig.dtype, load)
            a(f"        if (ok{r}) {{")
            for ln in lines:
                a("          " + ln)
            if STORE_HINT:
                a(f"          asm volatile(\"st.global.L2::cache_hint.{'f64' if elem == 8 else 'f32'} [%0], %1, %2;\""
                  f" :: \"l\"(orow + {r} * opy), \"{'d' if elem == 8 else 'f'}\"({res}), \"l\"(st_pol) : \"memory\");")
            else:
                a(f"          orow[{r} * opy] = {res};")
            a("        }")
        a("        orow += opz;")
        a("        __syncwarp();")
        for s_, ((rz, _ry, _rx), _wh, stages, _pl, _off) in enumerate(slots):
            a(f"        if (lane == 0) mbar_arrive(empty{s_} + st{s_});  // plane z of slot {s_} is dead")
            a(f"        if (++st{s_} == {stages}) {{ st{s_} = 0; ph{s_} ^= 1; }}")
        a("      }")
    a("    }")
    for s_, ((rz, _ry, _rx), _wh, stages, _pl, _off) in enumerate(slots):
        a(f"    for (int k = nzl; k < nzl + {2 * rz}; ++k) if (lane == 0) mbar_arrive(empty{s_} + (fill{s_} + k) % {stages});")
        a(f"    fill{s_} += nzl + {2 * rz};")
    a("  }")
    a("}")
    src = "\n".join(L) + "\n"
    return src, "est_stream", (CT + 32, 1, 1), smem, 1, {"slots": slots, "smem": smem, "cfg": cfg}


def _choose_zchunks(nz: int, n_xy: int, capacity: int) -> int:
    """Number of z-chunks balancing the persistent grid's last round."""
    best, best_eff = 1, -1.0
    for nzc in range(1, max(1, nz // MIN_ZCHUNK) + 1):
        zc = -(-nz // nzc)
        items = n_xy * nzc
        rounds = -(-items // capacity)
        eff = items / (rounds * capacity) * zc / (zc + 2)  # ~2 halo planes re-read per chunk
        if eff > best_eff + 1e-9:
            best, best_eff = nzc, eff
    return best


def item_geometry(item: dict, sm_count: int, geom: dict) -> None:
    cfg = geom["cfg"]
    item["nbx"] = -(-item["nx"] // cfg.bx)
    item["nby"] = -(-item["ny"] // cfg.by)
    n_xy = item["nbx"] * item["nby"]
    if cfg.persistent:
        cap = sm_count * blocks_per_sm(geom["smem"], cfg)
        nzc = _choose_zchunks(item["nz"], n_xy, cap)
        item["zc"] = -(-item["nz"] // nzc)
    else:
        item["zc"] = min(cfg.zchunk, item["nz"])
        cap = sm_count * blocks_per_sm(geom["smem"], cfg)
        if n_xy * -(-item["nz"] // item["zc"]) < 4 * cap:
            # thin slab (e.g. 1024^3 split over 8 GPUs): split z finer so the
            # grid is several waves deep, balancing the last wave
            nzc = _choose_zchunks(item["nz"], n_xy, cap)
            item["zc"] = -(-item["nz"] // nzc)
    item["nzc"] = -(-item["nz"] // item["zc"])
    n_items = n_xy * item["nzc"]
    item["blocks"] = min(n_items, sm_count * blocks_per_sm(geom["smem"], cfg)) if cfg.persistent else n_items


def pack_params(item: dict, tmaps: list, n_in: int) -> bytes:
    out = bytearray()
    for tm in tmaps:
        assert len(tm) == 128
        out += tm
    out += struct.pack("<Qqqqqqqqqq", item["out"], item["opy"], item["opz"], item["nx"], item["ny"],
                       item["nz"], item["zc"], item["nbx"], item["nby"], item["nzc"])
    for key in ("cx0", "cy0", "cz0"):
        out += struct.pack(f"<{n_in}q", *item[key])
    return bytes(out) + b"\0" * ((-len(out)) % 64)
