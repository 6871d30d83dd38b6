"""The "tb" skeleton: temporal blocking of K consecutive ping-pong sweeps.

A batch of heat/Jacobi iterations is a chain of single-statement rank-3 nodes
`B[S] = f(A[S + offsets]); A[S] = f(B[S + offsets]); ...` (
reference semantics executor.py:258-348: nodes run in order, statement at a
time). On one GPU with one tile no halo exchange happens between them, so K of
them (K even) can run as ONE kernel that reads A once from HBM, keeps the
intermediate sweeps in shared memory and writes only the arrays' final values:
24 B per K updates instead of 16 B per update (12 B/LUP at K = 2).

Every point is still computed by the same generated expression
(codegen._emit_expr: one correctly rounded IEEE op per plan instruction, no
contraction), so results are bit-identical to K separate sweeps. Epochs,
rounds and launch counts are kept per node by the executor.

Kernel structure (warp-specialised like stream.source_ws2):
* work item = a BX x BY output column of S over ZC planes; step j (1..K) of
  the chain covers the item tile expanded by (K-j)*r in y/x (overlapped
  tiling) and trails step j-1 by rz planes in z;
* producer warp: one TMA (`cp.async.bulk.tensor.3d`) per input plane of A
  (tile + K*r halo) into an mbarrier-gated ring (full/empty barriers);
* compute warps, per input plane: step 1 reads the TMA ring, step j > 1 reads
  step j-1's shared-memory plane ring (2rz+2 planes); one named barrier
  between steps. Cells of a step's region outside S keep the array's stored
  value (read from its home buffer; S's complement is never written);
* stores: step K-1 (array B, final) in place inside S; step K (array A,
  final) into A's *other* home buffer, because neighbouring CTAs still read A
  through TMA. The executor alternates A between its tile buffer and a
  scratch twin (chains come in pairs, so A ends in its own buffer) and copies
  S's complement into the twin at the start of each run.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

from .codegen import CTYPE, ELEM, StmtSig, _emit_expr, slot_radius
from .stream import _PTX_HELPERS

MAX_RADIUS = 2
SMEM_BUDGET = 200 * 1024
SMEM_PER_SM = 228 * 1024
SKIP_MID_B = os.environ.get("EST_TB_SKIPB", "1") == "1"


@dataclass(frozen=True)
class TbCfg:
    k: int = 2              # sweeps per launch (even)
    bx: int = 48            # output columns per item
    by: int = 32            # output rows per item
    rpt: int = 2            # rows of the step-1 region per compute thread
    prefetch: int = 2       # input planes in flight beyond the z window
    zchunk: int = 192       # planes per item (C4: 5 full chunks + 62; 1-2 % over 128, profiles/r1s2_tb_skipb.md)
    l2promo: int = 2        # TMA L2 promotion: 0 none, 1 64B, 2 128B, 3 256B
    persistent: bool = False
    minb: int = 0           # __launch_bounds__ min blocks per SM (0: from smem/threads, >= 48 regs)
    variant: str = "block"  # "block" (smem ring per step) or "warp" (intermediate sweep in registers + shuffles)
    wx: int = 2             # (warp) warps across x; each warp owns 30 output columns
    wy: int = 4             # (warp) warps across y
    r: int = 4              # (warp) output rows per warp


def _env_cfg() -> TbCfg:
    e = os.environ.get
    d = TbCfg()
    return TbCfg(k=int(e("EST_TB_K", d.k)), bx=int(e("EST_TB_BX", d.bx)), by=int(e("EST_TB_BY", d.by)),
                 rpt=int(e("EST_TB_RPT", d.rpt)), prefetch=int(e("EST_TB_PREFETCH", d.prefetch)),
                 zchunk=int(e("EST_TB_ZCHUNK", d.zchunk)), l2promo=int(e("EST_TB_L2PROMO", d.l2promo)),
                 persistent=e("EST_TB_PERSISTENT", "0") == "1", minb=int(e("EST_TB_MINB", d.minb)),
                 variant=e("EST_TB_VARIANT", d.variant), wx=int(e("EST_TB_WX", d.wx)),
                 wy=int(e("EST_TB_WY", d.wy)), r=int(e("EST_TB_R", d.r)))


DEFAULT = _env_cfg()
ENABLED = os.environ.get("EST_TB", "1") == "1"
# measured crossover (profiles/r1s2_tb_skipb.md): at 1022^3 outputs the chain
# beats two single sweeps by 18 %, at 510^3 it is 1.5-4 % slower (too few
# items per SM to hide each item's pipeline fill)
MIN_POINTS = int(os.environ.get("EST_TB_MIN_POINTS", 1 << 28))
# chain depths that passed the GPU parity suite (EST_TB_VALIDATED_K widens it for experiments)
VALIDATED_K = tuple(int(k) for k in os.environ.get("EST_TB_VALIDATED_K", "2").split(","))


def _round(v: int, m: int) -> int:
    return -(-v // m) * m


def z_star(st: StmtSig) -> bool:
    """Every load off the centre plane is a pure z offset (dz, 0, 0)."""
    return all(i[2][0] == 0 or (i[2][1] == 0 and i[2][2] == 0) for i in st.instructions if i[0] == "load")


def layout(rad, dtype: int, cfg: TbCfg) -> dict:
    """Shared memory: the input TMA ring (tile + K*r halo) and, per
    intermediate step, a ring of 2rz+2 planes in the step-1 frame (W1 x H1)
    with one mbarrier per plane slot (count = compute warps)."""
    rz, ry, rx = rad
    elem = ELEM[dtype]
    q = 16 // elem
    K = cfg.k
    w0 = _round(cfg.bx + 2 * K * rx + q - 1, q)
    h0 = cfg.by + 2 * K * ry
    s0 = rz + 1 + cfg.prefetch
    pl0 = _round(w0 * h0 * elem, 1024)
    w1, h1 = cfg.bx + 2 * (K - 1) * rx, cfg.by + 2 * (K - 1) * ry
    pl1 = _round(w1 * h1 * elem, 128)
    off = s0 * pl0
    rings = []
    nr = 2 * rz + 2  # slots: a warp may run one plane ahead (split arrive / wait)
    for _j in range(1, K):
        rings.append({"off": off, "n": nr})
        off += nr * pl1
    data = _round(off, 8)
    smem = data + 8 * (2 * s0 + (K - 1) * nr) + 1024
    hg = h1 // cfg.rpt if h1 % cfg.rpt == 0 else 0
    nt = _round(w1 * hg, 32)
    return {"rad": (rz, ry, rx), "w0": w0, "h0": h0, "s0": s0, "pl0": pl0, "w1": w1, "h1": h1,
            "pl1": pl1, "hg": hg, "nt": nt, "rings": rings, "data": data, "smem": smem,
            "cfg": cfg, "elem": elem, "q": q}


def warp_eligible(st: StmtSig, dtype: int, cfg: TbCfg) -> bool:
    """Warp-tiled variant: K = 2, one input slot, every offset within +-1, z-star."""
    if cfg.variant != "warp" or cfg.k != 2 or st.arity != 1 or dtype not in ELEM or not z_star(st):
        return False
    rad = slot_radius(st).get(0)
    return rad is not None and max(rad) <= 1 and rad[0] == 1 and cfg.r >= 1


def eligible(st: StmtSig, dtype: int, cfg: TbCfg | None = None) -> bool:
    """Single input slot, z-star loads, 1 <= rz, radius <= MAX_RADIUS, fits."""
    cfg = cfg or DEFAULT
    if warp_eligible(st, dtype, cfg):
        return True
    # K = 4 chains are bit-exact since the padded-z guard of the fast path
    # (scripts/debug_tb_k4.py) but 1.5-1.7x slower than K = 2 on C4
    # (profiles/r1s2_tb_skipb.md), so only K = 2 is scheduled by default
    if cfg.k not in VALIDATED_K or st.arity != 1 or dtype not in ELEM or not z_star(st):
        return False
    rad = slot_radius(st).get(0)
    if rad is None or max(rad) > MAX_RADIUS or rad[0] < 1:
        return False
    lay = layout(rad, dtype, cfg)
    if lay["w0"] > 256 or lay["h0"] > 256 or lay["hg"] == 0 or lay["nt"] + 32 > 1024:
        return False
    return lay["smem"] <= SMEM_BUDGET


def blocks_per_sm(smem: int, nt: int) -> int:
    return max(1, min(SMEM_PER_SM // (smem + 1024), 2048 // (nt + 32)))


def source(st: StmtSig, dtype: int, cfg: TbCfg | None = None) -> tuple:
    cfg = cfg or DEFAULT
    if warp_eligible(st, dtype, cfg):
        return source_warp(st, dtype, cfg)
    return source_block(st, dtype, cfg)


def source_block(st: StmtSig, dtype: int, cfg: TbCfg | None = None) -> tuple:
    """-> (source, kernel name, block, smem, geometry).

    Each compute thread owns RPT points of the step-1 region (W1 x H1, rows
    interleaved by H1/RPT so warps run along x) for every plane: its own
    column of every step lives in registers (the pure-z operands), the centre
    plane of each step is published in shared memory for the neighbours'
    (dy, dx) operands. Per input plane: one mbarrier wait (TMA), one named
    barrier, then step 1 .. K each one plane further behind."""
    cfg = cfg or DEFAULT
    rad = slot_radius(st)[0]
    lay = layout(rad, dtype, cfg)
    rz, ry, rx = rad
    K, BX, BY, RPT = cfg.k, cfg.bx, cfg.by, cfg.rpt
    NT, HG, W1, H1 = lay["nt"], lay["hg"], lay["w1"], lay["h1"]
    NW = NT // 32
    T = CTYPE[dtype]
    q = lay["q"]
    s0, pl0, w0, h0 = lay["s0"], lay["pl0"], lay["w0"], lay["h0"]
    E = lay["elem"]
    L = []
    a = L.append
    a(f'// generated by paper_2512_19851_b200/temporal.py — skeleton "tb" (K={K} fused sweeps) {cfg}')
    a(f"typedef {T} T;")
    a("struct __align__(64) Tmap { unsigned long long w[16]; };")
    a("struct __align__(64) Params { Tmap tm;")
    a("  unsigned long long src, bhome, adst;  // padded-box origins: A now, B (in place), A next")
    a("  long long py, pz;")
    a("  int npz, npy, npx, xoff, sz0, sz1, sy0, sy1, sx0, sx1, nbx, nby, zc, nzc, wb; };")
    L.append(_PTX_HELPERS)
    a("__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {")
    a("  asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(smem_u32(b)) : \"memory\"); }")
    minb = cfg.minb or max(1, min(blocks_per_sm(lay["smem"], NT), 65536 // ((NT + 32) * 96)))
    lay["min_blocks"] = minb
    a(f'extern "C" __global__ void __launch_bounds__({NT + 32}, {minb})')
    a("est_tb(const __grid_constant__ Params p) {")
    a("  extern __shared__ __align__(1024) unsigned char smem[];")
    a(f"  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + {lay['data']});")
    a(f"  unsigned long long* empty = full + {s0};")
    a("  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;")
    a("  const int n_items = p.nbx * p.nby * p.nzc;")
    a("  if (tid == 0) {")
    a(f"    for (int i = 0; i < {s0}; ++i) {{ mbar_init(full + i, 1); mbar_init(empty + i, {NW}); }}")
    a(f"    for (int i = 0; i < {(K - 1) * lay['rings'][0]['n'] if K > 1 else 0}; ++i) mbar_init(empty + {s0} + i, {NW});")
    a("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");")
    a("  }")
    a("  __syncthreads();")

    def item_decode(ind):
        a(f"{ind}const int bx = item % p.nbx, rest = item / p.nbx;")
        a(f"{ind}const int by = rest % p.nby, bzc = rest / p.nby;")
        a(f"{ind}const int x0 = p.sx0 + bx * {BX}, y0 = p.sy0 + by * {BY};")
        a(f"{ind}const int zs = p.sz0 + bzc * p.zc;")
        a(f"{ind}const int nzl = min(p.zc, p.sz1 - zs);")
        a(f"{ind}const int n0 = nzl + {2 * K * rz};")

    # ---------------- producer warp
    a(f"  if (warp == {NW}) {{")
    a("    if (lane != 0) return;")
    a("    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&p.tm) : \"memory\");")
    a("    int fill = 0;")
    a("    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
    item_decode("      ")
    a(f"      const int xs = p.xoff + x0 - {K * rx};")
    a(f"      const int xa = xs - (xs & {q - 1});")
    a("      for (int k = 0; k < n0; ++k) {")
    a(f"        const int g = fill + k, stg = g % {s0};")
    a(f"        if (g >= {s0}) mbar_wait(empty + stg, ((g / {s0}) - 1) & 1);")
    a(f"        mbar_expect(full + stg, {w0 * h0 * E});")
    a(f"        tma_load3(smem + stg * {pl0}, &p.tm, xa, y0 - {K * ry}, zs - {K * rz} + k, full + stg);")
    a("      }")
    a("      fill += n0;")
    a("    }")
    a("    return;")
    a("  }")
    # ---------------- compute threads
    a("  const T* __restrict__ asrc = reinterpret_cast<const T*>(p.src);")
    a("  T* __restrict__ bmem = reinterpret_cast<T*>(p.bhome);")
    a("  T* __restrict__ adst = reinterpret_cast<T*>(p.adst);")
    a(f"  const bool act = tid < {W1 * HG};")
    a(f"  const int lx = tid % {W1}, lyg = tid / {W1};")
    # per-row thread constants (item independent)
    for r in range(RPT):
        ly = f"(lyg * {RPT} + {r})"
        a(f"  const int ly{r} = {ly};")
        for j in range(2, K + 1):
            lo_y, hi_y = (j - 1) * ry, H1 - (j - 1) * ry
            lo_x, hi_x = (j - 1) * rx, W1 - (j - 1) * rx
            a(f"  const bool inT{j}_{r} = act && ly{r} >= {lo_y} && ly{r} < {hi_y} && lx >= {lo_x} && lx < {hi_x};")
        a(f"  const int so{r} = ly{r} * {W1} + lx;  // step-1 frame smem index")
        a(f"  const int io{r} = (ly{r} + {ry}) * {w0} + lx + {rx};  // input frame (before the alignment shift)")
    a("  int fill = 0;")
    for j in range(1, K):
        a(f"  unsigned long long* rb{j} = empty + {s0 + (j - 1) * lay['rings'][0]['n']};  // ring {j} slot barriers")
        a(f"  int f{j} = 0;  // step-{j} planes produced so far (all items)")
    # register columns: c{j}_{r}_{k} = step-j value (j = 0: input) at the thread point, k = 0..2rz
    for j in range(0, K):
        for r in range(RPT):
            a(f"  T {', '.join(f'c{j}_{r}_{k} = 0' for k in range(2 * rz + 1))};")
    a("  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
    item_decode("    ")
    a(f"    const int sh = (p.xoff + x0 - {K * rx}) & {q - 1};")
    for r in range(RPT):
        a(f"    const int gy{r} = y0 - {(K - 1) * ry} + ly{r}, gx{r} = x0 - {(K - 1) * rx} + lx;")
        a(f"    const bool sxy{r} = act && gy{r} >= p.sy0 && gy{r} < p.sy1 && gx{r} >= p.sx0 && gx{r} < p.sx1;")
        a(f"    const bool pxy{r} = act && gy{r} >= 0 && gy{r} < p.npy && gx{r} >= 0 && gx{r} < p.npx;")
        a(f"    const long long go{r} = (long long)gy{r} * p.py + gx{r};")
    a(f"    const bool fast = (x0 - {(K - 1) * rx} >= p.sx0) && (x0 + {BX + (K - 1) * rx} <= p.sx1) &&"
      f" (y0 - {(K - 1) * ry} >= p.sy0) && (y0 + {BY + (K - 1) * ry} <= p.sy1);")
    a("    if (fast) {")
    emit_fast_loop(a, st, dtype, lay)
    a("    } else {")
    a("    for (int t = 0; t < n0; ++t) {")
    # prefetch out-of-S values of intermediate steps (home buffers), before any wait
    for j in range(1, K):
        home = "bmem" if j % 2 == 1 else "asrc"
        a(f"      const int z{j} = zs - {(K - j) * rz} + t - {2 * j * rz};")
        a(f"      const bool zi{j} = z{j} >= p.sz0 && z{j} < p.sz1, zp{j} = z{j} >= 0 && z{j} < p.npz;")
        for r in range(RPT):
            inT = "act" if j == 1 else f"inT{j}_{r}"
            a(f"      T h{j}_{r} = (T)0;")
            a(f"      if (t >= {2 * j * rz} && {inT} && zp{j} && pxy{r} && !(zi{j} && sxy{r}))"
              f" h{j}_{r} = {home}[(long long)z{j} * p.pz + go{r}];  // outside S: stored value")
    a(f"      {{ const int g = fill + t; mbar_wait(full + g % {s0}, (g / {s0}) & 1); }}")
    a(f"      const T* inC = reinterpret_cast<const T*>(smem) + ((fill + t) % {s0}) * {pl0 // E} + sh;")
    for r in range(RPT):
        a(f"      c0_{r}_{2 * rz} = act ? inC[io{r}] : (T)0;")
    for j in range(1, K + 1):
        emit_step_b(a, st, dtype, lay, j)
        if j == 1:
            a(f"      if (t >= {rz}) {{ __syncwarp(); if (lane == 0) mbar_arrive(empty + (fill + t - {rz}) % {s0}); }}")
    # rotate the register columns (step j's column only moves once step j ran)
    for j in range(0, K):
        cond = "true" if j == 0 else f"t >= {2 * j * rz}"
        a(f"      if ({cond}) {{")
        for r in range(RPT):
            for k in range(2 * rz):
                a(f"        c{j}_{r}_{k} = c{j}_{r}_{k + 1};")
        a("      }")
    a("    }")
    a("    }  // general path")
    a(f"    for (int k = (n0 > {rz} ? n0 - {rz} : 0); k < n0; ++k) if (lane == 0) mbar_arrive(empty + (fill + k) % {s0});")
    a("    fill += n0;")
    for j in range(1, K):
        a(f"    f{j} += nzl + {2 * (K - j) * rz};")
    a("  }")
    a("}")
    src = "\n".join(L) + "\n"
    lay["blocks_per_sm"] = minb
    return src, "est_tb", (NT + 32, 1, 1), lay["smem"], lay


def source_warp(st: StmtSig, dtype: int, cfg: TbCfg) -> tuple:
    """K = 2 warp-tiled chain kernel.

    CTA output tile = (30*WX) x (R*WY) columns x rows, streamed along z; the
    producer warp TMA-loads each input plane (tile + 2-cell halo) into an
    mbarrier ring. Each compute warp owns 30 output columns x R rows: lane l
    holds column l-1, so lanes 0 and 31 carry the x-halo of the intermediate
    sweep. Step 1 (B at t+1) is computed for rows -1..R of the warp from the
    shared input plane (z-neighbours from a per-lane register window); step 2
    (A at t+2) reads step 1 only from registers: own rows / y-neighbours
    directly, x-neighbours through warp shuffles. No shared memory for the
    intermediate sweep and no barrier between warps."""
    rz, ry, rx = slot_radius(st)[0]
    T = CTYPE[dtype]
    elem = ELEM[dtype]
    q = 16 // elem
    WX, WY, R = cfg.wx, cfg.wy, cfg.r
    BX, BY = 30 * WX, R * WY
    NW = WX * WY
    NT = 32 * NW
    w0 = _round(BX + 4 + q - 1, q)
    h0 = BY + 4
    s0 = 2 + cfg.prefetch
    pl0 = _round(w0 * h0 * elem, 1024)
    data = s0 * pl0
    smem = data + 8 * 2 * s0 + 1024
    minb = cfg.minb or max(1, min(SMEM_PER_SM // (smem + 1024), 65536 // ((NT + 32) * 96), 2048 // (NT + 32)))
    lay = {"rad": (rz, ry, rx), "w0": w0, "h0": h0, "s0": s0, "pl0": pl0, "data": data, "smem": smem,
           "cfg": cfg, "elem": elem, "q": q, "bx": BX, "by": BY, "nt": NT, "min_blocks": minb,
           "blocks_per_sm": minb, "variant": "warp"}
    ROWS = list(range(-1, R + 1))          # step-1 rows of a warp (rr = r + 1)
    L = []
    a = L.append
    a(f'// generated by paper_2512_19851_b200/temporal.py — skeleton "tb" warp-tiled (K=2) {cfg}')
    a(f"typedef {T} T;")
    a("struct __align__(64) Tmap { unsigned long long w[16]; };")
    a("struct __align__(64) Params { Tmap tm;")
    a("  unsigned long long src, bhome, adst;  // padded-box origins: A now, B (in place), A next")
    a("  long long py, pz;")
    a("  int npz, npy, npx, xoff, sz0, sz1, sy0, sy1, sx0, sx1, nbx, nby, zc, nzc, wb; };")
    L.append(_PTX_HELPERS)
    a("__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {")
    a("  asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(smem_u32(b)) : \"memory\"); }")
    a(f'extern "C" __global__ void __launch_bounds__({NT + 32}, {minb})')
    a("est_tb(const __grid_constant__ Params p) {")
    a("  extern __shared__ __align__(1024) unsigned char smem[];")
    a(f"  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + {data});")
    a(f"  unsigned long long* empty = full + {s0};")
    a("  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;")
    a("  const int n_items = p.nbx * p.nby * p.nzc;")
    a("  if (tid == 0) {")
    a(f"    for (int i = 0; i < {s0}; ++i) {{ mbar_init(full + i, 1); mbar_init(empty + i, {NW}); }}")
    a("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");")
    a("  }")
    a("  __syncthreads();")

    def item_decode(ind):
        a(f"{ind}const int bx = item % p.nbx, rest = item / p.nbx;")
        a(f"{ind}const int by = rest % p.nby, bzc = rest / p.nby;")
        a(f"{ind}const int x0 = p.sx0 + bx * {BX}, y0 = p.sy0 + by * {BY};")
        a(f"{ind}const int zs = p.sz0 + bzc * p.zc;")
        a(f"{ind}const int nzl = min(p.zc, p.sz1 - zs);")
        a(f"{ind}const int n0 = nzl + 4;")

    # ---------------- producer warp
    a(f"  if (warp == {NW}) {{")
    a("    if (lane != 0) return;")
    a("    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&p.tm) : \"memory\");")
    a("    int fill = 0;")
    a("    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
    item_decode("      ")
    a("      const int xs = p.xoff + x0 - 2;")
    a(f"      const int xa = xs - (xs & {q - 1});")
    a("      for (int k = 0; k < n0; ++k) {")
    a(f"        const int g = fill + k, stg = g % {s0};")
    a(f"        if (g >= {s0}) mbar_wait(empty + stg, ((g / {s0}) - 1) & 1);")
    a(f"        mbar_expect(full + stg, {w0 * h0 * elem});")
    a(f"        tma_load3(smem + stg * {pl0}, &p.tm, xa, y0 - 2, zs - 2 + k, full + stg);")
    a("      }")
    a("      fill += n0;")
    a("    }")
    a("    return;")
    a("  }")
    # ---------------- compute warps
    a("  const T* __restrict__ asrc = reinterpret_cast<const T*>(p.src); (void)asrc;")
    a("  T* __restrict__ bmem = reinterpret_cast<T*>(p.bhome);")
    a("  T* __restrict__ adst = reinterpret_cast<T*>(p.adst);")
    a(f"  const int wxi = warp % {WX}, wyi = warp / {WX};")
    a("  const bool own = lane >= 1 && lane <= 30;")
    a("  const long long py = p.py, pz = p.pz;")
    a("  int fill = 0;")
    for j in (0, 1):
        for rr in range(len(ROWS)):
            a(f"  T {', '.join(f'c{j}_{rr}_{k} = 0' for k in range(3))};")
    a("  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
    item_decode("    ")
    a(f"    const int sh = (p.xoff + x0 - 2) & {q - 1};")
    a(f"    const int scol = sh + 30 * wxi + lane + 1;   // smem column of this lane (output column lane-1)")
    a(f"    const int srow = {R} * wyi + 2;               // smem row of warp row 0")
    a("    const int gx = x0 + 30 * wxi + lane - 1;")
    a("    const bool colS = gx >= p.sx0 && gx < p.sx1, colP = gx >= 0 && gx < p.npx;")
    a(f"    const int gy0 = y0 + {R} * wyi;")
    for rr, r in enumerate(ROWS):
        a(f"    const bool rS{rr} = (gy0 + {r}) >= p.sy0 && (gy0 + {r}) < p.sy1 && colS;")
        a(f"    const bool rP{rr} = (gy0 + {r}) >= 0 && (gy0 + {r}) < p.npy && colP;")
    a("    const long long cb = (long long)gy0 * py + gx;  // row-0 offset of this lane within a plane")
    a("    const T* ring = reinterpret_cast<const T*>(smem) + sh * 0;")
    a(f"    for (int t0 = 0; t0 < n0; t0 += 3) {{")
    for m in range(3):
        def col(j, rr, k, m=m):
            return f"c{j}_{rr}_{(k + m) % 3}"
        a(f"      if (t0 + {m} < n0) {{")
        a(f"      const int t = t0 + {m};")
        a(f"      {{ const int g = fill + t; mbar_wait(full + g % {s0}, (g / {s0}) & 1); }}")
        a(f"      const T* Pn = ring + ((fill + t) % {s0}) * {pl0 // elem} + srow * {w0} + scol;  // input plane t")
        for rr, r in enumerate(ROWS):
            a(f"      {col(0, rr, 2)} = Pn[{r * w0}];")
        # ---- step 1: plane index t-1 of the input is the centre plane
        a("      if (t >= 2) {")
        a(f"        const T* Pc = ring + ((fill + t - 1) % {s0}) * {pl0 // elem} + srow * {w0} + scol;")
        a("        const int z1 = zs - 1 + (t - 2);")
        a("        const bool zin1 = z1 >= p.sz0 && z1 < p.sz1, zp1 = z1 >= 0 && z1 < p.npz;")
        a("        const long long zo1 = (long long)z1 * pz + cb;")
        for rr, r in enumerate(ROWS):
            def load1(slot, off3, rr=rr, r=r):
                dz, dy, dx = off3
                if dz != 0 or (dy == 0 and dx == 0):
                    return col(0, rr, 1 + dz)
                if dx == 0 and 0 <= rr + dy < len(ROWS):
                    return col(0, rr + dy, 1)
                return f"Pc[{(r + dy) * w0 + dx}]"
            lines, res = _emit_expr(st, dtype, load1)
            a(f"        {{ T v;")
            a(f"          if (zin1 && rS{rr}) {{")
            for ln in lines:
                a(f"            {ln}")
            a(f"            v = {res};")
            if 0 <= r < R:
                a(f"            if (own && p.wb) bmem[zo1 + {r} * py] = v;")
            a(f"          }} else {{")
            a(f"            v = (zp1 && rP{rr}) ? bmem[zo1 + {r} * py] : ({T})0;  // outside S: stored value")
            a("          }")
            a(f"          {col(1, rr, 2)} = v; }}")
        a("      }")
        a(f"      if (t >= 1) {{ __syncwarp(); if (lane == 0) mbar_arrive(empty + (fill + t - 1) % {s0}); }}")
        # ---- step 2: step-1 index t-3 is the centre
        a("      if (t >= 4) {")
        a("        const int z2 = zs + (t - 4);")
        a("        const bool zin2 = z2 >= p.sz0 && z2 < p.sz1;")
        a("        const long long zo2 = (long long)z2 * pz + cb;")
        # shuffled neighbours needed
        need = set()
        for i in st.instructions:
            if i[0] == "load" and i[2][0] == 0 and i[2][2] != 0:
                need.add((i[2][1], i[2][2]))
        shf = {}
        for r in range(R):
            rr = r + 1
            for dy, dx in sorted(need):
                key = (rr + dy, dx)
                if key not in shf:
                    nm = f"sf{rr + dy}_{'m' if dx < 0 else 'p'}{abs(dx)}"
                    shf[key] = nm
                    a(f"        const T {nm} = __shfl_sync(0xffffffffu, {col(1, rr + dy, 1)}, (lane + ({dx})) & 31);")
        for r in range(R):
            rr = r + 1
            def load2(slot, off3, rr=rr):
                dz, dy, dx = off3
                if dz != 0 or (dy == 0 and dx == 0):
                    return col(1, rr, 1 + dz)
                if dx == 0:
                    return col(1, rr + dy, 1)
                return shf[(rr + dy, dx)]
            lines, res = _emit_expr(st, dtype, load2)
            a(f"        if (zin2 && rS{rr} && own) {{")
            for ln in lines:
                a(f"          {ln}")
            a(f"          adst[zo2 + {r} * py] = {res};")
            a("        }")
        a("      }")
        a("      }")
    a("    }")
    a(f"    if (lane == 0) mbar_arrive(empty + (fill + n0 - 1) % {s0});")
    a("    fill += n0;")
    a("  }")
    a("}")
    src = "\n".join(L) + "\n"
    return src, "est_tb", (NT + 32, 1, 1), smem, lay


def emit_fast_loop(a, st: StmtSig, dtype: int, lay: dict) -> None:
    """Items whose whole step-1 region lies inside S in y/x: no per-point
    S tests (planes outside S's z range take a uniform branch), store
    pointers advanced per plane, ring slots as counters, and the plane loop
    unrolled 2rz+1 times so the register columns rotate by renaming."""
    cfg = lay["cfg"]
    K, RPT = cfg.k, cfg.rpt
    rz, ry, rx = lay["rad"]
    s0, E = lay["s0"], lay["elem"]
    pl0, pl1 = lay["pl0"] // E, lay["pl1"] // E
    Z = 2 * rz + 1          # register column length = unroll factor
    ind = "      "
    a(f"{ind}const long long pz = p.pz;")
    for r in range(RPT):
        a(f"{ind}T* bp{r} = bmem + (long long)(zs - {rz}) * pz + go{r};  // step K-1 (B) plane 0")
        a(f"{ind}T* ap{r} = adst + (long long)zs * pz + go{r};  // step K (A next) plane 0")
    a(f"{ind}int is = fill % {s0}, ip = (fill / {s0}) & 1;  // input slot / phase of index t")
    a(f"{ind}const T* ring0 = reinterpret_cast<const T*>(smem) + sh;")
    a(f"{ind}for (int t0 = 0; t0 < n0; t0 += {Z}) {{")
    for m in range(Z):
        # logical column index k (0 = oldest of the window) lives in name (k + m) % Z
        def col(j, r, k, m=m):
            return f"c{j}_{r}_{(k + m) % Z}"
        a(f"{ind}  if (t0 + {m} < n0) {{  // plane iteration t = t0 + {m}")
        a(f"{ind}  const int t = t0 + {m};")
        a(f"{ind}  mbar_wait(full + is, ip);")
        a(f"{ind}  {{ const T* inC = ring0 + is * {pl0};")
        for r in range(RPT):
            a(f"{ind}    {col(0, r, 2 * rz)} = inC[io{r}];")
        a(f"{ind}  }}")
        a(f"{ind}  int ir = is - {rz}; if (ir < 0) ir += {s0};  // slot of index t - rz")
        for j in range(1, K + 1):
            final = j == K
            a(f"{ind}  if (t >= {2 * j * rz}) {{  // step {j}")
            a(f"{ind}    const bool zin = (zs - {(K - j) * rz} + t - {2 * j * rz}) >= p.sz0 &&"
              f" (zs - {(K - j) * rz} + t - {2 * j * rz}) < p.sz1;")
            if j == 1:
                a(f"{ind}    const T* P = ring0 + ir * {pl0};")
            else:
                rp = lay["rings"][j - 2]
                nr = rp["n"]
                a(f"{ind}    const int gr = f{j - 1} + t - {(2 * j - 1) * rz};")
                a(f"{ind}    mbar_wait(rb{j - 1} + gr % {nr}, (gr / {nr}) & 1);")
                a(f"{ind}    const T* P = reinterpret_cast<const T*>(smem + {rp['off']}) + (gr % {nr}) * {pl1};")
            if not final:
                rg = lay["rings"][j - 1]
                a(f"{ind}    const int gw = f{j} + t - {2 * j * rz};")
                a(f"{ind}    T* Wr = reinterpret_cast<T*>(smem + {rg['off']}) + (gw % {rg['n']}) * {pl1};")
                home = "bmem" if j % 2 == 1 else "asrc"
                a(f"{ind}    const long long zo = (long long)(zs - {(K - j) * rz} + t - {2 * j * rz}) * pz;")
            a(f"{ind}    if (zin) {{")
            for r in range(RPT):
                inT = "act" if j == 1 else f"inT{j}_{r}"
                base = f"io{r}" if j == 1 else f"so{r}"
                pitch = lay["w0"] if j == 1 else lay["w1"]

                def load(slot, off3, r=r, base=base, pitch=pitch, j=j):
                    dz, dy, dx = off3
                    if dz != 0 or (dy == 0 and dx == 0):
                        return col(j - 1, r, rz + dz)
                    if dx == 0 and 0 <= r + dy < RPT:
                        return col(j - 1, r + dy, rz)
                    return f"P[{base} + {dy * pitch + dx}]"

                lines, res = _emit_expr(st, dtype, load)
                a(f"{ind}      if ({inT}) {{")
                for ln in lines:
                    a(f"{ind}        {ln}")
                if final:
                    a(f"{ind}        *ap{r} = {res};")
                else:
                    a(f"{ind}        Wr[so{r}] = {res};")
                    a(f"{ind}        {col(j, r, 2 * rz)} = {res};")
                    if j == K - 1:
                        a(f"{ind}        if (p.wb && inT{K}_{r}) *bp{r} = {res};")
                a(f"{ind}      }}")
            a(f"{ind}    }}")
            if not final:
                a(f"{ind}    else {{  // plane outside S: the array's stored value (0 beyond the padded box,")
                a(f"{ind}           // which deeper chains reach at the first and last planes)")
                a(f"{ind}      const int zq = zs - {(K - j) * rz} + t - {2 * j * rz};")
                a(f"{ind}      const bool zp = zq >= 0 && zq < p.npz;")
                for r in range(RPT):
                    inT = "act" if j == 1 else f"inT{j}_{r}"
                    a(f"{ind}      if ({inT}) {{ const T v = zp ? {home}[zo + go{r}] : (T)0; Wr[so{r}] = v;"
                      f" {col(j, r, 2 * rz)} = v; }}")
                a(f"{ind}    }}")
            for r in range(RPT):
                if final:
                    a(f"{ind}    ap{r} += pz;")
                elif j == K - 1:
                    a(f"{ind}    bp{r} += pz;")
            if not final:
                a(f"{ind}    __syncwarp(); if (lane == 0) mbar_arrive(rb{j} + gw % {lay['rings'][j - 1]['n']});")
            a(f"{ind}  }}")
            if j == 1:
                a(f"{ind}  if (t >= {rz}) {{ __syncwarp(); if (lane == 0) mbar_arrive(empty + ir); }}")
        a(f"{ind}  if (++is == {s0}) {{ is = 0; ip ^= 1; }}")
        a(f"{ind}  }}")
    a(f"{ind}}}")


def emit_step_b(a, st: StmtSig, dtype: int, lay: dict, j: int) -> None:
    """Step j at input iteration t: index u = t - 2*j*rz, centre plane of the
    previous step at index u + rz (input ring for j = 1, ring j-1 otherwise)."""
    cfg = lay["cfg"]
    K, RPT = cfg.k, cfg.rpt
    rz, ry, rx = lay["rad"]
    W1 = lay["w1"]
    E = lay["elem"]
    final = j == K
    ind = "        "
    a(f"      if (t >= {2 * j * rz}) {{  // step {j}")
    a(f"{ind}const int u = t - {2 * j * rz};")
    a(f"{ind}const int zj = zs - {(K - j) * rz} + u;")
    a(f"{ind}const bool zin = zj >= p.sz0 && zj < p.sz1;")
    a(f"{ind}const long long zoff = (long long)zj * p.pz;")
    if j == 1:
        a(f"{ind}const T* P = reinterpret_cast<const T*>(smem) + ((fill + t - {rz}) % {lay['s0']}) * {lay['pl0'] // E} + sh;")
    else:
        rp = lay["rings"][j - 2]
        nr = rp["n"]
        a(f"{ind}const int gr = f{j - 1} + t - {(2 * j - 1) * rz};  // step-{j - 1} plane read")
        a(f"{ind}mbar_wait(rb{j - 1} + gr % {nr}, (gr / {nr}) & 1);")
        a(f"{ind}const T* P = reinterpret_cast<const T*>(smem + {rp['off']}) + (gr % {nr}) * {lay['pl1'] // E};")
    if not final:
        rg = lay["rings"][j - 1]
        a(f"{ind}const int gw = f{j} + u;")
        a(f"{ind}T* W = reinterpret_cast<T*>(smem + {rg['off']}) + (gw % {rg['n']}) * {lay['pl1'] // E};")
    for r in range(RPT):
        inT = "act" if j == 1 else f"inT{j}_{r}"
        base = f"io{r}" if j == 1 else f"so{r}"
        pitch = lay["w0"] if j == 1 else W1

        def load(slot, off3, r=r, base=base, pitch=pitch):
            dz, dy, dx = off3
            if dz != 0 or (dy == 0 and dx == 0):
                return f"c{j - 1}_{r}_{rz + dz}"
            if dx == 0 and 0 <= r + dy < RPT:
                return f"c{j - 1}_{r + dy}_{rz}"  # the thread's own neighbouring row
            return f"P[{base} + {dy * pitch + dx}]"

        lines, res = _emit_expr(st, dtype, load)
        a(f"{ind}if ({inT}) {{")
        a(f"{ind}  T v;")
        a(f"{ind}  if (zin && sxy{r}) {{")
        for ln in lines:
            a(f"{ind}    {ln}")
        a(f"{ind}    v = {res};")
        if final:
            a(f"{ind}    adst[zoff + go{r}] = v;")
        elif j == K - 1:
            a(f"{ind}    if (p.wb && inT{K}_{r}) bmem[zoff + go{r}] = v;")
        a(f"{ind}  }} else {{")
        a(f"{ind}    v = {'(T)0' if final else f'h{j}_{r}'};")
        a(f"{ind}  }}")
        if not final:
            a(f"{ind}  W[so{r}] = v;")
            a(f"{ind}  c{j}_{r}_{2 * rz} = v;")
        a(f"{ind}}}")
    if not final:
        a(f"{ind}__syncwarp(); if (lane == 0) mbar_arrive(rb{j} + gw % {lay['rings'][j - 1]['n']});")
    a("      }")


def item_geometry(s_lo, s_hi, sm_count: int, lay: dict) -> dict:
    """Work-item tiling of the output box S (padded coordinates)."""
    cfg = lay["cfg"]
    nz, ny, nx = (b - a for a, b in zip(s_lo, s_hi))
    nbx, nby = -(-nx // lay.get("bx", cfg.bx)), -(-ny // lay.get("by", cfg.by))
    zc = min(cfg.zchunk, nz)
    nzc = -(-nz // zc)
    n_items = nbx * nby * nzc
    cap = sm_count * lay.get("min_blocks", 1)
    blocks = min(n_items, cap) if cfg.persistent else n_items
    return {"nbx": nbx, "nby": nby, "zc": zc, "nzc": nzc, "blocks": blocks}


def pack_params(tmap: bytes, src: int, bhome: int, adst: int, buf, s_lo, s_hi, geo: dict,
                write_b: bool = True) -> bytes:
    """Params block (layout mirrored in `source`). Pointers are padded-box
    origins (buffer base + xoff elements). `write_b` False skips B's stores:
    inside a run only the last chain's B survives (the next chain overwrites
    B before anything reads it), so earlier chains move 16 B per K LUP."""
    assert len(tmap) == 128
    npz, npy, npx = buf.nz, buf.pz // buf.py, buf.ext[2] + 2 * buf.depth[2]
    out = bytearray(tmap)
    out += struct.pack("<QQQqq", src, bhome, adst, buf.py, buf.pz)
    out += struct.pack("<15i", npz, npy, npx, buf.xoff, s_lo[0], s_hi[0], s_lo[1], s_hi[1],
                       s_lo[2], s_hi[2], geo["nbx"], geo["nby"], geo["zc"], geo["nzc"], int(write_b))
    return bytes(out) + b"\0" * ((-len(out)) % 64)


def complement_boxes(buf, src_base: int, dst_base: int, s_lo, s_hi) -> list:
    """Copy descriptors covering the padded box minus S (<= 6 boxes), from the
    buffer at `src_base` to an identically laid out one at `dst_base`."""
    from ._lib import EstBox

    npx = buf.ext[2] + 2 * buf.depth[2]
    n = (buf.nz, buf.pz // buf.py, npx)
    (z0, y0, x0), (z1, y1, x1) = s_lo, s_hi
    boxes = [((0, 0, 0), (z0, n[1], n[2])), ((z1, 0, 0), (n[0], n[1], n[2])),
             ((z0, 0, 0), (z1, y0, n[2])), ((z0, y1, 0), (z1, n[1], n[2])),
             ((z0, y0, 0), (z1, y1, x0)), ((z0, y0, x1), (z1, y1, n[2]))]
    out = []
    for lo, hi in boxes:
        ext = [b - a for a, b in zip(lo, hi)]
        if min(ext) <= 0:
            continue
        off = (buf.xoff + lo[0] * buf.pz + lo[1] * buf.py + lo[2]) * buf.elem
        out.append(EstBox(src_base + off, dst_base + off, buf.py, buf.pz, buf.py, buf.pz,
                          ext[2], ext[1], ext[0]))
    return out
