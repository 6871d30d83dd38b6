"""The "tb" skeleton: temporal blocking of K consecutive ping-pong sweeps.

A batch of heat/Jacobi iterations is a chain of single-statement rank-3 nodes
`B[S] = f(A[S + offsets]); A[S] = f(B[S + offsets]); ...` (
reference semantics executor.py:258-348: nodes run in order, statement at a
time). On one GPU with one tile no halo exchange happens between them, so K of
them (K even) run as ONE kernel that reads A once from HBM, keeps the
intermediate sweeps on chip and writes only the arrays' final values: A read
and A written once per K sweeps, B written only by a run's last chain
(`write_b`), i.e. 8 B/LUP for fp64 at K = 2 instead of 16 B/LUP for single
sweeps.

Every point is computed by the generated expression of codegen._emit_expr
(one correctly rounded IEEE op per plan instruction, no contraction), so the
results are bit-identical to K separate sweeps. Epochs, rounds and launch
counts are kept per node by the executor.

Kernel structure (one warp-specialised CTA per work item, one resident per SM):

* work item = a BX x BY output column of S over a z-chunk of ZC planes
  (chunks balanced so every item has the same depth; ~96 planes, shorter on
  small grids so there are >= 2048 items). Items are launched in order, one
  CTA each: the hardware dispatches the next item to whichever SM frees up,
  so the ~148 items in flight stay a contiguous band whose neighbours walk z
  together and share their overlapping halo columns / rows through L2. A
  persistent grid (CTA b taking items b, b+148, ...) lets CTAs drift apart by
  tens of planes over a launch and loses that reuse: C4 DRAM reads 12.6 GB vs
  10.6 GB per launch, 450 vs 525 GLUP/s (profiles/r2_tb_persistent_vs_inorder.md);
  `persistent=True` keeps the old schedule. x tiles start at a
  16-byte aligned padded column so every thread's V = 16/elem consecutive
  points are one 128-bit vector (fp64 pairs, fp32 quads) in shared memory and
  in HBM;
* step j (1..K) covers the tile expanded by m_j columns / (K-j)*ry rows
  (overlapped tiling; m_j rounded up to V) and trails step j-1 by rz planes;
* producer warp: one elected lane issues one TMA (`cp.async.bulk.tensor.3d`)
  per input plane (tile + halo) into an mbarrier ring (full/empty barriers),
  `prefetch` planes ahead of the compute window (persistent mode: running
  ahead into the CTA's next item);
* compute threads: thread (c, g) owns vector column c and RPT consecutive
  rows of the step-1 frame for every step and every plane. Its z-window of
  every step (2rz+1 planes) lives in registers and rotates by renaming (the
  plane loop is unrolled 2rz+1 times); in-plane neighbours come from shared
  memory: the TMA plane for step 1, step j's plane ring (rz+1 slots, the
  step-1 frame) for step j+1. Per plane a thread does one mbarrier wait, its
  vector loads / expressions / one vector store per row and step, and ONE
  named barrier; one thread releases the input slot after that barrier;
* items whose step-1 frame lies inside S in y/x take a predicate-free path;
  edge items keep the array's stored value at points outside S (prefetched
  before the plane's mbarrier wait) and store per component;
* stores: step K-1 (array B, final) in place, only in a run's last chain;
  step K (array A, final) into A's *other* home buffer, because neighbouring
  CTAs still read A through TMA. The executor alternates A between its tile
  buffer and a scratch twin (chains come in pairs, so A ends in its own
  buffer) and copies S's complement into the twin at the start of each run.

Earlier variants (a 2-row-per-thread scalar kernel with per-step mbarrier
rings, a warp-shuffle variant, an L2-forwarded wavefront and an L2-resident
grid-barrier chain) were measured slower and removed; their numbers are in
profiles/r1_tb_sweep.md and profiles/r1s2_tb_skipb.md.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

from .codegen import CTYPE, ELEM, StmtSig, _emit_expr, slot_radius
from .stream import _PTX_HELPERS

MAX_RADIUS = 2
SMEM_BUDGET = 220 * 1024
SMEM_PER_SM = 228 * 1024
SKIP_MID_B = os.environ.get("EST_TB_SKIPB", "1") == "1"
# measurement probes (wrong results, never scheduled by default): "noshared"
# replaces every in-plane operand by the centre value (no shared-memory loads)
PROBE = os.environ.get("EST_TB_PROBE", "")


@dataclass(frozen=True)
class TbCfg:
    k: int = 2              # sweeps per launch (even)
    bx: int = 64            # output columns per item (multiple of 16/elem)
    by: int = 32            # output rows per item
    rpt: int = 2            # consecutive step-1-frame rows per compute thread
    prefetch: int = 3       # input planes in flight beyond the z window
    zchunk: int = 96        # target planes per item (chunks are balanced)
    min_items: int = 2048   # shorter z chunks on small grids until there are this many items
    l2promo: int = 2        # TMA L2 promotion: 0 none, 1 64B, 2 128B, 3 256B
    persistent: bool = False  # one CTA per SM slot looping over items (else one CTA per item)
    hoist: bool = False     # issue every step's shared-memory loads at the top of a plane iteration


def _env_cfg() -> TbCfg:
    e = os.environ.get
    d = TbCfg()
    return TbCfg(k=int(e("EST_TB_K", d.k)), bx=int(e("EST_TB_BX", d.bx)), by=int(e("EST_TB_BY", d.by)),
                 rpt=int(e("EST_TB_RPT", d.rpt)), prefetch=int(e("EST_TB_PREFETCH", d.prefetch)),
                 zchunk=int(e("EST_TB_ZCHUNK", d.zchunk)), min_items=int(e("EST_TB_MIN_ITEMS", d.min_items)),
                 l2promo=int(e("EST_TB_L2PROMO", d.l2promo)),
                 persistent=e("EST_TB_PERSISTENT", "0") == "1", hoist=e("EST_TB_HOIST", "0") == "1")


DEFAULT = _env_cfg()
ENABLED = os.environ.get("EST_TB", "1") == "1"
# chains are scheduled from this many output points (smaller grids: too few
# items per SM to hide each item's pipeline fill)
MIN_POINTS = int(os.environ.get("EST_TB_MIN_POINTS", 1 << 26))
# chain depths that passed the GPU parity suite (EST_TB_VALIDATED_K widens it for experiments)
VALIDATED_K = tuple(int(k) for k in os.environ.get("EST_TB_VALIDATED_K", "2,4").split(","))


def _round(v: int, m: int) -> int:
    return -(-v // m) * m


def z_star(st: StmtSig) -> bool:
    """Every load off the centre plane is a pure z offset (dz, 0, 0)."""
    return all(i[2][0] == 0 or (i[2][1] == 0 and i[2][2] == 0) for i in st.instructions if i[0] == "load")


def layout(rad, dtype: int, cfg: TbCfg) -> dict:
    """Frames, margins, thread grid and shared memory of the chain kernel.

    x margins m_j (columns each side of the output tile that step j computes)
    are rounded to the vector width V so every frame starts on a vector; y
    margins are e_j = (K-j)*ry. Frame 0 is the TMA input plane, frames 1..K-1
    are the intermediate steps' plane rings (all in the step-1 geometry)."""
    rz, ry, rx = rad
    elem = ELEM[dtype]
    V = 16 // elem
    K = cfg.k
    m = [0] * (K + 1)
    for j in range(K - 1, -1, -1):
        m[j] = _round(m[j + 1] + rx, V)
    e = [(K - j) * ry for j in range(K + 1)]
    W0, H0 = cfg.bx + 2 * m[0], cfg.by + 2 * e[0]
    W1, H1 = cfg.bx + 2 * m[1], cfg.by + 2 * e[1]
    P1 = W1 // V
    G1 = -(-H1 // cfg.rpt)
    nact = P1 * G1
    NT = _round(nact, 32)
    Z = 2 * rz + 1
    s0 = rz + 1 + cfg.prefetch
    # every thread (active or not) computes its whole footprint unpredicated:
    # the frames are padded with the rows the last row group reads
    rows_t = -(-NT // P1) * cfg.rpt
    pl0 = _round(W0 * max(H0, (e[0] - e[1]) + rows_t + ry) * elem + 2 * elem * V, 128)
    pl1 = _round(W1 * max(H1, rows_t + ry) * elem + 2 * elem * V, 128)
    rings = []
    off = s0 * pl0
    R = rz + 1  # plane slots per intermediate ring (written at t, read rz iterations later)
    for _j in range(1, K):
        rings.append(off)
        off += R * pl1
    data = _round(off, 8)
    smem = data + 8 * 2 * s0 + 1024
    return {"rad": (rz, ry, rx), "V": V, "m": m, "e": e, "w0": W0, "h0": H0, "w1": W1, "h1": H1,
            "p1": P1, "g1": G1, "nact": nact, "nt": NT, "Z": Z, "R": R, "s0": s0, "pl0": pl0, "pl1": pl1,
            "rings": rings, "data": data, "smem": smem, "cfg": cfg, "elem": elem, "bx": cfg.bx, "by": cfg.by}


def eligible(st: StmtSig, dtype: int, cfg: TbCfg | None = None) -> bool:
    """Single input slot, z-star loads, 1 <= rz, radius <= MAX_RADIUS, fits."""
    cfg = cfg or DEFAULT
    if (cfg.k not in VALIDATED_K or cfg.k % 2 or st.arity != 1 or dtype not in ELEM or not z_star(st)
            or cfg.bx % (16 // ELEM.get(dtype, 8))):
        return False
    rad = slot_radius(st).get(0)
    if rad is None or max(rad) > MAX_RADIUS or rad[0] < 1:
        return False
    lay = layout(rad, dtype, cfg)
    if lay["w0"] > 256 or lay["h0"] > 256 or lay["nt"] + 32 > 1024:
        return False
    return lay["smem"] <= SMEM_BUDGET


def blocks_per_sm(smem: int, nt: int) -> int:
    return max(1, min(SMEM_PER_SM // (smem + 1024), 2048 // (nt + 32)))


class _Emitter:
    """Source text builder for one (statement, dtype, cfg, buffer layout) chain kernel."""

    def __init__(self, st: StmtSig, dtype: int, lay: dict, py: int, pz: int, xoff: int):
        self.st, self.dtype, self.lay = st, dtype, lay
        self.py, self.pz, self.xoff = py, pz, xoff
        self.T = CTYPE[dtype]
        self.VT = {8: "double2", 4: "float4"}[lay["elem"]]
        self.L: list = []

    def a(self, s: str) -> None:
        self.L.append(s)

    @staticmethod
    def _rn(x: int) -> str:
        return f"m{-x}" if x < 0 else str(x)

    def step_body(self, j: int, mm: int) -> tuple:
        """Expression lines of step j for every (row, component) of the
        thread at unroll position mm, and the shared-memory operands they
        need, grouped by (thread-relative row, vector group)."""
        lay = self.lay
        V, RPT, Z = lay["V"], lay["cfg"].rpt, lay["Z"]
        rz = lay["rad"][0]
        need: dict = {}
        body = []
        for r in range(RPT):
            for v in range(V):
                def load(slot, off3, r=r, v=v):
                    dz, dy, dx = off3
                    if PROBE == "noshared":  # measurement probe: in-plane operands from registers
                        dy, dx = 0, 0
                    if dz != 0 or (dy == 0 and dx == 0):
                        return f"c{j - 1}_{r}_{v}_{(rz + dz + mm) % Z}"
                    rr, xc = r + dy, v + dx
                    if 0 <= rr < RPT and 0 <= xc < V:
                        return f"c{j - 1}_{rr}_{xc}_{(rz + mm) % Z}"
                    g, comp = xc // V, xc % V
                    need.setdefault((rr, g), set()).add(comp)
                    return f"n{j}_{self._rn(rr)}_{self._rn(g)}_{comp}"
                lines, res = _emit_expr(self.st, self.dtype, load)
                body.append((r, v, lines, res))
        return body, need

    def emit_smem_loads(self, ind: str, j: int, need: dict, base: str, pitch: int) -> None:
        """Step j's shared-memory operands: one vector load per group with >= 2
        needed components, else scalars.

        A row's west / east neighbours (the last component of the vector to
        the left, the first of the vector to the right) are loaded as a
        crossed pair: half of the lanes of every bank phase (8 lanes for
        64-bit loads, which the LSU serves per half-warp; 16 for 32-bit)
        fetch west then east, the other half east then west. At a 16-byte
        lane stride each scalar load of one neighbour alone uses half of the
        banks twice; the crossed halves use disjoint bank sets."""
        V = self.lay["V"]
        need = dict(need)
        for rr in sorted({k[0] for k in need}):
            if need.get((rr, -1)) == {V - 1} and need.get((rr, 1)) == {0}:
                del need[(rr, -1)], need[(rr, 1)]
                t = f"{j}_{self._rn(rr)}"
                self.a(f"{ind}const {self.T} xa{t} = {base}[{rr * pitch - 1} + sw];")
                self.a(f"{ind}const {self.T} xb{t} = {base}[{rr * pitch + V} - sw];")
                self.a(f"{ind}const {self.T} n{t}_m1_{V - 1} = xw ? xb{t} : xa{t};")
                self.a(f"{ind}const {self.T} n{t}_1_0 = xw ? xa{t} : xb{t};")
        for (rr, g), comps in sorted(need.items()):
            off = rr * pitch + g * V
            tag = f"{j}_{self._rn(rr)}_{self._rn(g)}"
            if len(comps) >= 2:
                self.a(f"{ind}const {self.VT} q{tag} = *reinterpret_cast<const {self.VT}*>({base} + ({off}));")
                for c in sorted(comps):
                    self.a(f"{ind}const {self.T} n{tag}_{c} = q{tag}.{'xyzw'[c]};")
            else:
                (c,) = tuple(comps)
                self.a(f"{ind}const {self.T} n{tag}_{c} = {base}[{off + c}];")

    # -- kernel ---------------------------------------------------------------
    def source(self) -> str:
        lay = self.lay
        cfg = lay["cfg"]
        K, RPT, V, Z = cfg.k, cfg.rpt, lay["V"], lay["Z"]
        rz = lay["rad"][0]
        m, e = lay["m"], lay["e"]
        W0, H0, W1, H1, P1 = lay["w0"], lay["h0"], lay["w1"], lay["h1"], lay["p1"]
        NT, s0, E = lay["nt"], lay["s0"], lay["elem"]
        a = self.a
        NW = NT // 32
        minb = max(1, min(blocks_per_sm(lay["smem"], NT), 65536 // ((NT + 32) * 96)))
        lay["min_blocks"] = minb
        a(f'// generated by paper_2512_19851_b200/temporal.py — skeleton "tb" (K={K} fused sweeps, '
          f'V={V} vectors) {cfg} py={self.py} pz={self.pz} xoff={self.xoff}')
        a(f"typedef {self.T} T;")
        a("struct __align__(64) Tmap { unsigned long long w[16]; };")
        a("struct __align__(64) Params { Tmap tm;")
        a("  unsigned long long src, bhome, adst;  // padded-box origins: A now, B (in place), A next")
        a("  int npz, npy, npx, sz0, sz1, sy0, sy1, sx0, sx1, xt0, nbx, nby, zc, nzc, wb, cz0, cz1; };")
        a(_PTX_HELPERS)
        a("__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {")
        a("  asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(smem_u32(b)) : \"memory\"); }")
        a("__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {")
        a("  unsigned ok; asm volatile(\"{\\n .reg .pred p;\\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\\n\"")
        a("  \" selp.u32 %0, 1, 0, p;\\n}\" : \"=r\"(ok) : \"r\"(smem_u32(b)), \"r\"(parity) : \"memory\"); return ok; }")
        a("__device__ __forceinline__ void mbar_wait2(unsigned long long* b, unsigned parity) {")
        a("  if (!mbar_try(b, parity)) mbar_wait(b, parity); }  // fast first probe, bounded slow path")
        a(f'extern "C" __global__ void __launch_bounds__({NT + 32}, {minb})')
        a("est_tb(const __grid_constant__ Params p) {")
        a("  extern __shared__ __align__(1024) unsigned char smem[];")
        a(f"  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + {lay['data']});")
        a(f"  unsigned long long* empty = full + {s0};")
        a("  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;")
        a("  const int n_items = p.nbx * p.nby * p.nzc;")
        a("  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");")
        a("  if (tid == 0) {")
        a(f"    for (int i = 0; i < {s0}; ++i) {{ mbar_init(full + i, 1); mbar_init(empty + i, 1); }}")
        a("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");")
        a("  }")
        a("  __syncthreads();")
        a("  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");  // the previous chain's stores are visible")

        def item_decode(ind):
            a(f"{ind}const int bx = item % p.nbx, rest = item / p.nbx;")
            a(f"{ind}const int by = rest % p.nby, bzc = rest / p.nby;")
            a(f"{ind}const int x0 = p.xt0 + bx * {cfg.bx}, y0 = p.sy0 + by * {cfg.by};")
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
        a("      for (int k = 0; k < n0; ++k) {")
        a(f"        const int g = fill + k, stg = g % {s0};")
        a(f"        if (g >= {s0}) mbar_wait(empty + stg, ((g / {s0}) - 1) & 1);")
        a(f"        mbar_expect(full + stg, {W0 * H0 * E});")
        a(f"        tma_load3(smem + stg * {lay['pl0']}, &p.tm, x0 + {self.xoff - m[0]}, y0 - {e[0]}, "
          f"zs - {K * rz} + k, full + stg);")
        a("      }")
        a("      fill += n0;")
        a("    }")
        a("    return;")
        a("  }")
        # ---------------- compute threads
        a("  const T* __restrict__ asrc = reinterpret_cast<const T*>(p.src);")
        a("  T* __restrict__ bmem = reinterpret_cast<T*>(p.bhome);")
        a("  T* __restrict__ adst = reinterpret_cast<T*>(p.adst);")
        a(f"  const bool act = tid < {lay['nact']};")
        a(f"  const bool xw = (lane & {8 if V == 2 else 16}) != 0;  // crossed west/east neighbour loads")
        a(f"  const int sw = xw ? {V + 1} : 0;")
        a("  const int wb = p.wb, cz0 = p.cz0, cz1 = p.cz1, npz = p.npz;  // cz: S's planes in reach")
        a(f"  const int cc = tid % {P1}, gg = tid / {P1};  // vector column / row group in the step-1 frame")
        a(f"  const int off0 = ({e[0] - e[1]} + gg * {RPT}) * {W0} + {m[0] - m[1]} + cc * {V};  // input frame")
        a(f"  const int off1 = gg * {RPT} * {W1} + cc * {V};  // step-1 frame (rings)")
        for j in range(1, K + 1):
            dm, de = (m[1] - m[j]) // V, e[1] - e[j]
            for r in range(RPT):
                a(f"  const bool in{j}_{r} = act && (gg * {RPT} + {r}) >= {de} && (gg * {RPT} + {r}) < {H1 - de}"
                  f" && cc >= {dm} && cc < {P1 - dm};")
        for j in range(0, K):
            for r in range(RPT):
                for v in range(V):
                    a(f"  T {', '.join(f'c{j}_{r}_{v}_{k} = 0' for k in range(Z))};")
        a("  int is = 0, ip = 0;  // input ring slot / phase of plane t")
        a("  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {")
        item_decode("    ")
        a(f"    const long long gb = (long long)(y0 - {e[1]} + gg * {RPT}) * {self.py} + (x0 - {m[1]} + cc * {V});")
        a(f"    const bool fast = (x0 - {m[1]} >= p.sx0) && (x0 + {cfg.bx + m[1]} <= p.sx1) &&"
          f" (y0 - {e[1]} >= p.sy0) && (y0 + {cfg.by + e[1]} <= p.sy1);")
        a("    if (fast) {")
        self.emit_loop("      ", edge=False)
        a("    } else {")
        # per-thread S / padded-box predicates of the item (edge items only)
        for r in range(RPT):
            a(f"      const int gy{r} = y0 - {e[1]} + gg * {RPT} + {r};")
            a(f"      const bool ys{r} = gy{r} >= p.sy0 && gy{r} < p.sy1, yp{r} = gy{r} >= 0 && gy{r} < p.npy;")
        for v in range(V):
            a(f"      const int gx{v} = x0 - {m[1]} + cc * {V} + {v};")
            a(f"      const bool xs{v} = gx{v} >= p.sx0 && gx{v} < p.sx1, xp{v} = gx{v} >= 0 && gx{v} < p.npx;")
        self.emit_loop("      ", edge=True)
        a("    }")
        a("  }")
        a("}")
        return "\n".join(self.L) + "\n"

    def emit_loop(self, ind: str, edge: bool) -> None:
        """The plane loop of one item, unrolled Z = 2rz+1 times (register
        windows rotate by renaming). Every thread computes every row and
        component of its footprint (no divergent branches; frames are padded
        so out-of-region operands stay inside shared memory); only stores
        and global loads are predicated."""
        lay = self.lay
        cfg = lay["cfg"]
        K, RPT, V, Z = cfg.k, cfg.rpt, lay["V"], lay["Z"]
        rz = lay["rad"][0]
        W0, W1, s0, E = lay["w0"], lay["w1"], lay["s0"], lay["elem"]
        pl0, pl1 = lay["pl0"] // E, lay["pl1"] // E
        PY, PZ = self.py, self.pz
        NT = lay["nt"]
        VT = self.VT
        a = self.a
        a(f"{ind}T* ap = adst + (long long)zs * {PZ} + gb;  // step-K plane (A next)")
        a(f"{ind}T* bp = bmem + (long long)(zs - {rz}) * {PZ} + gb;  // step-(K-1) plane (B)")
        a(f"{ind}const T* ring0 = reinterpret_cast<const T*>(smem);")
        a(f"{ind}int tr = 0;  // t mod R (intermediate ring slots)")
        a(f"{ind}for (int t0 = 0; t0 < n0; t0 += {Z}) {{")
        for mm in range(Z):
            i2 = ind + "  "
            a(f"{i2}if (t0 + {mm} < n0) {{  // plane iteration t = t0 + {mm}")
            i3 = i2 + "  "
            a(f"{i3}const int t = t0 + {mm};")
            for j in range(1, K):
                a(f"{i3}const int u{j} = zs - {(K + j) * rz} + t;  // step-{j} plane")
                a(f"{i3}const bool zs{j} = u{j} >= cz0 && u{j} < cz1, zp{j} = u{j} >= 0 && u{j} < npz;")
                if edge:
                    # stored values outside S, prefetched before the plane's wait
                    home = "bmem" if j % 2 == 1 else "asrc"
                    for r in range(RPT):
                        for v in range(V):
                            a(f"{i3}T h{j}_{r}_{v} = (T)0;")
                            a(f"{i3}if (t >= {2 * j * rz} && in{j}_{r} && zp{j} && yp{r} && xp{v} && "
                              f"!(zs{j} && ys{r} && xs{v})) h{j}_{r}_{v} = "
                              f"{home}[(long long)u{j} * {PZ} + gb + {r * PY + v}];")
            a(f"{i3}mbar_wait2(full + is, ip);")
            a(f"{i3}{{ const T* S0 = ring0 + is * {pl0} + off0;  // own points of input plane t")
            for r in range(RPT):
                a(f"{i3}  {{ const {VT} q = *reinterpret_cast<const {VT}*>(S0 + {r * W0});")
                a(f"{i3}    " + " ".join(f"c0_{r}_{v}_{(2 * rz + mm) % Z} = q.{'xyzw'[v]};" for v in range(V)) + " }")
            a(f"{i3}}}")
            a(f"{i3}int ir = is - {rz}; if (ir < 0) ir += {s0};  // slot of plane t - rz")
            # with cfg.hoist every step's in-plane operands are loaded first: step 1
            # reads the TMA plane of t - rz, step j > 1 the ring plane step j-1
            # wrote rz iterations ago (behind the previous iteration's barrier),
            # so all loads of the iteration are in flight before the first
            # expression needs them (more live registers)
            bodies, loads = {}, {}
            for j in range(1, K + 1):
                if j == 1:
                    ptr = f"const T* P1 = ring0 + ir * {pl0} + off0;"
                    pitch = W0
                else:
                    R = lay["R"]
                    c = (rz + 2 * (j - 1) * rz) % R
                    ptr = (f"int rs{j} = tr - {c}; if (rs{j} < 0) rs{j} += {R};  // ring {j - 1} slot of plane u{j}\n"
                           f"const T* P{j} = reinterpret_cast<const T*>(smem + {lay['rings'][j - 2]}) + "
                           f"rs{j} * {pl1} + off1;")
                    pitch = W1
                body, need = self.step_body(j, mm)
                bodies[j] = body
                loads[j] = (ptr, need, pitch)
                if cfg.hoist:
                    for ln in ptr.split("\n"):
                        a(f"{i3}{ln}")
                    self.emit_smem_loads(i3, j, need, f"P{j}", pitch)
            for j in range(1, K + 1):
                final = j == K
                a(f"{i3}if (t >= {2 * j * rz}) {{  // step {j}")
                i4 = i3 + "  "
                if not final:
                    R = lay["R"]
                    c = (2 * j * rz) % R
                    a(f"{i4}int ws = tr - {c}; if (ws < 0) ws += {R};  // ring {j} slot of plane u{j}")
                    a(f"{i4}T* Wr = reinterpret_cast<T*>(smem + {lay['rings'][j - 1]}) + ws * {pl1} + off1;")
                    a(f"{i4}if (zs{j}) {{")
                else:
                    a(f"{i4}{{")
                i5 = i4 + "  "
                if not cfg.hoist:
                    ptr, need, pitch = loads[j]
                    for ln in ptr.split("\n"):
                        a(f"{i5}{ln}")
                    self.emit_smem_loads(i5, j, need, f"P{j}", pitch)
                body = bodies[j]
                for r, v, lines, res in body:
                    a(f"{i5}T o{r}_{v};")
                    a(f"{i5}{{ " + " ".join(lines) + f" o{r}_{v} = {res}; }}")
                for r in range(RPT):
                    outs = [f"o{r}_{v}" for v in range(V)]
                    if edge and not final:
                        for v in range(V):
                            a(f"{i5}if (!(ys{r} && xs{v})) o{r}_{v} = h{j}_{r}_{v};")
                    vec = f"make_{VT}({', '.join(outs)})"
                    if not final:
                        a(f"{i5}*reinterpret_cast<{VT}*>(Wr + {r * W1}) = {vec};")
                        a(f"{i5}" + " ".join(f"c{j}_{r}_{v}_{(2 * rz + mm) % Z} = o{r}_{v};" for v in range(V)))
                    targets = []
                    if final:
                        targets.append(("ap", f"in{K}_{r}"))
                    if j == K - 1:
                        targets.append(("bp", f"wb && in{K}_{r} && u{j} >= zs && u{j} < zs + nzl"))
                    for ptr, cond in targets:
                        if not edge:
                            a(f"{i5}if ({cond}) *reinterpret_cast<{VT}*>({ptr} + {r * PY}) = {vec};")
                        else:
                            allin = " && ".join(f"xs{v}" for v in range(V))
                            a(f"{i5}if ({cond} && ys{r}) {{")
                            a(f"{i5}  if ({allin}) *reinterpret_cast<{VT}*>({ptr} + {r * PY}) = {vec};")
                            a(f"{i5}  else {{ " + " ".join(f"if (xs{v}) {ptr}[{r * PY + v}] = o{r}_{v};"
                                                          for v in range(V)) + " }")
                            a(f"{i5}}}")
                a(f"{i4}}}")
                if not final:
                    # plane outside S: the array's stored value (0 beyond the padded box)
                    home = "bmem" if j % 2 == 1 else "asrc"
                    a(f"{i4}else {{")
                    for r in range(RPT):
                        vals = []
                        for v in range(V):
                            guard = f"zp{j} && in{j}_{r}" + (f" && yp{r} && xp{v}" if edge else "")
                            a(f"{i4}  const T s{r}_{v} = ({guard}) ? "
                              f"{home}[(long long)u{j} * {PZ} + gb + {r * PY + v}] : (T)0;")
                            vals.append(f"s{r}_{v}")
                        a(f"{i4}  *reinterpret_cast<{VT}*>(Wr + {r * W1}) = make_{VT}({', '.join(vals)});")
                        a(f"{i4}  " + " ".join(f"c{j}_{r}_{v}_{(2 * rz + mm) % Z} = s{r}_{v};" for v in range(V)))
                    a(f"{i4}}}")
                if final:
                    a(f"{i4}ap += {PZ};")
                if j == K - 1:
                    a(f"{i4}bp += {PZ};")
                a(f"{i3}}}")
            a(f"{i3}asm volatile(\"bar.sync 1, {NT};\" ::: \"memory\");")
            a(f"{i3}if (tid == 0 && t >= {rz}) mbar_arrive(empty + ir);  // plane t - rz fully consumed")
            a(f"{i3}if (++is == {s0}) {{ is = 0; ip ^= 1; }}")
            if K > 1:
                a(f"{i3}if (++tr == {lay['R']}) tr = 0;")
            a(f"{i2}}}")
        a(f"{ind}}}")
        # planes never used as a step-1 centre plane in this item: release their slots
        a(f"{ind}if (tid == 0) for (int k = (n0 > {rz} ? n0 - {rz} : 0); k < n0; ++k) {{")
        a(f"{ind}  int sl = is - n0 + k; while (sl < 0) sl += {s0}; mbar_arrive(empty + sl); }}")


def source(st: StmtSig, dtype: int, cfg: TbCfg | None = None, py: int = 1056, pz: int = 1056 * 1026,
           xoff: int = 15) -> tuple:
    """-> (source, kernel name, block, smem, layout). The buffer pitches (and
    the padded-box x offset) are compile-time constants so row and plane
    offsets are immediates; `py`/`pz` default to the C4 layout (1024^3 fp64,
    depth 1) for prebuilding."""
    cfg = cfg or DEFAULT
    rad = slot_radius(st)[0]
    lay = layout(rad, dtype, cfg)
    src = _Emitter(st, dtype, lay, py, pz, xoff).source()
    lay["blocks_per_sm"] = lay["min_blocks"]
    return src, "est_tb", (lay["nt"] + 32, 1, 1), lay["smem"], lay


def item_geometry(s_lo, s_hi, sm_count: int, lay: dict, xoff: int = 0) -> dict:
    """Work-item tiling of the output box S (padded coordinates): x tiles
    start at the vector-aligned column at or below S's first column, z chunks
    are balanced (every item has the same number of planes but the last)."""
    cfg = lay["cfg"]
    V = lay["V"]
    nz, ny = s_hi[0] - s_lo[0], s_hi[1] - s_lo[1]
    xt0 = s_lo[2] - ((xoff + s_lo[2]) % V)
    nbx = -(-(s_hi[2] - xt0) // cfg.bx)
    nby = -(-ny // cfg.by)
    nzc = max(1, -(-nz // max(1, cfg.zchunk)))
    if nbx * nby * nzc < cfg.min_items:  # small grids: more, shorter items (C2 510^3: 32-plane chunks)
        nzc = max(nzc, min(-(-cfg.min_items // (nbx * nby)), max(1, nz // 16)))
    zc = -(-nz // nzc)
    nzc = -(-nz // zc)
    n_items = nbx * nby * nzc
    cap = sm_count * lay.get("min_blocks", 1)
    blocks = min(n_items, cap) if cfg.persistent else n_items
    return {"nbx": nbx, "nby": nby, "zc": zc, "nzc": nzc, "blocks": blocks, "xt0": xt0}


def pack_params(tmap: bytes, src: int, bhome: int, adst: int, buf, s_lo, s_hi, geo: dict,
                write_b: bool = True, cz=None) -> bytes:
    """Params block (layout mirrored in `source`). Pointers are padded-box
    origins (buffer base + xoff elements). `write_b` False skips B's stores:
    inside a run only the last chain's B survives (the next chain overwrites
    B before anything reads it), so earlier chains move 16 B per K LUP.
    `cz` = the padded planes [cz0, cz1) where the intermediate steps COMPUTE
    the statement (the global output slice within reach of this tile): on a
    slab of a multi-tile job it extends past the tile's own output planes
    into the ghost planes that belong to the neighbour's output (default:
    the tile's own output planes [s_lo[0], s_hi[0]))."""
    assert len(tmap) == 128
    npz, npy, npx = buf.nz, buf.pz // buf.py, buf.ext[2] + 2 * buf.depth[2]
    cz0, cz1 = cz if cz is not None else (s_lo[0], s_hi[0])
    out = bytearray(tmap)
    out += struct.pack("<QQQ", src, bhome, adst)
    out += struct.pack("<17i", npz, npy, npx, s_lo[0], s_hi[0], s_lo[1], s_hi[1],
                       s_lo[2], s_hi[2], geo["xt0"], geo["nbx"], geo["nby"], geo["zc"], geo["nzc"], int(write_b),
                       cz0, cz1)
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
