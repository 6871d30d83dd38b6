"""The "tc" skeleton: two fused sweeps of a rank-2 chain in one launch.

Large 2-D runs stream from HBM (BASELINE C3: the acoustic wave at 16384^2
fp32; the paper's 2-D Laplace at 16384^2 fp64). Two consecutive nodes of such
a run are fused into one kernel that reads the run's inputs once and keeps the
intermediate sweep on chip (reference semantics
executor.py:258-348: nodes run in order, statement at a time). Two chain
shapes are recognised (executor.temporal_schedule):

* ping-pong (arity 1): `B[S] = f(A[S+o]); A[S] = f(B[S+o])` — the 2-D
  counterpart of temporal.py;
* rotation (arity 2, a second input read at the centre only):
  `X1[S] = f(Q[S+o], P[S]); P[S] = f(X1[S+o], Q[S])` — three arrays rotating,
  as the second-order-in-time wave `u2 = f(u1, u0)` (programs.wave2d_steps).

Traffic per two LUP: ping-pong reads A and writes A (B only in a run's last
chain), rotation reads Q and P and writes X1 and P — 8 B/LUP in fp32
rotation / fp64 ping-pong instead of 12 / 16 B for single sweeps.

Every point is the codegen expression (one correctly rounded IEEE op per plan
instruction), so the results are bit-identical to node-by-node execution.

Kernel (one CTA per work item, several CTAs per SM):

* work item = BX output columns of S over a chunk of rows, streamed along y
  (axis 0) in stages of RB rows: a producer warp issues per stage one TMA of
  the RB rows of Q (the input frame: BX + 2*m0 columns) and, for rotations,
  one of P (same frame; the step-1 frame is its centre) onto the stage's
  mbarrier;
* compute thread c owns one 16-byte vector column (fp32 quads, fp64 pairs)
  of the step-1 frame. Its y-neighbours of both steps live in registers
  (windows of RB + 2*ry rows), x-neighbours come from shared memory: the Q
  stage for step 1, a ring of step-1 rows (three banks of RB rows: written
  by this stage, read back by this stage and the next) for step 2;
* per stage: step 1 for RB rows (row t - ry of input row t), one named
  barrier, step 2 for RB rows (row t - 2*ry), so one barrier per RB rows;
  interior stages of items inside S in x run a variant without row / column
  checks;
* step-1 rows / columns outside S take the intermediate array's stored value
  (the state of node-by-node execution); stores: X1 in place at S (a
  ping-pong skips it except in a run's last chain), the step-2 array into its
  OTHER buffer, because neighbouring CTAs still read its current one (P's
  margin through TMA, or A itself). The executor alternates that array
  between its tile buffer and a twin.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

from .codegen import CTYPE, ELEM, StmtSig, _emit_expr, slot_radius
from .stream import _PTX_HELPERS

MAX_RADIUS = 2
SMEM_PER_SM = 228 * 1024


@dataclass(frozen=True)
class TcCfg:
    bx: int = 0          # output columns per item (0: the widest whose TMA box fits 256)
    rb: int = 0          # rows per stage (0: auto, 2*ry + 1 and at least 4 for ping-pong)
    prefetch: int = 1    # stages in flight beyond the two being read
    ychunk: int = 512    # target rows per item (chunks are balanced)
    min_items: int = 2048
    l2promo: int = 2
    vec: int = 0         # bytes per thread vector (0: auto, 8 = fp32 pairs for rotations, else 16)


def _env_cfg() -> TcCfg:
    e = os.environ.get
    d = TcCfg()
    return TcCfg(bx=int(e("EST_TC_BX", d.bx)), rb=int(e("EST_TC_RB", d.rb)),
                 prefetch=int(e("EST_TC_PREFETCH", d.prefetch)), ychunk=int(e("EST_TC_YCHUNK", d.ychunk)),
                 min_items=int(e("EST_TC_MIN_ITEMS", d.min_items)), l2promo=int(e("EST_TC_L2PROMO", d.l2promo)),
                 vec=int(e("EST_TC_VEC", d.vec)))


DEFAULT = _env_cfg()
ENABLED = os.environ.get("EST_TC", "1") == "1"
# rotation chains (the wave) are correct but lose to single sweeps at C3
# (523 vs 548 GLUP/s: the single-sweep kernel already moves 12 B/LUP at the
# copy roofline, the chain's 8 B/LUP run at ~4.2 TB/s); opt-in
ROTATIONS = os.environ.get("EST_TC_ROT", "0") == "1"
# chains are scheduled from this many output points (below: the single-sweep
# stream kernel or the shared-memory-resident chain)
MIN_POINTS = int(os.environ.get("EST_TC_MIN_POINTS", 1 << 24))


def _round(v: int, m: int) -> int:
    return -(-v // m) * m


def _loads(st: StmtSig, slot: int) -> list:
    return [i[2] for i in st.instructions if i[0] == "load" and i[1] == slot]


def roles(st: StmtSig):
    """(stencil slot, centre slot or None) of a chainable statement, else None.

    The stencil slot's loads are y-star (off the centre row only pure y
    offsets) with 1 <= ry and radius <= MAX_RADIUS; the centre slot (arity 2)
    is read at offset 0 only."""
    if st.arity not in (1, 2):
        return None
    rad = slot_radius(st)
    centre = [s for s in range(st.arity) if all(o == (0, 0, 0) for o in _loads(st, s))]
    if st.arity == 1:
        sten = 0
        cen = None
    else:
        if len(centre) != 1:
            return None
        cen = centre[0]
        sten = 1 - cen
    r = rad.get(sten)
    if r is None or r[0] != 0 or r[1] < 1 or max(r) > MAX_RADIUS:
        return None
    if any(o[1] != 0 and o[2] != 0 for o in _loads(st, sten)):
        return None
    return sten, cen


def layout(st: StmtSig, dtype: int, cfg: TcCfg) -> dict:
    sten, cen = roles(st)
    _rz, ry, rx = slot_radius(st)[sten]
    elem = ELEM[dtype]
    vec = cfg.vec or (8 if (cen is not None and elem == 4) else 16)
    V = max(2, vec // elem)
    A = 16 // elem  # TMA boxes must start on a 16-byte aligned column
    m1 = _round(rx, V)
    m0 = _round(m1 + rx, A)
    bx = cfg.bx or (256 - 2 * m0) // A * A
    W0, W1 = bx + 2 * m0, bx + 2 * m1
    RB = cfg.rb or (2 * ry + 1 if cen is not None else max(2 * ry + 1, 4))
    RB = max(RB, ry)
    P1 = W1 // V
    NT = _round(P1, 32)
    S0 = 2 + cfg.prefetch
    qb = _round(RB * W0 * elem, 128)
    # P is staged in the Q frame geometry (W0 columns): both TMA boxes then
    # have the same inner extent, a multiple of 32 bytes
    pb = _round(RB * W0 * elem, 128) if cen is not None else 0
    stage = qb + pb
    C1 = 3 * RB  # three banks of RB step-1 rows (this stage, the previous, the next)
    W1p = W1 + 2 * V
    ring1 = S0 * stage
    data = _round(ring1 + C1 * W1p * elem, 8)
    smem = data + 16 * S0 + 128
    return {"sten": sten, "cen": cen, "ry": ry, "rx": rx, "V": V, "m0": m0, "m1": m1, "bx": bx,
            "w0": W0, "w1": W1, "rb": RB, "p1": P1, "nt": NT, "s0": S0, "qb": qb, "pb": pb,
            "stage": stage, "c1": C1, "w1p": W1p, "ring1": ring1, "data": data, "smem": smem,
            "cfg": cfg, "elem": elem}


def eligible(st: StmtSig, dtype: int, cfg: TcCfg | None = None) -> bool:
    cfg = cfg or DEFAULT
    if dtype not in ELEM or roles(st) is None:
        return False
    lay = layout(st, dtype, cfg)
    if (lay["bx"] < lay["V"] or lay["bx"] % (16 // lay["elem"]) or (lay["m0"] - lay["m1"]) % lay["V"]
            or lay["w0"] > 256 or lay["nt"] + 32 > 1024):
        return False
    return lay["smem"] <= 200 * 1024


def blocks_per_sm(lay: dict) -> int:
    return max(1, min(SMEM_PER_SM // (lay["smem"] + 1024), 2048 // (lay["nt"] + 32), 32))


class _Emitter:
    def __init__(self, st: StmtSig, dtype: int, lay: dict, py: int, xoff: int):
        self.st, self.dtype, self.lay, self.py, self.xoff = st, dtype, lay, py, xoff
        self.T = CTYPE[dtype]
        self.VT = {(8, 2): "double2", (4, 4): "float4", (4, 2): "float2"}[(lay["elem"], lay["V"])]
        self.L: list = []

    def a(self, s: str) -> None:
        self.L.append(s)

    def _expr(self, step: int, i: int, v: int, need: dict) -> tuple:
        """Expression of component v at unroll position i of `step`.

        Step 1: stencil slot = Q (y-neighbours q[i+ry+dy], x-neighbours from
        the Q stage row of iteration t-ry), centre slot = P (stage row i).
        Step 2: stencil slot = X1 (x[i+ry+dy], x-neighbours from the ring row
        of iteration t-ry), centre slot = Q (q[i])."""
        lay = self.lay
        V, ry = lay["V"], lay["ry"]
        sten, cen = lay["sten"], lay["cen"]
        win = "q" if step == 1 else "x"

        def load(slot, off3):
            _dz, dy, dx = off3
            if slot == cen:
                return f"p{i}_{v}" if step == 1 else f"q{i}_{v}"
            if dx == 0:
                return f"{win}{i + ry + dy}_{v}"
            xc = v + dx
            if 0 <= xc < V:
                return f"{win}{i + ry}_{xc}"
            side = "l" if xc < 0 else "r"
            comp = xc % V
            need.setdefault(side, set()).add(comp)
            return f"n{step}{side}{i}_{comp}"

        return _emit_expr(self.st, self.dtype, load)

    def _nbr_loads(self, ind: str, step: int, i: int, need: dict, base: str) -> None:
        for side, comps in sorted(need.items()):
            off = -self.lay["V"] if side == "l" else self.lay["V"]
            self.a(f"{ind}const {self.VT} nv{step}{side}{i} = *reinterpret_cast<const {self.VT}*>({base} + ({off}));")
            for c in sorted(comps):
                self.a(f"{ind}const {self.T} n{step}{side}{i}_{c} = nv{step}{side}{i}.{'xyzw'[c]};")

    def emit_stage(self, ind: str, fast: bool) -> None:
        """One stage: step 1 for RB rows, the named barrier, step 2 for RB rows.
        The fast variant (interior stages of items inside S in x) has no row
        or column checks."""
        lay, a = self.lay, self.a
        V, ry, RB, NT = lay["V"], lay["ry"], lay["rb"], lay["nt"]
        W0, W1p = lay["w0"], lay["w1p"]
        rot = lay["cen"] is not None
        PY, VT, T = self.py, self.VT, self.T
        a(f"{ind}const long long r1 = (long long)(ys - {3 * ry} + tb) * {PY} + gx;  // step-1 row of unroll 0")
        for i in range(RB):
            i3 = ind + "  "
            a(f"{ind}{{  // step 1, unroll {i}: input row t = tb + {i}, step-1 row t - {ry}")
            a(f"{i3}{{ const {VT} v = *reinterpret_cast<const {VT}*>(QS + {i * W0}); "
              + " ".join(f"q{2 * ry + i}_{v} = v.{'xyzw'[v]};" for v in range(V)) + " }")
            if rot:
                a(f"{i3}const {VT} pv{i} = *reinterpret_cast<const {VT}*>(PS + {i * W0});")
                for v in range(V):
                    a(f"{i3}const T p{i}_{v} = pv{i}.{'xyzw'[v]};")
            need: dict = {}
            bodies = [self._expr(1, i, v, need) for v in range(V)]
            # x-neighbours of step 1 at row t - ry: this stage's row i - ry or the previous stage's
            src_row = i - ry
            base = f"(QS + {src_row * W0})" if src_row >= 0 else f"(QP + {(src_row + RB) * W0})"
            out = [f"x{2 * ry + i}_{v}" for v in range(V)]
            vec = f"make_{VT}({', '.join(out)})"
            if fast:
                self._nbr_loads(i3, 1, i, need, base)
                for v, (lines, res) in enumerate(bodies):
                    a(f"{i3}{{ " + " ".join(lines) + f" {out[v]} = {res}; }}")
                a(f"{i3}*reinterpret_cast<{VT}*>(WB + {i * W1p}) = {vec};")
                a(f"{i3}if (p.wb && own) *reinterpret_cast<{VT}*>(x1m + r1 + {i * PY}) = {vec};")
                a(f"{ind}}}")
                continue
            a(f"{i3}const int t = tb + {i};")
            a(f"{i3}if (t >= {2 * ry} && t < n0) {{")
            i4 = i3 + "  "
            i5 = i4 + "  "
            a(f"{i4}const int u1 = ys - {3 * ry} + t;  // padded row of this step-1 row")
            a(f"{i4}if (u1 >= p.sy0 && u1 < p.sy1) {{")
            self._nbr_loads(i5, 1, i, need, base)
            for v, (lines, res) in enumerate(bodies):
                a(f"{i5}{{ " + " ".join(lines) + f" {out[v]} = {res}; }}")
            a(f"{i5}if (!xin) {{")
            for v in range(V):
                a(f"{i5}  if (!xs{v}) {out[v]} = xp{v} ? x1m[r1 + {i * PY + v}] : (T)0;")
            a(f"{i5}}}")
            a(f"{i4}}} else {{  // row outside S: the stored value (0 beyond the padded box)")
            a(f"{i5}const bool yp = u1 >= 0 && u1 < p.npy;")
            for v in range(V):
                a(f"{i5}{out[v]} = (yp && xp{v}) ? x1m[r1 + {i * PY + v}] : (T)0;")
            a(f"{i4}}}")
            a(f"{i4}*reinterpret_cast<{VT}*>(WB + {i * W1p}) = {vec};")
            a(f"{i4}if (p.wb && own && u1 >= ys && u1 < ys + nyl) {{")
            a(f"{i5}T* dst = x1m + r1 + {i * PY};")
            a(f"{i5}if (xin) *reinterpret_cast<{VT}*>(dst) = {vec};")
            a(f"{i5}else {{ " + " ".join(f"if (xs{v}) dst[{v}] = {out[v]};" for v in range(V)) + " }")
            a(f"{i4}}}")
            a(f"{i3}}}")
            a(f"{ind}}}")
        a(f"{ind}asm volatile(\"bar.sync 1, {NT};\" ::: \"memory\");")
        a(f"{ind}if (tid == 0) {{ if (s > 0) mbar_arrive(empty + prv); if (s == nst - 1) mbar_arrive(empty + stg); }}")
        a(f"{ind}const long long r2 = r1 - {ry * PY};  // step-2 row of unroll 0")
        for i in range(RB):
            i3 = ind + "  "
            cond = "" if fast else f"if (tb + {i} >= {4 * ry} && tb + {i} < n0) "
            a(f"{ind}{cond}{{  // step 2, unroll {i}: row t - {2 * ry}")
            src = f"(WB + {(i - ry) * W1p})" if i >= ry else f"(WP + {(RB + i - ry) * W1p})"
            a(f"{i3}const T* R = {src};")
            need = {}
            bodies = [self._expr(2, i, v, need) for v in range(V)]
            self._nbr_loads(i3, 2, i, need, "R")
            for v, (lines, res) in enumerate(bodies):
                a(f"{i3}T o{v}; {{ " + " ".join(lines) + f" o{v} = {res}; }}")
            ov = f"make_{VT}({', '.join(f'o{v}' for v in range(V))})"
            if fast:
                a(f"{i3}if (own) *reinterpret_cast<{VT}*>(x2m + r2 + {i * PY}) = {ov};")
            else:
                a(f"{i3}if (own) {{")
                a(f"{i3}  T* dst = x2m + r2 + {i * PY};")
                a(f"{i3}  if (xin) *reinterpret_cast<{VT}*>(dst) = {ov};")
                a(f"{i3}  else {{ " + " ".join(f"if (xs{v}) dst[{v}] = o{v};" for v in range(V)) + " }")
                a(f"{i3}}}")
            a(f"{ind}}}")

    def source(self) -> str:
        lay, a = self.lay, self.a
        cfg = lay["cfg"]
        V, ry, RB, S0, C1 = lay["V"], lay["ry"], lay["rb"], lay["s0"], lay["c1"]
        W0, W1, W1p, P1, NT, E = lay["w0"], lay["w1"], lay["w1p"], lay["p1"], lay["nt"], lay["elem"]
        m0, m1, BX = lay["m0"], lay["m1"], lay["bx"]
        rot = lay["cen"] is not None
        PY, VT, T = self.py, self.VT, self.T
        NW = NT // 32
        H = RB + 2 * ry  # register window rows
        # the min-blocks hint caps the registers per thread: at most 4 so the
        # register windows are not spilled (the hardware still runs more CTAs
        # per SM when registers and shared memory allow)
        minb = min(blocks_per_sm(lay), 4)
        lay["min_blocks"] = minb
        a(f'// generated by paper_2512_19851_b200/temporal2d.py - skeleton "tc" (2 fused sweeps, rank 2, '
          f'{"rotation" if rot else "ping-pong"}) {cfg} bx={BX} rb={RB} py={PY} xoff={self.xoff}')
        a(f"typedef {T} T;")
        a("struct __align__(64) Tmap { unsigned long long w[16]; };")
        a("struct __align__(64) Params { Tmap tq; Tmap tp;")
        a("  unsigned long long x1, x2;  // padded-box origins: X1 (in place), step-2 array (other buffer)")
        a("  int npy, npx, sy0, sy1, sx0, sx1, xt0, nbx, yc, nyc, wb; };")
        a(_PTX_HELPERS)
        a("__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {")
        a("  asm volatile(\"mbarrier.arrive.shared::cta.b64 _, [%0];\" :: \"r\"(smem_u32(b)) : \"memory\"); }")
        a(f'extern "C" __global__ void __launch_bounds__({NT + 32}, {minb})')
        a("est_tc(const __grid_constant__ Params p) {")
        a("  extern __shared__ __align__(1024) unsigned char smem[];")
        a(f"  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + {lay['data']});")
        a(f"  unsigned long long* empty = full + {S0};")
        a("  const int tid = threadIdx.x, warp = tid >> 5;")
        a("  asm volatile(\"griddepcontrol.launch_dependents;\" ::: \"memory\");")
        a("  if (tid == 0) {")
        a(f"    for (int i = 0; i < {S0}; ++i) {{ mbar_init(full + i, 1); mbar_init(empty + i, 1); }}")
        a("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");")
        a("  }")
        a("  __syncthreads();")
        a("  asm volatile(\"griddepcontrol.wait;\" ::: \"memory\");  // the previous launch's stores are visible")
        a("  const int item = blockIdx.x;")
        a("  const int bxi = item % p.nbx, byi = item / p.nbx;")
        a(f"  const int x0 = p.xt0 + bxi * {BX};")
        a("  const int ys = p.sy0 + byi * p.yc;")
        a("  const int nyl = min(p.yc, p.sy1 - ys);")
        a(f"  const int n0 = nyl + {4 * ry};  // input rows of the item")
        a(f"  const int nst = (n0 + {RB - 1}) / {RB};  // stages")
        # ---------------- producer
        a(f"  if (warp == {NW}) {{")
        a("    if ((tid & 31) != 0) return;")
        a("    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&p.tq) : \"memory\");")
        if rot:
            a("    asm volatile(\"prefetch.tensormap [%0];\" :: \"l\"(&p.tp) : \"memory\");")
        a("    for (int s = 0; s < nst; ++s) {")
        a(f"      const int stg = s % {S0};")
        a(f"      if (s >= {S0}) mbar_wait(empty + stg, ((s / {S0}) - 1) & 1);")
        a(f"      mbar_expect(full + stg, {RB * W0 * E * (2 if rot else 1)});")
        a(f"      unsigned char* sb = smem + stg * {lay['stage']};")
        a(f"      tma_load3(sb, &p.tq, x0 + {self.xoff - m0}, ys - {2 * ry} + s * {RB}, 0, full + stg);")
        if rot:
            a(f"      tma_load3(sb + {lay['qb']}, &p.tp, x0 + {self.xoff - m0}, ys - {3 * ry} + s * {RB}, 0, full + stg);")
        a("    }")
        a("    return;")
        a("  }")
        # ---------------- compute threads
        a(f"  const bool act = tid < {P1};")
        a(f"  const int c = act ? tid : {P1 - 1};  // vector column of the step-1 frame")
        a(f"  const bool own = act && c >= {m1 // V} && c < {(m1 + BX) // V};  // output column of this item")
        a("  T* __restrict__ x1m = reinterpret_cast<T*>(p.x1);")
        a("  T* __restrict__ x2m = reinterpret_cast<T*>(p.x2);")
        a(f"  const int gx = x0 - {m1} + c * {V};  // first padded column of the thread's vector")
        a(f"  T* ring1 = reinterpret_cast<T*>(smem + {lay['ring1']}) + {V} + c * {V};")
        for v in range(V):
            a(f"  const bool xs{v} = gx + {v} >= p.sx0 && gx + {v} < p.sx1;  // column in S")
            a(f"  const bool xp{v} = gx + {v} >= 0 && gx + {v} < p.npx;  // column in the padded box")
        a("  const bool xin = " + " && ".join(f"xs{v}" for v in range(V)) + ";")
        for k in range(H):
            a(f"  T {', '.join(f'q{k}_{v} = 0' for v in range(V))};")
            a(f"  T {', '.join(f'x{k}_{v} = 0' for v in range(V))};")
        a("  int stg = 0, ph = 0, prv = 0, bk = 0, bp = 2;  // stage slot / phase, previous slot, ring banks")
        a(f"  const bool xfast = (x0 - {m1} >= p.sx0) && (x0 + {BX + m1} <= p.sx1);  // frame inside S in x")
        a("  for (int s = 0; s < nst; ++s) {")
        i2 = "    "
        a(f"{i2}const int tb = s * {RB};")
        a(f"{i2}mbar_wait(full + stg, ph);")
        a(f"{i2}const T* QS = reinterpret_cast<const T*>(smem + stg * {lay['stage']}) + {m0 - m1} + c * {V};")
        a(f"{i2}const T* QP = reinterpret_cast<const T*>(smem + prv * {lay['stage']}) + {m0 - m1} + c * {V};")
        if rot:
            a(f"{i2}const T* PS = reinterpret_cast<const T*>(smem + stg * {lay['stage']} + {lay['qb']}) + {m0 - m1} + c * {V};")

        a(f"{i2}T* WB = ring1 + bk * {RB * W1p};  // ring bank of this stage's step-1 rows")
        a(f"{i2}const T* WP = ring1 + bp * {RB * W1p};  // ... and of the previous stage's")
        # fast stage: every step-1 row lies in the item's own output rows (so
        # inside S), every step-2 row is valid and the frame is inside S in x
        a(f"{i2}if (xfast && tb >= {4 * ry} && tb + {RB} <= nyl + {3 * ry}) {{")
        self.emit_stage(i2 + "  ", fast=True)
        a(f"{i2}}} else {{")
        self.emit_stage(i2 + "  ", fast=False)
        a(f"{i2}}}")
        # ---- shift the register windows by RB rows
        for k in range(2 * ry):
            a(f"{i2}" + " ".join(f"q{k}_{v} = q{k + RB}_{v}; x{k}_{v} = x{k + RB}_{v};" for v in range(V)))
        a(f"{i2}prv = stg;")
        a(f"{i2}if (++stg == {S0}) {{ stg = 0; ph ^= 1; }}")
        a(f"{i2}bp = bk; if (++bk == 3) bk = 0;")
        a("  }")
        a("}")
        return "\n".join(self.L) + "\n"


def source(st: StmtSig, dtype: int, cfg: TcCfg | None = None, py: int = 16448, xoff: int = 28) -> tuple:
    """-> (source, kernel name, block, smem, layout). Row pitch and x offset are
    compile-time constants (defaults: the C3 layout, 16384^2 fp32, depth 2)."""
    cfg = cfg or DEFAULT
    lay = layout(st, dtype, cfg)
    src = _Emitter(st, dtype, lay, py, xoff).source()
    return src, "est_tc", (lay["nt"] + 32, 1, 1), lay["smem"], lay


def item_geometry(s_lo, s_hi, lay: dict, xoff: int = 0) -> dict:
    """Items of the output box S (padded coordinates, rank 2 as (y, x)): x
    tiles from the 16-byte aligned column at or below S's first column (a TMA
    box must start on a 16-byte aligned address: an 8-byte aligned start
    faults as an illegal instruction), y chunks balanced."""
    cfg = lay["cfg"]
    A, BX = 16 // lay["elem"], lay["bx"]
    ny = s_hi[0] - s_lo[0]
    xt0 = s_lo[1] - ((xoff + s_lo[1]) % A)  # 16-byte aligned tiles (TMA box starts)
    nbx = -(-(s_hi[1] - xt0) // BX)
    nyc = max(1, -(-ny // max(1, cfg.ychunk)))
    if nbx * nyc < cfg.min_items:
        nyc = max(nyc, min(-(-cfg.min_items // nbx), max(1, ny // (8 * lay["rb"]))))
    yc = -(-ny // nyc)
    nyc = -(-ny // yc)
    return {"nbx": nbx, "yc": yc, "nyc": nyc, "blocks": nbx * nyc, "xt0": xt0}


def pack_params(tq: bytes, tp: bytes, x1: int, x2: int, npy: int, npx: int, s_lo, s_hi, geo: dict,
                write_x1: bool = True) -> bytes:
    """Params block (layout mirrored in `source`); pointers are padded-box
    origins (buffer base + xoff elements)."""
    assert len(tq) == 128 and len(tp) == 128
    out = bytearray(tq) + bytearray(tp)
    out += struct.pack("<QQ", x1, x2)
    out += struct.pack("<11i", npy, npx, s_lo[0], s_hi[0], s_lo[1], s_hi[1], geo["xt0"], geo["nbx"],
                       geo["yc"], geo["nyc"], int(write_x1))
    return bytes(out) + b"\0" * ((-len(out)) % 64)
