// round_kernels.cu -- device kernels of one round of the batched round rule.
//
//   k_init       a2  R0 initialisation: one draw per pair, T = 1
//   k_select     a6+a7  per-query rank split (radix select of the k-th and
//                (k+h)-th composite keys), d1/d2, A, B, Eq. (5)  (P:144-153,
//                P:178-184)
//   k_filter     a8  blocker predicate -> action bytes + per-slot counts
//   k_plan       prefix of slot counts -> list offsets and warp-chunk plan
//   k_scatter    a8  compaction of the action bytes into per-slot work lists
//   k_advance    a3+a4  level gathers (T -> 2T draws, Philox + uint8 gather,
//                exact int sums) and exact fallbacks
//   k_output     a9  candidate set in rank order, d_hat, counters
//
// All state is integer; the only floating point is the fp64 estimate/bounds
// arithmetic, written with explicit round-to-nearest intrinsics (no FMA).
#include "internal.cuh"
#include "launch.h"
#include "select.cuh"
#include "round_common.cuh"

namespace aknn {

// ---------------------------------------------------------------------------
// a2: initialisation -- S_i = (X[i][j] - x[j])^2 for j = Draw(i, 0), T_i = 1.
// Grid (q, point chunks) when the chunk count fits grid.y: CTAs are issued query-fastest,
// so the q draws into one chunk's point rows come close together and the rows stay in
// L2 (one HBM read of X; query-major order streamed X's random sectors once per query:
// C4: 4 GB of sectors).  PM = false: grid (chunks, q), when the chunks exceed grid.y.
template <bool PM>
__global__ void k_init(Geom g) {
  const int qi = PM ? blockIdx.x : blockIdx.y;
  const int i = (PM ? blockIdx.y : blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= g.npad) return;
  const size_t o = (size_t)qi * g.npad + i;
  if (i >= g.n) {
    g.S[o] = 0;
    g.lvl[o] = LVL_EXACT;  // padding: never selected
    g.act[o] = 0;
    return;
  }
  uint32_t j;
  if (g.wor) {  // pi(0) of the arm's permutation (reading R23)
    j = wor_coord(wor_keys(g.rk0, g.rk1, (uint32_t)i + g.id_offset, rng_qi(g, (uint32_t)qi)), g.wor_z,
                  (uint32_t)g.d, 0u);
  } else {
    const uint4 w = philox4x32_10(make_uint4(0u, (uint32_t)i + g.id_offset, rng_qi(g, (uint32_t)qi), 0u),
                                  g.seed_lo, g.seed_hi);
    j = coord_of(w.x, (uint32_t)g.d);
  }
  const int diff = (int)__ldg(g.X + (size_t)i * g.pitch + j) - (int)__ldg(g.Q + (size_t)qi * g.pitch + j);
  g.S[o] = diff * diff;
  g.lvl[o] = (g.d == 1) ? LVL_EXACT : (uint8_t)0;  // d = 1: the draw is exact
  g.act[o] = 0;
}

__global__ void k_init_qstate(Geom g) {
  const int qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= g.q) return;
  QState s;
  s.thr_k = s.thr_kh = 0;
  s.A = s.B = s.a_d2 = 0.0;
  s.d1 = s.d2 = -1;
  s.done = 0;
  s.fallback = 0;
  s.rounds = 0;
  s.draws = 0;  // tallied at the end (k_tally)
  s.nexact = 0;
  s.exact_evals = 0;
  s.blocks = 0;
  g.qs[qi] = s;
}

// a6 + a7: rank split, d1/d2/A/B, Eq. (5).  One CTA per query.
// Multi-pass radix version; runs only for queries the pivot select flagged.
__global__ void __launch_bounds__(SEL_NT) k_select(Geom g, int nbits) {
  __shared__ SelSmem sm;
  __shared__ Best wbest[2][SEL_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done || !st->fallback) return;
  const int tid = threadIdx.x;
  ArmKeys keys{&g, qi};
  unsigned long long thk, thkh;
  select2(sm, keys, g.n, nbits, (unsigned)g.k, (unsigned)(g.k + g.h), &thk, &thkh);

  // bounds pass: A = max_C U (tie: smaller i), B = min_F L (tie: smaller i)
  Best bu{-1.0e300, 0x7fffffff, 0.0}, bl{1.0e300, 0x7fffffff, 0.0};
  for (int i0 = tid * 4; i0 < g.n; i0 += SEL_NT * 4) {
    const Arm4 a = load_arm4(g, qi, i0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e;
      if (i >= g.n) break;
      const unsigned long long key = arm_key(a.S[e], a.l(e), (uint32_t)i, g);
      if (key <= thk) {
        const double U = __dadd_rn(dhat_of(a.S[e], a.l(e), g.d, g.growth), alpha_of(a.l(e), g.alpha, g.growth));
        if (U > bu.v || (U == bu.v && i < bu.i)) bu = Best{U, i, 0.0};
      } else if (key > thkh) {
        const double al = alpha_of(a.l(e), g.alpha, g.growth);
        const double L = __dsub_rn(dhat_of(a.S[e], a.l(e), g.d, g.growth), al);
        if (L < bl.v || (L == bl.v && i < bl.i)) bl = Best{L, i, al};
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double uv = __shfl_xor_sync(FULL, bu.v, o);
    const int ui = __shfl_xor_sync(FULL, bu.i, o);
    if (uv > bu.v || (uv == bu.v && ui < bu.i)) { bu.v = uv; bu.i = ui; }
    const double lv = __shfl_xor_sync(FULL, bl.v, o);
    const int li = __shfl_xor_sync(FULL, bl.i, o);
    const double la = __shfl_xor_sync(FULL, bl.a, o);
    if (lv < bl.v || (lv == bl.v && li < bl.i)) { bl.v = lv; bl.i = li; bl.a = la; }
  }
  if (lane_id() == 0) {
    wbest[0][tid >> 5] = bu;
    wbest[1][tid >> 5] = bl;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < SEL_NT / 32; ++w) {
      const Best u = wbest[0][w], l = wbest[1][w];
      if (u.v > bu.v || (u.v == bu.v && u.i < bu.i)) bu = u;
      if (l.v < bl.v || (l.v == bl.v && l.i < bl.i)) bl = l;
    }
    st->thr_k = thk;
    st->thr_kh = thkh;
    st->A = bu.v;
    st->B = bl.v;
    st->d1 = bu.i;
    st->d2 = bl.i;
    st->a_d2 = bl.a;
    st->rounds += 1;
    const int stop = bu.v <= bl.v;  // Eq. (5), "<=" as written
    st->done = stop;
    if (!stop) atomicAdd(&g.ctl->n_active, 1u);
  }
}

// ---------------------------------------------------------------------------
// a8: blocker filter.  Active = {C: U > B} u {F: L < A} u {M: alpha > alpha_d2}
// minus exact arms; an active arm with 2T >= d goes exact.
//
// One CTA per block of FIL_ROWS queries x FIL_NT * 4 arms: each thread owns 4
// consecutive arms and walks the block's query rows (the next row's state is loaded
// before the current one is decided).  Per CTA: one global atomic per action slot
// (the list plan), and -- with tiles on -- the exact draw count of every (R x P)
// tile it covers (R | FIL_ROWS, P | FIL_NT * 4: each tile lies in one CTA), written
// with a plain store.
constexpr int FIL_NT = 256;
constexpr int FIL_ROWS = 32;
#ifndef AKNN_FIL_AHEAD
#define AKNN_FIL_AHEAD 2
#endif
constexpr int FIL_AHEAD = AKNN_FIL_AHEAD;

// The round's blocker predicate as integer thresholds (see THR_STRIDE): one warp per
// undecided query, lane c bisects S in [0, 65025 * 2^c] with the very fp64 operations
// the predicate is defined by (dhat_of, __dadd_rn / __dsub_rn, P:118-138 estimates and
// radii; R15), so the integer test decides every arm identically.
__global__ void __launch_bounds__(128) k_thresholds(Geom g) {
  const int qi = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int c = lane_id();
  if (qi >= g.q) return;
  const QState &st = g.qs[qi];
  if (st.done) return;
  const int nlev = g.cmax + 1, hdr = thr_hdr(nlev);
  int32_t *t = g.thr + (size_t)qi * thr_stride(nlev);
  const unsigned long long kmask = (1ull << g.kbits) - 1ull;
  bool mbit = false, eqk = false, eqkh = false;
  if (c < MAX_LEVELS && c <= g.cmax) {
    const uint8_t l = (uint8_t)c;
    const double al = alpha_of(l, g.alpha, g.growth);
    const int32_t smax = (int32_t)(65025u * lvl_count((uint32_t)c, g.growth));  // every draw (a - b)^2 <= 255^2
    // Su: first S with U(S) > B (smax + 1: none)
    int32_t lo = 0, hi = smax + 1;
    while (lo < hi) {
      const int32_t mid = lo + ((hi - lo) >> 1);
      if (__dadd_rn(dhat_of(mid, l, g.d, g.growth), al) > st.B) hi = mid; else lo = mid + 1;
    }
    const int32_t su = lo;
    // Sl: first S with L(S) >= A (blocker iff S < Sl)
    lo = 0;
    hi = smax + 1;
    while (lo < hi) {
      const int32_t mid = lo + ((hi - lo) >> 1);
      if (!(__dsub_rn(dhat_of(mid, l, g.d, g.growth), al) < st.A)) hi = mid; else lo = mid + 1;
    }
    const int32_t sl = lo;
    // the key thresholds on S at this level: S * mul <=> K = thr >> kbits
    const unsigned long long mul = lvl_mul((uint32_t)c, g.L, g.L3, g.growth);
    const unsigned long long Kk = st.thr_k >> g.kbits, Kkh = st.thr_kh >> g.kbits;
    const unsigned long long ck = (Kk + mul - 1) / mul, ckh = (Kkh + mul - 1) / mul;
    eqk = Kk % mul == 0;
    eqkh = Kkh % mul == 0;
    const int4 v = make_int4(su, sl, (int32_t)(ck > 0x7fffffffull ? 0x7fffffffull : ck),
                             (int32_t)(ckh > 0x7fffffffull ? 0x7fffffffull : ckh));
    *reinterpret_cast<int4 *>(t + 4 * c) = v;
    mbit = al > st.a_d2;
  }
  const unsigned m = __ballot_sync(FULL, mbit), mk = __ballot_sync(FULL, eqk), mkh = __ballot_sync(FULL, eqkh);
  if (c == 0) {
    t[hdr + 0] = (int32_t)m;
    t[hdr + 1] = (int32_t)mk;
    t[hdr + 2] = (int32_t)mkh;
    t[hdr + 3] = (int32_t)(uint32_t)(st.thr_k & kmask);
    t[hdr + 4] = (int32_t)(uint32_t)(st.thr_kh & kmask);
  }
}

cudaError_t launch_thresholds(const Geom &g, cudaStream_t s) {
  k_thresholds<<<(unsigned)((g.q + 3) / 4), 128, 0, s>>>(g);
  return cudaGetLastError();
}

// Branch-free decision of 4 arms (R5 with the integer thresholds of reading R20):
// one 16-byte table load per level (once for the 4 arms when they share it -- the
// lock-step case), no 64-bit key arithmetic, no floating point.
__device__ __forceinline__ uint32_t filter_arm(const Geom &g, const int4 &t, uint32_t c, uint8_t l, int32_t S, int i,
                                               uint32_t mmask, uint32_t eqk, uint32_t eqkh, uint32_t idk,
                                               uint32_t idkh, uint32_t *dr, uint32_t *lwb) {
  const bool live = i < g.n && !lvl_exact(l);
  bool inC = S < t.z, inM = S < t.w;
  if ((S == t.z) | (S == t.w)) {  // rare: the id decides a tie with the k-th / (k+h)-th key
    const uint32_t gid = (uint32_t)i + g.id_offset;
    inC = inC || (((eqk >> c) & 1u) && S == t.z && gid <= idk);
    inM = inM || (((eqkh >> c) & 1u) && S == t.w && gid <= idkh);
  }
  const bool blk = live && (inC ? S >= t.x : (inM ? ((mmask >> c) & 1u) != 0u : S < t.y));
  // P:176 (reading R8): exact when the next count would reach d (bit c of g.exnext)
  const bool ex = (g.exnext >> c) & 1u;
  *dr += (blk && !ex) ? (1u << c) : 0u;  // tiles (doubling only): the advance draws T_c
  *lwb = (blk && !ex && inM) ? 1u : 0u;  // inM: ranks 1..k+h (C or M)
  return blk ? (ex ? (uint32_t)ACT_EXACT : c + 1u) : 0u;
}

__device__ __forceinline__ uint32_t filter_arms(const Geom &g, const int32_t *thr, const Arm4 &a, int i0,
                                                uint32_t *draws, uint32_t *leadw) {
  uint32_t actw = 0, dr = 0, lw = 0;
  // thr: the row's table staged in shared memory by k_filter
  const int ho = thr_hdr(g.cmax + 1);
  const int4 hdr = *reinterpret_cast<const int4 *>(thr + ho);
  const uint32_t mmask = (uint32_t)hdr.x, eqk = (uint32_t)hdr.y, eqkh = (uint32_t)hdr.z;
  const uint32_t idk = (uint32_t)hdr.w, idkh = (uint32_t)thr[ho + 4];
  const uint32_t c0 = a.l(0) & 31u;
  if (a.lw == (uint32_t)a.l(0) * 0x01010101u) {  // one level for the 4 arms (lock-step)
    // Away from the two rank thresholds the predicate is a union of S intervals:
    //   S < Ck: C, blocker iff S >= Su;  Ck <= S < Ckh: M, iff mbit;  S >= Ckh: F, iff S < Sl
    // so blk = S in [Su, Ck) or (mbit and S in [Ck, Ckh)) or S in [Ckh, Sl): three unsigned
    // range tests per arm.  S equal to Ck or Ckh (the id decides the band) takes filter_arm.
    const int4 t = reinterpret_cast<const int4 *>(thr)[c0];  // Su, Sl, Ck, Ckh
    const bool mb = (mmask >> c0) & 1u;
    auto span = [](int32_t lo, int32_t hi) { return hi > lo ? (uint32_t)((int64_t)hi - (int64_t)lo) : 0u; };
    const uint32_t l1 = span(t.x, t.z), l2 = mb ? span(t.z, t.w) : 0u, l3 = span(t.w, t.y);
    uint32_t bm = 0, mm = 0, tie = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int32_t S = a.S[e];
      const bool b = ((uint32_t)S - (uint32_t)t.x < l1) | ((uint32_t)S - (uint32_t)t.z < l2) |
                     ((uint32_t)S - (uint32_t)t.w < l3);
      bm |= (uint32_t)b << e;
      mm |= (uint32_t)(S < t.w) << e;  // ranks 1..k+h (C or M), away from the thresholds
      tie |= (uint32_t)((S == t.z) | (S == t.w)) << e;
    }
    const int nlive = g.n - i0;  // arms past the end are never blockers
    const uint32_t live = lvl_exact(a.l(0)) ? 0u : (nlive >= 4 ? 0xFu : (nlive > 0 ? (1u << nlive) - 1u : 0u));
    bm &= live;
    // P:176 (reading R8): exact when the next count would reach d (bit c of g.exnext)
    const bool ex = (g.exnext >> c0) & 1u;
    const uint32_t av = ex ? (uint32_t)ACT_EXACT : c0 + 1u;
    actw = ((bm * 0x00204081u) & 0x01010101u) * av;  // bit e -> byte e
    dr = ex ? 0u : (uint32_t)__popc(bm) << c0;       // tiles (doubling only): T_c draws each
    lw = ex ? 0u : (((mm & bm) * 0x00204081u) & 0x01010101u);
    if (tie) {  // rare: redo the arms at a threshold with the id rule
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!((tie >> e) & 1u)) continue;
        uint32_t d1 = 0, lb;
        const uint32_t act = filter_arm(g, t, c0, a.l(0), a.S[e], i0 + e, mmask, eqk, eqkh, idk, idkh, &d1, &lb);
        const uint32_t was = (actw >> (8 * e)) & 0xFFu;
        actw = (actw & ~(0xFFu << (8 * e))) | (act << (8 * e));
        lw = (lw & ~(0xFFu << (8 * e))) | (lb << (8 * e));
        dr = dr - ((was && !ex) ? (1u << c0) : 0u) + d1;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint8_t l = a.l(e);
      const uint32_t c = l & 31u;
      const int4 t = reinterpret_cast<const int4 *>(thr)[c];
      uint32_t lb;
      actw |= filter_arm(g, t, c, l, a.S[e], i0 + e, mmask, eqk, eqkh, idk, idkh, &dr, &lb) << (8 * e);
      lw |= lb << (8 * e);
    }
  }
  *draws = dr;
  *leadw = lw;
  return actw;
}

// A lead pass (reading R24): the arms flagged in leadb advance once more from the
// level they reached (exact when the next level would reach d).
__device__ __forceinline__ uint32_t lead_arms(const Geom &g, const Arm4 &a, uint32_t lb, int i0, uint32_t *draws) {
  uint32_t actw = 0, dr = 0;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint8_t l = a.l(e);
    const uint32_t c = l & 31u;
    const bool go = i0 + e < g.n && ((lb >> (8 * e)) & 0xFFu) && !lvl_exact(l);
    const bool ex = (g.exnext >> c) & 1u;
    const uint32_t act = go ? (ex ? (uint32_t)ACT_EXACT : c + 1u) : 0u;
    dr += (go && !ex) ? (1u << c) : 0u;
    actw |= act << (8 * e);
  }
  *draws = dr;
  return actw;
}

// Per-thread run-length counter of action slots: flushes to the CTA's shared counts
// only when the slot changes (under lockstep levels: almost never).
struct SlotRun {
  unsigned slot = NONE, n = 0;
  __device__ __forceinline__ void add(unsigned s, unsigned *scnt, unsigned k = 1) {
    if (s == slot) {
      n += k;
      return;
    }
    if (slot != NONE && n) atomicAdd(&scnt[slot], n);
    slot = s;
    n = k;
  }
  __device__ __forceinline__ void flush(unsigned *scnt) {
    if (slot != NONE && n) atomicAdd(&scnt[slot], n);
  }
};

// MODE 0: the round's filter; 1: the same, also writing the lead bytes (lead > 1);
// 2: a lead pass (reading R24).  Separate instantiations keep MODE 0's registers.
template <int MODE>
__global__ void __launch_bounds__(FIL_NT) k_filter(Geom g) {
  // dynamic: [FIL_ROWS][thr stride] blocker thresholds (modes 0, 1), then the tile counts
  // [FIL_ROWS / R][FIL_NT * 4 / P] (tiles on)
  extern __shared__ __align__(16) uint32_t fsm[];
  const int tstride = thr_stride(g.cmax + 1);
  int32_t *sthr = reinterpret_cast<int32_t *>(fsm);
  uint32_t *tcnt = fsm + (MODE == 2 ? 0 : FIL_ROWS * tstride);
  __shared__ unsigned scnt[NSLOT];
  __shared__ unsigned lvc[(FIL_NT * 4 / 128) * MAX_LEVELS];
  const int q0 = blockIdx.y * FIL_ROWS;
  const int rows = min(FIL_ROWS, g.q - q0);
  const int i0 = (blockIdx.x * FIL_NT + threadIdx.x) * 4;
  const int lane = lane_id();
  const int tcols = g.tile_on ? (FIL_NT * 4) >> g.tile_lp : 0;
  const int ntc = g.tile_on ? (FIL_ROWS >> g.tile_lr) * tcols : 0;
  for (int s = threadIdx.x; s < NSLOT; s += FIL_NT) scnt[s] = 0;
  for (int t = threadIdx.x; t < ntc; t += FIL_NT) tcnt[t] = 0;
  for (int t = threadIdx.x; t < (FIL_NT * 4 / 128) * MAX_LEVELS; t += FIL_NT) lvc[t] = 0;
  __shared__ uint32_t srow_any;  // bit r: row r has an action in this chunk
  if (threadIdx.x == 0) srow_any = 0;
  // the CTA's rows of blocker thresholds (reading R20), staged once
  if (MODE != 2)
    for (int t = threadIdx.x; t < rows * (tstride / 4); t += FIL_NT)
      reinterpret_cast<int4 *>(sthr)[t] = __ldg(reinterpret_cast<const int4 *>(g.thr + (size_t)q0 * tstride) + t);
  __syncthreads();
  const bool arms = i0 < g.n;
  // the rows' done flags as one bit mask (read once: a per-row flag load was consumed
  // at once -- as a uniform register -- and stalled every row on its latency)
  uint32_t donem;
  {
    const int lane_r = lane;
    const bool dflag = lane_r < rows ? g.qs[q0 + lane_r].done != 0 : true;
    donem = __ballot_sync(FULL, dflag);
  }
  // FIL_AHEAD rows of arm loads in flight ahead of the row being decided (the pass is
  // load-latency bound: 20 bytes per thread and row)
  Arm4 aq[FIL_AHEAD];
#pragma unroll
  for (int j = 0; j < FIL_AHEAD; ++j) {
    aq[j] = Arm4{};
    if (arms && j < rows && !((donem >> j) & 1u)) aq[j] = load_arm4(g, q0 + j, i0);
  }
  SlotRun run, lrun;      // lrun: the thread's pairs per level in its 128 x 128 level tile
  unsigned ex_acc = 0;     // exact fallbacks of this thread (one 128-query tile row: 32 | 128)
  uint32_t dr_acc = 0;     // sampled draws of this thread in the current tile row
  uint32_t rany = 0;       // bit r: this thread's arms of row r have an action
  int tr_cur = 0;
  for (int r = 0; r < rows; ++r) {
    const int qi = q0 + r;
    const Arm4 ca = aq[0];
#pragma unroll
    for (int j = 0; j + 1 < FIL_AHEAD; ++j) aq[j] = aq[j + 1];
    if (r + FIL_AHEAD < rows && arms && !((donem >> (r + FIL_AHEAD)) & 1u))  // prefetch row r + FIL_AHEAD
      aq[FIL_AHEAD - 1] = load_arm4(g, qi + FIL_AHEAD, i0);
    if ((donem >> r) & 1u) continue;  // uniform: one query row at a time
    uint32_t dr = 0, actw = 0, lw = 0;
    if (MODE == 2) {
      if (arms) actw = lead_arms(g, ca, *reinterpret_cast<const uint32_t *>(g.leadb + (size_t)qi * g.npad + i0), i0, &dr);
    } else {
      if (arms) actw = filter_arms(g, sthr + r * tstride, ca, i0, &dr, &lw);
      if (MODE == 1 && i0 < g.npad) *reinterpret_cast<uint32_t *>(g.leadb + (size_t)qi * g.npad + i0) = lw;
    }
    if (i0 < g.npad) *reinterpret_cast<uint32_t *>(g.act + (size_t)qi * g.npad + i0) = actw;
    rany |= (actw != 0u ? 1u : 0u) << r;
    if (actw) {
      const uint32_t a0 = actw & 0xFFu;
      if (actw == a0 * 0x01010101u) {  // 4 equal actions (lock-step): one count update
        ex_acc += a0 == ACT_EXACT ? 4u : 0u;
        run.add(a0 == ACT_EXACT ? (unsigned)MAX_LEVELS : a0 - 1u, scnt, 4u);
        if (g.level_mma && a0 != ACT_EXACT) lrun.add(a0 - 1u, lvc + ((threadIdx.x * 4) >> 7) * MAX_LEVELS, 4u);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t act = (actw >> (8 * e)) & 0xFFu;
          ex_acc += act == ACT_EXACT;
          if (act) run.add(act == ACT_EXACT ? (unsigned)MAX_LEVELS : act - 1u, scnt);
        }
        if (g.level_mma) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t act = (actw >> (8 * e)) & 0xFFu;
            if (act && act != ACT_EXACT) lrun.add(act - 1u, lvc + ((threadIdx.x * 4) >> 7) * MAX_LEVELS);
          }
        }
      }
    }
    if (g.tile_on) {
      const int tr = r >> g.tile_lr;
      if (tr != tr_cur) {  // entering the next tile row of this CTA: flush
        if (dr_acc) atomicAdd(&tcnt[tr_cur * tcols + ((threadIdx.x * 4) >> g.tile_lp)], dr_acc);
        dr_acc = 0;
        tr_cur = tr;
      }
      dr_acc += dr;
    }
  }
  run.flush(scnt);
  if (g.level_mma) lrun.flush(lvc + ((threadIdx.x * 4) >> 7) * MAX_LEVELS);
  if (g.tile_on && dr_acc) atomicAdd(&tcnt[tr_cur * tcols + ((threadIdx.x * 4) >> g.tile_lp)], dr_acc);
  {
    const uint32_t w = __reduce_or_sync(FULL, rany);
    if (lane == 0 && w) atomicOr(&srow_any, w);
  }
  if (g.exact_mma) {
    // a warp's 128 arms lie in one 128 x 256 tile of the tensor-core pass: count them
    const unsigned wex = __reduce_add_sync(FULL, ex_acc);
    if (wex && lane == 0) atomicAdd(&g.xflags[(size_t)(q0 >> 7) * g.xf_cols + (i0 >> 8)], wex);
  }
  __syncthreads();
  if (threadIdx.x < NSLOT && scnt[threadIdx.x]) atomicAdd(&g.ctl->cnt[threadIdx.x], scnt[threadIdx.x]);
  if (threadIdx.x == 0) g.rowany[(size_t)blockIdx.y * g.rowany_cols + blockIdx.x] = srow_any;
  if (g.level_mma)
    for (int t = threadIdx.x; t < (FIL_NT * 4 / 128) * MAX_LEVELS; t += FIL_NT) {
      const int lc = ((blockIdx.x * FIL_NT * 4) >> 7) + t / MAX_LEVELS;
      if (lvc[t] && lc < g.lv_cols)
        atomicAdd(&g.lvcnt[((size_t)(q0 >> 7) * g.lv_cols + lc) * MAX_LEVELS + t % MAX_LEVELS], lvc[t]);
    }
  // every tile of this CTA, including those of finished queries (count 0)
  uint32_t tmax = 0, tmin = 0xFFFFFFFFu;
  for (int t = threadIdx.x; t < ntc; t += FIL_NT) {
    const int tr = (q0 >> g.tile_lr) + t / tcols;
    const int tc = ((blockIdx.x * FIL_NT * 4) >> g.tile_lp) + t % tcols;
    if ((tr << g.tile_lr) < g.q && tc < g.tile_cols) {
      g.tilework[(size_t)tr * g.tile_cols + tc] = tcnt[t];
      tmax = max(tmax, tcnt[t]);
      if ((float)tcnt[t] >= g.tile_min_draws) tmin = min(tmin, tcnt[t]);
    }
  }
  if (g.tile_on) {
    tmax = __reduce_max_sync(FULL, tmax);
    tmin = __reduce_min_sync(FULL, tmin);
    if (lane == 0 && tmax) atomicMax(&g.ctl->tile_max, tmax);
    if (lane == 0 && tmin != 0xFFFFFFFFu) atomicMin(&g.ctl->tile_min, tmin);
  }
}

// Work decomposition of one advance level c (s = 2^c draws = nb Philox blocks of 4
// draws per pair).  Every lane runs ADV_P independent Philox blocks at a time (ILP
// across the 10 dependent rounds):
//   nb <= ADV_P        a lane owns ADV_P / nb whole pairs (no cross-lane reduce)
//   nb <= 32 * ADV_P   nb / ADV_P lanes per pair (shuffle reduce inside the group)
//   otherwise          a warp per pair, lanes loop over ADV_P-block groups
// Exact fallbacks (slot MAX_LEVELS): ADV_XP pairs per warp, rows streamed with
// 16-B loads.  A warp-chunk is one warp's share of a slot.
constexpr int ADV_P = 4;
constexpr int ADV_XP = 4;

// Philox blocks per pair of the advance out of level c (doubling: max(1, 2^(c-2))).
__host__ __device__ __forceinline__ unsigned nblk_of(int c, int growth) {
  const LevelAdvance a = lvl_advance((uint32_t)c, growth);
  return a.cnt < 4u ? 1u : a.cnt / 4u;
}
// Lanes per pair at levels with nb > ADV_P blocks: each lane runs >= ADV_BPL blocks
// (two rounds of ADV_P independent Philox blocks) before the group reduce.
__host__ __device__ __forceinline__ unsigned lanes_per_pair(unsigned nb, unsigned bpl) {
  const unsigned t = nb / bpl;
  return t < 1u ? 1u : (t > 32u ? 32u : t);
}
__host__ __device__ __forceinline__ unsigned pairs_per_chunk(int slot, unsigned bpl, int stage_lo, int growth) {
  if (slot == MAX_LEVELS) return ADV_XP;
  if (slot >= stage_lo) return 1u;  // row-staged levels: one pair per warp
  const unsigned nb = nblk_of(slot, growth);
  return nb <= (unsigned)ADV_P ? 32u * ADV_P / nb : 32u / lanes_per_pair(nb, bpl);
}

// One thread per slot (NSLOT <= 64): counts and warp-chunks per slot, then the prefix
// sums across the two warps.
__global__ void k_plan(RoundCtl *ctl, unsigned bpl, int stage_lo, int level_mma, unsigned level_min, int growth) {
  __shared__ unsigned wsum_c[2];
  __shared__ unsigned long long wsum_ch[2];
  const int s = threadIdx.x, lane = s & 31, w = s >> 5;
  const unsigned c = s < NSLOT ? ctl->cnt[s] : 0u;
  const unsigned ppc = s < NSLOT ? pairs_per_chunk(s, bpl, stage_lo, growth) : 1u;
  const unsigned long long chs = (c + ppc - 1) / ppc;
  unsigned ic = c;
  unsigned long long ich = chs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned a = __shfl_up_sync(FULL, ic, o);
    const unsigned long long b = __shfl_up_sync(FULL, ich, o);
    if (lane >= o) {
      ic += a;
      ich += b;
    }
  }
  if (lane == 31) {
    wsum_c[w] = ic;
    wsum_ch[w] = ich;
  }
  __syncthreads();
  const unsigned base_c = w ? wsum_c[0] : 0u;
  const unsigned long long base_ch = w ? wsum_ch[0] : 0ull;
  if (s < NSLOT) {
    ctl->off[s] = base_c + ic - c;
    ctl->chunk_off[s] = base_ch + ich - chs;
    ctl->cursor[s] = 0;
  }
  if (s == 0) {
    const unsigned tot = wsum_c[0] + wsum_c[1];
    ctl->off[NSLOT] = tot;
    ctl->chunk_off[NSLOT] = wsum_ch[0] + wsum_ch[1];
    ctl->advanced += tot;
    int best = -1;
    unsigned bc = 0;
    if (level_mma)  // shared draws: the most populated sampled level goes to the tensor cores
      for (int t = 0; t < MAX_LEVELS; ++t)
        if (ctl->cnt[t] > bc) {
          bc = ctl->cnt[t];
          best = t;
        }
    ctl->gemm_level = (best >= 0 && bc >= level_min) ? best : -1;
  }
}

// After the scatter: the lists hold only the pairs of sparse tiles (and the exact
// fallbacks of sparse tensor-core tiles), cursor[s] of them per slot; the advance
// kernels walk exactly those.
__global__ void k_plan_lists(RoundCtl *ctl, unsigned bpl, int stage_lo, int growth) {
  __shared__ unsigned long long wsum_ch[2];
  const int s = threadIdx.x, lane = s & 31, w = s >> 5;
  const unsigned c = s < NSLOT ? ctl->cursor[s] : 0u;
  const unsigned ppc = s < NSLOT ? pairs_per_chunk(s, bpl, stage_lo, growth) : 1u;
  const unsigned long long chs = (c + ppc - 1) / ppc;
  unsigned long long ich = chs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long b = __shfl_up_sync(FULL, ich, o);
    if (lane >= o) ich += b;
  }
  if (lane == 31) wsum_ch[w] = ich;
  __syncthreads();
  const unsigned long long base_ch = w ? wsum_ch[0] : 0ull;
  if (s < NSLOT) {
    ctl->cnt[s] = c;
    ctl->chunk_off[s] = base_ch + ich - chs;
  }
  if (s == 0) ctl->chunk_off[NSLOT] = wsum_ch[0] + wsum_ch[1];
}

// a8: compaction of the action bytes into per-slot lists of (qi << ibits | i).
// One CTA per (query, 1024-arm chunk); thread t owns arms chunk + t + 256 e, so for
// each e a warp covers 32 consecutive arms.  Slots are counted in shared memory
// (warp-aggregated), the CTA reserves one range per slot with ONE global atomic,
// and writes its entries there: list order within a slot follows the arm order
// of each warp, so the advance kernel reads S / level nearly sequentially.
// A CTA walks `cpb` consecutive 1,024-arm chunks of its query row (one CTA per chunk
// spent most of the pass launching and retiring CTAs that exit at once: in lock-step
// rounds nearly every chunk lies in dense tiles and lists nothing).  The list order
// follows the CTA order -- the chunk's queries together -- so the list advance finds a
// chunk's point rows in L2; cpb stays 1 when cpb chunks of rows would not fit there.
__global__ void __launch_bounds__(FIL_NT) k_scatter(Geom g, int cpb) {
  const int qi = blockIdx.x;
  __shared__ unsigned scnt[NSLOT], sbase[NSLOT];
  __shared__ uint8_t sdense[FIL_NT * 4 / 4];  // the chunk's (R x P) tiles: dense?
  __shared__ uint8_t smma[FIL_NT * 4 / 256];   // its 128 x 256 exact tiles: tensor cores?
  __shared__ int any_listed;
  __shared__ uint8_t slv[FIL_NT * 4 / 128];  // the chunk's 128 x 128 level tiles: tensor cores?
  const int nch = (int)((g.npad + FIL_NT * 4 - 1) / (FIL_NT * 4));
  for (int cy = blockIdx.y * cpb; cy < min(nch, (int)(blockIdx.y + 1) * cpb); ++cy) {
  // nothing to list in this row's chunk (k_filter's per-row action mask; finished
  // queries have no actions): skip it before the tile decisions (uniform over the CTA)
  if (!((g.rowany[(size_t)(qi >> 5) * g.rowany_cols + cy] >> (qi & 31)) & 1u)) continue;
  __syncthreads();  // the previous chunk's readers of the shared arrays are done
  const int c0 = cy * FIL_NT * 4;
  const int ntile = g.tile_on ? (FIL_NT * 4) >> g.tile_lp : 0;
  for (int s = threadIdx.x; s < NSLOT; s += FIL_NT) scnt[s] = 0;
  if (threadIdx.x == 0) any_listed = 0;
  __syncthreads();
  // the chunk's tile decisions, once; a chunk whose sampled pairs all lie in dense
  // tiles and whose exact ones all go to the tensor cores lists nothing
  for (int t = threadIdx.x; t < ntile; t += FIL_NT) {
    const int tc = (c0 >> g.tile_lp) + t;
    const bool dense = tc < g.tile_cols &&
                       (float)g.tilework[(size_t)(qi >> g.tile_lr) * g.tile_cols + tc] >=
                           g.tile_min_draws;
    sdense[t] = dense;
    if (!dense) any_listed = 1;
  }
  if (!g.tile_on && !g.level_mma && threadIdx.x == 0) any_listed = 1;
  const int glev = g.level_mma ? g.ctl->gemm_level : -1;
  if (g.level_mma && threadIdx.x < (FIL_NT * 4) / 128) {
    // a level tile lists nothing when all its sampled pairs sit at the GEMM level, the
    // GEMM takes it and no point of the round overflows its w planes
    const int lc = (c0 >> 7) + (int)threadIdx.x;
    bool mma = false, other = false;
    if (lc < g.lv_cols) {
      const uint32_t *f = g.lvcnt + ((size_t)(qi >> 7) * g.lv_cols + lc) * MAX_LEVELS;
      for (int s = 0; s < MAX_LEVELS; ++s) {
        const uint32_t v = f[s];
        if (s == glev) mma = v >= g.lmin;
        else other |= v != 0u;
      }
      if (glev >= 0 && !mma && f[glev] != 0u) other = true;
    }
    slv[threadIdx.x] = mma;
    if (other || (mma && g.ctl->wovf_any)) any_listed = 1;
  }
  if (threadIdx.x < (FIL_NT * 4) / 256) {
    const int xc = (c0 >> 8) + (int)threadIdx.x;
    const uint32_t cnt = (g.exact_mma && xc < g.xf_cols) ? g.xflags[(size_t)(qi >> 7) * g.xf_cols + xc] : 0u;
    smma[threadIdx.x] = g.exact_mma && cnt >= g.xmin;
    if (cnt != 0u && cnt < g.xmin) any_listed = 1;
    if (!g.exact_mma) any_listed = 1;
  }
  __syncthreads();
  if (!any_listed) continue;
  const int base_i = c0 + threadIdx.x;
  const uint8_t *arow = g.act + (size_t)qi * g.npad;
  const int lane = lane_id();
  unsigned slot[4], loc[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int i = base_i + e * FIL_NT;
    const uint8_t act = i < g.n ? arow[i] : (uint8_t)0;
    slot[e] = act == 0 ? NONE : (act == ACT_EXACT ? (unsigned)MAX_LEVELS : act - 1u);
    if (slot[e] == (unsigned)MAX_LEVELS && smma[(i - c0) >> 8])
      slot[e] = NONE;  // a dense tile of the tensor-core exact pass takes it
    if (g.tile_on && slot[e] < (unsigned)MAX_LEVELS && sdense[(i - c0) >> g.tile_lp])
      slot[e] = NONE;  // k_advance_tiles takes it
    if (g.level_mma && (int)slot[e] == glev && slv[(i - c0) >> 7] && !g.wovf[i])
      slot[e] = NONE;  // k_level_mma takes it
    const unsigned m = __match_any_sync(FULL, slot[e]);
    const int leader = __ffs(m) - 1;
    unsigned b = 0;
    if (slot[e] != NONE && lane == leader) b = atomicAdd(&scnt[slot[e]], (unsigned)__popc(m));
    b = __shfl_sync(FULL, b, leader);
    loc[e] = b + __popc(m & ((1u << lane) - 1u));
  }
  __syncthreads();
  if (threadIdx.x < NSLOT && scnt[threadIdx.x])
    sbase[threadIdx.x] = g.ctl->off[threadIdx.x] + atomicAdd(&g.ctl->cursor[threadIdx.x], scnt[threadIdx.x]);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (slot[e] != NONE)
      g.list[sbase[slot[e]] + loc[e]] = ((uint32_t)qi << g.ibits) | (uint32_t)(base_i + e * FIL_NT);
  }
}

// ---------------------------------------------------------------------------
// a3 + a4: advance every listed pair.  Grid-stride over warp-chunks.
constexpr int ADV_NT = 256;

// Sum of the squared differences of the draws u = 4*blk .. 4*blk+3 (< s) of pair
// (qi, i) at level b = c + 1 (T -> 2T, t = T + u), for ADV_P blocks at once.
struct BlockTask {
  const uint8_t *xr, *qr;  // rows of X and of the query
  uint32_t i, qi, blk;      // global point id, RNG query index, Philox block
  bool valid;
};

// The advance out of level c draws the in-level ordinals u0 .. u0 + s - 1 of sample
// level b (doubling: b = c + 1, u0 = 0, s = 2^c); with s < 4 the block's words
// w0 = u0 & 3 .. w0 + s - 1 are the draws, the others are discarded.
__device__ __forceinline__ void draw_blocks(const Geom &g, const BlockTask (&t)[ADV_P], const LevelAdvance &av,
                                            uint32_t (&acc)[ADV_P]) {
  const uint32_t s = av.cnt, w0 = av.u0 & 3u, blk0 = av.u0 >> 2;
  uint4 w[ADV_P];  // Philox words, or the arm's permutation keys (without replacement)
#pragma unroll
  for (int k = 0; k < ADV_P; ++k)
    w[k] = g.wor ? wor_keys(g.rk0, g.rk1, t[k].i, t[k].qi)
                 : philox4x32_10_rk(make_uint4(blk0 + t[k].blk, t[k].i, t[k].qi, av.b), g.rk0, g.rk1);
#pragma unroll
  for (int k = 0; k < ADV_P; ++k) {
    const uint32_t ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
    uint32_t a = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // s < 4 only at the first levels (1 or 2 draws); other words are discarded
      if (t[k].valid && (s >= 4 || ((uint32_t)e >= w0 && (uint32_t)e < w0 + s))) {
        const uint32_t j = g.wor ? wor_coord(w[k], g.wor_z, (uint32_t)g.d, s + 4u * t[k].blk + (uint32_t)e)
                                 : coord_of(ws[e], (uint32_t)g.d);
        const int diff = (int)__ldg(t[k].xr + j) - (int)__ldg(t[k].qr + j);
        a += (uint32_t)(diff * diff);
      }
    }
    acc[k] = a;
  }
}

// Without replacement: the draws 4 blk0 .. 4 (blk0 + ADV_P) - 1 of the level are
// pi(2^c + u) under the arm's keys kk (reading R23).
__device__ __forceinline__ uint32_t draw4_pair_wor(const Geom &g, const uint8_t *__restrict__ xr,
                                                   const uint8_t *__restrict__ qr, uint4 kk, uint32_t lv,
                                                   uint32_t blk0) {
  const uint32_t t0 = (1u << (lv - 1u)) + 4u * blk0;
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < ADV_P; ++k) {
    const uint4 j4 = wor_coords4(kk, g.wor_z, (uint32_t)g.d, t0 + 4u * (uint32_t)k);
    const uint32_t js[4] = {j4.x, j4.y, j4.z, j4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int diff = (int)__ldg(xr + js[e]) - (int)__ldg(qr + js[e]);
      acc += (uint32_t)(diff * diff);
    }
  }
  return acc;
}

// ADV_P consecutive Philox blocks blk0.. of ONE pair (all 4 draws of each used: s >= 4).
__device__ __forceinline__ uint32_t draw4_pair(const Geom &g, const uint8_t *__restrict__ xr,
                                               const uint8_t *__restrict__ qr, uint32_t gi, uint32_t gq,
                                               uint32_t lv, uint32_t blk0) {
  const PhiloxPair pc = philox_pair(gi, gq, g.rk0);
  uint4 w[ADV_P];
#pragma unroll
  for (int k = 0; k < ADV_P; ++k) w[k] = philox_from_pair(blk0 + k, lv, pc, g.rk0, g.rk1);
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < ADV_P; ++k) {
    const uint32_t ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t j = coord_of(ws[e], (uint32_t)g.d);
      const int diff = (int)__ldg(xr + j) - (int)__ldg(qr + j);
      acc += (uint32_t)(diff * diff);
    }
  }
  return acc;
}

__device__ __forceinline__ void decode(const Geom &g, uint32_t code, uint32_t imask, uint32_t &qi,
                                       uint32_t &i) {
  qi = code >> g.ibits;
  i = code & imask;
}

__device__ __forceinline__ void commit(const Geom &g, uint32_t qi, uint32_t i, uint32_t add,
                                       uint8_t lvl) {
  const size_t o = (size_t)qi * g.npad + i;
  g.S[o] += (int32_t)add;
  g.lvl[o] = lvl;
}

// Exact fallback of up to ADV_XP pairs per warp: S = sum_j (x_j - q_j)^2.
__device__ __forceinline__ void exact_rows(const Geom &g, const uint32_t *codes, unsigned cnt,
                                           uint32_t imask) {
  const int lane = lane_id();
  const int nv = (int)(g.pitch >> 4);
  const uint4 *xr[ADV_XP], *qr[ADV_XP];
  uint32_t acc[ADV_XP];
#pragma unroll
  for (int p = 0; p < ADV_XP; ++p) {
    uint32_t qi = 0, i = 0;
    if ((unsigned)p < cnt) decode(g, codes[p], imask, qi, i);
    xr[p] = reinterpret_cast<const uint4 *>(g.X + (size_t)i * g.pitch);
    qr[p] = reinterpret_cast<const uint4 *>(g.Q + (size_t)qi * g.pitch);
    acc[p] = 0;
  }
  for (int v0 = 0; v0 < nv; v0 += 64) {
    uint4 a[ADV_XP][2], b[ADV_XP][2];
#pragma unroll
    for (int p = 0; p < ADV_XP; ++p)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int v = v0 + h * 32 + lane;
        const bool ok = (unsigned)p < cnt && v < nv;
        a[p][h] = ok ? __ldg(xr[p] + v) : make_uint4(0, 0, 0, 0);
        b[p][h] = ok ? __ldg(qr[p] + v) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int p = 0; p < ADV_XP; ++p)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t t;
        t = __vabsdiffu4(a[p][h].x, b[p][h].x); acc[p] = __dp4a(t, t, acc[p]);
        t = __vabsdiffu4(a[p][h].y, b[p][h].y); acc[p] = __dp4a(t, t, acc[p]);
        t = __vabsdiffu4(a[p][h].z, b[p][h].z); acc[p] = __dp4a(t, t, acc[p]);
        t = __vabsdiffu4(a[p][h].w, b[p][h].w); acc[p] = __dp4a(t, t, acc[p]);
      }
  }
#pragma unroll
  for (int p = 0; p < ADV_XP; ++p)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[p] += __shfl_xor_sync(FULL, acc[p], o);
  if (lane < ADV_XP && (unsigned)lane < cnt) {
    uint32_t mine = acc[0];
#pragma unroll
    for (int p = 1; p < ADV_XP; ++p)
      if (lane == p) mine = acc[p];
    uint32_t qi, i;
    decode(g, codes[lane], imask, qi, i);
    const size_t o = (size_t)qi * g.npad + i;
    g.S[o] = (int32_t)mine;
    g.lvl[o] = lvl_to_exact(g.lvl[o]);
  }
}

__global__ void __launch_bounds__(ADV_NT) k_advance(Geom g) {
  __shared__ unsigned long long coff[NSLOT + 1];
  __shared__ unsigned scnt[NSLOT], soff[NSLOT];
  for (int s = threadIdx.x; s <= NSLOT; s += ADV_NT) {
    coff[s] = g.ctl->chunk_off[s];
    if (s < NSLOT) {
      scnt[s] = g.ctl->cnt[s];
      soff[s] = g.ctl->off[s];
    }
  }
  __syncthreads();
  // this kernel takes the levels below stage_lo and the exact fallbacks; the
  // row-staged levels [stage_lo, MAX_LEVELS) belong to k_advance_staged
  const int slo = g.stage_lo < MAX_LEVELS ? g.stage_lo : MAX_LEVELS;
  const unsigned long long total_a = coff[slo], skip = coff[MAX_LEVELS] - coff[slo];
  // (exact fallbacks of dense tensor-core tiles are not listed: k_mma_tiles takes them)
  const unsigned long long total = coff[NSLOT] - skip;
  const unsigned long long nwarps = (unsigned long long)gridDim.x * (ADV_NT / 32);
  const int lane = lane_id();
  const uint32_t imask = (1u << g.ibits) - 1u;
  int slot = 0;
  for (unsigned long long vch = (unsigned long long)blockIdx.x * (ADV_NT / 32) + (threadIdx.x >> 5);
       vch < total; vch += nwarps) {
    const unsigned long long ch = vch < total_a ? vch : vch + skip;
    while (coff[slot + 1] <= ch) ++slot;  // chunks are visited in increasing order
    const unsigned long long rel = ch - coff[slot];
    if (slot == MAX_LEVELS) {
      const unsigned p0 = (unsigned)rel * ADV_XP;
      const unsigned cnt = min((unsigned)ADV_XP, scnt[slot] - p0);
      exact_rows(g, g.list + soff[slot] + p0, cnt, imask);
      continue;
    }
    const int c = slot;
    const LevelAdvance av = lvl_advance((uint32_t)c, g.growth);
    const unsigned nb = nblk_of(c, g.growth);
    const uint8_t newlvl = (uint8_t)(c + 1);
    const unsigned ppc = pairs_per_chunk(c, g.adv_bpl, g.stage_lo, g.growth);
    const unsigned pbase = (unsigned)rel * ppc;  // first pair of this chunk
    const uint32_t *lst = g.list + soff[c];
    const unsigned cnt = scnt[c];
    if (nb <= (unsigned)ADV_P) {
      // lane owns ppt pairs: pbase + j*32 + lane, each with nb blocks
      constexpr int dummy = 0;
      (void)dummy;
      const unsigned ppt = ADV_P / nb;
      BlockTask t[ADV_P];
      uint32_t code[ADV_P];
#pragma unroll
      for (int k = 0; k < ADV_P; ++k) {
        const unsigned j = k / nb, blk = k % nb;  // nb is a power of two <= ADV_P
        const unsigned p = pbase + j * 32 + lane;
        const bool ok = j < ppt && p < cnt;
        uint32_t qi = 0, i = 0;
        code[k] = ok ? lst[p] : 0u;
        decode(g, code[k], imask, qi, i);
        t[k] = BlockTask{g.X + (size_t)i * g.pitch, g.Q + (size_t)qi * g.pitch, i + g.id_offset,
                         rng_qi(g, qi), blk, ok};
      }
      uint32_t acc[ADV_P];
      draw_blocks(g, t, av, acc);
#pragma unroll
      for (int k = 0; k < ADV_P; ++k) {
        if (k % nb != 0 || !t[k].valid) continue;
        uint32_t sum = 0;
#pragma unroll
        for (int e = 0; e < ADV_P; ++e)
          if (e / nb == k / nb) sum += acc[e];
        uint32_t qi, i;
        decode(g, code[k], imask, qi, i);
        commit(g, qi, i, sum, newlvl);
      }
    } else {
      // tpp lanes per pair (a warp holds 32/tpp pairs); lane `sub` of a pair runs the
      // blocks (it*tpp + sub)*ADV_P + k, ADV_P independent Philox chains at a time
      const unsigned tpp = lanes_per_pair(nb, g.adv_bpl);
      const unsigned p = pbase + lane / tpp, sub = lane % tpp;
      const bool ok = p < cnt;
      uint32_t qi = 0, i = 0, sum = 0;
      if (ok) decode(g, lst[p], imask, qi, i);
      // keep the two row pointers live in registers: otherwise ptxas re-derives
      // X + i*pitch + j for every draw with an IMAD.WIDE on the fma-heavy pipe, the
      // pipe Philox saturates (ncu: fmaheavy 73 %).  A shuffle result cannot be
      // rematerialised, so the pointers stay put.
      const uint8_t *xr = reinterpret_cast<const uint8_t *>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(g.X + (size_t)i * g.pitch), lane));
      const uint8_t *qr = reinterpret_cast<const uint8_t *>(
          __shfl_sync(FULL, reinterpret_cast<unsigned long long>(g.Q + (size_t)qi * g.pitch), lane));
      if (ok) {
        const uint32_t gi = i + g.id_offset, gq = rng_qi(g, qi), lv = av.b, blk0 = av.u0 >> 2;
        if (g.wor) {  // (doubling only: u0 = 0)
          const uint4 kk = wor_keys(g.rk0, g.rk1, gi, gq);
          for (unsigned b0 = sub * ADV_P; b0 < nb; b0 += tpp * ADV_P) sum += draw4_pair_wor(g, xr, qr, kk, lv, b0);
        } else {
          for (unsigned b0 = sub * ADV_P; b0 < nb; b0 += tpp * ADV_P)
            sum += draw4_pair(g, xr, qr, gi, gq, lv, blk0 + b0);
        }
      }
      for (unsigned o = tpp >> 1; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
      if (ok && sub == 0) commit(g, qi, i, sum, newlvl);
    }
  }
}

// Row-staged levels (large d, many draws per pair): the warp copies the point's
// row into shared memory with 16-byte loads (one streaming read of d bytes instead
// of one random 32-byte sector per draw), then gathers its draws from there.
__device__ __forceinline__ uint32_t draw4_pair_srow(const Geom &g, const uint8_t *sx, const uint8_t *__restrict__ qr,
                                                    uint32_t gi, uint32_t gq, uint32_t lv, uint32_t blk0) {
  const PhiloxPair pc = philox_pair(gi, gq, g.rk0);
  uint4 w[ADV_P];
#pragma unroll
  for (int k = 0; k < ADV_P; ++k) w[k] = philox_from_pair(blk0 + k, lv, pc, g.rk0, g.rk1);
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < ADV_P; ++k) {
    const uint32_t ws[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t j = coord_of(ws[e], (uint32_t)g.d);
      const int diff = (int)sx[j] - (int)__ldg(qr + j);
      acc += (uint32_t)(diff * diff);
    }
  }
  return acc;
}

__global__ void __launch_bounds__(ADV_NT) k_advance_staged(Geom g) {
  extern __shared__ uint4 srow[];
  __shared__ unsigned long long coff[NSLOT + 1];
  __shared__ unsigned soff[NSLOT];
  for (int s = threadIdx.x; s <= NSLOT; s += ADV_NT) {
    coff[s] = g.ctl->chunk_off[s];
    if (s < NSLOT) soff[s] = g.ctl->off[s];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = lane_id();
  const int nv = (int)(g.pitch >> 4);
  uint4 *sx = srow + (size_t)warp * nv;
  const uint32_t imask = (1u << g.ibits) - 1u;
  const unsigned long long c0 = coff[g.stage_lo], total = coff[MAX_LEVELS] - c0;
  const unsigned long long nwarps = (unsigned long long)gridDim.x * (ADV_NT / 32);
  int slot = g.stage_lo;
  for (unsigned long long vch = (unsigned long long)blockIdx.x * (ADV_NT / 32) + warp; vch < total;
       vch += nwarps) {
    const unsigned long long ch = c0 + vch;
    while (coff[slot + 1] <= ch) ++slot;
    const int c = slot;  // (doubling only: staged levels are off under growth 2)
    const unsigned nb = nblk_of(c, g.growth);
    const uint32_t code = g.list[soff[c] + (ch - coff[c])];
    uint32_t qi, i;
    decode(g, code, imask, qi, i);
    const uint4 *xg = reinterpret_cast<const uint4 *>(g.X + (size_t)i * g.pitch);
    __syncwarp();
    for (int v = lane; v < nv; v += 32) sx[v] = __ldg(xg + v);
    __syncwarp();
    const uint8_t *sxb = reinterpret_cast<const uint8_t *>(sx);
    const uint8_t *qr = g.Q + (size_t)qi * g.pitch;
    const uint32_t gi = i + g.id_offset, gq = rng_qi(g, qi), lv = (uint32_t)(c + 1);
    uint32_t sum = 0;
    if (g.wor) {  // reading R23: pi(2^c + u) under the arm's keys
      const uint4 kk = wor_keys(g.rk0, g.rk1, gi, gq);
      const uint32_t t0 = 1u << c;  // staged levels draw >= 64 per pair: 4 per lane step
      for (unsigned u = 4 * lane; u < (1u << c); u += 128) {
        const uint4 j4 = wor_coords4(kk, g.wor_z, (uint32_t)g.d, t0 + u);
        const uint32_t js[4] = {j4.x, j4.y, j4.z, j4.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int diff = (int)sxb[js[e]] - (int)__ldg(qr + js[e]);
          sum += (uint32_t)(diff * diff);
        }
      }
    } else {
      for (unsigned b0 = lane * ADV_P; b0 < nb; b0 += 32 * ADV_P) sum += draw4_pair_srow(g, sxb, qr, gi, gq, lv, b0);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    if (lane == 0) commit(g, qi, i, sum, (uint8_t)(c + 1));
  }
}

// ---------------------------------------------------------------------------
// a9: output.  The k+h arms with key <= thr_kh, in rank order.
constexpr int OUT_NT = 256;
constexpr int OUT_MAXKH = 4096;

__global__ void __launch_bounds__(OUT_NT) k_output(Geom g, OutPtrs o) {
  const int qi = blockIdx.x;
  const QState st = g.qs[qi];
  const int kh = g.k + g.h;
  extern __shared__ unsigned char osm[];
  unsigned long long *key = reinterpret_cast<unsigned long long *>(osm);
  int32_t *sv = reinterpret_cast<int32_t *>(key + kh);
  int32_t *iv = sv + kh;
  uint8_t *lv = reinterpret_cast<uint8_t *>(iv + kh);
  __shared__ unsigned cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i0 = threadIdx.x * 4; i0 < g.n; i0 += OUT_NT * 4) {
    const Arm4 a = load_arm4(g, qi, i0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e;
      if (i >= g.n) break;
      const unsigned long long kk = arm_key(a.S[e], a.l(e), (uint32_t)i, g);
      if (kk <= st.thr_kh) {
        const unsigned p = atomicAdd(&cnt, 1u);
        if (p < (unsigned)kh) {
          key[p] = kk;
          sv[p] = a.S[e];
          iv[p] = i;
          lv[p] = a.l(e);
        }
      }
    }
  }
  __syncthreads();
  const int m = min((int)cnt, kh);
  for (int r = threadIdx.x; r < m; r += OUT_NT) {
    int rank = 0;
    for (int t = 0; t < m; ++t) rank += key[t] < key[r];
    const size_t oo = (size_t)(o.row0 + qi) * kh + rank;
    o.sets[oo] = (int32_t)(iv[r] + g.id_offset);
    if (o.dhat) o.dhat[oo] = dhat_of(sv[r], lv[r], g.d, g.growth);
  }
  if (threadIdx.x == 0) {
    const size_t row = (size_t)(o.row0 + qi);
    if (o.draws) o.draws[row] = st.draws;
    if (o.evals) o.evals[row] = st.draws + st.exact_evals;
    if (o.rounds) o.rounds[row] = st.rounds;
  }
}

// Per-query counters from the final arm states (SPEC S:250-258 accounting): an arm
// at sampled level c drew T_c coordinates (1 at initialisation, then the advances);
// an exact arm drew T_c before its fallback, which is charged d (d = 1: exact at
// initialisation, no fallback).  Philox blocks of the level gathers: the advance out
// of level l used nblk_of(l) (doubling: max(1, 2^(l-2))).
// Every statistic is a function of the arm's level byte alone, so the pass only counts
// the arms per byte value (a per-thread run-length count: in lock-step rows a 4-byte
// word of one level adds 4 at once; a shared histogram takes the runs), and 256 threads
// then turn the histogram into the sums.  (Per-arm 64-bit sums over 16-byte loads left
// the pass latency-bound: C4 1.8 ms per query batch.)
template <int NT>
__global__ void __launch_bounds__(NT) k_tally(Geom g) {
  const int qi = blockIdx.x;
  __shared__ unsigned hist[256];
  __shared__ unsigned long long red[4][NT / 32];
  for (int t = threadIdx.x; t < 256; t += NT) hist[t] = 0;
  __syncthreads();
  const uint8_t *lrow = g.lvl + (size_t)qi * g.npad;
  uint32_t cur = 0xFFFFFFFFu, run = 0;
  auto add = [&](uint32_t b, uint32_t k) {
    if (b == cur) {
      run += k;
      return;
    }
    if (run) atomicAdd(&hist[cur], run);
    cur = b;
    run = k;
  };
  // 16 level bytes per load (npad is a multiple of 16; bytes past n are skipped)
  for (int i0 = threadIdx.x * 16; i0 < g.n; i0 += NT * 16) {
    const uint4 v = *reinterpret_cast<const uint4 *>(lrow + i0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int j0 = i0 + 4 * q4;
      if (j0 + 4 <= g.n && w[q4] == (w[q4] & 0xFFu) * 0x01010101u) {
        add(w[q4] & 0xFFu, 4u);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (j0 + e < g.n) add((w[q4] >> (8 * e)) & 0xFFu, 1u);
      }
    }
  }
  if (run) atomicAdd(&hist[cur], run);
  __syncthreads();
  unsigned long long dr = 0, ex = 0, bl = 0, xe = 0;
  for (int b = threadIdx.x; b < 256; b += NT) {
    const unsigned long long m = hist[b];
    if (!m) continue;
    const uint8_t l = (uint8_t)b;
    const uint32_t c = l & 0x7Fu;
    const unsigned long long T = lvl_count(c, g.growth);
    unsigned long long cb = 0;  // Philox blocks drawn to reach level c
    for (uint32_t c2 = 0; c2 < c && c2 < (uint32_t)MAX_LEVELS; ++c2) cb += nblk_of((int)c2, g.growth);
    dr += m * T;
    const bool fb = lvl_exact(l) && g.d > 1;
    ex += fb ? m : 0ull;
    // charge of the fallback: d, or without replacement the d - T_c coordinates the
    // arm's permutation had not drawn yet (reading R23)
    xe += fb ? m * (g.wor ? (unsigned long long)g.d - T : (unsigned long long)g.d) : 0ull;
    bl += m * cb;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dr += __shfl_xor_sync(FULL, dr, o);
    ex += __shfl_xor_sync(FULL, ex, o);
    bl += __shfl_xor_sync(FULL, bl, o);
    xe += __shfl_xor_sync(FULL, xe, o);
  }
  if (lane_id() == 0) {
    red[0][threadIdx.x >> 5] = dr;
    red[1][threadIdx.x >> 5] = ex;
    red[2][threadIdx.x >> 5] = bl;
    red[3][threadIdx.x >> 5] = xe;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < NT / 32; ++w) {
      dr += red[0][w];
      ex += red[1][w];
      bl += red[2][w];
      xe += red[3][w];
    }
    g.qs[qi].draws = (long long)dr;
    g.qs[qi].nexact = (long long)ex;
    g.qs[qi].exact_evals = (long long)xe;
    g.qs[qi].blocks = (long long)bl;
  }
}

cudaError_t launch_tally(const Geom &g, cudaStream_t s) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g.q <= sms)
    k_tally<1024><<<g.q, 1024, 0, s>>>(g);
  else
    k_tally<256><<<g.q, 256, 0, s>>>(g);
  return cudaGetLastError();
}

__global__ void k_counts(Geom g, OutPtrs o) {
  const int qi = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const size_t src = (size_t)qi * g.npad + i;
  const size_t dst = (size_t)(o.row0 + qi) * o.ncols + o.col0 + i;
  const uint8_t l = g.lvl[src];
  if (o.counts) o.counts[dst] = (int32_t)count_of(l, g.d, g.growth);
  if (o.sums) o.sums[dst] = (int64_t)(uint32_t)g.S[src];
}

// ---------------------------------------------------------------------------
// Launch wrappers.
static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

cudaError_t launch_init(const Geom &g, cudaStream_t s) {
  const long long nch = cdiv(g.npad, 256);
  if (nch <= 65535)
    k_init<true><<<dim3(g.q, (unsigned)nch), 256, 0, s>>>(g);
  else
    k_init<false><<<dim3((unsigned)nch, g.q), 256, 0, s>>>(g);
  k_init_qstate<<<cdiv(g.q, 128), 128, 0, s>>>(g);
  if (g.level_mma) {
    const cudaError_t e = launch_q2_planes(g, s);
    if (e != cudaSuccess) return e;
  }
  if (g.tile_on) {
    const size_t rows = ((size_t)g.q + (1u << g.tile_lr) - 1) >> g.tile_lr;
    const cudaError_t e = cudaMemsetAsync(g.tilework, 0, sizeof(uint32_t) * rows * g.tile_cols, s);
    if (e != cudaSuccess) return e;
  }
  if (g.exact_mma) {
    cudaError_t e = cudaMemsetAsync(g.xflags, 0, sizeof(uint32_t) * (size_t)cdiv(g.q, 128) * g.xf_cols, s);
    if (e == cudaSuccess) e = launch_row_norms(g.Q, g.pitch, g.q, g.nq, s);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_select(const Geom &g, int nbits, cudaStream_t s) {
  const cudaError_t e = launch_select_pivot(g, s);
  if (e != cudaSuccess) return e;
  k_select<<<g.q, SEL_NT, 0, s>>>(g, nbits);
  return launch_thresholds(g, s);
}

cudaError_t launch_filter(const Geom &g, cudaStream_t s) {
  const size_t smem = (g.lead_pass ? 0 : sizeof(int32_t) * (size_t)FIL_ROWS * thr_stride(g.cmax + 1)) +
                      (g.tile_on ? sizeof(uint32_t) * (size_t)(FIL_ROWS >> g.tile_lr) * ((FIL_NT * 4) >> g.tile_lp) : 0);
  const dim3 grid(cdiv(g.npad, FIL_NT * 4), cdiv(g.q, FIL_ROWS));
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, FIL_NT, smem, s>>>(g);
    return cudaGetLastError();
  };
  if (g.lead_pass) return go(k_filter<2>);
  if (g.lead > 1) return go(k_filter<1>);
  return go(k_filter<0>);
}

cudaError_t launch_compact(const Geom &g, cudaStream_t s) {
  k_plan<<<1, 64, 0, s>>>(g.ctl, g.adv_bpl, g.stage_lo, g.level_mma, 1u << 16, g.growth);
  if (g.level_mma) {
    const cudaError_t e = launch_build_w(g, s);
    if (e != cudaSuccess) return e;
  }
  const int cpb = (long long)4 * FIL_NT * 4 * g.pitch <= (16ll << 20) ? 4 : 1;  // 4 chunks' rows <= 16 MB
  k_scatter<<<dim3(g.q, cdiv(cdiv(g.npad, FIL_NT * 4), cpb)), FIL_NT, 0, s>>>(g, cpb);
  k_plan_lists<<<1, 64, 0, s>>>(g.ctl, g.adv_bpl, g.stage_lo, g.growth);  // the lists as written
  return cudaGetLastError();
}

// The list-path advance (and the tensor-core exact fallbacks); the dense tiles are
// launch_advance_tiles.
cudaError_t launch_advance(const Geom &g, int num_sms, cudaStream_t s) {
  if (g.exact_mma) {
    const cudaError_t e = launch_exact_fallback_mma(g, s);
    if (e != cudaSuccess) return e;
  }
  k_advance<<<num_sms * 8, ADV_NT, 0, s>>>(g);
  if (g.stage_lo < MAX_LEVELS) {
    const size_t smem = (size_t)(ADV_NT / 32) * (size_t)g.pitch;
    cudaError_t e = cudaFuncSetAttribute(k_advance_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int per_sm = (int)((200u * 1024u) / (smem + 1024));
    k_advance_staged<<<num_sms * (per_sm < 1 ? 1 : per_sm), ADV_NT, smem, s>>>(g);
  }
  return cudaGetLastError();
}

// First level whose advance stages the point row in shared memory, or MAX_LEVELS for
// none: rows of >= 4 KB (an L1 cannot hold a warp-row per resident warp) and levels
// drawing at least pitch/64 coordinates (random sectors then cost more than one
// streaming pass over the row); rows up to 24 KB (8 warps x pitch <= 192 KB).
int stage_level(int64_t pitch) {
  if (pitch < 4096 || pitch > 24 * 1024) return MAX_LEVELS;
  int c = 0;
  while ((1ll << c) * 64 < pitch) ++c;
  return c < MAX_LEVELS ? c : MAX_LEVELS;
}

cudaError_t launch_output(const Geom &g, const OutPtrs &o, cudaStream_t s) {
  const cudaError_t te = launch_tally(g, s);
  if (te != cudaSuccess) return te;
  const int kh = g.k + g.h;
  const size_t smem = (size_t)kh * (8 + 4 + 4 + 1);
  k_output<<<g.q, OUT_NT, smem, s>>>(g, o);
  if (o.counts || o.sums) k_counts<<<dim3(cdiv(g.n, 256), g.q), 256, 0, s>>>(g, o);
  return cudaGetLastError();
}

int output_max_kh() { return OUT_MAXKH; }

// ---------------------------------------------------------------------------
// Device-side round control for the graph-launched loop: the rank split leaves
// n_active (queries failing Eq. (5)) in the control block; k_round_ctl counts the
// round and sets the WHILE condition = n_active > 0 and the round cap not reached
// (the same rule as the host loop: stop at Eq. (5) for all, or EMAXROUNDS).
__global__ void k_ctl_reset(RoundCtl *ctl, unsigned q) {
  RoundCtl z{};
  z.evaluated = q;
  *ctl = z;
}

__global__ void k_zero_round(RoundCtl *ctl) {
  unsigned *p = reinterpret_cast<unsigned *>(ctl);
  for (int t = threadIdx.x; t < (int)(offsetof(RoundCtl, advanced) / 4); t += blockDim.x) p[t] = 0;
}

__global__ void k_round_ctl(RoundCtl *ctl, cudaGraphConditionalHandle h, int max_rounds) {
  const unsigned r = ++ctl->round;
  const unsigned nact = ctl->n_active;
  ctl->qrounds += ctl->evaluated;
  ctl->brounds += nact;
  ctl->evaluated = nact;
  const bool cont = nact > 0 && (max_rounds <= 0 || (int)r < max_rounds);
  cudaGraphSetConditional(h, cont ? 1u : 0u);
}

cudaError_t launch_ctl_reset(RoundCtl *ctl, unsigned q, cudaStream_t s) {
  k_ctl_reset<<<1, 1, 0, s>>>(ctl, q);
  return cudaGetLastError();
}

cudaError_t launch_zero_round(const Geom &g, cudaStream_t s) {
  k_zero_round<<<1, 128, 0, s>>>(g.ctl);
  return cudaGetLastError();
}

cudaError_t launch_round_ctl(RoundCtl *ctl, cudaGraphConditionalHandle h, int max_rounds, cudaStream_t s) {
  k_round_ctl<<<1, 1, 0, s>>>(ctl, h, max_rounds);
  return cudaGetLastError();
}

}  // namespace aknn
