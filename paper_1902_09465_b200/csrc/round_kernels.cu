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

namespace aknn {

// ---------------------------------------------------------------------------
// Pair state loading: 4 consecutive arms of query row `qi` starting at i0
// (i0 % 4 == 0, rows padded to npad % 16 == 0, so the loads are aligned).
struct Arm4 {
  int32_t S[4];
  uint8_t l[4];
};

__device__ __forceinline__ Arm4 load_arm4(const Geom &g, int qi, int i0) {
  Arm4 a;
  const int4 s = *reinterpret_cast<const int4 *>(g.S + (size_t)qi * g.npad + i0);
  const uint32_t lv = *reinterpret_cast<const uint32_t *>(g.lvl + (size_t)qi * g.npad + i0);
  a.S[0] = s.x; a.S[1] = s.y; a.S[2] = s.z; a.S[3] = s.w;
#pragma unroll
  for (int e = 0; e < 4; ++e) a.l[e] = (uint8_t)(lv >> (8 * e));
  return a;
}

// ---------------------------------------------------------------------------
// a2: initialisation -- S_i = (X[i][j] - x[j])^2 for j = Draw(i, 0), T_i = 1.
__global__ void k_init(Geom g) {
  const int qi = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.npad) return;
  const size_t o = (size_t)qi * g.npad + i;
  if (i >= g.n) {
    g.S[o] = 0;
    g.lvl[o] = LVL_EXACT;
    g.act[o] = 0;
    return;
  }
  const uint4 w = philox4x32_10(make_uint4(0u, (uint32_t)i + g.id_offset, (uint32_t)qi + g.qi0, 0u),
                                g.seed_lo, g.seed_hi);
  const uint32_t j = coord_of(w.x, (uint32_t)g.d);
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
  s.rounds = 0;
  s.draws = g.n;  // one initial draw per arm
  s.nexact = 0;
  g.qs[qi] = s;
}

struct ArmKeys {
  const Geom *g;
  int qi;
  __device__ __forceinline__ void operator()(int i0, unsigned long long key[4]) const {
    if (i0 >= g->n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) key[e] = KEY_INVALID;
      return;
    }
    const Arm4 a = load_arm4(*g, qi, i0);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      key[e] = (i0 + e < g->n) ? arm_key(a.S[e], a.l[e], (uint32_t)(i0 + e), *g) : KEY_INVALID;
  }
};

struct Best {
  double v;
  int i;
  double a;
};

// a6 + a7: rank split, d1/d2/A/B, Eq. (5).  One CTA per query.
__global__ void __launch_bounds__(SEL_NT) k_select(Geom g, int nbits) {
  __shared__ SelSmem sm;
  __shared__ Best wbest[2][SEL_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
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
      const unsigned long long key = arm_key(a.S[e], a.l[e], (uint32_t)i, g);
      if (key <= thk) {
        const double U = __dadd_rn(dhat_of(a.S[e], a.l[e], g.d), alpha_of(a.l[e], g.alpha));
        if (U > bu.v || (U == bu.v && i < bu.i)) bu = Best{U, i, 0.0};
      } else if (key > thkh) {
        const double al = alpha_of(a.l[e], g.alpha);
        const double L = __dsub_rn(dhat_of(a.S[e], a.l[e], g.d), al);
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
constexpr int FIL_NT = 256;

__global__ void __launch_bounds__(FIL_NT) k_filter(Geom g) {
  const int qi = blockIdx.y;
  const QState st = g.qs[qi];
  if (st.done) return;
  const int i0 = (blockIdx.x * FIL_NT + threadIdx.x) * 4;
  __shared__ unsigned scnt[NSLOT];
  __shared__ unsigned long long sdraw, sexact;
  for (int s = threadIdx.x; s < NSLOT; s += FIL_NT) scnt[s] = 0;
  if (threadIdx.x == 0) sdraw = sexact = 0;
  __syncthreads();
  unsigned long long mydraw = 0, myexact = 0;
  uint32_t actw = 0;
  if (i0 < g.npad) {
    if (i0 < g.n) {
      const Arm4 a = load_arm4(g, qi, i0);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = i0 + e;
        uint8_t act = 0;
        if (i < g.n && a.l[e] != LVL_EXACT) {
          const unsigned long long key = arm_key(a.S[e], a.l[e], (uint32_t)i, g);
          const double dh = dhat_of(a.S[e], a.l[e], g.d);
          const double al = alpha_of(a.l[e], g.alpha);
          bool blk;
          if (key <= st.thr_k)
            blk = __dadd_rn(dh, al) > st.B;
          else if (key <= st.thr_kh)
            blk = al > st.a_d2;
          else
            blk = __dsub_rn(dh, al) < st.A;
          if (blk) {
            if ((2u << a.l[e]) >= (unsigned)g.d) {
              act = ACT_EXACT;
              myexact += 1;
            } else {
              act = (uint8_t)(a.l[e] + 1);
              mydraw += 1ull << a.l[e];
            }
          }
        }
        actw |= (uint32_t)act << (8 * e);
      }
    }
    *reinterpret_cast<uint32_t *>(g.act + (size_t)qi * g.npad + i0) = actw;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint8_t act = (uint8_t)(actw >> (8 * e));
    const unsigned slot = act == 0 ? NONE : (act == ACT_EXACT ? (unsigned)MAX_LEVELS : act - 1u);
    hist_add(scnt, slot);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mydraw += __shfl_xor_sync(FULL, mydraw, o);
    myexact += __shfl_xor_sync(FULL, myexact, o);
  }
  if (lane_id() == 0 && (mydraw | myexact)) {
    atomicAdd(&sdraw, mydraw);
    atomicAdd(&sexact, myexact);
  }
  __syncthreads();
  if (threadIdx.x < NSLOT && scnt[threadIdx.x]) atomicAdd(&g.ctl->cnt[threadIdx.x], scnt[threadIdx.x]);
  if (threadIdx.x == 0 && (sdraw | sexact)) {
    atomicAdd(reinterpret_cast<unsigned long long *>(&g.qs[qi].draws), sdraw);
    atomicAdd(reinterpret_cast<unsigned long long *>(&g.qs[qi].nexact), sexact);
  }
}

// Pairs per warp-chunk for level c (2^c draws = ceil(2^c / 4) Philox blocks).
__host__ __device__ __forceinline__ unsigned nblk_of(int c) { return c < 2 ? 1u : (1u << (c - 2)); }

__global__ void k_plan(RoundCtl *ctl) {
  if (threadIdx.x != 0) return;
  unsigned off = 0;
  unsigned long long ch = 0, adv = 0;
  for (int s = 0; s < NSLOT; ++s) {
    const unsigned c = ctl->cnt[s];
    ctl->off[s] = off;
    ctl->chunk_off[s] = ch;
    ctl->cursor[s] = 0;
    off += c;
    adv += c;
    if (s == MAX_LEVELS) {
      ch += c;  // one warp per exact pair
    } else {
      const unsigned nb = nblk_of(s);
      ch += nb <= 32 ? (c + (32 / nb) - 1) / (32 / nb) : c;
    }
  }
  ctl->off[NSLOT] = off;
  ctl->chunk_off[NSLOT] = ch;
  ctl->advanced += adv;
}

// a8: compaction of the action bytes into per-slot lists of (qi << ibits | i).
// blockIdx.x = query, so consecutive CTAs append the same point chunk of
// different queries (point-major list order, X-row locality in L2).
__global__ void __launch_bounds__(FIL_NT) k_scatter(Geom g) {
  const int qi = blockIdx.x;
  if (g.qs[qi].done) return;
  const int i0 = (blockIdx.y * FIL_NT + threadIdx.x) * 4;
  uint32_t actw = 0;
  if (i0 < g.n) actw = *reinterpret_cast<const uint32_t *>(g.act + (size_t)qi * g.npad + i0);
  const int lane = lane_id();
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint8_t act = (uint8_t)(actw >> (8 * e));
    const unsigned slot = act == 0 ? NONE : (act == ACT_EXACT ? (unsigned)MAX_LEVELS : act - 1u);
    const unsigned m = __match_any_sync(FULL, slot);
    if (slot == NONE) continue;
    const int leader = __ffs(m) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(&g.ctl->cursor[slot], (unsigned)__popc(m));
    base = __shfl_sync(m, base, leader);
    const unsigned r = __popc(m & ((1u << lane) - 1u));
    g.list[g.ctl->off[slot] + base + r] = ((uint32_t)qi << g.ibits) | (uint32_t)(i0 + e);
  }
}

// ---------------------------------------------------------------------------
// a3 + a4: advance every listed pair.  Grid-stride over warp-chunks.
constexpr int ADV_NT = 256;

// Sum of the squared differences of the draws u = 4*blk .. 4*blk+3 (< s) of
// pair (qi, i) at level b = c + 1 (T -> 2T, t = T + u).
__device__ __forceinline__ uint32_t draw_block(const Geom &g, uint32_t qi, uint32_t i, int c,
                                               uint32_t blk, uint32_t s) {
  const uint4 w = philox4x32_10(make_uint4(blk, i + g.id_offset, qi + g.qi0, (uint32_t)(c + 1)),
                                g.seed_lo, g.seed_hi);
  const uint8_t *xr = g.X + (size_t)i * g.pitch;
  const uint8_t *qr = g.Q + (size_t)qi * g.pitch;
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  uint32_t acc = 0;
  const uint32_t u0 = blk * 4;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (u0 + t < s) {
      const uint32_t j = coord_of(ws[t], (uint32_t)g.d);
      const int diff = (int)__ldg(xr + j) - (int)__ldg(qr + j);
      acc += (uint32_t)(diff * diff);
    }
  }
  return acc;
}

__device__ __forceinline__ uint32_t exact_row(const Geom &g, uint32_t qi, uint32_t i) {
  const uint4 *xr = reinterpret_cast<const uint4 *>(g.X + (size_t)i * g.pitch);
  const uint4 *qr = reinterpret_cast<const uint4 *>(g.Q + (size_t)qi * g.pitch);
  const int nv = (int)(g.pitch >> 4);
  uint32_t acc = 0;
  for (int v = lane_id(); v < nv; v += 32) {
    const uint4 a = __ldg(xr + v), b = __ldg(qr + v);
    uint32_t t;
    t = __vabsdiffu4(a.x, b.x); acc = __dp4a(t, t, acc);
    t = __vabsdiffu4(a.y, b.y); acc = __dp4a(t, t, acc);
    t = __vabsdiffu4(a.z, b.z); acc = __dp4a(t, t, acc);
    t = __vabsdiffu4(a.w, b.w); acc = __dp4a(t, t, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  return acc;
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
  const unsigned long long total = coff[NSLOT];
  const unsigned long long nwarps = (unsigned long long)gridDim.x * (ADV_NT / 32);
  const int lane = lane_id();
  const uint32_t imask = (1u << g.ibits) - 1u;
  int slot = 0;
  for (unsigned long long ch = (unsigned long long)blockIdx.x * (ADV_NT / 32) + (threadIdx.x >> 5);
       ch < total; ch += nwarps) {
    while (coff[slot + 1] <= ch) ++slot;  // chunks are visited in increasing order
    const unsigned long long rel = ch - coff[slot];
    if (slot == MAX_LEVELS) {
      const uint32_t code = g.list[soff[slot] + rel];
      const uint32_t qi = code >> g.ibits, i = code & imask;
      const uint32_t acc = exact_row(g, qi, i);
      if (lane == 0) {
        const size_t o = (size_t)qi * g.npad + i;
        g.S[o] = (int32_t)acc;
        g.lvl[o] = LVL_EXACT;
      }
      continue;
    }
    const int c = slot;
    const uint32_t s = 1u << c;
    const unsigned nb = nblk_of(c);
    if (nb <= 32) {
      const unsigned ppw = 32 / nb;
      const unsigned long long p = rel * ppw + lane / nb;
      const uint32_t blk = lane % nb;
      const bool valid = p < scnt[c];
      uint32_t code = 0, acc = 0;
      if (valid) {
        code = g.list[soff[c] + p];
        acc = draw_block(g, code >> g.ibits, code & imask, c, blk, s);
      }
      for (unsigned o = nb >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      if (valid && blk == 0) {
        const size_t o = (size_t)(code >> g.ibits) * g.npad + (code & imask);
        g.S[o] += (int32_t)acc;
        g.lvl[o] = (uint8_t)(c + 1);
      }
    } else {
      const uint32_t code = g.list[soff[c] + rel];
      const uint32_t qi = code >> g.ibits, i = code & imask;
      uint32_t acc = 0;
      for (uint32_t blk = lane; blk < nb; blk += 32) acc += draw_block(g, qi, i, c, blk, s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      if (lane == 0) {
        const size_t o = (size_t)qi * g.npad + i;
        g.S[o] += (int32_t)acc;
        g.lvl[o] = (uint8_t)(c + 1);
      }
    }
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
      const unsigned long long kk = arm_key(a.S[e], a.l[e], (uint32_t)i, g);
      if (kk <= st.thr_kh) {
        const unsigned p = atomicAdd(&cnt, 1u);
        if (p < (unsigned)kh) {
          key[p] = kk;
          sv[p] = a.S[e];
          iv[p] = i;
          lv[p] = a.l[e];
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
    if (o.dhat) o.dhat[oo] = dhat_of(sv[r], lv[r], g.d);
  }
  if (threadIdx.x == 0) {
    const size_t row = (size_t)(o.row0 + qi);
    if (o.draws) o.draws[row] = st.draws;
    if (o.evals) o.evals[row] = st.draws + (long long)g.d * st.nexact;
    if (o.rounds) o.rounds[row] = st.rounds;
  }
}

__global__ void k_counts(Geom g, OutPtrs o) {
  const int qi = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const size_t src = (size_t)qi * g.npad + i;
  const size_t dst = (size_t)(o.row0 + qi) * g.n + i;
  const uint8_t l = g.lvl[src];
  if (o.counts) o.counts[dst] = (l == LVL_EXACT) ? g.d : (int32_t)(1u << l);
  if (o.sums) o.sums[dst] = (int64_t)(uint32_t)g.S[src];
}

// ---------------------------------------------------------------------------
// Launch wrappers.
static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

cudaError_t launch_init(const Geom &g, cudaStream_t s) {
  k_init<<<dim3(cdiv(g.npad, 256), g.q), 256, 0, s>>>(g);
  k_init_qstate<<<cdiv(g.q, 128), 128, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_select(const Geom &g, int nbits, cudaStream_t s) {
  k_select<<<g.q, SEL_NT, 0, s>>>(g, nbits);
  return cudaGetLastError();
}

cudaError_t launch_filter(const Geom &g, cudaStream_t s) {
  k_filter<<<dim3(cdiv(g.npad, FIL_NT * 4), g.q), FIL_NT, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_compact(const Geom &g, cudaStream_t s) {
  k_plan<<<1, 32, 0, s>>>(g.ctl);
  k_scatter<<<dim3(g.q, cdiv(g.npad, FIL_NT * 4)), FIL_NT, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_advance(const Geom &g, int num_sms, cudaStream_t s) {
  k_advance<<<num_sms * 8, ADV_NT, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_output(const Geom &g, const OutPtrs &o, cudaStream_t s) {
  const int kh = g.k + g.h;
  const size_t smem = (size_t)kh * (8 + 4 + 4 + 1);
  k_output<<<g.q, OUT_NT, smem, s>>>(g, o);
  if (o.counts || o.sums) k_counts<<<dim3(cdiv(g.n, 256), g.q), 256, 0, s>>>(g, o);
  return cudaGetLastError();
}

int output_max_kh() { return OUT_MAXKH; }

}  // namespace aknn
