// select_pivot.cu -- the per-round rank split in ONE pass over the arm state
// (P:144-146 ranks, P:148-153 d1/d2, Eq. 5).
//
// Only the k+h smallest composite keys matter (the split C | M | F).  Per undecided
// query (one CTA):
//   1. sample SS keys (evenly spaced runs of 8 consecutive arms) and take the (r_s+1)-th smallest as a
//      pivot tau (r_s+1 = twice the expected sample rank of k+h, plus 10), found by
//      r_s+1 rounds of block-wide arg-min over the samples held in registers;
//   2. ONE pass over the n arms: keys <= tau go to a shared-memory buffer, and every
//      other arm feeds a running arg-min of L = d_hat - alpha (ties: smaller id),
//      screened in fp32 so that only arms that can beat the running minimum pay the
//      fp64 division;
//   3. rank the buffer (by counting when small, else bitonic sort): ranks k and k+h
//      are exact (keys are unique), A / d1 come from the k smallest, B / d2 =
//      min(outside arg-min, buffer entries ranked > k+h), then Eq. (5).
// If the buffer holds fewer than k+h keys or overflows (tau too small or too
// large; rare), the query is flagged and the multi-pass radix select (k_select)
// decides it instead.  Either way the result is the exact order statistics, so
// the outputs are identical.
#include "internal.cuh"
#include "launch.h"
#include "round_common.cuh"
#include "select.cuh"


namespace aknn {

constexpr unsigned PIV_CAP_MAX = 8192;  // buffer keys (64 KB of dynamic shared memory + ranks)
constexpr unsigned PIV_BRUTE = 384;  // buffers up to this size are ranked by counting (O(c^2));
                                     // larger ones by a bitonic sort (O(c log^2 c), a barrier per stage)

__host__ __device__ __forceinline__ unsigned piv_sample_size(int n, unsigned cap) {
  unsigned ss = 1024;  // >= n / 16 samples (capped): tau's rank, hence the buffer, stays small
  while (ss < cap && (int)(ss * 16u) < n) ss <<= 1;
  return ss;
}

__device__ void bitonic_keys(unsigned long long *buf, unsigned P) {
  for (unsigned k = 2; k <= P; k <<= 1)
    for (unsigned j = k >> 1; j > 0; j >>= 1) {
      for (unsigned idx = threadIdx.x; idx < P; idx += blockDim.x) {
        const unsigned ixj = idx ^ j;
        if (ixj > idx) {
          const unsigned long long a = buf[idx], b = buf[ixj];
          if ((a > b) == ((idx & k) == 0)) {
            buf[idx] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
}

// Per-level table of the streaming pass (one 16-byte shared-memory load per arm):
//   key <= tau   as integer tests on S (no 64-bit key per arm): with Kt = tau >> kbits,
//                S * mul_c < Kt  <=>  S < ceil(Kt / mul_c) = lt, and S * mul_c == Kt <=>
//                S == Kt / mul_c = eq when mul_c divides Kt (else eq = -1), in which case
//                the id decides (gid <= tau's id);
//   fp32 screen  for the arg-min of L = d_hat - alpha over the arms outside the buffer:
//                r = fma(S, inv(65025 T), -(alpha_c + eps_c)) in fp32 differs from
//                S / (65025 T) - alpha - eps_c by less than (alpha_c + 2) 2^-23 (d_hat <= 1:
//                every sample is <= 1; each fp32 rounding is a relative 2^-24), and
//                eps_c = (alpha_c + 2) 2^-20 exceeds that, so r > bound (rounded up to
//                fp32) proves L > bound: such an arm cannot be the arg-min and skips the
//                fp64 division; the rest are decided in fp64 as before.
struct PivLevel {
  int32_t lt, eq;  // key <= tau  <=>  S < lt  ||  (S == eq && gid <= id(tau))
  float invT, nae;  // 1 / (65025 T) and -(alpha + eps) in fp32
  double Tm;        // 65025 T (the fast screen's threshold estimate)
  double pad;
};

// The fast screen of the streaming pass for arms at level byte lc: every arm with
// S > piv_hi(...) is neither a key <= tau (S >= lt and S != eq) nor through the fp32
// screen (f(S) = fma((float)S, invT, nae) > boundf).  f is non-decreasing in S, so
// checking f(sthr + 1) > boundf once proves it for every S > sthr; the fp64 estimate
// of the crossing only has to be close (a bad estimate fails the check and the group
// takes the per-arm path -- slower, never wrong).
__device__ __forceinline__ int32_t piv_hi(uint32_t lvt_s, uint32_t lc, float boundf) {
  const uint32_t a = lvt_s + 32u * ((lc & LVL_EXACT) ? (uint32_t)MAX_LEVELS : lc);
  uint4 vv;
  double Tm;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(vv.x), "=r"(vv.y), "=r"(vv.z), "=r"(vv.w) : "r"(a));
  asm("ld.shared.f64 %0, [%1];" : "=d"(Tm) : "r"(a + 16u));
  const float invT = __uint_as_float(vv.z), nae = __uint_as_float(vv.w);
  int32_t sthr = 0x7fffffff;
  if (!(nae > boundf)) {  // else f(0) = nae > boundf: no arm passes (sthr = -1 below)
    const double est = ((double)boundf - (double)nae) * Tm;
    if (est < 1.0e9) {
      const int32_t e = (int32_t)est;
      const int32_t cand = e + 4 + (e >> 20);
      if (__fmaf_rn((float)(cand + 1), invT, nae) > boundf) sthr = cand;
    }
  } else {
    sthr = -1;
  }
  return max(max((int32_t)vv.x - 1, (int32_t)vv.y), sthr);
}

// Fills buf[0..cnt) with every key <= tau (unsorted) and rank[t] = the rank of buf[t]
// among them (0-based; keys are unique), and returns the arg-min of L over the arms
// with key > tau.  Returns false (and the caller falls back) when fewer than `need`
// keys are <= tau or the buffer overflows.
template <int PIV_NT, unsigned PIV_CAP>
__device__ bool pivot_pass(const Geom &g, int qi, unsigned need, unsigned long long *buf, unsigned *rank,
                           unsigned *cnt_out, RecBest *outside, RecBest *wsm) {
  __shared__ unsigned cnt;
  __shared__ unsigned long long tau_s;
  __shared__ unsigned long long wmin[PIV_NT / 32];
  __shared__ double wbnd[PIV_NT / 32];
  __shared__ double bound0_s;  // min L over the sampled arms with key > tau (screen start)
  __shared__ __align__(32) PivLevel lvt[MAX_LEVELS + 1];
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const int n = g.n;
  // the per-level table, fp32 screen part first (the sample phase uses it)
  if (tid <= MAX_LEVELS) {
    const bool ex = tid == MAX_LEVELS;  // slot MAX_LEVELS: exact arms (T = d, alpha = 0)
    const bool live = !ex && tid <= g.cmax;
    const double T = ex ? (double)g.d : (double)lvl_count((uint32_t)tid, g.growth);
    const float alf = live ? (float)g.alpha[lvl_count((uint32_t)tid, g.growth)] : 0.f;
    const float eps = (alf + 2.f) * 9.5367431640625e-07f;  // 2^-20
    PivLevel v;
    v.lt = 0;
    v.eq = -1;
    v.invT = (float)(1.0 / (T * 65025.0));
    v.nae = -__fadd_ru(alf, eps);
    v.Tm = T * 65025.0;
    v.pad = 0.0;
    lvt[tid] = v;
  }
  if (tid == 0) tau_s = KEY_INVALID;
  __syncthreads();
  if (n > (int)PIV_CAP) {
    // tau = the rounds-th smallest of ss sample keys, rounds about twice the expected
    // sample rank of need, plus 10.  The samples are ss / 8 evenly spaced runs of 8
    // consecutive arms (one 32-byte sector of S): single strided arms cost a sector of S
    // and of the level bytes each, and those sectors did not survive in L2 until the
    // streaming pass (ncu C2: 604 MB of DRAM reads for 300 MB of arm state)
    const unsigned ss = piv_sample_size(n, PIV_CAP);
    const unsigned per = ss / PIV_NT;  // <= 16 samples per thread
    const unsigned nruns = ss / 8u;
    unsigned long long mine[PIV_CAP / PIV_NT];
#pragma unroll
    for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) {
      mine[u] = KEY_INVALID;
      if (u < per) {
        const unsigned j = tid + u * PIV_NT;
        const int i = (int)((((unsigned long long)(j >> 3) * (unsigned)n) / nruns) & ~7ull) + (int)(j & 7u);
        if (i < n) {
          const size_t o = (size_t)qi * g.npad + i;
          mine[u] = arm_key(g.S[o], g.lvl[o], (uint32_t)i, g);
        }
      }
    }
    // keys <= tau ~ (n / ss) Gamma(rounds): with rounds = 2 expect + 10 the buffer holds
    // fewer than `need` keys with probability < 1e-9 at expect = 1 (C4: 0.82 sample ranks;
    // 2 expect + 4 failed about once per 5,000 query-rounds, and the radix fallback of one
    // query costs five times a whole pivot pass)
    const unsigned expect = (unsigned)(((unsigned long long)need * ss + n - 1) / n);
    const unsigned rounds = 2 * expect + 10;
    // the thread's smallest remaining sample; only the owner of a round's minimum
    // rescans its registers (keys are unique)
    unsigned long long head = KEY_INVALID;
#pragma unroll
    for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) head = mine[u] < head ? mine[u] : head;
    auto pop_min = [&](unsigned long long m) {
      if (head == m) {  // unique keys: exactly one owner
        head = KEY_INVALID;
#pragma unroll
        for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) {
          if (mine[u] == m) mine[u] = KEY_INVALID;
          head = mine[u] < head ? mine[u] : head;
        }
      }
    };
    auto warp_min = [&](unsigned long long m) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(FULL, m, o);
        m = y < m ? y : m;
      }
      return m;
    };
    {  // rounds of block arg-min (a per-warp pre-selection measured slower on C2)
      unsigned long long t = KEY_INVALID;
      for (unsigned r = 0; r < rounds; ++r) {
        unsigned long long m = warp_min(head);
        if (lane == 0) wmin[warp] = m;
        __syncthreads();
        m = wmin[0];
#pragma unroll
        for (int w = 1; w < PIV_NT / 32; ++w) m = wmin[w] < m ? wmin[w] : m;
        t = m;
        pop_min(m);
        __syncthreads();
      }
      if (tid == 0) tau_s = t;
    }
    __syncthreads();
    // samples with keys > tau are arms outside the buffer, so the L of any of them bounds
    // the outside arg-min from above -- the screen starts there instead of at +inf
    // (which sent the whole first stretch of arms to fp64).  The rounds popped exactly
    // the samples with keys <= tau, so `head` is the thread's smallest outside sample:
    // one exact fp64 L per thread (at one level, the smallest key is the smallest L).
    double b = 1.0e300;
    if (head != KEY_INVALID) {
      const uint32_t i = (uint32_t)(head & ((1ull << g.kbits) - 1ull)) - g.id_offset;
      const size_t o = (size_t)qi * g.npad + i;
      b = lower_of(g.S[o], g.lvl[o], g.d, g.alpha, g.growth);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) b = fmin(b, __shfl_xor_sync(FULL, b, o));
    if (lane == 0) wbnd[warp] = b;
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < PIV_NT / 32; ++w) b = fmin(b, wbnd[w]);
      bound0_s = fmin(b, wbnd[0]);
    }
  } else if (tid == 0) {
    tau_s = KEY_INVALID - 1;  // every arm
    bound0_s = 1.0e300;
  }
  if (tid == 0) cnt = 0;
  __syncthreads();
  const unsigned long long tau = tau_s;
  if (tid <= MAX_LEVELS) {  // the integer key <= tau tests
    const bool ex = tid == MAX_LEVELS;
    const bool live = !ex && tid <= g.cmax;
    const unsigned long long mul = ex ? g.Ld : (live ? lvl_mul((uint32_t)tid, g.L, g.L3, g.growth) : 1ull),
                             Kt = tau >> g.kbits;
    const unsigned long long qt = Kt / mul, rt = Kt % mul, lt = qt + (rt != 0);
    lvt[tid].lt = lt > 0x7fffffffull ? 0x7fffffff : (int32_t)lt;
    lvt[tid].eq = (rt == 0 && qt <= 0x7fffffffull) ? (int32_t)qt : -1;
  }
  __syncthreads();
  const uint32_t idt = (uint32_t)(tau & ((1ull << g.kbits) - 1ull));
  const uint32_t lvt_s = (uint32_t)__cvta_generic_to_shared(lvt);
  const uint32_t gid0 = g.id_offset;
  const int32_t *Srow = g.S + (size_t)qi * g.npad;
  const uint8_t *Lrow = g.lvl + (size_t)qi * g.npad;
  RecBest bl{1.0e300, 0xffffffffu, 0, 0};
  float boundf = __double2float_ru(bound0_s);  // min L known so far, rounded up to fp32
  constexpr int U = 4;  // arm groups in flight per thread (the pass is load-latency bound)
  for (int wb0 = (tid - lane) * 4; wb0 < n; wb0 += PIV_NT * 4 * U) {  // warp-uniform trips
    const int b0 = wb0 + lane * 4;
    int4 sg[U];
    uint32_t lg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i0 = b0 + u * PIV_NT * 4;
      sg[u] = make_int4(0, 0, 0, 0);
      lg[u] = 0;
      if (i0 < n) {
        sg[u] = *reinterpret_cast<const int4 *>(Srow + i0);
        lg[u] = *reinterpret_cast<const uint32_t *>(Lrow + i0);
      }
    }
    // fast screen: a full group of 4 arms at the thread's common level whose S all
    // exceed piv_hi is decided (outside, not the arg-min) by 5 integer compares; in
    // lock-step rounds that is nearly every group
    const uint32_t lc = lg[0] & 0xFFu;
    const int32_t hi = piv_hi(lvt_s, lc, boundf);
    const uint32_t l4 = lc * 0x01010101u;
    uint32_t slow = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i0 = b0 + u * PIV_NT * 4;
      const bool quiet = i0 + 4 <= n && lg[u] == l4 && min(min(sg[u].x, sg[u].y), min(sg[u].z, sg[u].w)) > hi;
      slow |= (uint32_t)(!quiet && i0 < n) << u;
    }
    if (slow) {
      // per-arm classification of the other groups: `inb` key <= tau, `cand` outside
      // and through the fp32 screen (bit u*4+e); their handling (64-bit keys, the fp64
      // division) runs below from one call site each, re-reading the arm from L1
      uint32_t inb = 0, cand = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!((slow >> u) & 1u)) continue;
        const int i0 = b0 + u * PIV_NT * 4;
        const int32_t Sv[4] = {sg[u].x, sg[u].y, sg[u].z, sg[u].w};
        const int ne = min(4, n - i0);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e < ne) {
            const uint32_t l = (lg[u] >> (8 * e)) & 0xFFu;
            const int32_t S = Sv[e];
            uint4 vv;
            asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                : "=r"(vv.x), "=r"(vv.y), "=r"(vv.z), "=r"(vv.w)
                : "r"(lvt_s + 32u * ((l & LVL_EXACT) ? (uint32_t)MAX_LEVELS : l)));
            const uint32_t gid = (uint32_t)(i0 + e) + gid0;
            const bool in = S < (int32_t)vv.x || (S == (int32_t)vv.y && gid <= idt);  // key <= tau
            const bool pass = !(__fmaf_rn((float)S, __uint_as_float(vv.z), __uint_as_float(vv.w)) > boundf);
            inb |= (uint32_t)in << (u * 4 + e);
            cand |= (uint32_t)(!in && pass) << (u * 4 + e);
          }
        }
      }
      while (inb) {
        const int j = __ffs(inb) - 1;
        inb &= inb - 1;
        const int i = b0 + (j >> 2) * PIV_NT * 4 + (j & 3);
        const unsigned p = atomicAdd(&cnt, 1u);
        if (p < PIV_CAP) buf[p] = arm_key(Srow[i], Lrow[i], (uint32_t)i, g);
      }
      while (cand) {  // could be the arg-min of L
        const int j = __ffs(cand) - 1;
        cand &= cand - 1;
        const int i = b0 + (j >> 2) * PIV_NT * 4 + (j & 3);
        const int32_t S = Srow[i];
        const uint8_t l = Lrow[i];
        const uint32_t gid = (uint32_t)i + gid0;
        // at the level of the thread's best so far, L = fl(fl(S / (65025 T)) - alpha) is
        // strictly increasing in S (distinct S give estimates many ulps apart, reading R9),
        // so the integer order (S, id) decides and the fp64 division runs only for an
        // improvement
        const bool same = bl.gid != 0xffffffffu && l == bl.lvl;
        if (same && !(S < bl.S || (S == bl.S && gid < bl.gid))) continue;
        const RecBest c{lower_of(S, l, g.d, g.alpha, g.growth), gid, S, l};
        if (same || better_min(c, bl)) bl = c;
      }
    }
    // share the warp's best: an arm above it cannot be the arg-min (fp32, rounded up:
    // the minimum of the rounded-up values is the rounded-up minimum)
    float wb = __double2float_ru(bl.v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wb = fminf(wb, __shfl_xor_sync(FULL, wb, o));
    boundf = fminf(boundf, wb);
  }
  __syncthreads();
  const unsigned c = cnt;
  *outside = block_best<false>(bl, wsm);
  *cnt_out = c;
  if (c < need || c > PIV_CAP) return false;
  if (c <= PIV_BRUTE) {
    for (unsigned t = tid; t < c; t += PIV_NT) {  // rank by counting (no sync stages)
      const unsigned long long k = buf[t];
      unsigned r = 0;
      for (unsigned j = 0; j < c; ++j) r += buf[j] < k;
      rank[t] = r;
    }
  } else {
    unsigned P = 2;
    while (P < c) P <<= 1;
    for (unsigned t = c + tid; t < P; t += PIV_NT) buf[t] = KEY_INVALID;
    __syncthreads();
    bitonic_keys(buf, P);
    for (unsigned t = tid; t < c; t += PIV_NT) rank[t] = t;
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ RecBest rec_of_key(const Geom &g, int qi, unsigned long long key, bool upper) {
  const uint32_t gid = (uint32_t)(key & ((1ull << g.kbits) - 1ull));
  const uint32_t i = gid - g.id_offset;
  const size_t o = (size_t)qi * g.npad + i;
  const int32_t S = g.S[o];
  const uint8_t l = g.lvl[o];
  return RecBest{upper ? upper_of(S, l, g.d, g.alpha, g.growth) : lower_of(S, l, g.d, g.alpha, g.growth), gid, S, l};
}

// Unsharded rank split + bounds + Eq. (5) (same contract as k_select).
template <int PIV_NT, unsigned PIV_CAP>
__global__ void __launch_bounds__(PIV_NT, 1024 / PIV_NT) k_select_pivot(Geom g) {
  extern __shared__ unsigned long long pbuf[];
  unsigned *prank = reinterpret_cast<unsigned *>(pbuf + PIV_CAP);
  __shared__ RecBest wsm[PIV_NT / 32];
  __shared__ unsigned long long sthr[2];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
  const unsigned k = (unsigned)g.k, kh = (unsigned)(g.k + g.h);
  unsigned cnt;
  RecBest outside;
  if (g.force_radix || !pivot_pass<PIV_NT, PIV_CAP>(g, qi, kh, pbuf, prank, &cnt, &outside, wsm)) {
    if (threadIdx.x == 0) st->fallback = 1;
    return;
  }
  RecBest bu{-1.0e300, 0xffffffffu, 0, 0}, bl = outside;
  for (unsigned t = threadIdx.x; t < cnt; t += PIV_NT) {
    const unsigned r = prank[t];
    if (r == k - 1) sthr[0] = pbuf[t];
    if (r == kh - 1) sthr[1] = pbuf[t];
    if (r < k) {
      const RecBest c = rec_of_key(g, qi, pbuf[t], true);
      if (better_max(c, bu)) bu = c;
    } else if (r >= kh) {
      const RecBest c = rec_of_key(g, qi, pbuf[t], false);
      if (better_min(c, bl)) bl = c;
    }
  }
  bu = block_best<true>(bu, wsm);
  bl = block_best<false>(bl, wsm);
  if (threadIdx.x == 0) {
    st->fallback = 0;
    st->thr_k = sthr[0];
    st->thr_kh = sthr[1];
    st->A = bu.v;
    st->B = bl.v;
    st->d1 = (int)(bu.gid - g.id_offset);
    st->d2 = (int)(bl.gid - g.id_offset);
    st->a_d2 = alpha_of(bl.lvl, g.alpha, g.growth);
    st->rounds += 1;
    const int stop = bu.v <= bl.v;  // Eq. (5), "<=" as written
    st->done = stop;
    if (!stop) atomicAdd(&g.ctl->n_active, 1u);
  }
}

// Sharded local summary (same contract as k_select_local): the local top-(k+h)
// records and the remainder's minimum-L record.
template <int PIV_NT, unsigned PIV_CAP>
__global__ void __launch_bounds__(PIV_NT, 1024 / PIV_NT) k_select_local_pivot(Geom g) {
  extern __shared__ unsigned long long pbuf[];
  unsigned *prank = reinterpret_cast<unsigned *>(pbuf + PIV_CAP);
  __shared__ RecBest wsm[PIV_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
  const unsigned kh = (unsigned)(g.k + g.h);
  unsigned cnt;
  RecBest outside;
  if (g.force_radix || !pivot_pass<PIV_NT, PIV_CAP>(g, qi, kh, pbuf, prank, &cnt, &outside, wsm)) {
    if (threadIdx.x == 0) st->fallback = 1;
    return;
  }
  ShardRec *out = g.send + (size_t)qi * (kh + 1);
  RecBest bl = outside;
  for (unsigned t = threadIdx.x; t < cnt; t += PIV_NT) {
    const unsigned long long key = pbuf[t];
    const unsigned r = prank[t];
    const uint32_t i = (uint32_t)(key & ((1ull << g.kbits) - 1ull)) - g.id_offset;
    const size_t o = (size_t)qi * g.npad + i;
    if (r < kh) {  // the local top-(k+h) in rank order
      ShardRec rr;
      rr.key = key;
      rr.S = g.S[o];
      rr.lvl = g.lvl[o];
      rr.pad[0] = rr.pad[1] = rr.pad[2] = 0;
      out[r] = rr;
    } else {
      const RecBest c = rec_of_key(g, qi, key, false);
      if (better_min(c, bl)) bl = c;
    }
  }
  bl = block_best<false>(bl, wsm);
  if (threadIdx.x == 0) {
    st->fallback = 0;
    ShardRec rr;
    rr.S = bl.S;
    rr.lvl = bl.lvl;
    rr.key = arm_key(bl.S, bl.lvl, bl.gid - g.id_offset, g);
    rr.pad[0] = rr.pad[1] = rr.pad[2] = 0;
    out[kh] = rr;
  }
}

static size_t pivot_smem_bytes(unsigned cap) { return (size_t)cap * (sizeof(unsigned long long) + sizeof(unsigned)); }

// One CTA per query: 512 threads (two CTAs per SM); with at most one query per SM
// (C4: q = 128) 1,024 threads, so that each SM has twice the arm loads in flight (the
// pass is load-latency bound there: ncu long-scoreboard stalls); for short rows (n <=
// 65,536, C2) 256 threads with a 4,096-key buffer, four CTAs per SM, so the per-query
// fixed phases (samples, arg-min rounds, ranking) of different queries overlap.
template <class K256, class K512, class K1024>
static cudaError_t launch_piv(const Geom &g, cudaStream_t s, K256 k256, K512 k512, K1024 k1024) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nt = g.q <= sms ? 1024 : (g.n <= 65536 ? 256 : 512);
  const size_t smem = pivot_smem_bytes(nt == 256 ? 4096u : PIV_CAP_MAX);
  cudaError_t e = nt == 1024 ? cudaFuncSetAttribute(k1024, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                  : nt == 512 ? cudaFuncSetAttribute(k512, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                              : cudaFuncSetAttribute(k256, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (nt == 1024)
    k1024<<<g.q, 1024, smem, s>>>(g);
  else if (nt == 512)
    k512<<<g.q, 512, smem, s>>>(g);
  else
    k256<<<g.q, 256, smem, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_select_pivot(const Geom &g, cudaStream_t s) {
  return launch_piv(g, s, k_select_pivot<256, 4096>, k_select_pivot<512, PIV_CAP_MAX>,
                    k_select_pivot<1024, PIV_CAP_MAX>);
}

cudaError_t launch_select_local_pivot(const Geom &g, cudaStream_t s) {
  return launch_piv(g, s, k_select_local_pivot<256, 4096>, k_select_local_pivot<512, PIV_CAP_MAX>,
                    k_select_local_pivot<1024, PIV_CAP_MAX>);
}

}  // namespace aknn
