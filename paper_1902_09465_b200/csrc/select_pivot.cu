// select_pivot.cu -- the per-round rank split in ONE pass over the arm state
// (P:144-146 ranks, P:148-153 d1/d2, Eq. 5).
//
// Only the k+h smallest composite keys matter (the split C | M | F).  Per undecided
// query (one CTA):
//   1. sample SS keys at fixed strided positions and take the (r_s+1)-th smallest as a
//      pivot tau (r_s+1 = twice the expected sample rank of k+h, plus 4), found by
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

constexpr int PIV_NT = 512;
constexpr unsigned PIV_CAP = 8192;    // buffer keys (64 KB of dynamic shared memory)
constexpr unsigned PIV_BRUTE = 1536;  // buffers up to this size are ranked by counting

__host__ __device__ __forceinline__ unsigned piv_sample_size(int n) {
  unsigned ss = 1024;  // >= n / 16 samples (capped): tau's rank, hence the buffer, stays small
  while (ss < PIV_CAP && (int)(ss * 16u) < n) ss <<= 1;
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
};

// Fills buf[0..cnt) with every key <= tau (unsorted) and rank[t] = the rank of buf[t]
// among them (0-based; keys are unique), and returns the arg-min of L over the arms
// with key > tau.  Returns false (and the caller falls back) when fewer than `need`
// keys are <= tau or the buffer overflows.
__device__ bool pivot_pass(const Geom &g, int qi, unsigned need, unsigned long long *buf, unsigned *rank,
                           unsigned *cnt_out, RecBest *outside, RecBest *wsm) {
  __shared__ unsigned cnt;
  __shared__ unsigned long long tau_s;
  __shared__ unsigned long long wmin[PIV_NT / 32];
  __shared__ double wbnd[PIV_NT / 32];
  __shared__ double bound0_s;  // min L over the sampled arms with key > tau (screen start)
  __shared__ __align__(16) PivLevel lvt[MAX_LEVELS + 1];
  const int tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
  const int n = g.n;
  if (n > (int)PIV_CAP) {
    // tau = the (rs+1)-th smallest of ss strided sample keys, rs+1 about twice the
    // expected sample rank of need, plus 8: found by rs+1 rounds of block arg-min
    const unsigned ss = piv_sample_size(n);
    const unsigned per = ss / PIV_NT;  // <= 16 samples per thread
    unsigned long long mine[PIV_CAP / PIV_NT];
#pragma unroll
    for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) {
      mine[u] = KEY_INVALID;
      if (u < per) {
        const unsigned j = tid + u * PIV_NT;
        const int i = (int)(((unsigned long long)j * (unsigned)n) / ss);
        const size_t o = (size_t)qi * g.npad + i;
        mine[u] = arm_key(g.S[o], g.lvl[o], (uint32_t)i, g);
      }
    }
    const unsigned expect = (unsigned)(((unsigned long long)need * ss + n - 1) / n);
    const unsigned rounds = 2 * expect + 4;
    unsigned long long t = KEY_INVALID;
    // the thread's smallest remaining sample; only the owner of a round's minimum
    // rescans its registers (keys are unique), so a round costs one warp reduction
    unsigned long long head = KEY_INVALID;
#pragma unroll
    for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) head = mine[u] < head ? mine[u] : head;
    for (unsigned r = 0; r < rounds; ++r) {
      unsigned long long m = head;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(FULL, m, o);
        m = y < m ? y : m;
      }
      if (lane == 0) wmin[warp] = m;
      __syncthreads();
      m = wmin[0];
#pragma unroll
      for (int w = 1; w < PIV_NT / 32; ++w) m = wmin[w] < m ? wmin[w] : m;
      t = m;
      if (head == m) {  // unique keys: exactly one owner
        head = KEY_INVALID;
#pragma unroll
        for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) {
          if (mine[u] == m) mine[u] = KEY_INVALID;
          head = mine[u] < head ? mine[u] : head;
        }
      }
      __syncthreads();
    }
    if (tid == 0) tau_s = t;
    // the samples left in `mine` have keys > tau: they are arms outside the buffer, so
    // their minimum L bounds the outside arg-min from above -- the screen starts there
    // instead of at +inf (which sent the whole first stretch of arms to fp64)
    double b = 1.0e300;
#pragma unroll
    for (unsigned u = 0; u < PIV_CAP / PIV_NT; ++u) {
      if (u < per && mine[u] != KEY_INVALID) {
        const unsigned j = tid + u * PIV_NT;
        const int i = (int)(((unsigned long long)j * (unsigned)n) / ss);
        const size_t o = (size_t)qi * g.npad + i;
        b = fmin(b, lower_of(g.S[o], g.lvl[o], g.d, g.alpha, g.growth));
      }
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
  if (tid <= MAX_LEVELS) {
    const bool ex = tid == MAX_LEVELS;  // slot MAX_LEVELS: exact arms (T = d, alpha = 0)
    const bool live = !ex && tid <= g.cmax;
    const double T = ex ? (double)g.d : (double)lvl_count((uint32_t)tid, g.growth);
    const unsigned long long mul = ex ? g.Ld : (live ? lvl_mul((uint32_t)tid, g.L, g.L3, g.growth) : 1ull),
                             Kt = tau >> g.kbits;
    const unsigned long long qt = Kt / mul, rt = Kt % mul, lt = qt + (rt != 0);
    const float alf = live ? (float)g.alpha[lvl_count((uint32_t)tid, g.growth)] : 0.f;
    const float eps = (alf + 2.f) * 9.5367431640625e-07f;  // 2^-20
    PivLevel v;
    v.lt = lt > 0x7fffffffull ? 0x7fffffff : (int32_t)lt;
    v.eq = (rt == 0 && qt <= 0x7fffffffull) ? (int32_t)qt : -1;
    v.invT = (float)(1.0 / (T * 65025.0));
    v.nae = -__fadd_ru(alf, eps);
    lvt[tid] = v;
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
      if (i0 < n) {
        sg[u] = *reinterpret_cast<const int4 *>(Srow + i0);
        lg[u] = *reinterpret_cast<const uint32_t *>(Lrow + i0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i0 = b0 + u * PIV_NT * 4;
      const int32_t Sv[4] = {sg[u].x, sg[u].y, sg[u].z, sg[u].w};
      const int ne = min(4, n - i0);  // arms of this group (<= 0 past the end)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = i0 + e;
        if (e >= ne) break;
        const uint32_t l = (lg[u] >> (8 * e)) & 0xFFu;
        const int32_t S = Sv[e];
        // the level's 16-byte entry (shared-window address hoisted out of the loop)
        uint4 vv;
        asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
            : "=r"(vv.x), "=r"(vv.y), "=r"(vv.z), "=r"(vv.w)
            : "r"(lvt_s + 16u * ((l & LVL_EXACT) ? (uint32_t)MAX_LEVELS : l)));
        PivLevel v;
        v.lt = (int32_t)vv.x;
        v.eq = (int32_t)vv.y;
        v.invT = __uint_as_float(vv.z);
        v.nae = __uint_as_float(vv.w);
        const uint32_t gid = (uint32_t)i + gid0;
        if (S < v.lt || (S == v.eq && gid <= idt)) {  // key <= tau
          const unsigned p = atomicAdd(&cnt, 1u);
          if (p < PIV_CAP) buf[p] = arm_key(S, (uint8_t)l, (uint32_t)i, g);
        } else if (!(__fmaf_rn((float)S, v.invT, v.nae) > boundf)) {  // could be the arg-min
          // at the level of the thread's best so far, L = fl(fl(S / (65025 T)) - alpha) is
          // strictly increasing in S (distinct S give estimates many ulps apart, reading R9),
          // so the integer order (S, id) decides and the fp64 division runs only for an
          // improvement; in lock-step rounds nearly every candidate is at that level
          if (bl.gid != 0xffffffffu && (uint8_t)l == bl.lvl) {
            if (S < bl.S || (S == bl.S && gid < bl.gid))
              bl = RecBest{lower_of(S, (uint8_t)l, g.d, g.alpha, g.growth), gid, S, (uint8_t)l};
          } else {
            const RecBest c{lower_of(S, (uint8_t)l, g.d, g.alpha, g.growth), gid, S, (uint8_t)l};
            if (better_min(c, bl)) bl = c;
          }
        }
      }
    }
    double wb = bl.v;  // share the warp's best: an arm above it cannot be the arg-min
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wb = fmin(wb, __shfl_xor_sync(FULL, wb, o));
    boundf = fminf(boundf, __double2float_ru(wb));
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
__global__ void __launch_bounds__(PIV_NT, 2) k_select_pivot(Geom g) {
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
  if (g.force_radix || !pivot_pass(g, qi, kh, pbuf, prank, &cnt, &outside, wsm)) {
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
__global__ void __launch_bounds__(PIV_NT, 2) k_select_local_pivot(Geom g) {
  extern __shared__ unsigned long long pbuf[];
  unsigned *prank = reinterpret_cast<unsigned *>(pbuf + PIV_CAP);
  __shared__ RecBest wsm[PIV_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
  const unsigned kh = (unsigned)(g.k + g.h);
  unsigned cnt;
  RecBest outside;
  if (g.force_radix || !pivot_pass(g, qi, kh, pbuf, prank, &cnt, &outside, wsm)) {
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

size_t pivot_smem_bytes() { return (size_t)PIV_CAP * (sizeof(unsigned long long) + sizeof(unsigned)); }

cudaError_t launch_select_pivot(const Geom &g, cudaStream_t s) {
  const size_t smem = pivot_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(k_select_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_select_pivot<<<g.q, PIV_NT, smem, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_select_local_pivot(const Geom &g, cudaStream_t s) {
  const size_t smem = pivot_smem_bytes();
  cudaError_t e =
      cudaFuncSetAttribute(k_select_local_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_select_local_pivot<<<g.q, PIV_NT, smem, s>>>(g);
  return cudaGetLastError();
}

}  // namespace aknn
