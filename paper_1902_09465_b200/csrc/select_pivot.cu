// select_pivot.cu -- the per-round rank split in ONE pass over the arm state
// (P:144-146 ranks, P:148-153 d1/d2, Eq. 5).
//
// Only the k+h smallest composite keys matter (the split C | M | F).  Per undecided
// query (one CTA):
//   1. sample SS keys at fixed strided positions, bitonic-sort them, and take the
//      sample key of rank r_s (about twice the expected rank of k+h in the sample,
//      plus 16) as a pivot tau;
//   2. ONE pass over the n arms: keys <= tau go to a shared-memory buffer, and every
//      other arm feeds a running arg-min of L = d_hat - alpha (ties: smaller id);
//   3. sort the buffer: ranks k and k+h are exact (keys are unique), A / d1 come
//      from the first k entries, B / d2 = min(outside arg-min, buffer entries
//      ranked > k+h), then Eq. (5).
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
constexpr unsigned PIV_CAP = 8192;  // buffer keys (64 KB of dynamic shared memory)

__host__ __device__ __forceinline__ unsigned piv_sample_size(int n) {
  unsigned ss = 1024;
  while (ss < PIV_CAP && (int)(ss * 64u) < n) ss <<= 1;
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

// Fills buf[0..cnt) (sorted ascending, cnt <= PIV_CAP) with every key <= tau and
// returns the arg-min of L over the arms with key > tau.  Returns false (and the
// caller falls back) when fewer than `need` keys are <= tau or the buffer overflows.
__device__ bool pivot_pass(const Geom &g, int qi, unsigned need, unsigned long long *buf,
                           unsigned *cnt_out, RecBest *outside, RecBest *wsm) {
  __shared__ unsigned cnt;
  __shared__ unsigned long long tau_s;
  const int tid = threadIdx.x;
  const int n = g.n;
  if (n > (int)PIV_CAP) {
    const unsigned ss = piv_sample_size(n);
    for (unsigned j = tid; j < ss; j += PIV_NT) {
      const int i = (int)(((unsigned long long)j * (unsigned)n) / ss);
      const size_t o = (size_t)qi * g.npad + i;
      buf[j] = arm_key(g.S[o], g.lvl[o], (uint32_t)i, g);
    }
    __syncthreads();
    bitonic_keys(buf, ss);
    if (tid == 0) {
      const unsigned expect = (unsigned)(((unsigned long long)need * ss + n - 1) / n);
      unsigned rs = 2 * expect + 16;
      if (rs > ss - 1) rs = ss - 1;
      tau_s = buf[rs];
    }
  } else if (tid == 0) {
    tau_s = KEY_INVALID - 1;  // every arm
  }
  if (tid == 0) cnt = 0;
  __syncthreads();
  const unsigned long long tau = tau_s;
  RecBest bl{1.0e300, 0xffffffffu, 0, 0};
  for (int i0 = tid * 4; i0 < n; i0 += PIV_NT * 4) {
    const Arm4 a = load_arm4(g, qi, i0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e;
      if (i >= n) break;
      const unsigned long long key = arm_key(a.S[e], a.l[e], (uint32_t)i, g);
      if (key <= tau) {
        const unsigned p = atomicAdd(&cnt, 1u);
        if (p < PIV_CAP) buf[p] = key;
      } else {
        const RecBest c{lower_of(a.S[e], a.l[e], g.d, g.alpha), (uint32_t)i + g.id_offset, a.S[e], a.l[e]};
        if (better_min(c, bl)) bl = c;
      }
    }
  }
  __syncthreads();
  const unsigned c = cnt;
  *outside = block_best<false>(bl, wsm);
  *cnt_out = c;
  if (c < need || c > PIV_CAP) return false;
  unsigned P = 2;
  while (P < c) P <<= 1;
  for (unsigned t = c + tid; t < P; t += PIV_NT) buf[t] = KEY_INVALID;
  __syncthreads();
  bitonic_keys(buf, P);
  return true;
}

__device__ __forceinline__ RecBest rec_of_key(const Geom &g, int qi, unsigned long long key, bool upper) {
  const uint32_t gid = (uint32_t)(key & ((1ull << g.kbits) - 1ull));
  const uint32_t i = gid - g.id_offset;
  const size_t o = (size_t)qi * g.npad + i;
  const int32_t S = g.S[o];
  const uint8_t l = g.lvl[o];
  return RecBest{upper ? upper_of(S, l, g.d, g.alpha) : lower_of(S, l, g.d, g.alpha), gid, S, l};
}

// Unsharded rank split + bounds + Eq. (5) (same contract as k_select).
__global__ void __launch_bounds__(PIV_NT) k_select_pivot(Geom g) {
  extern __shared__ unsigned long long pbuf[];
  __shared__ RecBest wsm[PIV_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
  const unsigned k = (unsigned)g.k, kh = (unsigned)(g.k + g.h);
  unsigned cnt;
  RecBest outside;
  if (g.force_radix || !pivot_pass(g, qi, kh, pbuf, &cnt, &outside, wsm)) {
    if (threadIdx.x == 0) st->fallback = 1;
    return;
  }
  RecBest bu{-1.0e300, 0xffffffffu, 0, 0}, bl = outside;
  for (unsigned t = threadIdx.x; t < cnt; t += PIV_NT) {
    if (t < k) {
      const RecBest c = rec_of_key(g, qi, pbuf[t], true);
      if (better_max(c, bu)) bu = c;
    } else if (t >= kh) {
      const RecBest c = rec_of_key(g, qi, pbuf[t], false);
      if (better_min(c, bl)) bl = c;
    }
  }
  bu = block_best<true>(bu, wsm);
  bl = block_best<false>(bl, wsm);
  if (threadIdx.x == 0) {
    st->fallback = 0;
    st->thr_k = pbuf[k - 1];
    st->thr_kh = pbuf[kh - 1];
    st->A = bu.v;
    st->B = bl.v;
    st->d1 = (int)(bu.gid - g.id_offset);
    st->d2 = (int)(bl.gid - g.id_offset);
    st->a_d2 = alpha_of(bl.lvl, g.alpha);
    st->rounds += 1;
    const int stop = bu.v <= bl.v;  // Eq. (5), "<=" as written
    st->done = stop;
    if (!stop) atomicAdd(&g.ctl->n_active, 1u);
  }
}

// Sharded local summary (same contract as k_select_local): the local top-(k+h)
// records and the remainder's minimum-L record.
__global__ void __launch_bounds__(PIV_NT) k_select_local_pivot(Geom g) {
  extern __shared__ unsigned long long pbuf[];
  __shared__ RecBest wsm[PIV_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
  const unsigned kh = (unsigned)(g.k + g.h);
  unsigned cnt;
  RecBest outside;
  if (g.force_radix || !pivot_pass(g, qi, kh, pbuf, &cnt, &outside, wsm)) {
    if (threadIdx.x == 0) st->fallback = 1;
    return;
  }
  ShardRec *out = g.send + (size_t)qi * (kh + 1);
  RecBest bl = outside;
  for (unsigned t = threadIdx.x; t < cnt; t += PIV_NT) {
    const unsigned long long key = pbuf[t];
    const uint32_t i = (uint32_t)(key & ((1ull << g.kbits) - 1ull)) - g.id_offset;
    const size_t o = (size_t)qi * g.npad + i;
    if (t < kh) {
      ShardRec r;
      r.key = key;
      r.S = g.S[o];
      r.lvl = g.lvl[o];
      r.pad[0] = r.pad[1] = r.pad[2] = 0;
      out[t] = r;
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

size_t pivot_smem_bytes() { return (size_t)PIV_CAP * sizeof(unsigned long long); }

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
