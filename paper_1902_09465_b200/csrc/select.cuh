// select.cuh -- block-wide radix select of two ranks over unique 64-bit keys
// (the rank split of P:144-146 on composite keys (d_hat-order key, index)).
#pragma once
#include "internal.cuh"

namespace aknn {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned NONE = 0xffffffffu;
constexpr unsigned long long KEY_INVALID = ~0ull;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Warp-aggregated shared-memory histogram increment (bins may collide).
__device__ __forceinline__ void hist_add(unsigned *hist, unsigned bin) {
  const unsigned m = __match_any_sync(FULL, bin);
  if (bin != NONE && lane_id() == __ffs(m) - 1) atomicAdd(&hist[bin], (unsigned)__popc(m));
}

constexpr int SEL_NT = 512;
constexpr int SEL_CAP = 2048;

struct SelSmem {
  unsigned hist[2 * 256];
  unsigned long long buf[2][SEL_CAP];
  unsigned bufn[2];
  unsigned long long pref[2], mask[2];
  unsigned rank[2], cand[2];
  int mode[2];  // 0 histogram, 1 collect + sort, 2 resolved
  int same;
};

__device__ __forceinline__ void bitonic_sort(unsigned long long *buf, unsigned n_used) {
  unsigned P = 2;
  while (P < n_used) P <<= 1;
  for (unsigned i = n_used + threadIdx.x; i < P; i += blockDim.x) buf[i] = KEY_INVALID;
  __syncthreads();
  for (unsigned k = 2; k <= P; k <<= 1)
    for (unsigned j = k >> 1; j > 0; j >>= 1) {
      for (unsigned idx = threadIdx.x; idx < P; idx += blockDim.x) {
        const unsigned ixj = idx ^ j;
        if (ixj > idx) {
          const unsigned long long a = buf[idx], b = buf[ixj];
          const bool up = (idx & k) == 0;
          if ((a > b) == up) {
            buf[idx] = b;
            buf[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
}

// One warp: find the bin where the cumulative count reaches `rank` (1-based).
__device__ __forceinline__ void scan_bins(const unsigned *hist, unsigned rank, unsigned *bin_out,
                          unsigned *below_out, unsigned *count_out) {
  const int lane = lane_id();
  unsigned loc[8];
  unsigned sum = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    loc[b] = hist[lane * 8 + b];
    sum += loc[b];
  }
  unsigned incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += v;
  }
  const unsigned excl = incl - sum;
  const unsigned ball = __ballot_sync(FULL, excl < rank && incl >= rank);
  const int src = __ffs(ball) - 1;
  if (lane == src) {
    unsigned c = excl;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      if (c + loc[b] >= rank) {
        *bin_out = lane * 8 + b;
        *below_out = c;
        *count_out = loc[b];
        break;
      }
      c += loc[b];
    }
  }
}

// Finds the keys of ranks r0 <= r1 (1-based) among the keys produced by
// `keys4(i0, out[4])` for i0 = 0, 4, 8, ... < n (invalid -> KEY_INVALID).
template <class F>
__device__ void select2(SelSmem &sm, F &keys4, int n, int nbits, unsigned r0, unsigned r1,
                        unsigned long long *th0, unsigned long long *th1) {
  const int tid = threadIdx.x;
  if (tid < 2) {
    sm.pref[tid] = 0;
    sm.mask[tid] = 0;
    sm.rank[tid] = tid == 0 ? r0 : r1;
    sm.cand[tid] = (unsigned)n;
    sm.mode[tid] = 0;
  }
  __syncthreads();
  int shift = ((nbits - 1) / 8) * 8;
  const int iters = (n + SEL_NT * 4 - 1) / (SEL_NT * 4);
  for (;;) {
    if (tid == 0) {
      for (int t = 0; t < 2; ++t)
        if (sm.mode[t] != 2) sm.mode[t] = (sm.cand[t] <= SEL_CAP) ? 1 : 0;
      sm.same = sm.mode[0] != 2 && sm.mode[1] != 2 && sm.pref[0] == sm.pref[1] &&
                sm.mask[0] == sm.mask[1] && sm.mode[0] == sm.mode[1];
      sm.bufn[0] = sm.bufn[1] = 0;
    }
    for (int b = tid; b < 512; b += SEL_NT) sm.hist[b] = 0;
    __syncthreads();
    const int mode0 = sm.mode[0], mode1 = sm.mode[1], same = sm.same;
    const unsigned long long p0 = sm.pref[0], m0 = sm.mask[0], p1 = sm.pref[1], m1 = sm.mask[1];
    for (int it = 0; it < iters; ++it) {
      const int i0 = (it * SEL_NT + tid) * 4;
      unsigned long long key[4];
      keys4(i0, key);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const unsigned long long kk = key[e];
        const bool valid = kk != KEY_INVALID;
        // target 0
        const bool in0 = valid && mode0 != 2 && (kk & m0) == p0;
        if (mode0 == 1) {
          if (in0) sm.buf[0][atomicAdd(&sm.bufn[0], 1u)] = kk;
        } else if (mode0 == 0) {
          hist_add(sm.hist, in0 ? (unsigned)((kk >> shift) & 255u) : NONE);
        }
        if (!same) {
          const bool in1 = valid && mode1 != 2 && (kk & m1) == p1;
          if (mode1 == 1) {
            if (in1) sm.buf[1][atomicAdd(&sm.bufn[1], 1u)] = kk;
          } else if (mode1 == 0) {
            hist_add(sm.hist, in1 ? 256u + (unsigned)((kk >> shift) & 255u) : NONE);
          }
        }
      }
    }
    __syncthreads();
    // resolve histogram targets (warp t handles target t)
    const int warp = tid >> 5;
    if (warp < 2) {
      const int t = warp;
      if (sm.mode[t] == 0) {
        const int src = (t == 1 && same) ? 0 : t;
        unsigned bin = 0, below = 0, cnt = 0;
        scan_bins(sm.hist + src * 256, sm.rank[t], &bin, &below, &cnt);
        // broadcast from the finding lane: all lanes of this warp wrote? only one did
        bin = __reduce_max_sync(FULL, bin);
        below = __reduce_max_sync(FULL, below);
        cnt = __reduce_max_sync(FULL, cnt);
        if (lane_id() == 0) {
          sm.pref[t] |= (unsigned long long)bin << shift;
          sm.mask[t] |= 255ull << shift;
          sm.rank[t] -= below;
          sm.cand[t] = cnt;
          if (shift == 0) sm.mode[t] = 2;
        }
      }
    }
    __syncthreads();
    // resolve collected targets
    for (int t = 0; t < 2; ++t) {
      if (sm.mode[t] != 1) continue;
      if (t == 1 && same) {
        // buffer 0 already sorted, same prefix
        if (tid == 0) {
          sm.pref[1] = sm.buf[0][sm.rank[1] - 1];
          sm.mode[1] = 2;
        }
        continue;
      }
      bitonic_sort(sm.buf[t], sm.bufn[t]);
      if (tid == 0) {
        sm.pref[t] = sm.buf[t][sm.rank[t] - 1];
        sm.mode[t] = 2;
      }
      __syncthreads();
    }
    __syncthreads();
    if (sm.mode[0] == 2 && sm.mode[1] == 2) break;
    shift -= 8;
    __syncthreads();
  }
  *th0 = sm.pref[0];
  *th1 = sm.pref[1];
}

}  // namespace aknn
