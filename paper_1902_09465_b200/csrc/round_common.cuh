// round_common.cuh -- per-arm state access shared by the round kernels.
#pragma once
#include "internal.cuh"
#include "select.cuh"

namespace aknn {

// ---------------------------------------------------------------------------
// Pair state loading: 4 consecutive arms of query row `qi` starting at i0
// (i0 % 4 == 0, rows padded to npad % 16 == 0, so the loads are aligned).
struct Arm4 {
  int32_t S[4];
  uint32_t lw;  // the 4 level bytes, packed: unpacked only where used, so a load issued
                // ahead (k_filter's prefetch) is not waited on at the load site
  __device__ __forceinline__ uint8_t l(int e) const { return (uint8_t)(lw >> (8 * e)); }
};

__device__ __forceinline__ Arm4 load_arm4(const Geom &g, int qi, int i0) {
  Arm4 a;
  const int4 s = *reinterpret_cast<const int4 *>(g.S + (size_t)qi * g.npad + i0);
  a.lw = *reinterpret_cast<const uint32_t *>(g.lvl + (size_t)qi * g.npad + i0);
  a.S[0] = s.x; a.S[1] = s.y; a.S[2] = s.z; a.S[3] = s.w;
  return a;
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
      key[e] = (i0 + e < g->n) ? arm_key(a.S[e], a.l(e), (uint32_t)(i0 + e), *g) : KEY_INVALID;
  }
};

struct Best {
  double v;
  int i;
  double a;
};

struct RecBest {  // a candidate for d1 (max U) or d2 (min L), ties to the smaller global id
  double v;
  uint32_t gid;
  int32_t S;
  uint8_t lvl;
};

__device__ __forceinline__ bool better_min(const RecBest &a, const RecBest &b) {
  return a.v < b.v || (a.v == b.v && a.gid < b.gid);
}
__device__ __forceinline__ bool better_max(const RecBest &a, const RecBest &b) {
  return a.v > b.v || (a.v == b.v && a.gid < b.gid);
}

__device__ __forceinline__ RecBest shfl_best(const RecBest &b, int o) {
  RecBest r;
  r.v = __shfl_xor_sync(FULL, b.v, o);
  r.gid = __shfl_xor_sync(FULL, b.gid, o);
  r.S = __shfl_xor_sync(FULL, b.S, o);
  r.lvl = (uint8_t)__shfl_xor_sync(FULL, (unsigned)b.lvl, o);
  return r;
}

// Block-wide arg-min (want_max = false) or arg-max; result valid in every thread.
template <bool want_max>
__device__ RecBest block_best(RecBest b, RecBest *wsm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const RecBest t = shfl_best(b, o);
    if (want_max ? better_max(t, b) : better_min(t, b)) b = t;
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane_id() == 0) wsm[w] = b;
  __syncthreads();
  RecBest r = wsm[0];
  for (int i = 1; i < nw; ++i)
    if (want_max ? better_max(wsm[i], r) : better_min(wsm[i], r)) r = wsm[i];
  return r;
}

}  // namespace aknn
