// a1_kernels.cu -- the literal Algorithm 1 schedule.
//
// Algorithm 1 samples exactly two arms per iteration, {d1, b2}, one
// coordinate each, then re-evaluates the rank split, Eq. (2)-(3) and Eq. (5).
// Iterations of one query are dependent, so the GPU runs one WARP per query and
// many queries side by side.  The warp keeps, per arm, the exact integer sum S,
// the sample count T, the cached estimate d_hat = S / (65025 T) and the cached
// lower bound L = d_hat - alpha(T), and the top-(k+h) arms as a
// list `cm` sorted by (d_hat, id) -- the bands of the paper's §4.1 heaps:
//   C = cm[0..k), M = cm[k..k+h), F = every other arm.
// Each iteration:
//   R2  restore "max key of cm <= min key of F" (swap the two while violated;
//       only the arms sampled last iteration can have broken it)
//   R3  d1 = argmax_C U, A = U_d1; d2 = argmin_F L, B = L_d2 (ties: smaller id)
//   R4  stop iff A <= B
//   Eq. (4) b2 = argmax_{{d2} u M} alpha (ties: d2, then smaller id)
//   a3  sample d1 and b2 once each (T += 1); at T == d the arm's S becomes the
//       exact sum, charged d evaluations (without replacement, reading
//       R23: the d samples are every coordinate once, so no extra charge)
// The per-arm sample stream is the batched rule's (Philox counter
// (u >> 2, id, qi, b) of the t-th sample, b = its doubling level), so the two
// schedules see the same coordinates.  Ranking by the cached fp64 d_hat with the
// id as tie-break is the exact rational order (reading R9).
#include <cstdint>
#include <cstdio>

#include "internal.cuh"
#include "launch.h"

namespace aknn {

namespace {

#ifdef AKNN_A1_CHECK
#define A1_CHECK(c, ...) do { if (!(c)) { printf("A1_CHECK %s line %d: ", #c, __LINE__); printf(__VA_ARGS__); printf("\n"); __trap(); } } while (0)
#else
#define A1_CHECK(c, ...) do { } while (0)
#endif

constexpr int A1_WARPS = 4;  // queries per CTA
constexpr unsigned FULL = 0xffffffffu;

struct A1Arm {  // per-query state, one workspace slice per query
  double *dh, *L;
  int32_t *S, *T, *cm;
  uint8_t *incm;
  const double *alpha;  // [d+1]: a shared-memory copy in shared-memory mode
};

__device__ __forceinline__ A1Arm a1_state(const A1Geom &g, unsigned char *b) {
  const size_t n = (size_t)g.n;
  A1Arm a;
  a.dh = reinterpret_cast<double *>(b);
  a.L = a.dh + n;
  a.S = reinterpret_cast<int32_t *>(a.L + n);
  a.T = a.S + n;
  a.cm = a.T + n;
  a.incm = reinterpret_cast<uint8_t *>(a.cm + g.kh);
  a.alpha = g.alpha;
  return a;
}

__device__ __forceinline__ bool key_less(double da, int ia, double db, int ib) {
  return da < db || (da == db && ia < ib);
}

__device__ __forceinline__ double a1_alpha(const A1Geom &g, const A1Arm &a, int T) { return T >= g.d ? 0.0 : a.alpha[T]; }

__device__ __forceinline__ double a1_dhat(int32_t S, int32_t T) {
  return (double)S / ((double)T * 65025.0);  // reading R15: one pinned expression
}

// (X[i][j] - x[j])^2 of the t-th sample of arm i (t = 0, 1, ...; level b = 0 for
// t = 0, else 1 + floor(log2 t); in-level ordinal u = t - 2^(b-1)).
__device__ __forceinline__ int32_t a1_draw(const A1Geom &g, const uint8_t *x, int i, int32_t t, uint32_t qrng) {
  uint32_t b = 0, u = 0;
  if (t > 0) {
    const uint32_t lg = 31u - (uint32_t)__clz(t);
    b = lg + 1u;
    u = (uint32_t)t - (1u << lg);
  }
  uint32_t j;
  if (g.wor) {  // reading R23: pi(t) of the arm's permutation
    j = wor_coord(wor_keys(g.rk0, g.rk1, (uint32_t)i + g.id_offset, qrng), g.wor_z, (uint32_t)g.d, (uint32_t)t);
  } else {
    const uint4 w = philox4x32_10_rk(make_uint4(u >> 2, (uint32_t)i + g.id_offset, qrng, b), g.rk0, g.rk1);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    j = coord_of(ws[u & 3u], (uint32_t)g.d);
  }
  A1_CHECK(i >= 0 && i < g.n && j < (uint32_t)g.d && t >= 0 && t < g.d, "i %d j %u t %d", i, j, t);
  const int32_t diff = (int32_t)g.X[(size_t)i * g.pitch + j] - (int32_t)x[j];
  return diff * diff;
}

// Warp: exact sum_j (X[i][j] - x[j])^2, result in every lane.
__device__ __forceinline__ int32_t a1_exact(const A1Geom &g, const uint8_t *x, int i, int lane) {
  const uint8_t *xr = g.X + (size_t)i * g.pitch;
  int32_t s = 0;
  for (int j = lane; j < g.d; j += 32) {
    const int32_t diff = (int32_t)xr[j] - (int32_t)x[j];
    s += diff * diff;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
  return s;
}

struct KeyArg {  // running argmin of (v, id)
  double v;
  int i;
};

__device__ __forceinline__ KeyArg warp_min(KeyArg a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    KeyArg b{__shfl_xor_sync(FULL, a.v, o), __shfl_xor_sync(FULL, a.i, o)};
    if (b.i >= 0 && (a.i < 0 || key_less(b.v, b.i, a.v, a.i))) a = b;
  }
  return a;
}

__device__ __forceinline__ KeyArg warp_max(KeyArg a) {  // ties: smaller id
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    KeyArg b{__shfl_xor_sync(FULL, a.v, o), __shfl_xor_sync(FULL, a.i, o)};
    if (b.i >= 0 && (a.i < 0 || b.v > a.v || (b.v == a.v && b.i < a.i))) a = b;
  }
  return a;
}

// The lane's share of F (arms i = lane mod 32 outside cm): its minimum key
// (d_hat, id) and its argmin of L (ties: smaller id).  Kept in registers and
// rescanned only when an arm of the lane left F or changed inside it.
__device__ __forceinline__ void lane_scan(const A1Geom &g, const A1Arm &a, int lane, KeyArg *pk, KeyArg *pl) {
  KeyArg km{0.0, -1}, lm{0.0, -1};
#pragma unroll 4
  for (int i = lane; i < g.n; i += 32) {
    if (a.incm[i]) continue;
    const double dh = a.dh[i], L = a.L[i];
    if (km.i < 0 || key_less(dh, i, km.v, km.i)) km = KeyArg{dh, i};
    if (lm.i < 0 || key_less(L, i, lm.v, lm.i)) lm = KeyArg{L, i};
  }
  *pk = km;
  *pl = lm;
}

__device__ __forceinline__ void fold_min(KeyArg *m, double v, int i) {
  if (m->i < 0 || key_less(v, i, m->v, m->i)) *m = KeyArg{v, i};
}

// cm without the entry at position p, then `arm` inserted at its rank: every lane
// buffers the entries it moves before the warp writes them back.
constexpr int A1_CM_PER_LANE = A1_MAX_KH / 32;

__device__ void cm_reinsert(const A1Geom &g, const A1Arm &a, int p, int arm, int lane) {
  const int kh = g.kh;
  const double da = a.dh[arm];
  // rank of `arm` among the other kh - 1 entries
  int r = 0;
  for (int j = lane; j < kh; j += 32) {
    if (j == p) continue;
    const int e = a.cm[j];
    r += key_less(a.dh[e], e, da, arm) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
  // new[j]: j < min(p, r) or j > max(p, r): unchanged; r == p: unchanged but arm
  int v[A1_CM_PER_LANE];
#pragma unroll
  for (int m = 0; m < A1_CM_PER_LANE; ++m) {
    const int j = lane + 32 * m;
    v[m] = -1;
    if (j >= kh) continue;
    if (j == r) v[m] = arm;
    else if (p < r && j >= p && j < r) v[m] = a.cm[j + 1];
    else if (r < p && j > r && j <= p) v[m] = a.cm[j - 1];
  }
  __syncwarp();
#pragma unroll
  for (int m = 0; m < A1_CM_PER_LANE; ++m) {
    const int j = lane + 32 * m;
    if (j < kh && v[m] >= 0) a.cm[j] = v[m];
  }
  __syncwarp();
}

__device__ __forceinline__ int cm_find(const A1Geom &g, const A1Arm &a, int arm, int lane) {
  int p = -1;
  for (int j = lane; j < g.kh; j += 32)
    if (a.cm[j] == arm) p = j;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) p = max(p, __shfl_xor_sync(FULL, p, o));
  return p;
}

__global__ void __launch_bounds__(32 * A1_WARPS) k_a1(A1Geom g) {
  extern __shared__ __align__(16) unsigned char a1sm[];
  const int lane = threadIdx.x & 31;
  const int wpc = g.smem ? 1 : A1_WARPS;  // warps per CTA
  const int slot = blockIdx.x * wpc + (threadIdx.x >> 5);
  const int qi = g.q0 + slot;
  if (slot >= g.qb || (threadIdx.x >> 5) >= wpc) return;  // warp-uniform
  A1Arm a = a1_state(g, g.smem ? a1sm : g.ws + (size_t)slot * g.ws_per_query);
  const uint8_t *x = g.Q + (size_t)qi * g.d;
  if (g.smem) {  // alpha and the query row next to the state (latency of every iteration)
    const size_t off = ((size_t)g.n * 24 + (size_t)g.kh * 4 + (size_t)g.n + 7) & ~(size_t)7;
    double *al = reinterpret_cast<double *>(a1sm + off);
    uint8_t *xs = reinterpret_cast<uint8_t *>(al + g.d + 1);
    for (int t = lane; t <= g.d; t += 32) al[t] = g.alpha[t];
    for (int j = lane; j < g.d; j += 32) xs[j] = x[j];
    __syncwarp();
    a.alpha = al;
    x = xs;
  }
  const uint32_t qrng = (uint32_t)qi + g.qi0;
  const int n = g.n, k = g.k, kh = g.kh, d = g.d;

  // R0: one sample per arm, T = 1 (d = 1: that sample is the exact sum)
  for (int i = lane; i < n; i += 32) {
    const int32_t S = a1_draw(g, x, i, 0, qrng);
    const int32_t T = d == 1 ? d : 1;
    a.S[i] = S;
    a.T[i] = T;
    const double dh = a1_dhat(S, T);
    a.dh[i] = dh;
    a.L[i] = dh - a1_alpha(g, a, T);
    a.incm[i] = 0;
  }
  __syncwarp();
  long long draws = n, nexact = 0;
  KeyArg pk, pl;  // the lane's share of F
  lane_scan(g, a, lane, &pk, &pl);
  // the initial top-(k + h), in rank order
  for (int r = 0; r < kh; ++r) {
    const KeyArg km = warp_min(pk);
    if (lane == 0) {
      a.cm[r] = km.i;
      a.incm[km.i] = 1;
    }
    __syncwarp();
    if ((km.i & 31) == lane) lane_scan(g, a, lane, &pk, &pl);
  }
  int it = 0, status = 0;
  for (;;) {
    ++it;
    // R2: the top-(k + h) band against F
    KeyArg km, d2;
    for (;;) {
      km = warp_min(pk);
      d2 = warp_min(pl);
      const int last = a.cm[kh - 1];
      A1_CHECK(km.i >= 0 && km.i < n && d2.i >= 0 && d2.i < n && last >= 0 && last < n, "km %d d2 %d last %d it %d", km.i, d2.i, last, it);
      const double dl = a.dh[last];
      if (!key_less(km.v, km.i, dl, last)) break;
      if (lane == 0) {
        a.incm[last] = 0;
        a.incm[km.i] = 1;
      }
      __syncwarp();
      cm_reinsert(g, a, kh - 1, km.i, lane);
      if ((km.i & 31) == lane) lane_scan(g, a, lane, &pk, &pl);  // its minimum left F
      if ((last & 31) == lane) {  // `last` joins F
        fold_min(&pk, dl, last);
        fold_min(&pl, a.L[last], last);
      }
    }
    // R3: d1 over C
    KeyArg d1{0.0, -1};
    for (int r = lane; r < k; r += 32) {
      const int i = a.cm[r];
      const double U = a.dh[i] + a1_alpha(g, a, a.T[i]);
      if (d1.i < 0 || U > d1.v || (U == d1.v && i < d1.i)) d1 = KeyArg{U, i};
    }
    d1 = warp_max(d1);
    const double A = d1.v, B = d2.v;
    if (A <= B) break;  // R4, Eq. (5)
    if (g.max_iters > 0 && it >= g.max_iters) {
      status = 1;
      break;
    }
    // Eq. (4): b2 = argmax over {d2} u M of alpha (ties: d2, then smaller id)
    KeyArg bm{0.0, -1};
    for (int r = k + lane; r < kh; r += 32) {
      const int i = a.cm[r];
      const double al = a1_alpha(g, a, a.T[i]);
      if (bm.i < 0 || al > bm.v || (al == bm.v && i < bm.i)) bm = KeyArg{al, i};
    }
    bm = warp_max(bm);
    const int b2 = (bm.i >= 0 && bm.v > a1_alpha(g, a, a.T[d2.i])) ? bm.i : d2.i;
    A1_CHECK(d1.i >= 0 && d1.i < n && b2 >= 0 && b2 < n && d1.i != b2, "d1 %d b2 %d it %d", d1.i, b2, it);
    // a3: one sample of d1 and one of b2 (distinct arms: d1 in C, b2
    // not), drawn side by side by lanes 0 and 1
    const int32_t T1 = a.T[d1.i], T2 = a.T[b2];
    int32_t v = 0;
    if (lane < 2) {
      const int l = lane == 0 ? d1.i : b2;
      const int32_t T = lane == 0 ? T1 : T2;
      if (T + 1 < d) v = a1_draw(g, x, l, T, qrng);
    }
    int32_t S1 = a.S[d1.i] + __shfl_sync(FULL, v, 0), S2 = a.S[b2] + __shfl_sync(FULL, v, 1);
    if (T1 + 1 == d) S1 = a1_exact(g, x, d1.i, lane);  // "If T_l = m ... exactly"
    if (T2 + 1 == d) S2 = a1_exact(g, x, b2, lane);
    draws += (T1 < d) + (T2 < d);
    nexact += (T1 + 1 == d) + (T2 + 1 == d);
    // apply one arm at a time: cm_reinsert ranks an arm against a band whose other
    // entries are in order
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const int l = s2 == 0 ? d1.i : b2;
      const int32_t T = s2 == 0 ? T1 : T2;
      if (T >= d) continue;  // uniform
      __syncwarp();
      if (lane == 0) {
        const int32_t S = s2 == 0 ? S1 : S2;
        a.S[l] = S;
        a.T[l] = T + 1;
        const double dh = a1_dhat(S, T + 1);
        a.dh[l] = dh;
        a.L[l] = dh - a1_alpha(g, a, T + 1);
      }
      __syncwarp();
      if (a.incm[l]) {
        const int p = cm_find(g, a, l, lane);
        A1_CHECK(p >= 0 && p < kh, "cm_find %d arm %d it %d", p, l, it);
        cm_reinsert(g, a, p, l, lane);
      }
      else if ((l & 31) == lane) lane_scan(g, a, lane, &pk, &pl);  // an F arm moved
    }
  }
  // outputs: the band in rank order, its estimates, the per-arm state
  const OutPtrs &o = g.out;
  const size_t row = (size_t)(o.row0 + qi);
  for (int r = lane; r < kh; r += 32) {
    const int i = a.cm[r];
    o.sets[row * kh + r] = (int32_t)(i + g.id_offset);
    if (o.dhat) o.dhat[row * kh + r] = a.dh[i];
  }
  for (int i = lane; i < n; i += 32) {
    if (o.counts) o.counts[row * o.ncols + i] = a.T[i];
    if (o.sums) o.sums[row * o.ncols + i] = a.S[i];
  }
  if (lane == 0) {
    if (o.draws) o.draws[row] = draws;
    // without replacement an arm reaching T = d drew every coordinate once: no charge
    if (o.evals) o.evals[row] = g.wor ? draws : draws + (long long)d * nexact;
    if (o.rounds) o.rounds[row] = it;
    if (status) atomicOr(g.status, 1);
  }
}

}  // namespace

// State in shared memory (one warp per CTA) when a query's slice fits
// A1_SMEM_MAX, else in the global workspace (A1_WARPS warps per CTA).
cudaError_t launch_a1(const A1Geom &g, cudaStream_t s) {
  if (g.qb <= 0) return cudaSuccess;
  if (g.smem) {
    cudaError_t e = cudaFuncSetAttribute(k_a1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.ws_per_query);
    if (e != cudaSuccess) return e;
    k_a1<<<(unsigned)g.qb, 32, g.ws_per_query, s>>>(g);
  } else {
    k_a1<<<(unsigned)((g.qb + A1_WARPS - 1) / A1_WARPS), 32 * A1_WARPS, 0, s>>>(g);
  }
  return cudaGetLastError();
}

size_t a1_ws_per_query(int64_t n, int kh, int d, bool tables) {
  size_t b = ((size_t)n * (8 + 8 + 4 + 4) + (size_t)kh * 4 + (size_t)n + 7) & ~(size_t)7;
  if (tables) b += (size_t)(d + 1) * 8 + (size_t)d;
  return (b + 255) / 256 * 256;
}

}  // namespace aknn
