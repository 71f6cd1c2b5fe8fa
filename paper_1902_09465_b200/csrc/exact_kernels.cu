// exact_kernels.cu -- the exact comparison pass (brute force): every
// distance D(q, i) = sum_j (x_ij - q_j)^2 exactly in integers, then the k
// nearest per query by (D, i).
//
// v1: CUDA-core tiles (vabsdiff4 + dp4a), 64 queries x 64 points per CTA,
// then the block radix select of select.cuh and a rank sort of the k winners.
#include "internal.cuh"
#include "launch.h"
#include "select.cuh"

namespace aknn {

constexpr int EX_TQ = 64, EX_TP = 64, EX_TK = 64;  // tile: queries, points, bytes

__global__ void __launch_bounds__(256) k_exact_tiles(ExactGeom e) {
  __shared__ uint32_t sq[EX_TQ][EX_TK / 4 + 1];
  __shared__ uint32_t sx[EX_TP][EX_TK / 4 + 1];
  const int q0 = blockIdx.y * EX_TQ, p0 = blockIdx.x * EX_TP;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4 x 4 each
  uint32_t acc[4][4] = {};
  for (int64_t k0 = 0; k0 < e.pitch; k0 += EX_TK) {
    for (int t = threadIdx.x; t < EX_TQ * (EX_TK / 4); t += 256) {
      const int r = t / (EX_TK / 4), w = t % (EX_TK / 4);
      const int64_t col = k0 + w * 4;
      uint32_t vq = 0, vx = 0;
      if (q0 + r < e.q && col < e.pitch)
        vq = *reinterpret_cast<const uint32_t *>(e.Q + (size_t)(q0 + r) * e.pitch + col);
      if (p0 + r < e.n && col < e.pitch)
        vx = __ldg(reinterpret_cast<const uint32_t *>(e.X + (size_t)(p0 + r) * e.pitch + col));
      sq[r][w] = vq;
      sx[r][w] = vx;
    }
    __syncthreads();
#pragma unroll 4
    for (int w = 0; w < EX_TK / 4; ++w) {
      uint32_t a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = sq[ty * 4 + u][w];
        b[u] = sx[tx * 4 + u][w];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t t = __vabsdiffu4(a[u], b[v]);
          acc[u][v] = __dp4a(t, t, acc[u][v]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int qq = q0 + ty * 4 + u, pp = p0 + tx * 4 + v;
      if (qq < e.q && pp < e.n) e.D[(size_t)qq * e.npad + pp] = (int32_t)acc[u][v];
    }
}

struct DistKeys {
  const ExactGeom *e;
  int qi;
  __device__ __forceinline__ void operator()(int i0, unsigned long long key[4]) const {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = i0 + t;
      key[t] = (i < e->n) ? (((unsigned long long)(uint32_t)e->D[(size_t)qi * e->npad + i] << e->ibits) | (uint32_t)i)
                          : KEY_INVALID;
    }
  }
};

__global__ void __launch_bounds__(SEL_NT) k_exact_topk(ExactGeom e) {
  __shared__ SelSmem sm;
  __shared__ unsigned long long win[1024];
  __shared__ unsigned cnt;
  const int qi = blockIdx.x;
  DistKeys keys{&e, qi};
  unsigned long long th, th2;
  select2(sm, keys, e.n, e.nbits, (unsigned)e.k, (unsigned)e.k, &th, &th2);
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < e.n; i += SEL_NT) {
    const unsigned long long kk = ((unsigned long long)(uint32_t)e.D[(size_t)qi * e.npad + i] << e.ibits) | (uint32_t)i;
    if (kk <= th) {
      const unsigned p = atomicAdd(&cnt, 1u);
      if (p < 1024) win[p] = kk;
    }
  }
  __syncthreads();
  const int m = min((int)cnt, e.k);
  for (int r = threadIdx.x; r < m; r += SEL_NT) {
    int rank = 0;
    for (int t = 0; t < m; ++t) rank += win[t] < win[r];
    const unsigned long long kk = win[r];
    const uint32_t i = (uint32_t)(kk & ((1ull << e.ibits) - 1));
    e.idx[(size_t)qi * e.k + rank] = (int32_t)(i + e.id_offset);
    e.dist2[(size_t)qi * e.k + rank] = (int32_t)(kk >> e.ibits);
  }
}

cudaError_t launch_exact(const ExactGeom &e, cudaStream_t s) {
  dim3 grid((e.n + EX_TP - 1) / EX_TP, (e.q + EX_TQ - 1) / EX_TQ);
  k_exact_tiles<<<grid, 256, 0, s>>>(e);
  k_exact_topk<<<e.q, SEL_NT, 0, s>>>(e);
  return cudaGetLastError();
}

cudaError_t launch_exact_topk(const ExactGeom &e, cudaStream_t s) {
  k_exact_topk<<<e.q, SEL_NT, 0, s>>>(e);
  return cudaGetLastError();
}

}  // namespace aknn
