// exact_kernels.cu -- the exact comparison pass (brute force): every
// distance D(q, i) = sum_j (x_ij - q_j)^2 exactly in integers, then the k
// nearest per query by (D, i).
//
// Used for k > exact_fused_max_k() only: the tcgen05 distance matrix of exact_mma.cu
// is ranked here by the block radix select of select.cuh and a rank sort of the k
// winners (k <= 128 runs the fused kernel of exact_fused.cu instead).
#include "internal.cuh"
#include "launch.h"
#include "select.cuh"

namespace aknn {

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

cudaError_t launch_exact_topk(const ExactGeom &e, cudaStream_t s) {
  k_exact_topk<<<e.q, SEL_NT, 0, s>>>(e);
  return cudaGetLastError();
}

}  // namespace aknn
