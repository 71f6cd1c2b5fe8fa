// probes.cu -- microbenchmarks that MEASURE the roofline denominators of the hot
// kernels on the box bench.py runs on (not part of libaknn.so, not on the hot path):
//
//   probe_philox   the achievable rate of Philox4x32-10 blocks + the multiply-high
//                  coordinate map (the integer work per 4 draws of k_advance), with
//                  no memory traffic: the ALU ceiling of the sampled levels.
//   probe_gather   the achievable rate of random one-byte gathers (one 32-B sector
//                  each) from a buffer of a given footprint: the sector ceiling
//                  (L2-resident footprint vs HBM footprint).
//   probe_shared   the achievable rate of the shared-draw tile gathers:
//                  per 4 draws one broadcast 16-byte load of packed (32 j | x << 24)
//                  words, 4 conflict-free byte gathers from a transposed 32-row query
//                  tile, VABSDIFF4 + IDP.4A -- the same instruction mix as
//                  k_advance_tiles' accumulate loop, with nothing else: its ceiling.
//
// C-ABI: each returns the best device time in ms over `reps` launches (CUDA events).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ uint4 philox(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * c.x;
    const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ (k0 + r * 0x9E3779B9u), (uint32_t)p1,
                   (uint32_t)(p0 >> 32) ^ c.w ^ (k1 + r * 0xBB67AE85u), (uint32_t)p0);
  }
  return c;
}

__global__ void __launch_bounds__(256) k_probe_philox(long long blocks_per_thread, uint32_t d, uint32_t k0,
                                                      uint32_t k1, uint32_t *out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (long long b = 0; b < blocks_per_thread; b += 4) {
    uint4 w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = philox(make_uint4((uint32_t)b + k, t, 7u, 3u), k0, k1);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      acc += __umulhi(w[k].x, d) + __umulhi(w[k].y, d) + __umulhi(w[k].z, d) + __umulhi(w[k].w, d);
  }
  out[t] = acc;
}

__global__ void __launch_bounds__(256) k_probe_gather(const uint8_t *__restrict__ buf, uint64_t bytes,
                                                      int loads_per_thread, uint32_t *out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t x = 0x9E3779B97F4A7C15ull * (t + 1);
  uint32_t acc = 0;
  for (int l = 0; l < loads_per_thread; l += 8) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x ^= x << 13;
      x ^= x >> 7;
      x ^= x << 17;
      v[k] = __ldg(buf + (x & (bytes - 1)));  // bytes is a power of two
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  out[t] = acc;
}

__global__ void __launch_bounds__(256) k_probe_shared(int iters, uint32_t *out) {
  __shared__ uint8_t qt[784 * 32];
  __shared__ uint32_t dbuf[8][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 784 * 32; i += 256) qt[i] = (uint8_t)(i * 2654435761u >> 24);
  for (int i = tid; i < 8 * 256; i += 256) {
    const uint32_t j = (i * 2654435761u) % 784u;
    (&dbuf[0][0])[i] = (j * 32u) | ((uint32_t)(i * 40503u) << 24);
  }
  __syncthreads();
  const uint32_t ql = (uint32_t)__cvta_generic_to_shared(qt) + lane;
  const uint4 *dp = reinterpret_cast<const uint4 *>(dbuf[warp]);
  uint32_t sum = 0;
  for (int it = 0; it < iters; ++it) {
    for (int u = 0; u < 64; ++u) {
      const uint4 pk = dp[u];
      uint32_t q[4];
      const uint32_t v[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(q[e]) : "r"(ql + (v[e] & 0x1FFFFFu)));
      const uint32_t x4 = __byte_perm(__byte_perm(pk.x, pk.y, 0x0073), __byte_perm(pk.z, pk.w, 0x0073), 0x5410);
      const uint32_t q4 = __byte_perm(__byte_perm(q[0], q[1], 0x0040), __byte_perm(q[2], q[3], 0x0040), 0x5410);
      const uint32_t t = __vabsdiffu4(x4, q4);
      sum = __dp4a(t, t, sum);
    }
  }
  out[blockIdx.x * 256 + tid] = sum;
}

template <class F>
double best_ms(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best;
}

}  // namespace

extern "C" {

// Blocks computed = grid_threads * blocks_per_thread; returns best ms.
double probe_philox(int grid_threads, long long blocks_per_thread, uint32_t d, int reps) {
  uint32_t *out = nullptr;
  if (cudaMalloc(&out, sizeof(uint32_t) * grid_threads) != cudaSuccess) return -1.0;
  const int nb = (grid_threads + 255) / 256;
  const double ms = best_ms([&] { k_probe_philox<<<nb, 256>>>(blocks_per_thread, d, 1u, 2u, out); }, reps);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(out);
  return e == cudaSuccess ? ms : -1.0;
}

// Random byte loads = grid_threads * loads_per_thread over a `bytes` (power of two) footprint.
double probe_gather(int grid_threads, int loads_per_thread, unsigned long long bytes, int reps) {
  if (bytes == 0 || (bytes & (bytes - 1))) return -1.0;
  uint8_t *buf = nullptr;
  uint32_t *out = nullptr;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return -1.0;
  if (cudaMalloc(&out, sizeof(uint32_t) * grid_threads) != cudaSuccess) {
    cudaFree(buf);
    return -1.0;
  }
  cudaMemset(buf, 1, bytes);
  const int nb = (grid_threads + 255) / 256;
  const double ms = best_ms([&] { k_probe_gather<<<nb, 256>>>(buf, bytes, loads_per_thread, out); }, reps);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(buf);
  cudaFree(out);
  return e == cudaSuccess ? ms : -1.0;
}

// (query, point) draws = blocks * 256 * iters * 256; returns best ms.
double probe_shared(int blocks, int iters, int reps) {
  uint32_t *out = nullptr;
  if (cudaMalloc(&out, sizeof(uint32_t) * 256 * (size_t)blocks) != cudaSuccess) return -1.0;
  const double ms = best_ms([&] { k_probe_shared<<<blocks, 256>>>(iters, out); }, reps);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFree(out);
  return e == cudaSuccess ? ms : -1.0;
}

}  // extern "C"
