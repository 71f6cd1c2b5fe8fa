// exact_fused.cu -- the exact comparison pass (row a10; "compute all distances,
// then sort") as ONE persistent tensor-core kernel whose epilogue keeps each query's
// running top-k, so the [q][n] distance matrix is never written.
//
//   D(q, i) = ||x_i||^2 + ||q||^2 - 2 <x_i, q>   (u8 x u8 -> s32 on tcgen05, exact:
//   d * 255^2 < 2^31 for d <= 33025), ranked by the composite key (D << 32 | i), i.e.
//   by (distance, smaller id) -- the oracle's brute-force order (orc_bruteforce).
//
// Work split.  Queries in 128-row m-blocks (TMEM lanes), points in 256-column tiles.
// A launch covers mt <= #SMs m-blocks; CTA b takes m-block b % mt and the b / mt-th of
// G = #SMs / mt contiguous ranges of point tiles, so the mt CTAs of one range stream
// the same X tiles at the same time (X read from HBM about once, the other m-blocks
// hit L2).  Per CTA:
//   warp 0 lane 0   TMA producer: Q k-block (128 x 128 B) + X k-block (256 x 128 B) per
//                   stage, 4-stage ring, running ahead across the CTA's tiles
//   warp 1          TMEM owner (512 columns = two 128 x 256 int32 accumulators) and,
//                   lane 0, the MMA issuer: 4 x tcgen05.mma kind::i8 (K = 32 B) per
//                   stage into accumulator t & 1, commit -> stage free / tile done
//   warps 4..11     epilogue (TMEM lane quadrant = warp % 4, column half = (warp-4)/4):
//                   thread = one (query row, column half) STREAM with a candidate
//                   buffer (global, L2-resident) and a threshold tau = the k-th
//                   smallest key kept so far; a key < tau is appended.  When a buffer
//                   is full the warp compacts it to its k smallest with a warp radix
//                   select (tau = the k-th).  The accumulator is released as soon as
//                   its last chunk is in registers, so the MMAs of tile t+2 overlap.
//   end of range    each stream's k smallest -> part[]; k_exact_merge then picks each
//                   query's k smallest of its 2 G lists and sorts them.
// Expected appends per stream ~ CAP * log_{CAP/k}(points/CAP): a few compactions per
// stream.
#include <cuda.h>

#include <algorithm>

#include "internal.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace aknn {

constexpr int XF_BM = 128, XF_BN = 256, XF_STAGES = 4;
constexpr int XF_EPI_WARP0 = 4, XF_EPI_WARPS = 8, XF_NT = 32 * (XF_EPI_WARP0 + XF_EPI_WARPS);
constexpr uint32_t XF_A_BYTES = XF_BM * MM_BK, XF_B_BYTES = XF_BN * MM_BK;
constexpr uint32_t XF_STAGE_BYTES = XF_A_BYTES + XF_B_BYTES;
constexpr int XF_CAP = 512;             // compaction threshold of a stream's buffer
constexpr int XF_BUF = XF_CAP + 32;     // + one 32-column chunk of slack
constexpr int XF_E = XF_BUF / 32;       // keys per lane in a warp compaction
constexpr int XF_MAX_K = 128;
constexpr int XF_STREAMS = 2 * XF_BM;   // streams per CTA: (column half, row)
constexpr size_t XF_SMEM = (size_t)XF_STAGES * XF_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                           (size_t)XF_EPI_WARPS * 256 * 4 /*radix histograms*/;
constexpr unsigned long long XF_NONE = ~0ull;

struct XfGeom {
  int q, n, k;          // queries of this launch, points, neighbours
  int mt, G, nt;        // m-blocks, point-tile ranges per m-block, point tiles
  int nk;               // 128-byte k-blocks of d
  uint32_t id_offset;
  const int32_t *nq;    // [q] ||q||^2 of this launch's queries
  const int32_t *nx;    // [>= nt * 256] ||x_i||^2 (zero padded)
  unsigned long long *buf;   // [grid][XF_STREAMS][XF_BUF]
  unsigned long long *part;  // [grid][XF_STREAMS][k]
  const unsigned long long *bound;  // [q] initial per-query threshold (the pilot's k-th key), or null
};

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((unsigned long long)hi << 32) | lo;
}

// Warp-cooperative: the c keys in b[0..c) (unique), k <= c.  Finds the k-th smallest by
// an 8-bit radix select (histogram in `hist`, 256 words of this warp's shared memory),
// moves the k smallest to b[0..k) (any order) and returns the k-th smallest.
__device__ unsigned long long warp_compact(unsigned long long *b, int c, int k, uint32_t *hist, int lane) {
  unsigned long long key[XF_E];
  unsigned long long orr = 0;
#pragma unroll
  for (int e = 0; e < XF_E; ++e) {
    const int i = lane + 32 * e;
    key[e] = i < c ? b[i] : XF_NONE;
    if (i < c) orr |= key[e];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) orr |= shfl64(orr, lane ^ o);
  const int top = orr ? 63 - __clzll((long long)orr) : 0;
  unsigned long long prefix = 0, pmask = 0, kth = 0;
  int want = k;
  bool found = false;
  for (int shift = (top >> 3) << 3; shift >= 0; shift -= 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < XF_E; ++e)
      if (key[e] != XF_NONE && (key[e] & pmask) == prefix) atomicAdd(&hist[(uint32_t)(key[e] >> shift) & 255u], 1u);
    __syncwarp();
    uint32_t h[8], loc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      h[i] = hist[lane * 8 + i];
      loc += h[i];
    }
    uint32_t inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t exc = inc - loc;
    int bin = -1;
    uint32_t before = 0, cb = 0;
    if (exc < (uint32_t)want && (uint32_t)want <= inc) {
      uint32_t acc = exc;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (bin < 0 && acc + h[i] >= (uint32_t)want) {
          bin = lane * 8 + i;
          before = acc;
          cb = h[i];
        }
        acc += h[i];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, bin >= 0)) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    before = __shfl_sync(0xffffffffu, before, src);
    cb = __shfl_sync(0xffffffffu, cb, src);
    prefix |= (unsigned long long)bin << shift;
    pmask |= 255ull << shift;
    want -= (int)before;
    if (cb == 1u) {  // the k-th key is the only one with this prefix
      unsigned long long mine = 0;
      bool has = false;
#pragma unroll
      for (int e = 0; e < XF_E; ++e)
        if (key[e] != XF_NONE && (key[e] & pmask) == prefix) {
          mine = key[e];
          has = true;
        }
      const int s2 = __ffs(__ballot_sync(0xffffffffu, has)) - 1;
      kth = shfl64(mine, s2);
      found = true;
      break;
    }
    __syncwarp();
  }
  if (!found) kth = prefix;  // all 64 bits decided
  // keep the keys <= kth: exactly k of them (keys are unique)
  int base = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int e = 0; e < XF_E; ++e) {
    const bool keep = key[e] <= kth;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (keep) b[base + __popc(bal & lt)] = key[e];
    base += __popc(bal);
  }
  __syncwarp();
  return kth;
}

__global__ void __launch_bounds__(XF_NT, 1)
    k_exact_fused(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ XfGeom g) {
  const int b = blockIdx.x, mb = b % g.mt, seg = b / g.mt;
  const int t_begin = (int)((long long)seg * g.nt / g.G), t_end = (int)((long long)(seg + 1) * g.nt / g.G);
  const int ntl = t_end - t_begin;
  const int m0 = mb * XF_BM;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + XF_STAGES * XF_STAGE_BYTES);
  uint64_t *empty = full + XF_STAGES;
  uint64_t *tfull = empty + XF_STAGES;  // [2]
  uint64_t *tempty = tfull + 2;         // [2]
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(tempty + 2);
  uint32_t *hist_all = reinterpret_cast<uint32_t *>(sm + XF_STAGES * XF_STAGE_BYTES + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < XF_STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, XF_EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t kg = 0;
      for (int t = 0; t < ntl; ++t) {
        const int n0 = (t_begin + t) * XF_BN;
        for (int kb = 0; kb < g.nk; ++kb, ++kg) {
          const uint32_t s = kg % XF_STAGES;
          if (kg >= XF_STAGES) mbar_wait(empty + s, ((kg / XF_STAGES) - 1) & 1);
          unsigned char *sa = sm + s * XF_STAGE_BYTES;
          mbar_expect_tx(full + s, XF_STAGE_BYTES);
          tma_load_2d(sa, &tmQ, full + s, kb * MM_BK, m0);
          tma_load_2d(sa + XF_A_BYTES, &tmX, full + s, kb * MM_BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = umma_idesc_u8(XF_BM, XF_BN);
      uint32_t kg = 0;
      for (int t = 0; t < ntl; ++t) {
        const uint32_t a = (uint32_t)t & 1u;
        if (t >= 2) {  // the epilogue has drained accumulator a (tile t - 2)
          mbar_wait(tempty + a, (uint32_t)((t >> 1) - 1) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t acc_addr = tmem + a * XF_BN;
        for (int kb = 0; kb < g.nk; ++kb, ++kg) {
          const uint32_t s = kg % XF_STAGES;
          mbar_wait(full + s, (kg / XF_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(sm + s * XF_STAGE_BYTES), sb = sa + XF_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < MM_BK / 32; ++kk) {
            const uint64_t da = umma_desc_sw128(sa + kk * 32), db = umma_desc_sw128(sb + kk * 32);
            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_addr),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(empty + s))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(tfull + a))
                     : "memory");
      }
    }
  } else if (warp >= XF_EPI_WARP0) {
    const int quad = warp & 3, half = (warp - XF_EPI_WARP0) >> 2;
    const int lrow = quad * 32 + lane, row = m0 + lrow;
    const int stream = half * XF_BM + lrow;
    uint32_t *hist = hist_all + (warp - XF_EPI_WARP0) * 256;
    unsigned long long *mybuf = g.buf + ((size_t)b * XF_STREAMS + stream) * XF_BUF;
    const bool vrow = row < g.q;
    const int32_t nqr = vrow ? __ldg(g.nq + row) : 0;
    // an invalid row appends nothing; with a pilot bound (the k-th smallest key of a
    // point sample, itself >= the k-th smallest key overall) only keys <= it are kept
    unsigned long long tau = !vrow ? 0ull : (g.bound ? g.bound[row] + 1ull : XF_NONE);
    int cnt = 0;
    for (int t = 0; t < ntl; ++t) {
      const uint32_t a = (uint32_t)t & 1u;
      mbar_wait(tfull + a, (uint32_t)(t >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int cbase = (t_begin + t) * XF_BN + half * (XF_BN / 2);
#pragma unroll 1
      for (int c0 = 0; c0 < XF_BN / 2; c0 += 32) {
        // room for this chunk: compact the streams of this warp whose buffer is full
        uint32_t need = __ballot_sync(0xffffffffu, cnt + 32 > XF_BUF);
        while (need) {
          const int L = __ffs(need) - 1;
          need &= need - 1u;
          unsigned long long *bl = reinterpret_cast<unsigned long long *>(
              shfl64(reinterpret_cast<unsigned long long>(mybuf), L));
          const int cl = __shfl_sync(0xffffffffu, cnt, L);
          const unsigned long long th = warp_compact(bl, cl, g.k, hist, lane);
          if (lane == L) {
            tau = th;
            cnt = g.k;
          }
        }
        uint32_t v[32];
        tmem_ld32(tmem + a * XF_BN + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * (XF_BN / 2) + c0), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c0 + 32 == XF_BN / 2) {  // the accumulator is in registers: release it
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty + a);
        }
        const int col0 = cbase + c0;
        const uint32_t gid0 = g.id_offset + (uint32_t)col0;
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4) {
          const int4 xn = __ldg(reinterpret_cast<const int4 *>(g.nx + col0 + j4));
          const int32_t xv[4] = {xn.x, xn.y, xn.z, xn.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = j4 + e;
            const int32_t D = xv[e] + nqr - 2 * (int32_t)v[j];
            const unsigned long long key = ((unsigned long long)(uint32_t)D << 32) | (gid0 + (uint32_t)j);
            if (key < tau && col0 + j < g.n) mybuf[cnt++] = key;
          }
        }
      }
    }
    // end of the range: each stream's k smallest -> part
    __syncwarp();
    uint32_t need = __ballot_sync(0xffffffffu, cnt > g.k);
    while (need) {
      const int L = __ffs(need) - 1;
      need &= need - 1u;
      unsigned long long *bl =
          reinterpret_cast<unsigned long long *>(shfl64(reinterpret_cast<unsigned long long>(mybuf), L));
      const int cl = __shfl_sync(0xffffffffu, cnt, L);
      warp_compact(bl, cl, g.k, hist, lane);
      if (lane == L) cnt = g.k;
    }
    __syncwarp();
    unsigned long long *out = g.part + ((size_t)b * XF_STREAMS + stream) * g.k;
    for (int j = 0; j < g.k; ++j) out[j] = j < cnt ? mybuf[j] : XF_NONE;
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// One CTA per query: the k smallest keys of its 2 G partial lists (block radix select,
// 8-bit digits from the top set bit), ranked, -> idx / dist2 rows in (D, id) order.
constexpr int XM_NT = 512;
// idx == nullptr: the pilot pass -- write the k-th smallest key to bound[row0 + r].
__global__ void __launch_bounds__(XM_NT) k_exact_merge(XfGeom g, int row0, int32_t *idx, int32_t *dist2,
                                                       unsigned long long *bound) {
  __shared__ uint32_t hist[256];
  __shared__ unsigned long long red[XM_NT / 32];
  __shared__ int sh_bin, sh_before, sh_cb;
  __shared__ unsigned long long win[XF_MAX_K];
  __shared__ unsigned wcount;
  const int r = blockIdx.x;  // query of this launch
  const int mb = r / XF_BM, lrow = r % XF_BM, k = g.k;
  const int nlist = 2 * g.G, M = nlist * k;
  auto cand = [&](int c) -> unsigned long long {
    const int l = c / k, j = c - l * k;
    const int seg = l >> 1, half = l & 1;
    const size_t cta = (size_t)seg * g.mt + mb;
    return g.part[(cta * XF_STREAMS + half * XF_BM + lrow) * k + j];
  };
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned long long orr = 0;
  for (int c = tid; c < M; c += XM_NT) {
    const unsigned long long v = cand(c);
    if (v != XF_NONE) orr |= v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) orr |= shfl64(orr, lane ^ o);
  if (lane == 0) red[wid] = orr;
  __syncthreads();
  if (tid == 0) {
    unsigned long long a = 0;
    for (int w = 0; w < XM_NT / 32; ++w) a |= red[w];
    red[0] = a;
  }
  __syncthreads();
  orr = red[0];
  const int top = orr ? 63 - __clzll((long long)orr) : 0;
  unsigned long long prefix = 0, pmask = 0, kth = 0;
  int want = k;
  bool found = false;
  for (int shift = (top >> 3) << 3; shift >= 0 && !found; shift -= 8) {
    for (int i = tid; i < 256; i += XM_NT) hist[i] = 0;
    __syncthreads();
    for (int c = tid; c < M; c += XM_NT) {
      const unsigned long long v = cand(c);
      if (v != XF_NONE && (v & pmask) == prefix) atomicAdd(&hist[(uint32_t)(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      int bin = 255;
      for (int i = 0; i < 256; ++i) {
        if (acc + hist[i] >= (uint32_t)want) {
          bin = i;
          break;
        }
        acc += hist[i];
      }
      sh_bin = bin;
      sh_before = (int)acc;
      sh_cb = (int)hist[bin];
    }
    __syncthreads();
    prefix |= (unsigned long long)sh_bin << shift;
    pmask |= 255ull << shift;
    want -= sh_before;
    if (sh_cb == 1) {
      for (int c = tid; c < M; c += XM_NT) {
        const unsigned long long v = cand(c);
        if (v != XF_NONE && (v & pmask) == prefix) red[0] = v;
      }
      __syncthreads();
      kth = red[0];
      found = true;
    }
    __syncthreads();
  }
  if (!found) kth = prefix;
  if (!idx) {  // pilot: every one of the k keys <= kth is a real point's key
    if (tid == 0) bound[row0 + r] = kth;
    return;
  }
  if (tid == 0) wcount = 0;
  __syncthreads();
  for (int c = tid; c < M; c += XM_NT) {
    const unsigned long long v = cand(c);
    if (v <= kth && v != XF_NONE) {
      const unsigned p = atomicAdd(&wcount, 1u);
      if (p < XF_MAX_K) win[p] = v;
    }
  }
  __syncthreads();
  const int m = min((int)wcount, k);
  for (int j = tid; j < m; j += XM_NT) {
    int rank = 0;
    for (int t = 0; t < m; ++t) rank += win[t] < win[j];
    const unsigned long long v = win[j];
    idx[(size_t)(row0 + r) * k + rank] = (int32_t)(uint32_t)(v & 0xffffffffu);
    dist2[(size_t)(row0 + r) * k + rank] = (int32_t)(v >> 32);
  }
}

int exact_fused_max_k() { return XF_MAX_K; }

// Pilot sample: the first XF_PILOT points (when n >= 4 XF_PILOT) give every query an
// initial threshold, so the streams of the full pass append only keys that can still
// reach the top k (without it every stream fills its buffer from the first tiles).
constexpr int XF_PILOT = 2048;

size_t exact_fused_ws_bytes(int num_sms, int k) {
  return (size_t)num_sms * XF_STREAMS * (XF_BUF + k) * sizeof(unsigned long long) +
         (size_t)num_sms * XF_BM * sizeof(unsigned long long);  // pilot bounds of one launch
}

// Queries in chunks of at most num_sms m-blocks; ws >= exact_fused_ws_bytes(num_sms, k).
// nx must be readable (zero padded) up to round_up(n, 256).
cudaError_t launch_exact_fused(const ExactGeom &e, const int32_t *nq, const int32_t *nx, void *ws, int num_sms,
                               cudaStream_t s) {
  if (e.k < 1 || e.k > XF_MAX_K || e.q < 1) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t err = cudaFuncSetAttribute(k_exact_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XF_SMEM);
    if (err != cudaSuccess) return err;
    attr = true;
  }
  const bool pilot = e.n >= 4 * XF_PILOT && e.k <= XF_PILOT;
  CUtensorMap tx, txp;
  cudaError_t err = make_map(&tx, e.X, e.n, e.d, e.pitch, XF_BN);
  if (err == cudaSuccess && pilot) err = make_map(&txp, e.X, XF_PILOT, e.d, e.pitch, XF_BN);
  if (err != cudaSuccess) return err;
  const int mt_all = (e.q + XF_BM - 1) / XF_BM;
  unsigned long long *buf = static_cast<unsigned long long *>(ws);
  unsigned long long *part = buf + (size_t)num_sms * XF_STREAMS * XF_BUF;
  unsigned long long *bnd = part + (size_t)num_sms * XF_STREAMS * e.k;
  for (int mb0 = 0; mb0 < mt_all; mb0 += num_sms) {
    const int mt = std::min(num_sms, mt_all - mb0);
    const int row0 = mb0 * XF_BM, qn = std::min(e.q - row0, mt * XF_BM);
    CUtensorMap tq;
    err = make_map(&tq, e.Q + (size_t)row0 * e.pitch, qn, e.d, e.pitch, XF_BM);
    if (err != cudaSuccess) return err;
    XfGeom g{};
    g.q = qn;
    g.k = e.k;
    g.mt = mt;
    g.nk = (e.d + MM_BK - 1) / MM_BK;
    g.id_offset = e.id_offset;
    g.nq = nq + row0;
    g.nx = nx;
    g.buf = buf;
    g.part = part;
    if (pilot) {  // the same kernel over the sample, then its k-th key per query
      g.n = XF_PILOT;
      g.nt = XF_PILOT / XF_BN;
      g.G = std::max(1, std::min(g.nt, num_sms / mt));
      g.bound = nullptr;
      k_exact_fused<<<mt * g.G, XF_NT, XF_SMEM, s>>>(tq, txp, g);
      k_exact_merge<<<qn, XM_NT, 0, s>>>(g, 0, nullptr, nullptr, bnd);
    }
    g.n = e.n;
    g.nt = (e.n + XF_BN - 1) / XF_BN;
    g.G = std::max(1, std::min(g.nt, num_sms / mt));
    g.bound = pilot ? bnd : nullptr;
    k_exact_fused<<<mt * g.G, XF_NT, XF_SMEM, s>>>(tq, tx, g);
    k_exact_merge<<<qn, XM_NT, 0, s>>>(g, row0, e.idx, e.dist2, nullptr);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

}  // namespace aknn
