// exact_fused.cu -- the exact comparison pass (row a10; "compute all distances,
// then sort") as ONE persistent tensor-core kernel whose epilogue keeps each query's
// running top-k candidates, so the [q][n] distance matrix is never written.
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
//   warp 0 lane 0   TMA producer.  d <= 1152 (QRES): the CTA's 128 query rows are
//                   loaded into shared memory ONCE (nk k-blocks of 128 x 128 B), then
//                   only X k-blocks (256 x 128 B) stream through a ring of 2-6 stages;
//                   wider rows stream Q and X k-blocks together through 4 stages
//   warp 1          TMEM owner (512 columns = two 128 x 256 int32 accumulators) and,
//                   lane 0, the MMA issuer: 4 x tcgen05.mma kind::i8 (K = 32 B) per
//                   k-block into accumulator t & 1, commit -> stage free / tile done
//   warps 4..11     epilogue (TMEM lane quadrant = warp % 4, column half = (warp-4)/4):
//                   thread = one (query row, column half) STREAM with a candidate
//                   buffer (global, L2-resident) and a threshold tau; a key < tau is
//                   appended.  tau starts at the pilot bound (below) and, when a buffer
//                   fills, the warp compacts it to its k smallest (warp radix select,
//                   tau = the k-th).  The accumulator is released as soon as its last
//                   chunk is in registers, so the MMAs of tile t+2 overlap.
//   end             each stream leaves its candidates (unsorted) and their count;
//                   k_exact_merge selects each query's k smallest of all its streams'
//                   candidates (block radix select in shared memory) and sorts them.
// Pilot: for n >= 4 * 2048 the same two kernels first run over the first 2048 points
// (8192 when n >= 65536); each query's k-th smallest key there bounds its k-th smallest
// key overall, so the full pass appends only keys that can still reach the top k.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace aknn {

constexpr int XF_BM = 128, XF_BN = 256;
constexpr int XF_EPI_WARP0 = 4, XF_EPI_WARPS = 8, XF_NT = 32 * (XF_EPI_WARP0 + XF_EPI_WARPS);
constexpr uint32_t XF_A_BYTES = XF_BM * MM_BK, XF_B_BYTES = XF_BN * MM_BK;
constexpr int XF_CAP = 512;             // compaction threshold of a stream's buffer
constexpr int XF_BUF = XF_CAP + 32;     // + one 32-column chunk of slack
constexpr int XF_E = XF_BUF / 32;       // keys per lane in a warp compaction
constexpr int XF_MAX_K = 128;
constexpr int XF_STREAMS = 2 * XF_BM;   // streams per CTA: (column half, row)
constexpr int XF_PILOT = 2048, XF_PILOT_BIG = 8192;  // pilot samples: n >= 4x / 8x them
constexpr size_t XF_SMEM_MAX = 227 * 1024;
constexpr size_t XF_HIST_BYTES = (size_t)XF_EPI_WARPS * 256 * 4;  // static: radix histograms
constexpr size_t XF_FIXED = 1024 /*align*/ + 256 /*barriers*/;
constexpr int XF_QRES_MAXK = 9;         // Q resident for d <= 9 * 128
constexpr unsigned long long XF_NONE = ~0ull;

struct XfGeom {
  int q, n, k;          // queries of this launch, points, neighbours
  int mt, G, nt;        // m-blocks, point-tile ranges per m-block, point tiles
  int nk;               // 128-byte k-blocks of d
  int nstages;          // ring stages
  uint32_t id_offset;
  const int32_t *nq;    // [q] ||q||^2 of this launch's queries
  const int32_t *nx;    // [>= nt * 256] ||x_i||^2 (zero padded)
  unsigned long long *buf;   // [grid][XF_STREAMS][XF_BUF] candidate keys
  uint32_t *pcnt;            // [grid][XF_STREAMS] candidates per stream
  const unsigned long long *bound;  // [q] initial per-query threshold (the pilot's k-th key), or null
  unsigned long long *qbound;       // [q] shared per-query bound: the smallest k-th key any stream
                                    // of the query has compacted to (atomicMin), reset to ~0
  int first_cap;                    // a stream's first compaction when it holds more keys
};

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((unsigned long long)hi << 32) | lo;
}

// Radix digit start: the highest 8-bit digit in which the valid keys differ (the
// common higher bits are fixed at once, so no pass piles every key into one bin).
__device__ __forceinline__ int radix_top_shift(unsigned long long andk, unsigned long long ork) {
  const unsigned long long diff = andk ^ ork;
  return diff ? ((63 - __clzll((long long)diff)) >> 3) << 3 : -8;
}

// Warp-cooperative: the c keys in b[0..c) (unique), k <= c.  Finds the k-th smallest by
// an 8-bit radix select (histogram `hist`: 256 words of this warp's shared memory,
// warp-aggregated increments), moves the k smallest to b[0..k) (any order) and returns
// the k-th smallest.
__device__ unsigned long long warp_compact(unsigned long long *b, int c, int k, uint32_t *hist, int lane) {
  unsigned long long key[XF_E];
  unsigned long long orr = 0, andk = XF_NONE;
#pragma unroll
  for (int e = 0; e < XF_E; ++e) {
    const int i = lane + 32 * e;
    key[e] = i < c ? b[i] : XF_NONE;
    if (i < c) {
      orr |= key[e];
      andk &= key[e];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    orr |= shfl64(orr, lane ^ o);
    andk &= shfl64(andk, lane ^ o);
  }
  int shift = radix_top_shift(andk, orr);
  unsigned long long pmask = shift >= 0 ? ~((1ull << (shift + 8)) - 1ull) : XF_NONE;
  unsigned long long prefix = andk & pmask, kth = prefix;
  int want = k;
  for (; shift >= 0; shift -= 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) hist[lane * 8 + i] = 0;
    __syncwarp();
#pragma unroll
    for (int e = 0; e < XF_E; ++e) {
      const bool v = key[e] != XF_NONE && (key[e] & pmask) == prefix;
      const uint32_t bin = v ? (uint32_t)(key[e] >> shift) & 255u : 256u;
      const uint32_t m = __match_any_sync(0xffffffffu, bin);
      if (v && lane == __ffs(m) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(m));
    }
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
    kth = prefix;
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
      break;
    }
    __syncwarp();
  }
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

template <bool QRES>
__global__ void __launch_bounds__(XF_NT, 1)
    k_exact_fused(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                  const __grid_constant__ XfGeom g) {
  __shared__ uint32_t hist_all[XF_EPI_WARPS][256];
  const int b = blockIdx.x, mb = b % g.mt, seg = b / g.mt;
  const int t_begin = (int)((long long)seg * g.nt / g.G), t_end = (int)((long long)(seg + 1) * g.nt / g.G);
  const int ntl = t_end - t_begin;
  const int m0 = mb * XF_BM;
  const uint32_t stage_bytes = QRES ? XF_B_BYTES : XF_A_BYTES + XF_B_BYTES;
  const uint32_t qres_bytes = QRES ? (uint32_t)g.nk * XF_A_BYTES : 0u;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char *ring = sm + qres_bytes;  // QRES: [Q k-blocks][ring]; else [ring of Q|X]
  uint64_t *full = reinterpret_cast<uint64_t *>(ring + (size_t)g.nstages * stage_bytes);
  uint64_t *empty = full + 8;
  uint64_t *tfull = empty + 8;   // [2]
  uint64_t *tempty = tfull + 2;  // [2]
  uint64_t *qfull = tempty + 2;
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(qfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t S = (uint32_t)g.nstages;

  if (warp == 0 && lane == 0) {
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, XF_EPI_WARPS);
    }
    mbar_init(qfull, 1);
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
      if (QRES) {     // the CTA's query rows, once
        mbar_expect_tx(qfull, qres_bytes);
        for (int kb = 0; kb < g.nk; ++kb) tma_load_2d(sm + (size_t)kb * XF_A_BYTES, &tmQ, qfull, kb * MM_BK, m0);
      }
      uint32_t kg = 0;
      for (int t = 0; t < ntl; ++t) {
        const int n0 = (t_begin + t) * XF_BN;
        for (int kb = 0; kb < g.nk; ++kb, ++kg) {
          const uint32_t s = kg % S;
          if (kg >= S) mbar_wait(empty + s, ((kg / S) - 1) & 1);
          unsigned char *sa = ring + s * stage_bytes;
          mbar_expect_tx(full + s, stage_bytes);
          if (QRES) {
            tma_load_2d(sa, &tmX, full + s, kb * MM_BK, n0);
          } else {
            tma_load_2d(sa, &tmQ, full + s, kb * MM_BK, m0);
            tma_load_2d(sa + XF_A_BYTES, &tmX, full + s, kb * MM_BK, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = umma_idesc_u8(XF_BM, XF_BN);
      if (QRES) mbar_wait(qfull, 0);
      uint32_t kg = 0;
      for (int t = 0; t < ntl; ++t) {
        const uint32_t a = (uint32_t)t & 1u;
        if (t >= 2) {  // the epilogue has drained accumulator a (tile t - 2)
          mbar_wait(tempty + a, (uint32_t)((t >> 1) - 1) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t acc_addr = tmem + a * XF_BN;
        for (int kb = 0; kb < g.nk; ++kb, ++kg) {
          const uint32_t s = kg % S;
          mbar_wait(full + s, (kg / S) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t st = smem_u32(ring + s * stage_bytes);
          const uint32_t sa = QRES ? smem_u32(sm + (size_t)kb * XF_A_BYTES) : st;
          const uint32_t sb = QRES ? st : st + XF_A_BYTES;
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
    uint32_t *hist = hist_all[warp - XF_EPI_WARP0];
    unsigned long long *mybuf = g.buf + ((size_t)b * XF_STREAMS + stream) * XF_BUF;
    const bool vrow = row < g.q;
    const int32_t nqr = vrow ? __ldg(g.nq + row) : 0;
    // an invalid row appends nothing; with a pilot bound (the k-th smallest key of a
    // point sample, itself >= the k-th smallest key overall) only keys <= it are kept
    unsigned long long tau = !vrow ? 0ull : (g.bound ? g.bound[row] + 1ull : XF_NONE);
    int cnt = 0, lim = g.first_cap + 32;  // the first compaction comes early (a tight tau soon)
    for (int t = 0; t < ntl; ++t) {
      const uint32_t a = (uint32_t)t & 1u;
      // every stream's k-th key bounds the query's k-th key: adopt the query's best so far
      if (vrow && t > 0) {
        const unsigned long long qb = __ldcg(g.qbound + row);
        tau = qb < tau ? qb + 1ull : tau;
      }
      mbar_wait(tfull + a, (uint32_t)(t >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int cbase = (t_begin + t) * XF_BN + half * (XF_BN / 2);
#pragma unroll 1
      for (int c0 = 0; c0 < XF_BN / 2; c0 += 32) {
        // room for this chunk: compact the streams of this warp whose buffer is full
        uint32_t need = __ballot_sync(0xffffffffu, cnt + 32 > lim);
        while (need) {
          const int L = __ffs(need) - 1;
          need &= need - 1u;
          unsigned long long *bl = reinterpret_cast<unsigned long long *>(
              shfl64(reinterpret_cast<unsigned long long>(mybuf), L));
          const int cl = __shfl_sync(0xffffffffu, cnt, L);
          const unsigned long long th = warp_compact(bl, cl, g.k, hist, lane);
          if (lane == L) {
            tau = th;  // all kept keys are <= th; keys below it may still enter
            cnt = g.k;
            lim = XF_BUF;
            atomicMin(g.qbound + row, th);
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
    g.pcnt[(size_t)b * XF_STREAMS + stream] = (uint32_t)cnt;  // unsorted candidates for the merge
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// One CTA per query: the k smallest of the candidates of its 2 G streams.  The
// streams' counts are scanned into offsets; when they fit (cap_keys, sized by the host
// from the expected count) the candidates are copied into shared memory once, warp by
// stream; otherwise every pass re-reads them from the (L2-resident) stream buffers.
// Selection: 8-bit radix select from the highest differing digit, warp-aggregated
// histogram increments, the bin found by a warp scan.  The k winners are ranked.
// idx == nullptr: the pilot -- write the k-th smallest key to bound[row0 + r].
constexpr int XM_NT = 512, XM_NW = XM_NT / 32;
constexpr int XM_MAX_STREAMS = 2 * 160;
constexpr size_t XM_SMEM_MAX = 200 * 1024;

__global__ void __launch_bounds__(XM_NT) k_exact_merge(XfGeom g, int row0, int32_t *idx, int32_t *dist2,
                                                       unsigned long long *bound, int cap_keys) {
  extern __shared__ unsigned long long skeys[];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t soff[XM_MAX_STREAMS + 1];
  __shared__ unsigned long long red_o[XM_NW], red_a[XM_NW];
  __shared__ int sh_bin, sh_before, sh_cb;
  __shared__ unsigned long long sh_kth;
  __shared__ unsigned long long win[XF_MAX_K];
  __shared__ unsigned wcount;
  const int r = blockIdx.x;  // query of this launch
  const int mb = r / XF_BM, lrow = r % XF_BM, k = g.k;
  const int nl = 2 * g.G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  auto stream_base = [&](int l) -> size_t {
    const int seg = l >> 1, half = l & 1;
    return (((size_t)seg * g.mt + mb) * XF_STREAMS + half * XF_BM + lrow);
  };
  if (wid == 0) {  // offsets of the streams' candidates: warp scan
    uint32_t carry = 0;
    for (int l0 = 0; l0 < nl; l0 += 32) {
      const int l = l0 + lane;
      const uint32_t c = l < nl ? g.pcnt[stream_base(l)] : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (l < nl) soff[l] = carry + inc - c;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) soff[nl] = carry;
  }
  __syncthreads();
  const int M = (int)soff[nl];
  const bool in_smem = M <= cap_keys;
  if (in_smem)
    for (int l = wid; l < nl; l += XM_NW) {
      const unsigned long long *src = g.buf + stream_base(l) * XF_BUF;
      const int c = (int)(soff[l + 1] - soff[l]);
      for (int j = lane; j < c; j += 32) skeys[soff[l] + j] = src[j];
    }
  __syncthreads();
  // fn(key, valid) on every candidate, every lane of a warp in lockstep (full-warp match)
  auto visit = [&](auto &&fn) {
    if (in_smem) {
      for (int c0 = 0; c0 < M; c0 += XM_NT) {
        const int c = c0 + tid;
        const bool v = c < M;
        fn(v ? skeys[c] : XF_NONE, v);
      }
    } else {
      for (int l = wid; l < nl; l += XM_NW) {
        const unsigned long long *src = g.buf + stream_base(l) * XF_BUF;
        const int c = (int)(soff[l + 1] - soff[l]);
        for (int j0 = 0; j0 < c; j0 += 32) {
          const int j = j0 + lane;
          const bool v = j < c;
          fn(v ? src[j] : XF_NONE, v);
        }
      }
    }
  };
  // common high bits of all candidates
  unsigned long long orr = 0, andk = XF_NONE;
  visit([&](unsigned long long v, bool ok) {
    if (ok) {
      orr |= v;
      andk &= v;
    }
  });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    orr |= shfl64(orr, lane ^ o);
    andk &= shfl64(andk, lane ^ o);
  }
  if (lane == 0) {
    red_o[wid] = orr;
    red_a[wid] = andk;
  }
  __syncthreads();
  orr = 0;
  andk = XF_NONE;
  for (int w = 0; w < XM_NW; ++w) {
    orr |= red_o[w];
    andk &= red_a[w];
  }
  int shift = radix_top_shift(andk, orr);
  unsigned long long pmask = shift >= 0 ? ~((1ull << (shift + 8)) - 1ull) : XF_NONE;
  unsigned long long prefix = andk & pmask, kth = prefix;
  int want = k;
  for (; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += XM_NT) hist[i] = 0;
    __syncthreads();
    visit([&](unsigned long long v, bool ok) {
      ok = ok && (v & pmask) == prefix;
      const uint32_t bin = ok ? (uint32_t)(v >> shift) & 255u : 256u;
      const uint32_t m = __match_any_sync(0xffffffffu, bin);
      if (ok && lane == __ffs(m) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(m));
    });
    __syncthreads();
    if (wid == 0) {  // the bin holding the want-th key: warp scan over 8 bins per lane
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
      if (exc < (uint32_t)want && (uint32_t)want <= inc) {
        uint32_t acc = exc;
        int bin = -1;
        for (int i = 0; i < 8 && bin < 0; ++i) {
          if (acc + h[i] >= (uint32_t)want) {
            bin = lane * 8 + i;
            sh_bin = bin;
            sh_before = (int)acc;
            sh_cb = (int)h[i];
          }
          acc += h[i];
        }
      }
    }
    __syncthreads();
    prefix |= (unsigned long long)sh_bin << shift;
    pmask |= 255ull << shift;
    want -= sh_before;
    kth = prefix;
    if (sh_cb == 1) {  // unique: locate it
      visit([&](unsigned long long v, bool ok) {
        if (ok && (v & pmask) == prefix) sh_kth = v;
      });
      __syncthreads();
      kth = sh_kth;
      break;
    }
    __syncthreads();
  }
  if (!idx) {  // pilot: every one of the k keys <= kth is a real point's key
    if (tid == 0) bound[row0 + r] = kth;
    return;
  }
  if (tid == 0) wcount = 0;
  __syncthreads();
  visit([&](unsigned long long v, bool ok) {
    if (ok && v <= kth) {
      const unsigned p = atomicAdd(&wcount, 1u);
      if (p < XF_MAX_K) win[p] = v;
    }
  });
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

size_t exact_fused_ws_bytes(int num_sms, int k) {
  (void)k;
  return (size_t)num_sms * XF_STREAMS * XF_BUF * sizeof(unsigned long long) +  // candidates
         (size_t)num_sms * XF_STREAMS * sizeof(uint32_t) +                     // their counts
         2 * (size_t)num_sms * XF_BM * sizeof(unsigned long long);              // pilot + shared bounds
}

// Queries in chunks of at most num_sms m-blocks; ws >= exact_fused_ws_bytes(num_sms, k).
// nx must be readable (zero padded) up to round_up(n, 256).
cudaError_t launch_exact_fused(const ExactGeom &e, const int32_t *nq, const int32_t *nx, void *ws, int num_sms,
                               cudaStream_t s) {
  if (e.k < 1 || e.k > XF_MAX_K || e.q < 1 || 2 * num_sms > XM_MAX_STREAMS) return cudaErrorInvalidValue;
  const int nk = (e.d + MM_BK - 1) / MM_BK;
  const bool qres = nk <= XF_QRES_MAXK;
  const size_t stage = qres ? XF_B_BYTES : XF_A_BYTES + XF_B_BYTES;
  const size_t dyn_max = XF_SMEM_MAX - XF_HIST_BYTES;  // the histograms are static shared memory
  const size_t avail = dyn_max - XF_FIXED - (qres ? (size_t)nk * XF_A_BYTES : 0);
  const int nst = (int)std::min<size_t>(qres ? 6 : 4, avail / stage);
  if (nst < 2) return cudaErrorInvalidValue;
  const size_t smem = XF_FIXED + (qres ? (size_t)nk * XF_A_BYTES : 0) + (size_t)nst * stage;
  static bool attr = false;
  if (!attr) {
    cudaError_t err = cudaFuncSetAttribute(k_exact_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(k_exact_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn_max);
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(k_exact_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XM_SMEM_MAX);
    if (err != cudaSuccess) return err;
    attr = true;
  }
  // pilot sample: the larger one when n allows (the full pass then appends ~ k n / S
  // candidates per query instead of ~ k n / 2048)
  const int S = e.n >= 8 * XF_PILOT_BIG ? XF_PILOT_BIG : XF_PILOT;
  static const int pilot_env = [] {  // AKNN_EXACT_PILOT=0 / 1 forces it off / on (A/B)
    const char *v = getenv("AKNN_EXACT_PILOT");
    return v && v[0] ? atoi(v) : -1;
  }();
  const bool pilot = (pilot_env < 0 ? e.n >= 4 * S : pilot_env == 1 && e.n >= 2 * S) && e.k <= S;
  CUtensorMap tx, txp;
  cudaError_t err = make_map(&tx, e.X, e.n, e.d, e.pitch, XF_BN);
  if (err == cudaSuccess && pilot) err = make_map(&txp, e.X, S, e.d, e.pitch, XF_BN);
  if (err != cudaSuccess) return err;
  const int mt_all = (e.q + XF_BM - 1) / XF_BM;
  unsigned long long *buf = static_cast<unsigned long long *>(ws);
  uint32_t *pcnt = reinterpret_cast<uint32_t *>(buf + (size_t)num_sms * XF_STREAMS * XF_BUF);
  unsigned long long *bnd = reinterpret_cast<unsigned long long *>(pcnt + (size_t)num_sms * XF_STREAMS);
  unsigned long long *qbnd = bnd + (size_t)num_sms * XF_BM;
  // merge shared memory: 4x the expected candidates per query (capped); a query with
  // more takes the re-reading path
  auto merge_smem = [&](size_t expect) {
    size_t b = std::max<size_t>(16 * 1024, 4 * expect * sizeof(unsigned long long));
    return std::min(b, XM_SMEM_MAX);
  };
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
    g.nk = nk;
    g.nstages = nst;
    g.id_offset = e.id_offset;
    g.nq = nq + row0;
    g.nx = nx;
    g.buf = buf;
    g.pcnt = pcnt;
    g.qbound = qbnd;
    g.first_cap = std::max(128, 2 * e.k);
    auto run = [&](const CUtensorMap &txm) {
      if (qres)
        k_exact_fused<true><<<mt * g.G, XF_NT, smem, s>>>(tq, txm, g);
      else
        k_exact_fused<false><<<mt * g.G, XF_NT, smem, s>>>(tq, txm, g);
    };
    if (pilot) {  // the same kernels over the sample, then its k-th key per query
      g.n = S;
      g.nt = S / XF_BN;
      g.G = std::max(1, std::min(g.nt, num_sms / mt));
      g.bound = nullptr;
      err = cudaMemsetAsync(qbnd, 0xFF, sizeof(unsigned long long) * (size_t)qn, s);
      if (err != cudaSuccess) return err;
      run(txp);
      // every sample key is a candidate (no threshold yet): exactly S of them
      const size_t ms = std::min(XM_SMEM_MAX, std::max<size_t>(16 * 1024, (size_t)S * sizeof(unsigned long long)));
      k_exact_merge<<<qn, XM_NT, ms, s>>>(g, 0, nullptr, nullptr, bnd, (int)(ms / 8));
    }
    g.n = e.n;
    g.nt = (e.n + XF_BN - 1) / XF_BN;
    g.G = std::max(1, std::min(g.nt, num_sms / mt));
    g.bound = pilot ? bnd : nullptr;
    err = cudaMemsetAsync(qbnd, 0xFF, sizeof(unsigned long long) * (size_t)qn, s);
    if (err != cudaSuccess) return err;
    run(tx);
    const size_t ms = merge_smem(pilot ? (size_t)e.k * (size_t)e.n / (size_t)S + (size_t)e.k
                                       : (size_t)2 * g.G * XF_BUF);
    k_exact_merge<<<qn, XM_NT, ms, s>>>(g, row0, e.idx, e.dist2, nullptr, (int)(ms / 8));
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

}  // namespace aknn
