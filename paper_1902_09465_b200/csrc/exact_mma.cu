// exact_mma.cu -- the exact comparison pass (P:98 brute force) on the 5th-generation
// tensor cores: D(q, i) = ||x_i||^2 + ||q||^2 - 2 <x_i, q>, with the inner products
// an unsigned-8-bit contraction accumulated exactly in int32 (tcgen05.mma kind::i8,
// u8 x u8 -> s32; d * 255^2 < 2^31 for d <= 33025, and so is every D).
//
// One CTA per 128-query x 256-point tile, K in 128-byte blocks:
//   warp 0 lane 0   TMA producer: cp.async.bulk.tensor 2-D loads of the query tile
//                   (128 x 128 B) and the point tile (256 x 128 B) into a 4-stage
//                   ring, 128-byte swizzled, completion on mbarriers (expect_tx)
//   warp 1 lane 0   MMA issuer: 4 x tcgen05.mma (K = 32 bytes each) per stage into a
//                   128 x 256 int32 accumulator in TMEM (256 columns); tcgen05.commit
//                   frees the stage, the last one signals the epilogue
//   warp 2          TMEM allocator (tcgen05.alloc / dealloc, 256 columns)
//   warps 4-7       epilogue: tcgen05.ld 32x32b.x32 (lane = query row, 32 points per
//                   load), D = nx + nq - 2 dot, int32 stores
// The distances then go through the block radix top-k of exact_kernels.cu.
//
// The same tile kernel, with another epilogue (EpiFallback), computes the round
// loop's exact fallbacks (row a4) when they are dense: under the footnote-2
// radius nearly every arm of a query reaches 2T >= d and goes exact in the same
// round, which as per-pair row streams re-reads n*d bytes per query from L2.
#include <cuda.h>

#include "internal.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace aknn {

constexpr int MM_BM = 128, MM_BN = 256, MM_STAGES = 4, MM_NT = 256;
constexpr uint32_t MM_A_BYTES = MM_BM * MM_BK, MM_B_BYTES = MM_BN * MM_BK;
constexpr uint32_t MM_STAGE_BYTES = MM_A_BYTES + MM_B_BYTES;
constexpr size_t MM_SMEM = (size_t)MM_STAGES * MM_STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr uint32_t MM_TMEM_COLS = 256;

// Epilogue of the exact comparison pass: D = ||x||^2 + ||q||^2 - 2 dot, int32 rows.
struct EpiDistances {
  const int32_t *nq, *nx;
  int32_t *D;
  int64_t ldd;
  int q, n;
  __device__ __forceinline__ int rows() const { return q; }
  __device__ __forceinline__ bool tile_active(int, int) const { return true; }
  __device__ __forceinline__ void store(int row, int col0, const uint32_t (&v)[32]) const {
    if (row >= q) return;
    const int32_t nqr = __ldg(nq + row);
    int32_t *drow = D + (size_t)row * ldd + col0;
    if (col0 + 32 <= n) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const int4 xn = __ldg(reinterpret_cast<const int4 *>(nx + col0 + j));
        int4 o;
        o.x = xn.x + nqr - 2 * (int32_t)v[j + 0];
        o.y = xn.y + nqr - 2 * (int32_t)v[j + 1];
        o.z = xn.z + nqr - 2 * (int32_t)v[j + 2];
        o.w = xn.w + nqr - 2 * (int32_t)v[j + 3];
        *reinterpret_cast<int4 *>(drow + j) = o;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < n; ++j) drow[j] = __ldg(nx + col0 + j) + nqr - 2 * (int32_t)v[j];
    }
  }
};

// Epilogue of the round loop's exact fallbacks (row a4): for every pair of
// the tile whose action byte is ACT_EXACT, S = sum_j (x_j - q_j)^2 = D exactly and
// the level becomes exact.  k_filter counts the fallbacks per 128 x 256 tile; tiles
// with fewer than g.xmin of them exit before touching TMEM (k_scatter listed their
// pairs for the row-stream path instead); every CTA clears its count for the next round.
struct EpiFallback {
  Geom g;
  __device__ __forceinline__ int rows() const { return g.q; }
  __device__ __forceinline__ bool tile_active(int m0, int n0) const {
    __shared__ uint32_t sflag;
    uint32_t *f = g.xflags + (size_t)(m0 / MM_BM) * g.xf_cols + (n0 / MM_BN);
    if (threadIdx.x == 0) {
      sflag = *f;
      if (sflag) *f = 0u;
    }
    __syncthreads();
    return sflag >= g.xmin;
  }
  __device__ __forceinline__ void store(int row, int col0, const uint32_t (&v)[32]) const {
    if (row >= g.q || col0 >= g.n || g.qs[row].done) return;
    const int32_t nqr = __ldg(g.nq + row);
    const size_t o = (size_t)row * g.npad + col0;
    uint8_t a[32];
    if (col0 + 32 <= g.npad) {
      const uint4 a0 = *reinterpret_cast<const uint4 *>(g.act + o);
      const uint4 a1 = *reinterpret_cast<const uint4 *>(g.act + o + 16);
      memcpy(a, &a0, 16);
      memcpy(a + 16, &a1, 16);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) a[j] = (col0 + j < g.npad) ? g.act[o + j] : (uint8_t)0;
    }
    int32_t *srow = g.S + o;
    uint8_t *lrow = g.lvl + o;
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += 4) {
      const bool all = a[j0] == ACT_EXACT && a[j0 + 1] == ACT_EXACT && a[j0 + 2] == ACT_EXACT &&
                       a[j0 + 3] == ACT_EXACT && col0 + j0 + 4 <= g.n;
      if (all) {
        const int4 xn = __ldg(reinterpret_cast<const int4 *>(g.nx + col0 + j0));
        int4 s4;
        s4.x = xn.x + nqr - 2 * (int32_t)v[j0 + 0];
        s4.y = xn.y + nqr - 2 * (int32_t)v[j0 + 1];
        s4.z = xn.z + nqr - 2 * (int32_t)v[j0 + 2];
        s4.w = xn.w + nqr - 2 * (int32_t)v[j0 + 3];
        *reinterpret_cast<int4 *>(srow + j0) = s4;
        uint32_t *l4 = reinterpret_cast<uint32_t *>(lrow + j0);
        *l4 |= 0x80808080u;  // 4 x lvl_to_exact
      } else {
#pragma unroll
        for (int j = j0; j < j0 + 4; ++j)
          if (a[j] == ACT_EXACT && col0 + j < g.n) {
            srow[j] = __ldg(g.nx + col0 + j) + nqr - 2 * (int32_t)v[j];
            lrow[j] = lvl_to_exact(lrow[j]);
          }
      }
    }
  }
};

template <class Epi>
__global__ void __launch_bounds__(MM_NT, 1)
    k_mma_tiles(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX, int d,
                const __grid_constant__ Epi epi) {
  // query tiles fastest: the CTAs resident at once share each point tile through L2,
  // so X (or the level's w planes) streams from HBM about once per launch
  const int mt = (epi.rows() + MM_BM - 1) / MM_BM;
  const int m0 = (int)(blockIdx.x % mt) * MM_BM, n0 = (int)(blockIdx.x / mt) * MM_BN;
  if (!epi.tile_active(m0, n0)) return;  // uniform across the CTA
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + MM_STAGES * MM_STAGE_BYTES);
  uint64_t *empty = full + MM_STAGES;
  uint64_t *tfull = empty + MM_STAGES;
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (d + MM_BK - 1) / MM_BK;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < MM_STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                 "n"(MM_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % MM_STAGES;
        if (kb >= MM_STAGES) mbar_wait(empty + s, ((kb / MM_STAGES) - 1) & 1);
        unsigned char *sa = sm + s * MM_STAGE_BYTES;
        mbar_expect_tx(full + s, MM_STAGE_BYTES);
        tma_load_2d(sa, &tmQ, full + s, kb * MM_BK, m0);
        tma_load_2d(sa + MM_A_BYTES, &tmX, full + s, kb * MM_BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = umma_idesc_u8(MM_BM, MM_BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % MM_STAGES;
        mbar_wait(full + s, (kb / MM_STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t sa = smem_u32(sm + s * MM_STAGE_BYTES), sb = sa + MM_A_BYTES;
#pragma unroll
        for (int kk = 0; kk < MM_BK / 32; ++kk) {
          const uint64_t da = umma_desc_sw128(sa + kk * 32), db = umma_desc_sw128(sb + kk * 32);
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(empty + s))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(tfull))
                   : "memory");
    }
  } else if (warp >= 4) {  // epilogue: TMEM lanes 32*(warp-4) .. +31 = query rows
    const int quad = warp - 4;
    mbar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = m0 + quad * 32 + lane;
#pragma unroll 1
    for (int c0 = 0; c0 < MM_BN; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
            "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
            "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      epi.store(row, n0 + c0, v);
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(MM_TMEM_COLS));
  }
}

// ||row||^2 of each of `rows` uint8 rows (pitch bytes, zero padded): warp per row.
__global__ void k_row_norms(const uint8_t *A, int64_t pitch, int rows, int32_t *out) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rows) return;
  const uint4 *r = reinterpret_cast<const uint4 *>(A + (size_t)w * pitch);
  uint32_t acc = 0;
  for (int v = lane; v < (int)(pitch >> 4); v += 32) {
    const uint4 a = __ldg(r + v);
    acc = __dp4a(a.x, a.x, acc);
    acc = __dp4a(a.y, a.y, acc);
    acc = __dp4a(a.z, a.z, acc);
    acc = __dp4a(a.w, a.w, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[w] = (int32_t)acc;
}

cudaError_t launch_row_norms(const uint8_t *A, int64_t pitch, int rows, int32_t *out, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  k_row_norms<<<(rows + 7) / 8, 256, 0, s>>>(A, pitch, rows, out);
  return cudaGetLastError();
}

// --- TMA descriptors through the driver entry point (no libcuda link) -------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

cudaError_t make_map(CUtensorMap *m, const uint8_t *base, int rows, int d, int64_t pitch, int box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !p) return cudaErrorNotSupported;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch};
  const cuuint32_t box[2] = {(cuuint32_t)MM_BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_exact_mma(const ExactGeom &e, const int32_t *nq, const int32_t *nx, cudaStream_t s) {
  CUtensorMap tq, tx;
  cudaError_t err = make_map(&tq, e.Q, e.q, e.d, e.pitch, MM_BM);
  if (err != cudaSuccess) return err;
  err = make_map(&tx, e.X, e.n, e.d, e.pitch, MM_BN);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_mma_tiles<EpiDistances>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MM_SMEM);
  if (err != cudaSuccess) return err;
  const EpiDistances epi{nq, nx, e.D, e.npad, e.q, e.n};
  const unsigned grid = (unsigned)(((e.q + MM_BM - 1) / MM_BM) * ((e.n + MM_BN - 1) / MM_BN));
  k_mma_tiles<EpiDistances><<<grid, MM_NT, MM_SMEM, s>>>(tq, tx, e.d, epi);
  return cudaGetLastError();
}

// Exact fallbacks of one round on the tensor cores (g.exact_mma): every tile of the
// (batch query x point) grid that k_filter flagged computes its distances and writes
// them into S for the pairs whose action byte is ACT_EXACT.
cudaError_t launch_exact_fallback_mma(const Geom &g, cudaStream_t s) {
  CUtensorMap tq, tx;
  cudaError_t err = make_map(&tq, g.Q, g.q, g.d, g.pitch, MM_BM);
  if (err != cudaSuccess) return err;
  err = make_map(&tx, g.X, g.n, g.d, g.pitch, MM_BN);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_mma_tiles<EpiFallback>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MM_SMEM);
  if (err != cudaSuccess) return err;
  const EpiFallback epi{g};
  const unsigned grid = (unsigned)(((g.q + MM_BM - 1) / MM_BM) * ((g.n + MM_BN - 1) / MM_BN));
  k_mma_tiles<EpiFallback><<<grid, MM_NT, MM_SMEM, s>>>(tq, tx, g.d, epi);
  return cudaGetLastError();
}

int exact_tile_rows() { return MM_BM; }
int exact_tile_cols() { return MM_BN; }


// ===========================================================================
// Query-independent draws on the tensor cores.
//
// With shared draws every query sees the same s = 2^c coordinates j_1..j_s of point i
// at level c.  With w_j their multiplicities, the level's update of pair (q, i) is
//   sum_t (x_ij_t - q_j_t)^2 = sum_j w_j x_ij^2 - 2 sum_j (w_j x_ij) q_j + sum_j w_j q_j^2,
// i.e. two integer GEMMs over K = d for a (query x point) tile: Q . (w o x) and
// (Q o Q) . w.  Operands are unsigned bytes (kind::i8): w o x <= 255 w splits into
// two byte planes, q^2 <= 65025 into two, w (<= 255, else the point is left to the
// lists) is one: four tcgen05.mma accumulators of 128 x 128 int32 fill the 512 TMEM
// columns.  Exact in int32 (every partial sum < 2^31), so S is bit-identical to the
// per-draw sums.  k_build_w writes the planes of the round's level (one warp per
// point: Philox once per point, not per pair); k_level_mma runs the 128 x 128 tiles
// that k_filter found holding >= g.lmin pairs at that level; its epilogue updates
// exactly those pairs (S += wa + B - 2 C, level c -> c + 1).
constexpr int LM_BM = 128, LM_BN = 128, LM_STAGES = 2;
constexpr uint32_t LM_PLANE = LM_BM * MM_BK;                 // 16 KB per operand plane
constexpr uint32_t LM_STAGE_BYTES = 6 * LM_PLANE;            // Q, Q2lo, Q2hi | Wx0, Wx1, Wc
constexpr size_t LM_SMEM = (size_t)LM_STAGES * LM_STAGE_BYTES + 1024 + 256;
constexpr uint32_t LM_TMEM_COLS = 512;

__global__ void k_q2_planes(Geom g) {  // q_j^2 as two byte planes (low, high)
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x, tot = (size_t)g.q * g.pitch;
  if (t >= tot) return;
  const uint32_t v = g.Q[t], sq = v * v;
  g.q2lo[t] = (uint8_t)(sq & 255u);
  g.q2hi[t] = (uint8_t)(sq >> 8);
}

// The level's planes for every point: w_j (multiplicity of coordinate j among the
// s = 2^c shared draws), w_j x_j (two bytes), wa = sum_j w_j x_j^2.  wovf[i] = 1 when
// some w_j > 255 (the point's pairs then take the list path).  One warp per point.
__global__ void __launch_bounds__(256) k_build_w(Geom g) {
  extern __shared__ uint32_t wcnt[];  // [8 warps][pitch]
  const int c = g.ctl->gemm_level;
  if (c < 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 8 + warp;
  if (i >= g.n) return;
  const int pitch = (int)g.pitch;
  uint32_t *cnt = wcnt + (size_t)warp * pitch;
  for (int j = lane; j < pitch; j += 32) cnt[j] = 0;
  __syncwarp();
  const uint32_t s = 1u << c, nb = (s + 3) / 4, lv = (uint32_t)(c + 1), d = (uint32_t)g.d;
  for (uint32_t b = lane; b < nb; b += 32) {
    const uint4 w = philox4x32_10_rk(make_uint4(b, (uint32_t)i + g.id_offset, SHARED_QI, lv), g.rk0, g.rk1);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (4 * b + e < s) atomicAdd(&cnt[coord_of(ws[e], d)], 1u);
  }
  __syncwarp();
  const uint8_t *xr = g.X + (size_t)i * pitch;
  const size_t o = (size_t)i * pitch;
  int32_t wa = 0;
  bool ovf = false;
  for (int j = lane; j < pitch; j += 32) {
    const uint32_t wj = cnt[j], x = xr[j], wx = wj * x;
    ovf |= wj > 255u;
    g.wc[o + j] = (uint8_t)(wj > 255u ? 0u : wj);
    g.wx0[o + j] = (uint8_t)(wx & 255u);
    g.wx1[o + j] = (uint8_t)(wx >> 8);
    wa += (int32_t)(wj * x * x);
  }
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) wa += __shfl_xor_sync(0xffffffffu, wa, k);
  ovf = __any_sync(0xffffffffu, ovf);
  if (lane == 0) {
    g.wa[i] = wa;
    g.wovf[i] = ovf ? 1 : 0;
    if (ovf) atomicOr(&g.ctl->wovf_any, 1u);
  }
}

// Persistent: one CTA per SM walks the flagged 128 x 128 tiles (query tiles fastest,
// so the resident CTAs share each point tile's planes through L2).  Warp 0 issues
// the TMA loads and runs ahead across tiles through the LM_STAGES ring; warp 1
// issues the MMAs of a tile once the epilogue has drained the previous tile's
// accumulators (warp 1 also owns the TMEM allocation); warps 2..9 drain TMEM into registers (a warp: its 32-lane quadrant
// x 64 columns), release TMEM at once and then update S / lvl from registers while
// the next tile's loads and MMAs run.
constexpr int LM_EPI_WARP0 = 2, LM_EPI_WARPS = 8;
constexpr int LM_EPI_COLS = LM_BN * 4 / LM_EPI_WARPS;  // columns per epilogue thread
constexpr int LM_NT = 32 * (LM_EPI_WARP0 + LM_EPI_WARPS);


__device__ __forceinline__ bool level_tile_on(const Geom &g, int c, int mt, int t) {
  const int mi = t % mt, ni = t / mt;
  return g.lvcnt[((size_t)mi * g.lv_cols + ni) * MAX_LEVELS + c] >= g.lmin;
}



__global__ void __launch_bounds__(LM_NT, 1)
    k_level_mma(const __grid_constant__ CUtensorMap tQ, const __grid_constant__ CUtensorMap tQ2l,
                const __grid_constant__ CUtensorMap tQ2h, const __grid_constant__ CUtensorMap tWx0,
                const __grid_constant__ CUtensorMap tWx1, const __grid_constant__ CUtensorMap tWc, Geom g) {
  const int c = g.ctl->gemm_level;
  if (c < 0) return;  // uniform
  const int mt = (g.q + LM_BM - 1) / LM_BM;
  const int ntiles = mt * ((g.n + LM_BN - 1) / LM_BN);
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(sm + LM_STAGES * LM_STAGE_BYTES);
  uint64_t *empty = full + LM_STAGES;
  uint64_t *tfull = empty + LM_STAGES;
  uint64_t *tempty = tfull + 1;
  uint32_t *tmem_base = reinterpret_cast<uint32_t *>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (g.d + MM_BK - 1) / MM_BK;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < LM_STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, LM_EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base)),
                 "n"(LM_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: 6 planes per k-block, running ahead across tiles
      uint32_t kg = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (!level_tile_on(g, c, mt, t)) continue;
        const int m0 = (t % mt) * LM_BM, n0 = (t / mt) * LM_BN;
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const uint32_t s = kg % LM_STAGES;
          if (kg >= LM_STAGES) mbar_wait(empty + s, ((kg / LM_STAGES) - 1) & 1);
          unsigned char *sa = sm + s * LM_STAGE_BYTES;
          mbar_expect_tx(full + s, LM_STAGE_BYTES);
          tma_load_2d(sa + 0 * LM_PLANE, &tQ, full + s, kb * MM_BK, m0);
          tma_load_2d(sa + 1 * LM_PLANE, &tQ2l, full + s, kb * MM_BK, m0);
          tma_load_2d(sa + 2 * LM_PLANE, &tQ2h, full + s, kb * MM_BK, m0);
          tma_load_2d(sa + 3 * LM_PLANE, &tWx0, full + s, kb * MM_BK, n0);
          tma_load_2d(sa + 4 * LM_PLANE, &tWx1, full + s, kb * MM_BK, n0);
          tma_load_2d(sa + 5 * LM_PLANE, &tWc, full + s, kb * MM_BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: acc0 = Q.Wx0, acc1 = Q.Wx1, acc2 = Q2lo.Wc, acc3 = Q2hi.Wc
      constexpr uint32_t idesc = umma_idesc_u8(LM_BM, LM_BN);
      uint32_t kg = 0, tl = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (!level_tile_on(g, c, mt, t)) continue;
        if (tl > 0) {  // the epilogue has drained the previous tile's accumulators
          mbar_wait(tempty, (tl - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const uint32_t s = kg % LM_STAGES;
          mbar_wait(full + s, (kg / LM_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sb = smem_u32(sm + s * LM_STAGE_BYTES);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const uint32_t pa = sb + (uint32_t)(a < 2 ? 0 : a - 1) * LM_PLANE;  // Q, Q, Q2lo, Q2hi
            const uint32_t pb = sb + (uint32_t)(a == 0 ? 3 : (a == 1 ? 4 : 5)) * LM_PLANE;
#pragma unroll
            for (int kk = 0; kk < MM_BK / 32; ++kk) {
              const uint64_t da = umma_desc_sw128(pa + kk * 32), db = umma_desc_sw128(pb + kk * 32);
              const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
              asm volatile(
                  "{\n\t.reg .pred p;\n\t"
                  "setp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (uint32_t)a * LM_BN),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(empty + s))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(tfull))
                     : "memory");
        ++tl;
      }
    }
  } else if (warp >= LM_EPI_WARP0) {
    // epilogue: TMEM lanes 32 * (warp % 4) .. + 31 = query rows, LM_EPI_COLS columns per warp
    const int quad = warp & 3, part = (warp - LM_EPI_WARP0) >> 2;
    const uint8_t lvc = (uint8_t)(c + 1);
    uint32_t tl = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      if (!level_tile_on(g, c, mt, t)) continue;
      const int m0 = (t % mt) * LM_BM, n0 = (t / mt) * LM_BN;
      const int row = m0 + quad * 32 + lane, cb = n0 + part * LM_EPI_COLS;
      if (warp == LM_EPI_WARP0 && lane == 0) atomicAdd(&g.ctl->lmma_tiles, 1ull);
      // D = wa + B - 2C for the thread's pairs (uint32: the wrap-around sum is exact
      // because the final S fits 31 bits); wa is loaded while the MMAs run
      uint32_t D[LM_EPI_COLS];
#pragma unroll
      for (int j = 0; j < LM_EPI_COLS / 4; ++j) {
        const int4 w = (cb + j * 4 < g.npad) ? *reinterpret_cast<const int4 *>(g.wa + cb + j * 4)
                                             : make_int4(0, 0, 0, 0);
        D[j * 4 + 0] = (uint32_t)w.x;
        D[j * 4 + 1] = (uint32_t)w.y;
        D[j * 4 + 2] = (uint32_t)w.z;
        D[j * 4 + 3] = (uint32_t)w.w;
      }
      mbar_wait(tfull, tl & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(part * LM_EPI_COLS);
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const uint32_t mul = a == 0 ? 0xFFFFFFFEu : (a == 1 ? 0xFFFFFE00u : (a == 2 ? 1u : 256u));  // -2, -512, 1, 256
#pragma unroll
        for (int h = 0; h < LM_EPI_COLS / 16; ++h) {
          uint32_t v[16];
          tmem_ld16(ta + (uint32_t)a * LM_BN + (uint32_t)(h * 16), v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 16; ++j) D[h * 16 + j] += mul * v[j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);  // TMEM free for the next tile's MMAs
      ++tl;
      if (row < g.q && cb < g.npad && !g.qs[row].done) {
        const size_t o = (size_t)row * g.npad + cb;  // npad % 16 == 0: 16-column groups are aligned
#pragma unroll
        for (int b = 0; b < LM_EPI_COLS / 16; ++b) {  // 16 pairs at a time
          const int c16 = b * 16;
          if (cb + c16 >= g.npad) break;
          const uint4 a16 = *reinterpret_cast<const uint4 *>(g.act + o + c16);
          const uint4 w16 = *reinterpret_cast<const uint4 *>(g.wovf + cb + c16);
          const uint32_t aw[4] = {a16.x, a16.y, a16.z, a16.w};
          const uint32_t ww[4] = {w16.x, w16.y, w16.z, w16.w};
          uint32_t hit = 0;  // bit e: pair cb + c16 + e takes this level's update
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t av = (aw[e >> 2] >> (8 * (e & 3))) & 0xFFu, wv = (ww[e >> 2] >> (8 * (e & 3))) & 0xFFu;
            hit |= (av == lvc && wv == 0u) ? (1u << e) : 0u;
          }
          if (!hit) continue;
          int4 S4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if ((hit >> (j * 4)) & 15u) S4[j] = *reinterpret_cast<const int4 *>(g.S + o + c16 + j * 4);
          const uint4 l16 = *reinterpret_cast<const uint4 *>(g.lvl + o + c16);
          uint32_t lw[4] = {l16.x, l16.y, l16.z, l16.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t hv = (hit >> (j * 4)) & 15u;
            if (!hv) continue;
            uint32_t sv[4] = {(uint32_t)S4[j].x, (uint32_t)S4[j].y, (uint32_t)S4[j].z, (uint32_t)S4[j].w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if ((hv >> e) & 1u) {
                sv[e] += D[c16 + j * 4 + e];
                lw[j] = (lw[j] & ~(0xFFu << (8 * e))) | ((uint32_t)lvc << (8 * e));
              }
            *reinterpret_cast<int4 *>(g.S + o + c16 + j * 4) = make_int4((int)sv[0], (int)sv[1], (int)sv[2], (int)sv[3]);
          }
          *reinterpret_cast<uint4 *>(g.lvl + o + c16) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(LM_TMEM_COLS));
  }
}

cudaError_t launch_q2_planes(const Geom &g, cudaStream_t s) {
  const size_t tot = (size_t)g.q * g.pitch;
  if (tot) k_q2_planes<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_build_w(const Geom &g, cudaStream_t s) {
  const size_t smem = (size_t)8 * g.pitch * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(k_build_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_build_w<<<(unsigned)((g.n + 7) / 8), 256, smem, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_level_mma(const Geom &g, cudaStream_t s) {
  CUtensorMap tq, tq2l, tq2h, tw0, tw1, twc;
  cudaError_t err = make_map(&tq, g.Q, g.q, g.d, g.pitch, LM_BM);
  if (err == cudaSuccess) err = make_map(&tq2l, g.q2lo, g.q, g.d, g.pitch, LM_BM);
  if (err == cudaSuccess) err = make_map(&tq2h, g.q2hi, g.q, g.d, g.pitch, LM_BM);
  if (err == cudaSuccess) err = make_map(&tw0, g.wx0, g.n, g.d, g.pitch, LM_BN);
  if (err == cudaSuccess) err = make_map(&tw1, g.wx1, g.n, g.d, g.pitch, LM_BN);
  if (err == cudaSuccess) err = make_map(&twc, g.wc, g.n, g.d, g.pitch, LM_BN);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(k_level_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM_SMEM);
  if (err != cudaSuccess) return err;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) sms = 148;
  }
  const long long tiles = (long long)((g.q + LM_BM - 1) / LM_BM) * ((g.n + LM_BN - 1) / LM_BN);
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  if (grid) k_level_mma<<<grid, LM_NT, LM_SMEM, s>>>(tq, tq2l, tq2h, tw0, tw1, twc, g);
  return cudaGetLastError();
}

int level_tile_rows() { return LM_BM; }
int level_tile_cols() { return LM_BN; }

}  // namespace aknn
