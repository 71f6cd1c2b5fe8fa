// advance_tiles.cu -- level gathers (row a3) of DENSE tiles from shared memory.
//
// The batch's (query x point) grid is cut into tiles of R = 2^tile_lr queries x
// P = 2^tile_lp points.  k_filter adds, per tile, the draws its blockers take this
// round (tilework); a tile whose draws reach tile_min_draws is advanced here instead of
// through the work lists (k_scatter leaves its pairs out): the CTA copies the R
// query rows and P point rows into shared memory once with 16-byte loads, then every
// draw of every listed pair of the tile gathers its two bytes from there.
//
// Why: a draw gathered from global memory costs one random 32-byte sector (L2, or HBM
// when X does not fit L2) and two L1 wavefronts; in a dense tile the R + P rows are
// read once for R * P pairs, so the sector traffic per pair and level drops from
// ~min(s, d/32) sectors to (R + P) * d / (R * P) bytes and the gathers become
// shared-memory loads.  What remains is the Philox4x32-10 integer work (the ALU bound
// of DESIGN.md §7).  Under the footnote-2 radius every arm of a query walks every
// level in lockstep, so nearly every tile is dense at every level.
//
// Inside a tile the active pairs are grouped by level c (smem compaction); each
// pair's draws are summed by one thread or one group of consecutive lanes (shuffle
// reduce), ADV_TP independent Philox blocks in flight per thread.  Integer sums: the
// result does not depend on the order, so S matches the list path and the oracle bit
// for bit.
#include "internal.cuh"
#include "launch.h"
#include "select.cuh"

namespace aknn {

constexpr int TILE_NT = 256;
// A shape whose shared memory allows one CTA per SM (rows > 8 KB, e.g. C3's 12 KB) runs
// 20 warps in that CTA instead of 8: the Philox chains and the shared-memory gathers
// need the extra warps to hide their latency (ncu, C3 at 8 warps: fmaheavy 25-42 %).
constexpr int TILE_NT_WIDE = 640;
constexpr int ADV_TP = 4;  // items (Philox blocks) in flight per thread

// Row slots are 2^slot_l bytes (>= pitch) and start at multiples of 2^slot_l, so
// the shared-memory address of coordinate j of a row is (row base | j): one LOP3 on
// the ALU pipe.  With a plain add, ptxas folds the row base into the multiply-high of
// the coordinate map (IMAD.HI with a 64-bit addend, plus IMAD.MOVs to build it) and
// repeats that multiply for the query row -- all on the fma-heavy pipe, the one the
// Philox rounds saturate (ncu: fmaheavy 84 % at 256 draws per pair).
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t sq_diff(uint32_t xa, uint32_t qa, uint32_t j) {
  const int diff = (int)lds_u8(xa | j) - (int)lds_u8(qa | j);
  return (uint32_t)(diff * diff);
}

// Four draws of one Philox block: the bytes are packed four to a word (PRMT, ALU)
// and summed with one VABSDIFF4 + one IDP.4A, instead of four subtractions and four
// multiply-adds on the fma-heavy pipe.  Exact: |x - q|^2 summed in uint32.
__device__ __forceinline__ uint32_t sq_diff4_j(uint32_t xa, uint32_t qa, uint32_t j0, uint32_t j1, uint32_t j2,
                                               uint32_t j3, uint32_t acc) {
  const uint32_t x01 = __byte_perm(lds_u8(xa | j0), lds_u8(xa | j1), 0x1140);
  const uint32_t x23 = __byte_perm(lds_u8(xa | j2), lds_u8(xa | j3), 0x4011);
  const uint32_t q01 = __byte_perm(lds_u8(qa | j0), lds_u8(qa | j1), 0x1140);
  const uint32_t q23 = __byte_perm(lds_u8(qa | j2), lds_u8(qa | j3), 0x4011);
  const uint32_t t = __vabsdiffu4(__byte_perm(x01, x23, 0x7610), __byte_perm(q01, q23, 0x7610));
  return __dp4a(t, t, acc);
}

// Tight row slots (stride = pitch, not a power of two): coordinate address = row base + j.
__device__ __forceinline__ uint32_t sq_diff_t(uint32_t xa, uint32_t qa, uint32_t j) {
  const int diff = (int)lds_u8(xa + j) - (int)lds_u8(qa + j);
  return (uint32_t)(diff * diff);
}
__device__ __forceinline__ uint32_t sq_diff4_t(uint32_t xa, uint32_t qa, uint4 w, uint32_t d, uint32_t acc) {
  const uint32_t j0 = coord_of(w.x, d), j1 = coord_of(w.y, d), j2 = coord_of(w.z, d), j3 = coord_of(w.w, d);
  const uint32_t x01 = __byte_perm(lds_u8(xa + j0), lds_u8(xa + j1), 0x1140);
  const uint32_t x23 = __byte_perm(lds_u8(xa + j2), lds_u8(xa + j3), 0x4011);
  const uint32_t q01 = __byte_perm(lds_u8(qa + j0), lds_u8(qa + j1), 0x1140);
  const uint32_t q23 = __byte_perm(lds_u8(qa + j2), lds_u8(qa + j3), 0x4011);
  const uint32_t t = __vabsdiffu4(__byte_perm(x01, x23, 0x7610), __byte_perm(q01, q23, 0x7610));
  return __dp4a(t, t, acc);
}

__device__ __forceinline__ uint32_t sq_diff4(uint32_t xa, uint32_t qa, uint4 w, uint32_t d, uint32_t acc) {
  return sq_diff4_j(xa, qa, coord_of(w.x, d), coord_of(w.y, d), coord_of(w.z, d), coord_of(w.w, d), acc);
}

// Without replacement (reading R23): the draws t0 .. t0 + 3 are pi(t) under the keys w.
__device__ __forceinline__ uint32_t sq_diff4_wor(uint32_t xa, uint32_t qa, uint4 w, const WorRadix &z,
                                                 uint32_t d, uint32_t t0, uint32_t acc) {
  const uint4 j = wor_coords4(w, z, d, t0);
  return sq_diff4_j(xa, qa, j.x, j.y, j.z, j.w, acc);
}

// ---------------------------------------------------------------------------
// Query-independent draws (AKNN_FLAG_SHARED_DRAWS) with R = 32 query
// rows per tile: arm p's t-th coordinate is the same for every query, so a level's
// draws of a point column are generated ONCE (Philox + the point's byte) into a
// packed list (j | x_j << 16) and every query row of every tile of the column reuses
// them: the per-pair work is one conflict-free byte gather from the transposed query
// tile Qt[j][32] (lane = query row) and one multiply-add.  Philox work drops by the
// 32 query rows of a tile (and by the column's tile rows when a level fits one chunk).
constexpr int F1_R = 32;

// Qt[j * 32 + r] = Q[r0 + r][j] for the tile's 32 query rows: 4 x 4 byte blocks
// transposed with PRMT (4-byte loads, 4-byte stores); QT_U blocks per thread in flight.
constexpr int QT_U = 2;
__device__ __forceinline__ void f1_stage_qt(const Geom &g, int r0, uint32_t *qt) {
  const int nj4 = (int)(g.pitch >> 2);  // 4-byte columns (pitch is a multiple of 16)
  const int total = 8 * nj4;
  for (int it0 = threadIdx.x; it0 < total; it0 += TILE_NT * QT_U) {
    uint32_t a[QT_U][4];
#pragma unroll
    for (int u = 0; u < QT_U; ++u) {
      const int it = it0 + u * TILE_NT, rb = it & 7, jb = it >> 3;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = r0 + rb * 4 + k;
        a[u][k] = (it < total && r < g.q) ? __ldg(reinterpret_cast<const uint32_t *>(g.Q + (size_t)r * g.pitch) + jb) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < QT_U; ++u) {
      const int it = it0 + u * TILE_NT, rb = it & 7, jb = it >> 3;
      if (it >= total) break;
      const uint32_t t01 = __byte_perm(a[u][0], a[u][1], 0x5140), t23 = __byte_perm(a[u][2], a[u][3], 0x5140);
      const uint32_t u01 = __byte_perm(a[u][0], a[u][1], 0x7362), u23 = __byte_perm(a[u][2], a[u][3], 0x7362);
      uint32_t *col = qt + (size_t)(jb * 4) * (F1_R / 4) + rb;  // word (j * 32 + 4 rb) / 4
      col[0 * (F1_R / 4)] = __byte_perm(t01, t23, 0x5410);
      col[1 * (F1_R / 4)] = __byte_perm(t01, t23, 0x7632);
      col[2 * (F1_R / 4)] = __byte_perm(u01, u23, 0x5410);
      col[3 * (F1_R / 4)] = __byte_perm(u01, u23, 0x7632);
    }
  }
}

// The draws u0 .. u0+ch-1 of level c for the P points of the column: dbuf[p * ch + u]
// = 32 j | X[p0 + p][j] << 24 (32 j < 2^21: the Qt offset of coordinate j).  Returns
// the Philox blocks drawn.
__device__ __forceinline__ unsigned f1_generate(const Geom &g, int p0, int P, int c, unsigned u0, unsigned ch,
                                                uint32_t *dbuf) {
  const unsigned s = 1u << c;
  const unsigned nbk = (ch + 3) / 4;  // blocks of this chunk per point
  const uint32_t lv = (uint32_t)(c + 1), d = (uint32_t)g.d;
  for (unsigned it = threadIdx.x; it < (unsigned)P * nbk; it += TILE_NT) {
    const int p = (int)(it / nbk);
    const unsigned bk = it - (unsigned)p * nbk, u = u0 + 4 * bk;
    const int i = p0 + p;
    const uint8_t *xr = g.X + (size_t)(i < g.n ? i : 0) * g.pitch;
    const uint4 w = philox4x32_10_rk(make_uint4(u >> 2, (uint32_t)i + g.id_offset, SHARED_QI, lv), g.rk0, g.rk1);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (u + e < s && u + e < u0 + ch) {
        const uint32_t j = coord_of(ws[e], d);
        dbuf[p * ch + (u - u0) + e] = (j * F1_R) | ((uint32_t)__ldg(xr + j) << 24);
      }
    }
  }
  return (unsigned)P * nbk;
}

// Sum over the chunk's draws of (x_j - Qt[j][r])^2 for pair (r = lane, p): warp w takes
// points w, w + 8, ...; acc[k] accumulates point w + 8k.  qt_s / dbuf_s: shared-memory
// addresses; ch is a multiple of 4 except for levels 0 and 1 (1 and 2 draws).
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds_u128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ void f1_accumulate(uint32_t qt_s, uint32_t dbuf_s, int P, unsigned ch, uint32_t (&acc)[4]) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t ql = qt_s + lane;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t p = warp + 8 * k;
    if (p >= (uint32_t)P) break;
    const uint32_t dp = dbuf_s + p * ch * 4u;
    uint32_t sum = 0;
    if ((ch & 3u) == 0) {
      for (uint32_t u = 0; u < ch; u += 4) {
        const uint4 pk = lds_u128(dp + u * 4u);  // broadcast
        // the 4 point bytes (top bytes of the packed words) and the 4 query bytes, packed;
        // |x - q|^2 summed by VABSDIFF4 + IDP.4A
        const uint32_t x4 = __byte_perm(__byte_perm(pk.x, pk.y, 0x0073), __byte_perm(pk.z, pk.w, 0x0073), 0x5410);
        const uint32_t q0 = lds_u8(ql + (pk.x & 0x1FFFFFu)), q1 = lds_u8(ql + (pk.y & 0x1FFFFFu));
        const uint32_t q2 = lds_u8(ql + (pk.z & 0x1FFFFFu)), q3 = lds_u8(ql + (pk.w & 0x1FFFFFu));
        const uint32_t q4 = __byte_perm(__byte_perm(q0, q1, 0x0040), __byte_perm(q2, q3, 0x0040), 0x5410);
        const uint32_t t = __vabsdiffu4(x4, q4);
        sum = __dp4a(t, t, sum);
      }
    } else {
      for (uint32_t u = 0; u < ch; ++u) {
        const uint32_t v = lds_u32(dp + u * 4u);
        const int diff = (int)(v >> 24) - (int)lds_u8(ql + (v & 0x1FFFFFu));
        sum += (uint32_t)(diff * diff);
      }
    }
    acc[k] += sum;
  }
}

// MODE 0: per-query draws with replacement; 1: query-independent draws (R = 32);
// 2: per-query draws without replacement (reading R23).
template <int MODE, int NT>
__global__ void __launch_bounds__(NT) k_advance_tiles(Geom g) {
  if ((float)g.ctl->tile_max < g.tile_min_draws) return;  // no dense tile this pass
  static_assert(MODE != 1 || NT == NT, "shared-draw tiles run 8 warps (f1_accumulate)");
  extern __shared__ __align__(16) unsigned char tsm[];
  __shared__ unsigned lcnt[MAX_LEVELS], loff[MAX_LEVELS + 1], lfill[MAX_LEVELS];
  const int R = 1 << g.tile_lr, P = 1 << g.tile_lp, RP = R * P;
  const int pitch = (int)g.pitch, nv = pitch >> 4;
  const int sl = g.tile_slot_l;
  const uint32_t slot = 1u << sl;
  // rows: [R query rows][P point rows], slot-aligned; then acc [RP] int32, lst [RP] u16
  // dynamic shared memory: [acc RP int32 | lst RP u16 | sact RP u8] at its start, then
  // the R + P row slots from the next slot boundary (the host sized it for that)
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tsm);
  int32_t *acc = reinterpret_cast<int32_t *>(tsm);
  uint16_t *lst = reinterpret_cast<uint16_t *>(acc + RP);
  uint8_t *sact = reinterpret_cast<uint8_t *>(lst + RP);  // [RP] action bytes of the tile
  const uint32_t rows_s = (base + (uint32_t)RP * 7u + slot - 1) & ~(slot - 1);
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (rows_s + ((uint32_t)(R + P) << sl) > base + dyn) __trap();  // host sizing broken: fail loudly
  }
  const uint32_t xs = rows_s + ((uint32_t)R << sl);  // first point row
  const int tid = threadIdx.x;
  const int rows = (g.q + R - 1) >> g.tile_lr;
  const uint32_t d = (uint32_t)g.d;
  const long long cols = (g.n + P - 1) >> g.tile_lp;
  const long long ntot = (long long)rows * cols;
  const float dthr = g.tile_min_draws;
  __shared__ uint16_t dlist[NT];  // dense tiles of the chunk (offsets, in order)
  __shared__ unsigned wcnt[NT / 32];

  // each CTA walks a contiguous range of the point-major tile space (t = tp * rows +
  // tr), so consecutive dense tiles of one point column reuse the staged point rows;
  // density is read 256 tiles at a time and compacted in order
  const long long t0 = (long long)blockIdx.x * ntot / gridDim.x, t1 = (long long)(blockIdx.x + 1) * ntot / gridDim.x;
  int staged_tp = -1;
  __shared__ __align__(8) uint64_t tbar;  // row staging mbarrier (bulk TMA copies)
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&tbar);
  uint32_t bar_phase = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int gen_tp = -1, gen_c = -1;  // shared draws: the column / level whose draw list is in dbuf
  __shared__ unsigned long long s_blocks, s_draws;  // Philox blocks and pair draws (statistics)
  if (tid == 0) s_blocks = s_draws = 0;
  if (tid < MAX_LEVELS) lcnt[tid] = 0;  // (the chunk loop's first barrier orders it)
  for (long long c0 = t0; c0 < t1; c0 += NT) {
    __syncthreads();  // dlist of the previous chunk is consumed
    {
      const long long t = c0 + tid;
      bool dense = false;
      if (t < t1) {
        const int tp = (int)(t / rows), tr = (int)(t % rows);
        dense = (float)g.tilework[(size_t)tr * g.tile_cols + tp] >= dthr;
      }
      const unsigned m = __ballot_sync(FULL, dense);
      if (lane_id() == 0) wcnt[tid >> 5] = __popc(m);
      __syncthreads();
      unsigned before = 0;
      for (int w = 0; w < (tid >> 5); ++w) before += wcnt[w];
      if (dense) dlist[before + __popc(m & ((1u << lane_id()) - 1u))] = (uint16_t)(t - c0);
    }
    __syncthreads();
    unsigned nd = 0;
    for (int w = 0; w < NT / 32; ++w) nd += wcnt[w];
  for (unsigned ti = 0; ti < nd; ++ti) {
    const long long t = c0 + dlist[ti];
    const int tp = (int)(t / rows), tr = (int)(t % rows);
    const int r0 = tr << g.tile_lr, p0 = tp << g.tile_lp;
    const bool reuse_x = tp == staged_tp;  // the point rows of this column are staged
    staged_tp = tp;
    constexpr bool f1 = MODE == 1;  // query-independent draws with R = 32 (host-selected instantiation)
    constexpr bool wor = MODE == 2;
    __syncthreads();  // the previous tile's shared memory is no longer in use
    // (lcnt was cleared after the previous tile's last read of it, before this barrier:
    // clearing it here would race with the level histogram of the other warps)

    // stage the rows.  Bulk TMA copies (one cp.async.bulk per row, issued by thread 0,
    // completion counted in bytes on an mbarrier) unless g.tile_tma == 0; otherwise
    // 16-byte cp.async copies, all in flight at once.  Rows past q / n are never
    // referenced and are left as they are.  Shared draws: the query rows transposed
    // (Qt), no point rows (their bytes are in the draw list)
    const bool tma = !f1 && g.tile_tma;
    if (tma && tid == 0) {
      uint32_t bytes = 0;
      const int nrow = reuse_x ? R : R + P;
      for (int row = 0; row < nrow; ++row)
        bytes += (row < R ? r0 + row < g.q : p0 + row - R < g.n) ? (uint32_t)pitch : 0u;
      // the previous tile's generic-proxy reads of these slots precede the async writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(bytes) : "memory");
      for (int row = 0; row < nrow; ++row) {
        const uint8_t *src = row < R ? (r0 + row < g.q ? g.Q + (size_t)(r0 + row) * pitch : nullptr)
                                     : (p0 + row - R < g.n ? g.X + (size_t)(p0 + row - R) * pitch : nullptr);
        if (src)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  rows_s + ((uint32_t)row << sl)),
              "l"(src), "r"((uint32_t)pitch), "r"(bar_s)
              : "memory");
      }
    }
    if (f1) f1_stage_qt(g, r0, reinterpret_cast<uint32_t *>(tsm + (rows_s - base)));
    for (int v = tid; v < ((f1 || tma) ? 0 : (reuse_x ? R : R + P) * nv); v += NT) {
      const int row = v / nv, c = v - row * nv;
      const uint8_t *src = nullptr;
      if (row < R) {
        if (r0 + row < g.q) src = g.Q + (size_t)(r0 + row) * pitch + 16 * c;
      } else if (!reuse_x && p0 + row - R < g.n) {
        src = g.X + (size_t)(p0 + row - R) * pitch + 16 * c;
      }
      if (src)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rows_s + ((uint32_t)row << sl) + 16u * c),
                     "l"(src)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // thread -> 4 consecutive arms of one query row (RP <= 4 * NT, P >= 4): the
    // query's done flag, the action bytes, S and the level bytes in ONE round trip
    const int e4 = tid * 4;
    const bool in = e4 < RP;
    const int rr = in ? e4 >> g.tile_lp : 0, pp = e4 & (P - 1);
    const bool live = in && r0 + rr < g.q && p0 + pp < g.n;
    const size_t o4 = (size_t)(r0 + rr) * g.npad + p0 + pp;
    int4 S4 = make_int4(0, 0, 0, 0);
    uint32_t A4 = 0, L4 = 0;
    int dn = 1;
    if (live) {
      dn = g.qs[r0 + rr].done;
      A4 = *reinterpret_cast<const uint32_t *>(g.act + o4);
      S4 = *reinterpret_cast<const int4 *>(g.S + o4);
      L4 = *reinterpret_cast<const uint32_t *>(g.lvl + o4);
    }
    uint32_t act4 = 0;  // sampled actions only (exact fallbacks: tensor-core pass)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint8_t a = (uint8_t)(A4 >> (8 * k));
      if (dn || a > MAX_LEVELS || p0 + pp + k >= g.n) a = 0;  // stale bytes of finished queries
      act4 |= (uint32_t)a << (8 * k);
      hist_add(lcnt, a ? a - 1u : NONE);
    }
    if (in) *reinterpret_cast<uint32_t *>(sact + e4) = act4;
    __syncthreads();  // lcnt
    if (tid < 32) {  // per-level list offsets
      const unsigned v = tid < MAX_LEVELS ? lcnt[tid] : 0u;
      unsigned x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, x, o);
        if (tid >= o) x += y;
      }
      if (tid < MAX_LEVELS) {
        loff[tid] = x - v;
        lfill[tid] = x - v;
      }
      if (tid == MAX_LEVELS - 1) loff[MAX_LEVELS] = x;
    }
    __syncthreads();
    // list the pairs by level: one shared atomic per (warp, level)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint8_t a = (uint8_t)(act4 >> (8 * k));
      const unsigned key = a ? a - 1u : NONE;
      const unsigned m = __match_any_sync(FULL, key);
      const int leader = __ffs(m) - 1;
      unsigned b0 = 0;
      if (a && lane_id() == leader) b0 = atomicAdd(&lfill[key], (unsigned)__popc(m));
      b0 = __shfl_sync(FULL, b0, leader);
      if (a) lst[b0 + __popc(m & ((1u << lane_id()) - 1u))] = (uint16_t)(e4 + k);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (tma) {  // every thread waits for the tile's bytes (phase bar_phase)
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "TW_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra TW_%=;\n\t}" ::"r"(bar_s),
          "r"(bar_phase)
          : "memory");
      bar_phase ^= 1u;
    }
    __syncthreads();

    // the draws, level by level.  nb <= ADV_TP blocks per pair: a thread owns
    // ADV_TP / nb whole pairs per pass.  nb > ADV_TP: tpp lanes per pair (consecutive
    // lanes), each running ADV_TP independent Philox blocks at a time, then a shuffle
    // reduce inside the lane group; every pair's sum is written by one thread.
    // levels present in the tile (one load per lane + a ballot, in every warp) and the
    // tile's pair draws (warp 0 reduces them; tid 0 adds them up)
    static_assert(MAX_LEVELS == 32, "one level per lane");
    const unsigned lv_l = lcnt[lane_id()];
    unsigned lmask = __ballot_sync(FULL, lv_l != 0u);
    unsigned long long tile_bl = 0;  // the tile's Philox blocks (tid 0)
    if (tid < 32) {
      unsigned long long dr = (unsigned long long)lv_l << lane_id();
      unsigned long long bl = (unsigned long long)lv_l << (lane_id() < 2 ? 0 : lane_id() - 2);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dr += __shfl_xor_sync(FULL, dr, o);
        bl += __shfl_xor_sync(FULL, bl, o);
      }
      if (tid == 0) s_draws += dr;
      tile_bl = bl;
    }
    if (f1) {
      // shared draws: per level, the column's draw list (cached across the column's
      // tiles while a level fits one chunk), then every (row, point) pair of the tile
      uint32_t *dbuf = reinterpret_cast<uint32_t *>(tsm + (rows_s - base) + ((size_t)R << sl));
      const uint32_t qt_s = rows_s, dbuf_s = rows_s + ((uint32_t)R << sl);
      const unsigned chmax = min(256u, (1u << sl) / 4u);
      for (; lmask; lmask &= lmask - 1) {
        const int c = __ffs(lmask) - 1;
        const unsigned s = 1u << c;
        uint32_t accp[4] = {0u, 0u, 0u, 0u};
        for (unsigned u0 = 0; u0 < s; u0 += chmax) {
          const unsigned ch = min(chmax, s - u0);
          const bool cached = s <= chmax && gen_tp == tp && gen_c == c;
          if (!cached) {
            __syncthreads();  // the previous chunk's draws are consumed
            const unsigned nb = f1_generate(g, p0, P, c, u0, ch, dbuf);
            if (tid == 0) s_blocks += nb;
            __syncthreads();
            gen_tp = s <= chmax ? tp : -1;
            gen_c = c;
          }
          f1_accumulate(qt_s, dbuf_s, P, ch, accp);
        }
        // pair (lane, warp + 8k): its sum if it advances at this level
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int p = (tid >> 5) + 8 * k, e = lane_id() * P + p;
          if (p < P && sact[e] == (uint8_t)(c + 1)) acc[e] = (int32_t)accp[k];
        }
      }
      lmask = 0;  // done: skip the per-pair Philox path below
    } else if (tid == 0) {
      s_blocks += tile_bl;
    }
    for (; lmask; lmask &= lmask - 1) {
      const int c = __ffs(lmask) - 1;
      const unsigned m = lcnt[c];
      const int lb = c < 2 ? 0 : c - 2;  // log2 Philox blocks per pair
      const unsigned s = 1u << c, nb = 1u << lb;
      const uint16_t *L = lst + loff[c];
      const uint32_t lv = (uint32_t)(c + 1);
      if (nb <= (unsigned)ADV_TP) {
        const unsigned ppt = ADV_TP / nb;
        for (unsigned l0 = tid; l0 < m; l0 += NT * ppt) {
          uint4 w[ADV_TP];
          int pr[ADV_TP];
#pragma unroll
          for (int k = 0; k < ADV_TP; ++k) {
            const unsigned li = l0 + (k / nb) * NT;
            const bool ok = (unsigned)k / nb < ppt && li < m;
            pr[k] = ok ? (int)L[li] : -1;
            const int e = ok ? pr[k] : 0;
            const uint32_t gi = (uint32_t)(p0 + (e & (P - 1))) + g.id_offset;
            const uint32_t gq = rng_qi(g, (uint32_t)(r0 + (e >> g.tile_lp)));
            w[k] = wor ? wor_keys(g.rk0, g.rk1, gi, gq)
                       : philox4x32_10_rk(make_uint4((uint32_t)k & (nb - 1), gi, gq, lv), g.rk0, g.rk1);
          }
          uint32_t sum = 0;
#pragma unroll
          for (int k = 0; k < ADV_TP; ++k) {
            if (pr[k] >= 0) {
              const uint32_t xa = xs + ((uint32_t)(pr[k] & (P - 1)) << sl);
              const uint32_t qa = rows_s + ((uint32_t)(pr[k] >> g.tile_lp) << sl);
              if (wor) {  // draws t = s + 4 blk + e, e < min(s, 4)
                const uint32_t t0 = s + 4u * ((uint32_t)k & (nb - 1));
                if (s >= 4) {
                  sum = sq_diff4_wor(xa, qa, w[k], g.wor_z, d, t0, sum);
                } else {
                  sum += sq_diff(xa, qa, wor_coord(w[k], g.wor_z, d, t0));
                  if (s == 2) sum += sq_diff(xa, qa, wor_coord(w[k], g.wor_z, d, t0 + 1u));
                }
              } else if (s >= 4) {
                sum = sq_diff4(xa, qa, w[k], d, sum);
              } else {  // levels 0 and 1 use 1 and 2 words of the block
                sum += sq_diff(xa, qa, coord_of(w[k].x, d));
                if (s == 2) sum += sq_diff(xa, qa, coord_of(w[k].y, d));
              }
            }
            if ((unsigned)(k + 1) % nb == 0) {  // last block of this pair
              if (pr[k] >= 0) acc[pr[k]] = (int32_t)sum;
              sum = 0;
            }
          }
        }
      } else {
        // nb > ADV_TP blocks per pair: the level's (pair, ADV_TP-block group) items are
        // dealt to the threads in one flat range (every thread busy whatever the pair
        // count), each item's sum added to its pair with one shared atomic (integer:
        // the order does not matter, S stays bit-identical)
        for (unsigned l = tid; l < m; l += NT) acc[L[l]] = 0;
        __syncthreads();
        const unsigned lg = (unsigned)(lb - 2);  // log2 groups of ADV_TP blocks per pair
        const unsigned total = m << lg;
        if (!wor) {
          // a CONTIGUOUS run of items per thread: the pair's constants (row addresses,
          // Philox round-0/1 products) and its shared atomic once per run of one pair
          const unsigned per = (total + NT - 1) / NT;
          const unsigned it1 = min(total, (unsigned)tid * per + per);
          int pe = -1;
          uint32_t xa = 0, qa = 0, sum = 0;
          PhiloxPair pc{};
          for (unsigned it = (unsigned)tid * per; it < it1; ++it) {
            const unsigned li = it >> lg, b0 = (it & ((1u << lg) - 1u)) * ADV_TP;
            if (b0 == 0 || pe < 0) {  // a new pair
              if (pe >= 0) atomicAdd(reinterpret_cast<uint32_t *>(acc + pe), sum);
              sum = 0;
              pe = (int)L[li];
              xa = xs + ((uint32_t)(pe & (P - 1)) << sl);
              qa = rows_s + ((uint32_t)(pe >> g.tile_lp) << sl);
              const uint32_t gi = (uint32_t)(p0 + (pe & (P - 1))) + g.id_offset;
              const uint32_t gq = rng_qi(g, (uint32_t)(r0 + (pe >> g.tile_lp)));
              pc = philox_pair(gi, gq, g.rk0);
            }
            uint4 w[ADV_TP];
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) w[k] = philox_from_pair(b0 + k, lv, pc, g.rk0, g.rk1);
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) sum = sq_diff4(xa, qa, w[k], d, sum);
          }
          if (pe >= 0) atomicAdd(reinterpret_cast<uint32_t *>(acc + pe), sum);
          continue;  // the next level
        }
        for (unsigned it = tid; it < total; it += NT) {
          const unsigned li = it >> lg, b0 = (it & ((1u << lg) - 1u)) * ADV_TP;
          const int pe = (int)L[li];
          const uint32_t xa = xs + ((uint32_t)(pe & (P - 1)) << sl);
          const uint32_t qa = rows_s + ((uint32_t)(pe >> g.tile_lp) << sl);
          const uint32_t gi = (uint32_t)(p0 + (pe & (P - 1))) + g.id_offset;
          const uint32_t gq = rng_qi(g, (uint32_t)(r0 + (pe >> g.tile_lp)));
          uint32_t sum = 0;
          if (wor) {
            const uint4 kk = wor_keys(g.rk0, g.rk1, gi, gq);
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) sum = sq_diff4_wor(xa, qa, kk, g.wor_z, d, s + 4u * (b0 + k), sum);
          } else {
            const PhiloxPair pc = philox_pair(gi, gq, g.rk0);
            uint4 w[ADV_TP];
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) w[k] = philox_from_pair(b0 + k, lv, pc, g.rk0, g.rk1);
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) sum = sq_diff4(xa, qa, w[k], d, sum);
          }
          atomicAdd(reinterpret_cast<uint32_t *>(acc + pe), sum);
        }
      }
    }
    __syncthreads();
    if (tid < MAX_LEVELS) lcnt[tid] = 0;  // for the next tile (every read of it is done)
    // commit: S += the level's sum, T -> 2T (the thread's own 4 arms)
    if (act4) {
      int4 o = S4;
      uint32_t l4 = L4;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t a = (act4 >> (8 * k)) & 0xFFu;
        if (!a) continue;
        const int32_t add = acc[e4 + k];
        if (k == 0) o.x += add;
        if (k == 1) o.y += add;
        if (k == 2) o.z += add;
        if (k == 3) o.w += add;
        l4 = (l4 & ~(0xFFu << (8 * k))) | (a << (8 * k));
      }
      *reinterpret_cast<int4 *>(g.S + o4) = o;
      *reinterpret_cast<uint32_t *>(g.lvl + o4) = l4;
    }
  }
  }
  if (threadIdx.x == 0 && s_blocks) atomicAdd(&g.ctl->tile_blocks, s_blocks);
  if (threadIdx.x == 0 && s_draws) atomicAdd(&g.ctl->tile_draws, s_draws);
}

// ---------------------------------------------------------------------------
// Grouped tiles (one CTA per SM, rows wider than 8 KB: C3).  The CTA walks whole point
// columns: it stages the column's P point rows ONCE and its NG thread groups then work
// on different query tiles of that column at the same time -- group j takes query
// tiles j, j + NG, ... -- each with its own R query-row slots, its own named barrier
// and mbarrier.  A tile's fixed latency (its action / S / level round trip, the copy
// of its query rows, the per-level barriers) is hidden by the other groups, as NG
// CTAs per SM would hide it, while the point rows stay shared (NG CTAs would need NG
// copies: the shared memory holds NG R + P slots instead of NG (R + P)).  Per-query
// draws with replacement (MODE 0) only; same arithmetic and result as k_advance_tiles.
//
// QG (the smallest tiled levels): no query-row copies -- a draw's query byte is gathered
// from global memory (Q is small and L2-resident), its point byte from the staged point
// rows.  A tile of 8 pairs at s draws each gathers 8 s query sectors instead of copying
// a whole query row (12 KB on C3): fewer bytes below ~48 draws per pair, and no copy
// latency in the tile's chain at any s.
//
// Dense for this launch: the tiles with tile_lo <= tilework < tile_hi (launch_advance_tiles
// splits the dense tiles between the QG, plain and |x - q| kernels).
__device__ __forceinline__ bool grp_dense(const Geom &g, float tw, float dthr) {
  return tw >= fmaxf(dthr, g.tile_lo) && tw < g.tile_hi;
}

constexpr int QG_LR = 4;  // QG super tiles: 16 query rows x P = 8 points (RP = 128: one-warp bookkeeping)

__device__ __forceinline__ uint32_t ldg_u8(const uint8_t *p) {
  uint32_t v;
  asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// QG: point byte from shared memory (x row at xa, coordinate address xa + j or xa | j),
// query byte from global memory.
template <bool TIGHT>
__device__ __forceinline__ uint32_t sq_diff_g(uint32_t xa, const uint8_t *qp, uint32_t j) {
  const int diff = (int)lds_u8(TIGHT ? xa + j : (xa | j)) - (int)ldg_u8(qp + j);
  return (uint32_t)(diff * diff);
}
template <bool TIGHT>
__device__ __forceinline__ uint32_t sq_diff4_g(uint32_t xa, const uint8_t *qp, uint4 w, uint32_t d, uint32_t acc) {
  const uint32_t j0 = coord_of(w.x, d), j1 = coord_of(w.y, d), j2 = coord_of(w.z, d), j3 = coord_of(w.w, d);
  const uint32_t q0 = ldg_u8(qp + j0), q1 = ldg_u8(qp + j1), q2 = ldg_u8(qp + j2), q3 = ldg_u8(qp + j3);
  const uint32_t x0 = lds_u8(TIGHT ? xa + j0 : (xa | j0)), x1 = lds_u8(TIGHT ? xa + j1 : (xa | j1));
  const uint32_t x2 = lds_u8(TIGHT ? xa + j2 : (xa | j2)), x3 = lds_u8(TIGHT ? xa + j3 : (xa | j3));
  const uint32_t x4 = __byte_perm(__byte_perm(x0, x1, 0x0040), __byte_perm(x2, x3, 0x0040), 0x5410);
  const uint32_t q4 = __byte_perm(__byte_perm(q0, q1, 0x0040), __byte_perm(q2, q3, 0x0040), 0x5410);
  const uint32_t t = __vabsdiffu4(x4, q4);
  return __dp4a(t, t, acc);
}

template <int NG, bool TIGHT, bool DB, int NTT, bool QG = false>
__global__ void __launch_bounds__(NTT) k_advance_tiles_grp(Geom g) {
  // DB: each group double-buffers its query rows -- the next tile's copy runs during this
  // tile's draws (2 NG R query slots); QG: no query rows in shared memory
  constexpr int QB = QG ? 0 : (DB ? 2 : 1);
  // no dense tile of this launch's range [lo, hi) in this pass
  if ((float)g.ctl->tile_max < fmaxf(g.tile_min_draws, g.tile_lo) || (float)g.ctl->tile_min >= g.tile_hi) return;
  constexpr int GT = NTT / NG;  // threads per group (whole warps)
  static_assert(GT % 32 == 0, "groups of whole warps");
  extern __shared__ __align__(16) unsigned char tsm[];
  __shared__ unsigned lcnt[NG][MAX_LEVELS], loff[NG][MAX_LEVELS + 1], lfill[NG][MAX_LEVELS];
  __shared__ __align__(8) uint64_t qbar[NG][2], pbar;
  __shared__ unsigned long long s_blocks, s_draws;
  __shared__ unsigned lmask_s[NG];
  __shared__ unsigned char accz[NG];  // 1: the tile's acc entries were zeroed by the fast path
  constexpr int CM_WORDS = 1024;                   // dense-tile bits of the column (rows <= 32768)
  __shared__ uint32_t colmask[CM_WORDS];
  // QG: super tiles of R = 2^QG_LR consecutive query rows (the bookkeeping of a tile --
  // its level lists, barriers, scan -- amortised over R P pairs instead of P; the tile
  // rows of tilework stay single query rows, so a row that is not dense is masked out)
  const int LR = QG ? QG_LR : g.tile_lr;
  const int R = 1 << LR, P = 1 << g.tile_lp, RP = R * P;
  const int pitch = (int)g.pitch;
  const bool one_warp_tiles = RP <= 128;  // a tile's bookkeeping sits in warp 0
  const int sl = g.tile_slot_l;
  const uint32_t slot = 1u << sl;
  // row stride: a power-of-two slot (coordinate address = row | j) or, TIGHT, the pitch
  const uint32_t stride = TIGHT ? (uint32_t)pitch : slot;
  const int tid = threadIdx.x, grp = tid / GT, gtid = tid - grp * GT;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tsm);
  // per group: acc [RP] int32 | lst [RP] u16 | sact [RP] u8 (7 RP bytes, 16-aligned)
  const uint32_t gsz = ((uint32_t)RP * 7u + 15u) & ~15u;
  int32_t *acc = reinterpret_cast<int32_t *>(tsm + (size_t)grp * gsz);
  uint16_t *lst = reinterpret_cast<uint16_t *>(acc + RP);
  uint8_t *sact = reinterpret_cast<uint8_t *>(lst + RP);
  const uint32_t rows_s = TIGHT ? base + (uint32_t)NG * gsz : (base + (uint32_t)NG * gsz + slot - 1) & ~(slot - 1);
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (rows_s + (uint32_t)(QB * NG * R + P) * stride > base + dyn) __trap();  // host sizing broken: fail loudly
  }
  const uint32_t qs0 = rows_s + (uint32_t)(grp * QB * R) * stride;  // this group's query rows (buffer 0)
  const uint32_t xs = rows_s + (uint32_t)(QB * NG * R) * stride;     // the column's point rows
  const uint32_t qbar0 = (uint32_t)__cvta_generic_to_shared(&qbar[grp][0]);
  const uint32_t pbar_s = (uint32_t)__cvta_generic_to_shared(&pbar);
  const uint32_t d = (uint32_t)g.d;
  const int rows = (g.q + R - 1) >> LR;                               // (super) tile rows
  const int rows1 = (g.q + (1 << g.tile_lr) - 1) >> g.tile_lr;        // tilework rows
  const int cols = (g.n + P - 1) >> g.tile_lp;
  const float dthr = g.tile_min_draws;
  if (tid == 0) {
    s_blocks = s_draws = 0;
    for (int j = 0; j < NG; ++j)
      for (int b = 0; b < 2; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&qbar[j][b])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(pbar_s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t qphase = 0u, pphase = 0;  // qphase bit b: the parity of query buffer b's barrier
  int sel = 0;  // the query buffer of the current tile
  auto gsync = [&] { asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(GT) : "memory"); };
  auto wait_bar = [](uint32_t bar, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "GW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GW_%=;\n\t}" ::"r"(bar),
        "r"(ph)
        : "memory");
  };
  const int c0 = (int)((long long)blockIdx.x * cols / gridDim.x), c1 = (int)((long long)(blockIdx.x + 1) * cols / gridDim.x);
  unsigned long long my_dr = 0, my_bl = 0;  // this group's draws / Philox blocks (gtid 0)
  // rows1 <= NTT (C3: 256): thread tr holds tile row tr's tilework of the NEXT column in a
  // register, loaded while the current column is processed (the strided reads of a
  // column's tilework cost an L2 round trip at every column start otherwise)
  const bool row_per_thread = rows1 <= NTT && rows1 <= CM_WORDS * 32;
  uint32_t tw_next = (row_per_thread && tid < rows1 && c0 < c1) ? g.tilework[(size_t)tid * g.tile_cols + c0] : 0u;
  for (int tp = c0; tp < c1; ++tp) {
    // the column's dense query tiles as a bit mask, read once (all groups are done with
    // the previous column); a column without one is skipped
    bool mine = false;
    __syncthreads();  // every group has left the previous column (its mask reads included)
    for (int w = tid; w < CM_WORDS && w * 32 < rows1; w += NTT) colmask[w] = 0u;
    __syncthreads();
    if (row_per_thread) {
      const uint32_t tw = tw_next;
      if (tid < rows1 && tp + 1 < c1) tw_next = g.tilework[(size_t)tid * g.tile_cols + tp + 1];
      if (tid < rows1 && grp_dense(g, (float)tw, dthr)) {
        mine = true;
        atomicOr(&colmask[tid >> 5], 1u << (tid & 31));
      }
    } else {
      for (int tr = tid; tr < rows1; tr += NTT) {
        const bool dn = grp_dense(g, (float)g.tilework[(size_t)tr * g.tile_cols + tp], dthr);
        mine |= dn;
        if (dn && tr < CM_WORDS * 32) atomicOr(&colmask[tr >> 5], 1u << (tr & 31));
      }
    }
    if (!__syncthreads_or(mine)) continue;
    const int p0 = tp << g.tile_lp;
    if (tid == 0 && tp + 1 < c1) {  // the next column's point rows: into L2 now (HBM -> L2)
      for (int row = 0; row < P; ++row)
        if (p0 + P + row < g.n)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g.X + (size_t)(p0 + P + row) * pitch),
                       "r"((uint32_t)pitch)
                       : "memory");
    }
    if (tid == 0) {  // the column's point rows: bulk TMA copies
      uint32_t bytes = 0;
      for (int row = 0; row < P; ++row) bytes += p0 + row < g.n ? (uint32_t)pitch : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pbar_s), "r"(bytes) : "memory");
      for (int row = 0; row < P; ++row)
        if (p0 + row < g.n)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  xs + (uint32_t)row * stride),
              "l"(g.X + (size_t)(p0 + row) * pitch), "r"((uint32_t)pitch), "r"(pbar_s)
              : "memory");
    }
    bool have_x = false;
    auto row_dense = [&](int tr) {  // tilework row tr
      return tr < CM_WORDS * 32 ? ((colmask[tr >> 5] >> (tr & 31)) & 1u) != 0u
                                : grp_dense(g, (float)g.tilework[(size_t)tr * g.tile_cols + tp], dthr);
    };
    auto dense_at = [&](int tr) {  // (super) tile row tr
      if (!QG) return row_dense(tr);
      const int r0 = tr << LR;
      if (r0 + R <= CM_WORDS * 32) return ((colmask[r0 >> 5] >> (r0 & 31)) & ((1u << R) - 1u)) != 0u;
      bool any = false;
      for (int r = r0; r < r0 + R && r < rows1; ++r) any |= row_dense(r);
      return any;
    };
    auto next_dense = [&](int tr) {  // the group's next dense query tile at or after tr
      while (tr < rows && !dense_at(tr)) tr += NG;
      return tr;
    };
    // thread -> 4 consecutive arms of one query row (RP <= 4 GT): done flag, actions, S
    // and levels in one round trip, issued one tile AHEAD (the tiles hold disjoint pairs)
    const int e4 = gtid * 4;
    const bool in = e4 < RP;
    const int rr = in ? e4 >> g.tile_lp : 0, pp = e4 & (P - 1);
    struct TileState {
      int4 S4;
      uint32_t A4, L4;
      int dn;
    };
    auto load_state = [&](int tr) {
      TileState t{make_int4(0, 0, 0, 0), 0u, 0u, 1};
      const int r0n = tr << LR;
      if (tr < rows && in && r0n + rr < g.q && p0 + pp < g.n && (!QG || row_dense(r0n + rr))) {
        const size_t o = (size_t)(r0n + rr) * g.npad + p0 + pp;
        t.dn = g.qs[r0n + rr].done;
        t.A4 = *reinterpret_cast<const uint32_t *>(g.act + o);
        t.S4 = *reinterpret_cast<const int4 *>(g.S + o);
        t.L4 = *reinterpret_cast<const uint32_t *>(g.lvl + o);
      }
      return t;
    };
    int trn = next_dense(grp);
    TileState nxt = load_state(trn);
    bool first = true;
    while (trn < rows) {
      const int tr = trn;
      const TileState cur = nxt;
      trn = next_dense(tr + NG);
      nxt = load_state(trn);  // in flight while this tile is processed
      const int r0 = tr << LR;
      // (no barrier here: the previous tile ended with one after its last read of the
      // query slot, acc, lst and the level tables, and only warp 0 writes them next)
      if (!one_warp_tiles) gsync();
      if (gtid < MAX_LEVELS) lcnt[grp][gtid] = 0;
      // the query rows: this tile's were copied during the previous tile of the column
      // (DB) unless it is the group's first; then the next tile's copy is issued into
      // the other buffer, free since the gsync above
      auto issue_rows = [&](int trq, int b) {
        const int rq = trq << LR;
        const uint32_t bar = qbar0 + 8u * (uint32_t)b, dst = qs0 + (uint32_t)(b * R) * stride;
        uint32_t bytes = 0;
        for (int row = 0; row < R; ++row) bytes += rq + row < g.q ? (uint32_t)pitch : 0u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        for (int row = 0; row < R; ++row)
          if (rq + row < g.q)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dst + (uint32_t)row * stride),
                "l"(g.Q + (size_t)(rq + row) * pitch), "r"((uint32_t)pitch), "r"(bar)
                : "memory");
      };
      // single-buffered: the tile's query rows were issued right after the previous
      // tile's last barrier (below) unless this is the group's first tile of the column
      if (!QG && gtid == 0) {
        if (first) issue_rows(tr, sel);
        if (DB && trn < rows) issue_rows(trn, sel ^ 1);
      }
      const uint32_t qs = qs0 + (uint32_t)(sel * R) * stride;
      const size_t o4 = (size_t)(r0 + rr) * g.npad + p0 + pp;
      const int4 S4 = cur.S4;
      const uint32_t A4 = cur.A4, L4 = cur.L4;
      const int dn = cur.dn;
      // RP <= 128: the lcnt clear, the arms (4 per thread) and the scan all sit in warp 0,
      // so its bookkeeping steps sync that warp only (the other warps meet it below)
      const bool one_warp = RP <= 128;
      auto bsync = [&] {
        if (one_warp)
          __syncwarp();
        else
          gsync();
      };
      bsync();  // lcnt cleared
      // only the warps holding arms (4 per thread, RP <= 4 GT) list them
      const bool arm_warp = (gtid & ~31) * 4 < RP;
      uint32_t act4 = 0;  // sampled actions only (exact fallbacks: tensor-core pass)
      // Tiles of <= 32 arms (C3's one-query tiles: 8) whose sampled arms all sit at ONE
      // level (lock-step rounds): warp 0 lists them with a min/max reduction and an
      // 8-lane prefix sum -- no level histogram, scan or per-level match (the general
      // path below, ~2x the instructions of this tile's bookkeeping)
      bool fast = false;
      if (RP <= 32 && gtid < 32) {
        if (in) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t a = (A4 >> (8 * k)) & 0xFFu;
            if (dn || a > (uint32_t)MAX_LEVELS || p0 + pp + k >= g.n) a = 0;
            act4 |= a << (8 * k);
          }
          *reinterpret_cast<uint32_t *>(sact + e4) = act4;
        }
        uint32_t lo = 255u, hi = 0u, cnt = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t a = (act4 >> (8 * k)) & 0xFFu;
          if (a) {
            lo = min(lo, a);
            hi = max(hi, a);
            ++cnt;
          }
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        if (hi == 0u || lo == hi) {
          fast = true;
          uint32_t x = cnt;
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, x, o);
            if (gtid >= o) x += y;
          }
          uint32_t b = x - cnt;
          const uint32_t tot = __shfl_sync(FULL, x, 7);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if ((act4 >> (8 * k)) & 0xFFu) lst[b++] = (uint16_t)(e4 + k);
#pragma unroll
          for (int k = 0; k < 4; ++k)  // the level's sums start at 0 (no zeroing pass below)
            if (in) acc[e4 + k] = 0;
          if (gtid == 0) {
            accz[grp] = 1;
            if (hi) {
              const uint32_t c = hi - 1u;
              lcnt[grp][c] = tot;
              loff[grp][c] = 0u;
              lmask_s[grp] = 1u << c;
              my_dr += (unsigned long long)tot << c;
              my_bl += (unsigned long long)tot << (c < 2u ? 0u : c - 2u);
            } else {
              lmask_s[grp] = 0u;
            }
          }
        }
        if (!fast) act4 = 0;
        if (!fast && gtid == 0) accz[grp] = 0;
      }
      if (!fast && arm_warp) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint8_t a = (uint8_t)(A4 >> (8 * k));
          if (dn || a > MAX_LEVELS || p0 + pp + k >= g.n) a = 0;
          act4 |= (uint32_t)a << (8 * k);
          hist_add(lcnt[grp], a ? a - 1u : NONE);
        }
        if (in) *reinterpret_cast<uint32_t *>(sact + e4) = act4;
      }
      if (!fast) bsync();  // lcnt
      if (!fast && gtid < 32) {  // per-level offsets, the level mask and the statistics: one warp
        const unsigned v = gtid < MAX_LEVELS ? lcnt[grp][gtid] : 0u;
        unsigned x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(FULL, x, o);
          if (gtid >= o) x += y;
        }
        if (gtid < MAX_LEVELS) {
          loff[grp][gtid] = x - v;
          lfill[grp][gtid] = x - v;
        }
        if (gtid == MAX_LEVELS - 1) loff[grp][MAX_LEVELS] = x;
        const unsigned lm = __ballot_sync(FULL, v != 0u);
        unsigned long long dr = (unsigned long long)v << gtid, bl = (unsigned long long)v << (gtid < 2 ? 0 : gtid - 2);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          dr += __shfl_xor_sync(FULL, dr, o);
          bl += __shfl_xor_sync(FULL, bl, o);
        }
        if (gtid == 0) {
          lmask_s[grp] = lm;
          my_dr += dr;  // statistics: per group in a register, one shared atomic at the end
          my_bl += bl;  // (64-bit shared atomics are CAS loops: once per tile cost ~1 %)
        }
      }
      if (!fast) bsync();
      if (!fast && arm_warp) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint8_t a = (uint8_t)(act4 >> (8 * k));
          const unsigned key = a ? a - 1u : NONE;
          const unsigned m = __match_any_sync(FULL, key);
          const int leader = __ffs(m) - 1;
          unsigned b0 = 0;
          if (a && lane_id() == leader) b0 = atomicAdd(&lfill[grp][key], (unsigned)__popc(m));
          b0 = __shfl_sync(FULL, b0, leader);
          if (a) lst[b0 + __popc(m & ((1u << lane_id()) - 1u))] = (uint16_t)(e4 + k);
        }
      }
      if (!QG) {
        wait_bar(qbar0 + 8u * (uint32_t)sel, (qphase >> sel) & 1u);  // the query rows
        qphase ^= 1u << sel;
      }
      if (!have_x) {  // the column's point rows (once per column and group)
        wait_bar(pbar_s, pphase);
        have_x = true;
      }
      gsync();
      unsigned lmask = lmask_s[grp];
      for (; lmask; lmask &= lmask - 1) {
        const int c = __ffs(lmask) - 1;
        const unsigned m = lcnt[grp][c];
        const int lb = c < 2 ? 0 : c - 2;
        const unsigned s = 1u << c, nb = 1u << lb;
        const uint16_t *L = lst + loff[grp][c];
        const uint32_t lv = (uint32_t)(c + 1);
        if (nb <= (unsigned)ADV_TP) {
          const unsigned ppt = ADV_TP / nb;
          for (unsigned l0 = gtid; l0 < m; l0 += GT * ppt) {
            uint4 w[ADV_TP];
            int pr[ADV_TP];
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) {
              const unsigned li = l0 + (k / nb) * GT;
              const bool ok = (unsigned)k / nb < ppt && li < m;
              pr[k] = ok ? (int)L[li] : -1;
              const int e = ok ? pr[k] : 0;
              const uint32_t gi = (uint32_t)(p0 + (e & (P - 1))) + g.id_offset;
              const uint32_t gq = rng_qi(g, (uint32_t)(r0 + (e >> g.tile_lp)));
              w[k] = philox4x32_10_rk(make_uint4((uint32_t)k & (nb - 1), gi, gq, lv), g.rk0, g.rk1);
            }
            uint32_t sum = 0;
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) {
              if (QG && pr[k] >= 0) {
                const uint32_t xa = xs + (uint32_t)(pr[k] & (P - 1)) * stride;
                const uint8_t *qp = g.Q + (size_t)(r0 + (pr[k] >> g.tile_lp)) * pitch;
                if (s >= 4) {
                  sum = sq_diff4_g<TIGHT>(xa, qp, w[k], d, sum);
                } else {
                  sum += sq_diff_g<TIGHT>(xa, qp, coord_of(w[k].x, d));
                  if (s == 2) sum += sq_diff_g<TIGHT>(xa, qp, coord_of(w[k].y, d));
                }
              } else if (pr[k] >= 0) {
                const uint32_t xa = xs + (uint32_t)(pr[k] & (P - 1)) * stride;
                const uint32_t qa = qs + (uint32_t)(pr[k] >> g.tile_lp) * stride;
                if (s >= 4) {
                  sum = TIGHT ? sq_diff4_t(xa, qa, w[k], d, sum) : sq_diff4(xa, qa, w[k], d, sum);
                } else {
                  sum += TIGHT ? sq_diff_t(xa, qa, coord_of(w[k].x, d)) : sq_diff(xa, qa, coord_of(w[k].x, d));
                  if (s == 2)
                    sum += TIGHT ? sq_diff_t(xa, qa, coord_of(w[k].y, d)) : sq_diff(xa, qa, coord_of(w[k].y, d));
                }
              }
              if ((unsigned)(k + 1) % nb == 0) {
                if (pr[k] >= 0) acc[pr[k]] = (int32_t)sum;
                sum = 0;
              }
            }
          }
        } else {
          if (!(RP <= 32 && accz[grp])) {  // (the one-level fast path zeroed them)
            for (unsigned l = gtid; l < m; l += GT) acc[L[l]] = 0;
            gsync();
          }
          const unsigned lg = (unsigned)(lb - 2);
          const unsigned total = m << lg;
          // The plain kernel: each thread takes a CONTIGUOUS run of items, so the pair's
          // constants (its row addresses, Philox round-0/1 products) and its shared
          // atomic are paid once per run of one pair instead of once per item (C3 top
          // level 106.1 -> 103.0 ms, 2,048 draws 54.6 -> 53.5; the middle levels lose
          // ~0.5 ms each).  QG super tiles keep the strided deal (its registers: the
          // contiguous form spilled there and ran 6.1 vs 5.7 ms).
          const unsigned per = (total + GT - 1) / GT;
          if (QG) {
            for (unsigned it = gtid; it < total; it += GT) {
              const unsigned li = it >> lg, b0 = (it & ((1u << lg) - 1u)) * ADV_TP;
              const int pe1 = (int)L[li];
              const uint32_t xa1 = xs + (uint32_t)(pe1 & (P - 1)) * stride;
              const uint32_t qa1 = qs + (uint32_t)(pe1 >> g.tile_lp) * stride;
              const uint32_t gi = (uint32_t)(p0 + (pe1 & (P - 1))) + g.id_offset;
              const uint32_t gq = rng_qi(g, (uint32_t)(r0 + (pe1 >> g.tile_lp)));
              const PhiloxPair pc1 = philox_pair(gi, gq, g.rk0);
              uint4 w[ADV_TP];
#pragma unroll
              for (int k = 0; k < ADV_TP; ++k) w[k] = philox_from_pair(b0 + k, lv, pc1, g.rk0, g.rk1);
              uint32_t sum1 = 0;
              if (QG) {
                const uint8_t *qp1 = g.Q + (size_t)(r0 + (pe1 >> g.tile_lp)) * pitch;
#pragma unroll
                for (int k = 0; k < ADV_TP; ++k) sum1 = sq_diff4_g<TIGHT>(xa1, qp1, w[k], d, sum1);
              } else {
#pragma unroll
                for (int k = 0; k < ADV_TP; ++k)
                  sum1 = TIGHT ? sq_diff4_t(xa1, qa1, w[k], d, sum1) : sq_diff4(xa1, qa1, w[k], d, sum1);
              }
              atomicAdd(reinterpret_cast<uint32_t *>(acc + pe1), sum1);
            }
            continue;  // the next level
          }
          const unsigned it1 = min(total, (unsigned)gtid * per + per);
          int pe = -1;
          uint32_t xa = 0, qa = 0, sum = 0;
          PhiloxPair pc{};
          const uint8_t *qp = nullptr;
          for (unsigned it = (unsigned)gtid * per; it < it1; ++it) {
            const unsigned li = it >> lg, b0 = (it & ((1u << lg) - 1u)) * ADV_TP;
            if (b0 == 0 || pe < 0) {  // a new pair
              if (pe >= 0) atomicAdd(reinterpret_cast<uint32_t *>(acc + pe), sum);
              sum = 0;
              pe = (int)L[li];
              xa = xs + (uint32_t)(pe & (P - 1)) * stride;
              qa = qs + (uint32_t)(pe >> g.tile_lp) * stride;
              if (QG) qp = g.Q + (size_t)(r0 + (pe >> g.tile_lp)) * pitch;
              const uint32_t gi = (uint32_t)(p0 + (pe & (P - 1))) + g.id_offset;
              const uint32_t gq = rng_qi(g, (uint32_t)(r0 + (pe >> g.tile_lp)));
              pc = philox_pair(gi, gq, g.rk0);
            }
            uint4 w[ADV_TP];
#pragma unroll
            for (int k = 0; k < ADV_TP; ++k) w[k] = philox_from_pair(b0 + k, lv, pc, g.rk0, g.rk1);
            if (QG) {
#pragma unroll
              for (int k = 0; k < ADV_TP; ++k) sum = sq_diff4_g<TIGHT>(xa, qp, w[k], d, sum);
            } else {
#pragma unroll
              for (int k = 0; k < ADV_TP; ++k)
                sum = TIGHT ? sq_diff4_t(xa, qa, w[k], d, sum) : sq_diff4(xa, qa, w[k], d, sum);
            }
          }
          if (pe >= 0) atomicAdd(reinterpret_cast<uint32_t *>(acc + pe), sum);
        }
      }
      gsync();
      // the slot is free (every read of this tile's query rows is behind the barrier):
      // the next tile's copy starts now, ahead of the commit and the next bookkeeping
      if (!QG && !DB && gtid == 0 && trn < rows) issue_rows(trn, sel);
      if (act4) {  // commit: S += the level's sum, T -> 2T (the thread's own 4 arms)
        int4 o = S4;
        uint32_t l4 = L4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t a = (act4 >> (8 * k)) & 0xFFu;
          if (!a) continue;
          const int32_t add = acc[e4 + k];
          if (k == 0) o.x += add;
          if (k == 1) o.y += add;
          if (k == 2) o.z += add;
          if (k == 3) o.w += add;
          l4 = (l4 & ~(0xFFu << (8 * k))) | (a << (8 * k));
        }
        *reinterpret_cast<int4 *>(g.S + o4) = o;
        *reinterpret_cast<uint32_t *>(g.lvl + o4) = l4;
      }
      first = false;
      if (DB) sel ^= 1;
    }
    if (!have_x) wait_bar(pbar_s, pphase);  // a group without tiles in this column
    pphase ^= 1u;
  }
  if (gtid == 0) {
    if (my_bl) atomicAdd(&s_blocks, my_bl);
    if (my_dr) atomicAdd(&s_draws, my_dr);
  }
  __syncthreads();
  if (tid == 0 && s_blocks) atomicAdd(&g.ctl->tile_blocks, s_blocks);
  if (tid == 0 && s_draws) atomicAdd(&g.ctl->tile_draws, s_draws);
}

// ---------------------------------------------------------------------------
// |x - q| tiles: the largest levels of rows wider than 8 KB (C3's 2,048 and 4,096 draws
// per pair).  ncu on the grouped kernel at 4,096 draws: shared-memory wavefronts at ~95 %
// of one per cycle per SM (two random byte gathers per draw, ~4.6 wavefronts per warp
// load from bank conflicts) -- above the Philox work (fma-heavy 79 %).  Here a tile's
// pairs first get their row z_p[j] = |x_p[j] - q[j]| (u8, exact) written once, with
// 16-byte conflict-free loads and stores, and every draw then gathers ONE byte:
// (x_j - q_j)^2 = z_j^2 summed by IDP.4A, the same integer sum as k_advance_tiles_grp and
// the oracle.  Materialising z costs ~d bytes per pair, so it pays only where a pair
// draws a large share of d (tilework >= tile_z_draws, chosen on the host).
//
// One CTA per SM walks whole point columns (R = 1 query x P = 8 points per tile, the
// grouped shape): the column's P raw point rows are staged once by bulk TMA, the query
// row of each tile by bulk TMA one tile ahead.  Warp-specialised, a job = half a tile
// (TZ_H pairs) in one of two z buffers with full / empty mbarriers:
//   4 producer warps   write the job's z rows;
//   1 bookkeeper warp  loads each job's actions / S / levels one job ahead, publishes the
//                      actions, and commits a job (S += its sums, level set) once its
//                      buffer is released -- off the draw path;
//   16 consumer warps  run the Philox draws: per item (one pair, 4 Philox blocks) a warp
//                      reduction (REDUX) and one shared atomic into the job's pair sums.
// A job at 2,048 / 4,096 draws per pair is 512 / 1,024 items: one / two per consumer.
constexpr int TZ_PW = 4, TZ_BW = 1, TZ_CW = 16;  // producer / bookkeeper / consumer warps
constexpr int TZ_NT = 32 * (TZ_PW + TZ_BW + TZ_CW);
constexpr int TZ_H = 4;                             // pairs per job (half a P = 8 tile)
constexpr int TZ_CM = 256;                          // mask words: rows <= 8192

__device__ __forceinline__ void sts_u128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "ZW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra ZW_%=;\n\t}" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tma_row(uint32_t dst, const uint8_t *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// Four draws (one Philox block) from a z row: one byte gather each, |x - q|^2 summed.
__device__ __forceinline__ uint32_t z_sq4(uint32_t za, uint4 w, uint32_t d, uint32_t acc) {
  const uint32_t b0 = lds_u8(za + coord_of(w.x, d)), b1 = lds_u8(za + coord_of(w.y, d));
  const uint32_t b2 = lds_u8(za + coord_of(w.z, d)), b3 = lds_u8(za + coord_of(w.w, d));
  const uint32_t t = __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
  return __dp4a(t, t, acc);
}

// One job's arm state as the bookkeeper holds it until the commit.
struct ZJob {
  int4 S4;
  uint32_t L4, act4;
  long long o4;  // offset of the job's first arm in S / lvl / act
};

__global__ void __launch_bounds__(TZ_NT, 1) k_advance_tiles_z(Geom g) {
  if ((float)g.ctl->tile_max < fmaxf(g.tile_z_draws, g.tile_min_draws)) return;  // no z tile this pass
  extern __shared__ __align__(16) unsigned char tsm[];
  __shared__ __align__(8) uint64_t bar_zf[2], bar_ze[2], bar_q[2], bar_x;
  __shared__ uint32_t colmask[TZ_CM];
  __shared__ uint32_t zacc[2][TZ_H], zact[2], ztr[2];
  __shared__ unsigned long long s_blocks, s_draws;
  constexpr int NJ = 2;  // jobs per tile (P = 2 TZ_H)
  const int P = 1 << g.tile_lp;
  const uint32_t pitch = (uint32_t)g.pitch, d = (uint32_t)g.d;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(tsm);
  const uint32_t xs = base;                             // the column's P raw point rows
  const uint32_t zs = xs + (uint32_t)P * pitch;         // 2 buffers x TZ_H z rows
  const uint32_t qsm = zs + 2u * TZ_H * pitch;          // 2 query rows
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    if (P != NJ * TZ_H || qsm + 2u * pitch > base + dyn) __trap();  // host sizing broken: fail loudly
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int role = warp < TZ_PW ? 0 : (warp < TZ_PW + TZ_BW ? 1 : 2);  // producer / bookkeeper / consumer
  const int rows = g.q;  // R = 1
  const int cols = (g.n + P - 1) >> g.tile_lp;
  const int nw = (rows + 31) >> 5;
  // only DENSE tiles (k_scatter leaves their pairs out of the lists) are z tiles
  const float zthr = fmaxf(g.tile_z_draws, g.tile_min_draws);
  auto sa = [](const void *p) { return (uint32_t)__cvta_generic_to_shared(p); };
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar_zf[b])), "r"(TZ_PW * 32 + 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar_ze[b])), "r"(TZ_CW * 32));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_q[b])));
      for (int e = 0; e < TZ_H; ++e) zacc[b][e] = 0;
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar_x)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_blocks = s_draws = 0;
  }
  __syncthreads();
  auto issue_q = [&](int tr, uint32_t b) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar_q[b])), "r"(pitch) : "memory");
    tma_row(qsm + b * pitch, g.Q + (size_t)tr * pitch, pitch, sa(&bar_q[b]));
  };
  // bookkeeper: a job's arm state (actions filtered as the grouped kernel filters them)
  auto load_job = [&](int tr, int pb) {
    ZJob jb;
    jb.o4 = (long long)tr * g.npad + pb;
    const uint32_t a4 = g.qs[tr].done ? 0u : *reinterpret_cast<const uint32_t *>(g.act + jb.o4);
    jb.S4 = *reinterpret_cast<const int4 *>(g.S + jb.o4);
    jb.L4 = *reinterpret_cast<const uint32_t *>(g.lvl + jb.o4);
    jb.act4 = 0;
#pragma unroll
    for (int e = 0; e < TZ_H; ++e) {
      uint32_t a = (a4 >> (8 * e)) & 0xFFu;
      if (a > (uint32_t)MAX_LEVELS || pb + e >= g.n) a = 0;
      jb.act4 |= a << (8 * e);
    }
    return jb;
  };
  unsigned long long my_bl = 0, my_dr = 0;
  auto commit = [&](const ZJob &jb, uint32_t zb) {  // bookkeeper, after the job's buffer is released
    if (!jb.act4) return;
    int4 S4 = jb.S4;
    uint32_t l4 = jb.L4;
#pragma unroll
    for (int e = 0; e < TZ_H; ++e) {
      const uint32_t a = (jb.act4 >> (8 * e)) & 0xFFu;
      const int32_t v = (int32_t)zacc[zb][e];
      zacc[zb][e] = 0u;
      if (!a) continue;
      if (e == 0) S4.x += v;
      if (e == 1) S4.y += v;
      if (e == 2) S4.z += v;
      if (e == 3) S4.w += v;
      l4 = (l4 & ~(0xFFu << (8 * e))) | (a << (8 * e));
      my_dr += 1ull << (a - 1u);
      my_bl += a <= 3u ? 1ull : 1ull << (a - 3u);
    }
    *reinterpret_cast<int4 *>(g.S + jb.o4) = S4;
    *reinterpret_cast<uint32_t *>(g.lvl + jb.o4) = l4;
  };
  ZJob pend0{}, pend1{};  // bookkeeper: the jobs awaiting their commit, by buffer
  uint32_t jz = 0, tq = 0, xc = 0;  // jobs / tiles / columns so far (identical in every role)
  const int c0 = (int)((long long)blockIdx.x * cols / gridDim.x), c1 = (int)((long long)(blockIdx.x + 1) * cols / gridDim.x);
  for (int tp = c0; tp < c1; ++tp) {
    __syncthreads();  // every role is done with the previous column
    for (int w = tid; w < nw; w += TZ_NT) colmask[w] = 0u;
    __syncthreads();
    bool any = false;
    for (int tr = tid; tr < rows; tr += TZ_NT)
      if ((float)g.tilework[(size_t)tr * g.tile_cols + tp] >= zthr) {
        any = true;
        atomicOr(&colmask[tr >> 5], 1u << (tr & 31));
      }
    if (!__syncthreads_or(any)) continue;
    const int p0 = tp << g.tile_lp;
    auto next_tile = [&](int tr) {  // the first z tile at or after row tr
      for (int w = tr >> 5; w < nw; ++w) {
        uint32_t m = colmask[w];
        if (w == (tr >> 5)) m &= ~0u << (tr & 31);
        if (m) return w * 32 + __ffs(m) - 1;
      }
      return rows;
    };
    const int tr0 = next_tile(0);
    int ntl = 0;
    for (int w = 0; w < nw; ++w) ntl += __popc(colmask[w]);
    if (tid == 0) {  // the column's point rows, the first tile's query row
      uint32_t bytes = 0;
      for (int row = 0; row < P; ++row) bytes += p0 + row < g.n ? pitch : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar_x)), "r"(bytes) : "memory");
      for (int row = 0; row < P; ++row)
        if (p0 + row < g.n) tma_row(xs + (uint32_t)row * pitch, g.X + (size_t)(p0 + row) * pitch, pitch, sa(&bar_x));
      issue_q(tr0, tq & 1u);
    }
    if (role == 0) {
      uint32_t t = tq, j = jz;
      mbar_wait_parity(sa(&bar_x), xc & 1u);
      const uint32_t n16 = pitch >> 4;
      for (int tr = tr0; tr < rows;) {
        const int trn = next_tile(tr + 1);
        asm volatile("bar.sync 1, %0;" ::"r"(TZ_PW * 32) : "memory");  // the other query buffer is free
        if (tid == 0 && trn < rows) issue_q(trn, (t + 1u) & 1u);
        mbar_wait_parity(sa(&bar_q[t & 1u]), (t >> 1) & 1u);
        const uint32_t qa = qsm + (t & 1u) * pitch;
#pragma unroll 1
        for (int h = 0; h < NJ; ++h, ++j) {
          const uint32_t zb = j & 1u;
          if (j >= 2) mbar_wait_parity(sa(&bar_ze[zb]), ((j >> 1) + 1u) & 1u);  // job j - 2 consumed
          const uint32_t zdst = zs + zb * TZ_H * pitch, xsrc = xs + (uint32_t)(h * TZ_H) * pitch;
          // two 16-byte columns per step: 10 loads in flight before the stores
          for (uint32_t c = tid; c < n16; c += 2 * TZ_PW * 32) {
            const uint32_t c2 = c + TZ_PW * 32;
            const bool two = c2 < n16;
            const uint4 qv = lds_u128(qa + c * 16u), qw = two ? lds_u128(qa + c2 * 16u) : qv;
            uint4 xv[TZ_H], xw[TZ_H];
#pragma unroll
            for (int e = 0; e < TZ_H; ++e) {
              xv[e] = lds_u128(xsrc + (uint32_t)e * pitch + c * 16u);
              xw[e] = two ? lds_u128(xsrc + (uint32_t)e * pitch + c2 * 16u) : xv[e];
            }
#pragma unroll
            for (int e = 0; e < TZ_H; ++e) {
              sts_u128(zdst + (uint32_t)e * pitch + c * 16u,
                       make_uint4(__vabsdiffu4(xv[e].x, qv.x), __vabsdiffu4(xv[e].y, qv.y),
                                  __vabsdiffu4(xv[e].z, qv.z), __vabsdiffu4(xv[e].w, qv.w)));
              if (two)
                sts_u128(zdst + (uint32_t)e * pitch + c2 * 16u,
                         make_uint4(__vabsdiffu4(xw[e].x, qw.x), __vabsdiffu4(xw[e].y, qw.y),
                                    __vabsdiffu4(xw[e].z, qw.z), __vabsdiffu4(xw[e].w, qw.w)));
            }
          }
          mbar_arrive1(sa(&bar_zf[zb]));
        }
        ++t;
        tr = trn;
      }
    } else if (role == 1) {
      if (lane == 0) {
        uint32_t j = jz;
        int tr = tr0, h = 0;
        ZJob cur = load_job(tr, p0);
        while (tr < rows) {
          const int trc = tr;
          if (++h == NJ) {
            h = 0;
            tr = next_tile(tr + 1);
          }
          ZJob nxt{};
          if (tr < rows) nxt = load_job(tr, p0 + h * TZ_H);  // in flight during this job
          const uint32_t zb = j & 1u;
          if (j >= 2) mbar_wait_parity(sa(&bar_ze[zb]), ((j >> 1) + 1u) & 1u);  // job j - 2 consumed
          if (zb == 0) {
            if (j >= 2) commit(pend0, 0u);
            pend0 = cur;
          } else {
            if (j >= 2) commit(pend1, 1u);
            pend1 = cur;
          }
          zact[zb] = cur.act4;
          ztr[zb] = (uint32_t)trc;
          mbar_arrive1(sa(&bar_zf[zb]));
          cur = nxt;
          ++j;
        }
      }
      __syncwarp();
    } else {
      const uint32_t cw = (uint32_t)(warp - TZ_PW - TZ_BW);
      uint32_t j = jz;
      const int njobs = ntl * NJ;
      for (int jj = 0; jj < njobs; ++jj, ++j) {
        const uint32_t zb = j & 1u;
        mbar_wait_parity(sa(&bar_zf[zb]), (j >> 1) & 1u);
        const uint32_t act4 = zact[zb], trc = ztr[zb];
        const int pb = p0 + (jj & 1) * TZ_H;
        // items: (pair e, 4 consecutive Philox blocks of its level)
        uint32_t ni[TZ_H];
#pragma unroll
        for (int e = 0; e < TZ_H; ++e) {
          const uint32_t a = (act4 >> (8 * e)) & 0xFFu;
          ni[e] = a == 0u ? 0u : (a <= 5u ? 1u : (1u << (a - 5u)));  // ceil(nb / 4), nb = 2^max(c-2,0)
        }
        const uint32_t n0 = ni[0], n01 = n0 + ni[1], n012 = n01 + ni[2], nall = n012 + ni[3];
        const uint32_t gq = rng_qi(g, trc);
        const uint32_t zb0 = zs + zb * TZ_H * pitch;
        for (uint32_t it0 = cw * 32u; it0 < nall; it0 += TZ_CW * 32u) {  // warp-uniform
          const uint32_t it = it0 + (uint32_t)lane;
          const bool valid = it < nall;
          const uint32_t e = it < n01 ? (it < n0 ? 0u : 1u) : (it < n012 ? 2u : 3u);
          uint32_t sum = 0;
          if (valid) {
            const uint32_t k = it - (e == 0u ? 0u : e == 1u ? n0 : e == 2u ? n01 : n012);
            const uint32_t a = (act4 >> (8 * e)) & 0xFFu, c = a - 1u;
            const uint32_t gi = (uint32_t)(pb + (int)e) + g.id_offset;
            const PhiloxPair pc = philox_pair(gi, gq, g.rk0);
            const uint32_t za = zb0 + e * pitch;
            if (c >= 4u) {  // 4 whole blocks
              uint4 w[ADV_TP];
#pragma unroll
              for (int kk = 0; kk < ADV_TP; ++kk) w[kk] = philox_from_pair(4u * k + kk, a, pc, g.rk0, g.rk1);
#pragma unroll
              for (int kk = 0; kk < ADV_TP; ++kk) sum = z_sq4(za, w[kk], d, sum);
            } else {  // levels 0-3: 1, 2, 4 or 8 draws (blocks 0 and, at level 3, 1)
              const uint4 w0 = philox_from_pair(0u, a, pc, g.rk0, g.rk1);
              if (c >= 2u) {
                sum = z_sq4(za, w0, d, 0u);
                if (c == 3u) sum = z_sq4(za, philox_from_pair(1u, a, pc, g.rk0, g.rk1), d, sum);
              } else {
                const uint32_t b0 = lds_u8(za + coord_of(w0.x, d));
                sum = b0 * b0;
                if (c == 1u) {
                  const uint32_t b1 = lds_u8(za + coord_of(w0.y, d));
                  sum += b1 * b1;
                }
              }
            }
          }
          // the warp's items usually belong to one pair: one REDUX + one shared atomic
          const uint32_t e0 = __shfl_sync(FULL, e, 0);
          if (__all_sync(FULL, !valid || e == e0)) {
            const uint32_t tot = __reduce_add_sync(FULL, sum);
            if (lane == 0 && tot) atomicAdd(&zacc[zb][e0], tot);
          } else if (valid && sum) {
            atomicAdd(&zacc[zb][e], sum);
          }
        }
        mbar_arrive1(sa(&bar_ze[zb]));
      }
    }
    tq += (uint32_t)ntl;
    jz += (uint32_t)ntl * NJ;
    ++xc;
  }
  if (role == 1 && lane == 0) {  // the last two jobs: wait for their consumers, commit
    for (uint32_t j = jz >= 2 ? jz - 2 : 0; j < jz; ++j) {
      const uint32_t zb = j & 1u;
      mbar_wait_parity(sa(&bar_ze[zb]), (j >> 1) & 1u);
      commit(zb == 0 ? pend0 : pend1, zb);
    }
    if (my_bl) atomicAdd(&s_blocks, my_bl);
    if (my_dr) atomicAdd(&s_draws, my_dr);
  }
  __syncthreads();
  if (tid == 0 && s_blocks) atomicAdd(&g.ctl->tile_blocks, s_blocks);
  if (tid == 0 && s_draws) atomicAdd(&g.ctl->tile_draws, s_draws);
}

int tile_slot_log2(int64_t pitch) {
  int l = 4;
  while ((1ll << l) < pitch) ++l;
  return l;
}

// The tile kernel's shared-memory window per CTA (static + reserved + dynamic), given
// where its dynamic region starts (`base`): the small arrays, then the row slots from
// the next slot boundary.
static size_t tile_window(int lr, int lp, int64_t pitch, size_t base) {
  const size_t R = (size_t)1 << lr, P = (size_t)1 << lp, slot = (size_t)1 << tile_slot_log2(pitch);
  const size_t rows0 = (base + R * P * 7 + slot - 1) / slot * slot;
  return rows0 + (R + P) * slot;
}

static size_t tile_base() {  // static shared memory + the per-CTA system reservation
  static size_t b = [] {
    cudaFuncAttributes fa{};
    int dev = 0, rsv = 0;
    cudaFuncAttributes fb{};
    if (cudaFuncGetAttributes(&fa, k_advance_tiles<0, TILE_NT>) != cudaSuccess) fa.sharedSizeBytes = 2048;
    auto widen = [&](const void *f) {
      if (cudaFuncGetAttributes(&fb, f) == cudaSuccess && fb.sharedSizeBytes > fa.sharedSizeBytes)
        fa.sharedSizeBytes = fb.sharedSizeBytes;
    };
    widen((const void *)k_advance_tiles<1, TILE_NT>);
    widen((const void *)k_advance_tiles<2, TILE_NT>);
    widen((const void *)k_advance_tiles<0, TILE_NT_WIDE>);
    widen((const void *)k_advance_tiles<2, TILE_NT_WIDE>);
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess)
      rsv = 1024;
    return (size_t)fa.sharedSizeBytes + (size_t)rsv;
  }();
  return b;
}

// Shared memory per CTA of a tile shape (the occupancy the shape chooser reasons about).
size_t tile_smem_bytes(int lr, int lp, int64_t pitch) { return tile_window(lr, lp, pitch, tile_base()); }

// AKNN_TILE_WIDE=0 keeps 8-warp CTAs at one CTA per SM (A/B measurements).
static bool env_tile_wide() {
  static const bool v = [] {
    const char *e = getenv("AKNN_TILE_WIDE");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Dynamic shared memory of one instantiation: its own static size + the reservation
// places the dynamic window (the slot alignment of the rows depends on where it starts).
template <int MODE, int NT>
static size_t tiles_dyn_smem(const Geom &g) {
  cudaFuncAttributes fa{};
  int dev = 0, rsv = 0;
  if (cudaFuncGetAttributes(&fa, k_advance_tiles<MODE, NT>) != cudaSuccess) fa.sharedSizeBytes = 2048;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess)
    rsv = 1024;
  const size_t base = (size_t)fa.sharedSizeBytes + (size_t)rsv;
  return tile_window(g.tile_lr, g.tile_lp, g.pitch, base) - base;
}

template <int MODE, int NT>
static cudaError_t launch_tiles_nt(const Geom &g, int num_sms, int *per_sm, cudaStream_t s) {
  const size_t smem = tiles_dyn_smem<MODE, NT>(g);
  cudaError_t e = cudaFuncSetAttribute(k_advance_tiles<MODE, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_advance_tiles<MODE, NT>, NT, smem);
  if (e != cudaSuccess) return e;
  if (*per_sm < 1) return cudaErrorInvalidConfiguration;
  k_advance_tiles<MODE, NT><<<num_sms * *per_sm, NT, smem, s>>>(g);
  return cudaGetLastError();
}

// 8-warp CTAs, or one 20-warp CTA per SM when the shape leaves room for one CTA only
template <int MODE>
static cudaError_t launch_tiles_k(const Geom &g, int num_sms, cudaStream_t s) {
  int per_sm = 0;
  const size_t smem = tiles_dyn_smem<MODE, TILE_NT>(g);
  cudaError_t e = cudaFuncSetAttribute(k_advance_tiles<MODE, TILE_NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_advance_tiles<MODE, TILE_NT>, TILE_NT, smem);
  if (e != cudaSuccess) return e;
  // bulk TMA row staging pays at one CTA per SM (C3: -3 % tile time), where nothing else
  // hides the staging latency; with 2-3 CTAs per SM (C2, C4) 16-byte cp.async is faster
  // (bulk copies: +7 % / +10 % tile time, measured)
  Geom gt = g;
  if (MODE != 1 && per_sm <= 1 && env_tile_wide()) {
    int wide = 0;
    if (launch_tiles_nt<MODE == 1 ? 0 : MODE, TILE_NT_WIDE>(gt, num_sms, &wide, s) == cudaSuccess) return cudaSuccess;
    cudaGetLastError();
  }
  gt.tile_tma = per_sm <= 1 ? g.tile_tma : 0;
  return launch_tiles_nt<MODE, TILE_NT>(gt, num_sms, &per_sm, s);
}

template <int NG, bool TIGHT, bool DB, int NTT = TILE_NT_WIDE, bool QG = false>
static cudaError_t launch_tiles_grp(const Geom &g, int num_sms, cudaStream_t s) {
  cudaFuncAttributes fa{};
  int dev = 0, rsv = 0;
  if (cudaFuncGetAttributes(&fa, k_advance_tiles_grp<NG, TIGHT, DB, NTT, QG>) != cudaSuccess) fa.sharedSizeBytes = 4096;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev) != cudaSuccess)
    rsv = 1024;
  const size_t base = (size_t)fa.sharedSizeBytes + (size_t)rsv;
  const size_t R = (size_t)1 << (QG ? QG_LR : g.tile_lr), P = (size_t)1 << g.tile_lp, slot = (size_t)1 << g.tile_slot_l;
  const size_t gsz = (R * P * 7 + 15) & ~(size_t)15;
  const size_t rows0 = TIGHT ? base + NG * gsz : (base + NG * gsz + slot - 1) / slot * slot;
  const size_t smem = rows0 + ((QG ? 0 : DB ? 2 : 1) * NG * R + P) * (TIGHT ? (size_t)g.pitch : slot) - base;
  cudaError_t e = cudaFuncSetAttribute(k_advance_tiles_grp<NG, TIGHT, DB, NTT, QG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_advance_tiles_grp<NG, TIGHT, DB, NTT, QG><<<num_sms, NTT, smem, s>>>(g);
  return cudaGetLastError();
}

// Shared memory of a grouped shape (the chooser's test): tight = rows at the pitch.
size_t tile_grp_smem_bytes(int groups, int lr, int lp, int64_t pitch, bool tight, bool db) {
  const size_t R = (size_t)1 << lr, P = (size_t)1 << lp, slot = (size_t)1 << tile_slot_log2(pitch);
  const size_t base = 4096 + 1024, gsz = (R * P * 7 + 15) & ~(size_t)15, qrows = (db ? 2 : 1) * groups * R;
  if (tight) return base + groups * gsz + (qrows + P) * (size_t)pitch;
  return (base + groups * gsz + slot - 1) / slot * slot + (qrows + P) * slot;
}

static size_t tiles_z_smem(int lp, int64_t pitch) { return (size_t)((1 << lp) + 2 * TZ_H + 2) * (size_t)pitch; }

bool tile_z_ok(int lr, int lp, int64_t pitch, int64_t q) {
  if (lr != 0 || (1 << lp) != 2 * TZ_H || pitch % 16 != 0 || q > (int64_t)TZ_CM * 32) return false;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, k_advance_tiles_z) != cudaSuccess) return false;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  return fa.sharedSizeBytes + tiles_z_smem(lp, pitch) <= (size_t)optin;
}

static cudaError_t launch_tiles_z(const Geom &g, int num_sms, cudaStream_t s) {
  const size_t smem = tiles_z_smem(g.tile_lp, g.pitch);
  cudaError_t e = cudaFuncSetAttribute(k_advance_tiles_z, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_advance_tiles_z<<<num_sms, TZ_NT, smem, s>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_advance_tiles(const Geom &g0, int num_sms, cudaStream_t s) {
  if (g0.tile_groups && !g0.wor && !(g0.shared_draws && g0.tile_lr == 5)) {
    // the dense tiles by tilework: [0, qg) QG grouped kernel, [qg, z) grouped kernel,
    // [z, inf) |x - q| kernel (each bound 0 = that kernel off)
    const float zlo = g0.tile_z_draws > 0.f ? fmaxf(g0.tile_z_draws, g0.tile_min_draws) : INFINITY;
    const float qhi = fminf(g0.tile_qg_draws, zlo);
    if (g0.tile_z_draws > 0.f) {
      const cudaError_t e = launch_tiles_z(g0, num_sms, s);
      if (e != cudaSuccess) return e;
    }
    if (g0.tile_groups == 10 && qhi > g0.tile_min_draws) {
      Geom gq = g0;
      gq.tile_lo = 0.f;
      gq.tile_hi = qhi;
      const cudaError_t e = launch_tiles_grp<10, true, false, 640, true>(gq, num_sms, s);
      if (e != cudaSuccess) return e;
    }
    Geom g = g0;
    g.tile_lo = g0.tile_groups == 10 ? fmaxf(qhi, 0.f) : 0.f;
    g.tile_hi = zlo;
    if (g.tile_groups == 8) return launch_tiles_grp<8, true, false, 512>(g, num_sms, s);
    if (g.tile_groups == 10) return launch_tiles_grp<10, true, false, 640>(g, num_sms, s);
    if (g.tile_groups == 5) return launch_tiles_grp<5, true, false, 640>(g, num_sms, s);  // R = 2
    if (g.tile_groups == 24) return launch_tiles_grp<8, true, false, 768>(g, num_sms, s);  // 8 groups of 3 warps
    if (g.tile_groups == 4) return launch_tiles_grp<4, false, false>(g, num_sms, s);
    if (g.tile_groups == 2 && g.tile_tight) return launch_tiles_grp<2, true, false>(g, num_sms, s);
    if (g.tile_groups == 2 && g.tile_db) return launch_tiles_grp<2, false, true>(g, num_sms, s);
    if (g.tile_groups == 2) return launch_tiles_grp<2, false, false>(g, num_sms, s);
  }
  if (g0.shared_draws && g0.tile_lr == 5) return launch_tiles_k<1>(g0, num_sms, s);
  if (g0.wor) return launch_tiles_k<2>(g0, num_sms, s);
  return launch_tiles_k<0>(g0, num_sms, s);
}

}  // namespace aknn
