// internal.cuh -- shared device/host definitions of libaknn (product path).
//
// Nothing here is shared with oracle/: the Philox rounds, the Lemire map, the
// estimator and the key are written out again from the paper / DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace aknn {

// Level byte per (query, point) pair: c = log2 T (T = 2^c sampled draws so
// far); once the arm went exact (T = d) the byte is LVL_EXACT | c with c
// the last sampled level, so the arm's sampled draws (2^c) stay recoverable and
// the per-query counters are tallied from the final state (k_tally).
constexpr uint8_t LVL_EXACT = 0x80;
__host__ __device__ __forceinline__ bool lvl_exact(uint8_t l) { return (l & LVL_EXACT) != 0; }
__host__ __device__ __forceinline__ uint8_t lvl_to_exact(uint8_t l) { return (uint8_t)(l | LVL_EXACT); }
// Action byte written by the blocker filter: 0 = idle, c+1 = draw level c+1
// (T_c -> T_{c+1}), ACT_EXACT = exact fallback.
constexpr uint8_t ACT_EXACT = 0xFE;
// d <= 33025 -> sampled levels c in [0, 15] under doubling, [0, 30] under growth 2
// (reading R25); slot MAX_LEVELS = exact list.  Per-level bit masks are 32-bit.
constexpr int MAX_LEVELS = 32;
constexpr int NSLOT = MAX_LEVELS + 1;
static_assert(NSLOT <= 64, "k_plan: one thread per slot, two warps");

// Integer form of the blocker predicate of one query for a round (k_thresholds).
// Per sampled level c, int4 {Su, Sl, Ck, Ckh}:
//   U(S, c) > B            <=>  S >= Su
//   L(S, c) < A            <=>  S <  Sl
//   key(S, c, i) <= thr_k  <=>  S < Ck  or (eq_k bit c and S == Ck and gid <= id_k)
//   key(S, c, i) <= thr_kh <=>  S < Ckh or (eq_kh bit c and S == Ckh and gid <= id_kh)
// and a header {M mask (alpha(2^c) > alpha_d2), eq_k mask, eq_kh mask, id_k, id_kh}.
// Exact because U and L are monotone non-decreasing in S (one correctly rounded
// division, one addition) and the key is (S * (L / 2^c)) << kbits | gid.
// The table of a query holds nlev = cmax + 1 levels (only the sampled levels of the
// schedule): header at thr_hdr(nlev), row stride thr_stride(nlev) ints (16-B aligned).
constexpr int THR_LEVEL_INTS = 4 * MAX_LEVELS;
constexpr int THR_STRIDE = THR_LEVEL_INTS + 8;  // the largest stride
__host__ __device__ __forceinline__ int thr_hdr(int nlev) { return 4 * nlev; }
__host__ __device__ __forceinline__ int thr_stride(int nlev) { return 4 * nlev + 8; }

// Per-query state of the round loop (device memory, one per batch row).
struct QState {
  unsigned long long thr_k;   // composite key of rank k      (end of C)
  unsigned long long thr_kh;  // composite key of rank k + h  (end of M)
  double A;                   // max_{C} d_hat + alpha  (Eq. 2)
  double B;                   // min_{F} d_hat - alpha  (Eq. 3)
  double a_d2;                // alpha_{d2}             (Eq. 4 batched)
  int d1, d2;                 // local ids of d1, d2
  int done;                   // 1 once Eq. (5) held
  int fallback;               // 1: the one-pass pivot select could not decide this
                              //    round; the multi-pass radix select does
  int rounds;                 // rounds evaluated
  long long draws;            // sampled draws      } tallied from the final
  long long nexact;           // exact fallbacks    } arm states by k_tally
  long long exact_evals;      // evaluations charged for them (d each; d - T without replacement)
  long long blocks;           // Philox4x32-10 blocks the level gathers used
};

// Per-round control block (device memory; one per batch).
struct RoundCtl {
  unsigned int n_active;                  // queries failing Eq. (5) this round
  int gemm_level;                         // shared draws: the slot k_level_mma takes this round (-1: none)
  unsigned int cnt[NSLOT];                // pairs per action slot
  unsigned int off[NSLOT + 1];            // list offsets per slot
  unsigned int cursor[NSLOT];             // scatter cursors
  unsigned long long chunk_off[NSLOT + 1];// warp-chunk prefix per slot
  unsigned int wovf_any;                  // shared draws: some point's w_j > 255 this round
  unsigned int pad1;
  unsigned long long advanced;            // pairs advanced, cumulative
  unsigned long long tile_blocks;         // Philox blocks of the tile gathers, cumulative
  unsigned long long tile_draws;          // (query, point) draws of the tile gathers, cumulative
  unsigned long long lmma_tiles;          // 128 x 128 tiles run by k_level_mma, cumulative
  // cumulative, maintained on the device by k_round_ctl (graph-launched loop)
  unsigned int round;                     // rounds evaluated
  unsigned int evaluated;                 // queries the next rank split looks at
  unsigned long long qrounds, brounds;    // sums of evaluated / blocked queries
  unsigned int tile_max;                  // this pass: the largest tilework (k_filter), so the
                                          // tile kernels without a tile in their range exit at once
  unsigned int tile_min;                  // this pass: the smallest tilework of a dense tile
};

// One arm as exchanged between point shards: its composite key
// (global id in the low bits), exact integer sum S and level byte.  16 bytes.
struct ShardRec {
  unsigned long long key;
  int32_t S;
  uint8_t lvl;
  uint8_t pad[3];
};

// Everything a round kernel needs, passed by value.
// Domain Z_a x Z_b of the permutation network of sampling without replacement (R23).
struct WorRadix {
  uint32_t a, b, binv;  // binv = ceil(2^32 / b): x / b = umulhi(x, binv) for x < a b (b >= 2)
};

struct Geom {
  const uint8_t *X;      // [n][pitch] points (zero padded)
  const uint8_t *Q;      // [q][pitch] queries of this batch (zero padded)
  const double *alpha;   // [d+1]
  int32_t *S;            // [q][npad] exact integer sums
  uint8_t *lvl;          // [q][npad] level bytes
  uint8_t *act;          // [q][npad] action bytes
  uint32_t *list;        // work list, codes (qi << ibits) | i
  QState *qs;            // [q]
  RoundCtl *ctl;
  int64_t pitch;         // row pitch of X and Q (bytes, multiple of 16)
  int64_t npad;          // row pitch of S/lvl/act (elements, multiple of 16)
  int n;                 // local points
  int d;                 // dimension m
  int q;                 // queries in this batch
  int k, h;
  uint32_t id_offset;    // global id of local row 0
  uint32_t qi0;          // RNG query index of batch row 0
  int shared_draws;      // 1: query-independent draws: counter word 0xFFFFFFFF
  int lead;              // close-side lead L (aknn_opts.lead, reading R24): C/M blockers advance L times
  int lead_pass;         // 1: this filter decides a lead pass (from leadb and the levels reached)
  uint8_t *leadb;        // [q][npad] 1 = a blocker of this round ranked in C or M (lead > 1 only)
  int wor;               // 1: sampling without replacement (AKNN_FLAG_WITHOUT_REPLACEMENT, R23)
  WorRadix wor_z;        //    its Feistel domain Z_a x Z_b
  // shared draws on the tensor cores (exact_mma.cu, k_level_mma)
  int level_mma;         // 1: the round's dominant level runs as integer GEMMs
  uint8_t *q2lo, *q2hi;  // [q][pitch] q_j^2 byte planes
  uint8_t *wx0, *wx1, *wc;  // [n][pitch] w_j x_j (two bytes) and w_j of the level
  int32_t *wa;           // [n] sum_j w_j x_j^2
  uint8_t *wovf;         // [n] some w_j > 255: the point's pairs take the lists
  uint32_t *lvcnt;       // [ceil(q/128)][lv_cols][MAX_LEVELS] pairs per level in the 128 x 128 tile
  int lv_cols;
  uint32_t lmin;         // tiles with >= lmin pairs at the level run on the tensor cores
  uint32_t seed_lo, seed_hi;
  uint32_t rk0[10], rk1[10]; // Philox round keys of (seed_lo, seed_hi): kernel-param
                             // constants, so each round's key XOR is one LOP3
  unsigned long long L;  // lcm(T_0..T_cmax, d): K = S * (L / T) is an exact order key
  unsigned long long Ld; // L / d
  unsigned long long L3; // L / 3 (growth 2: the counts 3 * 2^j)
  int growth;            // sample-count schedule: 1 doubling (R7), 2 (reading R25)
  uint32_t exnext;       // bit c: the count after level c reaches d (the P:176 fallback)
  int ibits;             // bits of the local point index in a work-list code
  int kbits;             // bits of the GLOBAL point id in the composite key
  ShardRec *send;        // [q][k+h+1] this shard's summary (sharded query only)
  const ShardRec *recv;  // [world][recv_stride] every shard's summary
  int64_t recv_stride;   // records per shard slot of recv (qb * (k+h+1))
  int world;             // shards taking part (1 = unsharded)
  int cmax;              // largest sampled level (T_cmax < d)
  unsigned adv_bpl;      // advance: Philox blocks per lane before a lane-group reduce
  int force_radix;       // 1: skip the pivot select (aknn_opts.flags bit 0)
  int stage_lo;          // first row-staged advance level (MAX_LEVELS = none)
  // exact fallbacks on the tensor cores (exact_mma.cu, EpiFallback)
  int exact_mma;         // 1: k_filter flags tiles, k_mma_tiles<EpiFallback> computes them
  int xf_cols;           // columns of xflags (point tiles of 256)
  uint32_t *xflags;      // [ceil(q/128)][xf_cols] ACT_EXACT pairs of the tile this round
  uint32_t xmin;         // tiles with >= xmin of them run on the tensor cores
  const int32_t *nx;     // [n] ||x_i||^2
  int32_t *nq;           // [q] ||x_q||^2 of this batch
  // tile-staged level gathers (advance_tiles.cu)
  int tile_on;           // 1: dense (R x P) tiles advance from shared memory
  int tile_lr, tile_lp;  // log2 R (queries per tile), log2 P (points per tile); R | 32, 4 <= P <= 32
  int tile_cols;         // row length of tilework: ceil(npad / P)
  uint32_t *tilework;    // [ceil(qb / R)][tile_cols] draws of the tile's sampled blockers
  uint32_t *rowany;      // [ceil(qb / 32)][rowany_cols] bit r: row r of the 32-row group has an
  int rowany_cols;       //   action in this 1024-arm chunk (k_filter -> k_scatter early exit)
  float tile_min_draws;  // dense iff tilework >= tile_min_draws
  int tile_slot_l;       // log2 of a row slot in shared memory (>= pitch)
  int tile_tma;          // 1: rows staged by bulk TMA copies (cp.async.bulk), 0: 16-byte cp.async
  int tile_groups;       // > 0: k_advance_tiles_grp with this many thread groups per CTA
  int tile_tight;        // 1: its row slots are the pitch apart (not a power of two)
  int tile_db;           // 1: its groups double-buffer their query rows
  float tile_z_draws;    // > 0: dense tiles with tilework >= this run in k_advance_tiles_z
                         //   (|x - q| rows materialised; the grouped kernel skips them)
  float tile_qg_draws;   // > 0: dense tiles with tilework < this gather the query bytes from
                         //   global memory (k_advance_tiles_grp<..., QG>: no query-row copies)
  float tile_lo, tile_hi;  // this grouped launch takes the dense tiles with lo <= tilework < hi
  unsigned long long *advanced;  // pairs advanced (statistics), device counter
  // the blocker predicate as integer thresholds per (query, level) (k_thresholds)
  int32_t *thr;          // [q][THR_STRIDE]: Su[c], Sl[c] (c < MAX_LEVELS), M-mask
};

// ---- Philox4x32-10 (Salmon et al.), counter (x,y,z,w), key (k0,k1) --------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * c.x;
    const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1,
                   (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Same permutation with precomputed round keys rk0[r] = k0 + r*0x9E3779B9,
// rk1[r] = k1 + r*0xBB67AE85 (kernel-parameter constants).
__device__ __forceinline__ uint4 philox4x32_10_rk(uint4 c, const uint32_t *rk0, const uint32_t *rk1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned long long p0 = (unsigned long long)0xD2511F53u * c.x;
    const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ rk0[r], (uint32_t)p1,
                   (uint32_t)(p0 >> 32) ^ c.w ^ rk1[r], (uint32_t)p0);
  }
  return c;
}

// The same permutation for counters (blk, gi, gq, lv) that share (gi, gq): round 0's
// second product (of the counter word gq) and round 1's first product (of round 0's
// first output word, a function of gi and gq only) are the pair's constants, computed
// once by philox_pair and reused for every block of the pair: 18 instead of 20
// 32 x 32 -> 64-bit multiplies per block on the fma-heavy pipe.  Bit-identical.
struct PhiloxPair {
  uint32_t y0;        // round 0 output word y = lo(M1 * gq)
  uint32_t x0;        // round 0 output word x = hi(M1 * gq) ^ gi ^ rk0[0]
  uint32_t hp1, lp1;  // round 1: M0 * x0
};
__device__ __forceinline__ PhiloxPair philox_pair(uint32_t gi, uint32_t gq, const uint32_t *rk0) {
  const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * gq;
  PhiloxPair c;
  c.x0 = (uint32_t)(p1 >> 32) ^ gi ^ rk0[0];
  c.y0 = (uint32_t)p1;
  const unsigned long long q0 = (unsigned long long)0xD2511F53u * c.x0;
  c.hp1 = (uint32_t)(q0 >> 32);
  c.lp1 = (uint32_t)q0;
  return c;
}
__device__ __forceinline__ uint4 philox_from_pair(uint32_t blk, uint32_t lv, const PhiloxPair &pc,
                                                  const uint32_t *rk0, const uint32_t *rk1) {
  // round 0: c = (blk, gi, gq, lv)
  const unsigned long long p0 = (unsigned long long)0xD2511F53u * blk;
  const uint32_t z0 = (uint32_t)(p0 >> 32) ^ lv ^ rk1[0], w0 = (uint32_t)p0;
  // round 1: c = (x0, y0, z0, w0); M0 * x0 is the pair's constant
  const unsigned long long p1 = (unsigned long long)0xCD9E8D57u * z0;
  uint4 c = make_uint4((uint32_t)(p1 >> 32) ^ pc.y0 ^ rk0[1], (uint32_t)p1, pc.hp1 ^ w0 ^ rk1[1], pc.lp1);
#pragma unroll
  for (int r = 2; r < 10; ++r) {
    const unsigned long long q0 = (unsigned long long)0xD2511F53u * c.x;
    const unsigned long long q1 = (unsigned long long)0xCD9E8D57u * c.z;
    c = make_uint4((uint32_t)(q1 >> 32) ^ c.y ^ rk0[r], (uint32_t)q1, (uint32_t)(q0 >> 32) ^ c.w ^ rk1[r],
                   (uint32_t)q0);
  }
  return c;
}

// The query word of the Philox counter of batch row qi (R19): the query's
// RNG index, or -- with query-independent draws -- one word shared by
// every query, so that arm i's t-th coordinate is the same for all queries.
constexpr uint32_t SHARED_QI = 0xFFFFFFFFu;
__device__ __forceinline__ uint32_t rng_qi(const Geom &g, uint32_t qi) { return g.shared_draws ? SHARED_QI : qi + g.qi0; }

// Multiply-high map of a 32-bit word onto [0, d) (reading R5).
__device__ __forceinline__ uint32_t coord_of(uint32_t w, uint32_t d) { return __umulhi(w, d); }

// ---- Sampling without replacement (AKNN_FLAG_WITHOUT_REPLACEMENT; R23) ----
// The t-th sample of an arm is pi(t), pi a permutation of [0, d) keyed by the arm's
// Philox block w of counter (0, i, qi, WOR_LEVEL): rho = a 6-round mixed-radix Feistel
// network on Z_a x Z_b (a = ceil(sqrt d), b = ceil(d / a); x = L b + R), round r:
// (L, R) -> (R, (L + F_r(R)) mod m), m = a for even r, b for odd r,
// F_r(R) = umulhi(g((R ^ k_r) * 0x9E3779B1), m), g(h) = (h ^ (h >> 16)) * 0x85EBCA6B,
// k_r = w[r mod 4] + r * 0x9E3779B9, walked until the value is < d (rare: a b < d + a);
// pi(t) = (rho(t) + rot) mod d with rot = (w.x ^ w.z) mapped onto [0, d).
constexpr uint32_t WOR_LEVEL = 0x80000000u;  // a level word no draw uses
__host__ inline WorRadix wor_radix(int d) {
  uint32_t r = 1;
  while (r * r < (uint32_t)d) ++r;
  WorRadix w;
  w.a = r;
  w.b = ((uint32_t)d + r - 1) / r;
  w.binv = w.b >= 2 ? (uint32_t)(((1ull << 32) + w.b - 1) / w.b) : 0u;
  return w;
}
__device__ __forceinline__ uint4 wor_keys(const uint32_t *rk0, const uint32_t *rk1, uint32_t gi, uint32_t gq) {
  return philox4x32_10_rk(make_uint4(0u, gi, gq, WOR_LEVEL), rk0, rk1);
}
__device__ __forceinline__ uint32_t wor_feistel(uint4 w, const WorRadix &z, uint32_t x) {
  uint32_t L = z.b >= 2 ? __umulhi(x, z.binv) : x;
  uint32_t R = x - L * z.b;
#pragma unroll
  for (uint32_t r = 0; r < 6; ++r) {
    const uint32_t m = (r & 1u) ? z.b : z.a;
    const uint32_t kw = (r & 3u) == 0 ? w.x : (r & 3u) == 1 ? w.y : (r & 3u) == 2 ? w.z : w.w;
    uint32_t h = (R ^ (kw + r * 0x9E3779B9u)) * 0x9E3779B1u;
    h = (h ^ (h >> 16)) * 0x85EBCA6Bu;
    uint32_t nr = L + __umulhi(h, m);  // L < m and the map < m: one conditional subtract
    nr = nr >= m ? nr - m : nr;
    L = R;
    R = nr;
  }
  return L * z.b + R;
}
// Four consecutive draws t0 .. t0 + 3 of one arm (independent chains: ILP).
__device__ __forceinline__ uint4 wor_coords4(uint4 w, const WorRadix &z, uint32_t d, uint32_t t0) {
  uint32_t x[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) x[e] = wor_feistel(w, z, t0 + (uint32_t)e);
#pragma unroll
  for (int e = 0; e < 4; ++e)
    while (x[e] >= d) x[e] = wor_feistel(w, z, x[e]);
  const uint32_t rot = coord_of(w.x ^ w.z, d);
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    x[e] += rot;
    x[e] = x[e] >= d ? x[e] - d : x[e];
  }
  return make_uint4(x[0], x[1], x[2], x[3]);
}
__device__ __forceinline__ uint32_t wor_coord(uint4 w, const WorRadix &z, uint32_t d, uint32_t t) {
  uint32_t x = t;
  do {
    x = wor_feistel(w, z, x);
  } while (x >= d);
  x += coord_of(w.x ^ w.z, d);
  return x >= d ? x - d : x;
}

// The sample-count schedule: level c holds T_c samples.  growth 1 (readings R7): T_c =
// 2^c; growth 2 (reading R25): 1, 2, 3, 4, 6, 8, 12, 16, ... (factors
// 3/2 and 4/3), i.e. T_c = 2^((c+1)/2) for odd c and 3 * 2^((c-2)/2) for even c >= 2.
// Every power of two is a count, so the advance [T_c, T_{c+1}) stays inside one sample
// level b of the Draw stream (reading R19).
__host__ __device__ __forceinline__ uint32_t lvl_count(uint32_t c, int growth) {
  if (growth <= 1) return c < 32u ? 1u << c : 0xFFFFFFFFu;
  if (c == 0) return 1u;
  return (c & 1u) ? (1u << ((c + 1) >> 1)) : (3u << ((c - 2) >> 1));
}
// The samples of an arm in level byte l: d once exact, else T_c.
__host__ __device__ __forceinline__ uint32_t count_of(uint8_t l, int d, int growth) {
  return lvl_exact(l) ? (uint32_t)d : lvl_count(l & 0x7Fu, growth);
}
// L / T_c for the exact order key (L = lcm of every sampled count and d; L3 = L / 3).
__host__ __device__ __forceinline__ unsigned long long lvl_mul(uint32_t c, unsigned long long L,
                                                               unsigned long long L3, int growth) {
  if (growth <= 1) return L >> c;
  if (c == 0) return L;
  return (c & 1u) ? (L >> ((c + 1) >> 1)) : (L3 >> ((c - 2) >> 1));
}
// The advance out of level c draws the samples t = T_c .. T_{c+1} - 1: sample level
// b = 1 + floor(log2 T_c), in-level ordinals u = u0 .. u0 + cnt - 1 (reading R19).
struct LevelAdvance {
  uint32_t b, u0, cnt;
};
__host__ __device__ __forceinline__ LevelAdvance lvl_advance(uint32_t c, int growth) {
  const uint32_t t0 = lvl_count(c, growth), t1 = lvl_count(c + 1, growth);
#ifdef __CUDA_ARCH__
  const uint32_t b = 31u - (uint32_t)__clz(t0);  // floor(log2 t0)
#else
  uint32_t b = 0;
  while ((t0 >> b) > 1u) ++b;
#endif
  return LevelAdvance{b + 1u, t0 - (1u << b), t1 - t0};
}

// Exact order key of an arm: K = S * (L / T).  S/T ranks exactly like the
// fp64 estimate S/(65025 T) (reading R9), and with the local index
// in the low bits every key is unique: (d_hat, i) lexicographic order.
// i is the LOCAL index; the key carries the global id i + id_offset, so keys of
// different shards are comparable and unique.
__device__ __forceinline__ unsigned long long arm_key(int32_t S, uint8_t l, uint32_t i,
                                                      const Geom &g) {
  const unsigned long long mul = lvl_exact(l) ? g.Ld : lvl_mul(l, g.L, g.L3, g.growth);
  return (((unsigned long long)(uint32_t)S * mul) << g.kbits) | (i + g.id_offset);
}

// d_hat = S / (T * 65025), one correctly rounded fp64 division (P:121-124,
// DESIGN.md reading R15).  T * 65025 is exact in fp64.
__host__ __device__ __forceinline__ double dhat_of(int32_t S, uint8_t l, int d, int growth) {
  const double T = (double)count_of(l, d, growth);
#ifdef __CUDA_ARCH__
  return __ddiv_rn((double)S, __dmul_rn(T, 65025.0));
#else
  return (double)S / (T * 65025.0);  // host: -ffp-contract=off, one rounding each
#endif
}

__host__ __device__ __forceinline__ double alpha_of(uint8_t l, const double *alpha, int growth) {
#ifdef __CUDA_ARCH__
  return lvl_exact(l) ? 0.0 : __ldg(alpha + lvl_count(l, growth));
#else
  return lvl_exact(l) ? 0.0 : alpha[lvl_count(l, growth)];
#endif
}

__host__ __device__ __forceinline__ double upper_of(int32_t S, uint8_t l, int d, const double *alpha, int growth) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(dhat_of(S, l, d, growth), alpha_of(l, alpha, growth));
#else
  return dhat_of(S, l, d, growth) + alpha_of(l, alpha, growth);
#endif
}

__host__ __device__ __forceinline__ double lower_of(int32_t S, uint8_t l, int d, const double *alpha, int growth) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(dhat_of(S, l, d, growth), alpha_of(l, alpha, growth));
#else
  return dhat_of(S, l, d, growth) - alpha_of(l, alpha, growth);
#endif
}

}  // namespace aknn
