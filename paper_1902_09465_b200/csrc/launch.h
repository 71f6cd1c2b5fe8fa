// launch.h -- internal launch wrappers (host side of the kernels).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "internal.cuh"

namespace aknn {

// Device output pointers of one query batch (rows row0 .. row0 + q - 1).
struct OutPtrs {
  int row0;
  int64_t col0;     // first column of this shard in counts/sums rows
  int64_t ncols;    // row length of counts/sums
  int accumulate;   // 1: atomically add draws/evals (several shards, one device)
  int32_t *sets;
  double *dhat;
  int32_t *counts;
  int64_t *sums;
  int64_t *evals;
  int64_t *draws;
  int32_t *rounds;
};

// Literal Algorithm 1 (a1_kernels.cu): one warp per query, state in `ws`.
constexpr int A1_MAX_KH = 512;
struct A1Geom {
  const uint8_t *X;      // [n][pitch]
  int64_t pitch;
  const uint8_t *Q;      // [q][d] queries of the call (unpadded)
  const double *alpha;   // [d+1]
  int n, d, k, kh;
  int q0, qb;            // this launch: queries q0 .. q0 + qb - 1
  uint32_t id_offset, qi0;
  int max_iters;         // 0 = unlimited
  uint32_t rk0[10], rk1[10];
  unsigned char *ws;     // qb slices of ws_per_query bytes
  size_t ws_per_query;
  int *status;           // bit 0: some query reached max_iters
  int smem;              // 1: state in shared memory (ws_per_query <= A1_SMEM_MAX)
  int wor;               // 1: sampling without replacement (R23)
  WorRadix wor_z;
  OutPtrs out;
};
constexpr size_t A1_SMEM_MAX = 96 * 1024;
cudaError_t launch_a1(const A1Geom &g, cudaStream_t s);
size_t a1_ws_per_query(int64_t n, int kh, int d, bool tables);

cudaError_t launch_init(const Geom &g, cudaStream_t s);
cudaError_t launch_select(const Geom &g, int nbits, cudaStream_t s);
cudaError_t launch_filter(const Geom &g, cudaStream_t s);
cudaError_t launch_thresholds(const Geom &g, cudaStream_t s);  // after every rank split / merge
cudaError_t launch_compact(const Geom &g, cudaStream_t s);
cudaError_t launch_advance(const Geom &g, int num_sms, cudaStream_t s);
int stage_level(int64_t pitch);
// Tile-staged level gathers of dense tiles (advance_tiles.cu).
cudaError_t launch_advance_tiles(const Geom &g, int num_sms, cudaStream_t s);
size_t tile_smem_bytes(int lr, int lp, int64_t pitch);
size_t tile_grp_smem_bytes(int groups, int lr, int lp, int64_t pitch, bool tight, bool db);
int tile_slot_log2(int64_t pitch);
// |x - q| tiles (k_advance_tiles_z): usable for this shape (P = 8 points, R = 1, rows fit)
bool tile_z_ok(int lr, int lp, int64_t pitch, int64_t q);
// Per-query counters from the final arm states (before the outputs).
cudaError_t launch_tally(const Geom &g, cudaStream_t s);
// Device-driven round loop (CUDA graph with a conditional WHILE node).
cudaError_t launch_ctl_reset(RoundCtl *ctl, unsigned q, cudaStream_t s);
cudaError_t launch_zero_round(const Geom &g, cudaStream_t s);
cudaError_t launch_round_ctl(RoundCtl *ctl, cudaGraphConditionalHandle h, int max_rounds, cudaStream_t s);
cudaError_t launch_output(const Geom &g, const OutPtrs &o, cudaStream_t s);
// Sharded rounds (shard_kernels.cu).
cudaError_t launch_select_local(const Geom &g, int nbits, cudaStream_t s);
// One-pass pivot selects (select_pivot.cu); flag QState.fallback when undecided.
cudaError_t launch_select_pivot(const Geom &g, cudaStream_t s);
cudaError_t launch_select_local_pivot(const Geom &g, cudaStream_t s);
cudaError_t launch_merge(const Geom &g, const OutPtrs &o, cudaStream_t s);
cudaError_t launch_output_sharded(const Geom &g, const OutPtrs &o, cudaStream_t s);
size_t merge_smem_bytes(int world, int kh);
int output_max_kh();

// Exact comparison pass (exact_kernels.cu).
struct ExactGeom {
  const uint8_t *X;   // [n][pitch]
  const uint8_t *Q;   // [q][pitch]
  int64_t pitch;
  int n, d, q, k;
  uint32_t id_offset;
  int32_t *D;         // [q][npad] scratch distances
  int64_t npad;
  int ibits, nbits;
  int32_t *idx;       // [q][k] out (device)
  int32_t *dist2;     // [q][k] out (device)
};
cudaError_t launch_exact_topk(const ExactGeom &e, cudaStream_t s);   // top-k of e.D only
// D via tcgen05 kind::i8 (exact_mma.cu); nq [q], nx [n] squared row norms.
cudaError_t launch_exact_mma(const ExactGeom &e, const int32_t *nq, const int32_t *nx, cudaStream_t s);
// Exact fallbacks of a round on the tensor cores (flagged tiles only).
cudaError_t launch_exact_fallback_mma(const Geom &g, cudaStream_t s);
// The fused exact pass (exact_fused.cu): persistent tcgen05 kernel with a running top-k
// epilogue + per-query merge; k <= exact_fused_max_k().  nx zero padded to n rounded up
// to 256; ws >= exact_fused_ws_bytes(num_sms, k).
cudaError_t launch_exact_fused(const ExactGeom &e, const int32_t *nq, const int32_t *nx, void *ws, int num_sms,
                               cudaStream_t s);
int exact_fused_max_k();
size_t exact_fused_ws_bytes(int num_sms, int k);
int exact_tile_rows();
// Shared draws on the tensor cores (exact_mma.cu).
cudaError_t launch_q2_planes(const Geom &g, cudaStream_t s);
cudaError_t launch_build_w(const Geom &g, cudaStream_t s);
cudaError_t launch_level_mma(const Geom &g, cudaStream_t s);
int level_tile_rows();
int level_tile_cols();
int exact_tile_cols();
cudaError_t launch_row_norms(const uint8_t *A, int64_t pitch, int rows, int32_t *out, cudaStream_t s);

}  // namespace aknn
