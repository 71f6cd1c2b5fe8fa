/*
 * aknn.h -- C-ABI of libaknn.so, the B200 (sm_100a) hot path of the adaptive
 * k-NN algorithm of LeJeune, Baraniuk & Heckel (arXiv 1902.09465).
 *
 * Citations: "P:<line>" = /root/reference/PAPER.md, "S:<line>" = SPEC.md.
 * The readings of ambiguous passages (R1..R18) are listed in DESIGN.md §3.
 *
 * Problem (§3): given points X = {x_1..x_n} in R^m and a query x,
 * return a set of size k+h that contains the k nearest neighbours of x in
 * l2 distance.  Points and queries are uint8 vectors; one sampled squared
 * coordinate difference is (a-b)^2/65025 in [0,1] (reading R2).
 *
 * Method (Algorithm 1, run under the batched round rule BR of
 * DESIGN.md §2): per query, estimate D_i = (1/m)||x - x_i||^2
 * by uniformly sampled coordinates with confidence radius
 * alpha(T_i); split arms by rank into close / middle / far
 * (P:144-146); stop when Eq. (5) holds; return the
 * top k+h by estimate.
 *
 * Conventions for every entry point:
 *   - All sizes are element counts.  Matrices are dense row-major with no
 *     padding: points [n][d], queries [q][d], sets [q][k+h], counts [q][n].
 *   - Buffers belong to the caller; the library never frees or retains a
 *     caller pointer after the call returns.  An aknn_index owns a device
 *     copy of X until aknn_free.
 *   - Host variants take host pointers and are synchronous.  *_async
 *     variants take DEVICE pointers and a cudaStream_t (as void*) and enqueue
 *     their device work on that stream.
 *   - On any status other than AKNN_OK no output is written, except
 *     AKNN_EMAXROUNDS, which writes the state reached (see aknn_opts).
 *     aknn_last_error() returns a thread-local message for the last failure.
 *   - Not thread-safe per index: calls on one aknn_index must be serialised.
 */
#ifndef AKNN_H
#define AKNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aknn_index aknn_index; /* opaque; owns a device copy of X */

typedef enum {
  AKNN_OK = 0,
  AKNN_EINVAL = -1,     /* argument outside the domain stated below              */
  AKNN_ENOMEM = -2,     /* device or host allocation failed                      */
  AKNN_ECUDA = -3,      /* a CUDA runtime call or kernel launch failed           */
  AKNN_ENCCL = -4,      /* an NCCL call failed or timed out (sharded index)      */
  AKNN_EMAXROUNDS = -5  /* aknn_opts.max_rounds reached before Eq. (5) held      */
} aknn_status;

/* Outputs of a query batch.  `sets` is required; every other field may be
 * NULL to skip that output.  Host pointers for aknn_query[_ex], device
 * pointers for aknn_query_async.                                            */
typedef struct {
  int32_t *sets;   /* [q][k+h] point ids of (1)..(k+h), rank order    */
  double *dhat;    /* [q][k+h] fp64 estimates d_hat of those arms     */
  int32_t *counts; /* [q][n_local] per-pair sample count T_i; T_i == d means
                      the arm went exact                              */
  int64_t *sums;   /* [q][n_local] exact integer S_i = sum of sampled (a-b)^2
                      (or the exact sum once T_i == d); d_hat = S/(65025 T)   */
  int64_t *evals;  /* [q] draws + d * (#exact fallbacks)          */
  int64_t *draws;  /* [q] sampled coordinate draws, including initialisation  */
  int32_t *rounds; /* [q] rounds of the batched rule until Eq. (5) held       */
} aknn_result;

/* Optional per-call settings; pass NULL for the defaults (all zero).        */
typedef struct {
  int32_t qi_offset;  /* RNG query index of queries[0] (default 0): query a uses
                         counter word qi = qi_offset + a                      */
  int32_t max_rounds; /* 0 = unlimited; otherwise stop after this many rounds
                         and return AKNN_EMAXROUNDS with the state reached    */
  int32_t timing;     /* 1 = time each kernel class with CUDA events on the
                         launching stream and fill aknn_stats.ms_*           */
  int32_t flags;      /* bit 0 (AKNN_FLAG_RADIX_SELECT): decide every rank split
                         with the multi-pass radix select instead of the one-pass
                         pivot select (diagnostics; results are identical);
                         bits 1, 2 (AKNN_FLAG_EXACT_ROWS, AKNN_FLAG_NO_TILES): see
                         below                                                   */
  int32_t lead;       /* close-side lead L (DESIGN.md
                         reading R24): 0 or 1 = the batched rule; L > 1 = the
                         blockers of a round that rank in C or M (ranks 1..k+h)
                         advance L times (each the doubling / P:176 exact step),
                         the far blockers once.  1 <= L <= 8 (else EINVAL);
                         ignored by the Algorithm-1 entry points.              */
  int32_t batch_queries; /* 0 = automatic; else at most this many queries per
                         internal sub-batch (the round workspace is ~10 B per
                         (query, point) pair; the automatic size fits 60 % of
                         free device memory).  Results do not depend on it.
                         Ignored by the Algorithm-1 entry points.  < 0: EINVAL */
  int32_t growth;     /* sample-count schedule of an advance (SURVEY.md §8(f) row 4,
                         DESIGN.md reading R25): 0 or 1 = doubling T -> 2T (reading
                         R7); 2 = growth factor < 2: T runs through 1, 2, 3, 4, 6,
                         8, 12, 16, ... (factors 3/2 and 4/3; the advance from T
                         draws the next count minus T samples, the exact fallback
                         of P:176 when the next count would reach d).  Growth 2
                         runs the list path (no shared-memory tiles) and needs
                         per-query draws with replacement (EINVAL with
                         AKNN_FLAG_SHARED_DRAWS / _WITHOUT_REPLACEMENT); other
                         values: EINVAL.  Ignored by the Algorithm-1 entry points. */
} aknn_opts;

#define AKNN_FLAG_RADIX_SELECT 1
/* bit 1: compute the exact fallbacks by streaming each pair's row on the
   CUDA cores instead of the tensor-core tile pass (diagnostics; identical results) */
#define AKNN_FLAG_EXACT_ROWS 2
/* bit 2: advance every pair through the work lists (global-memory gathers) instead
   of staging dense (query x point) tiles in shared memory (diagnostics; identical
   results)                                                                   */
#define AKNN_FLAG_NO_TILES 4
/* bit 3: every 128 x 256 tile with an exact fallback runs on the tensor cores (by
   default tiles with fewer than 512 of them stream rows instead; identical results) */
#define AKNN_FLAG_EXACT_MMA_ALL 8
/* bit 4: query-independent coordinate draws: the Philox counter's
   query word is 0xFFFFFFFF for every query, so arm i's t-th sampled coordinate is the
   same for all queries (each query's samples stay i.i.d. uniform, so the
   guarantee of P:395-399 holds per query).  A different -- equally valid -- stream:
   results differ from the default and match the oracle run with qids = 0xFFFFFFFF. */
#define AKNN_FLAG_SHARED_DRAWS 16
/* bit 5: with shared draws, keep every level on the per-pair gathers instead of the
   tensor-core level GEMMs (k_level_mma; diagnostics, identical results)      */
#define AKNN_FLAG_NO_LEVEL_MMA 32
/* bit 6: sampling WITHOUT replacement (footnote 1 to P:120; SURVEY.md §8(f) row 4;
   DESIGN.md reading R23): the t-th sample of arm (qi, i) is coordinate pi(t) of a
   permutation of [0, d) keyed per arm: a 6-round mixed-radix Feistel network on
   Z_a x Z_b (a = ceil(sqrt d), b = ceil(d / a)) cycle-walked into [0, d), then a
   keyed rotation; its keys are the Philox4x32-10 block of counter
   (0, i, qi, 0x80000000).  Estimates stay unbiased
   and the footnote-2 / §5 radii stay valid (Hoeffding's bound holds without
   replacement).  An exact fallback is charged only the d - T coordinates
   not drawn yet, so evals = the sum of the final counts <= n d; in Algorithm 1 an
   arm reaching T = d has drawn every coordinate once (no extra charge).  Results
   differ from the default stream and match the oracle's without_replacement mode.
   Not combinable with AKNN_FLAG_SHARED_DRAWS (EINVAL).                        */
#define AKNN_FLAG_WITHOUT_REPLACEMENT 64

/* Execution statistics of the last query call on an index (aknn_get_stats).
 * Kernel classes: init (a2), select (a6-a7: rank split, bounds, Eq. 5),
 * filter (a8 blocker predicate), compact (a8 list plan + scatter), advance
 * (a3-a4 list-path level gathers and exact fallbacks), tiles (a3 level gathers
 * of dense tiles from shared memory), output (a9).  ms_* are device
 * times from CUDA events recorded on the launching stream around every
 * launch of that class (timing = 1 only; events are read after the call's
 * final synchronisation, so timing adds no host round trips).              */
typedef struct {
  int32_t rounds;             /* host rounds executed (max over sub-batches)   */
  int32_t query_batches;      /* internal query sub-batches                    */
  int64_t kernel_launches;    /* device kernels launched by the call           */
  int64_t pairs;              /* q * n_local                                   */
  int64_t draws;              /* total sampled draws incl. init (sum over q)   */
  int64_t exact_fallbacks;    /* total arms that went exact                    */
  int64_t active_pair_rounds; /* sum over rounds of advanced (listed) pairs    */
  int64_t query_rounds;       /* sum over rounds of queries the rank split
                                 evaluated (not yet stopped)                   */
  int64_t blocked_query_rounds;/* ... of those, queries that failed Eq. (5)    */
  double ms_total;            /* device time of the whole call (timing=1)      */
  double ms_init, ms_select, ms_filter, ms_compact, ms_advance, ms_output;
  int64_t launches_init, launches_select, launches_filter, launches_compact,
      launches_advance, launches_output;
  int64_t philox_blocks;      /* Philox4x32-10 blocks the level gathers drew
                                 (one per 4 draws; levels 1 and 2 use one)      */
  int32_t graph_builds;       /* round-loop graphs captured + instantiated by
                                 this call (0 when the cached graph was reused) */
  int32_t pad0;
  double ms_tiles;            /* device time of the dense-tile gathers: shared-memory
                                 tiles (k_advance_tiles) or, with shared draws, the
                                 tensor-core level GEMMs (k_level_mma); rows a3  */
  int64_t launches_tiles;
  int64_t tile_blocks;        /* Philox blocks drawn by the tile gathers        */
  int64_t tile_draws;         /* (query, point) draws summed by the tile gathers */
  int64_t level_mma_tiles;    /* 128 x 128 tiles of shared-draw levels run as tensor-core GEMMs */
} aknn_stats;

/* ------------------------------------------------------------------------ */
/* Index construction.                                                       */
/* ------------------------------------------------------------------------ */

/* Copy points (host, uint8 [n][d]) to the current CUDA device: the point set X
 * of the problem statement (§3; one point per row, one uint8 coordinate
 * per byte, reading R2).  The device copy is row-major with the row pitch padded
 * to 16 bytes (zero filled); ||x_i||^2 is computed lazily by the first exact pass.
 * Domain (EINVAL otherwise): n >= 2, n < 2^31, 1 <= d <= 33025 (so that
 * d * 255^2 < 2^31), and the composite rank key of DESIGN.md reading R9 fits 63
 * bits: bit_length(65025 * lcm(2^c, d)) + bit_length(n - 1) <= 63 with c the
 * largest integer such that 2^c < d (c = 0 for d <= 2).  Every d <= 258 fits
 * for any n < 2^31, every d <= 4128 for n <= 8e6, every d <= 16384 for
 * n <= 1e6 and every d <= 33025 for n <= 1e5 (all five BASELINE configs fit).
 * ENOMEM when the device copy does not fit; ECUDA on a
 * failed copy.  The caller may free `points` on return.                     */
aknn_status aknn_build(const uint8_t *points, int64_t n, int32_t d, aknn_index **out);

/* Same, from a DEVICE buffer, copied on `cuda_stream` (the index keeps its own
 * copy; the caller's buffer may be freed after the stream completes; queries on
 * another stream must be ordered after it by the caller).  Same domain.      */
aknn_status aknn_build_async(const uint8_t *points_dev, int64_t n, int32_t d,
                             void *cuda_stream, aknn_index **out);

/* Sharded index: this process holds rows
 * [offset, offset + n_local) of an n_global-point set.  Point ids in the RNG
 * counter and in the returned sets are global ids.  `nccl_unique_id` points
 * to an ncclUniqueId (128 bytes) shared by the `world` ranks (rank 0 creates
 * it with aknn_nccl_unique_id and broadcasts it out of band).  With
 * world == 1 no communicator is created.                                    */
aknn_status aknn_build_shard(const uint8_t *shard, int64_t n_local, int64_t n_global,
                             int64_t offset, int32_t d, const void *nccl_unique_id,
                             int32_t rank, int32_t world, aknn_index **out);
/* Domain as aknn_build with n = n_global for the key, plus
 * 0 <= offset, offset + n_local <= n_global, 0 <= rank < world (EINVAL);
 * ENCCL when world > 1 and the communicator cannot be created.               */
/* aknn_query* on an index built with world > 1 runs the point-sharded round
 * loop: one ncclAllGather per round of (k+h+1) 16-byte records per query and
 * rank, a deterministic merge on every rank, and at the end an ncclAllReduce of
 * draws/evals.  Every rank must call it with the same arguments; sets, d_hat,
 * evals, draws and rounds are then identical on every rank (global ids), and
 * counts/sums hold this rank's n_local columns.  Needs world * (k+h) <= 16384
 * and n_local > k + h on every rank.                                          */

/* Failure detection of the sharded query: while a rank waits for a
 * round it also polls ncclCommGetAsyncError and a wall-clock deadline; on a peer
 * error or when no progress is made for timeout_ms (default 300000; 0 = no
 * deadline) it calls ncclCommAbort -- the pending collective then fails on every
 * rank instead of hanging -- and returns AKNN_ENCCL.  An aborted index returns
 * AKNN_ENCCL from every later sharded query (rebuild it).  EINVAL: NULL index or
 * timeout_ms < 0.  No effect on indexes without a communicator.              */
aknn_status aknn_set_timeout(aknn_index *ix, double timeout_ms);

/* Write a fresh ncclUniqueId (128 bytes) to `id_out`.                       */
aknn_status aknn_nccl_unique_id(void *id_out);

/* ------------------------------------------------------------------------ */
/* The adaptive query (the hot path).                                        */
/* ------------------------------------------------------------------------ */

/* Run the batched round rule for q queries (host uint8 [q][d]).
 * k >= 1, h >= 0, k + h < n_global; delta in (0,1); seed = the 64-bit Philox
 * key (low word = key[0]).  alpha: host fp64 [d+1], alpha[u] for 1 <= u < d
 * (alpha[0] and alpha[d] are ignored; an exact arm has alpha 0); NULL
 * selects the footnote-2 table of (n_global, delta) built by
 * aknn_alpha_table (EINVAL when delta/n_global >= 1/e).
 * Results are bit-identical to the oracle's for the same inputs.            */
aknn_status aknn_query(const aknn_index *ix, const uint8_t *queries, int32_t q, int32_t k,
                       int32_t h, double delta, uint64_t seed, const double *alpha,
                       aknn_result *out);

/* aknn_query with options (NULL = defaults).                                */
aknn_status aknn_query_ex(const aknn_index *ix, const uint8_t *queries, int32_t q, int32_t k,
                          int32_t h, double delta, uint64_t seed, const double *alpha,
                          const aknn_opts *opts, aknn_result *out);

/* Device-pointer variant: queries_dev uint8 [q][d], alpha_dev fp64 [d+1]
 * (NULL = footnote-2 table), outputs in `out` are device pointers.  All work
 * is enqueued on `cuda_stream`.  With timing = 0 the round loop runs on the
 * device (one CUDA graph per query sub-batch, a conditional WHILE node decides
 * the rounds); with max_rounds = 0 as well the call returns WITHOUT waiting for
 * the device (the status cannot be EMAXROUNDS) and the statistics of the call
 * are completed by aknn_get_stats or by the next call on this index.  Otherwise
 * it returns after the loop has finished.  Outputs are complete when the
 * stream is.  Calls on one index must be ordered (one stream, or synchronised). */
aknn_status aknn_query_async(const aknn_index *ix, const uint8_t *queries_dev, int32_t q,
                             int32_t k, int32_t h, double delta, uint64_t seed,
                             const double *alpha_dev, const aknn_opts *opts,
                             aknn_result *out, void *cuda_stream);

/* One query batch over a point set split into `nshards` shard indices that all
 * live on the CURRENT device (built with aknn_build_shard(..., world = 1)),
 * driven in lockstep by this process.  Shard s must hold rows
 * [offset_s, offset_s + n_s) with the shards tiling [0, n_global) in order, and
 * n_s > k + h.  Each round every shard writes its summary (local top-(k+h)
 * arms + its minimum-L remainder arm) into one receive buffer and
 * every shard merges them identically -- the same kernels as the NCCL path,
 * without the transport.  Outputs as aknn_query, except counts/sums rows have
 * n_global columns (shard s at columns offset_s ..).  Results are bit-identical
 * to aknn_query on the unsharded set.  Stats go to shards[0].                */
aknn_status aknn_query_multi(const aknn_index *const *shards, int32_t nshards,
                             const uint8_t *queries, int32_t q, int32_t k, int32_t h,
                             double delta, uint64_t seed, const double *alpha,
                             const aknn_opts *opts, aknn_result *out);

/* The literal Algorithm 1 schedule for q
 * queries (host uint8 [q][d]) on an unsharded index.  Each iteration
 * re-evaluates the rank split (C = ranks 1..k, M = k+1..k+h, F = the rest, by
 * (d_hat, id)), d1 = argmax_C U and d2 = argmin_F L (Eq. 2-3), stops when
 * Eq. (5) A <= B holds, and otherwise samples one coordinate of d1 and of
 * b2 = argmax_{{d2} u M} alpha (Eq. 4; ties to d2, then the smaller id); an arm
 * whose count reaches T = d takes its exact distance, charged d
 * evaluations.  The t-th sample of an arm is the batched rule's (the same
 * Philox counter), so only the schedule differs.  Arguments as aknn_query_ex;
 * opts->max_rounds caps the ITERATIONS (AKNN_EMAXROUNDS, outputs = the state
 * reached), opts->timing is ignored, and of opts->flags only
 * AKNN_FLAG_WITHOUT_REPLACEMENT applies (reading R23; evals = draws then).
 * Outputs: sets/dhat of the final top-(k+h) in rank order, counts = T_i (1..d), sums = S_i,
 * draws, evals = draws + d * (#arms that went exact), rounds = iterations
 * (including the last, stopping one).  EINVAL: the aknn_query_ex domain, a
 * sharded index, or k + h > 512.  Bit-identical to the oracle's A1 mode.     */
aknn_status aknn_query_a1(const aknn_index *ix, const uint8_t *queries, int32_t q, int32_t k,
                          int32_t h, double delta, uint64_t seed, const double *alpha,
                          const aknn_opts *opts, aknn_result *out);

/* aknn_query_a1 on device buffers (queries_dev uint8 [q][d], alpha_dev fp64
 * [d+1] or NULL = footnote-2 table, `out` device pointers), enqueued on
 * `cuda_stream`; returns after the stream has finished the call (the status
 * reports the iteration cap).                                                 */
aknn_status aknn_query_a1_device(const aknn_index *ix, const uint8_t *queries_dev, int32_t q,
                                 int32_t k, int32_t h, double delta, uint64_t seed,
                                 const double *alpha_dev, const aknn_opts *opts,
                                 aknn_result *out, void *cuda_stream);

/* Statistics of the last aknn_query* call on `ix`.                          */
aknn_status aknn_get_stats(const aknn_index *ix, aknn_stats *out);

/* ------------------------------------------------------------------------ */
/* Exact comparison pass (P:98 brute force): all distances, then top-k.      */
/* ------------------------------------------------------------------------ */

/* For each of q host queries: the k nearest points by the exact integer
 * distance sum_j (a_j - b_j)^2, ties to the smaller id; idx/dist2 host
 * [q][k] in ascending (dist2, id) order.  1 <= k <= min(n_local, 1024).
 * Computed as ||x'||^2 + ||q'||^2 - 2 x'.q' with x' = x - 128 (int8) on the
 * tensor cores (int8 -> int32), exact for d <= 33025.                        */
aknn_status aknn_exact(const aknn_index *ix, const uint8_t *queries, int32_t q, int32_t k,
                       int32_t *idx, int32_t *dist2);

/* Device-pointer variant on `cuda_stream`.                                   */
aknn_status aknn_exact_async(const aknn_index *ix, const uint8_t *queries_dev, int32_t q,
                             int32_t k, int32_t *idx_dev, int32_t *dist2_dev,
                             void *cuda_stream);

/* ------------------------------------------------------------------------ */
/* Host reference of the shard exchange.  Not on the hot path:  */
/* the same records, keys and merge the device kernels use, so the N > 1      */
/* protocol can be tested on CPUs (gloo) without a GPU.                        */
/* ------------------------------------------------------------------------ */

/* A shard record is 16 bytes: uint64 composite key (exact order key of the
 * estimate S/(65025 T) in the high bits, GLOBAL id in the low bits), int32 S,
 * uint8 level (log2 T, 0xFF = exact), 3 pad bytes.                            */
#define AKNN_SHARD_REC_BYTES 16

/* Summary of one query's arms on one shard: the k+h smallest composite keys
 * (ascending) then the arm with the smallest L = d_hat - alpha among the rest
 * (ties: smaller id) -> recs_out[(k+h+1) * 16 bytes].  S, lvl: [n_local] arm
 * state (lvl = log2 T or 0xFF for exact); ids are offset + i.                 */
aknn_status aknn_shard_summary_host(const int32_t *S, const uint8_t *lvl, int64_t n_local,
                                    int64_t offset, int64_t n_global, int32_t d, int32_t k,
                                    int32_t h, const double *alpha, void *recs_out);

typedef struct {
  int32_t *sets;         /* [k+h] global ids of ranks 1..k+h (required)          */
  double *dhat;          /* [k+h] their estimates (nullable)                     */
  uint64_t thr_k, thr_kh;/* composite keys of ranks k and k+h                    */
  double A, B;           /* Eq. (2)-(3) bounds                       */
  int64_t d1, d2;        /* their global ids                                     */
  double alpha_d2;       /* alpha of d2 (the middle-set rule, Eq. 4 batched)     */
  int32_t stop;          /* 1 iff A <= B, Eq. (5)                                */
} aknn_merge_result;

/* Merge `world` summaries (recs: [world][(k+h+1) * 16 bytes], rank order) of
 * one query into the global round quantities, exactly as k_merge does.       */
aknn_status aknn_shard_merge_host(const void *recs, int32_t world, int64_t n_global, int32_t d,
                                  int32_t k, int32_t h, const double *alpha,
                                  aknn_merge_result *res);

/* ------------------------------------------------------------------------ */
/* Confidence radius tables (host).                                           */
/* ------------------------------------------------------------------------ */

/* kind 0 = footnote 2: alpha(u) = sqrt(2 beta(u, delta/n)/u),
 *          beta = log(1/d') + 3 log log(1/d') + 1.5 log(1 + log u); needs
 *          delta/n < 1/e.
 * kind 1 = §5: alpha(u) = sqrt(c_alpha log(1 + (1 + log u) n/delta)/u).
 * Writes alpha_out[0..d]; alpha_out[0] = alpha_out[d] = 0.                  */
aknn_status aknn_alpha_table(int32_t kind, int64_t n, double delta, double c_alpha, int32_t d,
                             double *alpha_out);

/* ------------------------------------------------------------------------ */
/* Housekeeping.                                                             */
/* ------------------------------------------------------------------------ */

int64_t aknn_index_n_local(const aknn_index *ix);
int64_t aknn_index_n_global(const aknn_index *ix);
int32_t aknn_index_dim(const aknn_index *ix);
void aknn_free(aknn_index *ix);
const char *aknn_strerror(aknn_status s);
const char *aknn_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* AKNN_H */
