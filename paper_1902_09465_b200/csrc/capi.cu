// capi.cu -- the C-ABI of libaknn.so (include/aknn.h) and the host round
// driver of the batched round rule.
//
// The driver owns: the device copy of X (row pitch padded to 16 B, zero
// filled), a workspace sized for one query sub-batch, and one CUDA stream.
// Per sub-batch: k_init, then rounds of {k_select -> 4-byte D2H of the
// active-query count -> k_filter/k_plan/k_scatter -> k_advance}, then
// k_output.  Every device step is a kernel of round_kernels.cu; the host
// only sequences launches and validates arguments.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/aknn.h"
#include "host_wait.h"
#include "internal.cuh"
#include "launch.h"

#ifdef AKNN_WITH_NCCL
#include <nccl.h>
#endif

using namespace aknn;

namespace {

thread_local std::string g_last_error;

aknn_status fail(aknn_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? AKNN_ENOMEM : AKNN_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                     \
  } while (0)

#define TRY(call)                       \
  do {                                  \
    aknn_status s_ = (call);            \
    if (s_ != AKNN_OK) return s_;       \
  } while (0)

int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

int bit_length(unsigned long long v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

unsigned long long gcd_u64(unsigned long long a, unsigned long long b) {
  while (b) {
    const unsigned long long t = a % b;
    a = b;
    b = t;
  }
  return a;
}

// Pinned host staging (device->host reads of the round control block and query
// states): a pageable destination would make cudaMemcpyAsync block in the driver.
struct HostBuf {
  void *p = nullptr;
  size_t bytes = 0;
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  cudaError_t ensure(size_t want) {
    if (bytes >= want) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
};

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  aknn_status ensure(size_t want) {
    if (bytes >= want) return AKNN_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(AKNN_ENOMEM, "cudaMalloc(%zu): %s", want, cudaGetErrorString(e));
    }
    bytes = want;
    return AKNN_OK;
  }
  template <class T>
  T *as(size_t byte_off = 0) const {
    return reinterpret_cast<T *>(static_cast<char *>(p) + byte_off);
  }
};

struct EventPool {
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  ~EventPool() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
  cudaEvent_t get() {
    if (used == ev.size()) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      ev.push_back(e);
    }
    return ev[used++];
  }
};

}  // namespace

struct aknn_index {
  int device = 0;
  int num_sms = 148;
  int64_t n_local = 0, n_global = 0, offset = 0;
  int32_t d = 0;
  int64_t pitch = 0;
  DevBuf X;                // [n_local][pitch]
  cudaStream_t stream = nullptr;
  DevBuf ws;               // round workspace
  DevBuf qbuf;             // padded query staging
  DevBuf alpha;            // [d+1]
  DevBuf outs;             // device outputs for the host API
  DevBuf exact_ws;
  HostBuf host;            // pinned: n_active | RoundCtl | QState[qb]
  DevBuf nx;               // [n_local] ||x_i||^2 for the tensor-core exact pass (lazy)
  bool nx_ready = false;   // the row-norm kernel has been enqueued ...
  cudaEvent_t nx_ev = nullptr;  // ... and completes at this event (other streams wait on it)
  EventPool events;
  // cached graph of the device-driven round loop (one query sub-batch shape)
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  std::vector<unsigned char> loop_key;
  int rank = 0, world = 1;
#ifdef AKNN_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  bool nccl_failed = false;        // the communicator was aborted (peer error / timeout)
  double nccl_timeout_ms = 300000.0;  // aknn_set_timeout
  aknn_stats stats{};
  // statistics of an aknn_query_async call whose control blocks are still being
  // copied to `host` (graph loop, no round cap): finished on the next call on this
  // index or by aknn_get_stats, so the call itself never waits for the device
  struct Pending {
    bool on = false;
    cudaEvent_t ev = nullptr;
    std::vector<int> qn;  // queries per sub-batch
    size_t slot = 0;      // bytes per sub-batch in `host`
  } pending;
  Geom pending_geom{};
  int pending_outputs_per_batch = 0;
};

namespace {


aknn_status make_index(int64_t n_local, int64_t n_global, int64_t offset, int32_t d,
                       aknn_index **out) {
  aknn_index *ix = new (std::nothrow) aknn_index();
  if (!ix) return fail(AKNN_ENOMEM, "host allocation failed");
  ix->n_local = n_local;
  ix->n_global = n_global;
  ix->offset = offset;
  ix->d = d;
  ix->pitch = round_up(d, 16);
  cudaError_t e = cudaGetDevice(&ix->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ix->num_sms, cudaDevAttrMultiProcessorCount, ix->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ix;
    return fail(AKNN_ECUDA, "CUDA device setup failed: %s", cudaGetErrorString(e));
  }
  aknn_status s = ix->X.ensure((size_t)n_local * ix->pitch);
  if (s != AKNN_OK) {
    cudaStreamDestroy(ix->stream);
    delete ix;
    return s;
  }
  *out = ix;
  return AKNN_OK;
}

// Philox blocks per lane in the advance kernel's lane groups (tuning knob; the
// results do not depend on it).  AKNN_ADV_BPL overrides for experiments.
unsigned adv_bpl() {
  static const unsigned v = [] {
    const char *e = getenv("AKNN_ADV_BPL");
    const unsigned x = e ? (unsigned)atoi(e) : 8u;
    return (x >= 4 && (x & (x - 1)) == 0) ? x : 8u;
  }();
  return v;
}

// Exact fallbacks on the tensor cores (exact_mma.cu) unless AKNN_FLAG_EXACT_ROWS.
// Workspace: nq [qb] int32 and the tile flags [ceil(qb/128)][ceil(npad/256)].
size_t exact_mma_ws_bytes(int64_t qb, int64_t npad) {
  const int64_t rt = (qb + exact_tile_rows() - 1) / exact_tile_rows();
  const int64_t ct = (npad + exact_tile_cols() - 1) / exact_tile_cols();
  return round_up((size_t)qb * 4, 256) + round_up((size_t)(rt * ct) * 4, 256);
}

// ||x_i||^2 for the tensor-core passes: computed once per index on the first
// stream that needs it; every later user (possibly on another stream) waits on the
// event recorded behind that kernel, so it never reads the norms early.
aknn_status ensure_row_norms(aknn_index *ix, cudaStream_t st) {
  if (!ix->nx_ready) {
    const int64_t npad = round_up(ix->n_local, 256);  // the fused exact pass reads whole 256-point tiles
    TRY(ix->nx.ensure(sizeof(int32_t) * (size_t)npad));
    if (!ix->nx_ev) CU(cudaEventCreateWithFlags(&ix->nx_ev, cudaEventDisableTiming));
    CU(cudaMemsetAsync(ix->nx.p, 0, sizeof(int32_t) * (size_t)npad, st));
    CU(launch_row_norms(ix->X.as<uint8_t>(), ix->pitch, (int)ix->n_local, ix->nx.as<int32_t>(), st));
    CU(cudaEventRecord(ix->nx_ev, st));
    ix->nx_ready = true;
    return AKNN_OK;
  }
  CU(cudaStreamWaitEvent(st, ix->nx_ev, 0));
  return AKNN_OK;
}

aknn_status setup_exact_mma(aknn_index *ix, Geom &g, int64_t qb, uint8_t *ws, const aknn_opts &o,
                            cudaStream_t st) {
  g.exact_mma = (o.flags & AKNN_FLAG_EXACT_ROWS) ? 0 : 1;
  if (!g.exact_mma) return AKNN_OK;
  TRY(ensure_row_norms(ix, st));
  g.nx = ix->nx.as<int32_t>();
  g.nq = reinterpret_cast<int32_t *>(ws);
  g.xflags = reinterpret_cast<uint32_t *>(ws + round_up((size_t)qb * 4, 256));
  g.xf_cols = (int)((g.npad + exact_tile_cols() - 1) / exact_tile_cols());
  // a 128 x 256 tile costs about as much as streaming ~800 pairs' rows: smaller counts
  // take the row path (AKNN_XMIN overrides)
  static const int xmin = [] {
    const char *e = getenv("AKNN_XMIN");
    return e && e[0] ? atoi(e) : 512;
  }();
  g.xmin = (o.flags & AKNN_FLAG_EXACT_MMA_ALL) ? 1u : (uint32_t)(xmin < 1 ? 1 : xmin);
  return AKNN_OK;
}

// Tile-staged level gathers (advance_tiles.cu) unless AKNN_FLAG_NO_TILES / AKNN_TILE=0.
// Tile shape: the largest R x P (powers of two, R <= P, 4 <= P <= 32) whose shared
// memory fits 3 CTAs per SM, else 2, else 1.  AKNN_TILE_LR / AKNN_TILE_LP override (experiments).  A tile is dense
// (staged) when its draws, at one 32-byte sector each on the list path, cost at least
// AKNN_TILE_F (default 4) times its staging bytes (R + P) * pitch.
struct TileShape {
  int on, lr, lp;
  float row_draws;
  int groups;  // > 0: grouped tiles (one CTA per SM, point rows shared by the groups)
  int tight;   // grouped, rows at the pitch
  int db;      // grouped, double-buffered query rows
};

int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e && e[0] ? atoi(e) : dflt;
}

TileShape tile_shape(int64_t pitch, int64_t n) {
  TileShape t{0, 0, 0, 0.f, 0, 0, 0};
  if (env_int("AKNN_TILE", 1) == 0) return t;
  // the largest tile (R * P) whose shared memory fits 3, 2 or 1 CTAs per SM (228 KB);
  // rows wider than 8 KB: the largest tile at one CTA per SM (C3, d = 12,288: 4 x 8 at
  // one CTA beat 2 x 4 at two by 14 % -- staging amortised over 4x the pairs)
  int lr = -1, lp = -1;
  const std::vector<size_t> caps = pitch > 8192 ? std::vector<size_t>{(size_t)233472}
                                                 : std::vector<size_t>{(size_t)233472 / 3, (size_t)233472 / 2, (size_t)233472};
  for (size_t cap : caps) {
    for (int a = 5; a >= 0; --a)
      for (int b = 5; b >= 2; --b)
        if (a <= b && tile_smem_bytes(a, b, pitch) <= cap && (lr < 0 || a + b > lr + lp)) {
          lr = a;
          lp = b;
        }
    if (lr >= 0) break;
  }
  if (lr < 0) return t;
  t.lr = env_int("AKNN_TILE_LR", lr);
  t.lp = env_int("AKNN_TILE_LP", lp);
  // rows wider than 8 KB: NG thread groups share the column's P = 8 point rows
  // (AKNN_TILE_GROUPS: 10 = default, 2-warp groups of one query row at the pitch; 8; 24 =
  // 8 groups of 3 warps; 5 = 4-warp groups of two query rows; 4 = power-of-two slots;
  // 2; 0 = the classic kernel)
  // AKNN_TILE_TIGHT = 1: rows at the pitch (not in power-of-two slots), so 16 point rows
  // fit with 2 groups of one query row (the query rows restaged per pair halve)
  // AKNN_TILE_GROUPS = 2 with AKNN_TILE_DB = 1: 2 groups of one query row, each double-
  // buffering its query rows (the next tile's copy overlaps this tile's draws)
  const int ng0 = pitch > 8192 ? env_int("AKNN_TILE_GROUPS", 10) : 0;
  // the default (10 groups at the pitch) needs 18 rows: narrower CTAs when it does not fit
  const int ng = (ng0 == 10 && tile_grp_smem_bytes(10, 0, 3, pitch, true, false) > (size_t)227 * 1024)
                     ? (tile_grp_smem_bytes(8, 0, 3, pitch, true, false) <= (size_t)227 * 1024 ? 8 : 4)
                     : ng0;
  const int tight = env_int("AKNN_TILE_TIGHT", 0), db = env_int("AKNN_TILE_DB", 1);
  if ((ng == 8 || ng == 10 || ng == 24) && tile_grp_smem_bytes(ng == 24 ? 8 : ng, 0, 3, pitch, true, false) <= (size_t)227 * 1024) {
    t.groups = ng;  // 8 / 10 groups of 2 warps (24: 8 groups of 3 warps), rows at the pitch
    t.tight = 1;
    t.lr = 0;
    t.lp = 3;
  } else if (ng == 5 && tile_grp_smem_bytes(5, 1, 3, pitch, true, false) <= (size_t)227 * 1024) {
    t.groups = 5;  // 5 groups of 4 warps, each on two query rows (R = 2) at the pitch
    t.tight = 1;
    t.lr = 1;
    t.lp = 3;
  } else if (ng == 2 && tight && tile_grp_smem_bytes(2, 0, 4, pitch, true, false) <= (size_t)227 * 1024) {
    t.groups = 2;
    t.tight = 1;
    t.lr = 0;
    t.lp = 4;
  } else if (ng == 2 && db && tile_grp_smem_bytes(2, 0, 3, pitch, false, true) <= (size_t)227 * 1024) {
    t.groups = 2;
    t.db = 1;
    t.lr = 0;
    t.lp = 3;
  } else if ((ng == 2 || ng == 4) && tile_grp_smem_bytes(ng, ng == 4 ? 0 : 1, 3, pitch, false, false) <= (size_t)227 * 1024) {
    t.groups = ng;
    t.lr = ng == 4 ? 0 : 1;
    t.lp = 3;
  }
  if (t.lr < 0 || t.lr > 5 || t.lp < 2 || t.lp > 5 ||
      (!t.groups && tile_smem_bytes(t.lr, t.lp, pitch) > (size_t)233472))
    return TileShape{0, 0, 0, 0.f, 0, 0, 0};
  // X in L2 (C2: 47 MB): a list draw costs one L2 sector, tiles must amortise their
  // staging over >= 4 sectors' worth of draws; X in HBM (C3-C5): a list draw is a
  // random HBM sector (~1/15 the Philox rate): F = 1 on C4 (F = 0.25 / 1 / 4: 101.0 /
  // 100.0 / 100.4 ms), 0.25 with the grouped tiles of rows > 8 KB (C3, 8 groups: 277.6
  // / 279.2 / 290.9 ms at F = 0.25 / 0.5 / 1)
  const char *fe = getenv("AKNN_TILE_F");
  const bool x_in_l2 = (double)n * (double)pitch <= 100e6;
  const double f = fe && fe[0] ? atof(fe) : (x_in_l2 ? 4.0 : (pitch > 8192 ? 0.25 : 1.0));
  t.row_draws = (float)(f * (double)pitch / 32.0);
  t.on = 1;
  return t;
}

size_t tile_ws_bytes(int64_t qb, int64_t npad, const TileShape &t) {
  if (!t.on) return 0;
  const int64_t rows = (qb + (1ll << t.lr) - 1) >> t.lr, cols = (npad + (1ll << t.lp) - 1) >> t.lp;
  return round_up((size_t)(rows * cols) * 4, 256);  // tilework
}

void setup_tiles(Geom &g, const TileShape &t, const aknn_opts &o, int64_t qb, uint8_t *ws) {
  // (the tile kernels implement the doubling schedule; growth 2 takes the lists)
  g.tile_on = (t.on && !(o.flags & AKNN_FLAG_NO_TILES) && g.growth <= 1) ? 1 : 0;
  g.advanced = &g.ctl->advanced;
  if (!g.tile_on) return;
  g.tile_lr = t.lr;
  g.tile_lp = t.lp;
  // (shared draws run per-pair Philox with the shared counter word there: same kernel)
  g.tile_groups = (o.flags & AKNN_FLAG_WITHOUT_REPLACEMENT) ? 0 : t.groups;
  g.tile_tight = t.tight;
  g.tile_db = t.db;
  g.tile_cols = (int)((g.npad + (1ll << t.lp) - 1) >> t.lp);
  g.tilework = reinterpret_cast<uint32_t *>(ws);
  g.tile_slot_l = tile_slot_log2(g.pitch);
  g.tile_tma = env_int("AKNN_TILE_TMA", 1) ? 1 : 0;  // A/B measurements only
  // consecutive tiles of a point column share the staged point rows: a tile stages
  // about its R query rows (+ one point row's share)
  g.tile_min_draws = t.row_draws * (float)((1 << t.lr) + 1);
  // AKNN_TILE_ZS = s > 0: the grouped shape's tiles whose pairs draw >= s each take the
  // |x - q| kernel (k_advance_tiles_z).  Off by default: on C3 it cut the shared-memory
  // wavefronts of the largest level by 41 % but ran 112.7 / 68.1 ms at 4,096 / 2,048
  // draws per pair against the grouped kernel's 108.4 / 57.2
  const int zs = env_int("AKNN_TILE_ZS", 0);
  // AKNN_TILE_QG = s: the 10-group shape's tiles whose pairs draw < s each gather their
  // query bytes from global memory (no query-row copies; 0 = off)
  const int qgs = env_int("AKNN_TILE_QG", 128);
  g.tile_qg_draws = (g.tile_groups == 10 && qgs > 0) ? (float)qgs * (float)(1 << t.lp) : 0.f;
  g.tile_z_draws = (g.tile_groups && zs > 0 && tile_z_ok(t.lr, t.lp, g.pitch, qb)) ? (float)zs * (float)(1 << t.lp) : 0.f;

}

// One round after the rank split: filter -> plan/scatter (+ dense-tile list) ->
// advance (tensor-core exact fallbacks, list levels) -> dense tiles.  timer(k): per-class
// event brackets of the host-driven loop (0 start, 1 filter, 2 compact, 3 advance,
// 4 tiles).
size_t lvcnt_bytes(int64_t qb, int64_t npad);  // (below)

template <class Timer>
cudaError_t launch_round_pass(const Geom &g, int num_sms, cudaStream_t st, Timer &timer) {
  timer(0);
  cudaError_t e = cudaSuccess;
  if (g.level_mma) e = cudaMemsetAsync(g.lvcnt, 0, lvcnt_bytes(g.q, g.npad), st);
  if (e == cudaSuccess && g.tile_on) e = cudaMemsetAsync(&g.ctl->tile_max, 0, sizeof(unsigned int), st);
  if (e == cudaSuccess && g.tile_on) e = cudaMemsetAsync(&g.ctl->tile_min, 0xFF, sizeof(unsigned int), st);
  if (e == cudaSuccess) e = launch_filter(g, st);
  timer(1);
  if (e == cudaSuccess) e = launch_compact(g, st);
  timer(2);
  if (e == cudaSuccess) e = launch_advance(g, num_sms, st);
  timer(3);
  if (e == cudaSuccess && g.tile_on) e = launch_advance_tiles(g, num_sms, st);
  if (e == cudaSuccess && g.level_mma) e = launch_level_mma(g, st);
  timer(4);
  return e;
}

// One round's advances: every blocker once, then (close-side lead L > 1, reading R24)
// L - 1 lead passes in which the blockers ranked in C or M advance again.
template <class Timer>
cudaError_t launch_round_body(const Geom &g, int num_sms, cudaStream_t st, Timer &&timer) {
  cudaError_t e = launch_round_pass(g, num_sms, st, timer);
  if (g.lead > 1) {
    Geom gl = g;
    gl.lead_pass = 1;
    for (int p = 1; p < g.lead && e == cudaSuccess; ++p) {
      e = launch_zero_round(g, st);  // the per-pass slot counters
      if (e == cudaSuccess) e = launch_round_pass(gl, num_sms, st, timer);
    }
  }
  return e;
}

// Shared draws on the tensor cores (k_level_mma): q^2 planes [qb][pitch] x 2, the
// level's w planes [n][pitch] x 3, wa [n], wovf [n], per-(128 x 128, level) counts.
// k_build_w keeps 8 warps' coordinate counts in shared memory (8 * pitch * 4 B): rows
// wider than 6 KB take the shared-draw tiles / lists instead
bool level_mma_on(const aknn_opts &o, int64_t pitch) {
  return (o.flags & AKNN_FLAG_SHARED_DRAWS) && !(o.flags & AKNN_FLAG_NO_LEVEL_MMA) && env_int("AKNN_LEVEL_MMA", 1) &&
         pitch <= 6144;
}
size_t lvcnt_bytes(int64_t qb, int64_t npad) {
  return (size_t)((qb + level_tile_rows() - 1) / level_tile_rows()) *
         (size_t)((npad + level_tile_cols() - 1) / level_tile_cols()) * MAX_LEVELS * sizeof(uint32_t);
}
size_t level_ws_bytes(int64_t qb, int64_t n, int64_t npad, int64_t pitch, const aknn_opts &o) {
  if (!level_mma_on(o, pitch)) return 0;
  return 2 * round_up((size_t)qb * pitch, 256) + 3 * round_up((size_t)n * pitch, 256) +
         round_up((size_t)npad * 4, 256) + round_up((size_t)n, 256) + round_up(lvcnt_bytes(qb, npad), 256);
}
void setup_level_mma(Geom &g, int64_t qb, uint8_t *ws, const aknn_opts &o) {
  g.level_mma = level_mma_on(o, g.pitch) ? 1 : 0;
  if (!g.level_mma) return;
  g.tile_on = 0;  // the non-GEMM pairs take the lists
  const size_t qp = round_up((size_t)qb * g.pitch, 256), np = round_up((size_t)g.n * g.pitch, 256);
  g.q2lo = ws;
  g.q2hi = ws + qp;
  g.wx0 = ws + 2 * qp;
  g.wx1 = g.wx0 + np;
  g.wc = g.wx1 + np;
  g.wa = reinterpret_cast<int32_t *>(g.wc + np);
  g.wovf = reinterpret_cast<uint8_t *>(g.wa) + round_up((size_t)g.npad * 4, 256);  // wa: npad ints
  g.lvcnt = reinterpret_cast<uint32_t *>(g.wovf + round_up((size_t)g.n, 256));
  g.lv_cols = (int)((g.npad + level_tile_cols() - 1) / level_tile_cols());
  static const int lmin = env_int("AKNN_LMIN", 2048);
  g.lmin = (uint32_t)(lmin < 1 ? 1 : lmin);
}

// Builds the level geometry of the composite key (R9) for a count
// schedule (growth 1: doubling, reading R7; growth 2: reading R25).
struct KeyGeom {
  unsigned long long L, Ld, L3;
  int cmax, ibits, kbits, nbits, growth;
};

// ibits: local index bits of a work-list code; kbits: GLOBAL id bits of the key.
// L = lcm(T_0 .. T_cmax, d) over the sampled counts, so S * (L / T) is an integer order
// key for every level.
aknn_status key_geom(int64_t n_local, int64_t n_global, int32_t d, KeyGeom *kg, int growth = 1) {
  int cmax = 0;
  while (d >= 2 && cmax + 1 < MAX_LEVELS && lvl_count((uint32_t)cmax + 1u, growth) < (uint32_t)d) ++cmax;
  unsigned long long L = (unsigned long long)d;
  for (int c = 0; c <= cmax; ++c) {
    const unsigned long long t = lvl_count((uint32_t)c, growth);
    L = L / gcd_u64(L, t) * t;
  }
  kg->growth = growth;
  kg->L = L;
  kg->Ld = L / (unsigned long long)d;
  kg->L3 = L % 3ull == 0 ? L / 3ull : 0ull;
  kg->cmax = cmax;
  kg->ibits = bit_length((unsigned long long)(n_local - 1));
  if (kg->ibits < 1) kg->ibits = 1;
  kg->kbits = bit_length((unsigned long long)(n_global - 1));
  if (kg->kbits < 1) kg->kbits = 1;
  kg->nbits = bit_length(65025ull * L) + kg->kbits;
  if (kg->nbits > 63)
    return fail(AKNN_EINVAL, "composite key needs %d bits (> 63) for n=%lld, d=%d, growth %d", kg->nbits,
                (long long)n_global, d, growth);
  return AKNN_OK;
}

// Bit c set: an arm advancing out of level c would reach d samples, so it goes exact
// instead (reading R8).
uint32_t exnext_mask(int32_t d, int growth) {
  uint32_t m = 0;
  for (uint32_t c = 0; c < (uint32_t)MAX_LEVELS; ++c)
    if (lvl_count(c + 1u, growth) >= (uint32_t)d) m |= 1u << c;
  return m;
}

// Build-time domain (include/aknn.h): sizes, and the composite rank key of the
// whole point set must fit 63 bits, so every later query on the index can rank.
aknn_status validate_build(int64_t n, int32_t d, int64_t n_global) {
  if (n < 2 || n >= (1ll << 31)) return fail(AKNN_EINVAL, "n=%lld outside [2, 2^31)", (long long)n);
  if (d < 1 || d > 33025) return fail(AKNN_EINVAL, "d=%d outside [1, 33025]", d);
  if (n_global < n || n_global >= (1ll << 31))
    return fail(AKNN_EINVAL, "n_global=%lld outside [n_local, 2^31)", (long long)n_global);
  KeyGeom kg;
  return key_geom(n, n_global, d, &kg);
}

aknn_status host_alpha_table(int kind, int64_t n, double delta, double c_alpha, int32_t d,
                             double *a) {
  if (n < 1 || d < 1 || !(delta > 0.0 && delta < 1.0))
    return fail(AKNN_EINVAL, "alpha table: need n >= 1, d >= 1, delta in (0,1)");
  a[0] = 0.0;
  a[d] = 0.0;
  if (kind == 0) {
    // footnote 2
    const double inv = (double)n / delta;  // 1 / delta'
    const double lg = std::log(inv);
    if (!(lg > 1.0)) return fail(AKNN_EINVAL, "footnote-2 alpha needs delta/n < 1/e");
    const double base = lg + 3.0 * std::log(lg);
    for (int32_t u = 1; u < d; ++u) {
      const double beta = base + 1.5 * std::log(1.0 + std::log((double)u));
      a[u] = std::sqrt(2.0 * beta / (double)u);
    }
    return AKNN_OK;
  }
  if (kind == 1) {
    // §5
    if (!(c_alpha > 0.0)) return fail(AKNN_EINVAL, "c_alpha must be > 0");
    for (int32_t u = 1; u < d; ++u)
      a[u] = std::sqrt(c_alpha * std::log(1.0 + (1.0 + std::log((double)u)) * (double)n / delta) / (double)u);
    return AKNN_OK;
  }
  return fail(AKNN_EINVAL, "alpha kind %d unknown (0 = footnote 2, 1 = section 5)", kind);
}

// Waits for `st` by polling an event instead of blocking in cudaStreamSynchronize:
// a blocked host thread can be descheduled (seen on the VM hosts: wake-ups 100+ ms
// late), and every round trip of the host loop -- and the return of every call --
// would pay for it.  The spin costs one host core while the device works.
cudaError_t sync_spin(cudaStream_t st) {
  thread_local cudaEvent_t ev = nullptr;
  if (!ev) {
    const cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaEventRecord(ev, st);
  if (e != cudaSuccess) return e;
  for (;;) {
    e = cudaEventQuery(ev);
    if (e != cudaErrorNotReady) return e;
  }
}

// Waits for `st` on an index of an NCCL communicator: the event poll of sync_spin plus
// the communicator's asynchronous error state and a wall-clock deadline (host_wait.h);
// on a peer error or a timeout the communicator is aborted -- the pending collective
// then fails on every rank instead of hanging -- and the call returns AKNN_ENCCL.
aknn_status wait_stream(aknn_index *ix, cudaStream_t st) {
#ifdef AKNN_WITH_NCCL
  if (ix->world > 1) {
    if (ix->nccl_failed || !ix->comm) return fail(AKNN_ENCCL, "the communicator was aborted by an earlier failure");
    thread_local cudaEvent_t ev = nullptr;
    if (!ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CU(cudaEventRecord(ev, st));
    cudaError_t dev_err = cudaSuccess;
    ncclResult_t peer = ncclSuccess;
    const WaitResult w = wait_loop(
        [&] {
          const cudaError_t e = cudaEventQuery(ev);
          if (e == cudaSuccess) return 1;
          if (e == cudaErrorNotReady) return 0;
          dev_err = e;
          return -1;
        },
        [&] {
          ncclResult_t r = ncclSuccess;
          if (ncclCommGetAsyncError(ix->comm, &r) != ncclSuccess) r = ncclInternalError;
          peer = r;
          return r != ncclSuccess && r != ncclInProgress;
        },
        [&] {
          ncclCommAbort(ix->comm);
          ix->comm = nullptr;
          ix->nccl_failed = true;
        },
        [] {
          return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
              .count();
        },
        ix->nccl_timeout_ms);
    if (w == WAIT_DEVICE_ERROR)
      return fail(AKNN_ECUDA, "waiting for the sharded round: %s", cudaGetErrorString(dev_err));
    if (w == WAIT_PEER_ERROR)
      return fail(AKNN_ENCCL, "NCCL reported %s on rank %d; communicator aborted", ncclGetErrorString(peer),
                  ix->rank);
    if (w == WAIT_TIMEOUT)
      return fail(AKNN_ENCCL, "no progress for %.0f ms on rank %d (dead peer?); communicator aborted",
                  ix->nccl_timeout_ms, ix->rank);
    return AKNN_OK;
  }
#endif
  CU(sync_spin(st));
  return AKNN_OK;
}

// Per-launch CUDA events on the launching stream, read after the call's final
// synchronisation (no extra host round trips).  Events are pooled per index.
enum Phase { PH_INIT = 0, PH_SELECT, PH_FILTER, PH_COMPACT, PH_ADVANCE, PH_TILES, PH_OUTPUT, PH_ALL, PH_N };

struct PhaseTimer {
  bool on;
  cudaStream_t s;
  EventPool *pool;
  struct Rec {
    int ph;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  cudaEvent_t open_a = nullptr;
  PhaseTimer(bool on_, cudaStream_t s_, EventPool *p) : on(on_), s(s_), pool(p) {
    if (on) pool->used = 0;
  }
  void start() {
    if (!on) return;
    open_a = pool->get();
    if (open_a) cudaEventRecord(open_a, s);
  }
  void stop(int ph) {
    if (!on || !open_a) return;
    cudaEvent_t b = pool->get();
    if (!b) return;
    cudaEventRecord(b, s);
    recs.push_back(Rec{ph, open_a, b});
    open_a = nullptr;
  }
  // call after the stream has been synchronised past every recorded event
  void resolve(double ms[PH_N]) {
    for (int i = 0; i < PH_N; ++i) ms[i] = 0.0;
    for (const Rec &r : recs) {
      float m = 0.f;
      if (cudaEventElapsedTime(&m, r.a, r.b) == cudaSuccess) ms[r.ph] += m;
    }
  }
};

// The round loop of one query sub-batch as ONE CUDA graph: reset, init (a2), rank
// split (a6-a7), then a conditional WHILE node whose body is filter -> plan ->
// scatter -> advance -> zero -> rank split -> k_round_ctl, the last of which sets the
// condition on the device.  No host round trip per round.  The instantiated graph is
// cached on the index and reused while the launch parameters are unchanged.
aknn_status loop_graph(aknn_index *ix, const Geom &g, int nbits, int max_rounds, cudaGraphExec_t *out,
                       int32_t *builds) {
  std::vector<unsigned char> key(sizeof(Geom) + 2 * sizeof(int));
  memcpy(key.data(), &g, sizeof(Geom));
  memcpy(key.data() + sizeof(Geom), &nbits, sizeof(int));
  memcpy(key.data() + sizeof(Geom) + sizeof(int), &max_rounds, sizeof(int));
  if (ix->loop_exec && key == ix->loop_key) {
    *out = ix->loop_exec;
    return AKNN_OK;
  }
  if (ix->loop_exec) {
    cudaGraphExecDestroy(ix->loop_exec);
    ix->loop_exec = nullptr;
  }
  if (!ix->cap_stream) CU(cudaStreamCreateWithFlags(&ix->cap_stream, cudaStreamNonBlocking));
  cudaStream_t cs = ix->cap_stream;
  cudaGraph_t graph = nullptr;
  CU(cudaGraphCreate(&graph, 0));
  struct GraphFree {
    cudaGraph_t g;
    ~GraphFree() {
      if (g) cudaGraphDestroy(g);
    }
  } gf{graph};
  cudaGraphConditionalHandle h;
  CU(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
  CU(cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  cudaError_t e = launch_ctl_reset(g.ctl, (unsigned)g.q, cs);
  if (e == cudaSuccess) e = launch_init(g, cs);
  if (e == cudaSuccess) e = launch_select(g, nbits, cs);
  if (e == cudaSuccess) e = launch_round_ctl(g.ctl, h, max_rounds, cs);
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t *deps = nullptr;
  size_t ndeps = 0;
  if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps);
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode = nullptr;
  if (e == cudaSuccess) e = cudaGraphAddNode(&cnode, graph, deps, ndeps, &cp);
  if (e == cudaSuccess) e = cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies);
  cudaGraph_t captured = nullptr;
  const cudaError_t e2 = cudaStreamEndCapture(cs, &captured);
  if (e != cudaSuccess || e2 != cudaSuccess) {
    cudaGetLastError();
    return fail(AKNN_ECUDA, "capturing the round-loop graph: %s",
                cudaGetErrorString(e != cudaSuccess ? e : e2));
  }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CU(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  e = launch_round_body(g, ix->num_sms, cs, [](int) {});
  if (e == cudaSuccess) e = launch_zero_round(g, cs);
  if (e == cudaSuccess) e = launch_select(g, nbits, cs);
  if (e == cudaSuccess) e = launch_round_ctl(g.ctl, h, max_rounds, cs);
  cudaGraph_t body_out = nullptr;
  const cudaError_t e3 = cudaStreamEndCapture(cs, &body_out);
  if (e != cudaSuccess || e3 != cudaSuccess) {
    cudaGetLastError();
    return fail(AKNN_ECUDA, "capturing the loop body: %s", cudaGetErrorString(e != cudaSuccess ? e : e3));
  }
  cudaGraphExec_t exec = nullptr;
  CU(cudaGraphInstantiate(&exec, graph, 0));
  ++*builds;
  ix->loop_exec = exec;
  ix->loop_key = key;
  *out = exec;
  return AKNN_OK;
}

// Kernel launches per class (for aknn_stats; memset nodes excluded).
int launches_init_of(const Geom &g) { return 2 + (g.exact_mma ? 1 : 0) + (g.level_mma ? 1 : 0); }  // init, qstate, norms, q^2
// (every pass of a round: with a close-side lead L, L passes and L - 1 counter resets)
int launches_filter_of(const Geom &g) { return g.lead; }
int launches_compact_of(const Geom &g) { return (3 + (g.level_mma ? 1 : 0)) * g.lead; }  // plan, (w planes,) scatter, list sizes
int launches_advance_of(const Geom &g) {
  return (1 + (g.exact_mma ? 1 : 0) + (g.stage_lo < MAX_LEVELS ? 1 : 0)) * g.lead + (g.lead - 1);
}
int launches_tiles_of(const Geom &g) { return ((g.tile_on ? 1 : 0) + (g.level_mma ? 1 : 0)) * g.lead; }
int launches_output_of(const OutPtrs &o) { return 2 + ((o.counts || o.sums) ? 1 : 0); }  // tally, output

// Folds one sub-batch's control block and query states (copied to the host) into
// the statistics; graph = the device-driven loop counted the rounds itself.
void fold_batch_stats(aknn_stats &stats, const RoundCtl &ctl_h, const QState *qs, int qn, bool graph,
                      const Geom &g, int r, aknn_status *status) {
  if (graph) {
    r = (int)ctl_h.round;
    stats.query_rounds += (int64_t)ctl_h.qrounds;
    stats.blocked_query_rounds += (int64_t)ctl_h.brounds;
    stats.launches_init += 1 + launches_init_of(g);  // + loop reset
    stats.launches_select += 4 * r;                  // pivot, radix fallback, thresholds, round control
    stats.launches_filter += launches_filter_of(g) * (r - 1);
    stats.launches_compact += launches_compact_of(g) * (r - 1);
    stats.launches_advance += (launches_advance_of(g) + 1) * (r - 1);  // + counter reset
    stats.launches_tiles += launches_tiles_of(g) * (r - 1);
    if (ctl_h.n_active > 0 && status) *status = AKNN_EMAXROUNDS;
  }
  if (r > stats.rounds) stats.rounds = r;
  stats.active_pair_rounds += (int64_t)ctl_h.advanced;
  stats.tile_blocks += (int64_t)ctl_h.tile_blocks;
  stats.tile_draws += (int64_t)ctl_h.tile_draws;
  stats.level_mma_tiles += (int64_t)ctl_h.lmma_tiles;
  for (int a = 0; a < qn; ++a) {
    stats.draws += qs[a].draws;
    stats.exact_fallbacks += qs[a].nexact;
    stats.philox_blocks += qs[a].blocks;
  }
}

void total_launches(aknn_stats &stats) {
  stats.kernel_launches = stats.launches_init + stats.launches_select + stats.launches_filter +
                          stats.launches_compact + stats.launches_advance + stats.launches_tiles +
                          stats.launches_output;
}

// Completes the statistics of a deferred aknn_query_async call (waits for its copies).
aknn_status finish_pending(aknn_index *ix) {
  if (!ix->pending.on) return AKNN_OK;
  ix->pending.on = false;
  for (;;) {
    const cudaError_t e = cudaEventQuery(ix->pending.ev);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) return fail(AKNN_ECUDA, "waiting for the query: %s", cudaGetErrorString(e));
  }
  aknn_stats &stats = ix->stats;
  const Geom &g = ix->pending_geom;
  for (size_t b = 0; b < ix->pending.qn.size(); ++b) {
    const char *base = static_cast<const char *>(ix->host.p) + 256 + b * ix->pending.slot;
    const RoundCtl &ctl_h = *reinterpret_cast<const RoundCtl *>(base);
    const QState *qs = reinterpret_cast<const QState *>(base + sizeof(RoundCtl));
    fold_batch_stats(stats, ctl_h, qs, ix->pending.qn[b], true, g, 0, nullptr);
    stats.launches_output += ix->pending_outputs_per_batch;
  }
  total_launches(stats);
  return AKNN_OK;
}

// Runs the whole query on device pointers.  Q rows have stride `qstride`
// bytes in `queries_dev` (device).  Outputs are device pointers.
// Flag combinations the path does not define.
aknn_status check_flags(const aknn_opts &o) {
  if ((o.flags & AKNN_FLAG_WITHOUT_REPLACEMENT) && (o.flags & AKNN_FLAG_SHARED_DRAWS))
    return fail(AKNN_EINVAL, "AKNN_FLAG_WITHOUT_REPLACEMENT cannot be combined with AKNN_FLAG_SHARED_DRAWS");
  if (o.lead < 0 || o.lead > 8) return fail(AKNN_EINVAL, "lead must be in [0, 8] (got %d)", o.lead);
  if (o.batch_queries < 0) return fail(AKNN_EINVAL, "batch_queries must be >= 0 (got %d)", o.batch_queries);
  if (o.growth < 0 || o.growth > 2) return fail(AKNN_EINVAL, "growth must be 0, 1 or 2 (got %d)", o.growth);
  if (o.growth == 2 && (o.flags & (AKNN_FLAG_SHARED_DRAWS | AKNN_FLAG_WITHOUT_REPLACEMENT)))
    return fail(AKNN_EINVAL, "growth 2 runs with per-query draws with replacement only");
  return AKNN_OK;
}

aknn_status run_query(aknn_index *ix, const uint8_t *queries_dev, int64_t qstride, int32_t q,
                      int32_t k, int32_t h, uint64_t seed, const double *alpha_dev,
                      const aknn_opts *opts, const aknn_result *out, cudaStream_t st,
                      bool may_defer = false) {
  TRY(finish_pending(ix));
  const int64_t n = ix->n_local;
  const int32_t d = ix->d;
  KeyGeom kg;
  const aknn_opts o = opts ? *opts : aknn_opts{};
  TRY(check_flags(o));
  const int growth = o.growth > 1 ? o.growth : 1;
  TRY(key_geom(n, ix->n_global, d, &kg, growth));
  if (k + h > output_max_kh())
    return fail(AKNN_EINVAL, "k+h=%d exceeds the supported %d", k + h, output_max_kh());
  const int64_t npad = round_up(n, 16);
  // sub-batch size: the code (qi << ibits | i) must fit 32 bits; the
  // workspace (S 4 B + lvl 1 B + act 1 B + list 4 B per pair) fits in memory.
  int64_t qb = o.batch_queries > 0 ? std::min<int64_t>(q, o.batch_queries) : q;
  const int64_t code_cap = 1ll << (32 - kg.ibits);
  if (qb > code_cap) qb = code_cap;
  const size_t per_q = (size_t)npad * 10 + ix->pitch + sizeof(QState) + 64;
  if ((size_t)qb * per_q > ix->ws.bytes) {
    // only when the workspace must grow: cudaMemGetInfo is a driver round trip that
    // sometimes stalls the enqueueing thread for tens of ms
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    const size_t budget = (size_t)(0.6 * (double)(free_b + ix->ws.bytes));
    if ((size_t)qb * per_q > budget) qb = (int64_t)(budget / per_q);
  }
  if (qb < 1) return fail(AKNN_ENOMEM, "not enough device memory for one query row");
  // workspace layout
  const size_t szS = (size_t)qb * npad * 4, szL = (size_t)qb * npad, szA = szL,
               szList = (size_t)qb * npad * 4, szQ = (size_t)qb * ix->pitch,
               szQS = (size_t)qb * sizeof(QState), szCtl = sizeof(RoundCtl);
  size_t off = 0;
  const size_t oS = off; off = round_up(off + szS, 256);
  const size_t oL = off; off = round_up(off + szL, 256);
  const size_t oA = off; off = round_up(off + szA, 256);
  const size_t oList = off; off = round_up(off + szList, 256);
  const size_t oQ = off; off = round_up(off + szQ, 256);
  const size_t oQS = off; off = round_up(off + szQS, 256);
  const size_t oCtl = off; off = round_up(off + szCtl, 256);
  const size_t oXm = off; off = round_up(off + exact_mma_ws_bytes(qb, npad), 256);
  const TileShape tsh = tile_shape(ix->pitch, ix->n_local);
  const size_t oTw = off; off = round_up(off + tile_ws_bytes(qb, npad, tsh), 256);
  const size_t oThr = off; off = round_up(off + sizeof(int32_t) * THR_STRIDE * (size_t)qb, 256);  // (max stride)
  const size_t oLm = off; off = round_up(off + level_ws_bytes(qb, n, npad, ix->pitch, o), 256);
  const size_t oLead = off; off = round_up(off + (o.lead > 1 ? szL : 0), 256);
  const int rowany_cols = (int)((npad + 1023) / 1024);
  const size_t oRany = off; off = round_up(off + (size_t)((qb + 31) / 32) * rowany_cols * 4, 256);
  TRY(ix->ws.ensure(off));

  Geom g{};
  g.thr = ix->ws.as<int32_t>(oThr);
  g.X = ix->X.as<uint8_t>();
  g.Q = ix->ws.as<uint8_t>(oQ);
  g.alpha = alpha_dev;
  g.S = ix->ws.as<int32_t>(oS);
  g.lvl = ix->ws.as<uint8_t>(oL);
  g.act = ix->ws.as<uint8_t>(oA);
  g.lead = o.lead > 1 ? o.lead : 1;
  g.leadb = o.lead > 1 ? ix->ws.as<uint8_t>(oLead) : nullptr;
  g.rowany = ix->ws.as<uint32_t>(oRany);
  g.rowany_cols = rowany_cols;
  g.list = ix->ws.as<uint32_t>(oList);
  g.qs = ix->ws.as<QState>(oQS);
  g.ctl = ix->ws.as<RoundCtl>(oCtl);
  g.pitch = ix->pitch;
  g.npad = npad;
  g.n = (int)n;
  g.d = d;
  g.k = k;
  g.h = h;
  g.id_offset = (uint32_t)ix->offset;
  g.seed_lo = (uint32_t)(seed & 0xffffffffu);
  g.seed_hi = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    g.rk0[r] = g.seed_lo + (uint32_t)r * 0x9E3779B9u;
    g.rk1[r] = g.seed_hi + (uint32_t)r * 0xBB67AE85u;
  }
  g.L = kg.L;
  g.Ld = kg.Ld;
  g.L3 = kg.L3;
  g.growth = kg.growth;
  g.exnext = exnext_mask(d, kg.growth);
  g.ibits = kg.ibits;
  g.kbits = kg.kbits;
  g.world = 1;
  g.cmax = kg.cmax;
  g.adv_bpl = adv_bpl();
  g.force_radix = (o.flags & AKNN_FLAG_RADIX_SELECT) ? 1 : 0;
  g.shared_draws = (o.flags & AKNN_FLAG_SHARED_DRAWS) ? 1 : 0;
  g.wor = (o.flags & AKNN_FLAG_WITHOUT_REPLACEMENT) ? 1 : 0;
  g.wor_z = wor_radix(d);
  g.stage_lo = g.growth > 1 ? MAX_LEVELS : stage_level(g.pitch);  // staged rows: doubling only
  TRY(setup_exact_mma(ix, g, qb, ix->ws.as<uint8_t>(oXm), o, st));
  setup_tiles(g, tsh, o, qb, ix->ws.as<uint8_t>(oTw));
  setup_level_mma(g, qb, ix->ws.as<uint8_t>(oLm), o);

  aknn_stats stats{};
  stats.pairs = (int64_t)q * n;
  // the device-driven (graph) loop unless per-kernel timing was asked for, which
  // needs the host loop to bracket each launch with events
  static const bool no_graph = getenv("AKNN_NO_GRAPH") && getenv("AKNN_NO_GRAPH")[0] == '1';
  const bool use_graph = o.timing == 0 && !no_graph;
  PhaseTimer tm(o.timing != 0, st, &ix->events);
  tm.start();
  cudaEvent_t all_a = tm.open_a;
  // pinned host staging: [256 B: active count][per sub-batch: RoundCtl | QState[qb]]
  const int64_t nbatch = (q + qb - 1) / qb;
  const size_t slot = round_up(sizeof(RoundCtl) + sizeof(QState) * (size_t)qb, 64);
  CU(ix->host.ensure(256 + (size_t)nbatch * slot));
  unsigned int *h_active = static_cast<unsigned int *>(ix->host.p);
  // defer the statistics (no host wait at all) on the async graph path without a
  // round cap: the status cannot be EMAXROUNDS there
  const bool defer = may_defer && use_graph && o.max_rounds <= 0;
  const int outs_per_batch = (out->counts || out->sums) ? 3 : 2;  // tally, output, counts
  std::vector<int> batch_qn;
  tm.open_a = nullptr;
  aknn_status status = AKNN_OK;
  for (int64_t r0 = 0; r0 < q; r0 += qb) {
    const int qn = (int)std::min<int64_t>(qb, q - r0);
    const int64_t b = r0 / qb;
    RoundCtl *h_ctl = reinterpret_cast<RoundCtl *>(static_cast<char *>(ix->host.p) + 256 + (size_t)b * slot);
    QState *h_qs = reinterpret_cast<QState *>(h_ctl + 1);
    batch_qn.push_back(qn);
    g.q = qn;
    g.qi0 = (uint32_t)(o.qi_offset + r0);
    ++stats.query_batches;
    // stage queries into the zero-padded pitch layout
    CU(cudaMemsetAsync(ix->ws.as<uint8_t>(oQ), 0, szQ, st));
    CU(cudaMemcpy2DAsync(ix->ws.as<uint8_t>(oQ), ix->pitch, queries_dev + r0 * qstride, qstride, d,
                         qn, cudaMemcpyDeviceToDevice, st));
    int r = 0;
    if (use_graph) {
      // device-driven loop: one graph launch per sub-batch; the outputs are enqueued
      // behind it and the control block is read back once, at the end
      cudaGraphExec_t exec = nullptr;
      TRY(loop_graph(ix, g, kg.nbits, o.max_rounds, &exec, &stats.graph_builds));
      CU(cudaGraphLaunch(exec, st));
    }
    if (!use_graph) {
    CU(cudaMemsetAsync(g.ctl, 0, sizeof(RoundCtl), st));
    tm.start();
    CU(launch_init(g, st));
    tm.stop(PH_INIT);
    stats.launches_init += launches_init_of(g);
    unsigned evaluated = (unsigned)qn;  // queries the rank split looks at this round
    for (;;) {
      ++r;
      // zero the per-round counters (everything but the cumulative `advanced`)
      CU(launch_zero_round(g, st));
      tm.start();
      CU(launch_select(g, kg.nbits, st));
      tm.stop(PH_SELECT);
      stats.launches_select += 3;
      stats.query_rounds += evaluated;
      CU(cudaMemcpyAsync(h_active, &g.ctl->n_active, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
      CU(sync_spin(st));
      const unsigned nact = *h_active;
      stats.blocked_query_rounds += nact;
      evaluated = nact;
      if (nact == 0) break;
      if (o.max_rounds > 0 && r >= o.max_rounds) {
        status = AKNN_EMAXROUNDS;
        break;
      }
      CU(launch_round_body(g, ix->num_sms, st, [&](int k) {
        if (k == 0) {
          tm.start();
        } else if (k == 1) {
          tm.stop(PH_FILTER);
          tm.start();
        } else if (k == 2) {
          tm.stop(PH_COMPACT);
          tm.start();
        } else if (k == 3) {
          tm.stop(PH_ADVANCE);
          tm.start();
        } else {
          tm.stop(PH_TILES);
        }
      }));
      stats.launches_tiles += launches_tiles_of(g);
      stats.launches_filter += launches_filter_of(g);
      stats.launches_compact += launches_compact_of(g);
      stats.launches_advance += launches_advance_of(g);
      if (r > 1 + 64 * 64) return fail(AKNN_ECUDA, "round loop did not terminate (internal error)");
    }
    }  // host-driven loop
    OutPtrs op{(int)r0, 0, n, 0, out->sets, out->dhat, out->counts, out->sums, out->evals, out->draws, out->rounds};
    tm.start();
    CU(launch_output(g, op, st));
    tm.stop(PH_OUTPUT);
    CU(cudaMemcpyAsync(h_ctl, g.ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(h_qs, g.qs, sizeof(QState) * qn, cudaMemcpyDeviceToHost, st));
    if (defer) continue;  // folded in by finish_pending
    stats.launches_output += launches_output_of(op);
    CU(sync_spin(st));
    // EMAXROUNDS is recorded and the remaining sub-batches still run, so every
    // output row holds the state its query reached
    fold_batch_stats(stats, *h_ctl, h_qs, qn, use_graph, g, r, &status);
  }
  tm.open_a = all_a;
  tm.stop(PH_ALL);
  if (defer) {
    if (!ix->pending.ev) CU(cudaEventCreateWithFlags(&ix->pending.ev, cudaEventDisableTiming));
    CU(cudaEventRecord(ix->pending.ev, st));
    ix->pending.on = true;
    ix->pending.qn = batch_qn;
    ix->pending.slot = slot;
    ix->pending_geom = g;
    ix->pending_outputs_per_batch = outs_per_batch;
    ix->stats = stats;  // completed by finish_pending
    CU(cudaGetLastError());
    return AKNN_OK;
  }
  CU(sync_spin(st));
  double ms[PH_N];
  tm.resolve(ms);
  stats.ms_init = ms[PH_INIT];
  stats.ms_select = ms[PH_SELECT];
  stats.ms_filter = ms[PH_FILTER];
  stats.ms_compact = ms[PH_COMPACT];
  stats.ms_advance = ms[PH_ADVANCE];
  stats.ms_tiles = ms[PH_TILES];
  stats.ms_output = ms[PH_OUTPUT];
  stats.ms_total = ms[PH_ALL];
  total_launches(stats);
  ix->stats = stats;
  CU(cudaGetLastError());
  return status;
}

// ---------------------------------------------------------------------------
// The point-sharded round loop.  `shards` are either the one
// local shard of an NCCL communicator (nccl = true: one process per GPU, one
// ncclAllGather per round), or several shards of one point set on the current
// device driven in lockstep by this process (nccl = false: the exchange is
// that every shard writes its summary straight into the shared receive
// buffer).  Both run the same kernels and the same merge, so the results are
// identical to each other, to the unsharded path and to the oracle.
aknn_status run_query_sharded(const std::vector<aknn_index *> &shards, bool nccl,
                              const uint8_t *queries_dev, int32_t q, int32_t k, int32_t h,
                              uint64_t seed, const double *alpha_dev, const aknn_opts *opts,
                              const aknn_result *out, int64_t out_ncols, cudaStream_t st) {
  aknn_index *ix0 = shards[0];
  if (nccl && ix0->nccl_failed) return fail(AKNN_ENCCL, "the communicator was aborted by an earlier failure");
  for (aknn_index *sh : shards) TRY(finish_pending(sh));
  const int32_t d = ix0->d;
  const int W = nccl ? ix0->world : (int)shards.size();
  const int kh = k + h;
  if ((int64_t)W * kh > 16384)
    return fail(AKNN_EINVAL, "world * (k+h) = %lld exceeds 16384 (merge buffer)", (long long)W * kh);
  const aknn_opts o = opts ? *opts : aknn_opts{};
  TRY(check_flags(o));
  std::vector<KeyGeom> kg(shards.size());
  const int growth = o.growth > 1 ? o.growth : 1;
  for (size_t s = 0; s < shards.size(); ++s) TRY(key_geom(shards[s]->n_local, ix0->n_global, d, &kg[s], growth));
  // sub-batch size: list codes fit 32 bits on every shard; memory on this device
  int64_t qb = o.batch_queries > 0 ? std::min<int64_t>(q, o.batch_queries) : q;
  size_t free_b = 0, total_b = 0;
  CU(cudaMemGetInfo(&free_b, &total_b));
  size_t held = 0, per_q = (size_t)W * (kh + 1) * sizeof(ShardRec);
  for (size_t s = 0; s < shards.size(); ++s) {
    qb = std::min<int64_t>(qb, 1ll << (32 - kg[s].ibits));
    held += shards[s]->ws.bytes;
    per_q += (size_t)round_up(shards[s]->n_local, 16) * 10 + shards[s]->pitch + sizeof(QState) + 64 +
             (size_t)(kh + 1) * sizeof(ShardRec);
  }
  const size_t budget = (size_t)(0.6 * (double)(free_b + held));
  if ((size_t)qb * per_q > budget) qb = (int64_t)(budget / per_q);
#ifdef AKNN_WITH_NCCL
  if (nccl) {  // every rank must use the same sub-batches
    DevBuf tmp;
    TRY(tmp.ensure(sizeof(int64_t)));
    CU(cudaMemcpyAsync(tmp.p, &qb, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (ncclAllReduce(tmp.p, tmp.p, 1, ncclInt64, ncclMin, ix0->comm, st) != ncclSuccess)
      return fail(AKNN_ENCCL, "ncclAllReduce(qb) failed");
    CU(cudaMemcpyAsync(&qb, tmp.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    TRY(wait_stream(ix0, st));
  }
#endif
  if (qb < 1) return fail(AKNN_ENOMEM, "not enough device memory for one query row");
  const int64_t recv_stride = qb * (kh + 1);
  // per-shard workspace: S | lvl | act | list | Q | QState | RoundCtl | send | [recv]
  std::vector<Geom> G(shards.size());
  std::vector<size_t> oQv(shards.size()), szQv(shards.size());
  ShardRec *recv_shared = nullptr;
  for (size_t si = 0; si < shards.size(); ++si) {
    aknn_index *ix = shards[si];
    const int64_t npad = round_up(ix->n_local, 16);
    const bool has_recv = nccl || si == 0;
    const size_t szS = (size_t)qb * npad * 4, szL = (size_t)qb * npad,
                 szList = (size_t)qb * npad * 4, szQ = (size_t)qb * ix->pitch,
                 szQS = (size_t)qb * sizeof(QState), szCtl = sizeof(RoundCtl),
                 szSend = nccl ? (size_t)recv_stride * sizeof(ShardRec) : 0,
                 szRecv = has_recv ? (size_t)W * recv_stride * sizeof(ShardRec) : 0;
    size_t off = 0;
    const size_t oS = off; off = round_up(off + szS, 256);
    const size_t oL = off; off = round_up(off + szL, 256);
    const size_t oA = off; off = round_up(off + szL, 256);
    const size_t oList = off; off = round_up(off + szList, 256);
    const size_t oQ = off; off = round_up(off + szQ, 256);
    const size_t oQS = off; off = round_up(off + szQS, 256);
    const size_t oCtl = off; off = round_up(off + szCtl, 256);
    const size_t oSend = off; off = round_up(off + szSend, 256);
    const size_t oRecv = off; off = round_up(off + szRecv, 256);
    const size_t oXm = off; off = round_up(off + exact_mma_ws_bytes(qb, npad), 256);
    const TileShape tsh = tile_shape(ix->pitch, ix->n_local);
    const size_t oTw = off; off = round_up(off + tile_ws_bytes(qb, npad, tsh), 256);
    const size_t oThr = off; off = round_up(off + sizeof(int32_t) * THR_STRIDE * (size_t)qb, 256);  // (max stride)  // (max stride)
    const size_t oLm = off; off = round_up(off + level_ws_bytes(qb, ix->n_local, npad, ix->pitch, o), 256);
    const size_t oLead = off; off = round_up(off + (o.lead > 1 ? szL : 0), 256);
    const int rowany_cols = (int)((npad + 1023) / 1024);
    const size_t oRany = off; off = round_up(off + (size_t)((qb + 31) / 32) * rowany_cols * 4, 256);
    TRY(ix->ws.ensure(off));
    Geom &g = G[si];
    g = Geom{};
    g.thr = ix->ws.as<int32_t>(oThr);
    g.X = ix->X.as<uint8_t>();
    g.Q = ix->ws.as<uint8_t>(oQ);
    g.alpha = alpha_dev;
    g.S = ix->ws.as<int32_t>(oS);
    g.lvl = ix->ws.as<uint8_t>(oL);
    g.act = ix->ws.as<uint8_t>(oA);
    g.lead = o.lead > 1 ? o.lead : 1;
    g.leadb = o.lead > 1 ? ix->ws.as<uint8_t>(oLead) : nullptr;
    g.rowany = ix->ws.as<uint32_t>(oRany);
    g.rowany_cols = rowany_cols;
    g.list = ix->ws.as<uint32_t>(oList);
    g.qs = ix->ws.as<QState>(oQS);
    g.ctl = ix->ws.as<RoundCtl>(oCtl);
    g.pitch = ix->pitch;
    g.npad = npad;
    g.n = (int)ix->n_local;
    g.d = d;
    g.k = k;
    g.h = h;
    g.id_offset = (uint32_t)ix->offset;
    g.seed_lo = (uint32_t)(seed & 0xffffffffu);
    g.seed_hi = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) {
      g.rk0[r] = g.seed_lo + (uint32_t)r * 0x9E3779B9u;
      g.rk1[r] = g.seed_hi + (uint32_t)r * 0xBB67AE85u;
    }
    g.L = kg[si].L;
    g.Ld = kg[si].Ld;
    g.L3 = kg[si].L3;
    g.growth = kg[si].growth;
    g.exnext = exnext_mask(d, kg[si].growth);
    g.ibits = kg[si].ibits;
    g.kbits = kg[si].kbits;
    g.cmax = kg[si].cmax;
    g.adv_bpl = adv_bpl();
    g.force_radix = (o.flags & AKNN_FLAG_RADIX_SELECT) ? 1 : 0;
    g.shared_draws = (o.flags & AKNN_FLAG_SHARED_DRAWS) ? 1 : 0;
    g.wor = (o.flags & AKNN_FLAG_WITHOUT_REPLACEMENT) ? 1 : 0;
    g.wor_z = wor_radix(d);
    g.stage_lo = g.growth > 1 ? MAX_LEVELS : stage_level(g.pitch);  // staged rows: doubling only
    g.world = W;
    g.recv_stride = recv_stride;
    TRY(setup_exact_mma(ix, g, qb, ix->ws.as<uint8_t>(oXm), o, st));
    setup_tiles(g, tsh, o, qb, ix->ws.as<uint8_t>(oTw));
    setup_level_mma(g, qb, ix->ws.as<uint8_t>(oLm), o);
    if (has_recv) g.recv = ix->ws.as<ShardRec>(oRecv);
    if (si == 0 && !nccl) recv_shared = ix->ws.as<ShardRec>(oRecv);
    if (nccl) g.send = ix->ws.as<ShardRec>(oSend);
    oQv[si] = oQ;
    szQv[si] = szQ;
  }
  if (!nccl)
    for (size_t si = 0; si < shards.size(); ++si) {
      G[si].recv = recv_shared;
      G[si].send = recv_shared + (size_t)si * recv_stride;
    }

  aknn_stats stats{};
  for (aknn_index *ix : shards) stats.pairs += (int64_t)q * ix->n_local;
  PhaseTimer tm(o.timing != 0, st, &ix0->events);
  tm.start();
  cudaEvent_t all_a = tm.open_a;
  tm.open_a = nullptr;
  CU(ix0->host.ensure(256 + sizeof(RoundCtl) + sizeof(QState) * (size_t)qb));
  unsigned int *h_active = static_cast<unsigned int *>(ix0->host.p);
  RoundCtl *h_ctl = reinterpret_cast<RoundCtl *>(static_cast<char *>(ix0->host.p) + 256);
  QState *h_qs = reinterpret_cast<QState *>(h_ctl + 1);
  const size_t nS = shards.size();
  aknn_status status = AKNN_OK;
  for (int64_t r0 = 0; r0 < q; r0 += qb) {
    const int qn = (int)std::min<int64_t>(qb, q - r0);
    ++stats.query_batches;
    tm.start();
    for (size_t si = 0; si < nS; ++si) {
      Geom &g = G[si];
      g.q = qn;
      g.qi0 = (uint32_t)(o.qi_offset + r0);
      CU(cudaMemsetAsync(shards[si]->ws.as<uint8_t>(oQv[si]), 0, szQv[si], st));
      CU(cudaMemcpy2DAsync(shards[si]->ws.as<uint8_t>(oQv[si]), g.pitch, queries_dev + r0 * d, d, d,
                           qn, cudaMemcpyDeviceToDevice, st));
      CU(cudaMemsetAsync(g.ctl, 0, sizeof(RoundCtl), st));
      CU(launch_init(g, st));
      stats.launches_init += launches_init_of(g);
    }
    tm.stop(PH_INIT);
    if (!nccl && nS > 1) {  // shards add their counters into the output rows
      if (out->draws) CU(cudaMemsetAsync(out->draws + r0, 0, sizeof(int64_t) * qn, st));
      if (out->evals) CU(cudaMemsetAsync(out->evals + r0, 0, sizeof(int64_t) * qn, st));
    }
    int r = 0;
    unsigned evaluated = (unsigned)qn;
    for (;;) {
      ++r;
      tm.start();
      for (size_t si = 0; si < nS; ++si) {
        CU(launch_zero_round(G[si], st));
        CU(launch_select_local(G[si], kg[si].nbits, st));
        ++stats.launches_select;
      }
#ifdef AKNN_WITH_NCCL
      if (nccl) {
        if (ncclAllGather(G[0].send, const_cast<ShardRec *>(G[0].recv),
                          (size_t)recv_stride * sizeof(ShardRec), ncclUint8, ix0->comm, st) != ncclSuccess)
          return fail(AKNN_ENCCL, "ncclAllGather of the round summaries failed");
      }
#endif
      for (size_t si = 0; si < nS; ++si) {
        OutPtrs op{(int)r0, 0, 0, 0, (nccl || si == 0) ? out->sets : nullptr,
                   (nccl || si == 0) ? out->dhat : nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        CU(launch_merge(G[si], op, st));
        CU(launch_thresholds(G[si], st));
        stats.launches_select += 2;  // merge + thresholds
      }
      tm.stop(PH_SELECT);
      stats.query_rounds += evaluated;
      CU(cudaMemcpyAsync(h_active, &G[0].ctl->n_active, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
      TRY(wait_stream(ix0, st));
      const unsigned nact = *h_active;
      stats.blocked_query_rounds += nact;
      evaluated = nact;
      if (nact == 0) break;
      if (o.max_rounds > 0 && r >= o.max_rounds) {
        status = AKNN_EMAXROUNDS;
        break;
      }
      tm.start();
      for (size_t si = 0; si < nS; ++si) CU(launch_round_body(G[si], shards[si]->num_sms, st, [](int) {}));
      tm.stop(PH_ADVANCE);  // sharded: the whole round body is timed as one class (advance)
      stats.launches_filter += launches_filter_of(G[0]) * (int)nS;
      stats.launches_compact += launches_compact_of(G[0]) * (int)nS;
      stats.launches_advance += launches_advance_of(G[0]) * (int)nS;
      stats.launches_tiles += launches_tiles_of(G[0]) * (int)nS;
      if (r > 1 + 64 * 64) return fail(AKNN_ECUDA, "round loop did not terminate (internal error)");
    }
    if (r > stats.rounds) stats.rounds = r;
    tm.start();
    for (size_t si = 0; si < nS; ++si) {
      OutPtrs op{(int)r0, nccl ? 0 : shards[si]->offset, out_ncols, (!nccl && nS > 1) ? 1 : 0,
                 nullptr, nullptr, out->counts, out->sums, out->evals, out->draws, out->rounds};
      CU(launch_output_sharded(G[si], op, st));
      stats.launches_output += launches_output_of(op);
    }
#ifdef AKNN_WITH_NCCL
    if (nccl) {
      if (out->draws && ncclAllReduce(out->draws + r0, out->draws + r0, qn, ncclInt64, ncclSum, ix0->comm, st) != ncclSuccess)
        return fail(AKNN_ENCCL, "ncclAllReduce(draws) failed");
      if (out->evals && ncclAllReduce(out->evals + r0, out->evals + r0, qn, ncclInt64, ncclSum, ix0->comm, st) != ncclSuccess)
        return fail(AKNN_ENCCL, "ncclAllReduce(evals) failed");
    }
#endif
    tm.stop(PH_OUTPUT);
    for (size_t si = 0; si < nS; ++si) {
      CU(cudaMemcpyAsync(h_ctl, G[si].ctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
      CU(cudaMemcpyAsync(h_qs, G[si].qs, sizeof(QState) * qn, cudaMemcpyDeviceToHost, st));
      TRY(wait_stream(ix0, st));
      const RoundCtl &ctl_h = *h_ctl;
      const QState *qs = h_qs;
      stats.active_pair_rounds += (int64_t)ctl_h.advanced;
      stats.tile_blocks += (int64_t)ctl_h.tile_blocks;
      stats.tile_draws += (int64_t)ctl_h.tile_draws;
      stats.level_mma_tiles += (int64_t)ctl_h.lmma_tiles;
      for (int a = 0; a < qn; ++a) {
        stats.draws += qs[a].draws;
        stats.exact_fallbacks += qs[a].nexact;
        stats.philox_blocks += qs[a].blocks;
      }
    }
  }
  tm.open_a = all_a;
  tm.stop(PH_ALL);
  TRY(wait_stream(ix0, st));
  double ms[PH_N];
  tm.resolve(ms);
  stats.ms_init = ms[PH_INIT];
  stats.ms_select = ms[PH_SELECT];
  stats.ms_filter = ms[PH_FILTER];
  stats.ms_compact = ms[PH_COMPACT];
  stats.ms_advance = ms[PH_ADVANCE];
  stats.ms_tiles = ms[PH_TILES];
  stats.ms_output = ms[PH_OUTPUT];
  stats.ms_total = ms[PH_ALL];
  stats.kernel_launches = stats.launches_init + stats.launches_select + stats.launches_filter +
                          stats.launches_compact + stats.launches_advance + stats.launches_tiles +
                          stats.launches_output;
  ix0->stats = stats;
  CU(cudaGetLastError());
  return status;
}

aknn_status check_query_args(const aknn_index *ix, int32_t q, int32_t k, int32_t h, double delta,
                             const aknn_result *out) {
  if (!ix) return fail(AKNN_EINVAL, "index is NULL");
  if (!out || !out->sets) return fail(AKNN_EINVAL, "out->sets is required");
  if (q < 0) return fail(AKNN_EINVAL, "q=%d < 0", q);
  if (k < 1 || h < 0) return fail(AKNN_EINVAL, "need k >= 1 and h >= 0 (k=%d, h=%d)", k, h);
  if ((int64_t)k + h >= ix->n_global)
    return fail(AKNN_EINVAL, "k+h=%d must be < n=%lld (DESIGN.md R13)", k + h, (long long)ix->n_global);
  if ((int64_t)k + h >= ix->n_local)
    return fail(AKNN_EINVAL, "k+h=%d must be < n_local=%lld", k + h, (long long)ix->n_local);
  if (!(delta > 0.0 && delta < 1.0)) return fail(AKNN_EINVAL, "delta=%g outside (0,1)", delta);
  return AKNN_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

aknn_status aknn_build(const uint8_t *points, int64_t n, int32_t d, aknn_index **out) {
  if (!points || !out) return fail(AKNN_EINVAL, "NULL argument");
  TRY(validate_build(n, d, n));
  aknn_index *ix = nullptr;
  TRY(make_index(n, n, 0, d, &ix));
  cudaError_t e = cudaMemsetAsync(ix->X.p, 0, ix->X.bytes, ix->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(ix->X.p, ix->pitch, points, d, d, n, cudaMemcpyHostToDevice, ix->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ix->stream);
  if (e != cudaSuccess) {
    aknn_free(ix);
    return fail(AKNN_ECUDA, "copying points: %s", cudaGetErrorString(e));
  }
  *out = ix;
  return AKNN_OK;
}

aknn_status aknn_build_async(const uint8_t *points_dev, int64_t n, int32_t d, void *cuda_stream,
                             aknn_index **out) {
  if (!points_dev || !out) return fail(AKNN_EINVAL, "NULL argument");
  TRY(validate_build(n, d, n));
  aknn_index *ix = nullptr;
  TRY(make_index(n, n, 0, d, &ix));
  cudaStream_t s = (cudaStream_t)cuda_stream;
  cudaError_t e = cudaMemsetAsync(ix->X.p, 0, ix->X.bytes, s);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(ix->X.p, ix->pitch, points_dev, d, d, n, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) {
    aknn_free(ix);
    return fail(AKNN_ECUDA, "copying points: %s", cudaGetErrorString(e));
  }
  *out = ix;
  return AKNN_OK;
}

aknn_status aknn_nccl_unique_id(void *id_out) {
  if (!id_out) return fail(AKNN_EINVAL, "NULL argument");
#ifdef AKNN_WITH_NCCL
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return fail(AKNN_ENCCL, "ncclGetUniqueId failed");
  memcpy(id_out, &id, sizeof id);
  return AKNN_OK;
#else
  return fail(AKNN_ENCCL, "libaknn was built without NCCL");
#endif
}

aknn_status aknn_build_shard(const uint8_t *shard, int64_t n_local, int64_t n_global, int64_t offset,
                             int32_t d, const void *nccl_unique_id, int32_t rank, int32_t world,
                             aknn_index **out) {
  if (!shard || !out) return fail(AKNN_EINVAL, "NULL argument");
  if (n_global < n_local || n_global >= (1ll << 31))
    return fail(AKNN_EINVAL, "n_global=%lld < n_local=%lld", (long long)n_global, (long long)n_local);
  TRY(validate_build(n_local, d, n_global));
  if (n_global < n_local || offset < 0 || offset + n_local > n_global || n_global >= (1ll << 31))
    return fail(AKNN_EINVAL, "shard [%lld, %lld) outside [0, %lld)", (long long)offset,
                (long long)(offset + n_local), (long long)n_global);
  if (world < 1 || rank < 0 || rank >= world) return fail(AKNN_EINVAL, "rank %d of %d", rank, world);
  if (world > 1) {
#ifndef AKNN_WITH_NCCL
    return fail(AKNN_ENCCL, "sharded query across %d ranks needs NCCL (not built in)", world);
#endif
  }
  aknn_index *ix = nullptr;
  TRY(make_index(n_local, n_global, offset, d, &ix));
  ix->rank = rank;
  ix->world = world;
  cudaError_t e = cudaMemsetAsync(ix->X.p, 0, ix->X.bytes, ix->stream);
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(ix->X.p, ix->pitch, shard, d, d, n_local, cudaMemcpyHostToDevice, ix->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ix->stream);
  if (e != cudaSuccess) {
    aknn_free(ix);
    return fail(AKNN_ECUDA, "copying shard: %s", cudaGetErrorString(e));
  }
#ifdef AKNN_WITH_NCCL
  if (world > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof id);
    if (ncclCommInitRank(&ix->comm, world, id, rank) != ncclSuccess) {
      aknn_free(ix);
      return fail(AKNN_ENCCL, "ncclCommInitRank failed");
    }
  }
#else
  (void)nccl_unique_id;
#endif
  *out = ix;
  return AKNN_OK;
}

aknn_status aknn_alpha_table(int32_t kind, int64_t n, double delta, double c_alpha, int32_t d,
                             double *alpha_out) {
  if (!alpha_out) return fail(AKNN_EINVAL, "NULL argument");
  return host_alpha_table(kind, n, delta, c_alpha, d, alpha_out);
}

aknn_status aknn_query_async(const aknn_index *cix, const uint8_t *queries_dev, int32_t q, int32_t k,
                             int32_t h, double delta, uint64_t seed, const double *alpha_dev,
                             const aknn_opts *opts, aknn_result *out, void *cuda_stream) {
  aknn_index *ix = const_cast<aknn_index *>(cix);
  TRY(check_query_args(ix, q, k, h, delta, out));
  if (q > 0 && !queries_dev) return fail(AKNN_EINVAL, "queries is NULL");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const double *al = alpha_dev;
  if (!al) {
    std::vector<double> a(ix->d + 1);
    TRY(host_alpha_table(0, ix->n_global, delta, 0.0, ix->d, a.data()));
    TRY(ix->alpha.ensure(sizeof(double) * (ix->d + 1)));
    CU(cudaMemcpyAsync(ix->alpha.p, a.data(), sizeof(double) * (ix->d + 1), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
    al = ix->alpha.as<double>();
  }
  if (q == 0) return AKNN_OK;
  if (ix->world > 1) {
    std::vector<aknn_index *> one{ix};
    return run_query_sharded(one, true, queries_dev, q, k, h, seed, al, opts, out, ix->n_local, st);
  }
  return run_query(ix, queries_dev, ix->d, q, k, h, seed, al, opts, out, st, /*may_defer=*/true);
}

}  // extern "C"

namespace {
// Host-pointer query over one index (unsharded, or one NCCL shard) or over several
// shards of one point set on the current device (multi = true).
// Literal Algorithm 1 on device buffers: one warp per
// query (a1_kernels.cu), queries in launches whose workspace fits `budget`.
aknn_status run_query_a1(aknn_index *ix, const uint8_t *queries_dev, int32_t q, int32_t k, int32_t h,
                         uint64_t seed, const double *alpha_dev, const aknn_opts *opts,
                         const aknn_result *out, cudaStream_t st) {
  const int kh = k + h;
  if (kh > A1_MAX_KH) return fail(AKNN_EINVAL, "Algorithm 1 mode supports k+h <= %d (got %d)", A1_MAX_KH, kh);
  // shared-memory mode needs the state AND the alpha / query tables in one CTA's
  // window; otherwise every query's state lives in the global workspace
  const size_t per_s = a1_ws_per_query(ix->n_local, kh, ix->d, true);
  const bool smem = per_s <= A1_SMEM_MAX;
  const size_t per = smem ? per_s : a1_ws_per_query(ix->n_local, kh, ix->d, false);
  const size_t budget = (size_t)1 << 30;
  const int qb = smem ? q : (int)std::max<size_t>(1, std::min<size_t>((size_t)q, budget / per));
  TRY(ix->ws.ensure(256 + (smem ? 0 : per * (size_t)qb)));
  A1Geom g{};
  g.X = ix->X.as<uint8_t>();
  g.pitch = ix->pitch;
  g.Q = queries_dev;
  g.alpha = alpha_dev;
  g.n = (int)ix->n_local;
  g.d = ix->d;
  g.k = k;
  g.kh = kh;
  g.id_offset = (uint32_t)ix->offset;
  g.qi0 = opts ? (uint32_t)opts->qi_offset : 0u;
  g.max_iters = opts ? opts->max_rounds : 0;
  const uint32_t lo = (uint32_t)(seed & 0xffffffffu), hi = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    g.rk0[r] = lo + (uint32_t)r * 0x9E3779B9u;
    g.rk1[r] = hi + (uint32_t)r * 0xBB67AE85u;
  }
  g.status = ix->ws.as<int>();
  g.ws = ix->ws.as<unsigned char>(256);
  g.ws_per_query = per;
  g.smem = smem ? 1 : 0;
  g.wor = (opts && (opts->flags & AKNN_FLAG_WITHOUT_REPLACEMENT)) ? 1 : 0;
  g.wor_z = wor_radix(ix->d);
  g.out = OutPtrs{0, 0, ix->n_local, 0, out->sets, out->dhat, out->counts, out->sums,
                  out->evals, out->draws, out->rounds};
  CU(cudaMemsetAsync(g.status, 0, sizeof(int), st));
  int64_t launches = 0;
  for (int q0 = 0; q0 < q; q0 += qb) {
    g.q0 = q0;
    g.qb = std::min(qb, q - q0);
    CU(launch_a1(g, st));
    ++launches;
  }
  int *hs = nullptr;
  CU(ix->host.ensure(sizeof(int)));
  hs = static_cast<int *>(ix->host.p);
  CU(cudaMemcpyAsync(hs, g.status, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(sync_spin(st));
  ix->stats = aknn_stats{};
  ix->stats.query_batches = (int32_t)((q + qb - 1) / qb);
  ix->stats.kernel_launches = launches;
  ix->stats.pairs = (int64_t)q * ix->n_local;
  return (*hs & 1) ? AKNN_EMAXROUNDS : AKNN_OK;
}

aknn_status host_query(const std::vector<aknn_index *> &shards, bool multi, const uint8_t *queries,
                       int32_t q, int32_t k, int32_t h, double delta, uint64_t seed,
                       const double *alpha, const aknn_opts *opts, aknn_result *out, bool a1 = false) {
  aknn_index *ix = shards[0];
  if (q == 0) return AKNN_OK;
  cudaStream_t st = ix->stream;
  const int32_t d = ix->d;
  const int64_t n = multi ? ix->n_global : ix->n_local;  // row length of counts/sums
  const int kh = k + h;
  std::vector<double> a(d + 1);
  if (alpha) {
    memcpy(a.data(), alpha, sizeof(double) * (d + 1));
  } else {
    TRY(host_alpha_table(0, ix->n_global, delta, 0.0, d, a.data()));
  }
  // device staging: alpha | queries | outputs
  const size_t szA = sizeof(double) * (d + 1), szQ = (size_t)q * d;
  const size_t szSets = (size_t)q * kh * 4, szDhat = out->dhat ? (size_t)q * kh * 8 : 0,
               szCnt = out->counts ? (size_t)q * n * 4 : 0, szSum = out->sums ? (size_t)q * n * 8 : 0,
               szEv = (size_t)q * 8, szDr = (size_t)q * 8, szRo = (size_t)q * 4;
  size_t off = 0;
  const size_t oA = off; off = round_up(off + szA, 256);
  const size_t oQ = off; off = round_up(off + szQ, 256);
  const size_t oSets = off; off = round_up(off + szSets, 256);
  const size_t oDhat = off; off = round_up(off + szDhat, 256);
  const size_t oCnt = off; off = round_up(off + szCnt, 256);
  const size_t oSum = off; off = round_up(off + szSum, 256);
  const size_t oEv = off; off = round_up(off + szEv, 256);
  const size_t oDr = off; off = round_up(off + szDr, 256);
  const size_t oRo = off; off = round_up(off + szRo, 256);
  TRY(ix->outs.ensure(off));
  CU(cudaMemcpyAsync(ix->outs.as<char>(oA), a.data(), szA, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(ix->outs.as<char>(oQ), queries, szQ, cudaMemcpyHostToDevice, st));
  aknn_result dout{ix->outs.as<int32_t>(oSets), out->dhat ? ix->outs.as<double>(oDhat) : nullptr,
                   out->counts ? ix->outs.as<int32_t>(oCnt) : nullptr,
                   out->sums ? ix->outs.as<int64_t>(oSum) : nullptr, ix->outs.as<int64_t>(oEv),
                   ix->outs.as<int64_t>(oDr), ix->outs.as<int32_t>(oRo)};
  aknn_status s;
  if (a1)
    s = run_query_a1(ix, ix->outs.as<uint8_t>(oQ), q, k, h, seed, ix->outs.as<double>(oA), opts, &dout, st);
  else if (multi || ix->world > 1)
    s = run_query_sharded(shards, !multi, ix->outs.as<uint8_t>(oQ), q, k, h, seed,
                          ix->outs.as<double>(oA), opts, &dout, n, st);
  else
    s = run_query(ix, ix->outs.as<uint8_t>(oQ), d, q, k, h, seed, ix->outs.as<double>(oA), opts,
                  &dout, st);
  if (s != AKNN_OK && s != AKNN_EMAXROUNDS) return s;
  CU(cudaMemcpyAsync(out->sets, dout.sets, szSets, cudaMemcpyDeviceToHost, st));
  if (out->dhat) CU(cudaMemcpyAsync(out->dhat, dout.dhat, szDhat, cudaMemcpyDeviceToHost, st));
  if (out->counts) CU(cudaMemcpyAsync(out->counts, dout.counts, szCnt, cudaMemcpyDeviceToHost, st));
  if (out->sums) CU(cudaMemcpyAsync(out->sums, dout.sums, szSum, cudaMemcpyDeviceToHost, st));
  if (out->evals) CU(cudaMemcpyAsync(out->evals, dout.evals, szEv, cudaMemcpyDeviceToHost, st));
  if (out->draws) CU(cudaMemcpyAsync(out->draws, dout.draws, szDr, cudaMemcpyDeviceToHost, st));
  if (out->rounds) CU(cudaMemcpyAsync(out->rounds, dout.rounds, szRo, cudaMemcpyDeviceToHost, st));
  TRY(wait_stream(ix, st));
  return s;
}
}  // namespace

extern "C" {

aknn_status aknn_query_ex(const aknn_index *cix, const uint8_t *queries, int32_t q, int32_t k,
                          int32_t h, double delta, uint64_t seed, const double *alpha,
                          const aknn_opts *opts, aknn_result *out) {
  aknn_index *ix = const_cast<aknn_index *>(cix);
  TRY(check_query_args(ix, q, k, h, delta, out));
  if (q > 0 && !queries) return fail(AKNN_EINVAL, "queries is NULL");
  std::vector<aknn_index *> one{ix};
  return host_query(one, false, queries, q, k, h, delta, seed, alpha, opts, out);
}

aknn_status aknn_query_multi(const aknn_index *const *shards, int32_t nshards, const uint8_t *queries,
                             int32_t q, int32_t k, int32_t h, double delta, uint64_t seed,
                             const double *alpha, const aknn_opts *opts, aknn_result *out) {
  if (!shards || nshards < 1) return fail(AKNN_EINVAL, "need at least one shard");
  std::vector<aknn_index *> v(nshards);
  int64_t covered = 0;
  int dev = -1;
  CU(cudaGetDevice(&dev));
  for (int32_t s = 0; s < nshards; ++s) {
    v[s] = const_cast<aknn_index *>(shards[s]);
    if (!v[s]) return fail(AKNN_EINVAL, "shard %d is NULL", s);
    TRY(check_query_args(v[s], q, k, h, delta, out));
    if (v[s]->world != 1) return fail(AKNN_EINVAL, "shard %d belongs to an NCCL communicator", s);
    if (v[s]->device != dev) return fail(AKNN_EINVAL, "shard %d is not on the current device", s);
    if (v[s]->d != v[0]->d || v[s]->n_global != v[0]->n_global)
      return fail(AKNN_EINVAL, "shard %d has another dimension or n_global", s);
    if (v[s]->offset != covered)
      return fail(AKNN_EINVAL, "shards must tile [0, n_global) in order (shard %d starts at %lld, expected %lld)",
                  s, (long long)v[s]->offset, (long long)covered);
    covered += v[s]->n_local;
  }
  if (covered != v[0]->n_global)
    return fail(AKNN_EINVAL, "shards cover %lld of n_global=%lld points", (long long)covered,
                (long long)v[0]->n_global);
  if (q > 0 && !queries) return fail(AKNN_EINVAL, "queries is NULL");
  return host_query(v, true, queries, q, k, h, delta, seed, alpha, opts, out);
}

aknn_status aknn_query_a1(const aknn_index *cix, const uint8_t *queries, int32_t q, int32_t k,
                          int32_t h, double delta, uint64_t seed, const double *alpha,
                          const aknn_opts *opts, aknn_result *out) {
  aknn_index *ix = const_cast<aknn_index *>(cix);
  TRY(check_query_args(ix, q, k, h, delta, out));
  if (ix->world != 1 || ix->n_local != ix->n_global)
    return fail(AKNN_EINVAL, "Algorithm 1 mode needs an unsharded index");
  if (q > 0 && !queries) return fail(AKNN_EINVAL, "queries is NULL");
  if (ix->pending.on) TRY(finish_pending(ix));
  std::vector<aknn_index *> one{ix};
  return host_query(one, false, queries, q, k, h, delta, seed, alpha, opts, out, true);
}

aknn_status aknn_query_a1_device(const aknn_index *cix, const uint8_t *queries_dev, int32_t q, int32_t k,
                                 int32_t h, double delta, uint64_t seed, const double *alpha_dev,
                                 const aknn_opts *opts, aknn_result *out, void *cuda_stream) {
  aknn_index *ix = const_cast<aknn_index *>(cix);
  TRY(check_query_args(ix, q, k, h, delta, out));
  if (ix->world != 1 || ix->n_local != ix->n_global)
    return fail(AKNN_EINVAL, "Algorithm 1 mode needs an unsharded index");
  if (q > 0 && !queries_dev) return fail(AKNN_EINVAL, "queries is NULL");
  if (ix->pending.on) TRY(finish_pending(ix));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const double *al = alpha_dev;
  if (!al) {
    std::vector<double> a(ix->d + 1);
    TRY(host_alpha_table(0, ix->n_global, delta, 0.0, ix->d, a.data()));
    TRY(ix->alpha.ensure(sizeof(double) * (ix->d + 1)));
    CU(cudaMemcpyAsync(ix->alpha.p, a.data(), sizeof(double) * (ix->d + 1), cudaMemcpyHostToDevice, st));
    al = ix->alpha.as<double>();
  }
  if (q == 0) return AKNN_OK;
  return run_query_a1(ix, queries_dev, q, k, h, seed, al, opts, out, st);
}

aknn_status aknn_query(const aknn_index *ix, const uint8_t *queries, int32_t q, int32_t k, int32_t h,
                       double delta, uint64_t seed, const double *alpha, aknn_result *out) {
  return aknn_query_ex(ix, queries, q, k, h, delta, seed, alpha, nullptr, out);
}

// ---------------------------------------------------------------------------
// Host reference of the shard protocol (the same records, keys, tie rules and
// merge as k_select_local / k_merge), for CPU tests of the N > 1 exchange.
namespace {
struct HostKey {
  KeyGeom kg;
  unsigned long long key(int32_t S, uint8_t l, uint32_t gid) const {
    const unsigned long long mul = lvl_exact(l) ? kg.Ld : lvl_mul(l, kg.L, kg.L3, kg.growth);
    return (((unsigned long long)(uint32_t)S * mul) << kg.kbits) | gid;
  }
};
}  // namespace

aknn_status aknn_shard_summary_host(const int32_t *S, const uint8_t *lvl, int64_t n_local,
                                    int64_t offset, int64_t n_global, int32_t d, int32_t k,
                                    int32_t h, const double *alpha, void *recs_out) {
  if (!S || !lvl || !alpha || !recs_out) return fail(AKNN_EINVAL, "NULL argument");
  if (k < 1 || h < 0 || (int64_t)k + h >= n_local || d < 1)
    return fail(AKNN_EINVAL, "need k >= 1, h >= 0, k + h < n_local, d >= 1");
  HostKey hk;
  TRY(key_geom(n_local, n_global, d, &hk.kg));
  const int kh = k + h;
  std::vector<std::pair<unsigned long long, int64_t>> v((size_t)n_local);
  for (int64_t i = 0; i < n_local; ++i) v[i] = {hk.key(S[i], lvl[i], (uint32_t)(i + offset)), i};
  std::nth_element(v.begin(), v.begin() + (kh - 1), v.end());
  const unsigned long long th = v[kh - 1].first;
  ShardRec *out = static_cast<ShardRec *>(recs_out);
  int p = 0;
  int64_t best = -1;
  double bl = 0.0;
  for (int64_t i = 0; i < n_local; ++i) {
    const unsigned long long kk = hk.key(S[i], lvl[i], (uint32_t)(i + offset));
    if (kk <= th) {
      ShardRec r{};
      r.key = kk;
      r.S = S[i];
      r.lvl = lvl[i];
      out[p++] = r;
    } else {
      const double L = lower_of(S[i], lvl[i], d, alpha, 1);
      if (best < 0 || L < bl) {  // ascending i: ties keep the smaller id
        best = i;
        bl = L;
      }
    }
  }
  std::sort(out, out + kh, [](const ShardRec &a, const ShardRec &b) { return a.key < b.key; });
  ShardRec r{};
  r.key = hk.key(S[best], lvl[best], (uint32_t)(best + offset));
  r.S = S[best];
  r.lvl = lvl[best];
  out[kh] = r;
  return AKNN_OK;
}

aknn_status aknn_shard_merge_host(const void *recs, int32_t world, int64_t n_global, int32_t d,
                                  int32_t k, int32_t h, const double *alpha, aknn_merge_result *res) {
  if (!recs || !alpha || !res || !res->sets) return fail(AKNN_EINVAL, "NULL argument");
  if (world < 1 || k < 1 || h < 0) return fail(AKNN_EINVAL, "need world >= 1, k >= 1, h >= 0");
  KeyGeom kg;
  TRY(key_geom(n_global, n_global, d, &kg));
  const int kh = k + h;
  const ShardRec *rc = static_cast<const ShardRec *>(recs);
  std::vector<const ShardRec *> top;
  for (int w = 0; w < world; ++w)
    for (int r = 0; r < kh; ++r) top.push_back(rc + (size_t)w * (kh + 1) + r);
  std::sort(top.begin(), top.end(), [](const ShardRec *a, const ShardRec *b) { return a->key < b->key; });
  const unsigned long long gmask = (1ull << kg.kbits) - 1ull;
  auto gid = [&](const ShardRec *r) { return (int64_t)(r->key & gmask); };
  // d1 = argmax U over ranks 1..k (Eq. 2), ties to the smaller id
  const ShardRec *b1 = nullptr;
  double A = 0.0;
  for (int t = 0; t < k; ++t) {
    const double U = upper_of(top[t]->S, top[t]->lvl, d, alpha, 1);
    if (!b1 || U > A || (U == A && gid(top[t]) < gid(b1))) { b1 = top[t]; A = U; }
  }
  // d2 = argmin L over ranks > k+h and every shard's remainder arm (Eq. 3)
  std::vector<const ShardRec *> far(top.begin() + kh, top.end());
  for (int w = 0; w < world; ++w) far.push_back(rc + (size_t)w * (kh + 1) + kh);
  const ShardRec *b2 = nullptr;
  double B = 0.0;
  for (const ShardRec *r : far) {
    const double L = lower_of(r->S, r->lvl, d, alpha, 1);
    if (!b2 || L < B || (L == B && gid(r) < gid(b2))) { b2 = r; B = L; }
  }
  for (int t = 0; t < kh; ++t) {
    res->sets[t] = (int32_t)gid(top[t]);
    if (res->dhat) res->dhat[t] = dhat_of(top[t]->S, top[t]->lvl, d, 1);
  }
  res->thr_k = top[k - 1]->key;
  res->thr_kh = top[kh - 1]->key;
  res->A = A;
  res->B = B;
  res->d1 = gid(b1);
  res->d2 = gid(b2);
  res->alpha_d2 = alpha_of(b2->lvl, alpha, 1);
  res->stop = A <= B;  // Eq. (5)
  return AKNN_OK;
}

aknn_status aknn_get_stats(const aknn_index *ix, aknn_stats *out) {
  if (!ix || !out) return fail(AKNN_EINVAL, "NULL argument");
  TRY(finish_pending(const_cast<aknn_index *>(ix)));
  *out = ix->stats;
  return AKNN_OK;
}

aknn_status aknn_exact_async(const aknn_index *cix, const uint8_t *queries_dev, int32_t q, int32_t k,
                             int32_t *idx_dev, int32_t *dist2_dev, void *cuda_stream) {
  aknn_index *ix = const_cast<aknn_index *>(cix);
  if (!ix || !idx_dev || !dist2_dev) return fail(AKNN_EINVAL, "NULL argument");
  if (q < 0 || k < 1 || k > ix->n_local || k > 1024)
    return fail(AKNN_EINVAL, "need q >= 0 and 1 <= k <= min(n_local, 1024) (k=%d)", k);
  if (q == 0) return AKNN_OK;
  if (!queries_dev) return fail(AKNN_EINVAL, "queries is NULL");
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int64_t n = ix->n_local, npad = round_up(n, 16);
  ExactGeom e{};
  e.ibits = std::max(1, bit_length((unsigned long long)(n - 1)));
  e.nbits = bit_length(65025ull * (unsigned long long)ix->d) + e.ibits;
  if (e.nbits > 63) return fail(AKNN_EINVAL, "exact key needs %d bits", e.nbits);
  TRY(ensure_row_norms(ix, st));
  e.X = ix->X.as<uint8_t>();
  e.pitch = ix->pitch;
  e.n = (int)n;
  e.d = ix->d;
  e.k = k;
  e.id_offset = (uint32_t)ix->offset;
  e.npad = npad;
  const bool fused = k <= exact_fused_max_k();
  // fused: queries staged in the pitch layout + their norms + the per-CTA candidate
  // buffers; otherwise chunks of queries whose [qc][npad] int32 distance matrix is
  // bounded by 2 GiB
  const int64_t qc = fused ? q : std::max<int64_t>(1, std::min<int64_t>(q, (int64_t)(2ll << 30) / (npad * 4)));
  const size_t szD = fused ? exact_fused_ws_bytes(ix->num_sms, k) : (size_t)qc * npad * 4,
               szQ = (size_t)qc * ix->pitch, szN = (size_t)qc * 4;
  TRY(ix->exact_ws.ensure(round_up(szD, 256) + round_up(szQ, 256) + szN));
  for (int64_t r0 = 0; r0 < q; r0 += qc) {
    const int qn = (int)std::min<int64_t>(qc, q - r0);
    uint8_t *qpad = ix->exact_ws.as<uint8_t>(round_up(szD, 256));
    int32_t *nq = ix->exact_ws.as<int32_t>(round_up(szD, 256) + round_up(szQ, 256));
    CU(cudaMemsetAsync(qpad, 0, szQ, st));
    CU(cudaMemcpy2DAsync(qpad, ix->pitch, queries_dev + r0 * ix->d, ix->d, ix->d, qn,
                         cudaMemcpyDeviceToDevice, st));
    e.Q = qpad;
    e.q = qn;
    e.idx = idx_dev + r0 * k;
    e.dist2 = dist2_dev + r0 * k;
    CU(launch_row_norms(qpad, ix->pitch, qn, nq, st));
    if (fused) {
      CU(launch_exact_fused(e, nq, ix->nx.as<int32_t>(), ix->exact_ws.p, ix->num_sms, st));
    } else {
      e.D = ix->exact_ws.as<int32_t>();
      CU(launch_exact_mma(e, nq, ix->nx.as<int32_t>(), st));
      CU(launch_exact_topk(e, st));
    }
  }
  return AKNN_OK;
}

aknn_status aknn_exact(const aknn_index *cix, const uint8_t *queries, int32_t q, int32_t k, int32_t *idx,
                       int32_t *dist2) {
  aknn_index *ix = const_cast<aknn_index *>(cix);
  if (!ix || !queries || !idx || !dist2) return fail(AKNN_EINVAL, "NULL argument");
  if (q == 0) return AKNN_OK;
  const size_t szQ = (size_t)q * ix->d, szO = (size_t)q * k * 4;
  TRY(ix->outs.ensure(round_up(szQ, 256) + 2 * round_up(szO, 256)));
  uint8_t *dq = ix->outs.as<uint8_t>();
  int32_t *di = ix->outs.as<int32_t>(round_up(szQ, 256));
  int32_t *dd = ix->outs.as<int32_t>(round_up(szQ, 256) + round_up(szO, 256));
  cudaStream_t st = ix->stream;
  CU(cudaMemcpyAsync(dq, queries, szQ, cudaMemcpyHostToDevice, st));
  TRY(aknn_exact_async(ix, dq, q, k, di, dd, st));
  CU(cudaMemcpyAsync(idx, di, szO, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(dist2, dd, szO, cudaMemcpyDeviceToHost, st));
  CU(sync_spin(st));
  return AKNN_OK;
}

aknn_status aknn_set_timeout(aknn_index *ix, double timeout_ms) {
  if (!ix) return fail(AKNN_EINVAL, "NULL argument");
  if (!(timeout_ms >= 0.0)) return fail(AKNN_EINVAL, "timeout_ms must be >= 0 (0 = no deadline)");
  ix->nccl_timeout_ms = timeout_ms;
  return AKNN_OK;
}

int64_t aknn_index_n_local(const aknn_index *ix) { return ix ? ix->n_local : -1; }
int64_t aknn_index_n_global(const aknn_index *ix) { return ix ? ix->n_global : -1; }
int32_t aknn_index_dim(const aknn_index *ix) { return ix ? ix->d : -1; }

void aknn_free(aknn_index *ix) {
  if (!ix) return;
  finish_pending(ix);  // its copies target ix->host
  if (ix->pending.ev) cudaEventDestroy(ix->pending.ev);
  if (ix->nx_ev) cudaEventDestroy(ix->nx_ev);
#ifdef AKNN_WITH_NCCL
  if (ix->comm) ncclCommDestroy(ix->comm);  // (an aborted communicator is already gone)
#endif
  if (ix->stream) cudaStreamSynchronize(ix->stream);
  if (ix->loop_exec) cudaGraphExecDestroy(ix->loop_exec);
  if (ix->cap_stream) cudaStreamDestroy(ix->cap_stream);
  if (ix->stream) cudaStreamDestroy(ix->stream);
  delete ix;
}

const char *aknn_strerror(aknn_status s) {
  switch (s) {
    case AKNN_OK: return "AKNN_OK: success";
    case AKNN_EINVAL: return "AKNN_EINVAL: invalid argument";
    case AKNN_ENOMEM: return "AKNN_ENOMEM: out of memory";
    case AKNN_ECUDA: return "AKNN_ECUDA: CUDA error";
    case AKNN_ENCCL: return "AKNN_ENCCL: NCCL error";
    case AKNN_EMAXROUNDS: return "AKNN_EMAXROUNDS: max_rounds reached before Eq. (5) held";
  }
  return "unknown aknn_status";
}

const char *aknn_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
