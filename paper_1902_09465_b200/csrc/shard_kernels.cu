// shard_kernels.cu -- the point-sharded round.
//
// The point set is split into `world` shards with global ids.  A round of the
// batched rule needs three global facts per query: the composite keys of ranks
// k and k+h (the C/M/F split) and the bounds A, B with d2 and
// alpha_{d2} (Eq. 2-3).  Every global top-(k+h) arm lies in the top
// (k+h) of its own shard, and every other arm is in F, so per shard it suffices
// to send
//   * its local top-(k+h) arms (key, S, level), and
//   * the arm with the smallest L = d_hat - alpha among the rest (ties: smaller id).
// After an allgather every shard merges the same records the same way:
//   k_select_local  local radix select of rank k+h + the summary records
//   k_merge         sort the world*(k+h) keys, thresholds, A/d1 over the top k,
//                   B/d2 over ranks > k+h plus the rest records, Eq. (5), and the
//                   candidate set of the query
// The filter / compaction / advance kernels then run locally, unchanged.
#include "internal.cuh"
#include "launch.h"
#include "round_common.cuh"
#include "select.cuh"

namespace aknn {

// ---------------------------------------------------------------------------
// Local summary of one query (one CTA per undecided query).
__global__ void __launch_bounds__(SEL_NT) k_select_local(Geom g, int nbits) {
  __shared__ SelSmem sm;
  __shared__ RecBest wsm[SEL_NT / 32];
  __shared__ unsigned cnt;
  const int qi = blockIdx.x;
  if (g.qs[qi].done || !g.qs[qi].fallback) return;  // the pivot select decided it
  const int tid = threadIdx.x;
  const unsigned kh = (unsigned)(g.k + g.h);
  ArmKeys keys{&g, qi};
  unsigned long long th, th2;
  select2(sm, keys, g.n, nbits, kh, kh, &th, &th2);
  ShardRec *out = g.send + (size_t)qi * (kh + 1);
  if (tid == 0) cnt = 0;
  __syncthreads();
  RecBest bl{1.0e300, 0xffffffffu, 0, 0};
  for (int i0 = tid * 4; i0 < g.n; i0 += SEL_NT * 4) {
    const Arm4 a = load_arm4(g, qi, i0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = i0 + e;
      if (i >= g.n) break;
      const unsigned long long key = arm_key(a.S[e], a.l(e), (uint32_t)i, g);
      if (key <= th) {
        const unsigned p = atomicAdd(&cnt, 1u);
        ShardRec r;
        r.key = key;
        r.S = a.S[e];
        r.lvl = a.l(e);
        r.pad[0] = r.pad[1] = r.pad[2] = 0;
        out[p] = r;
      } else {
        const RecBest c{lower_of(a.S[e], a.l(e), g.d, g.alpha, g.growth), (uint32_t)i + g.id_offset, a.S[e],
                        a.l(e)};
        if (better_min(c, bl)) bl = c;
      }
    }
  }
  const RecBest r = block_best<false>(bl, wsm);
  if (tid == 0) {
    ShardRec rr;
    rr.S = r.S;
    rr.lvl = r.lvl;
    rr.key = arm_key(r.S, r.lvl, r.gid - g.id_offset, g);
    rr.pad[0] = rr.pad[1] = rr.pad[2] = 0;
    out[kh] = rr;
  }
}

// ---------------------------------------------------------------------------
// Global merge (one CTA per undecided query; identical on every shard).
constexpr int MRG_NT = 256;

size_t merge_smem_bytes(int world, int kh) {
  unsigned m = (unsigned)world * (unsigned)kh, P = 2;
  while (P < m) P <<= 1;
  return (size_t)P * (sizeof(unsigned long long) + sizeof(uint32_t));
}

__device__ void bitonic_sort_kv(unsigned long long *key, uint32_t *val, unsigned P) {
  for (unsigned k = 2; k <= P; k <<= 1)
    for (unsigned j = k >> 1; j > 0; j >>= 1) {
      for (unsigned idx = threadIdx.x; idx < P; idx += blockDim.x) {
        const unsigned ixj = idx ^ j;
        if (ixj > idx) {
          const unsigned long long a = key[idx], b = key[ixj];
          const bool up = (idx & k) == 0;
          if ((a > b) == up) {
            key[idx] = b;
            key[ixj] = a;
            const uint32_t t = val[idx];
            val[idx] = val[ixj];
            val[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(MRG_NT) k_merge(Geom g, OutPtrs o) {
  extern __shared__ unsigned char msm[];
  __shared__ RecBest wsm[MRG_NT / 32];
  const int qi = blockIdx.x;
  QState *st = g.qs + qi;
  if (st->done) return;
  const unsigned kh = (unsigned)(g.k + g.h), W = (unsigned)g.world, m = W * kh;
  unsigned P = 2;
  while (P < m) P <<= 1;
  unsigned long long *key = reinterpret_cast<unsigned long long *>(msm);
  uint32_t *pos = reinterpret_cast<uint32_t *>(key + P);
  const ShardRec *rq = g.recv;
  auto rec = [&](unsigned w, unsigned r) -> const ShardRec & {
    return rq[(size_t)w * g.recv_stride + (size_t)qi * (kh + 1) + r];
  };
  for (unsigned t = threadIdx.x; t < P; t += MRG_NT) {
    if (t < m) {
      key[t] = rec(t / kh, t % kh).key;
      pos[t] = t;
    } else {
      key[t] = KEY_INVALID;
      pos[t] = 0;
    }
  }
  __syncthreads();
  bitonic_sort_kv(key, pos, P);
  const uint32_t gmask = (uint32_t)((1ull << g.kbits) - 1ull);
  // d1 = argmax U over ranks 1..k (Eq. 2); d2 = argmin L over ranks > k+h (Eq. 3)
  RecBest bu{-1.0e300, 0xffffffffu, 0, 0}, bl{1.0e300, 0xffffffffu, 0, 0};
  for (unsigned t = threadIdx.x; t < m + W; t += MRG_NT) {
    if (t < (unsigned)g.k) {
      const ShardRec &r = rec(pos[t] / kh, pos[t] % kh);
      const RecBest c{upper_of(r.S, r.lvl, g.d, g.alpha, g.growth), (uint32_t)(key[t] & gmask), r.S, r.lvl};
      if (better_max(c, bu)) bu = c;
    } else if (t >= kh) {
      const ShardRec &r = t < m ? rec(pos[t] / kh, pos[t] % kh) : rec(t - m, kh);
      const unsigned long long kk = t < m ? key[t] : r.key;
      const RecBest c{lower_of(r.S, r.lvl, g.d, g.alpha, g.growth), (uint32_t)(kk & gmask), r.S, r.lvl};
      if (better_min(c, bl)) bl = c;
    }
  }
  bu = block_best<true>(bu, wsm);
  bl = block_best<false>(bl, wsm);
  // the candidate set in rank order and its estimates, every round
  if (o.sets) {
    for (unsigned t = threadIdx.x; t < kh; t += MRG_NT) {
      const size_t oo = (size_t)(o.row0 + qi) * kh + t;
      o.sets[oo] = (int32_t)(key[t] & gmask);
      if (o.dhat) {
        const ShardRec &r = rec(pos[t] / kh, pos[t] % kh);
        o.dhat[oo] = dhat_of(r.S, r.lvl, g.d, g.growth);
      }
    }
  }
  if (threadIdx.x == 0) {
    st->thr_k = key[g.k - 1];
    st->thr_kh = key[kh - 1];
    st->A = bu.v;
    st->B = bl.v;
    st->d1 = (int)bu.gid;
    st->d2 = (int)bl.gid;
    st->a_d2 = alpha_of(bl.lvl, g.alpha, g.growth);
    st->rounds += 1;
    const int stop = bu.v <= bl.v;  // Eq. (5), "<=" as written
    st->done = stop;
    if (!stop) atomicAdd(&g.ctl->n_active, 1u);
  }
}

// Per-shard counters (draws, evals = draws + the exact fallbacks' charge), rounds, and the
// optional per-pair counts/sums at this shard's columns.
__global__ void k_counters_sharded(Geom g, OutPtrs o) {
  const int qi = blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= g.q) return;
  const QState st = g.qs[qi];
  const size_t row = (size_t)(o.row0 + qi);
  const long long ev = st.draws + st.exact_evals;
  if (o.accumulate) {
    if (o.draws) atomicAdd(reinterpret_cast<unsigned long long *>(o.draws + row), (unsigned long long)st.draws);
    if (o.evals) atomicAdd(reinterpret_cast<unsigned long long *>(o.evals + row), (unsigned long long)ev);
  } else {
    if (o.draws) o.draws[row] = st.draws;
    if (o.evals) o.evals[row] = ev;
  }
  if (o.rounds) o.rounds[row] = st.rounds;
}

__global__ void k_counts_sharded(Geom g, OutPtrs o) {
  const int qi = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  const size_t src = (size_t)qi * g.npad + i;
  const size_t dst = (size_t)(o.row0 + qi) * o.ncols + o.col0 + i;
  const uint8_t l = g.lvl[src];
  if (o.counts) o.counts[dst] = (int32_t)count_of(l, g.d, g.growth);
  if (o.sums) o.sums[dst] = (int64_t)(uint32_t)g.S[src];
}

static inline unsigned cdiv(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

cudaError_t launch_select_local(const Geom &g, int nbits, cudaStream_t s) {
  const cudaError_t e = launch_select_local_pivot(g, s);
  if (e != cudaSuccess) return e;
  k_select_local<<<g.q, SEL_NT, 0, s>>>(g, nbits);
  return cudaGetLastError();
}

cudaError_t launch_merge(const Geom &g, const OutPtrs &o, cudaStream_t s) {
  const size_t smem = merge_smem_bytes(g.world, g.k + g.h);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_merge<<<g.q, MRG_NT, smem, s>>>(g, o);
  return cudaGetLastError();
}

cudaError_t launch_output_sharded(const Geom &g, const OutPtrs &o, cudaStream_t s) {
  const cudaError_t te = launch_tally(g, s);
  if (te != cudaSuccess) return te;
  k_counters_sharded<<<cdiv(g.q, 128), 128, 0, s>>>(g, o);
  if (o.counts || o.sums) k_counts_sharded<<<dim3(cdiv(g.n, 256), g.q), 256, 0, s>>>(g, o);
  return cudaGetLastError();
}

}  // namespace aknn
