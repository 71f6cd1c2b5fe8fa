/*
 * aknn_oracle.c -- the CPU ORACLE for the adaptive k-NN hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1902_09465_b200/) never links, imports or calls
 * anything here, and this file includes nothing from the product path.
 *
 * Plain, slow, single-threaded C99, fp64, compiled -O2 -ffp-contract=off.
 * Every function cites the passage of /root/reference/PAPER.md ("P:<line>")
 * or SPEC.md ("S:<line>") it follows; the readings of ambiguous passages are
 * the ones listed in DESIGN.md §3.
 *
 * Parity status:
 *   orc_philox4x32_10     pinned: cuRAND curand_Philox4x32_10 (library routine)
 *   orc_lemire            pinned: exhaustive preimage counts over all 2^32 words
 *   orc_alpha_*           pinned: SPEC worked values S:78; monotonicity
 *   orc_bruteforce        pinned: numpy / torch._int_mm brute force
 *   orc_round_step        pinned: hand-built states (S:139-171 examples), brute sort
 *   orc_query_br          pinned: planted set, d=1, all-exact, Theorem-1 rate,
 *                         closed-form draw/eval accounting, A1 stream prefix;
 *                         growth schedule: hand-written count sequences, growth 1
 *                         = BR, per-arm sums = prefixes of the arm's own stream
 *   orc_next_count        pinned: hand-written sequences of G_1, G_2, G_4
 *   orc_wor_*             pinned: exhaustive bijection of [0, d) (many d, keys),
 *                         uniformity of pi(t) over keys, A1 full-permutation
 *                         sums equal brute force, evals = sum of counts
 *   per-arm counts, round numbers and the order of the returned set:
 *                         parity unpinned beyond the invariants above.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-2)
#define ORC_EMAXROUNDS (-5)
#define ORC_EINTERNAL (-9)

/* ------------------------------------------------------------------------ */
/* a1: the coordinate draw.  P:120-125 (§4): "sampling indices j_1..j_T      */
/* uniformly at random from all indices {1..m}".  The stream is Philox4x32-10 */
/* (Salmon et al., SC'11) keyed by the 64-bit seed, counter (u>>2, i, qi, b); */
/* SURVEY.md §8(c) "Draw(i,t)".                                              */
/* ------------------------------------------------------------------------ */

static void philox_round(uint32_t c[4], const uint32_t k[2]) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  uint32_t r[4];
  r[0] = hi1 ^ c[1] ^ k[0];
  r[1] = lo1;
  r[2] = hi0 ^ c[3] ^ k[1];
  r[3] = lo0;
  memcpy(c, r, sizeof r);
}

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    philox_round(c, k);
  }
  memcpy(out, c, sizeof c);
}

/* Multiply-high map of a 32-bit word onto [0, d) (reading R5). */
uint32_t orc_lemire(uint32_t w, uint32_t d) {
  return (uint32_t)(((uint64_t)w * (uint64_t)d) >> 32);
}

/* Exhaustive preimage histogram of orc_lemire over all 2^32 words (pin). */
void orc_lemire_histogram(uint32_t d, uint64_t *hist) {
  memset(hist, 0, sizeof(uint64_t) * d);
  uint32_t w = 0;
  do {
    hist[orc_lemire(w, d)]++;
  } while (++w != 0);
}

/* Level b and in-level ordinal u of the t-th sample (t = 0,1,2,...):
 * b = 0 for t = 0, else 1 + floor(log2 t); u = t - 2^(b-1).               */
static void level_of(int64_t t, uint32_t *b, uint32_t *u) {
  if (t == 0) {
    *b = 0;
    *u = 0;
    return;
  }
  uint32_t lg = 0;
  while (((int64_t)1 << (lg + 1)) <= t) ++lg;
  *b = lg + 1;
  *u = (uint32_t)(t - ((int64_t)1 << lg));
}

/* The coordinate j of the t-th sample of arm (qi, i).                      */
uint32_t orc_draw_index(uint64_t seed, uint32_t qi, uint32_t i, int64_t t, uint32_t d) {
  uint32_t b, u;
  level_of(t, &b, &u);
  const uint32_t ctr[4] = {u >> 2, i, qi, b};
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  uint32_t w[4];
  orc_philox4x32_10(ctr, key, w);
  return orc_lemire(w[u & 3u], d);
}

/* ------------------------------------------------------------------------ */
/* Sampling WITHOUT replacement (footnote 1 to P:120;  */
/* DESIGN.md reading R23).  The t-th sample of arm (qi, i), t = 0 .. d-1, is  */
/* coordinate pi(t) of a permutation pi of [0, d) keyed per arm:              */
/*   w = the Philox4x32-10 block of counter (0, i, qi, 0x80000000) under the  */
/*       seed (a level word no draw uses);                                    */
/*   E = a 6-round mixed-radix Feistel network on Z_a x Z_b, a = ceil(sqrt d),*/
/*       b = ceil(d / a) (so d <= a b < d + a): x = L b + R with L in Z_a,    */
/*       R in Z_b; round r maps (L, R) in Z_m x Z_m' to                       */
/*       (R, (L + F_r(R, m)) mod m) in Z_m' x Z_m, m = a for even r, b for    */
/*       odd r (each round is invertible, six rounds return to Z_a x Z_b);    */
/*       F_r(R, m) = floor(g((R xor k_r) * 0x9E3779B1 mod 2^32) * m / 2^32),  */
/*       g(h) = (h xor (h >> 16)) * 0x85EBCA6B mod 2^32,                      */
/*       k_r = w[r mod 4] + r * 0x9E3779B9 mod 2^32;                          */
/*   rho(t) = E^m(t) for the smallest m >= 1 with E^m(t) < d (cycle walking;  */
/*       needed only when a b > d, with probability < 1/b per step);          */
/*   pi(t) = (rho(t) + rot) mod d, rot = floor((w0 xor w2) * d / 2^32) (a    */
/*       uniform rotation: the position of every t is uniform over keys).     */
/* (An earlier power-of-two domain walked with probability up to 3/4 per      */
/* step; on the GPU the walk diverges inside a warp, so the domain is now the */
/* tight a x b one.)                                                          */
/* ------------------------------------------------------------------------ */
/* a = ceil(sqrt(d)), b = ceil(d / a).                                        */
void orc_wor_radix(uint32_t d, uint32_t *a, uint32_t *b) {
  uint32_t r = 1;
  while (r * r < d) ++r;
  *a = r;
  *b = (d + r - 1) / r;
}

void orc_wor_keys(uint64_t seed, uint32_t qi, uint32_t i, uint32_t keys[4]) {
  const uint32_t ctr[4] = {0u, i, qi, 0x80000000u};
  const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
  orc_philox4x32_10(ctr, key, keys);
}

uint32_t orc_feistel(const uint32_t keys[4], uint32_t a, uint32_t b, uint32_t x) {
  uint32_t L = x / b, R = x % b, m = a, m2 = b;
  for (uint32_t r = 0; r < 6; ++r) {
    const uint32_t kr = keys[r & 3u] + r * 0x9E3779B9u;
    uint32_t h = (R ^ kr) * 0x9E3779B1u;
    h = (h ^ (h >> 16)) * 0x85EBCA6Bu;
    const uint32_t f = (uint32_t)(((uint64_t)h * m) >> 32);
    const uint32_t nr = (L + f) % m;
    L = R;
    R = nr;
    const uint32_t t = m;  /* the halves swap roles */
    m = m2;
    m2 = t;
  }
  return L * b + R;
}

uint32_t orc_wor_index(const uint32_t keys[4], uint32_t d, uint32_t t) {
  uint32_t a, b;
  orc_wor_radix(d, &a, &b);
  uint32_t x = t;
  do {
    x = orc_feistel(keys, a, b, x);
  } while (x >= d);
  const uint32_t rot = orc_lemire(keys[0] ^ keys[2], d);
  return x + rot >= d ? x + rot - d : x + rot;
}

/* pi(0..d-1) of arm (qi, i), for the pins (a bijection of [0, d)).          */
void orc_wor_perm(uint64_t seed, uint32_t qi, uint32_t i, uint32_t d, uint32_t *out) {
  uint32_t keys[4];
  orc_wor_keys(seed, qi, i, keys);
  for (uint32_t t = 0; t < d; ++t) out[t] = orc_wor_index(keys, d, t);
}

/* One sampled squared coordinate difference |[x_i]_j - [x]_j|^2,
 * kept as the exact integer (a-b)^2; the [0,1] sample is that / 65025
 * (reading R2).                                            */
static int64_t draw_sq(const uint8_t *xi, const uint8_t *x, uint64_t seed, uint32_t qi,
                       uint32_t i, int64_t t, uint32_t d, int wor) {
  uint32_t j;
  if (wor) {
    uint32_t keys[4];
    orc_wor_keys(seed, qi, i, keys);
    j = orc_wor_index(keys, d, (uint32_t)t);
  } else {
    j = orc_draw_index(seed, qi, i, t, d);
  }
  const int64_t diff = (int64_t)xi[j] - (int64_t)x[j];
  return diff * diff;
}

/* Exact sum_j (a_j - b_j)^2 (brute force P:98).                  */
static int64_t exact_sq(const uint8_t *xi, const uint8_t *x, int32_t d) {
  int64_t s = 0;
  for (int32_t j = 0; j < d; ++j) {
    const int64_t diff = (int64_t)xi[j] - (int64_t)x[j];
    s += diff * diff;
  }
  return s;
}

/* ------------------------------------------------------------------------ */
/* The confidence radius alpha(u).                                          */
/* ------------------------------------------------------------------------ */

/* Footnote 2: alpha(u) = sqrt(2 beta(u, delta/n) / u),
 * beta(u, d') = log(1/d') + 3 log log(1/d') + 1.5 log(1 + log u).
 * Table layout: alpha[u] for 1 <= u < d; alpha[0] = alpha[d] = 0 (an exact
 * arm has alpha = 0).  Requires delta/n < 1/e (R3).        */
int orc_alpha_theory(int64_t n, double delta, int32_t d, double *alpha) {
  if (n < 1 || d < 1 || !(delta > 0.0 && delta < 1.0)) return ORC_EINVAL;
  const double dp = delta / (double)n;
  const double l1 = log(1.0 / dp);
  if (!(l1 > 1.0)) return ORC_EINVAL; /* log log(1/d') must be defined and > 0 */
  const double ll = log(l1);
  alpha[0] = 0.0;
  for (int32_t u = 1; u < d; ++u) {
    const double beta = l1 + 3.0 * ll + 1.5 * log(1.0 + log((double)u));
    alpha[u] = sqrt(2.0 * beta / (double)u);
  }
  alpha[d] = 0.0;
  return ORC_OK;
}

/* §5: alpha(u) = sqrt(C_alpha log(1 + (1 + log u) n / delta) / u).  */
int orc_alpha_experimental(int64_t n, double delta, double c_alpha, int32_t d, double *alpha) {
  if (n < 1 || d < 1 || !(delta > 0.0 && delta < 1.0) || !(c_alpha > 0.0)) return ORC_EINVAL;
  alpha[0] = 0.0;
  for (int32_t u = 1; u < d; ++u) {
    const double inner = 1.0 + (1.0 + log((double)u)) * (double)n / delta;
    alpha[u] = sqrt(c_alpha * log(inner) / (double)u);
  }
  alpha[d] = 0.0;
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Brute force: all distances, then sort by (distance, index).        */
/* ------------------------------------------------------------------------ */

typedef struct {
  int64_t key;
  int32_t idx;
} ikey_t;

static int cmp_ikey(const void *a, const void *b) {
  const ikey_t *x = (const ikey_t *)a, *y = (const ikey_t *)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

int orc_bruteforce(const uint8_t *X, int64_t n, int32_t d, const uint8_t *Q, int32_t q,
                   int32_t k, int32_t *idx, int64_t *dist2) {
  if (n < 1 || d < 1 || q < 0 || k < 1 || k > n) return ORC_EINVAL;
  ikey_t *v = (ikey_t *)malloc(sizeof(ikey_t) * (size_t)n);
  if (!v) return ORC_ENOMEM;
  for (int32_t a = 0; a < q; ++a) {
    for (int64_t i = 0; i < n; ++i) {
      v[i].key = exact_sq(X + (size_t)i * d, Q + (size_t)a * d, d);
      v[i].idx = (int32_t)i;
    }
    qsort(v, (size_t)n, sizeof(ikey_t), cmp_ikey);
    for (int32_t r = 0; r < k; ++r) {
      idx[(size_t)a * k + r] = v[r].idx;
      if (dist2) dist2[(size_t)a * k + r] = v[r].key;
    }
  }
  free(v);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* R1-R5 of one round on a given state.                    */
/* ------------------------------------------------------------------------ */

typedef struct {
  double dh;
  int32_t idx;
} dkey_t;

static int cmp_dkey(const void *a, const void *b) {
  const dkey_t *x = (const dkey_t *)a, *y = (const dkey_t *)b;
  if (x->dh != y->dh) return x->dh < y->dh ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* R1: d_hat_i(T_i) = (1/T_i) sum of T_i samples, each (a-b)^2/65025
 * (P:121-124), as one pinned fp64 expression (reading R15).       */
static double dhat_of(int64_t S, int32_t T) {
  return (double)S / ((double)T * 65025.0);
}

/* alpha_i = alpha(T_i); 0 once the arm is exact.                    */
static double alpha_of(int32_t T, int32_t d, const double *alpha) {
  return T == d ? 0.0 : alpha[T];
}

/*
 * One evaluation of the round quantities on state (S, T):
 *   R1 estimates and bounds; R2 the permutation (.) with
 *   d_hat_(1) <= ... <= d_hat_(n), ties by smaller index;
 *   R3 d1 = argmax_{(1)..(k)} d_hat + alpha, d2 = argmin_{(k+1+h)..(n)}
 *   d_hat - alpha (Eq. 2-3; ties to the smaller index);
 *   R4 the termination test Eq. (5), "<=" as written;
 *   R5 (batched round rule, R6): the blocker set
 *   {C: U > B} u {F: L < A} u {M: alpha > alpha_d2} minus exact arms, the
 *   M term being Eq. (4) batched.
 * order[0..n) receives the permutation; active[] (nullable) the blockers.
 * Returns 1 if Eq. (5) holds, 0 if not, <0 on error.
 */
int orc_round_step(int64_t n, int32_t d, const int64_t *S, const int32_t *T, int32_t k,
                   int32_t h, const double *alpha, int32_t *order, int32_t *d1_out,
                   int32_t *d2_out, double *A_out, double *B_out, uint8_t *active) {
  if (k < 1 || h < 0 || (int64_t)k + h >= n) return ORC_EINVAL;
  dkey_t *v = (dkey_t *)malloc(sizeof(dkey_t) * (size_t)n);
  if (!v) return ORC_ENOMEM;
  for (int64_t i = 0; i < n; ++i) {
    v[i].dh = dhat_of(S[i], T[i]);
    v[i].idx = (int32_t)i;
  }
  qsort(v, (size_t)n, sizeof(dkey_t), cmp_dkey);
  for (int64_t r = 0; r < n; ++r) order[r] = v[r].idx;

  /* d1 over the close set (1)..(k) */
  int32_t d1 = -1;
  double A = 0.0;
  for (int32_t r = 0; r < k; ++r) {
    const int32_t i = v[r].idx;
    const double U = v[r].dh + alpha_of(T[i], d, alpha);
    if (d1 < 0 || U > A || (U == A && i < d1)) {
      d1 = i;
      A = U;
    }
  }
  /* d2 over the far set (k+1+h)..(n) */
  int32_t d2 = -1;
  double B = 0.0;
  for (int64_t r = (int64_t)k + h; r < n; ++r) {
    const int32_t i = v[r].idx;
    const double L = v[r].dh - alpha_of(T[i], d, alpha);
    if (d2 < 0 || L < B || (L == B && i < d2)) {
      d2 = i;
      B = L;
    }
  }
  const int stop = (A <= B);
  if (active) {
    const double a_d2 = alpha_of(T[d2], d, alpha);
    memset(active, 0, (size_t)n);
    for (int64_t r = 0; r < n; ++r) {
      const int32_t i = v[r].idx;
      if (T[i] == d) continue; /* exact arms never advance */
      const double a = alpha_of(T[i], d, alpha);
      const double U = v[r].dh + a, L = v[r].dh - a;
      int blk;
      if (r < k)
        blk = U > B;
      else if (r < (int64_t)k + h)
        blk = a > a_d2;
      else
        blk = L < A;
      active[i] = (uint8_t)blk;
    }
  }
  if (d1_out) *d1_out = d1;
  if (d2_out) *d2_out = d2;
  if (A_out) *A_out = A;
  if (B_out) *B_out = B;
  free(v);
  return stop;
}

/* ------------------------------------------------------------------------ */
/* Growth schedule of R6 (reading R25).      */
/* The paper increments T by one per selection; the batched rule  */
/* doubles it (reading R7).  A growth factor < 2 takes the next count from the */
/* grid G_m = { (m + r) 2^j / m : j >= 0, 0 <= r < m } of integers: m = 1 is   */
/* doubling (1, 2, 4, 8, ...), m = 2 the schedule 1, 2, 3, 4, 6, 8, 12, 16, ... */
/* (factors 3/2 and 4/3, sqrt 2 per level on average).  Every power of two is  */
/* in G_m, so each advance [T, next(T)) lies inside one sample level b of the  */
/* Draw stream.                                                               */
/* ------------------------------------------------------------------------ */

/* The smallest integer of G_m greater than T (T >= 1, m in {1, 2, 4}).        */
int64_t orc_next_count(int64_t T, int32_t m) {
  int64_t best = -1;
  for (int32_t j = 0; j < 62; ++j) {
    for (int32_t r = 0; r < m; ++r) {
      const int64_t v = (int64_t)(m + r) << j;
      if (v % m != 0) continue;
      const int64_t c = v / m;
      if (c > T && (best < 0 || c < best)) best = c;
    }
    if (((int64_t)1 << j) > 2 * T) break;
  }
  return best;
}

/* ------------------------------------------------------------------------ */
/* The batched round rule BR, one query at a time.         */
/* ------------------------------------------------------------------------ */

/*
 * X uint8 [n][d] row-major; Qrows uint8 [q][d]; qids[a] is query a's index qi
 * in the RNG counter; id_offset is added to every point id in the counter
 * and in the returned sets (sharding).  alpha: fp64 [d+1].
 * Outputs (all per query a, row-major; nullable except sets):
 *   sets [q][k+h] point ids, rank order;  dhat [q][k+h];
 *   counts [q][n] T_i;  sums [q][n] S_i;  evals/draws [q];  rounds [q].
 * Returns ORC_OK, ORC_EINVAL, ORC_ENOMEM or ORC_EMAXROUNDS.
 */
int orc_query_br(const uint8_t *X, int64_t n, int32_t d, const uint8_t *Qrows, int32_t q,
                 const int32_t *qids, int64_t id_offset, int32_t k, int32_t h, uint64_t seed,
                 const double *alpha, int32_t max_rounds, int32_t wor, int32_t lead, int32_t growth,
                 int32_t *sets, double *dhat, int32_t *counts, int64_t *sums, int64_t *evals,
                 int64_t *draws, int32_t *rounds) {
  if (n < 2 || d < 1 || q < 0 || k < 1 || h < 0 || (int64_t)k + h >= n || !alpha || !sets ||
      !(growth == 0 || growth == 1 || growth == 2 || growth == 4))
    return ORC_EINVAL;
  int64_t *S = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int32_t *T = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  uint8_t *act = (uint8_t *)malloc((size_t)n);
  if (!S || !T || !order || !act) {
    free(S); free(T); free(order); free(act);
    return ORC_ENOMEM;
  }
  int status = ORC_OK, hit_max = 0;
  for (int32_t a = 0; a < q; ++a) {
    const uint8_t *x = Qrows + (size_t)a * d;
    const uint32_t qi = (uint32_t)qids[a];
    int64_t ndraws = 0, ncharge = 0;
    /* R0, Algorithm 1 initialisation: one sample per arm, T=1. */
    for (int64_t i = 0; i < n; ++i) {
      S[i] = draw_sq(X + (size_t)i * d, x, seed, qi, (uint32_t)(i + id_offset), 0, (uint32_t)d, wor);
      T[i] = 1;
      ndraws += 1;
      if (d == 1) T[i] = d; /* the single coordinate is the exact distance */
    }
    int32_t r = 0;
    int stop = 0;
    for (;;) {
      ++r;
      int32_t d1, d2;
      double A, B;
      stop = orc_round_step(n, d, S, T, k, h, alpha, order, &d1, &d2, &A, &B, act);
      if (stop < 0) { status = stop; break; }
      if (stop) break;                                   /* R4, Eq. (5) */
      if (max_rounds > 0 && r >= max_rounds) { status = ORC_EMAXROUNDS; break; }
      int64_t nact = 0;
      /* R6: every blocker advances once; with a close-side lead L > 1 (reading
       * R24) the blockers ranked in C or M this round
       * advance L - 1 more times (each the same P:176 / doubling step).     */
      for (int64_t r = 0; r < (int64_t)k + h; ++r) act[order[r]] |= (uint8_t)(act[order[r]] ? 2 : 0);
      for (int32_t pass = 0; pass < (lead > 1 ? lead : 1); ++pass) {
        for (int64_t i = 0; i < n; ++i) {
          if (!act[i] || (pass > 0 && !(act[i] & 2)) || T[i] == d) continue;
          if (pass == 0) ++nact;
          const uint8_t *xi = X + (size_t)i * d;
          /* the next count: 2T (reading R7), or the next grid value of reading R25 */
          const int64_t Tn = growth > 1 ? orc_next_count(T[i], growth) : 2 * (int64_t)T[i];
          if (Tn >= d) {
            /* P:176 exact fallback, taken before the draws that would reach m;
             * charged d evaluations, or without replacement the d - T
             * coordinates the permutation had not drawn yet (reading R23)   */
            S[i] = exact_sq(xi, x, d);
            ncharge += wor ? (int64_t)d - T[i] : (int64_t)d;
            T[i] = d;
          } else {
            for (int64_t t = T[i]; t < Tn; ++t)
              S[i] += draw_sq(xi, x, seed, qi, (uint32_t)(i + id_offset), t, (uint32_t)d, wor);
            ndraws += Tn - T[i];
            T[i] = (int32_t)Tn;
          }
        }
      }
      if (nact == 0) { status = ORC_EINTERNAL; break; } /* impossible, §8(c) */
    }
    const int32_t kh = k + h;
    for (int32_t rr = 0; rr < kh; ++rr) {                /* P:186-187 return */
      const int32_t i = order[rr];
      sets[(size_t)a * kh + rr] = (int32_t)(i + id_offset);
      if (dhat) dhat[(size_t)a * kh + rr] = dhat_of(S[i], T[i]);
    }
    if (counts) memcpy(counts + (size_t)a * n, T, sizeof(int32_t) * (size_t)n);
    if (sums) memcpy(sums + (size_t)a * n, S, sizeof(int64_t) * (size_t)n);
    if (draws) draws[a] = ndraws;
    if (evals) evals[a] = ndraws + ncharge;
    if (rounds) rounds[a] = r;
    if (status == ORC_EMAXROUNDS) {  /* every query still runs to its own cap */
      hit_max = 1;
      status = ORC_OK;
    }
    if (status != ORC_OK) break;
  }
  free(S); free(T); free(order); free(act);
  return status != ORC_OK ? status : (hit_max ? ORC_EMAXROUNDS : ORC_OK);
}

/* ------------------------------------------------------------------------ */
/* Literal Algorithm 1, mode A1: per iteration, sample {d1, b2}. */
/* Slow (one sort per iteration): tiny inputs only.                          */
/* ------------------------------------------------------------------------ */
int orc_query_a1(const uint8_t *X, int64_t n, int32_t d, const uint8_t *x, int32_t qi,
                 int32_t k, int32_t h, uint64_t seed, const double *alpha, int64_t max_iters,
                 int32_t wor, int32_t *set, int32_t *counts, int64_t *sums, int64_t *evals,
                 int64_t *draws, int64_t *iters) {
  if (n < 2 || d < 1 || k < 1 || h < 0 || (int64_t)k + h >= n || !alpha || !set)
    return ORC_EINVAL;
  int64_t *S = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  int32_t *T = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  if (!S || !T || !order) {
    free(S); free(T); free(order);
    return ORC_ENOMEM;
  }
  int64_t ndraws = 0, nexact = 0, it = 0;
  int status = ORC_OK;
  for (int64_t i = 0; i < n; ++i) {
    S[i] = draw_sq(X + (size_t)i * d, x, seed, (uint32_t)qi, (uint32_t)i, 0, (uint32_t)d, wor);
    T[i] = 1;
    ndraws += 1;
    if (d == 1) T[i] = d;
  }
  for (;;) {
    ++it;
    int32_t d1, d2;
    double A, B;
    const int stop = orc_round_step(n, d, S, T, k, h, alpha, order, &d1, &d2, &A, &B, NULL);
    if (stop < 0) { status = stop; break; }
    if (stop) break;
    if (max_iters > 0 && it >= max_iters) { status = ORC_EMAXROUNDS; break; }
    /* Eq. (4): b2 = argmax_{ {d2} u (k+1)..(k+h) } alpha_i; ties to d2, then
     * to the smaller index.                                        */
    int32_t b2 = d2;
    double ab = alpha_of(T[d2], d, alpha);
    for (int32_t r = k; r < k + h; ++r) {
      const int32_t i = order[r];
      const double a = alpha_of(T[i], d, alpha);
      if (a > ab || (a == ab && b2 != d2 && i < b2)) {
        b2 = i;
        ab = a;
      }
    }
    const int32_t sel[2] = {d1, b2};
    for (int s = 0; s < 2; ++s) {         /* "For l in {d1, b2}" */
      const int32_t l = sel[s];
      if (T[l] >= d) continue;
      S[l] += draw_sq(X + (size_t)l * d, x, seed, (uint32_t)qi, (uint32_t)l, T[l], (uint32_t)d, wor);
      T[l] += 1;
      ndraws += 1;
      if (T[l] == d) {                     /* "If T_l = m ... exactly" */
        const int64_t ex = exact_sq(X + (size_t)l * d, x, d);
        /* without replacement the d samples ARE every coordinate once: the
         * running sum already is the exact one, and nothing more is charged */
        if (wor && S[l] != ex) { status = ORC_EINTERNAL; break; }
        S[l] = ex;
        if (!wor) ++nexact;
      }
    }
    if (status != ORC_OK) break;
  }
  for (int32_t r = 0; r < k + h; ++r) set[r] = order[r];
  if (counts) memcpy(counts, T, sizeof(int32_t) * (size_t)n);
  if (sums) memcpy(sums, S, sizeof(int64_t) * (size_t)n);
  if (draws) *draws = ndraws;
  if (evals) *evals = ndraws + (int64_t)d * nexact;
  if (iters) *iters = it;
  free(S); free(T); free(order);
  return status;
}
