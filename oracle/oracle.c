/* TEST INFRASTRUCTURE ONLY — see oracle.h. Plain-C restatement of the
 * reference algorithms; every function cites the reference file:line
 * (paths relative to /root/reference/proj/core/src unless noted). */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ========================================================================
 * RNG: std::mt19937_64 (the C++ standard's parameters) wrapped as rng.hpp.
 * ======================================================================== */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL

void og_rng_seed(og_rng* r, uint64_t seed) { /* rng.hpp:16 Rng(seed) : engine_(seed) */
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(og_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t x = (r->mt[i] & MT_UM) | (r->mt[(i + 1) % MT_N] & MT_LM);
    uint64_t xa = x >> 1;
    if (x & 1ULL) xa ^= MT_A;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
  }
  r->idx = 0;
}

uint64_t og_rng_next(og_rng* r) { /* rng.hpp:18 next() */
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

double og_rng_uniform01(og_rng* r) { /* rng.hpp:21 top 53 bits */
  return (double)(og_rng_next(r) >> 11) * 0x1.0p-53;
}

uint64_t og_rng_below(og_rng* r, uint64_t bound) { /* rng.hpp:24-35 Lemire + rejection */
  unsigned __int128 product = (unsigned __int128)og_rng_next(r) * bound;
  uint64_t low = (uint64_t)product;
  if (low < bound) {
    const uint64_t threshold = (0 - bound) % bound;
    while (low < threshold) {
      product = (unsigned __int128)og_rng_next(r) * bound;
      low = (uint64_t)product;
    }
  }
  return (uint64_t)(product >> 64);
}

void og_rng_draws(uint64_t seed, uint64_t count, uint64_t bound, uint64_t* out) {
  og_rng r;
  og_rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = bound ? og_rng_below(&r, bound) : og_rng_next(&r);
}

/* ========================================================================
 * Philox4x32-10 (Salmon et al., SC'11), restated independently of the
 * product's device implementation so the KAT + cross-check pin both.
 * ======================================================================== */
void og_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c[0] = hi1 ^ c[1] ^ k0;
    c[1] = lo1;
    c[2] = hi0 ^ c[3] ^ k1;
    c[3] = lo0;
  }
  memcpy(out, c, sizeof c);
}

/* Lemire bounded draw with rejection (rng.hpp:24-35 semantics) over Philox
 * 64-bit words; redraws use counter word 3 = t + (retry << 24). */
static uint64_t philox_below(uint64_t first, uint64_t bound, uint32_t k, uint32_t v, uint32_t tag,
                             uint32_t t, const uint32_t key[2]) {
  unsigned __int128 product = (unsigned __int128)first * bound;
  uint64_t low = (uint64_t)product;
  if (low < bound) {
    const uint64_t threshold = (0 - bound) % bound;
    uint32_t retry = 1;
    while (low < threshold) {
      const uint32_t ctr[4] = {k, v, tag, t + (retry++ << 24)};
      uint32_t o[4];
      og_philox4x32_10(ctr, key, o);
      product = (unsigned __int128)(((uint64_t)o[3] << 32) | o[2]) * bound;
      low = (uint64_t)product;
    }
  }
  return (uint64_t)(product >> 64);
}

/* One alpha-random walk (walk_index.cpp:10-17 semantics: stop with
 * probability alpha, else move to a uniform effective out-neighbor, dead-ends
 * jump to `source`), drawing step t from Philox(key=seed, ctr=(k,v,tag,t)). */
uint32_t og_philox_walk(const uint64_t* off, const uint32_t* nbr, uint32_t start, uint32_t source,
                        double alpha, uint64_t seed, uint32_t k, uint32_t v, uint32_t tag) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t cur = start;
  for (uint32_t t = 0;; ++t) {
    const uint32_t ctr[4] = {k, v, tag, t};
    uint32_t o[4];
    og_philox4x32_10(ctr, key, o);
    const double u = (double)((((uint64_t)o[1] << 32) | o[0]) >> 11) * 0x1.0p-53;
    if (!(u >= alpha)) return cur;
    const uint64_t d = off[cur + 1] - off[cur];
    if (d == 0) {
      cur = source;
    } else {
      const uint64_t i = philox_below(((uint64_t)o[3] << 32) | o[2], d, k, v, tag, t, key);
      cur = nbr[off[cur] + i];
    }
  }
}

void og_philox_build_index(const uint64_t* off, const uint32_t* nbr, uint64_t n, double alpha,
                           uint64_t seed, uint32_t* endpoints) {
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t k = 0; k < off[v + 1] - off[v]; ++k)
      endpoints[off[v] + k] = og_philox_walk(off, nbr, (uint32_t)v, (uint32_t)v, alpha, seed,
                                             (uint32_t)k, (uint32_t)v, 0xFFFFFFFFu);
}

/* ========================================================================
 * Graph: graph.cpp:13-63, graph.hpp:23-86
 * ======================================================================== */
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

static uint64_t lower_bound_u64(const uint64_t* ids, uint64_t cnt, uint64_t key) {
  uint64_t lo = 0, hi = cnt;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (ids[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

/* build_graph_from_edges (graph.cpp:36-63): survivors = sorted unique
 * endpoints (:40-47); new id = rank (:48-51); offsets = scan of per-source
 * counts (:54-56); neighbors placed in input order by a cursor (:58-60). */
int og_build_graph_from_edges(const uint64_t* pairs, uint64_t count, uint64_t* off_out,
                              uint32_t* nbr_out, uint64_t* n_out) {
  if (count == 0) return 2; /* graph.cpp:37 */
  uint64_t* ids = (uint64_t*)malloc(16 * count);
  memcpy(ids, pairs, 16 * count);
  qsort(ids, 2 * count, 8, cmp_u64);
  uint64_t n = 0;
  for (uint64_t i = 0; i < 2 * count; ++i)
    if (n == 0 || ids[n - 1] != ids[i]) ids[n++] = ids[i];
  memset(off_out, 0, 8 * (n + 1));
  for (uint64_t i = 0; i < count; ++i) off_out[lower_bound_u64(ids, n, pairs[2 * i]) + 1]++;
  for (uint64_t i = 0; i < n; ++i) off_out[i + 1] += off_out[i];
  uint64_t* cursor = (uint64_t*)malloc(8 * n);
  memcpy(cursor, off_out, 8 * n);
  for (uint64_t i = 0; i < count; ++i)
    nbr_out[cursor[lower_bound_u64(ids, n, pairs[2 * i])]++] =
        (uint32_t)lower_bound_u64(ids, n, pairs[2 * i + 1]);
  free(cursor);
  free(ids);
  *n_out = n;
  return og_validate_graph(off_out, nbr_out, n, count);
}

int og_validate_graph(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint64_t m) {
  /* Graph::validate (graph.cpp:24-34) */
  if (off[0] != 0) return 2;
  for (uint64_t v = 0; v < n; ++v)
    if (off[v + 1] < off[v]) return 2;
  if (off[n] != m) return 2;
  for (uint64_t e = 0; e < m; ++e)
    if (nbr[e] >= n) return 2;
  return 0;
}

uint64_t og_dead_ends(const uint64_t* off, uint64_t n, uint32_t* out) { /* graph.cpp:19-20 */
  uint64_t c = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (off[v + 1] == off[v]) {
      if (out) out[c] = (uint32_t)v;
      ++c;
    }
  return c;
}

/* random_graph (synthetic.cpp:9-26): degrees drawn first for all nodes, then
 * targets, from one Rng. */
int og_random_graph(uint32_t n, uint32_t min_out, uint32_t max_out, uint64_t seed,
                    uint64_t* off_out, uint32_t* nbr_out, uint64_t* m_out) {
  if (n == 0 || min_out > max_out) return 1;
  og_rng r;
  og_rng_seed(&r, seed);
  uint32_t* deg = (uint32_t*)malloc(4ull * n);
  uint64_t m = 0;
  for (uint32_t v = 0; v < n; ++v) {
    deg[v] = min_out + (uint32_t)og_rng_below(&r, (uint64_t)(max_out - min_out) + 1);
    if (off_out) off_out[v] = m;
    m += deg[v];
  }
  if (off_out) off_out[n] = m;
  *m_out = m;
  if (nbr_out) {
    uint64_t e = 0;
    for (uint32_t v = 0; v < n; ++v)
      for (uint32_t k = 0; k < deg[v]; ++k) nbr_out[e++] = (uint32_t)og_rng_below(&r, n);
  }
  free(deg);
  return 0;
}

static inline uint64_t deg_eff(const uint64_t* off, uint64_t v) { /* graph.hpp:83-86 */
  const uint64_t d = off[v + 1] - off[v];
  return d ? d : 1;
}

/* ========================================================================
 * Push engines: push.cpp
 * ======================================================================== */
static int recompute_r_sum(const double* residue, uint64_t n, double* r_sum) { /* push.cpp:9-15 */
  double total = 0.0;
  for (uint64_t v = 0; v < n; ++v) total += residue[v];
  if (fabs(total - *r_sum) > 1e-6) return 3;
  *r_sum = total;
  return 0;
}

static void init_state(uint64_t n, uint32_t s, double* reserve, double* residue, og_stats* st) {
  memset(reserve, 0, 8 * n); /* PushState(n, s), push.hpp:51-55 */
  memset(residue, 0, 8 * n);
  residue[s] = 1.0;
  memset(st, 0, sizeof *st);
  st->r_sum = 1.0;
}

/* push_once (push.cpp:17-27): zero before the spread so self-loops keep
 * their share; dead-ends spread to the source. */
void og_push_once(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                  double* reserve, double* residue, og_stats* st, uint32_t v) {
  (void)n;
  const double r = residue[v];
  if (r <= 0.0) return;
  reserve[v] += alpha * r;
  residue[v] = 0.0;
  const uint64_t d = off[v + 1] - off[v];
  const uint64_t de = d ? d : 1;
  const double share = (1.0 - alpha) * r / (double)de;
  if (d == 0) residue[s] += share;
  for (uint64_t j = off[v]; j < off[v + 1]; ++j) residue[nbr[j]] += share;
  st->r_sum -= alpha * r;
  st->pushes += de;
}

/* FIFO ring of capacity n+1 (push.hpp:15-39) */
typedef struct {
  uint32_t* buf;
  uint64_t cap, head, tail;
} fifo;
static uint64_t fifo_size(const fifo* q) {
  return q->tail >= q->head ? q->tail - q->head : q->cap - q->head + q->tail;
}
static void fifo_push(fifo* q, uint32_t v) {
  q->buf[q->tail] = v;
  q->tail = q->tail + 1 == q->cap ? 0 : q->tail + 1;
}
static uint32_t fifo_pop(fifo* q) {
  const uint32_t v = q->buf[q->head];
  q->head = q->head + 1 == q->cap ? 0 : q->head + 1;
  return v;
}

/* drain_queue (push.cpp:34-59): pop while non-empty and size <= limit,
 * checking r_sum <= lambda_stop before every pop; enqueue u once when it
 * becomes active (residue > deg_eff * r_max). */
static void drain_queue(const uint64_t* off, const uint32_t* nbr, uint32_t s, double alpha,
                        double r_max, double lambda_stop, uint64_t limit, double* reserve,
                        double* residue, uint8_t* in_q, fifo* q, og_stats* st) {
  while (q->head != q->tail && fifo_size(q) <= limit) {
    if (lambda_stop > 0 && st->r_sum <= lambda_stop) break;
    const uint32_t v = fifo_pop(q);
    in_q[v] = 0;
    const double r = residue[v];
    if (r <= 0.0) continue;
    reserve[v] += alpha * r;
    residue[v] = 0.0;
    const uint64_t d = off[v + 1] - off[v];
    const uint64_t de = d ? d : 1;
    const double share = (1.0 - alpha) * r / (double)de;
    for (uint64_t i = 0; i < de; ++i) {
      const uint32_t u = d ? nbr[off[v] + i] : s;
      residue[u] += share;
      if (!in_q[u] && residue[u] > (double)deg_eff(off, u) * r_max) {
        in_q[u] = 1;
        fifo_push(q, u);
      }
    }
    st->r_sum -= alpha * r;
    st->pushes += de;
    st->local_node_pushes++;
  }
}

static void seed_source(const uint64_t* off, uint32_t s, double r_max, const double* residue,
                        uint8_t* in_q, fifo* q) { /* push.cpp:61-66 */
  if (residue[s] > (double)deg_eff(off, s) * r_max) {
    in_q[s] = 1;
    fifo_push(q, s);
  }
}

/* power_iteration (push.cpp:81-108): Jacobi sweeps over all v (zeros
 * included), exact r_sum after every iteration. */
int og_power_iteration(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                       double alpha, double lambda, double* reserve, double* residue,
                       og_stats* st, double* iter_r_sums, uint32_t cap) {
  init_state(n, s, reserve, residue, st);
  double* next = (double*)malloc(8 * n);
  while (st->r_sum > lambda) {
    memset(next, 0, 8 * n);
    for (uint64_t v = 0; v < n; ++v) {
      const double r = residue[v];
      reserve[v] += alpha * r;
      const uint64_t d = off[v + 1] - off[v];
      const uint64_t de = d ? d : 1;
      const double share = (1.0 - alpha) * r / (double)de;
      if (d == 0) next[s] += share;
      for (uint64_t j = off[v]; j < off[v + 1]; ++j) next[nbr[j]] += share;
      st->pushes += de;
    }
    memcpy(residue, next, 8 * n);
    double total = 0.0;
    for (uint64_t v = 0; v < n; ++v) total += residue[v];
    st->r_sum = total;
    if (iter_r_sums && st->iterations < cap) iter_r_sums[st->iterations] = total;
    st->iterations++;
  }
  free(next);
  return 0;
}

/* sim_forward_push (push.cpp:110-138): as power_iteration but zero residues
 * are skipped (r_max = 0 snapshot semantics). */
int og_sim_forward_push(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                        double alpha, double lambda, double* reserve, double* residue,
                        og_stats* st) {
  init_state(n, s, reserve, residue, st);
  double* next = (double*)malloc(8 * n);
  while (st->r_sum > lambda) {
    memset(next, 0, 8 * n);
    for (uint64_t v = 0; v < n; ++v) {
      const double r = residue[v];
      if (r == 0.0) continue;
      reserve[v] += alpha * r;
      const uint64_t d = off[v + 1] - off[v];
      const uint64_t de = d ? d : 1;
      const double share = (1.0 - alpha) * r / (double)de;
      if (d == 0) next[s] += share;
      for (uint64_t j = off[v]; j < off[v + 1]; ++j) next[nbr[j]] += share;
      st->pushes += de;
    }
    memcpy(residue, next, 8 * n);
    double total = 0.0;
    for (uint64_t v = 0; v < n; ++v) total += residue[v];
    st->r_sum = total;
    st->iterations++;
  }
  free(next);
  return 0;
}

/* fifo_forward_push (push.cpp:140-149) */
int og_fifo_forward_push(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                         double alpha, double r_max, double lambda_stop, double* reserve,
                         double* residue, og_stats* st) {
  if (!(r_max > 0.0)) return 1;
  init_state(n, s, reserve, residue, st);
  fifo q = {(uint32_t*)malloc(4 * (n + 1)), n + 1, 0, 0};
  uint8_t* in_q = (uint8_t*)calloc(n, 1);
  seed_source(off, s, r_max, residue, in_q, &q);
  drain_queue(off, nbr, s, alpha, r_max, lambda_stop, UINT64_MAX, reserve, residue, in_q, &q, st);
  const int rc = recompute_r_sum(residue, n, &st->r_sum);
  free(q.buf);
  free(in_q);
  return rc;
}

/* power_push_state (push.cpp:151-199) + finish_state: local FIFO phase up
 * to the scan threshold, then epochs i = 1..epoch_num with
 * lambda_i = lambda^(i/epoch_num), r_max_i = lambda_i / m_eff, in-place
 * id-ordered sweeps until r_sum <= lambda_i (exact recompute per sweep). */
int og_power_push(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                  double lambda, uint32_t epoch_num, int64_t scan_threshold, double* reserve,
                  double* residue, og_stats* st, double* epoch_r_max) {
  if (!(lambda > 0.0 && lambda <= 1.0)) return 1; /* push.cpp:154-155 */
  const double m_eff = (double)(off[n] + og_dead_ends(off, n, NULL));
  const double r_max = lambda / m_eff;
  const uint64_t threshold = scan_threshold < 0 ? n / 4 : (uint64_t)scan_threshold;
  init_state(n, s, reserve, residue, st);
  fifo q = {(uint32_t*)malloc(4 * (n + 1)), n + 1, 0, 0};
  uint8_t* in_q = (uint8_t*)calloc(n, 1);
  seed_source(off, s, r_max, residue, in_q, &q);
  drain_queue(off, nbr, s, alpha, r_max, lambda, threshold, reserve, residue, in_q, &q, st);
  int rc = recompute_r_sum(residue, n, &st->r_sum);
  free(q.buf);
  free(in_q);
  if (rc) return rc;
  if (st->r_sum > lambda) {
    st->used_scan_phase = 1;
    for (uint32_t epoch = 1; epoch <= epoch_num; ++epoch) {
      const double epoch_lambda = pow(lambda, (double)epoch / epoch_num);
      const double epoch_rmax = epoch_lambda / m_eff;
      if (epoch_r_max) epoch_r_max[epoch - 1] = epoch_rmax;
      while (st->r_sum > epoch_lambda) {
        for (uint64_t v = 0; v < n; ++v) {
          const double r = residue[v];
          const uint64_t d = off[v + 1] - off[v];
          const uint64_t de = d ? d : 1;
          if (r <= (double)de * epoch_rmax) continue;
          reserve[v] += alpha * r;
          residue[v] = 0.0;
          const double share = (1.0 - alpha) * r / (double)de;
          if (d == 0) residue[s] += share;
          for (uint64_t j = off[v]; j < off[v + 1]; ++j) residue[nbr[j]] += share;
          st->r_sum -= alpha * r;
          st->pushes += de;
        }
        if ((rc = recompute_r_sum(residue, n, &st->r_sum))) return rc;
        st->iterations++;
      }
    }
  }
  return 0;
}

/* refine (push.cpp:208-222): enqueue every active node in id order, drain
 * with no limit, recompute r_sum. */
int og_refine(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
              double r_max, double* reserve, double* residue, og_stats* st) {
  if (!(r_max > 0.0)) return 1;
  fifo q = {(uint32_t*)malloc(4 * (n + 1)), n + 1, 0, 0};
  uint8_t* in_q = (uint8_t*)calloc(n, 1);
  for (uint64_t v = 0; v < n; ++v)
    if (residue[v] > (double)deg_eff(off, v) * r_max) {
      in_q[v] = 1;
      fifo_push(&q, (uint32_t)v);
    }
  drain_queue(off, nbr, s, alpha, r_max, -1.0, UINT64_MAX, reserve, residue, in_q, &q, st);
  free(q.buf);
  free(in_q);
  return recompute_r_sum(residue, n, &st->r_sum);
}

/* ========================================================================
 * Truth: exact_ppr.cpp:45-90, metrics.cpp:27-42
 * ======================================================================== */
int og_exact_ppr(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                 double* pi) {
  if (n > 2000) return 1; /* kDenseSolveMaxNodes, exact_ppr.hpp:17 */
  if (!(alpha > 0.0 && alpha < 1.0)) return 1;
  if (s >= n) return 1;
  double* a = (double*)calloc(n * n, 8);
  for (uint64_t i = 0; i < n; ++i) a[i * n + i] = 1.0;
  for (uint64_t v = 0; v < n; ++v) { /* column system of pi (I - (1-a) P) = a e_s */
    const uint64_t d = off[v + 1] - off[v];
    const double share = (1.0 - alpha) / (double)(d ? d : 1);
    if (d == 0) a[(uint64_t)s * n + v] -= share;
    for (uint64_t j = off[v]; j < off[v + 1]; ++j) a[(uint64_t)nbr[j] * n + v] -= share;
  }
  double* b = pi;
  memset(b, 0, 8 * n);
  b[s] = alpha;
  for (uint64_t k = 0; k < n; ++k) { /* solve_inplace, exact_ppr.cpp:11-41 */
    uint64_t p = k;
    double best = fabs(a[k * n + k]);
    for (uint64_t i = k + 1; i < n; ++i)
      if (fabs(a[i * n + k]) > best) { best = fabs(a[i * n + k]); p = i; }
    if (best == 0.0) { free(a); return 3; }
    if (p != k) {
      for (uint64_t j = k; j < n; ++j) {
        const double t = a[k * n + j]; a[k * n + j] = a[p * n + j]; a[p * n + j] = t;
      }
      const double t = b[k]; b[k] = b[p]; b[p] = t;
    }
    const double inv = 1.0 / a[k * n + k];
    for (uint64_t i = k + 1; i < n; ++i) {
      const double f = a[i * n + k] * inv;
      if (f == 0.0) continue;
      a[i * n + k] = 0.0;
      for (uint64_t j = k + 1; j < n; ++j) a[i * n + j] -= f * a[k * n + j];
      b[i] -= f * b[k];
    }
  }
  for (uint64_t i = n; i-- > 0;) {
    double acc = b[i];
    for (uint64_t j = i + 1; j < n; ++j) acc -= a[i * n + j] * b[j];
    b[i] = acc / a[i * n + i];
  }
  free(a);
  double sum = 0.0;
  for (uint64_t v = 0; v < n; ++v) {
    if (pi[v] < 0.0) {
      if (pi[v] < -1e-12) return 3;
      pi[v] = 0.0;
    }
    sum += pi[v];
  }
  if (fabs(sum - 1.0) > 1e-10) return 3;
  return 0;
}

void og_compare_to_truth(const double* est, const double* truth, uint64_t n, double mu,
                         double eps, og_error_report* out) {
  memset(out, 0, sizeof *out);
  for (uint64_t i = 0; i < n; ++i) {
    const double diff = fabs(est[i] - truth[i]);
    out->l1 += diff;
    if (truth[i] >= mu) {
      out->nodes_above_mu++;
      const double rel = diff / truth[i];
      if (rel > out->max_rel_above_mu) out->max_rel_above_mu = rel;
      if (rel > eps) out->violations++;
    }
  }
}

/* ========================================================================
 * SpeedPPR: speedppr.cpp:8-111, walk_index.cpp:10-54
 * ======================================================================== */
double og_walk_budget_real(uint64_t n, double eps, double mu) { /* speedppr.cpp:8-14 */
  if (n < 2 || !(eps > 0.0) || !(mu > 0.0 && mu <= 1.0)) return -1.0;
  return 2.0 * (2.0 * eps / 3.0 + 2.0) * log((double)n) / (eps * eps * mu);
}

int og_compute_walk_budget(uint64_t n, double eps, double mu, uint64_t* out) {
  const double w = og_walk_budget_real(n, eps, mu);
  if (w < 0) return 1;
  *out = (uint64_t)ceil(w);
  return 0;
}

uint32_t og_random_walk(const uint64_t* off, const uint32_t* nbr, uint32_t start, uint32_t source,
                        double alpha, og_rng* rng) { /* walk_index.cpp:10-17 */
  uint32_t cur = start;
  while (og_rng_uniform01(rng) >= alpha) {
    const uint64_t d = off[cur + 1] - off[cur];
    const uint64_t i = og_rng_below(rng, d ? d : 1);
    cur = d ? nbr[off[cur] + i] : source;
  }
  return cur;
}

void og_build_index(const uint64_t* off, const uint32_t* nbr, uint64_t n, double alpha,
                    uint64_t seed, uint32_t* endpoints) { /* walk_index.cpp:44-54 */
  og_rng r;
  og_rng_seed(&r, seed);
  uint64_t pos = 0;
  for (uint64_t v = 0; v < n; ++v)
    for (uint64_t k = 0; k < off[v + 1] - off[v]; ++k)
      endpoints[pos++] = og_random_walk(off, nbr, (uint32_t)v, (uint32_t)v, alpha, &r);
}

/* run_monte_carlo (speedppr.cpp:23-50) with the index variant (:60-72). */
int og_monte_carlo(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                   double* reserve, double* residue, uint64_t W, const uint32_t* index_endpoints,
                   og_rng* rng, uint64_t* walks) {
  const double budget = (double)W;
  uint64_t total = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const double r = residue[v];
    if (r <= 0.0) continue;
    const uint64_t d = off[v + 1] - off[v];
    const uint64_t degree = d ? d : 1;
    uint64_t wc = (uint64_t)ceil(r * budget);
    if (wc > degree) {
      if (r * budget > (double)degree * (1.0 + 1e-9) + 1e-9) return 3; /* :33-37 */
      wc = degree;
    }
    const double contribution = r / (double)wc;
    for (uint64_t k = 0; k < wc; ++k) {
      uint32_t t;
      if (index_endpoints && d) t = index_endpoints[off[v] + k];
      else t = og_random_walk(off, nbr, (uint32_t)v, s, alpha, rng);
      reserve[t] += contribution;
    }
    total += wc;
    residue[v] = 0.0;
  }
  *walks = total;
  return 0;
}

int og_speedppr_query(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                      double alpha, double eps, double mu, uint64_t seed,
                      const uint32_t* index_endpoints, double* est, uint64_t* walks,
                      uint64_t* pushes) {
  if (!(alpha >= 0.0 && alpha < 1.0) || !(eps > 0.0)) return 1; /* QueryConfig::validate */
  if (mu > 0.0 && !(mu <= 1.0)) return 1;
  if (s >= n) return 1;
  const double mu_eff = mu > 0.0 ? mu : 1.0 / (double)n;
  uint64_t W;
  if (og_compute_walk_budget(n, eps, mu_eff, &W)) return 1;
  og_rng rng;
  og_rng_seed(&rng, seed);
  const uint64_t m_eff = off[n] + og_dead_ends(off, n, NULL);
  if (W <= m_eff) { /* speedppr.cpp:90-102 */
    memset(est, 0, 8 * n);
    const double contribution = 1.0 / (double)W;
    for (uint64_t k = 0; k < W; ++k) est[og_random_walk(off, nbr, s, s, alpha, &rng)] += contribution;
    *walks = W;
    *pushes = 0;
    return 0;
  }
  const double lambda = (double)m_eff / (double)W;
  double* residue = (double*)malloc(8 * n);
  og_stats st;
  int rc = og_power_push(off, nbr, n, s, alpha, lambda, 8, -1, est, residue, &st, NULL);
  if (!rc) rc = og_refine(off, nbr, n, s, alpha, 1.0 / (double)W, est, residue, &st);
  if (!rc) rc = og_monte_carlo(off, nbr, n, s, alpha, est, residue, W, index_endpoints, &rng, walks);
  *pushes = st.pushes;
  free(residue);
  return rc;
}

/* ========================================================================
 * Synthetic R-MAT input (SURVEY 8(d) "Synthetic inputs"), restated on the
 * host so the reference arm of bench.py never needs the GPU library to make
 * its input. The definition is the product's (pprg_graph_generate_rmat,
 * graph.cu k_rmat + sort_clean + build_from_sorted_keys) and is pinned to it
 * bit-for-bit by tests/test_gpu_configs.py:
 *   edge i descends `scale` levels; level l uses 32-bit word (l mod 4) of
 *   Philox4x32-10(ctr = (i_lo, i_hi, 'RMAT', l/4), key = seed); p = w/2^32
 *   selects quadrant a (0,0) / b (0,1) / c (1,0) / d (1,1) by p < a, < a+b,
 *   < a+b+c. Edges are sorted by (u, v), duplicates and self-loops dropped,
 *   surviving endpoint ids relabelled by rank (graph.cpp:40-51 semantics) and
 *   the CSR built with each row in ascending neighbour order.
 * ======================================================================== */
typedef struct {
  uint64_t lo, hi, seed;
  int scale;
  double a, ab, abc;
  uint64_t* keys;
} rmat_job;

static void* rmat_worker(void* arg) {
  const rmat_job* j = (const rmat_job*)arg;
  const uint32_t key[2] = {(uint32_t)j->seed, (uint32_t)(j->seed >> 32)};
  const int s = j->scale;
  for (uint64_t i = j->lo; i < j->hi; ++i) {
    uint32_t u = 0, v = 0, o[4] = {0, 0, 0, 0};
    for (int l = 0; l < s; ++l) {
      if ((l & 3) == 0) {
        const uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 0x524D4154u, (uint32_t)(l >> 2)};
        og_philox4x32_10(ctr, key, o);
      }
      const double p = (double)o[l & 3] * 0x1.0p-32;
      const uint32_t bu = p >= j->ab, bv = (p >= j->a && p < j->ab) || p >= j->abc;
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    j->keys[i] = ((uint64_t)u << s) | v; /* compact (u, v) key: 2*scale bits */
  }
  return NULL;
}

/* LSD radix sort of `cnt` keys of `bits` bits, 16 bits per pass. */
static void radix_sort_u64(uint64_t* keys, uint64_t* tmp, uint64_t cnt, int bits) {
  uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) << 16);
  uint64_t* const first = keys;
  for (int shift = 0; shift < bits; shift += 16) {
    memset(hist, 0, sizeof(uint64_t) << 16);
    for (uint64_t i = 0; i < cnt; ++i) ++hist[(keys[i] >> shift) & 0xFFFF];
    uint64_t run = 0;
    for (int d = 0; d < 65536; ++d) {
      const uint64_t c = hist[d];
      hist[d] = run;
      run += c;
    }
    for (uint64_t i = 0; i < cnt; ++i) tmp[hist[(keys[i] >> shift) & 0xFFFF]++] = keys[i];
    uint64_t* t = keys;
    keys = tmp;
    tmp = t;
  }
  if (keys != first) memcpy(first, keys, 8 * cnt); /* result in the caller's first buffer */
  free(hist);
}

int og_generate_rmat(int scale, uint64_t edge_factor, double a, double b, double c, uint64_t seed,
                     int threads, uint64_t* off_out, uint32_t* nbr_out, uint64_t* n_out,
                     uint64_t* m_out) {
  if (scale < 1 || scale > 31) return 1;
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) return 1;
  const uint64_t draws = edge_factor << scale, id_space = 1ull << scale;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  uint64_t* keys = (uint64_t*)malloc(8 * (draws ? draws : 1));
  uint64_t* tmp = (uint64_t*)malloc(8 * (draws ? draws : 1));
  if (!keys || !tmp) {
    free(keys);
    free(tmp);
    return 2;
  }
  pthread_t tid[256];
  rmat_job job[256];
  for (int t = 0; t < threads; ++t) {
    job[t] = (rmat_job){draws * t / threads, draws * (t + 1) / threads, seed, scale, a, a + b,
                        a + b + c, keys};
    pthread_create(&tid[t], NULL, rmat_worker, &job[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  radix_sort_u64(keys, tmp, draws, 2 * scale);
  const uint64_t vmask = id_space - 1;
  uint64_t cnt = 0; /* unique, no self-loops, compacted in place */
  for (uint64_t i = 0; i < draws; ++i) {
    const uint64_t k = keys[i];
    if ((i == 0 || keys[i - 1] != k) && (k >> scale) != (k & vmask)) tmp[cnt++] = k;
  }
  free(keys);
  if (cnt == 0) {
    free(tmp);
    return 2; /* "graph is empty after cleaning" */
  }
  uint32_t* rank = (uint32_t*)calloc(id_space + 1, 4);
  for (uint64_t i = 0; i < cnt; ++i) {
    rank[tmp[i] >> scale] = 1;
    rank[tmp[i] & vmask] = 1;
  }
  uint64_t n = 0;
  for (uint64_t v = 0; v <= id_space; ++v) {
    const uint32_t p = rank[v];
    rank[v] = (uint32_t)n;
    n += p;
  }
  memset(off_out, 0, 8 * (n + 1));
  for (uint64_t i = 0; i < cnt; ++i) {
    ++off_out[rank[tmp[i] >> scale] + 1];
    nbr_out[i] = rank[tmp[i] & vmask];
  }
  for (uint64_t v = 0; v < n; ++v) off_out[v + 1] += off_out[v];
  free(rank);
  free(tmp);
  *n_out = n;
  *m_out = cnt;
  return 0;
}
