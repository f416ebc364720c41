/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * Plain-C restatement of the reference's hot-path algorithms
 * (/root/reference/proj/core/src/ files), one function per reference symbol,
 * each citing the file:line it follows. Pinned by tests/test_oracle_*.py
 * against (a) the golden vectors the reference's own tests hold
 * (testutil.hpp:28-33, test_push_engines.cpp, test_walks.cpp, ...) and
 * (b) the reference library itself compiled unchanged into
 * oracle/_ref/libppr_ref.so (bit-for-bit on every engine, including the
 * mt19937_64 stream and therefore build_index / speedppr_query).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 *
 * Conventions: graphs are CSR (offsets u64[n+1], neighbors u32[m]);
 * vectors are caller-allocated double[n]; status 0 = ok, 1 = invalid
 * argument, 2 = runtime (data) error, 3 = logic error (broken invariant).
 */
#ifndef PPR_ORACLE_H
#define PPR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + rng.hpp:14-39 ------------------------------ */
typedef struct {
  uint64_t mt[312];
  int idx;
} og_rng;
void og_rng_seed(og_rng* r, uint64_t seed);
uint64_t og_rng_next(og_rng* r);
double og_rng_uniform01(og_rng* r);
uint64_t og_rng_below(og_rng* r, uint64_t bound);
void og_rng_draws(uint64_t seed, uint64_t count, uint64_t bound, uint64_t* out);

/* ---- Philox4x32-10 (independent restatement used to pin the product's) -- */
void og_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* The product's walk definition: step t of walk
 * (k, v) keyed by seed, tag = source (MC) or 0xFFFFFFFF (index). */
uint32_t og_philox_walk(const uint64_t* off, const uint32_t* nbr, uint32_t start,
                        uint32_t source, double alpha, uint64_t seed, uint32_t k, uint32_t v,
                        uint32_t tag);
void og_philox_build_index(const uint64_t* off, const uint32_t* nbr, uint64_t n, double alpha,
                           uint64_t seed, uint32_t* endpoints);

/* ---- graph: graph.cpp:13-63, synthetic.cpp:9-26 ------------------------- */
/* off_out needs room for 2*count+1 entries, nbr_out for count. */
int og_build_graph_from_edges(const uint64_t* pairs, uint64_t count, uint64_t* off_out,
                              uint32_t* nbr_out, uint64_t* n_out);
int og_validate_graph(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint64_t m);
uint64_t og_dead_ends(const uint64_t* off, uint64_t n, uint32_t* out /* may be NULL */);
/* two-call: pass nbr_out = NULL to get m (written to *m_out) */
int og_random_graph(uint32_t n, uint32_t min_out, uint32_t max_out, uint64_t seed,
                    uint64_t* off_out, uint32_t* nbr_out, uint64_t* m_out);

/* Synthetic R-MAT (the product's generator definition, restated on the host;
 * see oracle.c). off_out needs 2^scale+1 entries, nbr_out edge_factor<<scale.
 * Returns 1 on bad parameters, 2 on an empty graph or allocation failure. */
int og_generate_rmat(int scale, uint64_t edge_factor, double a, double b, double c, uint64_t seed,
                     int threads, uint64_t* off_out, uint32_t* nbr_out, uint64_t* n_out,
                     uint64_t* m_out);

/* ---- push engines: push.cpp ------------------------------------------- */
typedef struct {
  double r_sum;
  uint64_t pushes;     /* edge pushes: each push on v costs deg_eff(v) */
  uint32_t iterations; /* powitr/sim: iterations; powerpush: scan sweeps */
  int used_scan_phase; /* power_push trace */
  uint64_t local_node_pushes;
} og_stats;

void og_push_once(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                  double* reserve, double* residue, og_stats* st, uint32_t v);
/* iter_r_sums (optional) receives r_sum after each iteration, up to cap. */
int og_power_iteration(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                       double alpha, double lambda, double* reserve, double* residue,
                       og_stats* st, double* iter_r_sums, uint32_t cap);
int og_sim_forward_push(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                        double alpha, double lambda, double* reserve, double* residue,
                        og_stats* st);
/* lambda_stop <= 0 means none. */
int og_fifo_forward_push(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                         double alpha, double r_max, double lambda_stop, double* reserve,
                         double* residue, og_stats* st);
/* scan_threshold < 0 means default n/4. epoch_r_max (optional) gets epoch_num values. */
int og_power_push(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                  double lambda, uint32_t epoch_num, int64_t scan_threshold, double* reserve,
                  double* residue, og_stats* st, double* epoch_r_max);
/* refine in place on an existing (reserve, residue, st) state. */
int og_refine(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
              double r_max, double* reserve, double* residue, og_stats* st);

/* ---- truth: exact_ppr.cpp:45-90, metrics.cpp:27-55 --------------------- */
int og_exact_ppr(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                 double* pi);
typedef struct {
  double l1, max_rel_above_mu;
  uint64_t nodes_above_mu, violations;
} og_error_report;
void og_compare_to_truth(const double* est, const double* truth, uint64_t n, double mu,
                         double eps, og_error_report* out);

/* ---- SpeedPPR: speedppr.cpp, walk_index.cpp ---------------------------- */
double og_walk_budget_real(uint64_t n, double eps, double mu); /* <0 on invalid */
int og_compute_walk_budget(uint64_t n, double eps, double mu, uint64_t* out);
uint32_t og_random_walk(const uint64_t* off, const uint32_t* nbr, uint32_t start, uint32_t source,
                        double alpha, og_rng* rng);
void og_build_index(const uint64_t* off, const uint32_t* nbr, uint64_t n, double alpha,
                    uint64_t seed, uint32_t* endpoints);
/* Monte Carlo phase (speedppr.cpp:23-72) over a refined state; index
 * endpoints may be NULL. Consumes rng. */
int og_monte_carlo(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s, double alpha,
                   double* reserve, double* residue, uint64_t W, const uint32_t* index_endpoints,
                   og_rng* rng, uint64_t* walks);
/* speedppr_query (speedppr.cpp:74-111), mt19937_64 stream, bit-exact with the
 * reference. mu <= 0 means 1/n. */
int og_speedppr_query(const uint64_t* off, const uint32_t* nbr, uint64_t n, uint32_t s,
                      double alpha, double eps, double mu, uint64_t seed,
                      const uint32_t* index_endpoints, double* est, uint64_t* walks,
                      uint64_t* pushes);

#ifdef __cplusplus
}
#endif
#endif
