// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C shim over the *unmodified* reference library (compiled from the sources
// under /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libppr_ref.so). It lets pytest (ctypes), bench.py's
// `--impl reference` arm and the oracle self-checks call the reference's own
// C++ API:
//   ppr::build_graph_from_edges / Graph(offsets, neighbors)  graph.hpp:18,92
//   ppr::power_iteration / sim_forward_push / fifo_forward_push   push.hpp:80-95
//   ppr::power_push (+ PowerPushTrace) / power_push_state / refine push.hpp:105-119
//   ppr::speedppr_query / compute_walk_budget / monte_carlo_phase speedppr.hpp
//   ppr::build_index / random_walk / save_index / load_index       walk_index.hpp
//   ppr::exact_ppr / ground_truth / random_graph                    exact_ppr.hpp, metrics.hpp
// Exceptions are mapped to status codes: 1 invalid_argument, 2 runtime_error,
// 3 logic_error, 4 anything else; the message is kept per thread.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ppr/exact_ppr.hpp"
#include "ppr/graph.hpp"
#include "ppr/metrics.hpp"
#include "ppr/push.hpp"
#include "ppr/speedppr.hpp"
#include "ppr/synthetic.hpp"
#include "ppr/walk_index.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

struct Out {
  double* reserve;
  double* residue;
  double* r_sum;
  std::uint64_t* pushes;
  std::uint64_t* walks;
};

void emit(const ppr::PPRVector& v, std::uint32_t n, const Out& o) {
  if (o.reserve) std::memcpy(o.reserve, v.estimates.data(), 8ull * n);
  if (o.residue) std::memcpy(o.residue, v.residues.data(), 8ull * n);
  if (o.r_sum) *o.r_sum = v.achieved_r_sum;
  if (o.pushes) *o.pushes = v.pushes;
  if (o.walks) *o.walks = v.walks;
}

struct IterTrace : ppr::PushObserver {
  std::vector<double> r_sums;
  std::vector<double> reserves, residues;  // flattened per iteration (optional)
  bool keep_vectors = false;
  void on_iteration(const ppr::PushState& st, std::uint32_t) override {
    r_sums.push_back(st.r_sum);
    if (keep_vectors) {
      reserves.insert(reserves.end(), st.reserve.begin(), st.reserve.end());
      residues.insert(residues.end(), st.residue.begin(), st.residue.end());
    }
  }
};

ppr::QueryConfig make_cfg(double alpha, std::uint32_t epoch_num, std::int64_t scan_threshold) {
  ppr::QueryConfig cfg;
  cfg.alpha = alpha;
  cfg.epoch_num = epoch_num;
  if (scan_threshold >= 0) cfg.scan_threshold = static_cast<std::uint64_t>(scan_threshold);
  return cfg;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- graphs ------------------------------------------------------------------
int ref_graph_from_edges(const std::uint64_t* pairs, std::uint64_t count, void** out) {
  return guard([&] {
    std::vector<std::pair<std::uint64_t, std::uint64_t>> edges(count);
    for (std::uint64_t i = 0; i < count; ++i) edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    *out = new ppr::Graph(ppr::build_graph_from_edges(edges));
  });
}

int ref_graph_from_csr(const std::uint64_t* offsets, const std::uint32_t* nbrs, std::uint64_t n,
                       void** out) {
  return guard([&] {
    std::vector<std::uint64_t> off(offsets, offsets + n + 1);
    std::vector<ppr::NodeId> nb(nbrs, nbrs + offsets[n]);
    *out = new ppr::Graph(std::move(off), std::move(nb));
  });
}

int ref_random_graph(std::uint32_t n, std::uint32_t min_out, std::uint32_t max_out,
                     std::uint64_t seed, void** out) {
  return guard([&] { *out = new ppr::Graph(ppr::random_graph(n, min_out, max_out, seed)); });
}

int ref_load_graph_cache(const char* path, void** out) {
  return guard([&] { *out = new ppr::Graph(ppr::load_graph_cache(path)); });
}
int ref_save_graph_cache(const void* g, const char* path) {
  return guard([&] { ppr::save_graph_cache(*static_cast<const ppr::Graph*>(g), path); });
}
int ref_load_edge_list(const char* path, int undirected, void** out) {
  return guard([&] {
    *out = new ppr::Graph(undirected ? ppr::undirected_to_directed(path) : ppr::load_edge_list(path));
  });
}

void ref_graph_free(void* g) { delete static_cast<ppr::Graph*>(g); }
std::uint64_t ref_graph_n(const void* g) { return static_cast<const ppr::Graph*>(g)->n(); }
std::uint64_t ref_graph_m(const void* g) { return static_cast<const ppr::Graph*>(g)->m(); }
std::uint64_t ref_graph_dead_end_count(const void* g) {
  return static_cast<const ppr::Graph*>(g)->dead_ends().size();
}
void ref_graph_export(const void* gp, std::uint64_t* offsets, std::uint32_t* nbrs,
                      std::uint32_t* dead_ends) {
  const auto& g = *static_cast<const ppr::Graph*>(gp);
  if (offsets) std::memcpy(offsets, g.out_offsets().data(), 8ull * (g.n() + 1));
  if (nbrs) std::memcpy(nbrs, g.out_neighbors().data(), 4ull * g.m());
  if (dead_ends) std::memcpy(dead_ends, g.dead_ends().data(), 4ull * g.dead_ends().size());
}

// ---- high-precision engines --------------------------------------------------
int ref_power_iteration(const void* gp, std::uint32_t s, double alpha, double lambda,
                        double* reserve, double* residue, double* r_sum, std::uint64_t* pushes,
                        double* iter_r_sums, std::uint32_t iter_cap, std::uint32_t* iters) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    IterTrace tr;
    auto v = ppr::power_iteration(g, s, alpha, lambda, &tr);
    emit(v, g.n(), {reserve, residue, r_sum, pushes, nullptr});
    if (iters) *iters = static_cast<std::uint32_t>(tr.r_sums.size());
    for (std::size_t i = 0; iter_r_sums && i < tr.r_sums.size() && i < iter_cap; ++i)
      iter_r_sums[i] = tr.r_sums[i];
  });
}

// Per-iteration reserve/residue snapshots of power_iteration (small graphs).
int ref_power_iteration_trace(const void* gp, std::uint32_t s, double alpha, double lambda,
                              double* reserves, double* residues, std::uint32_t iter_cap,
                              std::uint32_t* iters) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    IterTrace tr;
    tr.keep_vectors = true;
    ppr::power_iteration(g, s, alpha, lambda, &tr);
    const std::uint32_t k = static_cast<std::uint32_t>(tr.r_sums.size());
    *iters = k;
    const std::uint64_t n = g.n();
    for (std::uint32_t i = 0; i < k && i < iter_cap; ++i) {
      std::memcpy(reserves + i * n, tr.reserves.data() + i * n, 8 * n);
      std::memcpy(residues + i * n, tr.residues.data() + i * n, 8 * n);
    }
  });
}

int ref_sim_forward_push(const void* gp, std::uint32_t s, double alpha, double lambda,
                         double* reserve, double* residue, double* r_sum, std::uint64_t* pushes) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    emit(ppr::sim_forward_push(g, s, alpha, lambda), g.n(), {reserve, residue, r_sum, pushes, nullptr});
  });
}

int ref_fifo_forward_push(const void* gp, std::uint32_t s, double alpha, double r_max,
                          double lambda_stop, double* reserve, double* residue, double* r_sum,
                          std::uint64_t* pushes) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    std::optional<double> stop;
    if (lambda_stop > 0) stop = lambda_stop;
    emit(ppr::fifo_forward_push(g, s, alpha, r_max, stop), g.n(),
         {reserve, residue, r_sum, pushes, nullptr});
  });
}

int ref_power_push(const void* gp, std::uint32_t s, double alpha, double lambda,
                   std::uint32_t epoch_num, std::int64_t scan_threshold, double* reserve,
                   double* residue, double* r_sum, std::uint64_t* pushes, int* used_scan,
                   double* epoch_r_max) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    ppr::PowerPushTrace tr;
    auto v = ppr::power_push(g, s, alpha, lambda, make_cfg(alpha, epoch_num, scan_threshold),
                             nullptr, &tr);
    emit(v, g.n(), {reserve, residue, r_sum, pushes, nullptr});
    if (used_scan) *used_scan = tr.used_scan_phase ? 1 : 0;
    for (std::size_t i = 0; epoch_r_max && i < tr.epoch_r_max.size(); ++i)
      epoch_r_max[i] = tr.epoch_r_max[i];
  });
}

// power_push_state followed by refine(r_max): the SpeedPPR pre-walk state.
int ref_power_push_refine(const void* gp, std::uint32_t s, double alpha, double lambda,
                          double r_max, double* reserve, double* residue, double* r_sum,
                          std::uint64_t* pushes) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    ppr::QueryConfig cfg;
    cfg.alpha = alpha;
    ppr::PushState st = ppr::power_push_state(g, s, alpha, lambda, cfg);
    ppr::refine(g, s, alpha, r_max, st);
    emit(ppr::finish_state(std::move(st), s, alpha), g.n(), {reserve, residue, r_sum, pushes, nullptr});
  });
}

// Many independent power_push queries on `threads` std::threads sharing the
// const Graph (graph.hpp:15). Outputs are optional (k*n each).
int ref_power_push_batch(const void* gp, const std::uint32_t* sources, std::uint32_t k,
                         double alpha, double lambda, std::uint32_t threads, double* reserve,
                         double* residue, double* r_sums, int use_powitr) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    const std::uint64_t n = g.n();
    std::atomic<std::uint32_t> next{0};
    std::vector<std::thread> pool;
    std::vector<std::string> errs(threads);
    for (std::uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          for (std::uint32_t i; (i = next.fetch_add(1)) < k;) {
            ppr::QueryConfig cfg;
            cfg.alpha = alpha;
            auto v = use_powitr ? ppr::power_iteration(g, sources[i], alpha, lambda)
                                : ppr::power_push(g, sources[i], alpha, lambda, cfg);
            if (reserve) std::memcpy(reserve + i * n, v.estimates.data(), 8 * n);
            if (residue) std::memcpy(residue + i * n, v.residues.data(), 8 * n);
            if (r_sums) r_sums[i] = v.achieved_r_sum;
          }
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// ---- SpeedPPR ---------------------------------------------------------------
double ref_walk_budget_real(std::uint64_t n, double eps, double mu) {
  double out = -1;
  if (guard([&] { out = ppr::walk_budget_real(n, eps, mu); })) return -1;
  return out;
}
int ref_compute_walk_budget(std::uint64_t n, double eps, double mu, std::uint64_t* out) {
  return guard([&] { *out = ppr::compute_walk_budget(n, eps, mu); });
}

int ref_build_index(const void* gp, double alpha, std::uint64_t seed, void** out) {
  return guard([&] {
    *out = new ppr::WalkIndex(ppr::build_index(*static_cast<const ppr::Graph*>(gp), alpha, seed));
  });
}
void ref_index_free(void* idx) { delete static_cast<ppr::WalkIndex*>(idx); }
void ref_index_export(const void* ip, std::uint32_t* endpoints) {
  const auto& idx = *static_cast<const ppr::WalkIndex*>(ip);
  std::uint64_t pos = 0;
  for (ppr::NodeId v = 0; v < idx.node_count(); ++v)
    for (auto e : idx.endpoints_of(v)) endpoints[pos++] = e;
}
int ref_save_index(const void* ip, const char* path) {
  return guard([&] { ppr::save_index(*static_cast<const ppr::WalkIndex*>(ip), path); });
}
int ref_load_index(const char* path, void** out) {
  return guard([&] { *out = new ppr::WalkIndex(ppr::load_index(path)); });
}

// Indices are passed as (offsets, endpoints) so a GPU-built index can be fed
// to the reference MC phase; rng_id is stored but the reference's loader-side
// check does not apply to in-memory construction.
int ref_index_from_arrays(double alpha, std::uint64_t seed, std::uint8_t rng_id,
                          const std::uint64_t* offsets, std::uint64_t n,
                          const std::uint32_t* endpoints, void** out) {
  return guard([&] {
    std::vector<std::uint64_t> off(offsets, offsets + n + 1);
    std::vector<ppr::NodeId> ep(endpoints, endpoints + offsets[n]);
    *out = new ppr::WalkIndex(alpha, seed, rng_id, std::move(off), std::move(ep));
  });
}

int ref_speedppr_query(const void* gp, std::uint32_t s, double alpha, double eps, double mu,
                       std::uint64_t seed, const void* index, double* est, std::uint64_t* walks,
                       std::uint64_t* pushes) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    ppr::QueryConfig cfg;
    cfg.alpha = alpha;
    cfg.epsilon = eps;
    if (mu > 0) cfg.mu = mu;
    cfg.seed = seed;
    auto v = ppr::speedppr_query(g, s, cfg, static_cast<const ppr::WalkIndex*>(index));
    emit(v, g.n(), {est, nullptr, nullptr, pushes, walks});
  });
}

int ref_speedppr_batch(const void* gp, const std::uint32_t* sources, std::uint32_t k, double alpha,
                       double eps, std::uint64_t seed, const void* index, std::uint32_t threads) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    std::atomic<std::uint32_t> next{0};
    std::vector<std::thread> pool;
    std::vector<std::string> errs(threads);
    for (std::uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        try {
          for (std::uint32_t i; (i = next.fetch_add(1)) < k;) {
            ppr::QueryConfig cfg;
            cfg.alpha = alpha;
            cfg.epsilon = eps;
            cfg.seed = seed;
            ppr::speedppr_query(g, sources[i], cfg, static_cast<const ppr::WalkIndex*>(index));
          }
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// ---- truth -------------------------------------------------------------------
int ref_exact_ppr(const void* gp, std::uint32_t s, double alpha, double* pi) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    auto d = ppr::exact_ppr(g, s, alpha);
    std::memcpy(pi, d.pi.data(), 8ull * g.n());
  });
}
int ref_ground_truth(const void* gp, std::uint32_t s, double alpha, double* pi) {
  return guard([&] {
    const auto& g = *static_cast<const ppr::Graph*>(gp);
    auto v = ppr::ground_truth(g, s, alpha);
    std::memcpy(pi, v.estimates.data(), 8ull * g.n());
  });
}

// Reference Rng (mt19937_64) draws, to pin the oracle's restatement.
void ref_rng_draws(std::uint64_t seed, std::uint64_t count, std::uint64_t bound, std::uint64_t* out) {
  ppr::Rng rng(seed);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = bound ? rng.below(bound) : rng.next();
}

}  // extern "C"
