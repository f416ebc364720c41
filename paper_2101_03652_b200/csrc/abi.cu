// extern "C" boundary (include/pprg.h): argument checks with the reference's
// error behaviour, exception -> status mapping, per-thread error message.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pprg.h"
#include "internal.h"

struct pprg_graph {
  std::unique_ptr<pprg::Graph> g;
};
struct pprg_part {
  pprg::PartSession* s = nullptr;
  pprg_graph* owner = nullptr;
  uint32_t k = 0;
};
struct pprg_index {
  std::unique_ptr<pprg::WalkIndex> w;
  pprg_graph* owner;
};

namespace pprg {
void release_workspaces(const Graph* g);
}

namespace {
thread_local std::string t_err;
std::atomic<int> g_det_default{0};

template <typename F>
int guard(F&& f) {
  pprg::DetScope det(g_det_default.load() != 0);  // PPRG_DETERMINISTIC flags add to it
  try {
    f();
    return PPRG_OK;
  } catch (const pprg::Error& e) {
    t_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    t_err = std::string("out of host memory: ") + e.what();
    return PPRG_EINTERNAL;
  } catch (const std::exception& e) {
    t_err = e.what();
    return PPRG_EINTERNAL;
  }
}

void require(bool ok, const char* msg) {
  if (!ok) pprg::fail(PPRG_EINVAL, msg);
}

void fill_stats(const std::vector<pprg::ColumnStats>& cs, const pprg::CallStats& call, uint32_t k,
                pprg_query_stats* q, pprg_call_stats* c) {
  if (q)
    for (uint32_t i = 0; i < k; ++i) {
      q[i].achieved_r_sum = cs[i].r_sum;
      q[i].pushes = cs[i].pushes;
      q[i].walks = cs[i].walks;
      q[i].sweeps = cs[i].sweeps;
      q[i].local_levels = cs[i].local_levels;
      q[i].used_scan_phase = cs[i].used_scan_phase;
      q[i].reserved = 0;
    }
  if (c) {
    c->device_ms = call.device_ms;
    c->sweep_ms = call.sweep_ms;
    c->local_ms = call.local_ms;
    c->final_ms = call.final_ms;
    c->alg_bytes = call.alg_bytes;
    c->sweep_launches = call.sweep_launches;
    c->max_sweeps = call.max_sweeps;
    c->kernel_launches = call.kernel_launches;
  }
}

// alpha in (0,1): the reference admits alpha = 0 (types.hpp:37) but then never
// terminates; the device path rejects it instead of spinning.
void check_alpha(double alpha) {
  require(alpha > 0.0 && alpha < 1.0, "alpha must be in (0,1)");
}

int push_engine(pprg_graph* g, pprg::Engine eng, const uint32_t* sources, uint32_t k, double alpha,
                double lambda, uint32_t epoch_num, int64_t scan_threshold, double r_max,
                double lambda_stop, double* reserve_out, double* residue_out, uint32_t flags,
                pprg_query_stats* q, pprg_call_stats* c) {
  return guard([&] {
    if (flags & PPRG_DETERMINISTIC) pprg::t_det = true;
    require(g && g->g, "null graph");
    require(k == 0 || sources, "null sources");
    check_alpha(alpha);
    std::vector<pprg::ColumnStats> cs(k);
    pprg::CallStats call;
    pprg::Outputs out{reserve_out, residue_out, (flags & PPRG_OUT_DEVICE) != 0,
                      (flags & PPRG_ASYNC_HOST) != 0};
    if (k)
      pprg::run_push_engine(*g->g, eng, sources, k, alpha, lambda, epoch_num, scan_threshold,
                            r_max, lambda_stop, out, cs.data(), &call);
    fill_stats(cs, call, k, q, c);
  });
}
}  // namespace

extern "C" {

const char* pprg_last_error(void) { return t_err.c_str(); }
int pprg_version(void) { return 1; }

int pprg_set_deterministic(int on) {
  g_det_default.store(on ? 1 : 0);
  return PPRG_OK;
}

int pprg_device_count(int* count) {
  return guard([&] { PPRG_CUDA(cudaGetDeviceCount(count)); });
}

int pprg_graph_create(const uint64_t* offsets, const uint32_t* neighbors, uint64_t n, int device,
                      pprg_graph** out) {
  return guard([&] {
    require(out && offsets, "null argument");
    require(neighbors || offsets[n] == 0, "null neighbors");
    auto h = new pprg_graph;
    try {
      h->g = pprg::graph_from_csr(offsets, neighbors, n, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pprg_graph_build_from_edges(const uint64_t* pairs, uint64_t count, int device,
                                pprg_graph** out) {
  return guard([&] {
    require(out && (pairs || count == 0), "null argument");
    auto h = new pprg_graph;
    try {
      h->g = pprg::graph_from_edges(pairs, count, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pprg_graph_load_cache(const char* path, int device, pprg_graph** out) {
  return guard([&] {
    require(path && out, "null argument");
    auto h = new pprg_graph;
    try {
      h->g = pprg::graph_load_cache(path, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pprg_graph_save_cache(pprg_graph* g, const char* path) {
  return guard([&] {
    require(g && g->g && path, "null argument");
    pprg::graph_save_cache(*g->g, path);
  });
}

int pprg_graph_generate_rmat(int scale, uint64_t edge_factor, double a, double b, double c,
                             uint64_t seed, int device, uint64_t* edges_out,
                             uint64_t* edge_count_out, pprg_graph** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    std::vector<uint64_t> edges;
    auto h = new pprg_graph;
    try {
      h->g = pprg::graph_rmat(scale, edge_factor, a, b, c, seed, device,
                              edges_out || edge_count_out ? &edges : nullptr);
    } catch (...) {
      delete h;
      throw;
    }
    if (edges_out) std::memcpy(edges_out, edges.data(), 8 * edges.size());
    if (edge_count_out) *edge_count_out = edges.size();
    *out = h;
  });
}

int pprg_graph_generate_chung_lu(uint64_t n, uint64_t draws, double beta, uint64_t seed, int device,
                                 uint64_t* edges_out, uint64_t* edge_count_out, pprg_graph** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    std::vector<uint64_t> edges;
    auto h = new pprg_graph;
    try {
      h->g = pprg::graph_chung_lu(n, draws, beta, seed, device,
                                  edges_out || edge_count_out ? &edges : nullptr);
    } catch (...) {
      delete h;
      throw;
    }
    if (edges_out) std::memcpy(edges_out, edges.data(), 8 * edges.size());
    if (edge_count_out) *edge_count_out = edges.size();
    *out = h;
  });
}

int pprg_graph_info(const pprg_graph* g, uint64_t* n, uint64_t* m, uint64_t* dead_ends) {
  return guard([&] {
    require(g && g->g, "null graph");
    if (n) *n = g->g->n;
    if (m) *m = g->g->m;
    if (dead_ends) *dead_ends = g->g->n_dead;
  });
}

int pprg_graph_export(const pprg_graph* g, uint64_t* offsets, uint32_t* neighbors,
                      uint32_t* dead_ends) {
  return guard([&] {
    require(g && g->g, "null graph");
    pprg::Graph& G = *g->g;
    pprg::DeviceGuard dg(G.device);
    std::lock_guard<std::mutex> lk(G.mu);
    if (offsets)
      PPRG_CUDA(cudaMemcpyAsync(offsets, G.off.get(), 8 * (G.n + 1), cudaMemcpyDeviceToHost, G.stream));
    if (neighbors && G.m)
      PPRG_CUDA(cudaMemcpyAsync(neighbors, G.nbr.get(), 4 * G.m, cudaMemcpyDeviceToHost, G.stream));
    if (dead_ends && G.n_dead)
      PPRG_CUDA(cudaMemcpyAsync(dead_ends, G.dead.get(), 4 * G.n_dead, cudaMemcpyDeviceToHost, G.stream));
    PPRG_CUDA(cudaStreamSynchronize(G.stream));
  });
}

int pprg_graph_export_transpose(pprg_graph* g, uint64_t* in_offsets, uint32_t* in_neighbors) {
  return guard([&] {
    require(g && g->g, "null graph");
    pprg::Graph& G = *g->g;
    pprg::DeviceGuard dg(G.device);
    std::lock_guard<std::mutex> lk(G.mu);
    G.ensure_transpose();
    if (in_offsets)
      PPRG_CUDA(cudaMemcpyAsync(in_offsets, G.in_off.get(), 8 * (G.n + 1), cudaMemcpyDeviceToHost, G.stream));
    if (in_neighbors && G.m)
      PPRG_CUDA(cudaMemcpyAsync(in_neighbors, G.in_nbr.get(), 4 * G.m, cudaMemcpyDeviceToHost, G.stream));
    PPRG_CUDA(cudaStreamSynchronize(G.stream));
  });
}

void pprg_graph_destroy(pprg_graph* g) {
  if (!g) return;
  try {
    pprg::DeviceGuard dg(g->g ? g->g->device : 0);
    pprg::release_workspaces(g->g.get());
    g->g.reset();
  } catch (...) {
  }
  delete g;
}

int pprg_power_iteration(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                         double lambda, double* reserve_out, double* residue_out, uint32_t flags,
                         pprg_query_stats* q, pprg_call_stats* c) {
  // power_iteration validates nothing; lambda >= 1 => 0 iterations
  return push_engine(g, pprg::Engine::PowItr, sources, k, alpha, lambda, 0, -1, 0, 0, reserve_out,
                     residue_out, flags, q, c);
}

int pprg_sim_forward_push(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                          double lambda, double* reserve_out, double* residue_out, uint32_t flags,
                          pprg_query_stats* q, pprg_call_stats* c) {
  return push_engine(g, pprg::Engine::SimFwdPush, sources, k, alpha, lambda, 0, -1, 0, 0,
                     reserve_out, residue_out, flags, q, c);
}

int pprg_fifo_forward_push(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                           double r_max, double lambda_stop, double* reserve_out,
                           double* residue_out, uint32_t flags, pprg_query_stats* q,
                           pprg_call_stats* c) {
  if (!(r_max > 0.0)) {  // push.cpp:142
    t_err = "fifo_forward_push: r_max must be positive";
    return PPRG_EINVAL;
  }
  return push_engine(g, pprg::Engine::Fifo, sources, k, alpha, 0.0, 0, -1, r_max, lambda_stop,
                     reserve_out, residue_out, flags, q, c);
}

int pprg_run_traced(pprg_graph* g, int algo, uint32_t source, double alpha, double lambda,
                    double* estimates_out, pprg_query_stats* q, pprg_checkpoint* points,
                    uint32_t capacity, uint32_t* count) {
  return guard([&] {
    require(g && g->g && count, "null argument");
    require(algo >= PPRG_ALGO_POWITR && algo <= PPRG_ALGO_POWERPUSH, "unknown algorithm");
    check_alpha(alpha);
    require(lambda > 0.0 && lambda <= 1.0, "lambda must be in (0,1]");
    pprg::Graph& G = *g->g;
    pprg::TraceSink sink;
    sink.dev_t0 = pprg::device_now_ns(G);
    sink.host_t0 = pprg::host_now_ns();
    struct Reset {
      ~Reset() { pprg::g_trace = nullptr; }
    } reset;
    pprg::g_trace = &sink;
    std::vector<pprg::ColumnStats> cs(1);
    pprg::CallStats call;
    pprg::Outputs out{estimates_out, nullptr, false};
    // run_high_precision (sweep.cpp:50-61)
    switch (algo) {
      case PPRG_ALGO_POWITR:
        pprg::run_push_engine(G, pprg::Engine::PowItr, &source, 1, alpha, lambda, 0, -1, 0, 0, out,
                              cs.data(), &call);
        break;
      case PPRG_ALGO_SIMFWDPUSH:
        pprg::run_push_engine(G, pprg::Engine::SimFwdPush, &source, 1, alpha, lambda, 0, -1, 0, 0,
                              out, cs.data(), &call);
        break;
      case PPRG_ALGO_FIFO:
        pprg::run_push_engine(G, pprg::Engine::Fifo, &source, 1, alpha, 0.0, 0, -1,
                              lambda / static_cast<double>(G.m_eff()), 0.0, out, cs.data(), &call);
        break;
      default:
        pprg::run_push_engine(G, pprg::Engine::PowerPush, &source, 1, alpha, lambda, 8, -1, 0, 0,
                              out, cs.data(), &call);
    }
    pprg::g_trace = nullptr;
    const uint32_t n = (uint32_t)std::min<size_t>(sink.pts.size(), capacity);
    for (uint32_t i = 0; i < n && points; ++i) {
      points[i].pushes = sink.pts[i].pushes;
      points[i].r_sum = sink.pts[i].r_sum;
      points[i].time_ns = sink.pts[i].time_ns;
    }
    *count = n;
    fill_stats(cs, call, 1, q, nullptr);
  });
}

int pprg_run_observed(pprg_graph* g, int algo, uint32_t source, double alpha, double param,
                      double lambda_stop, uint32_t epoch_num, int64_t scan_threshold,
                      double* reserve_out, double* residue_out, pprg_query_stats* q,
                      pprg_step_callback cb, void* user) {
  return guard([&] {
    require(g && g->g && cb, "null argument");
    require(algo >= PPRG_ALGO_POWITR && algo <= PPRG_ALGO_POWERPUSH, "unknown algorithm");
    check_alpha(alpha);
    pprg::Graph& G = *g->g;
    if (algo == PPRG_ALGO_FIFO)
      require(param > 0.0, "fifo_forward_push: r_max must be positive");  // push.cpp:142
    else if (algo == PPRG_ALGO_POWERPUSH)
      require(param > 0.0 && param <= 1.0, "power_push: lambda must be in (0,1]");
    pprg::StepSink sink;
    sink.cb = cb;
    sink.user = user;
    struct Reset {
      ~Reset() { pprg::g_obs = nullptr; }
    } reset;
    pprg::g_obs = &sink;
    std::vector<pprg::ColumnStats> cs(1);
    pprg::CallStats call;
    pprg::Outputs out{reserve_out, residue_out, false};
    const pprg::Engine eng = algo == PPRG_ALGO_POWITR       ? pprg::Engine::PowItr
                             : algo == PPRG_ALGO_SIMFWDPUSH ? pprg::Engine::SimFwdPush
                             : algo == PPRG_ALGO_FIFO       ? pprg::Engine::Fifo
                                                            : pprg::Engine::PowerPush;
    pprg::run_push_engine(G, eng, &source, 1, alpha, eng == pprg::Engine::Fifo ? 0.0 : param,
                          epoch_num ? epoch_num : 8, scan_threshold,
                          eng == pprg::Engine::Fifo ? param : 0.0,
                          lambda_stop > 0.0 ? lambda_stop : 0.0, out, cs.data(), &call);
    fill_stats(cs, call, 1, q, nullptr);
  });
}

int pprg_ground_truth(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                      double* estimates_out, uint32_t flags, pprg_query_stats* q,
                      pprg_call_stats* c) {
  return guard([&] {
    if (flags & PPRG_DETERMINISTIC) pprg::t_det = true;
    require(g && g->g, "null graph");
    require(k == 0 || (sources && estimates_out), "null argument");
    check_alpha(alpha);
    pprg::Graph& G = *g->g;
    const bool dev = (flags & PPRG_OUT_DEVICE) != 0;
    // kGroundTruthLambda = 1e-17 (metrics.hpp:10), the double-precision limit.
    // Power iteration keeps the residues explicit (no cancellation against
    // x), stops at r_sum <= 1e-17 (push.cpp:81-108) and is deterministic:
    // fixed-order row sums, hub rows combined in piece order.
    std::vector<pprg::ColumnStats> cs(k);
    pprg::CallStats call;
    if (k)
      pprg::run_push_engine(G, pprg::Engine::PowItr, sources, k, alpha, 1e-17, 0, -1, 0.0, 0.0,
                            pprg::Outputs{estimates_out, nullptr, dev}, cs.data(), &call);
    if (k && G.n <= 2000) {
      // metrics.cpp:48-53 cross-checks small graphs against the dense solve;
      // here an independent engine (FIFO push to lambda = 1e-14) plays that
      // role, with the reference's 1e-12 l1 bound.
      const uint64_t n = G.n;
      std::vector<double> chk(n * k), got(n * k);
      std::vector<pprg::ColumnStats> cs2(k);
      pprg::CallStats call2;
      const double r_max = 1e-14 / static_cast<double>(G.m_eff());
      pprg::run_push_engine(G, pprg::Engine::Fifo, sources, k, alpha, 0.0, 0, -1, r_max, 0.0,
                            pprg::Outputs{chk.data(), nullptr, false}, cs2.data(), &call2);
      if (dev)
        PPRG_CUDA(cudaMemcpy(got.data(), estimates_out, 8 * n * k, cudaMemcpyDeviceToHost));
      else
        std::memcpy(got.data(), estimates_out, 8 * n * k);
      for (uint32_t i = 0; i < k; ++i) {
        double l1 = 0.0;
        for (uint64_t v = 0; v < n; ++v) l1 += std::fabs(got[i * n + v] - chk[i * n + v]);
        if (l1 > 1e-12) pprg::fail(pprg::EINTERNAL, "ground_truth: disagrees with the dense solve");
      }
      call.kernel_launches += call2.kernel_launches;
    }
    fill_stats(cs, call, k, q, c);
  });
}

int pprg_power_push(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha,
                    double lambda, uint32_t epoch_num, int64_t scan_threshold,
                    double* reserve_out, double* residue_out, uint32_t flags,
                    pprg_query_stats* q, pprg_call_stats* c, double* epoch_r_max_out) {
  if (!(lambda > 0.0 && lambda <= 1.0)) {  // push.cpp:154-155
    t_err = "power_push: lambda must be in (0,1]";
    return PPRG_EINVAL;
  }
  if (epoch_num == 0) {  // types.hpp:45
    t_err = "epoch_num must be positive";
    return PPRG_EINVAL;
  }
  const int rc = push_engine(g, pprg::Engine::PowerPush, sources, k, alpha, lambda, epoch_num,
                             scan_threshold, 0, 0, reserve_out, residue_out, flags, q, c);
  if (rc == PPRG_OK && epoch_r_max_out) {
    const double m_eff = (double)g->g->m_eff();
    for (uint32_t e = 1; e <= epoch_num; ++e)
      epoch_r_max_out[e - 1] = std::pow(lambda, static_cast<double>(e) / epoch_num) / m_eff;
  }
  return rc;
}

static_assert(sizeof(pprg_column_state) == sizeof(pprg::ColInit), "column state layout");

int pprg_epoch_init(pprg_column_state* cols, uint32_t columns, const double* sum_x,
                    const double* sum_dead_x, const double* epoch_lambda, uint32_t epoch_num,
                    double alpha, int* need_sweeps) {
  return guard([&] {
    require(cols && sum_x && sum_dead_x && epoch_lambda && need_sweeps, "epoch: null argument");
    require(columns >= 1 && columns <= 64 && epoch_num >= 1 && epoch_num <= 64, "epoch: bad sizes");
    *need_sweeps = pprg::epoch_init(reinterpret_cast<pprg::ColInit*>(cols), (int)columns, sum_x,
                                    sum_dead_x, epoch_lambda, epoch_num, alpha);
  });
}

int pprg_epoch_advance(pprg_column_state* cols, uint32_t columns, const double* summed,
                       const double* epoch_lambda, uint32_t epoch_num, double alpha, int* done) {
  return guard([&] {
    require(cols && summed && epoch_lambda && done, "epoch: null argument");
    require(columns >= 1 && columns <= 64 && epoch_num >= 1 && epoch_num <= 64, "epoch: bad sizes");
    *done = pprg::epoch_advance(reinterpret_cast<pprg::ColInit*>(cols), (int)columns, summed,
                                epoch_lambda, epoch_num, alpha);
  });
}

int pprg_part_begin(pprg_graph* g, uint32_t nparts, uint32_t part, const uint32_t* sources,
                    uint32_t k, double alpha, double lambda, uint32_t epoch_num,
                    int64_t scan_threshold, double* partial_sums, uint64_t* node_lo,
                    uint64_t* node_hi, pprg_part** out) {
  return guard([&] {
    require(g && sources && partial_sums && node_lo && node_hi && out, "partition: null argument");
    auto h = new pprg_part;
    try {
      h->s = pprg::part_begin(*g->g, nparts, part, sources, k, alpha, lambda, epoch_num,
                              scan_threshold, partial_sums, node_lo, node_hi);
    } catch (...) {
      delete h;
      throw;
    }
    h->owner = g;
    h->k = k;
    *out = h;
  });
}

int pprg_part_start(pprg_part* p, const double* summed, int* need_sweeps) {
  return guard([&] {
    require(p && summed && need_sweeps, "partition: null argument");
    *need_sweeps = pprg::part_start(p->s, summed) ? 1 : 0;
  });
}

int pprg_part_buffers(pprg_part* p, double** y, uint32_t* columns, double** counters) {
  return guard([&] {
    require(p && y && columns && counters, "partition: null argument");
    *y = pprg::part_y(p->s, columns);
    *counters = pprg::part_counters(p->s);
  });
}

int pprg_part_local_x(pprg_part* p, double** x) {
  return guard([&] {
    require(p && x, "partition: null argument");
    *x = pprg::part_x(p->s);
  });
}

int pprg_part_resum(pprg_part* p, double* partial_sums) {
  return guard([&] {
    require(p && partial_sums, "partition: null argument");
    pprg::part_resum(p->s, partial_sums);
  });
}

int pprg_part_sweep(pprg_part* p, double* local_counters) {
  return guard([&] {
    require(p != nullptr, "partition: null argument");
    pprg::part_sweep(p->s, local_counters);
  });
}

int pprg_part_advance(pprg_part* p, const double* summed, int* done) {
  return guard([&] {
    require(p && summed && done, "partition: null argument");
    *done = pprg::part_advance(p->s, summed) ? 1 : 0;
  });
}

int pprg_part_finish(pprg_part* p, double* reserve_out, double* residue_out, uint32_t flags,
                     double* residue_sums) {
  return guard([&] {
    require(p && residue_sums, "partition: null argument");
    pprg::part_finish(p->s, reserve_out, residue_out, (flags & PPRG_OUT_DEVICE) != 0, residue_sums);
  });
}

int pprg_part_stats(const pprg_part* p, pprg_query_stats* q, pprg_call_stats* c) {
  return guard([&] {
    require(p != nullptr, "partition: null argument");
    std::vector<pprg::ColumnStats> cs(p->k);
    pprg::CallStats call;
    pprg::part_stats(p->s, cs.data(), &call);
    fill_stats(cs, call, p->k, q, c);
  });
}

int pprg_part_set_peers(pprg_part* p, double* const* peer_y, uint32_t npeers) {
  return guard([&] {
    require(p && (npeers == 0 || peer_y), "partition: null argument");
    pprg::part_set_peers(p->s, peer_y, npeers);
  });
}

int pprg_part_ipc_handle(pprg_part* p, void* handle) {
  return guard([&] {
    require(p && handle, "partition: null argument");
    pprg::DeviceGuard dg(pprg::part_device(p->s));
    uint32_t cols = 0;
    cudaIpcMemHandle_t h;
    PPRG_CUDA(cudaIpcGetMemHandle(&h, pprg::part_y(p->s, &cols)));
    std::memcpy(handle, &h, sizeof h);
  });
}

int pprg_ipc_open(int device, const void* handle, void** ptr) {
  return guard([&] {
    require(handle && ptr, "ipc: null argument");
    pprg::DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    PPRG_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int pprg_ipc_close(int device, void* ptr) {
  return guard([&] {
    pprg::DeviceGuard dg(device);
    PPRG_CUDA(cudaIpcCloseMemHandle(ptr));
  });
}

void pprg_part_destroy(pprg_part* p) {
  if (!p) return;
  pprg::part_destroy(p->s);
  delete p;
}

int pprg_refine(pprg_graph* g, const uint32_t* sources, uint32_t k, double alpha, double r_max,
                double* reserve_inout, double* residue_inout, uint32_t flags,
                pprg_query_stats* q, pprg_call_stats* c) {
  return guard([&] {
    if (flags & PPRG_DETERMINISTIC) pprg::t_det = true;
    require(g && g->g, "null graph");
    require(k == 0 || (sources && reserve_inout && residue_inout), "null argument");
    check_alpha(alpha);
    std::vector<pprg::ColumnStats> cs(k);
    pprg::CallStats call;
    if (k)
      pprg::refine_state(*g->g, sources, k, alpha, r_max, reserve_inout, residue_inout,
                         (flags & PPRG_OUT_DEVICE) != 0, cs.data(), &call);
    fill_stats(cs, call, k, q, c);
  });
}

int pprg_block_columns(const pprg_graph* g, uint32_t k, uint32_t* out) {
  return guard([&] {
    require(g != nullptr && out != nullptr, "block columns: null argument");
    *out = pprg::block_width(g->g->n, k);
  });
}

int pprg_uses_delta_sweeps(const pprg_graph* g, uint32_t k, int* out) {
  return guard([&] {
    require(g != nullptr && out != nullptr, "delta sweeps: null argument");
    *out = pprg::delta_block(*g->g, k) ? 1 : 0;
  });
}

int pprg_walk_budget(uint64_t n, double epsilon, double mu, uint64_t* out) {
  return guard([&] {
    // walk_budget_real, speedppr.cpp:8-14 (same checks)
    require(n >= 2, "walk budget: need n >= 2");
    require(epsilon > 0.0, "walk budget: epsilon must be positive");
    require(mu > 0.0 && mu <= 1.0, "walk budget: mu must be in (0,1]");
    *out = static_cast<uint64_t>(std::ceil(2.0 * (2.0 * epsilon / 3.0 + 2.0) *
                                           std::log(static_cast<double>(n)) /
                                           (epsilon * epsilon * mu)));
  });
}

int pprg_index_build(pprg_graph* g, double alpha, uint64_t seed, pprg_index** out) {
  return guard([&] {
    require(g && g->g && out, "null argument");
    check_alpha(alpha);
    auto h = new pprg_index;
    h->owner = g;
    try {
      h->w = pprg::index_build(*g->g, alpha, seed);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pprg_index_load(pprg_graph* g, const char* path, pprg_index** out) {
  return guard([&] {
    require(g && g->g && path && out, "null argument");
    auto h = new pprg_index;
    h->owner = g;
    try {
      h->w = pprg::index_load(*g->g, path);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pprg_index_save(const pprg_index* idx, const char* path) {
  return guard([&] {
    require(idx && idx->w && idx->owner && path, "null argument");
    pprg::index_save(*idx->owner->g, *idx->w, path);
  });
}

int pprg_index_from_host(pprg_graph* g, double alpha, uint64_t seed, const uint32_t* endpoints,
                         pprg_index** out) {
  return guard([&] {
    require(g && g->g && out && (endpoints || g->g->m == 0), "null argument");
    auto h = new pprg_index;
    h->owner = g;
    try {
      h->w = pprg::index_from_host(*g->g, alpha, seed, endpoints);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pprg_index_export(const pprg_index* idx, uint32_t* endpoints) {
  return guard([&] {
    require(idx && idx->w && endpoints, "null argument");
    pprg::DeviceGuard dg(idx->w->device);
    if (idx->w->m)
      PPRG_CUDA(cudaMemcpy(endpoints, idx->w->endpoints.get(), 4 * idx->w->m, cudaMemcpyDeviceToHost));
  });
}

void pprg_index_destroy(pprg_index* idx) {
  if (!idx) return;
  try {
    pprg::DeviceGuard dg(idx->w ? idx->w->device : 0);
    idx->w.reset();
  } catch (...) {
  }
  delete idx;
}

int pprg_speedppr(pprg_graph* g, const pprg_index* idx, const uint32_t* sources, uint32_t k,
                  double alpha, double epsilon, double mu, uint64_t seed, double* estimates_out,
                  uint32_t flags, pprg_query_stats* q, pprg_call_stats* c) {
  return guard([&] {
    if (flags & PPRG_DETERMINISTIC) pprg::t_det = true;
    require(g && g->g, "null graph");
    require(k == 0 || sources, "null sources");
    // QueryConfig::validate + speedppr.cpp:76-83
    require(epsilon > 0.0, "epsilon must be positive");
    require(!(mu > 0.0) || mu <= 1.0, "mu must be in (0,1]");
    check_alpha(alpha);
    if (idx) {
      if (idx->w->m != g->g->m || idx->owner->g->n != g->g->n)
        pprg::fail(PPRG_EDATA, "walk index does not match the graph shape");
      if (idx->w->alpha != alpha) pprg::fail(PPRG_EDATA, "walk index was built for a different alpha");
    }
    std::vector<pprg::ColumnStats> cs(k);
    pprg::CallStats call;
    if (k)
      pprg::speedppr(*g->g, idx ? idx->w.get() : nullptr, sources, k, alpha, epsilon, mu, seed,
                     estimates_out, (flags & PPRG_OUT_DEVICE) != 0, cs.data(), &call);
    fill_stats(cs, call, k, q, c);
  });
}

int pprg_monte_carlo(pprg_graph* g, const pprg_index* idx, uint32_t source, double alpha,
                     uint64_t walk_budget, uint64_t seed, const double* reserve,
                     const double* residue, double* estimates_out, uint64_t* walks_out) {
  return guard([&] {
    require(g && g->g && reserve && residue && estimates_out && walks_out, "null argument");
    check_alpha(alpha);
    require(walk_budget >= 1, "monte carlo: walk budget must be positive");
    if (idx) {  // walk_index.cpp:36-42, speedppr.cpp:62-64
      if (idx->owner != g && (idx->w->m != g->g->m || idx->owner->g->n != g->g->n))
        pprg::fail(pprg::EDATA, "walk index does not match the graph shape");
      if (idx->w->alpha != alpha) pprg::fail(pprg::EDATA, "walk index was built for a different alpha");
    }
    pprg::monte_carlo(*g->g, idx ? idx->w.get() : nullptr, source, alpha, walk_budget, seed,
                      reserve, residue, estimates_out, walks_out);
  });
}

int pprg_walk_terminals(pprg_graph* g, const uint32_t* starts, const uint32_t* ks,
                        const uint32_t* vs, uint64_t count, uint32_t source, uint32_t tag,
                        double alpha, uint64_t seed, uint32_t* out) {
  return guard([&] {
    require(g && g->g && out, "null argument");
    pprg::walk_terminals(*g->g, starts, ks, vs, count, source, tag, alpha, seed, out);
  });
}

int pprg_graph_sync(pprg_graph* g) {
  return guard([&] {
    require(g && g->g, "null graph");
    pprg::graph_sync(*g->g);
  });
}

int pprg_device_alloc(int device, uint64_t bytes, void** out) {
  return guard([&] {
    pprg::DeviceGuard dg(device);
    PPRG_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  });
}

int pprg_host_alloc(uint64_t bytes, void** out) {
  return guard([&] {
    require(out != nullptr, "null argument");
    PPRG_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}

int pprg_host_free(void* p) {
  return guard([&] { PPRG_CUDA(cudaFreeHost(p)); });
}

int pprg_device_free(int device, void* p) {
  return guard([&] {
    pprg::DeviceGuard dg(device);
    PPRG_CUDA(cudaFree(p));
  });
}

}  // extern "C"
