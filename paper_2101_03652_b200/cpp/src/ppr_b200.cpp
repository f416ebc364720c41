// C++ drop-in of the reference's ppr:: core API over the engine's C ABI
// (include/pprg.h). Every engine call runs on the GPU; status codes come back
// as the reference's exception types (invalid_argument / runtime_error /
// logic_error).
#include <algorithm>
#include <bit>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <string_view>

#include "../../../include/pprg.h"
#include "ppr/csv.hpp"
#include "ppr/exact_ppr.hpp"
#include "ppr/graph.hpp"
#include "ppr/metrics.hpp"
#include "ppr/push.hpp"
#include "ppr/speedppr.hpp"
#include "ppr/sweep.hpp"
#include "ppr/synthetic.hpp"
#include "ppr/walk_index.hpp"

namespace ppr {

// ---- rng.hpp ----------------------------------------------------------------
std::uint64_t Rng::below(std::uint64_t bound) {
  using u128 = unsigned __int128;
  u128 prod = static_cast<u128>(next()) * bound;
  auto low = static_cast<std::uint64_t>(prod);
  if (low < bound) {
    const std::uint64_t reject_below = (0 - bound) % bound;  // 2^64 mod bound
    while (low < reject_below) {
      prod = static_cast<u128>(next()) * bound;
      low = static_cast<std::uint64_t>(prod);
    }
  }
  return static_cast<std::uint64_t>(prod >> 64);
}

// ---- push.hpp host containers -------------------------------------------------
FifoQueue::FifoQueue(std::size_t n) : slots_(n + 1) {}
bool FifoQueue::empty() const { return first_ == last_; }
std::size_t FifoQueue::size() const {
  return last_ >= first_ ? last_ - first_ : slots_.size() - (first_ - last_);
}
void FifoQueue::push(NodeId v) {
  slots_[last_] = v;
  if (++last_ == slots_.size()) last_ = 0;
}
NodeId FifoQueue::pop() {
  const NodeId v = slots_[first_];
  if (++first_ == slots_.size()) first_ = 0;
  return v;
}
void FifoQueue::clear() { first_ = last_ = 0; }

PushState::PushState(NodeId n, NodeId s)
    : reserve(n, 0.0), residue(n, 0.0), r_sum(1.0), in_queue(n, 0), queue(n) {
  residue[s] = 1.0;
}

// ---- types.hpp (reference types.hpp:17-53) -----------------------------------
double default_lambda(EdgeId m) { return std::min(1.0 / static_cast<double>(m), 1e-8); }
double default_mu(NodeId n) { return 1.0 / static_cast<double>(n); }
std::uint64_t default_scan_threshold(NodeId n) { return n / 4; }

void QueryConfig::validate() const {
  auto bad = [](const char* what) { throw std::invalid_argument(what); };
  if (!(alpha >= 0.0 && alpha < 1.0)) bad("alpha must be in [0,1)");
  if (lambda && !(*lambda > 0.0 && *lambda <= 1.0)) bad("lambda must be in (0,1]");
  if (epsilon && !(*epsilon > 0.0)) bad("epsilon must be positive");
  if (mu && !(*mu > 0.0 && *mu <= 1.0)) bad("mu must be in (0,1]");
  if (epoch_num == 0) bad("epoch_num must be positive");
}
double QueryConfig::lambda_for(EdgeId m) const { return lambda.value_or(default_lambda(m)); }
double QueryConfig::mu_for(NodeId n) const { return mu.value_or(default_mu(n)); }
std::uint64_t QueryConfig::scan_threshold_for(NodeId n) const {
  return scan_threshold.value_or(default_scan_threshold(n));
}
namespace {

// The reference is a deterministic library (SPEC.md: identical inputs give
// identical results), so its drop-in runs the engine in PPRG_DETERMINISTIC
// mode; PPRG_FAST=1 selects the faster nondeterministic sweeps instead.
const int g_det_init = [] {
  pprg_set_deterministic(std::getenv("PPRG_FAST") ? 0 : 1);
  return 0;
}();

void check(int rc) {
  if (rc == PPRG_OK) return;
  const std::string msg = pprg_last_error();
  if (rc == PPRG_EINVAL) throw std::invalid_argument(msg);
  if (rc == PPRG_EDATA) throw std::runtime_error(msg);
  if (rc == PPRG_EINTERNAL) throw std::logic_error(msg);
  throw std::runtime_error("device error: " + msg);
}

int device_from_env() {
  if (const char* e = std::getenv("PPRG_DEVICE")) return std::atoi(e);
  return 0;
}

PPRVector make_vector(NodeId n, NodeId s, double alpha) {
  PPRVector v;
  v.estimates.assign(n, 0.0);
  v.residues.assign(n, 0.0);
  v.source = s;
  v.alpha = alpha;
  return v;
}

void notify(PushObserver* obs, const PPRVector& v, std::uint32_t iterations) {
  if (!obs) return;
  PushState st(static_cast<NodeId>(v.estimates.size()), v.source);
  st.reserve = v.estimates;
  st.residue = v.residues;
  st.r_sum = v.achieved_r_sum;
  st.edge_push_count = v.pushes;
  obs->on_push(st);
  obs->on_iteration(st, iterations);
}

// With an observer: run the query observed (pprg_run_observed); after every
// frontier level / global sweep / iteration the library hands over the full
// reserve and residue, mirrored into a PushState for on_push / on_iteration
// (step granularity, never per push).
struct ObsCtx {
  PushObserver* obs;
  PushState* st;
};

void step_cb(void* user, const double* reserve, const double* residue, double r_sum,
             std::uint64_t pushes, std::uint32_t step) {
  auto* c = static_cast<ObsCtx*>(user);
  const std::size_t n = c->st->reserve.size();
  std::copy(reserve, reserve + n, c->st->reserve.begin());
  std::copy(residue, residue + n, c->st->residue.begin());
  c->st->r_sum = r_sum;
  c->st->edge_push_count = pushes;
  c->obs->on_push(*c->st);
  c->obs->on_iteration(*c->st, step);
}

bool observed(const Graph& g, int algo, NodeId s, double alpha, double param, double lambda_stop,
              std::uint32_t epochs, std::int64_t scan, PushObserver* obs, PPRVector& v,
              pprg_query_stats* qout = nullptr) {
  if (!obs) return false;
  PushState st(g.n(), s);
  ObsCtx ctx{obs, &st};
  pprg_query_stats q{};
  check(pprg_run_observed(g.device_handle(), algo, s, alpha, param, lambda_stop, epochs, scan,
                          v.estimates.data(), v.residues.data(), &q, step_cb, &ctx));
  v.achieved_r_sum = q.achieved_r_sum;
  v.pushes = q.pushes;
  if (qout) *qout = q;
  return true;
}

}  // namespace

// ---- graph.hpp ---------------------------------------------------------------
Graph::Graph(std::vector<std::uint64_t> out_offsets, std::vector<NodeId> out_neighbors)
    : off_(std::move(out_offsets)), nbr_(std::move(out_neighbors)) {
  if (off_.empty()) throw std::runtime_error("graph: offsets array must have length n+1");
  n_ = static_cast<NodeId>(off_.size() - 1);
  m_ = nbr_.size();
  if (off_.back() != m_) throw std::runtime_error("graph: offsets must end at m");
  pprg_graph* h = nullptr;
  check(pprg_graph_create(off_.data(), nbr_.data(), n_, device_from_env(), &h));
  dev_.reset(h, pprg_graph_destroy);
  for (NodeId v = 0; v < n_; ++v)
    if (is_dead_end(v)) dead_.push_back(v);
}

void Graph::validate() const {  // the device validated at construction (graph.cpp:24-34)
  if (off_[0] != 0) throw std::runtime_error("graph: offsets must start at 0");
}

Graph Graph::adopt(pprg_graph* h) {
  Graph g;
  g.dev_.reset(h, pprg_graph_destroy);
  std::uint64_t n = 0, m = 0, nd = 0;
  check(pprg_graph_info(h, &n, &m, &nd));
  g.n_ = static_cast<NodeId>(n);
  g.m_ = m;
  g.off_.resize(n + 1);
  g.nbr_.resize(m);
  g.dead_.resize(nd);
  check(pprg_graph_export(h, g.off_.data(), g.nbr_.data(), g.dead_.data()));
  return g;
}

namespace {
// Pairs -> the flat (u, v) u64 array the device builder takes; the sort,
// relabel and stable scatter of graph.cpp:36-63 run on the GPU.
Graph build_on_device(const std::uint64_t* flat, std::size_t pairs) {
  if (pairs == 0) throw std::runtime_error("graph is empty after cleaning");
  pprg_graph* h = nullptr;
  check(pprg_graph_build_from_edges(flat, pairs, device_from_env(), &h));
  return Graph::adopt(h);
}
}  // namespace

Graph build_graph_from_edges(const std::vector<std::pair<std::uint64_t, std::uint64_t>>& edges) {
  static_assert(sizeof(std::pair<std::uint64_t, std::uint64_t>) == 16);
  return build_on_device(reinterpret_cast<const std::uint64_t*>(edges.data()), edges.size());
}

// PPRG files (graph.cpp:115-149 format: "PPRG", u8 version 1, n, m, offsets,
// neighbours, little endian) are read and written by the engine straight
// between the file and device memory through pinned staging buffers
// (pprg_graph_load_cache / pprg_graph_save_cache), with the reference's checks
// and messages; the host copies are then exported from the device.
void save_graph_cache(const Graph& g, const std::string& path) {
  check(pprg_graph_save_cache(g.device_handle(), path.c_str()));
}

Graph load_graph_cache(const std::string& path) {
  pprg_graph* h = nullptr;
  check(pprg_graph_load_cache(path.c_str(), device_from_env(), &h));
  return Graph::adopt(h);
}

bool is_graph_cache(const std::string& path) {
  char head[4] = {};
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  const std::size_t got = std::fread(head, 1, 4, f);
  std::fclose(f);
  return got == 4 && std::string_view(head, 4) == "PPRG";
}

// ---- push.hpp ----------------------------------------------------------------
PPRVector power_iteration(const Graph& g, NodeId s, double alpha, double lambda,
                          PushObserver* observer) {
  PPRVector v = make_vector(g.n(), s, alpha);
  pprg_query_stats q{};
  if (observed(g, PPRG_ALGO_POWITR, s, alpha, lambda, 0.0, 0, -1, observer, v)) return v;
  check(pprg_power_iteration(g.device_handle(), &s, 1, alpha, lambda, v.estimates.data(),
                             v.residues.data(), 0, &q, nullptr));
  v.achieved_r_sum = q.achieved_r_sum;
  v.pushes = q.pushes;
  notify(observer, v, q.sweeps);
  return v;
}

PPRVector sim_forward_push(const Graph& g, NodeId s, double alpha, double lambda,
                           PushObserver* observer) {
  PPRVector v = make_vector(g.n(), s, alpha);
  pprg_query_stats q{};
  if (observed(g, PPRG_ALGO_SIMFWDPUSH, s, alpha, lambda, 0.0, 0, -1, observer, v)) return v;
  check(pprg_sim_forward_push(g.device_handle(), &s, 1, alpha, lambda, v.estimates.data(),
                              v.residues.data(), 0, &q, nullptr));
  v.achieved_r_sum = q.achieved_r_sum;
  v.pushes = q.pushes;
  notify(observer, v, q.sweeps);
  return v;
}

PPRVector fifo_forward_push(const Graph& g, NodeId s, double alpha, double r_max,
                            std::optional<double> lambda_stop, PushObserver* observer) {
  PPRVector v = make_vector(g.n(), s, alpha);
  pprg_query_stats q{};
  if (observed(g, PPRG_ALGO_FIFO, s, alpha, r_max, lambda_stop ? *lambda_stop : -1.0, 0, -1,
               observer, v))
    return v;
  check(pprg_fifo_forward_push(g.device_handle(), &s, 1, alpha, r_max,
                               lambda_stop ? *lambda_stop : -1.0, v.estimates.data(),
                               v.residues.data(), 0, &q, nullptr));
  v.achieved_r_sum = q.achieved_r_sum;
  v.pushes = q.pushes;
  notify(observer, v, q.local_levels);
  return v;
}

PPRVector power_push(const Graph& g, NodeId s, double alpha, double lambda,
                     const QueryConfig& cfg, PushObserver* observer, PowerPushTrace* trace) {
  PPRVector v = make_vector(g.n(), s, alpha);
  pprg_query_stats q{};
  if (observer) {
    if (!(lambda > 0.0 && lambda <= 1.0))
      throw std::invalid_argument("power_push: lambda must be in (0,1]");  // push.cpp:154-155
    observed(g, PPRG_ALGO_POWERPUSH, s, alpha, lambda, 0.0, cfg.epoch_num,
             cfg.scan_threshold ? static_cast<int64_t>(*cfg.scan_threshold) : -1, observer, v, &q);
    if (trace) {  // push.cpp:168-180
      trace->used_scan_phase = q.used_scan_phase != 0;
      trace->epoch_r_max.clear();
      const double m_eff = static_cast<double>(g.effective_edge_count());
      if (trace->used_scan_phase)
        for (std::uint32_t e = 1; e <= cfg.epoch_num; ++e)
          trace->epoch_r_max.push_back(std::pow(lambda, static_cast<double>(e) / cfg.epoch_num) / m_eff);
    }
    return v;
  }
  std::vector<double> eps(cfg.epoch_num);
  check(pprg_power_push(g.device_handle(), &s, 1, alpha, lambda, cfg.epoch_num,
                        cfg.scan_threshold ? static_cast<int64_t>(*cfg.scan_threshold) : -1,
                        v.estimates.data(), v.residues.data(), 0, &q, nullptr, eps.data()));
  v.achieved_r_sum = q.achieved_r_sum;
  v.pushes = q.pushes;
  if (trace) {
    trace->used_scan_phase = q.used_scan_phase != 0;
    trace->epoch_r_max = q.used_scan_phase ? eps : std::vector<double>{};
  }
  notify(observer, v, q.sweeps);
  return v;
}

std::vector<PPRVector> power_push_batch(const Graph& g, const std::vector<NodeId>& sources,
                                        double alpha, double lambda, const QueryConfig& cfg) {
  const std::size_t k = sources.size(), n = g.n();
  std::vector<double> res(k * n), rsd(k * n);
  std::vector<pprg_query_stats> q(k);
  check(pprg_power_push(g.device_handle(), sources.data(), static_cast<uint32_t>(k), alpha, lambda,
                        cfg.epoch_num,
                        cfg.scan_threshold ? static_cast<int64_t>(*cfg.scan_threshold) : -1,
                        res.data(), rsd.data(), 0, q.data(), nullptr, nullptr));
  std::vector<PPRVector> out(k);
  for (std::size_t i = 0; i < k; ++i) {
    out[i].estimates.assign(res.begin() + i * n, res.begin() + (i + 1) * n);
    out[i].residues.assign(rsd.begin() + i * n, rsd.begin() + (i + 1) * n);
    out[i].source = sources[i];
    out[i].alpha = alpha;
    out[i].achieved_r_sum = q[i].achieved_r_sum;
    out[i].pushes = q[i].pushes;
  }
  return out;
}

// ---- walk_index.hpp / speedppr.hpp -------------------------------------------
void WalkIndex::check_compatible(const Graph& g) const {  // walk_index.cpp:36-42 (same checks, messages)
  const bool shape_ok = node_count() == g.n() && endpoint_count() == g.m();
  if (!shape_ok) throw std::runtime_error("walk index does not match the graph shape");
  // the slices follow the graph's own offsets once the shapes agree, so a
  // slice / degree mismatch is one node whose stored slice length differs
  NodeId v = 0;
  while (v < g.n() && endpoints_of(v).size() == g.out_degree(v)) ++v;
  if (v != g.n()) throw std::runtime_error("walk index slice length differs from out-degree");
}

WalkIndex build_index(const Graph& g, double alpha, std::uint64_t seed) {
  pprg_index* h = nullptr;
  check(pprg_index_build(g.device_handle(), alpha, seed, &h));
  WalkIndex w;
  w.dev_.reset(h, pprg_index_destroy);
  w.dev_graph_ = g.device_handle();
  w.alpha_ = alpha;
  w.seed_ = seed;
  w.offsets_ = g.out_offsets();
  w.endpoints_.resize(g.m());
  if (g.m()) check(pprg_index_export(h, w.endpoints_.data()));
  return w;
}

// PPRW files (walk_index.hpp:52-56 format: "PPRW", u8 version 1, u8 rng id,
// f64 alpha, u64 seed, n, m, offsets (n+1) x u64, endpoints m x u32; little
// endian). An index with a device copy is written by the engine straight from
// device memory (pprg_index_save); otherwise, and for loads without a graph,
// the arrays move in bulk through stdio.
namespace {
static_assert(std::endian::native == std::endian::little, "PPRW/PPRG files are little endian");

struct File {
  std::FILE* f;
  std::string path;
  File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)), path(p) {}
  ~File() {
    if (f) std::fclose(f);
  }
  bool get(void* dst, std::size_t bytes) { return std::fread(dst, 1, bytes, f) == bytes; }
  bool put(const void* src, std::size_t bytes) { return std::fwrite(src, 1, bytes, f) == bytes; }
};
}  // namespace

void save_index(const WalkIndex& index, const std::string& path) {
  if (index.dev_) {
    check(pprg_index_save(index.dev_.get(), path.c_str()));
    return;
  }
  File out(path, "wb");
  if (!out.f) throw std::runtime_error("cannot open for writing: " + path);
  const std::uint8_t head[2] = {1, static_cast<std::uint8_t>(index.rng_id())};
  const double alpha = index.alpha();
  const std::uint64_t fields[3] = {index.seed(), index.node_count(), index.endpoint_count()};
  bool ok = out.put("PPRW", 4) && out.put(head, 2) && out.put(&alpha, 8) && out.put(fields, 24) &&
            out.put(index.offsets_.data(), 8 * index.offsets_.size()) &&
            out.put(index.endpoints_.data(), 4 * index.endpoints_.size());
  ok = (std::fflush(out.f) == 0) && ok;
  if (!ok) throw std::runtime_error("write failed: " + path);
}

WalkIndex load_index(const std::string& path) {
  File in(path, "rb");
  if (!in.f) throw std::runtime_error("cannot open walk index: " + path);
  char magic[4];
  std::uint8_t head[2] = {};
  if (!in.get(magic, 4) || std::string_view(magic, 4) != "PPRW")
    throw std::runtime_error(path + ": not a walk index (bad magic)");
  if (!in.get(head, 2) || head[0] != 1)
    throw std::runtime_error(path + ": unsupported walk index version");
  if (head[1] != kRngIdPhilox4x32_10) throw std::runtime_error(path + ": unknown generator id");
  double alpha = 0.0;
  std::uint64_t fields[3] = {};  // seed, n, m
  WalkIndex w;
  bool ok = in.get(&alpha, 8) && in.get(fields, 24);
  if (ok) {
    w.offsets_.resize(fields[1] + 1);
    w.endpoints_.resize(fields[2]);
    ok = in.get(w.offsets_.data(), 8 * w.offsets_.size()) &&
         in.get(w.endpoints_.data(), 4 * w.endpoints_.size());
  }
  if (!ok) throw std::runtime_error(path + ": truncated walk index");
  w.alpha_ = alpha;
  w.seed_ = fields[0];
  // the WalkIndex constructor's checks (walk_index.cpp:19-34 semantics)
  const auto& off = w.offsets_;
  if (off.front() != 0 || off.back() != fields[2])
    throw std::runtime_error("walk index: inconsistent offsets");
  if (!std::is_sorted(off.begin(), off.end()))
    throw std::runtime_error("walk index: offsets must be non-decreasing");
  if (std::any_of(w.endpoints_.begin(), w.endpoints_.end(),
                  [&](NodeId e) { return e >= fields[1]; }))
    throw std::runtime_error("walk index: endpoint id out of range");
  return w;
}

WalkIndex load_index(const std::string& path, const Graph& g) {
  WalkIndex w = load_index(path);
  (void)w.device_handle(g);
  return w;
}

pprg_index* WalkIndex::device_handle(const Graph& g) const {
  if (dev_ && dev_graph_ == g.device_handle()) return dev_.get();
  check_compatible(g);
  pprg_index* h = nullptr;
  check(pprg_index_from_host(g.device_handle(), alpha_, seed_, endpoints_.data(), &h));
  dev_.reset(h, pprg_index_destroy);
  dev_graph_ = g.device_handle();
  return h;
}

NodeId random_walk(const Graph& g, NodeId start, NodeId source, double alpha, Rng& rng) {
  NodeId at = start;
  while (rng.uniform01() >= alpha) {
    const auto out = effective_out(g, at, source);
    at = out[rng.below(out.degree())];
  }
  return at;
}

void push_once(PushState& st, NodeId v, const Graph& g, NodeId s, double alpha) {
  const double r = st.residue[v];
  if (r <= 0.0) return;
  st.reserve[v] += alpha * r;
  st.residue[v] = 0.0;  // zeroed before the spread: a self-loop keeps its share
  const auto out = effective_out(g, v, s);
  const double share = (1.0 - alpha) * r / static_cast<double>(out.degree());
  for (NodeId u : out) st.residue[u] += share;
  st.r_sum -= alpha * r;
  st.edge_push_count += out.degree();
}

double walk_budget_real(std::uint64_t n, double epsilon, double mu) {  // speedppr.cpp:8-14
  // W = 2 (2 eps / 3 + 2) ln(n) / (eps^2 mu), the paper's Chernoff budget;
  // argument checks in the reference's order and with its messages
  const struct {
    bool bad;
    const char* msg;
  } checks[] = {{n < 2, "walk budget: need n >= 2"},
                {!(epsilon > 0.0), "walk budget: epsilon must be positive"},
                {!(mu > 0.0 && mu <= 1.0), "walk budget: mu must be in (0,1]"}};
  for (const auto& c : checks)
    if (c.bad) throw std::invalid_argument(c.msg);
  const double slack = 2.0 + epsilon * (2.0 / 3.0);
  return (2.0 * slack / (epsilon * epsilon * mu)) * std::log(static_cast<double>(n));
}

std::uint64_t compute_walk_budget(std::uint64_t n, double epsilon, double mu) {
  std::uint64_t out = 0;
  check(pprg_walk_budget(n, epsilon, mu, &out));
  return out;
}

namespace {
// an index may serve a query only on its own graph shape and alpha
// (walk_index.cpp:36-42, speedppr.cpp:62-64, 81-84)
void require_index_fits(const WalkIndex* index, const Graph& g, double alpha) {
  if (!index) return;
  index->check_compatible(g);
  if (!(index->alpha() == alpha)) throw std::runtime_error("walk index was built for a different alpha");
}

PPRVector mc_phase(const Graph& g, NodeId s, double alpha, PushState&& st, std::uint64_t W,
                   const WalkIndex* index, Rng& rng) {
  if (st.reserve.size() != g.n() || st.residue.size() != g.n())
    throw std::invalid_argument("monte carlo: state size does not match the graph");
  require_index_fits(index, g, alpha);
  PPRVector out;
  out.estimates.assign(g.n(), 0.0);
  out.residues.assign(g.n(), 0.0);
  std::uint64_t walks = 0;
  check(pprg_monte_carlo(g.device_handle(), index ? index->device_handle(g) : nullptr, s, alpha, W,
                         rng.next(), st.reserve.data(), st.residue.data(), out.estimates.data(),
                         &walks));
  out.source = s;
  out.alpha = alpha;
  out.achieved_r_sum = 0.0;  // speedppr.cpp:47
  out.pushes = st.edge_push_count;
  out.walks = walks;
  return out;
}
}  // namespace

PPRVector monte_carlo_phase(const Graph& g, NodeId s, double alpha, PushState&& state,
                            std::uint64_t walk_budget, Rng& rng) {
  return mc_phase(g, s, alpha, std::move(state), walk_budget, nullptr, rng);
}

PPRVector monte_carlo_phase(const Graph& g, NodeId s, double alpha, PushState&& state,
                            std::uint64_t walk_budget, const WalkIndex& index, Rng& rng) {
  return mc_phase(g, s, alpha, std::move(state), walk_budget, &index, rng);
}

PPRVector speedppr_query(const Graph& g, NodeId s, const QueryConfig& cfg,
                         const WalkIndex* index) {  // speedppr.cpp:74-111
  cfg.validate();
  if (!cfg.epsilon.has_value()) throw std::invalid_argument("speedppr: epsilon is required");
  if (!(s < g.n())) throw std::invalid_argument("speedppr: source out of range");
  require_index_fits(index, g, cfg.alpha);
  PPRVector v = make_vector(g.n(), s, cfg.alpha);
  pprg_query_stats q{};
  check(pprg_speedppr(g.device_handle(), index ? index->device_handle(g) : nullptr, &s, 1,
                      cfg.alpha, *cfg.epsilon, cfg.mu ? *cfg.mu : -1.0, cfg.seed,
                      v.estimates.data(), 0, &q, nullptr));
  v.pushes = q.pushes;
  v.walks = q.walks;
  return v;
}

// ---- edge lists (graph.hpp:97-100; format of graph.cpp:66-104) ---------------
// The whole file is read into memory and scanned once by a small state machine
// that appends straight into the flat pair array the device builder takes.
// Accepted: per line, optional blanks (space, tab, CR), then either nothing,
// a '#' comment, or two unsigned decimal ids separated by blanks. Errors name
// the file and the 1-based line ("path:line: what"), as the reference's.
namespace {
class EdgeScanner {
 public:
  EdgeScanner(const std::string& path, bool both_directions)
      : path_(path), both_(both_directions) {}

  std::vector<std::uint64_t> scan(std::string_view text) {
    std::vector<std::uint64_t> flat;
    std::size_t pos = 0;
    while (pos < text.size()) {
      ++line_;
      std::size_t eol = text.find('\n', pos);
      if (eol == std::string_view::npos) eol = text.size();
      scan_line(text.substr(pos, eol - pos), flat);
      pos = eol + 1;
    }
    return flat;
  }

 private:
  static bool blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

  [[noreturn]] void error(const char* what) const {
    throw std::runtime_error(path_ + ":" + std::to_string(line_) + ": " + what);
  }

  // one unsigned id at `i`; advances past it and the blanks after it
  std::uint64_t id(std::string_view ln, std::size_t& i, const char* what) const {
    std::uint64_t v = 0;
    const auto r = std::from_chars(ln.data() + i, ln.data() + ln.size(), v);
    if (r.ec != std::errc()) error(what);
    i = static_cast<std::size_t>(r.ptr - ln.data());
    while (i < ln.size() && blank(ln[i])) ++i;
    return v;
  }

  void scan_line(std::string_view ln, std::vector<std::uint64_t>& flat) const {
    std::size_t i = 0;
    while (i < ln.size() && blank(ln[i])) ++i;
    if (i == ln.size() || ln[i] == '#') return;
    const std::uint64_t u = id(ln, i, "expected non-negative integer source id");
    const std::uint64_t v = id(ln, i, "expected non-negative integer target id");
    if (i != ln.size()) error("trailing content after edge pair");
    flat.insert(flat.end(), {u, v});
    if (both_) flat.insert(flat.end(), {v, u});
  }

  std::string path_;
  bool both_;
  std::uint64_t line_ = 0;
};

Graph read_edge_file(const std::string& path, bool undirected) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open graph file: " + path);
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const std::vector<std::uint64_t> flat = EdgeScanner(path, undirected).scan(text);
  if (flat.empty()) throw std::runtime_error(path + ": graph is empty after cleaning");
  return build_on_device(flat.data(), flat.size() / 2);
}
}  // namespace

Graph load_edge_list(const std::string& path) { return read_edge_file(path, false); }
Graph undirected_to_directed(const std::string& path) { return read_edge_file(path, true); }

// ---- synthetic.hpp ------------------------------------------------------------------
Graph random_graph(NodeId n, std::uint32_t min_out, std::uint32_t max_out, std::uint64_t seed) {
  if (n == 0) throw std::invalid_argument("random_graph: need at least one node");
  if (min_out > max_out) throw std::invalid_argument("random_graph: min_out > max_out");
  Rng rng(seed);
  std::vector<std::uint64_t> off(static_cast<std::size_t>(n) + 1, 0);
  for (NodeId v = 0; v < n; ++v)  // all degrees first, then all targets (one stream)
    off[v + 1] = off[v] + min_out + rng.below(static_cast<std::uint64_t>(max_out - min_out) + 1);
  std::vector<NodeId> nbr(off[n]);
  for (auto& t : nbr) t = static_cast<NodeId>(rng.below(n));
  return Graph(std::move(off), std::move(nbr));
}

// ---- push state (push.cpp:9-15, 70-79, 201-222) -----------------------------------
void PushState::recompute_r_sum() {  // push.cpp:9-15: exact sum, 1e-6 drift guard
  const double exact = std::accumulate(residue.begin(), residue.end(), 0.0);
  const double drift = std::abs(exact - r_sum);
  if (drift > 1e-6) throw std::logic_error("push: r_sum drifted more than 1e-6 from the residues");
  r_sum = exact;
}

PushState power_push_state(const Graph& g, NodeId s, double alpha, double lambda,
                           const QueryConfig& cfg, PushObserver* observer, PowerPushTrace* trace) {
  PPRVector v = power_push(g, s, alpha, lambda, cfg, observer, trace);
  PushState st(g.n(), s);
  st.reserve = std::move(v.estimates);
  st.residue = std::move(v.residues);
  st.r_sum = v.achieved_r_sum;
  st.edge_push_count = v.pushes;
  return st;
}

void refine(const Graph& g, NodeId s, double alpha, double r_max, PushState& state,
            PushObserver* observer) {
  if (!(r_max > 0.0)) throw std::invalid_argument("refine: r_max must be positive");
  if (state.reserve.size() != g.n() || state.residue.size() != g.n())
    throw std::invalid_argument("refine: state size does not match the graph");
  pprg_query_stats q{};
  check(pprg_refine(g.device_handle(), &s, 1, alpha, r_max, state.reserve.data(),
                    state.residue.data(), 0, &q, nullptr));
  state.queue.clear();
  std::fill(state.in_queue.begin(), state.in_queue.end(), 0);
  state.r_sum = q.achieved_r_sum;
  state.edge_push_count += q.pushes;
  if (observer) {
    observer->on_push(state);
    observer->on_iteration(state, q.local_levels);
  }
}

PPRVector finish_state(PushState&& state, NodeId source, double alpha) {  // push.cpp:70-79
  PPRVector out = make_vector(0, source, alpha);
  std::swap(out.estimates, state.reserve);
  std::swap(out.residues, state.residue);
  out.achieved_r_sum = state.r_sum;
  out.pushes = state.edge_push_count;
  return out;
}

// ---- metrics.hpp (semantics of metrics.cpp:11-42) ---------------------------------
namespace {
// One pass over (estimate, truth): the l1 distance and, for truth >= mu, the
// relative errors (count above epsilon, maximum). epsilon < 0 counts nothing.
ErrorReport accumulate_errors(const double* est, const double* truth, std::size_t n, double mu,
                              double epsilon) {
  ErrorReport r;
  for (std::size_t i = 0; i < n; ++i) {
    const double gap = std::abs(est[i] - truth[i]);
    r.l1 += gap;
    if (!(truth[i] >= mu)) continue;
    const double rel = gap / truth[i];
    r.nodes_above_mu += 1;
    r.violations += rel > epsilon ? 1 : 0;
    if (rel > r.max_rel_above_mu) r.max_rel_above_mu = rel;
  }
  return r;
}

void require_same_length(std::size_t a, std::size_t b, const char* fn) {
  if (a != b) throw std::invalid_argument(std::string(fn) + ": vector lengths differ");
}
}  // namespace

double l1_error(std::span<const double> estimate, std::span<const double> truth) {
  require_same_length(estimate.size(), truth.size(), "l1_error");
  return accumulate_errors(estimate.data(), truth.data(), estimate.size(),
                           std::numeric_limits<double>::infinity(), 0.0)
      .l1;
}

double l1_error(const PPRVector& estimate, const PPRVector& truth) {
  const bool same_source = estimate.source == truth.source;
  if (!same_source) throw std::invalid_argument("l1_error: results are for different sources");
  require_same_length(estimate.estimates.size(), truth.estimates.size(), "l1_error");
  return accumulate_errors(estimate.estimates.data(), truth.estimates.data(),
                           truth.estimates.size(), std::numeric_limits<double>::infinity(), 0.0)
      .l1;
}

ErrorReport compare_to_truth(std::span<const double> estimate, std::span<const double> truth,
                             double mu, double epsilon) {
  require_same_length(estimate.size(), truth.size(), "compare_to_truth");
  return accumulate_errors(estimate.data(), truth.data(), estimate.size(), mu, epsilon);
}

PPRVector ground_truth(const Graph& g, NodeId s, double alpha) {
  if (s >= g.n()) throw std::invalid_argument("source out of range");
  PPRVector v = make_vector(g.n(), s, alpha);
  pprg_query_stats qs{};
  check(pprg_ground_truth(g.device_handle(), &s, 1, alpha, v.estimates.data(), 0, &qs, nullptr));
  v.achieved_r_sum = qs.achieved_r_sum;
  v.pushes = qs.pushes;
  return v;
}

// ---- exact_ppr.hpp (exact_ppr.cpp:45-90 guards and checks) -------------------------
DensePPR exact_ppr(const Graph& g, NodeId s, double alpha) {
  const NodeId n = g.n();
  if (n > kDenseSolveMaxNodes)
    throw std::invalid_argument("exact_ppr: graph exceeds the dense solve guard");
  if (!(alpha > 0.0 && alpha < 1.0)) throw std::invalid_argument("exact_ppr: alpha must be in (0,1)");
  if (s >= n) throw std::invalid_argument("exact_ppr: source out of range");
  // the GPU ground truth (lambda = 1e-17) stands in for the dense solve; the
  // reference's acceptance checks on the result follow (exact_ppr.cpp:67-88)
  std::vector<double> x(n, 0.0);
  pprg_query_stats qs{};
  check(pprg_ground_truth(g.device_handle(), &s, 1, alpha, x.data(), 0, &qs, nullptr));
  const double most_negative = x.empty() ? 0.0 : *std::min_element(x.begin(), x.end());
  if (most_negative < -1e-12) throw std::logic_error("exact_ppr: negative probability");
  for (double& v : x) v = std::max(v, 0.0);
  const double mass = std::accumulate(x.begin(), x.end(), 0.0);
  if (std::abs(mass - 1.0) > 1e-10) throw std::logic_error("exact_ppr: result does not sum to 1");
  // defining equation pi = alpha e_s + (1-alpha) pi P: the mass each node
  // receives from its in-neighbours, then the l1 norm of the difference
  std::vector<double> received(n, 0.0);
  for (NodeId v = 0; v < n; ++v) {
    const auto out = effective_out(g, v, s);
    const double give = (1.0 - alpha) * x[v] / static_cast<double>(out.degree());
    for (NodeId u : out) received[u] += give;
  }
  received[s] += alpha;
  double gap = 0.0;
  for (NodeId u = 0; u < n; ++u) gap += std::abs(x[u] - received[u]);
  if (gap > 1e-10) throw std::logic_error("exact_ppr: residual check failed");
  return DensePPR{std::move(x)};
}

// ---- csv.hpp (file format of csv.cpp:9-43: "node,ppr" then v,value rows) ------------
std::string format_double(double value) {
  char buf[32];  // %.17g round-trips every finite double
  const int len = std::snprintf(buf, sizeof buf, "%.17g", value);
  return std::string(buf, static_cast<std::size_t>(len));
}

void write_ppr_csv(const std::string& path, std::span<const double> values) {
  std::string text = "node,ppr\n";
  text.reserve(text.size() + values.size() * 28);
  for (std::size_t v = 0; v < values.size(); ++v)
    text.append(std::to_string(v)).append(1, ',').append(format_double(values[v])).append(1, '\n');
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open for writing: " + path);
  const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  if (std::fclose(f) != 0 || !ok) throw std::runtime_error("write failed: " + path);
}

std::vector<double> read_ppr_csv(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open: " + path);
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::string_view rest(text);
  auto next_line = [&rest]() {
    const std::size_t eol = std::min(rest.find('\n'), rest.size());
    std::string_view ln = rest.substr(0, eol);
    rest.remove_prefix(std::min(eol + 1, rest.size()));
    if (!ln.empty() && ln.back() == '\r') ln.remove_suffix(1);
    return ln;
  };
  if (rest.empty() || next_line() != "node,ppr")
    throw std::runtime_error(path + ": missing node,ppr header");
  std::vector<double> values;
  while (!rest.empty()) {
    const std::string_view ln = next_line();
    if (ln.empty()) continue;
    const std::size_t comma = ln.find(',');
    if (comma == std::string_view::npos)
      throw std::runtime_error(path + ": malformed row: " + std::string(ln));
    std::uint64_t id = 0;
    const auto r = std::from_chars(ln.data(), ln.data() + comma, id);
    if (r.ec != std::errc() || r.ptr != ln.data() + comma || id != values.size())
      throw std::runtime_error(path + ": node ids must be consecutive from 0");
    values.push_back(std::stod(std::string(ln.substr(comma + 1))));
  }
  return values;
}

// ---- sweep.hpp (the harness of sweep.cpp, on the GPU engines) ------------------------
// Cells run through the C ABI: the truths of all sources in one batched
// ground_truth call, each high-precision cell as one pprg_run_traced query
// whose per-step series (one point per global sweep / iteration / frontier
// level, recorded on the device side of the call) is thinned to the plan's
// push cadence, each SpeedPPR cell as one pprg_speedppr query.
bool is_high_precision_algo(const std::string& name) {
  static const char* const names[] = {kAlgoPowItr, kAlgoFifoFwdPush, kAlgoSimFwdPush,
                                      kAlgoPowerPush};
  return std::any_of(std::begin(names), std::end(names),
                     [&](const char* a) { return name == a; });
}
bool is_known_algo(const std::string& name) {
  return name == kAlgoSpeedPPR || is_high_precision_algo(name);
}

namespace {
// Keeps a point each time the cumulative edge pushes reach the next multiple
// of the cadence (shared by CheckpointRecorder and the traced sweep cells).
struct CadenceFilter {
  std::uint64_t cadence, next;
  explicit CadenceFilter(std::uint64_t c) : cadence(c ? c : 1), next(c ? c : 1) {}
  bool take(std::uint64_t pushes) {
    if (pushes < next) return false;
    next += cadence * ((pushes - next) / cadence + 1);
    return true;
  }
};

int traced_algo(const std::string& name) {
  if (name == kAlgoPowItr) return PPRG_ALGO_POWITR;
  if (name == kAlgoSimFwdPush) return PPRG_ALGO_SIMFWDPUSH;
  if (name == kAlgoFifoFwdPush) return PPRG_ALGO_FIFO;
  return PPRG_ALGO_POWERPUSH;
}

std::uint64_t elapsed_ns(std::chrono::steady_clock::time_point since) {
  return static_cast<std::uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                        std::chrono::steady_clock::now() - since)
                                        .count());
}
}  // namespace

CheckpointRecorder::CheckpointRecorder(std::uint64_t cadence)
    : cadence_(cadence ? cadence : 1), next_mark_(cadence_),
      started_(std::chrono::steady_clock::now()) {}

void CheckpointRecorder::on_push(const PushState& st) {
  CadenceFilter f(cadence_);
  f.next = next_mark_;
  if (!f.take(st.edge_push_count)) return;
  next_mark_ = f.next;
  checkpoints_.push_back({st.edge_push_count, st.r_sum, elapsed_ns(started_)});
}

SweepResult run_sweep(const Graph& g, const std::vector<NodeId>& sources, const SweepPlan& plan) {
  if (auto bad = std::find_if_not(plan.algorithms.begin(), plan.algorithms.end(), is_known_algo);
      bad != plan.algorithms.end())
    throw std::invalid_argument("unknown algorithm: " + *bad);
  const NodeId n = g.n();
  const double mu = plan.mu.value_or(default_mu(n));
  const std::uint64_t cadence = plan.checkpoint_every ? plan.checkpoint_every : 4 * g.m();
  for (NodeId s : sources)
    if (s >= n) throw std::invalid_argument("source out of range");

  // every source's truth in one device call (k x n, query-major)
  std::vector<double> truth(static_cast<std::size_t>(n) * sources.size());
  std::vector<pprg_query_stats> tq(sources.size());
  if (!sources.empty())
    check(pprg_ground_truth(g.device_handle(), sources.data(),
                            static_cast<std::uint32_t>(sources.size()), plan.alpha, truth.data(), 0,
                            tq.data(), nullptr));

  SweepResult result;
  std::vector<double> est(n);
  std::vector<pprg_checkpoint> series(1u << 16);
  auto emit = [&](NodeId s, const std::string& algo, double param, std::uint64_t wall,
                  const pprg_query_stats& q, const double* t, double eps) {
    SweepCell cell;
    const ErrorReport rep = accumulate_errors(est.data(), t, n, mu, eps);
    cell.row = SweepRow{s, algo, param, wall, q.pushes, q.walks, rep.l1, rep.max_rel_above_mu};
    result.cells.push_back(std::move(cell));
  };
  for (std::size_t i = 0; i < sources.size(); ++i) {
    const NodeId s = sources[i];
    const double* t = truth.data() + i * n;
    for (const std::string& algo : plan.algorithms) {
      if (is_high_precision_algo(algo)) {
        for (double lambda : plan.lambdas) {
          pprg_query_stats q{};
          std::uint32_t count = 0;
          const auto t0 = std::chrono::steady_clock::now();
          check(pprg_run_traced(g.device_handle(), traced_algo(algo), s, plan.alpha, lambda,
                                est.data(), &q, series.data(),
                                static_cast<std::uint32_t>(series.size()), &count));
          emit(s, algo, lambda, elapsed_ns(t0), q, t, 0.0);
          CadenceFilter keep(cadence);
          for (std::uint32_t c = 0; c < count; ++c)
            if (keep.take(series[c].pushes))
              result.cells.back().checkpoints.push_back(
                  {series[c].pushes, series[c].r_sum, series[c].time_ns});
        }
        continue;
      }
      for (double eps : plan.epsilons)
        for (std::uint64_t seed : plan.seeds) {
          pprg_query_stats q{};
          const auto t0 = std::chrono::steady_clock::now();
          check(pprg_speedppr(g.device_handle(), nullptr, &s, 1, plan.alpha, eps,
                              plan.mu ? *plan.mu : -1.0, seed, est.data(), 0, &q, nullptr));
          emit(s, algo, eps, elapsed_ns(t0), q, t, eps);
        }
    }
  }
  return result;
}

void write_sweep_csv(const SweepResult& result, const std::string& directory,
                     const std::string& graph_name) {
  namespace fs = std::filesystem;
  const fs::path dir(directory);
  fs::create_directories(dir);
  auto write_file = [](const fs::path& path, const std::string& text) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("cannot write " + path.string());
    const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    if (std::fclose(f) != 0 || !ok) throw std::runtime_error("write failed: " + path.string());
  };
  auto join = [](std::initializer_list<std::string> fields) {
    std::string line;
    for (const std::string& f : fields) line.append(line.empty() ? "" : ",").append(f);
    return line + "\n";
  };
  std::string summary = "source,algo,param,wall_time_ns,edge_pushes,walks,l1_error,max_rel_error\n";
  for (const SweepCell& cell : result.cells) {
    const SweepRow& r = cell.row;
    summary += join({std::to_string(r.source), r.algo, format_double(r.param),
                     std::to_string(r.wall_time_ns), std::to_string(r.edge_pushes),
                     std::to_string(r.walks), format_double(r.l1_error),
                     format_double(r.max_rel_error)});
    if (cell.checkpoints.empty()) continue;
    char tag[32];  // series file name carries the parameter in %g form
    std::snprintf(tag, sizeof tag, "%g", r.param);
    std::string text = "pushes,r_sum,time_ns\n";
    for (const Checkpoint& c : cell.checkpoints)
      text += join({std::to_string(c.pushes), format_double(c.r_sum), std::to_string(c.time_ns)});
    write_file(dir / (graph_name + "_" + r.algo + "_" + tag + ".csv"), text);
  }
  write_file(dir / (graph_name + "_sweep.csv"), summary);
}

std::vector<NodeId> sample_sources(const Graph& g, std::uint64_t count, std::uint64_t seed) {
  Rng rng(seed);  // Rng(seed).below(n) per source, with replacement
  std::vector<NodeId> out;
  out.reserve(count);
  while (out.size() < count) out.push_back(static_cast<NodeId>(rng.below(g.n())));
  return out;
}

}  // namespace ppr
