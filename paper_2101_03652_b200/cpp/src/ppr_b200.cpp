// C++ drop-in of the reference's ppr:: core API over the engine's C ABI
// (include/pprg.h). Every engine call runs on the GPU; status codes come back
// as the reference's exception types (invalid_argument / runtime_error /
// logic_error).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>

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

void write_u64(std::ofstream& o, std::uint64_t v) {
  char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  o.write(b, 8);
}
void write_u32(std::ofstream& o, std::uint32_t v) {
  char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  o.write(b, 4);
}
std::uint64_t read_u64(std::ifstream& in) {
  unsigned char b[8] = {};
  in.read(reinterpret_cast<char*>(b), 8);
  std::uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(b[i]) << (8 * i);
  return v;
}
std::uint32_t read_u32(std::ifstream& in) {
  unsigned char b[4] = {};
  in.read(reinterpret_cast<char*>(b), 4);
  std::uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= static_cast<std::uint32_t>(b[i]) << (8 * i);
  return v;
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

Graph build_graph_from_edges(const std::vector<std::pair<std::uint64_t, std::uint64_t>>& edges) {
  if (edges.empty()) throw std::runtime_error("graph is empty after cleaning");
  std::vector<std::uint64_t> flat(2 * edges.size());
  for (std::size_t i = 0; i < edges.size(); ++i) {
    flat[2 * i] = edges[i].first;
    flat[2 * i + 1] = edges[i].second;
  }
  pprg_graph* h = nullptr;
  check(pprg_graph_build_from_edges(flat.data(), edges.size(), device_from_env(), &h));
  std::uint64_t n = 0, m = 0, nd = 0;
  check(pprg_graph_info(h, &n, &m, &nd));
  std::vector<std::uint64_t> off(n + 1);
  std::vector<NodeId> nbr(m);
  check(pprg_graph_export(h, off.data(), nbr.data(), nullptr));
  pprg_graph_destroy(h);
  return Graph(std::move(off), std::move(nbr));
}

void save_graph_cache(const Graph& g, const std::string& path) {  // graph.cpp:115-125
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out.write("PPRG", 4);
  out.put(1);
  write_u64(out, g.n());
  write_u64(out, g.m());
  for (auto o : g.out_offsets()) write_u64(out, o);
  for (auto u : g.out_neighbors()) write_u32(out, u);
  if (!out) throw std::runtime_error("write failed: " + path);
}

Graph load_graph_cache(const std::string& path) {  // graph.cpp:127-143
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open graph cache: " + path);
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, "PPRG", 4) != 0)
    throw std::runtime_error(path + ": not a graph cache (bad magic)");
  if (in.get() != 1) throw std::runtime_error(path + ": unsupported graph cache version");
  const std::uint64_t n = read_u64(in), m = read_u64(in);
  std::vector<std::uint64_t> off(n + 1);
  for (auto& o : off) o = read_u64(in);
  std::vector<NodeId> nbr(m);
  for (auto& u : nbr) u = read_u32(in);
  if (!in) throw std::runtime_error(path + ": truncated graph cache");
  return Graph(std::move(off), std::move(nbr));
}

bool is_graph_cache(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  char magic[4];
  return in && in.read(magic, 4) && std::memcmp(magic, "PPRG", 4) == 0;
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
void WalkIndex::check_compatible(const Graph& g) const {  // walk_index.cpp:36-42
  if (node_count() != g.n() || endpoint_count() != g.m())
    throw std::runtime_error("walk index does not match the graph shape");
  for (NodeId v = 0; v < g.n(); ++v)
    if (endpoints_of(v).size() != g.out_degree(v))
      throw std::runtime_error("walk index slice length differs from out-degree");
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

void save_index(const WalkIndex& index, const std::string& path) {  // walk_index.cpp:61-81
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out.write("PPRW", 4);
  out.put(1);
  out.put(static_cast<char>(index.rng_id()));
  std::uint64_t bits;
  const double a = index.alpha();
  std::memcpy(&bits, &a, 8);
  write_u64(out, bits);
  write_u64(out, index.seed());
  write_u64(out, index.node_count());
  write_u64(out, index.endpoint_count());
  std::uint64_t off = 0;
  write_u64(out, 0);
  for (NodeId v = 0; v < index.node_count(); ++v) {
    off += index.endpoints_of(v).size();
    write_u64(out, off);
  }
  for (NodeId v = 0; v < index.node_count(); ++v)
    for (NodeId e : index.endpoints_of(v)) write_u32(out, e);
  if (!out) throw std::runtime_error("write failed: " + path);
}

WalkIndex load_index(const std::string& path) {  // walk_index.cpp:83-104
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open walk index: " + path);
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, "PPRW", 4) != 0)
    throw std::runtime_error(path + ": not a walk index (bad magic)");
  if (in.get() != 1) throw std::runtime_error(path + ": unsupported walk index version");
  if (in.get() != kRngIdPhilox4x32_10) throw std::runtime_error(path + ": unknown generator id");
  const std::uint64_t abits = read_u64(in);
  double alpha;
  std::memcpy(&alpha, &abits, 8);
  const std::uint64_t seed = read_u64(in), n = read_u64(in), m = read_u64(in);
  WalkIndex w;
  w.alpha_ = alpha;
  w.seed_ = seed;
  w.offsets_.resize(n + 1);
  for (auto& o : w.offsets_) o = read_u64(in);
  w.endpoints_.resize(m);
  for (auto& e : w.endpoints_) e = read_u32(in);
  if (!in) throw std::runtime_error(path + ": truncated walk index");
  // WalkIndex constructor checks (walk_index.cpp:19-34)
  if (w.offsets_.empty() || w.offsets_.front() != 0 || w.offsets_.back() != m)
    throw std::runtime_error("walk index: inconsistent offsets");
  for (std::size_t i = 0; i + 1 < w.offsets_.size(); ++i)
    if (w.offsets_[i + 1] < w.offsets_[i])
      throw std::runtime_error("walk index: offsets must be non-decreasing");
  for (NodeId e : w.endpoints_)
    if (e >= n) throw std::runtime_error("walk index: endpoint id out of range");
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
  if (n < 2) throw std::invalid_argument("walk budget: need n >= 2");
  if (!(epsilon > 0.0)) throw std::invalid_argument("walk budget: epsilon must be positive");
  if (!(mu > 0.0 && mu <= 1.0)) throw std::invalid_argument("walk budget: mu must be in (0,1]");
  return 2.0 * (2.0 * epsilon / 3.0 + 2.0) * std::log(static_cast<double>(n)) /
         (epsilon * epsilon * mu);
}

std::uint64_t compute_walk_budget(std::uint64_t n, double epsilon, double mu) {
  std::uint64_t out = 0;
  check(pprg_walk_budget(n, epsilon, mu, &out));
  return out;
}

namespace {
PPRVector mc_phase(const Graph& g, NodeId s, double alpha, PushState&& st, std::uint64_t W,
                   const WalkIndex* index, Rng& rng) {
  if (st.reserve.size() != g.n() || st.residue.size() != g.n())
    throw std::invalid_argument("monte carlo: state size does not match the graph");
  if (index) {
    index->check_compatible(g);
    if (index->alpha() != alpha) throw std::runtime_error("walk index was built for a different alpha");
  }
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
  if (!cfg.epsilon) throw std::invalid_argument("speedppr: epsilon is required");
  if (s >= g.n()) throw std::invalid_argument("speedppr: source out of range");
  if (index) {
    index->check_compatible(g);
    if (index->alpha() != cfg.alpha)
      throw std::runtime_error("walk index was built for a different alpha");
  }
  PPRVector v = make_vector(g.n(), s, cfg.alpha);
  pprg_query_stats q{};
  check(pprg_speedppr(g.device_handle(), index ? index->device_handle(g) : nullptr, &s, 1,
                      cfg.alpha, *cfg.epsilon, cfg.mu ? *cfg.mu : -1.0, cfg.seed,
                      v.estimates.data(), 0, &q, nullptr));
  v.pushes = q.pushes;
  v.walks = q.walks;
  return v;
}

// ---- edge lists (graph.cpp:66-113) ---------------------------------------------------
namespace {
Graph read_edge_file(const std::string& path, bool undirected) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open graph file: " + path);
  std::vector<std::pair<std::uint64_t, std::uint64_t>> edges;
  std::string line;
  for (std::uint64_t no = 1; std::getline(in, line); ++no) {
    const char* p = line.data();
    const char* const end = p + line.size();
    auto blank = [&] {
      while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    };
    auto bad = [&](const char* what) {
      throw std::runtime_error(path + ":" + std::to_string(no) + ": " + what);
    };
    blank();
    if (p == end || *p == '#') continue;
    std::uint64_t a = 0, b = 0;
    auto r = std::from_chars(p, end, a);
    if (r.ec != std::errc()) bad("expected non-negative integer source id");
    p = r.ptr;
    blank();
    r = std::from_chars(p, end, b);
    if (r.ec != std::errc()) bad("expected non-negative integer target id");
    p = r.ptr;
    blank();
    if (p != end) bad("trailing content after edge pair");
    edges.emplace_back(a, b);
    if (undirected) edges.emplace_back(b, a);
  }
  if (edges.empty()) throw std::runtime_error(path + ": graph is empty after cleaning");
  return build_graph_from_edges(edges);
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
void PushState::recompute_r_sum() {
  double total = 0.0;
  for (double r : residue) total += r;
  if (std::abs(total - r_sum) > 1e-6)
    throw std::logic_error("push: r_sum drifted more than 1e-6 from the residues");
  r_sum = total;
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

PPRVector finish_state(PushState&& state, NodeId source, double alpha) {
  PPRVector out;
  out.estimates = std::move(state.reserve);
  out.residues = std::move(state.residue);
  out.source = source;
  out.alpha = alpha;
  out.achieved_r_sum = state.r_sum;
  out.pushes = state.edge_push_count;
  return out;
}

// ---- metrics.hpp (metrics.cpp:11-55) ---------------------------------------------
double l1_error(std::span<const double> estimate, std::span<const double> truth) {
  if (estimate.size() != truth.size())
    throw std::invalid_argument("l1_error: vector lengths differ");
  double total = 0.0;
  for (std::size_t i = 0; i < estimate.size(); ++i) total += std::abs(estimate[i] - truth[i]);
  return total;
}

double l1_error(const PPRVector& estimate, const PPRVector& truth) {
  if (estimate.source != truth.source)
    throw std::invalid_argument("l1_error: results are for different sources");
  return l1_error(std::span<const double>(estimate.estimates),
                  std::span<const double>(truth.estimates));
}

ErrorReport compare_to_truth(std::span<const double> estimate, std::span<const double> truth,
                             double mu, double epsilon) {
  if (estimate.size() != truth.size())
    throw std::invalid_argument("compare_to_truth: vector lengths differ");
  ErrorReport r;
  for (std::size_t i = 0; i < estimate.size(); ++i) {
    const double d = std::abs(estimate[i] - truth[i]);
    r.l1 += d;
    if (truth[i] >= mu) {
      ++r.nodes_above_mu;
      r.max_rel_above_mu = std::max(r.max_rel_above_mu, d / truth[i]);
      if (d / truth[i] > epsilon) ++r.violations;
    }
  }
  return r;
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
  std::vector<double> x(n, 0.0);
  pprg_query_stats qs{};
  check(pprg_ground_truth(g.device_handle(), &s, 1, alpha, x.data(), 0, &qs, nullptr));
  double sum = 0.0;
  for (double& v : x) {
    if (v < 0.0) {
      if (v < -1e-12) throw std::logic_error("exact_ppr: negative probability");
      v = 0.0;
    }
    sum += v;
  }
  if (std::abs(sum - 1.0) > 1e-10) throw std::logic_error("exact_ppr: result does not sum to 1");
  std::vector<double> resid(x);  // pi - alpha e_s - (1-alpha) pi P
  resid[s] -= alpha;
  for (NodeId v = 0; v < n; ++v) {
    const auto out = effective_out(g, v, s);
    const double share = (1.0 - alpha) * x[v] / static_cast<double>(out.degree());
    for (NodeId u : out) resid[u] -= share;
  }
  double l1 = 0.0;
  for (double r : resid) l1 += std::abs(r);
  if (l1 > 1e-10) throw std::logic_error("exact_ppr: residual check failed");
  return DensePPR{std::move(x)};
}

// ---- csv.hpp (csv.cpp:9-43) --------------------------------------------------------
std::string format_double(double value) {
  char buffer[40];
  std::snprintf(buffer, sizeof(buffer), "%.17g", value);
  return buffer;
}

void write_ppr_csv(const std::string& path, std::span<const double> values) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw std::runtime_error("cannot open for writing: " + path);
  out << "node,ppr\n";
  for (std::size_t v = 0; v < values.size(); ++v) out << v << ',' << format_double(values[v]) << '\n';
  if (!out) throw std::runtime_error("write failed: " + path);
}

std::vector<double> read_ppr_csv(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open: " + path);
  std::string line;
  if (!std::getline(in, line) || line != "node,ppr")
    throw std::runtime_error(path + ": missing node,ppr header");
  std::vector<double> values;
  std::uint64_t expected = 0;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    const auto comma = line.find(',');
    if (comma == std::string::npos) throw std::runtime_error(path + ": malformed row: " + line);
    if (std::stoull(line.substr(0, comma)) != expected)
      throw std::runtime_error(path + ": node ids must be consecutive from 0");
    values.push_back(std::stod(line.substr(comma + 1)));
    ++expected;
  }
  return values;
}

// ---- sweep.hpp (sweep.cpp:16-147) ----------------------------------------------------
bool is_high_precision_algo(const std::string& name) {
  return name == kAlgoPowItr || name == kAlgoFifoFwdPush || name == kAlgoSimFwdPush ||
         name == kAlgoPowerPush;
}
bool is_known_algo(const std::string& name) {
  return is_high_precision_algo(name) || name == kAlgoSpeedPPR;
}

CheckpointRecorder::CheckpointRecorder(std::uint64_t cadence)
    : cadence_(cadence ? cadence : 1), next_mark_(cadence_),
      started_(std::chrono::steady_clock::now()) {}

void CheckpointRecorder::on_push(const PushState& st) {
  if (st.edge_push_count < next_mark_) return;
  const auto ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                      std::chrono::steady_clock::now() - started_)
                      .count();
  checkpoints_.push_back({st.edge_push_count, st.r_sum, static_cast<std::uint64_t>(ns)});
  while (next_mark_ <= st.edge_push_count) next_mark_ += cadence_;
}

namespace {
PPRVector run_high_precision(const Graph& g, NodeId s, const std::string& algo, double alpha,
                             double lambda, PushObserver* obs) {
  if (algo == kAlgoPowItr) return power_iteration(g, s, alpha, lambda, obs);
  if (algo == kAlgoSimFwdPush) return sim_forward_push(g, s, alpha, lambda, obs);
  if (algo == kAlgoFifoFwdPush)
    return fifo_forward_push(g, s, alpha, lambda / static_cast<double>(g.effective_edge_count()),
                             std::nullopt, obs);
  QueryConfig cfg;
  cfg.alpha = alpha;
  return power_push(g, s, alpha, lambda, cfg, obs);
}
std::uint64_t since_ns(std::chrono::steady_clock::time_point t0) {
  return static_cast<std::uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
          .count());
}
}  // namespace

SweepResult run_sweep(const Graph& g, const std::vector<NodeId>& sources, const SweepPlan& plan) {
  for (const auto& a : plan.algorithms)
    if (!is_known_algo(a)) throw std::invalid_argument("unknown algorithm: " + a);
  const std::uint64_t cadence = plan.checkpoint_every ? plan.checkpoint_every : 4 * g.m();
  const double mu = plan.mu ? *plan.mu : default_mu(g.n());
  SweepResult result;
  for (NodeId s : sources) {
    const PPRVector truth = ground_truth(g, s, plan.alpha);
    for (const auto& algo : plan.algorithms) {
      if (is_high_precision_algo(algo)) {
        for (double lambda : plan.lambdas) {
          CheckpointRecorder rec(cadence);
          const auto t0 = std::chrono::steady_clock::now();
          const PPRVector got = run_high_precision(g, s, algo, plan.alpha, lambda, &rec);
          const std::uint64_t wall = since_ns(t0);
          const ErrorReport rep = compare_to_truth(got.estimates, truth.estimates, mu, 0.0);
          SweepCell cell;
          cell.row = {s, algo, lambda, wall, got.pushes, got.walks, rep.l1, rep.max_rel_above_mu};
          cell.checkpoints = rec.checkpoints();
          result.cells.push_back(std::move(cell));
        }
      } else {
        for (double eps : plan.epsilons)
          for (std::uint64_t seed : plan.seeds) {
            QueryConfig cfg;
            cfg.alpha = plan.alpha;
            cfg.epsilon = eps;
            cfg.mu = plan.mu;
            cfg.seed = seed;
            const auto t0 = std::chrono::steady_clock::now();
            const PPRVector got = speedppr_query(g, s, cfg);
            const std::uint64_t wall = since_ns(t0);
            const ErrorReport rep = compare_to_truth(got.estimates, truth.estimates, mu, eps);
            SweepCell cell;
            cell.row = {s, algo, eps, wall, got.pushes, got.walks, rep.l1, rep.max_rel_above_mu};
            result.cells.push_back(std::move(cell));
          }
      }
    }
  }
  return result;
}

void write_sweep_csv(const SweepResult& result, const std::string& directory,
                     const std::string& graph_name) {
  namespace fs = std::filesystem;
  fs::create_directories(directory);
  const fs::path dir(directory);
  std::ofstream summary(dir / (graph_name + "_sweep.csv"), std::ios::trunc);
  if (!summary) throw std::runtime_error("cannot write sweep summary");
  summary << "source,algo,param,wall_time_ns,edge_pushes,walks,l1_error,max_rel_error\n";
  for (const auto& cell : result.cells) {
    const auto& r = cell.row;
    summary << r.source << ',' << r.algo << ',' << format_double(r.param) << ',' << r.wall_time_ns
            << ',' << r.edge_pushes << ',' << r.walks << ',' << format_double(r.l1_error) << ','
            << format_double(r.max_rel_error) << '\n';
    if (!cell.checkpoints.empty()) {
      char param[32];
      std::snprintf(param, sizeof(param), "%g", r.param);
      std::ofstream series(dir / (graph_name + "_" + r.algo + "_" + param + ".csv"), std::ios::trunc);
      series << "pushes,r_sum,time_ns\n";
      for (const auto& c : cell.checkpoints)
        series << c.pushes << ',' << format_double(c.r_sum) << ',' << c.time_ns << '\n';
    }
  }
}

std::vector<NodeId> sample_sources(const Graph& g, std::uint64_t count, std::uint64_t seed) {
  Rng rng(seed);
  std::vector<NodeId> out(count);
  for (auto& s : out) s = static_cast<NodeId>(rng.below(g.n()));
  return out;
}

}  // namespace ppr
