// The reference's own test cases (tests/test_power_push.cpp, test_push_engines.cpp,
// test_graph.cpp, test_walks.cpp, test_speedppr.cpp under /root/reference/proj),
// restated against the C++ drop-in (paper_2101_03652_b200/cpp): same API calls,
// same expectations, running on the GPU. Exit status = number of failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "ppr/csv.hpp"
#include "ppr/exact_ppr.hpp"
#include "ppr/graph.hpp"
#include "ppr/metrics.hpp"
#include "ppr/push.hpp"
#include "ppr/speedppr.hpp"
#include "ppr/synthetic.hpp"
#include "ppr/sweep.hpp"
#include "ppr/walk_index.hpp"

using namespace ppr;

static int failures = 0;
#define CHECK(x)                                                              \
  do {                                                                        \
    if (!(x)) {                                                               \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);               \
      ++failures;                                                             \
    }                                                                         \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                              \
  do {                                                                        \
    bool ok_ = false;                                                         \
    try {                                                                     \
      (void)(expr);                                                           \
    } catch (const T&) {                                                      \
      ok_ = true;                                                             \
    } catch (...) {                                                           \
    }                                                                         \
    if (!ok_) {                                                               \
      std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
      ++failures;                                                             \
    }                                                                         \
  } while (0)

static Graph five_node_graph() {  // testutil.hpp:18-24
  return build_graph_from_edges({{0, 1}, {0, 2}, {1, 0}, {1, 2}, {1, 3}, {1, 4}, {2, 1}, {2, 3},
                                 {3, 0}, {3, 1}, {3, 2}, {4, 1}, {4, 2}});
}
static const double kPi0[5] = {0.29366106080206994, 0.27166882276843485, 0.23285899094437276,
                               0.1474773609314361, 0.054333764553686985};  // testutil.hpp:28-33

static double l1(const std::vector<double>& a, const double* b) {
  double t = 0;
  for (std::size_t i = 0; i < a.size(); ++i) t += std::abs(a[i] - b[i]);
  return t;
}

int main() {
  const Graph g = five_node_graph();
  // test_graph.cpp:32-39
  CHECK(g.n() == 5 && g.m() == 13);
  const EdgeId deg[5] = {2, 4, 2, 3, 2};
  for (NodeId v = 0; v < 5; ++v) CHECK(g.out_degree(v) == deg[v]);
  // relabel keeps order, duplicates kept (test_graph.cpp:41-59)
  {
    const Graph sp = build_graph_from_edges({{10, 40}, {40, 25}});
    CHECK(sp.n() == 3 && sp.neighbors(0)[0] == 2 && sp.neighbors(2)[0] == 1);
    const Graph dup = build_graph_from_edges({{0, 1}, {0, 1}, {1, 1}, {1, 0}});
    CHECK(dup.m() == 4 && dup.out_degree(0) == 2 && dup.out_degree(1) == 2);
  }
  // test_power_push.cpp:32-54
  {
    PowerPushTrace trace;
    QueryConfig cfg;
    const PPRVector out = power_push(g, 0, 0.2, 1e-8, cfg, nullptr, &trace);
    CHECK(trace.used_scan_phase);
    CHECK(trace.epoch_r_max.size() == 8);
    for (std::size_t i = 1; i <= 8 && i <= trace.epoch_r_max.size(); ++i) {
      const double expected = std::pow(10.0, -static_cast<double>(i)) / 13.0;
      CHECK(std::abs(trace.epoch_r_max[i - 1] - expected) <= 1e-12 * expected);
    }
    CHECK(out.achieved_r_sum <= 1e-8);
    CHECK(l1(out.estimates, kPi0) <= 1e-8);
  }
  // test_power_push.cpp:89-94 and push.cpp:142
  {
    QueryConfig cfg;
    CHECK_THROWS_AS(power_push(g, 0, 0.2, 0.0, cfg), std::invalid_argument);
    CHECK_THROWS_AS(power_push(g, 0, 0.2, 1.5, cfg), std::invalid_argument);
    CHECK_THROWS_AS(fifo_forward_push(g, 0, 0.2, 0.0), std::invalid_argument);
  }
  // test_push_engines.cpp:148-154, 237-253
  {
    const PPRVector z = power_iteration(g, 0, 0.2, 1.0);
    for (double x : z.estimates) CHECK(x == 0.0);
    CHECK(z.achieved_r_sum == 1.0 && z.residues[0] == 1.0);
    CHECK(l1(power_iteration(g, 0, 0.2, 1e-8).estimates, kPi0) <= 1e-8);
    CHECK(l1(sim_forward_push(g, 0, 0.2, 1e-8).estimates, kPi0) <= 1e-8);
    CHECK(l1(fifo_forward_push(g, 0, 0.2, 1e-8 / 13).estimates, kPi0) <= 1e-8);
  }
  // batched queries agree with single queries within lambda
  {
    QueryConfig cfg;
    const auto many = power_push_batch(g, {0, 1, 2, 3, 4}, 0.2, 1e-10, cfg);
    CHECK(many.size() == 5);
    CHECK(l1(many[0].estimates, kPi0) <= 1e-10);
  }
  // test_walks.cpp:14-18, 71-79; test_graph.cpp:153-178 (cache round trip)
  CHECK(compute_walk_budget(5, 0.5, 0.2) == 151);
  {
    const WalkIndex idx = build_index(g, 0.2, 7);
    CHECK(idx.endpoint_count() == 13);
    const std::size_t expected[5] = {2, 4, 2, 3, 2};
    for (NodeId v = 0; v < 5; ++v) CHECK(idx.endpoints_of(v).size() == expected[v]);
    const std::string ip = "/tmp/ppr_dropin_idx.pprw", gp = "/tmp/ppr_dropin_g.pprg";
    save_index(idx, ip);
    const WalkIndex back = load_index(ip, g);
    for (NodeId v = 0; v < 5; ++v)
      for (std::size_t k = 0; k < expected[v]; ++k)
        CHECK(back.endpoints_of(v)[k] == idx.endpoints_of(v)[k]);
    save_graph_cache(g, gp);
    CHECK(is_graph_cache(gp));
    const Graph gb = load_graph_cache(gp);
    CHECK(gb.out_offsets() == g.out_offsets() && gb.out_neighbors() == g.out_neighbors());
    std::ifstream f(gp, std::ios::binary);
    const std::string bytes((std::istreambuf_iterator<char>(f)), {});
    CHECK(bytes.size() == 4 + 1 + 8 + 8 + 6 * 8 + 13 * 4);
    std::remove(ip.c_str());
    std::remove(gp.c_str());
  }
  // test_speedppr.cpp:148-173
  {
    QueryConfig cfg;
    CHECK_THROWS_AS(speedppr_query(g, 0, cfg), std::invalid_argument);
    cfg.epsilon = 3.0;
    cfg.seed = 9;
    const PPRVector out = speedppr_query(g, 0, cfg);
    CHECK(out.pushes == 0 && out.walks == compute_walk_budget(5, 3.0, 0.2));
    double sum = 0;
    for (double x : out.estimates) sum += x;
    CHECK(std::abs(sum - 1.0) < 1e-9);
    const WalkIndex other = build_index(g, 0.15, 3);
    QueryConfig c2;
    c2.epsilon = 0.5;
    CHECK_THROWS_AS(speedppr_query(g, 0, c2, &other), std::runtime_error);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  {  // test_metrics.cpp:66-76, 85-93
    const PPRVector a = ground_truth(g, 0, 0.2);
    const PPRVector b = ground_truth(g, 0, 0.2);
    CHECK(a.estimates == b.estimates);
    const double pi0[5] = {0.29366106080206994, 0.27166882276843485, 0.23285899094437276,
                           0.1474773609314361, 0.054333764553686985};
    double l1 = 0.0, total = 0.0;
    for (int v = 0; v < 5; ++v) l1 += std::fabs(a.estimates[v] - pi0[v]), total += a.estimates[v];
    CHECK(l1 <= 1e-12);
    CHECK(std::fabs(total - 1.0) <= 1e-12);
    CHECK(a.achieved_r_sum <= kGroundTruthLambda);
    CHECK(compare_to_truth(a.estimates, a.estimates, 0.2, 0.0).violations == 0);
    const std::vector<double> vals = {0.29366106080206994, 1e-17, 0.0, 2.0 / 3.0, 5.4333764553686985e-2};
    write_ppr_csv("/tmp/pprg_dropin_vals.csv", vals);
    CHECK(read_ppr_csv("/tmp/pprg_dropin_vals.csv") == vals);
    std::remove("/tmp/pprg_dropin_vals.csv");
  }
  {  // observers at step granularity (test_push_engines.cpp:22-46, 283-339; test_metrics.cpp:36-56)
    struct Probe : PushObserver {
      std::uint64_t calls = 0;
      double worst = 0.0;
      std::vector<double> last_reserve;
      double last_r_sum = 2.0;
      bool monotone = true;
      void on_push(const PushState& st) override {
        ++calls;
        double t = 0.0;
        for (double x : st.reserve) t += x;
        for (double x : st.residue) t += x;
        worst = std::max(worst, std::fabs(t - 1.0));
        if (!last_reserve.empty())
          for (std::size_t v = 0; v < st.reserve.size(); ++v)
            if (st.reserve[v] < last_reserve[v]) monotone = false;
        if (st.r_sum > last_r_sum + 1e-15) monotone = false;
        last_reserve = st.reserve;
        last_r_sum = st.r_sum;
      }
    };
    const std::vector<std::pair<std::uint64_t, std::uint64_t>> e = {
        {0, 1}, {1, 2}, {2, 0}, {2, 3}, {3, 4}, {4, 0}, {4, 5}, {5, 6}, {6, 2}, {6, 7}, {7, 8}, {3, 9}};
    const Graph gd = build_graph_from_edges(e);  // node 8, 9 are dead ends
    std::uint64_t total = 0;
    double worst = 0.0;
    {
      Probe p;
      fifo_forward_push(gd, 1, 0.2, 1e-9, std::nullopt, &p);
      CHECK(p.monotone);
      total += p.calls;
      worst = std::max(worst, p.worst);
    }
    {
      Probe p;
      power_push(gd, 1, 0.2, 1e-10, QueryConfig{}, &p);
      CHECK(p.monotone);
      total += p.calls;
      worst = std::max(worst, p.worst);
    }
    {
      Probe p;
      PushState st = power_push_state(gd, 1, 0.2, 1e-4, QueryConfig{});
      refine(gd, 1, 0.2, 1e-9, st, &p);
      for (NodeId v = 0; v < gd.n(); ++v)
        CHECK(st.residue[v] <= static_cast<double>(gd.out_degree(v) ? gd.out_degree(v) : 1) * 1e-9);
      total += p.calls;
      worst = std::max(worst, p.worst);
    }
    {
      Probe p;
      power_iteration(gd, 1, 0.2, 1e-13, &p);
      sim_forward_push(gd, 1, 0.2, 1e-13, &p);
      total += p.calls;
      worst = std::max(worst, p.worst);
    }
    CHECK(total >= 100);
    CHECK(worst <= 1e-9);

    struct Trace : PushObserver {
      std::vector<double> errors;
      const double* truth = nullptr;
      void on_iteration(const PushState& st, std::uint32_t) override {
        double err = 0.0;
        for (std::size_t v = 0; v < st.reserve.size(); ++v) err += std::fabs(st.reserve[v] - truth[v]);
        errors.push_back(err);
      }
    } tr;
    const double pi0[5] = {0.29366106080206994, 0.27166882276843485, 0.23285899094437276,
                           0.1474773609314361, 0.054333764553686985};
    tr.truth = pi0;
    power_iteration(g, 0, 0.2, 1e-9, &tr);
    CHECK(!tr.errors.empty());
    for (std::size_t j = 1; j <= tr.errors.size(); ++j)
      CHECK(std::fabs(tr.errors[j - 1] - std::pow(0.8, j)) < 1e-10);
  }
  {  // refine: already-inactive state is a fixed point (test_push_engines.cpp:342-350)
    PushState st = power_push_state(g, 0, 0.2, 1e-6, QueryConfig{});
    const std::uint64_t pushes_before = st.edge_push_count;
    const auto reserve_before = st.reserve;
    refine(g, 0, 0.2, 1.0, st);
    CHECK(st.edge_push_count == pushes_before);
    CHECK(st.reserve == reserve_before);
  }
  {  // refine enforces the per-node residue bound in O(m) pushes (test_push_engines.cpp:352-367)
    std::vector<std::pair<std::uint64_t, std::uint64_t>> e;
    for (std::uint64_t v = 0; v < 300; ++v)
      for (std::uint64_t j = 1; j <= 1 + v % 5; ++j) e.push_back({v, (v * 7 + j * 13) % 300});
    const Graph gr = build_graph_from_edges(e);
    const double r_max = 1e-7 / static_cast<double>(gr.m());
    const double lambda = static_cast<double>(gr.m()) * r_max;
    PushState st = power_push_state(gr, 4, 0.2, lambda, QueryConfig{});
    const std::uint64_t before = st.edge_push_count;
    refine(gr, 4, 0.2, r_max, st);
    for (NodeId v = 0; v < gr.n(); ++v)
      CHECK(st.residue[v] <= static_cast<double>(gr.out_degree(v)) * r_max);
    CHECK(static_cast<double>(st.edge_push_count - before) <= lambda / (0.2 * r_max) * 1.01);
    const PPRVector fin = finish_state(std::move(st), 4, 0.2);
    CHECK(fin.achieved_r_sum <= lambda);
  }
  {  // monte carlo phase (test_speedppr.cpp:35-107), on the GPU
    auto total = [](const std::vector<double>& xs) {
      double t = 0.0;
      for (double x : xs) t += x;
      return t;
    };
    {
      PushState st(5, 0);
      st.residue.assign(5, 0.0);
      st.reserve = {0.4, 0.3, 0.2, 0.1, 0.0};
      st.r_sum = 0.0;
      Rng rng(1);
      const PPRVector out = monte_carlo_phase(g, 0, 0.2, std::move(st), 100, rng);
      CHECK((out.estimates == std::vector<double>{0.4, 0.3, 0.2, 0.1, 0.0}));
      CHECK(out.walks == 0);
    }
    {
      const std::uint64_t W = 151;
      PushState st(5, 0);
      st.residue.assign(5, 0.0);
      st.residue[1] = 3.0 / W;
      st.r_sum = 3.0 / W;
      Rng rng(2);
      const PPRVector out = monte_carlo_phase(g, 0, 0.2, std::move(st), W, rng);
      CHECK(out.walks == 3);
      CHECK(std::fabs(total(out.estimates) - 3.0 / W) <= 1e-12 * 3.0 / W + 1e-18);
      for (double x : out.estimates) CHECK(std::fabs(x * W - std::round(x * W)) < 1e-9);
    }
    for (std::uint64_t seed : {3, 4, 5}) {
      const Graph gr = random_graph(40, 0, 4, seed);
      const NodeId s = static_cast<NodeId>(seed % gr.n());
      const std::uint64_t W = 4 * gr.effective_edge_count();
      QueryConfig cfg;
      PushState st = power_push_state(gr, s, 0.2, static_cast<double>(gr.effective_edge_count()) / W, cfg);
      refine(gr, s, 0.2, 1.0 / static_cast<double>(W), st);
      Rng rng(seed);
      const PPRVector out = monte_carlo_phase(gr, s, 0.2, std::move(st), W, rng);
      CHECK(std::fabs(total(out.estimates) - 1.0) < 1e-9);
      CHECK(out.achieved_r_sum == 0.0);
    }
    {
      PushState st(5, 0);  // residue[0] = 1 >> d/W
      Rng rng(1);
      CHECK_THROWS_AS(monte_carlo_phase(g, 0, 0.2, std::move(st), 100, rng), std::logic_error);
    }
    {
      const Graph gr = random_graph(30, 0, 4, 13);
      const WalkIndex idx = build_index(gr, 0.2, 21);
      PushState st(gr.n(), 5);
      Rng rng(7);
      CHECK_THROWS_AS(monte_carlo_phase(gr, 5, 0.15, PushState(gr.n(), 5), 100, idx, rng),
                      std::runtime_error);
      // stored prefixes: a residue of k/W on a node with out-edges consumes its first k terminals
      const std::uint64_t W = 1000;
      NodeId v = 0;
      while (gr.out_degree(v) < 3) ++v;
      st.residue.assign(gr.n(), 0.0);
      st.residue[v] = 3.0 / W;
      st.reserve.assign(gr.n(), 0.0);
      const PPRVector out = monte_carlo_phase(gr, 5, 0.2, std::move(st), W, idx, rng);
      std::vector<double> expect(gr.n(), 0.0);
      for (int k = 0; k < 3; ++k) expect[idx.endpoints_of(v)[k]] += (3.0 / W) / 3.0;
      for (NodeId t = 0; t < gr.n(); ++t) CHECK(std::fabs(out.estimates[t] - expect[t]) < 1e-15);
    }
  }
  {  // edge list parsing (test_graph.cpp "edge list parsing", "undirected loading doubles every edge")
    const std::string path = "/tmp/pprg_dropin_edges.txt";
    {
      std::ofstream out(path);
      out << "# comment\n\n0 1\n  1\t2\r\n2 0\n";
    }
    const Graph a = load_edge_list(path);
    CHECK(a.n() == 3 && a.m() == 3);
    const Graph u = undirected_to_directed(path);
    CHECK(u.m() == 6);
    {
      std::ofstream out(path);
      out << "0 1\n1 2 3\n";
    }
    bool threw = false;
    try {
      load_edge_list(path);
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()).find(":2: trailing content after edge pair") != std::string::npos;
    }
    CHECK(threw);
    std::remove(path.c_str());
  }
  {  // sweep harness (test_metrics.cpp sweep cases)
    SweepPlan plan;
    plan.algorithms = {kAlgoPowerPush, kAlgoPowItr, kAlgoSpeedPPR};
    plan.lambdas = {1e-4, 1e-8};
    plan.epsilons = {0.5};
    const SweepResult r = run_sweep(g, {0}, plan);
    CHECK(r.cells.size() == 5);
    CHECK(r.cells[0].row.edge_pushes <= r.cells[1].row.edge_pushes);  // pushes grow as lambda shrinks
    for (const auto& c : r.cells)
      if (c.row.algo != kAlgoSpeedPPR) CHECK(c.row.l1_error <= c.row.param + 1e-12);
    CHECK(!r.cells[1].checkpoints.empty());
    bool threw = false;
    try {
      SweepPlan bad;
      bad.algorithms = {"nosuch"};
      run_sweep(g, {0}, bad);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    write_sweep_csv(r, "/tmp/pprg_dropin_sweep", "five");
    std::ifstream in("/tmp/pprg_dropin_sweep/five_sweep.csv");
    std::string header;
    std::getline(in, header);
    CHECK(header == "source,algo,param,wall_time_ns,edge_pushes,walks,l1_error,max_rel_error");
    const auto src = sample_sources(g, 10, 3);
    CHECK(src.size() == 10);
    for (NodeId v : src) CHECK(v < g.n());
  }
  {  // exact_ppr (test_oracle.cpp: five-node frozen solve, two-cycle closed form, guards)
    const double pi0[5] = {0.29366106080206994, 0.27166882276843485, 0.23285899094437276,
                           0.1474773609314361, 0.054333764553686985};
    const DensePPR d = exact_ppr(g, 0, 0.2);
    for (int v = 0; v < 5; ++v) CHECK(std::fabs(d.pi[v] - pi0[v]) < 1e-12);
    const Graph two = build_graph_from_edges({{0, 1}, {1, 0}});
    const DensePPR t = exact_ppr(two, 0, 0.2);
    CHECK(std::fabs(t.pi[0] - 5.0 / 9.0) < 1e-12 && std::fabs(t.pi[1] - 4.0 / 9.0) < 1e-12);
    CHECK_THROWS_AS(exact_ppr(g, 9, 0.2), std::invalid_argument);
    CHECK_THROWS_AS(exact_ppr(g, 0, 0.0), std::invalid_argument);
    CHECK_THROWS_AS(exact_ppr(random_graph(2001, 1, 2, 1), 0, 0.2), std::invalid_argument);
  }
  return failures;
}
