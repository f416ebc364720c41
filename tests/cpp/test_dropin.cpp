// The reference's own test cases (tests/test_power_push.cpp, test_push_engines.cpp,
// test_graph.cpp, test_walks.cpp, test_speedppr.cpp under /root/reference/proj),
// restated against the C++ drop-in (paper_2101_03652_b200/cpp): same API calls,
// same expectations, running on the GPU. Exit status = number of failures.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "ppr/csv.hpp"
#include "ppr/graph.hpp"
#include "ppr/metrics.hpp"
#include "ppr/push.hpp"
#include "ppr/speedppr.hpp"
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
  return failures;
}
