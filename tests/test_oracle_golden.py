"""Pin the CPU oracle (oracle/oracle.c) to the golden vectors and known-answer
tests the reference's own suite holds. Each test cites the reference test it
restates (paths under /root/reference/proj/tests)."""
import math

import numpy as np
import pytest

from oracle.pyoracle import (FIVE_NODE_PI0, InvalidArgument, LogicError, OgStats,
                             five_node_edges)


@pytest.fixture(scope="module")
def g5(oracle):
    return oracle.build_graph_from_edges(five_node_edges())


def test_five_node_shape(g5):  # test_graph.cpp:32-39
    assert g5.n == 5 and g5.m == 13
    assert list(g5.degrees()) == [2, 4, 2, 3, 2]
    assert len(g5.dead_ends()) == 0


def test_star_dead_ends(oracle):  # test_graph.cpp:21-30
    g = oracle.build_graph_from_edges([(0, 1), (0, 2)])
    assert (g.n, g.m) == (3, 2)
    assert list(g.dead_ends()) == [1, 2] and g.m_eff == 4


def test_relabel_sparse_ids(oracle):  # test_graph.cpp:41-52
    g = oracle.build_graph_from_edges([(10, 40), (40, 25)])
    assert g.n == 3
    assert g.neighbors[g.offsets[0]] == 2 and g.neighbors[g.offsets[2]] == 1


def test_duplicates_and_self_loops_kept(oracle):  # test_graph.cpp:54-59
    g = oracle.build_graph_from_edges([(0, 1), (0, 1), (1, 1), (1, 0)])
    assert g.m == 4 and list(g.degrees()) == [2, 2]


def test_exact_five_node_golden(oracle, g5):  # test_oracle.cpp:26-32
    pi = oracle.exact_ppr(g5, 0, 0.2)
    assert np.max(np.abs(pi - FIVE_NODE_PI0)) < 1e-12


def test_exact_two_cycle(oracle):  # test_oracle.cpp:18-24
    g = oracle.build_graph_from_edges([(0, 1), (1, 0)])
    pi = oracle.exact_ppr(g, 0, 0.2)
    assert abs(pi[0] - 5 / 9) < 1e-14 and abs(pi[1] - 4 / 9) < 1e-14


def test_exact_guards(oracle, g5):  # test_oracle.cpp:66-73
    with pytest.raises(InvalidArgument):
        oracle.exact_ppr(g5, 0, 0.0)
    with pytest.raises(InvalidArgument):
        oracle.exact_ppr(g5, 9, 0.2)


def test_push_trace_running_example(oracle, g5):  # test_push_engines.cpp:50-76
    res, rsd, st = np.zeros(5), np.zeros(5), OgStats(1.0, 0, 0, 0, 0)
    rsd[0] = 1.0
    oracle.push_once(g5, 0, 0.2, res, rsd, st, 0)
    assert abs(res[0] - 0.2) < 1e-12 and abs(rsd[1] - 0.4) < 1e-12 and abs(rsd[2] - 0.4) < 1e-12
    oracle.push_once(g5, 0, 0.2, res, rsd, st, 2)
    assert abs(res[2] - 0.08) < 1e-12 and abs(rsd[1] - 0.56) < 1e-12 and abs(rsd[3] - 0.16) < 1e-12
    oracle.push_once(g5, 0, 0.2, res, rsd, st, 1)
    assert abs(res[1] - 0.112) < 1e-12
    assert np.max(np.abs(rsd - [0.112, 0.0, 0.112, 0.272, 0.112])) < 1e-12
    assert np.all(rsd <= g5.degrees() * 0.099)
    assert abs(res.sum() + rsd.sum() - 1.0) < 1e-12


def test_push_zero_residue_noop(oracle, g5):  # test_push_engines.cpp:78-84
    res, rsd, st = np.zeros(5), np.zeros(5), OgStats(1.0, 0, 0, 0, 0)
    rsd[0] = 1.0
    oracle.push_once(g5, 0, 0.2, res, rsd, st, 3)
    assert st.pushes == 0 and st.r_sum == 1.0


def test_self_loop_keeps_share(oracle):  # test_push_engines.cpp:86-95
    g = oracle.build_graph_from_edges([(0, 0), (0, 1), (1, 0)])
    res, rsd, st = np.zeros(2), np.array([1.0, 0.0]), OgStats(1.0, 0, 0, 0, 0)
    oracle.push_once(g, 0, 0.2, res, rsd, st, 0)
    assert abs(rsd[0] - 0.4) < 1e-12 and abs(rsd[1] - 0.4) < 1e-12 and abs(st.r_sum - 0.8) < 1e-12


def test_dead_end_push_and_count(oracle):  # test_push_engines.cpp:97-105, 370-377
    g = oracle.build_graph_from_edges([(0, 1), (0, 2), (2, 0)])
    res, rsd, st = np.zeros(3), np.array([1.0, 0, 0]), OgStats(1.0, 0, 0, 0, 0)
    oracle.push_once(g, 0, 0.2, res, rsd, st, 0)
    assert st.pushes == 2
    oracle.push_once(g, 0, 0.2, res, rsd, st, 1)
    assert st.pushes == 3
    g2 = oracle.build_graph_from_edges([(0, 1), (2, 0)])
    res, rsd, st = np.zeros(3), np.array([1.0, 0, 0]), OgStats(1.0, 0, 0, 0, 0)
    oracle.push_once(g2, 0, 0.2, res, rsd, st, 0)
    oracle.push_once(g2, 0, 0.2, res, rsd, st, 1)
    assert abs(res[1] - 0.16) < 1e-12 and abs(rsd[0] - 0.64) < 1e-12


def test_power_iteration_lambda_ge_1(oracle, g5):  # test_push_engines.cpp:148-154
    out = oracle.power_iteration(g5, 0, 0.2, 1.0)
    assert np.all(out.estimates == 0) and out.r_sum == 1.0 and out.residues[0] == 1.0


@pytest.mark.parametrize("seed", [31, 32])
def test_power_iteration_decay(oracle, seed):  # test_push_engines.cpp:156-166
    g = oracle.random_graph(60, 1, 5, seed)
    out = oracle.power_iteration(g, 3, 0.2, 1e-8, trace_cap=200)
    assert len(out.trace) >= 60
    for j in range(1, 61):
        assert abs(out.trace[j - 1] - 0.8 ** j) < 1e-12 * j


def test_power_iteration_count(oracle):  # test_push_engines.cpp:168-176
    g = oracle.random_graph(40, 1, 4, 7)
    out = oracle.power_iteration(g, 0, 0.2, 1e-6)
    assert out.iterations == math.ceil(math.log(1 / 1e-6) / math.log(1 / 0.8))


def test_fifo_running_example(oracle, g5):  # test_push_engines.cpp:209-221
    out = oracle.fifo_forward_push(g5, 0, 0.2, 0.099)
    assert np.max(np.abs(out.estimates - [0.2, 0.08, 0.096, 0, 0])) < 1e-12
    assert out.estimates[3] == 0.0 and out.estimates[4] == 0.0
    assert np.max(np.abs(out.residues - [0.08, 0.192, 0.0, 0.272, 0.08])) < 1e-12


@pytest.mark.parametrize("seed", [41, 42, 43])
def test_fifo_natural_stop(oracle, seed):  # test_push_engines.cpp:223-235
    g = oracle.random_graph(80, 0, 4, seed)
    s = (seed * 13) % g.n
    out = oracle.fifo_forward_push(g, s, 0.2, 1e-5)
    deg_eff = np.maximum(g.degrees(), 1)
    assert np.all(out.residues <= deg_eff * 1e-5)
    assert out.r_sum <= g.m_eff * 1e-5 * (1 + 1e-12)


def test_fifo_rmax_ge_1(oracle, g5):  # test_push_engines.cpp:255-269
    out = oracle.fifo_forward_push(g5, 0, 0.2, 0.49)
    assert abs(out.estimates[0] - 0.2) < 1e-12 and out.pushes == 2
    out = oracle.fifo_forward_push(g5, 0, 0.2, 1.0)
    assert np.all(out.estimates == 0) and out.pushes == 0 and out.r_sum == 1.0


def test_iterative_engines_reach_golden(oracle, g5):  # test_push_engines.cpp:237-253
    lam = 1e-8
    assert np.abs(oracle.power_iteration(g5, 0, 0.2, lam).estimates - FIVE_NODE_PI0).sum() <= lam
    assert np.abs(oracle.sim_forward_push(g5, 0, 0.2, lam).estimates - FIVE_NODE_PI0).sum() <= lam
    fifo = oracle.fifo_forward_push(g5, 0, 0.2, lam / g5.m)
    assert np.abs(fifo.estimates - FIVE_NODE_PI0).sum() <= lam


def test_power_push_golden_and_epochs(oracle, g5):  # test_power_push.cpp:32-54
    out = oracle.power_push(g5, 0, 0.2, 1e-8)
    assert out.used_scan_phase and len(out.epoch_r_max) == 8
    for i in range(1, 9):
        assert abs(out.epoch_r_max[i - 1] - 10.0 ** -i / 13) <= 1e-12 * 10.0 ** -i / 13
    assert out.r_sum <= 1e-8
    assert np.abs(out.estimates - FIVE_NODE_PI0).sum() <= 1e-8


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_power_push_dead_ends(oracle, seed):  # test_power_push.cpp:56-68
    g = oracle.random_graph(120, 0, 3, seed)
    assert len(g.dead_ends()) > 0
    s = seed % g.n
    out = oracle.power_push(g, s, 0.2, 1e-8)
    assert out.r_sum <= 1e-8
    assert np.abs(out.estimates - oracle.exact_ppr(g, s, 0.2)).sum() <= 1e-8


def test_power_push_dead_end_source(oracle):  # test_power_push.cpp:70-76
    g = oracle.build_graph_from_edges([(0, 1), (0, 2), (2, 0)])
    out = oracle.power_push(g, 1, 0.2, 1e-8)
    assert np.abs(out.estimates - oracle.exact_ppr(g, 1, 0.2)).sum() <= 1e-8


def test_power_push_overrides(oracle):  # test_power_push.cpp:78-87
    g = oracle.random_graph(200, 1, 4, 9)
    out = oracle.power_push(g, 0, 0.2, 1e-6, epoch_num=3, scan_threshold=0)
    assert out.used_scan_phase and len(out.epoch_r_max) == 3 and out.r_sum <= 1e-6


def test_power_push_lambda_validation(oracle, g5):  # test_power_push.cpp:89-94
    for lam in (0.0, 1.5):
        with pytest.raises(InvalidArgument):
            oracle.power_push(g5, 0, 0.2, lam)


def test_queue_only_path_equals_fifo(oracle):  # test_power_push.cpp:11-30
    g = oracle.build_graph_from_edges([(v, (v + 1) % 40) for v in range(40)])
    a = oracle.power_push(g, 0, 0.2, 1e-6)
    assert not a.used_scan_phase
    b = oracle.fifo_forward_push(g, 0, 0.2, 1e-6 / g.m, 1e-6)
    assert np.array_equal(a.estimates, b.estimates) and np.array_equal(a.residues, b.residues)
    assert a.r_sum <= 1e-6


def test_refine_fixed_point_and_bound(oracle, g5):  # test_push_engines.cpp:343-368
    base = oracle.power_push(g5, 0, 0.2, 1e-6)
    r = oracle.power_push_refine(g5, 0, 0.2, 1e-6, 1.0)
    assert r.pushes == base.pushes and np.array_equal(r.estimates, base.estimates)
    for seed in (61, 62):
        g = oracle.random_graph(300, 1, 5, seed)
        r_max = 1e-7 / g.m
        lam = g.m * r_max
        before = oracle.power_push(g, 4, 0.2, lam).pushes
        out = oracle.power_push_refine(g, 4, 0.2, lam, r_max)
        assert np.all(out.residues <= np.maximum(g.degrees(), 1) * r_max)
        assert out.pushes - before <= lam / (0.2 * r_max) * 1.01


def test_walk_budget(oracle):  # test_walks.cpp:14-37
    assert oracle.compute_walk_budget(5, 0.5, 0.2) == 151
    for eps in (0.1, 0.3, 0.5, 1.0):
        ratio = oracle.walk_budget_real(1000, eps / 2, 1e-3) / oracle.walk_budget_real(1000, eps, 1e-3)
        assert 3.4 < ratio <= 4.0
    for bad in ((5, 0.0, 0.2), (5, 0.5, 0.0), (5, 0.5, 1.5), (1, 0.5, 0.2)):
        with pytest.raises(InvalidArgument):
            oracle.compute_walk_budget(*bad)


def test_speedppr_pure_sampling_branch(oracle, g5):  # test_speedppr.cpp:162-173
    assert oracle.compute_walk_budget(5, 3.0, 0.2) <= g5.m_eff
    out = oracle.speedppr_query(g5, 0, 0.2, 3.0, seed=9)
    assert out.pushes == 0 and out.walks == oracle.compute_walk_budget(5, 3.0, 0.2)
    assert abs(out.estimates.sum() - 1.0) < 1e-9


def test_speedppr_normalized_deterministic(oracle):  # test_speedppr.cpp:175-185
    g = oracle.random_graph(80, 0, 4, 31)
    a = oracle.speedppr_query(g, 3, 0.2, 0.5, seed=4)
    b = oracle.speedppr_query(g, 3, 0.2, 0.5, seed=4)
    assert np.array_equal(a.estimates, b.estimates) and a.walks > 0
    assert abs(a.estimates.sum() - 1.0) < 1e-9


def test_speedppr_relative_error_golden(oracle, g5):  # test_speedppr.cpp:207-223
    exact = oracle.exact_ppr(g5, 0, 0.2)
    clean = sum(oracle.compare_to_truth(oracle.speedppr_query(g5, 0, 0.2, 0.5, seed=s).estimates,
                                        exact, 0.2, 0.5).violations == 0 for s in range(20))
    assert clean >= 19


def test_index_shape(oracle, g5):  # test_walks.cpp:71-95
    idx = oracle.build_index(g5, 0.2, 7)
    assert len(idx) == 13 and np.all(idx < 5)
    g = oracle.random_graph(60, 0, 4, 17)
    assert len(oracle.build_index(g, 0.2, 7)) == g.m


def test_philox_known_answers(oracle):
    """Random123 philox4x32-10 known-answer vectors (kat_vectors)."""
    assert list(oracle.philox([0, 0, 0, 0], [0, 0])) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C,
                                                         0x9B00DBD8]
    assert list(oracle.philox([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)) == [0x408F276D, 0x41C83B0E,
                                                                       0xA20BC7C6, 0x6D5451FD]
    assert list(oracle.philox([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                              [0xA4093822, 0x299F31D0])) == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                             0x24126EA1]


def test_philox_walk_distribution(oracle, g5):
    """Walk terminals of the product's Philox walk follow the exact PPR
    (the analogue of test_walks.cpp:48-58 for the counter-based stream)."""
    exact = oracle.exact_ppr(g5, 0, 0.2)
    hits = np.zeros(5)
    walks = 200000
    for k in range(walks):
        hits[oracle.philox_walk(g5, 0, 0, 0.2, 42, k, 0, 0)] += 1
    assert np.max(np.abs(hits / walks - exact)) < 0.005
