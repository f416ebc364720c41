"""Pin the oracle restatement bit-for-bit against the reference library itself
(oracle/_ref/libppr_ref.so, compiled unchanged from /root/reference). Skipped
where that library was not built."""
import numpy as np
import pytest

from oracle.pyoracle import five_node_edges


def _rand_edges(seed, n_ids, count, sparse=False):
    rng = np.random.default_rng(seed)
    e = rng.integers(0, n_ids, size=(count, 2), dtype=np.uint64)
    if sparse:
        e = e * np.uint64(1000003) + np.uint64(7)
    return e


def test_rng_stream_bit_exact(oracle, ref):
    for seed in (0, 1, 5489, 2**63 + 11):
        assert np.array_equal(oracle.rng_draws(seed, 2000), ref.rng_draws(seed, 2000))
        for bound in (1, 2, 3, 7, 1000, 2**33 + 1, 2**63 + 5):
            assert np.array_equal(oracle.rng_draws(seed, 500, bound), ref.rng_draws(seed, 500, bound))


@pytest.mark.parametrize("seed,sparse", [(1, False), (2, True), (3, False)])
def test_build_graph_bit_exact(oracle, ref, seed, sparse):
    edges = _rand_edges(seed, 300, 2000, sparse)  # duplicates + self-loops included
    a = oracle.build_graph_from_edges(edges)
    b = ref.graph_from_edges(edges)
    bc = b.csr()
    assert np.array_equal(a.offsets, bc.offsets) and np.array_equal(a.neighbors, bc.neighbors)
    assert np.array_equal(a.dead_ends(), b.dead_ends())


def test_random_graph_bit_exact(oracle, ref):
    for args in ((120, 0, 3, 101), (400, 0, 5, 99), (60, 1, 5, 31)):
        a = oracle.random_graph(*args)
        b = ref.random_graph(*args).csr()
        assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.neighbors, b.neighbors)


def _graphs(oracle):
    yield oracle.build_graph_from_edges(five_node_edges()), 0
    for seed in (101, 7, 99):
        g = oracle.random_graph(150 + seed, 0, 5, seed)
        yield g, seed % g.n


def _same(a, b):
    assert np.array_equal(a.estimates, b.estimates)
    assert np.array_equal(a.residues, b.residues)
    assert a.r_sum == b.r_sum and a.pushes == b.pushes


def test_engines_bit_exact(oracle, ref):
    for g, s in _graphs(oracle):
        rg = ref.graph(g)
        _same(oracle.power_iteration(g, s, 0.2, 1e-8), rg.power_iteration(s, 0.2, 1e-8))
        _same(oracle.sim_forward_push(g, s, 0.2, 1e-8), rg.sim_forward_push(s, 0.2, 1e-8))
        _same(oracle.fifo_forward_push(g, s, 0.2, 1e-9 / g.m),
              rg.fifo_forward_push(s, 0.2, 1e-9 / g.m))
        for lam in (1e-4, 1e-8, 1e-12):
            a, b = oracle.power_push(g, s, 0.2, lam), rg.power_push(s, 0.2, lam)
            _same(a, b)
            assert a.used_scan_phase == b.used_scan_phase
            assert np.array_equal(a.epoch_r_max, b.epoch_r_max)
        _same(oracle.power_push(g, s, 0.2, 1e-7, 3, 0), rg.power_push(s, 0.2, 1e-7, 3, 0))
        _same(oracle.power_push_refine(g, s, 0.2, 0.05, 1e-7),
              rg.power_push_refine(s, 0.2, 0.05, 1e-7))


def test_exact_and_index_and_speedppr_bit_exact(oracle, ref):
    for g, s in _graphs(oracle):
        rg = ref.graph(g)
        assert np.array_equal(oracle.exact_ppr(g, s, 0.2), rg.exact_ppr(s, 0.2))
        idx = oracle.build_index(g, 0.2, 21)
        assert np.array_equal(idx, rg.build_index(0.2, 21))
        for eps in (0.5, 3.0):
            a = oracle.speedppr_query(g, s, 0.2, eps, seed=4)
            b = rg.speedppr_query(s, 0.2, eps, seed=4)
            assert np.array_equal(a.estimates, b.estimates) and a.walks == b.walks
            a = oracle.speedppr_query(g, s, 0.2, eps, seed=4, index=idx)
            b = rg.speedppr_query(s, 0.2, eps, seed=4, index=idx, index_seed=21)
            assert np.array_equal(a.estimates, b.estimates) and a.walks == b.walks


def test_power_push_vs_ground_truth_within_lambda(oracle, ref):
    g = oracle.random_graph(1500, 0, 6, 5)
    rg = ref.graph(g)
    truth = rg.ground_truth(11, 0.2)
    out = oracle.power_push(g, 11, 0.2, 1e-8)
    assert out.r_sum <= 1e-8
    assert np.max(np.abs(out.estimates - truth)) <= 1e-8
