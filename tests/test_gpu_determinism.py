"""PPRG_DETERMINISTIC (the reference's rerun guarantee, SPEC.md
"two runs with identical argv produce identical result files"): with the mode
on, every engine returns bitwise-identical reserves, residues and r_sum on a
rerun, and still meets the parity bar against the CPU oracle (per node
|pi_gpu - pi_ref| <= lambda, r_sum <= lambda). Runs are interleaved with other
queries so the device schedule differs between the two runs."""
import numpy as np
import pytest

from oracle.pyoracle import CSR

pytestmark = pytest.mark.gpu

ALPHA, LAM = 0.2, 1e-8


@pytest.fixture(scope="module")
def P():
    import paper_2101_03652_b200 as P
    P.load_library()
    yield P
    P.set_deterministic(False)


def gcsr(g) -> CSR:
    return CSR(g.out_offsets().copy(), g.out_neighbors().copy())


def same(a, b):
    return a.tobytes() == b.tobytes()


def twice(P, fn, perturb):
    with P.deterministic():
        first = fn()
        perturb()
        second = fn()
    return first, second


def check_vectors(o1, o2):
    for a, b in zip(o1, o2):
        assert same(a.estimates, b.estimates)
        assert same(a.residues, b.residues)
        assert a.achieved_r_sum == b.achieved_r_sum
        assert a.sweeps == b.sweeps and a.pushes == b.pushes


@pytest.mark.parametrize("scale,k", [(13, 64), (13, 7), (13, 2), (13, 1), (15, 32)])
def test_power_push_batch_reruns_bit_identical(P, oracle, scale, k):
    g = P.generate_rmat(scale, 8, 3)
    src = P.sample_sources(np.diff(g.out_offsets()), k, 5)
    other = P.sample_sources(np.diff(g.out_offsets()), 5, 9)
    (o1, _), (o2, _) = twice(P, lambda: P.power_push_batch(g, src, ALPHA, LAM),
                             lambda: P.power_push_batch(g, other, ALPHA, LAM))
    check_vectors(o1, o2)
    csr = gcsr(g)
    for i in (0, k - 1):
        ref = oracle.power_push(csr, int(src[i]), ALPHA, LAM)
        assert o1[i].achieved_r_sum <= LAM
        assert float(np.max(np.abs(o1[i].estimates - ref.estimates))) <= LAM


def test_power_push_scan_phase_and_queue_limit(P, oracle):
    # a small queue limit: the local phase stops on it (level boundaries in
    # deterministic mode) and the global phase finishes
    g = P.generate_rmat(12, 8, 4)
    src = P.sample_sources(np.diff(g.out_offsets()), 8, 2)
    (o1, _), (o2, _) = twice(P, lambda: P.power_push_batch(g, src, ALPHA, LAM, scan_threshold=50),
                             lambda: P.power_push_batch(g, src[:3], ALPHA, LAM))
    check_vectors(o1, o2)
    assert all(o.used_scan_phase for o in o1)
    csr = gcsr(g)
    for i in range(len(src)):
        ref = oracle.power_push(csr, int(src[i]), ALPHA, LAM, scan_threshold=50)
        assert o1[i].achieved_r_sum <= LAM
        assert float(np.max(np.abs(o1[i].estimates - ref.estimates))) <= LAM


def test_power_push_k1_warp_tasks_deterministic(P, oracle):
    # >= 4M in-edges: K = 1 sweeps run as warp tasks
    g = P.generate_rmat(18, 16, 1)
    src = P.sample_sources(np.diff(g.out_offsets()), 1, 1)
    (o1, _), (o2, _) = twice(P, lambda: P.power_push_batch(g, src, ALPHA, LAM),
                             lambda: P.power_push_batch(g, src, ALPHA, 1e-4))
    check_vectors(o1, o2)
    ref = oracle.power_push(gcsr(g), int(src[0]), ALPHA, LAM)
    assert o1[0].achieved_r_sum <= LAM
    assert float(np.max(np.abs(o1[0].estimates - ref.estimates))) <= LAM


def test_dead_end_source_deterministic(P, oracle):
    csr = oracle.random_graph(3000, 0, 5, 11)
    dead = csr.dead_ends()
    assert len(dead) > 0
    g = P.Graph(csr.offsets, csr.neighbors)
    src = np.array([dead[0], 0, 17], np.uint32)
    (o1, _), (o2, _) = twice(P, lambda: P.power_push_batch(g, src, ALPHA, LAM),
                             lambda: P.power_push_batch(g, src[1:], ALPHA, LAM))
    check_vectors(o1, o2)
    for i, s in enumerate(src):
        ref = oracle.power_push(csr, int(s), ALPHA, LAM)
        assert float(np.max(np.abs(o1[i].estimates - ref.estimates))) <= LAM


def test_powitr_simfwd_fifo_ground_truth_deterministic(P, oracle):
    csr = oracle.random_graph(4000, 0, 8, 21)
    g = P.Graph(csr.offsets, csr.neighbors)
    src = np.array([3, 100, 2000], np.uint32)
    perturb = lambda: P.power_push_batch(g, src, ALPHA, 1e-6)  # noqa: E731
    (a1, _), (a2, _) = twice(P, lambda: P.power_iteration_batch(g, src, ALPHA, LAM), perturb)
    check_vectors(a1, a2)
    ref = oracle.power_iteration(csr, 3, ALPHA, LAM)
    assert float(np.max(np.abs(a1[0].estimates - ref.estimates))) <= 1e-12
    b1, b2 = twice(P, lambda: P.sim_forward_push(g, 100, ALPHA, LAM), perturb)
    check_vectors([b1], [b2])
    r_max = 1e-9 / csr.m_eff
    c1, c2 = twice(P, lambda: P.fifo_forward_push(g, 2000, ALPHA, r_max), perturb)
    check_vectors([c1], [c2])
    ref = oracle.fifo_forward_push(csr, 2000, ALPHA, r_max)
    assert float(np.max(np.abs(c1.estimates - ref.estimates))) <= 1e-9
    # ground truth (power iteration at lambda = 1e-17) on a graph the dense
    # oracle solves (n <= 2000)
    small = oracle.random_graph(1500, 0, 8, 22)
    gs = P.Graph(small.offsets, small.neighbors)
    d1, d2 = twice(P, lambda: P.ground_truth(gs, 3, ALPHA), perturb)
    assert same(d1.estimates, d2.estimates)
    assert float(np.abs(d1.estimates - oracle.exact_ppr(small, 3, ALPHA)).sum()) <= 1e-12


def test_speedppr_and_refine_deterministic(P, oracle):
    g = P.generate_rmat(14, 8, 6)
    idx = P.build_index(g, ALPHA, 4)
    src = P.sample_sources(np.diff(g.out_offsets()), 16, 4)
    cfg = P.QueryConfig(epsilon=0.5, seed=7)
    (s1, _), (s2, _) = twice(P, lambda: P.speedppr_batch(g, src, cfg, idx),
                             lambda: P.speedppr_batch(g, src[:4], cfg, idx))
    for a, b in zip(s1, s2):
        assert same(a.estimates, b.estimates)
        assert a.walks == b.walks
        assert abs(a.estimates.sum() - 1.0) < 1e-6
    # index-free (fresh Philox walks for every walk)
    t1, t2 = twice(P, lambda: P.speedppr_query(g, int(src[0]), cfg, None),
                   lambda: P.speedppr_query(g, int(src[1]), cfg, None))
    assert same(t1.estimates, t2.estimates)
    # refine from a caller state
    base = P.power_push(g, int(src[0]), ALPHA, 1e-4)
    r1, r2 = twice(P, lambda: P.refine(g, int(src[0]), ALPHA, 1e-9, base),
                   lambda: P.refine(g, int(src[1]), ALPHA, 1e-8, base))
    check_vectors([r1], [r2])


def test_fast_mode_unaffected(P, oracle):
    # the default (nondeterministic) mode still meets parity after deterministic calls
    P.set_deterministic(False)
    g = P.generate_rmat(13, 8, 3)
    src = P.sample_sources(np.diff(g.out_offsets()), 4, 5)
    outs, _ = P.power_push_batch(g, src, ALPHA, LAM)
    ref = oracle.power_push(gcsr(g), int(src[0]), ALPHA, LAM)
    assert float(np.max(np.abs(outs[0].estimates - ref.estimates))) <= LAM
