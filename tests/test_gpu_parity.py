"""GPU parity: every engine through the C ABI (lib/libpprg.so) against the CPU
oracle on the same inputs. Tolerances follow the north star: CSR / degree /
index structures bit-exact; high-precision fp64 results per node
|pi_gpu - pi_ref| <= lambda with final r_sum <= lambda; SpeedPPR within
relative error epsilon of the truth for nodes with pi >= mu."""
import math

import numpy as np
import pytest

from oracle.pyoracle import CSR, FIVE_NODE_PI0, five_node_edges

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2101_03652_b200 as P
    import ctypes
    L = P.load_library()
    cnt = ctypes.c_int()
    assert L.pprg_device_count(ctypes.byref(cnt)) == 0 and cnt.value >= 1, "no CUDA device"
    return P


def gcsr(g) -> CSR:
    return CSR(g.out_offsets().copy(), g.out_neighbors().copy())


def dev(P, csr: CSR):
    return P.Graph(csr.offsets, csr.neighbors)


# ---- (1) CSR build and device residency --------------------------------------
@pytest.mark.parametrize("seed,sparse", [(1, False), (2, True), (3, False)])
def test_build_from_edges_bit_exact(P, oracle, seed, sparse):
    rng = np.random.default_rng(seed)
    e = rng.integers(0, 500, size=(4000, 2), dtype=np.uint64)
    if sparse:
        e = e * np.uint64(1000003) + np.uint64(11)
    ref = oracle.build_graph_from_edges(e)
    g = P.build_graph_from_edges(e)
    assert g.n() == ref.n and g.m() == ref.m
    assert np.array_equal(g.out_offsets(), ref.offsets)
    assert np.array_equal(g.out_neighbors(), ref.neighbors)
    assert np.array_equal(g.dead_ends(), ref.dead_ends())


def test_graph_validation_messages(P):
    with pytest.raises(P.DataError, match="neighbor id out of range"):
        P.Graph([0, 1], [5])
    with pytest.raises(P.DataError, match="non-decreasing"):
        P.Graph([0, 2, 1, 3], [0, 1, 2])
    with pytest.raises(P.DataError, match="empty"):
        P.build_graph_from_edges(np.zeros((0, 2), np.uint64))


def test_transpose_is_exact(P, oracle):
    g = oracle.random_graph(3000, 0, 9, 5)
    d = dev(P, g)
    ioff, inbr = d.transpose()
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.offsets).astype(np.int64))
    order = np.lexsort((src, g.neighbors))  # by dst, then src ascending
    assert np.array_equal(inbr, src[order])
    assert np.array_equal(ioff, np.concatenate([[0], np.cumsum(np.bincount(g.neighbors, minlength=g.n))]).astype(np.uint64))


@pytest.mark.parametrize("scale,ef,seed", [(10, 8, 1), (17, 8, 1)])
def test_rmat_generator_csr_bit_exact(P, oracle, scale, ef, seed):
    g, edges = P.generate_rmat(scale, ef, seed, return_edges=True)
    assert np.all(edges[:, 0] != edges[:, 1])
    keys = (edges[:, 0] << np.uint64(32)) | edges[:, 1]
    assert np.all(np.diff(keys.astype(np.float64)) > 0) or np.all(keys[1:] > keys[:-1])
    ref = oracle.build_graph_from_edges(edges)
    assert np.array_equal(g.out_offsets(), ref.offsets)
    assert np.array_equal(g.out_neighbors(), ref.neighbors)


def test_chung_lu_generator_csr_bit_exact(P, oracle):
    g, edges = P.generate_chung_lu(1 << 12, 30 << 12, 4, return_edges=True)
    ref = oracle.build_graph_from_edges(edges)
    assert np.array_equal(g.out_offsets(), ref.offsets)
    assert np.array_equal(g.out_neighbors(), ref.neighbors)


# ---- PowItr / SimFwdPush -------------------------------------------------------
@pytest.mark.parametrize("seed", [31, 32, 101])
def test_power_iteration_matches_oracle(P, oracle, seed):
    g = oracle.random_graph(400, 0 if seed == 101 else 1, 5, seed)
    d = dev(P, g)
    s = seed % g.n
    ref = oracle.power_iteration(g, s, 0.2, 1e-8)
    got = P.power_iteration(d, s, 0.2, 1e-8)
    assert got.sweeps == ref.iterations and got.pushes == ref.pushes
    assert np.max(np.abs(got.estimates - ref.estimates)) <= 1e-12
    assert np.max(np.abs(got.residues - ref.residues)) <= 1e-12
    assert abs(got.achieved_r_sum - ref.r_sum) <= 1e-12


def test_power_iteration_lambda_ge_1(P, oracle):  # test_push_engines.cpp:148-154
    d = P.build_graph_from_edges(five_node_edges())
    out = P.power_iteration(d, 0, 0.2, 1.0)
    assert np.all(out.estimates == 0) and out.achieved_r_sum == 1.0 and out.residues[0] == 1.0


def test_sim_forward_push_matches_oracle(P, oracle):
    g = oracle.random_graph(300, 0, 4, 7)
    d = dev(P, g)
    ref = oracle.sim_forward_push(g, 3, 0.2, 1e-9)
    got = P.sim_forward_push(d, 3, 0.2, 1e-9)
    assert got.pushes == ref.pushes
    assert np.max(np.abs(got.estimates - ref.estimates)) <= 1e-12


# ---- PowerPush ------------------------------------------------------------------
def check_hp(got, ref, lam, slack=1e-15):
    assert got.achieved_r_sum <= lam
    assert np.max(np.abs(got.estimates - ref.estimates)) <= lam + slack
    assert np.abs(got.estimates - ref.estimates).sum() <= got.achieved_r_sum + ref.r_sum + 1e-13
    assert np.all(got.residues >= 0)
    assert abs(got.estimates.sum() + got.residues.sum() - 1.0) <= 1e-9
    assert abs(got.residues.sum() - got.achieved_r_sum) <= 1e-12


def test_power_push_five_node_golden(P):  # test_power_push.cpp:32-54
    d = P.build_graph_from_edges(five_node_edges())
    tr = P.PowerPushTrace()
    out = P.power_push(d, 0, 0.2, 1e-8, P.QueryConfig(), tr)
    assert tr.used_scan_phase and len(tr.epoch_r_max) == 8
    for i in range(1, 9):
        assert abs(tr.epoch_r_max[i - 1] - 10.0 ** -i / 13) <= 1e-12 * 10.0 ** -i / 13
    assert out.achieved_r_sum <= 1e-8
    assert np.abs(out.estimates - FIVE_NODE_PI0).sum() <= 1e-8


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_power_push_dead_ends_vs_exact(P, oracle, seed):  # test_power_push.cpp:56-68
    g = oracle.random_graph(120, 0, 3, seed)
    s = seed % g.n
    out = P.power_push(dev(P, g), s, 0.2, 1e-8)
    assert out.achieved_r_sum <= 1e-8
    assert np.abs(out.estimates - oracle.exact_ppr(g, s, 0.2)).sum() <= 1e-8
    check_hp(out, oracle.power_push(g, s, 0.2, 1e-8), 1e-8)


def test_power_push_dead_end_source(P, oracle):  # test_power_push.cpp:70-76
    g = oracle.build_graph_from_edges([(0, 1), (0, 2), (2, 0)])
    out = P.power_push(dev(P, g), 1, 0.2, 1e-8)
    assert np.abs(out.estimates - oracle.exact_ppr(g, 1, 0.2)).sum() <= 1e-8


def test_power_push_overrides_and_validation(P, oracle):  # test_power_push.cpp:78-94
    g = oracle.random_graph(200, 1, 4, 9)
    d = dev(P, g)
    tr = P.PowerPushTrace()
    out = P.power_push(d, 0, 0.2, 1e-6, P.QueryConfig(epoch_num=3, scan_threshold=0), tr)
    assert tr.used_scan_phase and len(tr.epoch_r_max) == 3 and out.achieved_r_sum <= 1e-6
    for lam in (0.0, 1.5):
        with pytest.raises(P.InvalidArgument):
            P.power_push(d, 0, 0.2, lam)
    with pytest.raises(P.InvalidArgument):
        P.power_push(d, g.n, 0.2, 1e-6)


def test_queue_only_path(P, oracle):  # test_power_push.cpp:11-30
    g = oracle.build_graph_from_edges([(v, (v + 1) % 40) for v in range(40)])
    d = dev(P, g)
    tr = P.PowerPushTrace()
    a = P.power_push(d, 0, 0.2, 1e-6, P.QueryConfig(), tr)
    assert not tr.used_scan_phase
    b = oracle.fifo_forward_push(g, 0, 0.2, 1e-6 / g.m, 1e-6)
    assert np.max(np.abs(a.estimates - b.estimates)) <= 1e-15
    assert a.achieved_r_sum <= 1e-6


@pytest.mark.parametrize("lam", [1e-4, 1e-8, 1e-11])
def test_power_push_random_graphs_vs_oracle(P, oracle, lam):
    for seed in (5, 6):
        g = oracle.random_graph(2500, 0, 8, seed)
        d = dev(P, g)
        for s in (0, 17, 1234):
            check_hp(P.power_push(d, s, 0.2, lam), oracle.power_push(g, s, 0.2, lam), lam)


@pytest.mark.parametrize("k", [3, 8, 32, 64])
def test_power_push_column_block(P, oracle, k):
    g = oracle.random_graph(1500, 0, 6, 11)
    d = dev(P, g)
    srcs = np.arange(k, dtype=np.uint32) * 7 % g.n
    outs, cs = P.power_push_batch(d, srcs, 0.2, 1e-8)
    assert cs.sweep_launches >= 1
    for s, o in zip(srcs, outs):
        check_hp(o, oracle.power_push(g, int(s), 0.2, 1e-8), 1e-8)


def test_power_iteration_column_block(P, oracle):
    g = oracle.random_graph(800, 0, 6, 12)
    d = dev(P, g)
    srcs = [0, 5, 9, 100, 799]
    outs, _ = P.power_iteration_batch(d, srcs, 0.2, 1e-8)
    for s, o in zip(srcs, outs):
        ref = oracle.power_iteration(g, s, 0.2, 1e-8)
        assert np.max(np.abs(o.estimates - ref.estimates)) <= 1e-12


def test_rmat17_power_push_vs_oracle(P, oracle):
    """Config-1 graph (R-MAT scale 17, ef 8, seed 1) against the CPU oracle."""
    d, edges = P.generate_rmat(17, 8, 1, return_edges=True)
    g = gcsr(d)
    srcs = P.sample_sources(np.diff(g.offsets), 4, 1)
    outs, cs = P.power_push_batch(d, srcs, 0.2, 1e-8)
    for s, o in zip(srcs, outs):
        ref = oracle.power_push(g, int(s), 0.2, 1e-8)
        check_hp(o, ref, 1e-8)
        assert o.used_scan_phase and ref.used_scan_phase


# ---- FIFO forward push ----------------------------------------------------------------
def test_fifo_running_example(P, oracle):  # test_push_engines.cpp:209-221
    """The reference pops one node at a time; the GPU drains a whole FIFO level
    per launch, so the push order (not the push rule) differs and the coarse
    r_max = 0.099 trace is not reproduced value for value. What is order-
    independent: natural stop, conservation, and est <= pi with
    pi - est <= r_sum pointwise, so two engines differ by at most the larger
    residual mass at every node."""
    g = oracle.build_graph_from_edges(five_node_edges())
    d = P.build_graph_from_edges(five_node_edges())
    out = P.fifo_forward_push(d, 0, 0.2, 0.099)
    ref = oracle.fifo_forward_push(g, 0, 0.2, 0.099)
    assert np.all(out.residues <= np.diff(g.offsets) * 0.099)
    assert abs(out.estimates.sum() + out.residues.sum() - 1) < 1e-12
    assert np.all(out.estimates <= FIVE_NODE_PI0 + 1e-15)
    assert np.all(np.abs(out.estimates - ref.estimates) <= max(out.achieved_r_sum, ref.r_sum))
    assert abs(out.estimates[0] - 0.2) < 1e-12  # the first pop is the source in both
    out = P.fifo_forward_push(d, 0, 0.2, 1.0)
    assert np.all(out.estimates == 0) and out.pushes == 0 and out.achieved_r_sum == 1.0
    out = P.fifo_forward_push(d, 0, 0.2, 0.49)  # test_push_engines.cpp:256-261
    assert abs(out.estimates[0] - 0.2) < 1e-12 and out.pushes == 2
    with pytest.raises(P.InvalidArgument):
        P.fifo_forward_push(d, 0, 0.2, 0.0)


@pytest.mark.parametrize("seed", [41, 42, 43])
def test_fifo_natural_stop(P, oracle, seed):  # test_push_engines.cpp:223-235
    g = oracle.random_graph(800, 0, 4, seed)
    s = (seed * 13) % g.n
    out = P.fifo_forward_push(dev(P, g), s, 0.2, 1e-7)
    assert np.all(out.residues <= np.maximum(np.diff(g.offsets), 1) * 1e-7)
    assert out.achieved_r_sum <= g.m_eff * 1e-7 * (1 + 1e-12)
    assert abs(out.estimates.sum() + out.residues.sum() - 1) < 1e-9


# ---- SpeedPPR --------------------------------------------------------------------
def test_walk_terminals_bit_exact(P, oracle):
    g = oracle.random_graph(300, 0, 5, 21)
    d = dev(P, g)
    rng = np.random.default_rng(0)
    starts = rng.integers(0, g.n, 2000).astype(np.uint32)
    ks = rng.integers(0, 50, 2000).astype(np.uint32)
    got = P.walk_terminals(d, starts, ks, starts, 7, 7, 0.2, 99)
    want = [oracle.philox_walk(g, int(a), 7, 0.2, 99, int(k), int(a), 7) for a, k in zip(starts, ks)]
    assert np.array_equal(got, np.asarray(want, np.uint32))


@pytest.mark.parametrize("seed", [7, 8])
def test_index_bit_exact_and_shape(P, oracle, seed):  # test_walks.cpp:71-110
    g = oracle.random_graph(500, 0, 6, 17)
    d = dev(P, g)
    idx = P.build_index(d, 0.2, seed)
    ep = idx.endpoints()
    assert np.array_equal(ep, oracle.philox_build_index(g, 0.2, seed))
    assert len(ep) == g.m and np.all(ep < g.n)
    for v in g.dead_ends()[:5]:
        assert len(idx.endpoints_of(int(v))) == 0
    assert np.array_equal(ep, P.build_index(d, 0.2, seed).endpoints())


def test_walk_budget(P):  # test_walks.cpp:14-37
    assert P.compute_walk_budget(5, 0.5, 0.2) == 151
    with pytest.raises(P.InvalidArgument):
        P.compute_walk_budget(1, 0.5, 0.2)


def test_speedppr_pure_sampling_branch(P):  # test_speedppr.cpp:162-173
    d = P.build_graph_from_edges(five_node_edges())
    out = P.speedppr_query(d, 0, P.QueryConfig(epsilon=3.0, seed=9))
    assert out.pushes == 0 and out.walks == P.compute_walk_budget(5, 3.0, 0.2)
    assert abs(out.estimates.sum() - 1.0) < 1e-9


def test_speedppr_requires_epsilon_and_alpha_match(P):  # test_speedppr.cpp:148-160
    d = P.build_graph_from_edges(five_node_edges())
    with pytest.raises(P.InvalidArgument):
        P.speedppr_query(d, 0, P.QueryConfig())
    idx = P.build_index(d, 0.15, 3)
    with pytest.raises(P.DataError):
        P.speedppr_query(d, 0, P.QueryConfig(epsilon=0.5), idx)


@pytest.mark.parametrize("use_index", [False, True])
def test_speedppr_relative_error(P, oracle, use_index):
    """Acceptance criteria 8-9 analogue: >= 95% of seeded runs have no node
    with pi >= 1/n off by more than epsilon (acceptance.cpp:223-290)."""
    g = oracle.random_graph(1000, 0, 6, 3)
    d = dev(P, g)
    idx = P.build_index(d, 0.2, 5) if use_index else None
    clean = 0
    for seed in range(20):
        s = (seed * 37) % g.n
        truth = oracle.exact_ppr(g, s, 0.2)
        out = P.speedppr_query(d, s, P.QueryConfig(epsilon=0.5, seed=seed), idx)
        assert abs(out.estimates.sum() - 1.0) < 1e-9
        rep = oracle.compare_to_truth(out.estimates, truth, 1.0 / g.n, 0.5)
        clean += rep.violations == 0
    assert clean >= 19


def test_speedppr_unbiased(P, oracle):
    """Mean of many seeded runs approaches the exact PPR (acceptance.cpp:294-321)."""
    g = oracle.random_graph(60, 1, 4, 11)
    d = dev(P, g)
    truth = oracle.exact_ppr(g, 2, 0.2)
    runs = np.stack([P.speedppr_query(d, 2, P.QueryConfig(epsilon=1.0, seed=s)).estimates
                     for s in range(300)])
    se = runs.std(axis=0, ddof=1) / math.sqrt(len(runs))
    assert np.all(np.abs(runs.mean(axis=0) - truth) <= 4 * se + 1e-12)


@pytest.mark.parametrize("use_index", [False, True])
def test_speedppr_batch_push_branch(P, oracle, use_index):
    """64 sources as one column block on a skewed graph where W > m_eff (push +
    refine + MC branch, speedppr.cpp:103-110): every query sums to 1 and at
    most one in 20 has a node with pi >= 1/n off by more than epsilon."""
    g = P.generate_rmat(11, 8, 21)
    n = g.n()
    c = gcsr(g)
    src = P.sample_sources(np.diff(g.out_offsets()), 64, 21)
    idx = P.build_index(g, 0.2, 8) if use_index else None
    outs, _ = P.speedppr_batch(g, src, P.QueryConfig(epsilon=0.5, seed=5), idx)
    assert P.compute_walk_budget(n, 0.5, 1.0 / n) > g.m() + len(g.dead_ends())
    clean = 0
    for q in range(0, 64, 4):
        est = outs[q].estimates
        assert abs(est.sum() - 1.0) < 1e-9 and outs[q].pushes > 0 and outs[q].walks > 0
        truth = oracle.exact_ppr(c, int(src[q]), 0.2)
        clean += oracle.compare_to_truth(est, truth, 1.0 / n, 0.5).violations == 0
    assert clean >= 15


# ---- (5) vertex-partitioned power_push (configs[4]) ----------------
@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("nparts,k", [(2, 1), (3, 4), (8, 1), (8, 64)])
def test_partitioned_power_push_virtual(P, oracle, nparts, k, fused):
    """P parts of one block on one GPU (sequential, slices copied between
    them) against the oracle's power_push: per node |diff| <= lambda, and the
    exact all-part r_sum <= lambda."""
    from paper_2101_03652_b200.partition import run_virtual_parts
    g = P.generate_rmat(13, 8, 31)
    c = gcsr(g)
    lam = 1e-8
    src = P.sample_sources(np.diff(g.out_offsets()), k, 31)
    res, rsd, rs, sweeps, parts = run_virtual_parts(g, nparts, src, 0.2, lam, fused=fused)
    bounds = [(p.lo, p.hi) for p in parts]
    assert bounds[0][0] == 0 and bounds[-1][1] == g.n()
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(nparts - 1))
    assert sweeps > 0
    for q in range(0, k, max(1, k // 4)):
        ref = oracle.power_push(c, int(src[q]), 0.2, lam)
        assert rs[q] <= lam
        assert abs(rsd[q].sum() - rs[q]) < 1e-12
        assert np.max(np.abs(res[q] - ref.estimates)) <= lam
        assert abs(res[q].sum() + rs[q] - 1.0) < 1e-9
    for p in parts:
        p.close()


@pytest.mark.parametrize("fused", [False, True])
def test_partitioned_local_phase_only(P, oracle, fused):
    """lambda reached by the queue phase: no sweeps, outputs still exact."""
    from paper_2101_03652_b200.partition import run_virtual_parts
    g = dev(P, oracle.random_graph(400, 1, 6, 9))
    c = gcsr(g)
    res, rsd, rs, sweeps, parts = run_virtual_parts(g, 3, [5], 0.2, 1e-2,
                                                    scan_threshold=10 ** 9, fused=fused)
    ref = oracle.power_push(c, 5, 0.2, 1e-2, scan_threshold=10 ** 9)
    assert sweeps == 0 and rs[0] <= 1e-2
    assert np.max(np.abs(res[0] - ref.estimates)) <= 1e-2
    q, _ = parts[0].stats()
    assert q[0].used_scan_phase == 0


def test_partitioned_single_rank_nccl(P, oracle):
    """The torch.distributed protocol at world size 1 over NCCL (the exchange
    degenerates to self-broadcasts, the sweeps are the real ones)."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2101_03652_b200.partition import GpuPart, run_partitioned
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = P.generate_rmat(12, 8, 5)
        c = gcsr(g)
        part = GpuPart(g, 1, 0, [int(np.argmax(np.diff(g.out_offsets())))], 0.2, 1e-8)
        n = g.n()
        out = np.zeros(n)
        r = run_partitioned(part, comm_device="cuda:0",
                            finish_kwargs=dict(reserve_ptr=out.ctypes.data))
        ref = oracle.power_push(c, int(part.src[0]), 0.2, 1e-8)
        assert r.r_sum[0] <= 1e-8 and r.bounds == [(0, n)]
        assert np.max(np.abs(out - ref.estimates)) <= 1e-8
        part.close()
    finally:
        dist.destroy_process_group()


# ---- ground_truth (metrics.cpp:44-55) ------------------------
def test_ground_truth_five_node_deterministic(P):  # test_metrics.cpp:66-76
    d = P.build_graph_from_edges(five_node_edges())
    a = P.ground_truth(d, 0, 0.2)
    b = P.ground_truth(d, 0, 0.2)
    assert np.array_equal(a.estimates, b.estimates)
    assert np.abs(a.estimates - FIVE_NODE_PI0).sum() <= 1e-12
    assert abs(a.estimates.sum() - 1.0) <= 1e-12
    assert a.achieved_r_sum <= P.GROUND_TRUTH_LAMBDA


def test_ground_truth_dead_ends(P, oracle):  # test_metrics.cpp:78-83
    g = oracle.random_graph(50, 0, 3, 71)
    d = dev(P, g)
    assert len(d.dead_ends()) > 0
    out = P.ground_truth(d, 7, 0.2)
    assert out.achieved_r_sum <= P.GROUND_TRUTH_LAMBDA
    assert np.abs(out.estimates - oracle.exact_ppr(g, 7, 0.2)).sum() <= 1e-12


def test_ground_truth_large_reproducible(P):
    """r_sum <= 1e-17 on exit, and two runs agree to the 1e-17 bound (the
    dead-end mass and r_sum are fp64 atomic sums, so bits may differ where
    the reference's sequential loop is bit-deterministic)."""
    g = P.generate_rmat(15, 16, 9)
    src = P.sample_sources(np.diff(g.out_offsets()), 3, 9)
    a, _ = P.ground_truth_batch(g, src, 0.2)
    b, _ = P.ground_truth_batch(g, src, 0.2)
    for x, y in zip(a, b):
        assert np.abs(x.estimates - y.estimates).sum() <= 2 * P.GROUND_TRUTH_LAMBDA + 1e-16
        assert x.achieved_r_sum <= P.GROUND_TRUTH_LAMBDA
        assert abs(x.estimates.sum() + x.achieved_r_sum - 1.0) < 1e-12
    # the 1e-8 PowerPush answer is within lambda of it everywhere
    pp, _ = P.power_push_batch(g, src, 0.2, 1e-8)
    for x, y in zip(a, pp):
        assert np.max(np.abs(x.estimates - y.estimates)) <= 1e-8


# ---- sweep harness progress series (sweep.cpp:25-61) --------------------------------
@pytest.mark.parametrize("algo", ["powerpush", "powitr", "simfwdpush", "fwdpush-fifo"])
def test_traced_progress_series(P, oracle, algo):
    from paper_2101_03652_b200 import harness
    g = P.generate_rmat(12, 8, 4)
    s = int(np.argmax(np.diff(g.out_offsets())))
    got, pts = harness.run_traced(g, algo, s, 0.2, 1e-8)
    assert len(pts) >= 5 and got.achieved_r_sum <= 1e-8
    push = [p.pushes for p in pts]
    assert push == sorted(push) and push[-1] <= got.pushes
    assert pts[-1].r_sum <= 1.0 and pts[0].r_sum <= 1.0
    assert all(b.time_ns >= a.time_ns for a, b in zip(pts, pts[1:]))
    ref = oracle.power_push(gcsr(g), s, 0.2, 1e-8)
    assert np.max(np.abs(got.estimates - ref.estimates)) <= 1e-8
    cp = harness.cadence_filter(pts, 4 * g.m())
    assert all(b.pushes - a.pushes >= 0 for a, b in zip(cp, cp[1:]))


# ---- refine on a caller state (push.cpp:208-222) ------------------------------------
def test_refine_from_caller_state(P, oracle):
    g = oracle.random_graph(500, 1, 5, 61)
    d = dev(P, g)
    m = int(g.offsets[-1])
    r_max = 1e-7 / m
    lam = m * r_max
    st = P.power_push(d, 4, 0.2, lam)
    out = P.refine(d, 4, 0.2, r_max, st)
    deg = np.diff(g.offsets).astype(np.float64)
    assert np.all(out.residues <= np.maximum(deg, 1) * r_max)
    assert out.pushes - st.pushes <= lam / (0.2 * r_max) * 1.01
    assert abs(out.estimates.sum() + out.residues.sum() - 1.0) < 1e-9
    ref = oracle.power_push_refine(g, 4, 0.2, lam, r_max)
    assert np.max(np.abs(out.estimates - ref.estimates)) <= lam
    # an already-inactive state is a fixed point, bit for bit
    same = P.refine(d, 4, 0.2, 1.0, st)
    assert np.array_equal(same.estimates, st.estimates) and same.pushes == st.pushes


# ---- device-direct PPRG / PPRW files (graph.cpp:115-143, walk_index.cpp:57-104) -------
def test_graph_cache_roundtrip_device_direct(P, oracle, tmp_path):
    from paper_2101_03652_b200 import formats
    g = oracle.random_graph(3000, 0, 7, 12)
    d = dev(P, g)
    ours, host = str(tmp_path / "a.pprg"), str(tmp_path / "b.pprg")
    formats.save_graph_cache(d, ours)
    formats.write_graph_cache(host, g.offsets, g.neighbors)
    assert open(ours, "rb").read() == open(host, "rb").read()
    back = formats.load_graph_cache(ours)
    assert np.array_equal(back.out_offsets(), g.offsets)
    assert np.array_equal(back.out_neighbors(), g.neighbors)
    assert np.array_equal(back.dead_ends(), d.dead_ends())


def test_graph_cache_interop_with_reference(P, ref, oracle, tmp_path):
    from paper_2101_03652_b200 import formats
    g = oracle.random_graph(800, 0, 5, 3)
    p1, p2 = str(tmp_path / "ours.pprg"), str(tmp_path / "ref.pprg")
    formats.save_graph_cache(dev(P, g), p1)
    rg = ref.load_graph_cache(p1)                # reference reads our file
    assert np.array_equal(rg.csr().offsets, g.offsets)
    rg.save(p2)                                  # and we read the reference's
    back = formats.load_graph_cache(p2)
    assert np.array_equal(back.out_neighbors(), g.neighbors)


def test_graph_cache_errors(P, tmp_path):
    from paper_2101_03652_b200 import formats
    bad = tmp_path / "bad.pprg"
    bad.write_bytes(b"XXXX\x01")
    with pytest.raises(P.DataError, match="not a graph cache"):
        formats.load_graph_cache(str(bad))
    bad.write_bytes(b"PPRG\x02")
    with pytest.raises(P.DataError, match="unsupported graph cache version"):
        formats.load_graph_cache(str(bad))
    bad.write_bytes(b"PPRG\x01" + np.array([5, 13], "<u8").tobytes() + b"\x00" * 10)
    with pytest.raises(P.DataError, match="truncated graph cache"):
        formats.load_graph_cache(str(bad))
    with pytest.raises(P.DataError, match="cannot open graph cache"):
        formats.load_graph_cache(str(tmp_path / "missing.pprg"))
    # a corrupt body is caught by the device validation (graph.cpp:24-34)
    off = np.array([0, 2, 1, 3], "<u8")
    bad.write_bytes(b"PPRG\x01" + np.array([3, 3], "<u8").tobytes() + off.tobytes() +
                    np.zeros(3, "<u4").tobytes())
    with pytest.raises(P.DataError, match="non-decreasing"):
        formats.load_graph_cache(str(bad))


def test_index_file_roundtrip_device_direct(P, oracle, tmp_path):
    from paper_2101_03652_b200 import formats
    g = oracle.random_graph(2000, 0, 6, 5)
    d = dev(P, g)
    idx = P.build_index(d, 0.2, 77)
    ours, host = str(tmp_path / "a.pprw"), str(tmp_path / "b.pprw")
    formats.save_index(idx, ours)
    formats.write_index_host(idx, host)
    assert open(ours, "rb").read() == open(host, "rb").read()
    back = formats.load_index(ours, d)
    assert np.array_equal(back.endpoints(), idx.endpoints())
    assert back.alpha() == 0.2 and back.seed() == 77
    # another graph's shape, a foreign generator id, out-of-range endpoints
    other = dev(P, oracle.random_graph(2000, 0, 6, 6))
    with pytest.raises(P.DataError, match="does not match the graph shape|slice length differs"):
        formats.load_index(ours, other)
    raw = bytearray(open(ours, "rb").read())
    raw[5] = 1
    open(host, "wb").write(bytes(raw))
    with pytest.raises(P.DataError, match="unknown generator id"):
        formats.load_index(host, d)
    raw[5] = 2
    raw[-4:] = np.array([10 ** 6], "<u4").tobytes()
    open(host, "wb").write(bytes(raw))
    with pytest.raises(P.DataError, match="endpoint id out of range"):
        formats.load_index(host, d)


def test_monte_carlo_expectation(P, oracle):
    """E[MC(state)] = reserve + sum_v residue(v) pi(v, .) (test_speedppr.cpp:84-107)."""
    g = oracle.random_graph(9, 1, 3, 11)
    d = dev(P, g)
    W = 60
    m_eff = int(g.offsets[-1]) + int(np.sum(np.diff(g.offsets) == 0))
    st = P.refine(d, 2, 0.2, 1.0 / W, P.power_push(d, 2, 0.2, m_eff / W))
    expected = st.estimates.copy()
    for v in range(g.n):
        if st.residues[v] > 0:
            expected += st.residues[v] * oracle.exact_ppr(g, v, 0.2)
    runs = np.stack([P.monte_carlo_phase(d, 2, 0.2, st, W, 1000 + r).estimates
                     for r in range(3000)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(len(runs))
    assert np.all(np.abs(runs.mean(axis=0) - expected) <= 4 * se + 1e-12)
    assert np.all(np.abs(runs.sum(axis=1) - 1.0) < 1e-9)


def test_async_host_outputs(P, oracle):
    """PPRG_ASYNC_HOST: results are complete after pprg_graph_sync."""
    import ctypes
    g = P.generate_rmat(14, 8, 2)
    src = P.sample_sources(np.diff(g.out_offsets()), 130, 2).astype(np.uint32)
    k, n = len(src), g.n()
    res, rsd = P.pinned_empty((k, n)), P.pinned_empty((k, n))
    res[:] = -1.0
    L = P.load_library()
    q = (P._abi.QStats * k)()
    P._abi._check(L.pprg_power_push(g.handle, src.ctypes.data, k, 0.2, 1e-8, 8, -1,
                                    res.ctypes.data, rsd.ctypes.data, 2, q, None, None))
    P._abi._check(L.pprg_graph_sync(g.handle))
    ref, _ = P.power_push_batch(g, src, 0.2, 1e-8)
    assert np.all(res >= 0.0)
    for i in (0, 64, 129):
        assert np.max(np.abs(res[i] - ref[i].estimates)) <= 2e-8
