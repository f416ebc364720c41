"""GPU parity at the BASELINE.json configs themselves (not scaled-down stand-ins):
the CUDA path through the C ABI against the reference library compiled
unchanged into oracle/_ref (push.cpp, speedppr.cpp, metrics.cpp) on the
identical CSR and sources.

Tolerances (north_star / SURVEY 8(c)):
  * high precision (PowerPush, PowItr; fp64): per node |pi_gpu - pi_ref| <= lambda,
    GPU r_sum <= lambda, and l1(pi_gpu, pi_ref) <= r_sum_gpu + r_sum_ref (both are
    pointwise under-estimates of pi, so their distance is bounded by the leftover
    residue mass), with 1e-15 of floating-point slack;
  * PowItr: every iterate within 1e-12 (l_inf) of the reference and the same
    iteration count (push.cpp:81-108);
  * SpeedPPR: compare_to_truth(mu = 1/n, eps = 0.5).violations == 0 per source
    (metrics.cpp:27-42) against a lambda = 1e-17 ground truth (metrics.cpp:44-55),
    itself cross-checked against the reference's power_push at lambda = 1e-12.
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import CSR

pytestmark = pytest.mark.gpu

ALPHA, LAM = 0.2, 1e-8
SLACK = 1e-15
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def P():
    import paper_2101_03652_b200 as P
    return P


def gcsr(g) -> CSR:
    return CSR(g.out_offsets().copy(), g.out_neighbors().copy())


def assert_high_precision(est_gpu, rs_gpu, est_ref, rs_ref, lam, what):
    assert rs_gpu <= lam, f"{what}: GPU r_sum {rs_gpu} > lambda"
    d = np.abs(est_gpu - est_ref)
    assert float(d.max()) <= lam + SLACK, f"{what}: max |delta| {d.max()}"
    l1 = float(d.sum())
    assert l1 <= rs_gpu + rs_ref + 1e-12, f"{what}: l1 {l1} > {rs_gpu} + {rs_ref}"
    return float(d.max()), l1


# ---- the host generator the reference arm uses is the product's, bit for bit --------
@pytest.mark.parametrize("scale,ef,seed", [(10, 8, 1), (17, 8, 1)])
def test_host_rmat_matches_device_generator(P, oracle, scale, ef, seed):
    g = P.generate_rmat(scale, ef, seed)
    h = oracle.generate_rmat(scale, ef, seed)
    assert np.array_equal(g.out_offsets(), h.offsets)
    assert np.array_equal(g.out_neighbors(), h.neighbors)


# ---- configs[0]: one source, R-MAT 17/8, graph + source from seed 1 -----------------
@pytest.fixture(scope="module")
def rmat17(P):
    return P.generate_rmat(17, 8, 1)


@pytest.fixture(scope="module")
def rmat17_ref(ref, rmat17):
    return ref.graph(gcsr(rmat17))


def test_config0_power_push(P, rmat17, rmat17_ref):
    s = int(P.sample_sources(np.diff(rmat17.out_offsets()), 1, 1)[0])
    tr = P.PowerPushTrace()
    got = P.power_push(rmat17, s, ALPHA, LAM, trace=tr)
    want = rmat17_ref.power_push(s, ALPHA, LAM)
    assert_high_precision(got.estimates, got.achieved_r_sum, want.estimates, want.r_sum,
                          LAM, "configs[0]")
    # the residue vector the GPU returns is the exact leftover mass
    assert abs(float(got.residues.sum()) - got.achieved_r_sum) <= 1e-12
    assert tr.used_scan_phase == want.used_scan_phase
    assert np.allclose(tr.epoch_r_max, want.epoch_r_max, rtol=1e-15, atol=0)


# ---- configs[1]: 64 sources (seed 2) as one 64-column block, PowerPush and PowItr ---
def test_config1_power_push_block(P, rmat17, rmat17_ref):
    src = P.sample_sources(np.diff(rmat17.out_offsets()), 64, 2)
    assert rmat17.block_columns(64) == 64
    outs, cs = P.power_push_batch(rmat17, src, ALPHA, LAM)
    res, rsd, rs = rmat17_ref.power_push_batch(list(src), ALPHA, LAM, THREADS, keep=True)
    for c in range(64):
        assert_high_precision(outs[c].estimates, outs[c].achieved_r_sum, res[c], rs[c], LAM,
                              f"configs[1] PowerPush column {c}")


def test_config1_power_iteration_block(P, rmat17, rmat17_ref):
    src = P.sample_sources(np.diff(rmat17.out_offsets()), 64, 2)
    outs, cs = P.power_iteration_batch(rmat17, src, ALPHA, LAM)
    res, rsd, rs = rmat17_ref.power_push_batch(list(src), ALPHA, LAM, THREADS, keep=True,
                                                powitr=True)
    it = rmat17_ref.power_iteration(int(src[0]), ALPHA, LAM)
    assert it.iterations == 83
    for c in range(64):
        assert outs[c].sweeps == it.iterations, (c, outs[c].sweeps)
        assert float(np.max(np.abs(outs[c].estimates - res[c]))) <= 1e-12
        assert float(np.max(np.abs(outs[c].residues - rsd[c]))) <= 1e-12
        assert abs(outs[c].achieved_r_sum - rs[c]) <= 1e-12


# ---- configs[2]: the bench's own path, R-MAT 22/16 seed 3, 256 sources, K = 64 ------
def test_config2_power_push_k64_blocks(P, ref):
    import torch
    g = P.generate_rmat(22, 16, 3)
    src = P.sample_sources(np.diff(g.out_offsets()), 256, 3)
    n, k = g.n(), len(src)
    assert g.block_columns(k) == 64
    dres = torch.empty((k, n), dtype=torch.float64, device="cuda:0")
    drsd = torch.empty((k, n), dtype=torch.float64, device="cuda:0")
    outs, cs = P.power_push_batch(g, src, ALPHA, LAM, device_out=(dres.data_ptr(),
                                                                  drsd.data_ptr()))
    assert cs.max_sweeps > 0
    # two columns from each of the four 64-column blocks, first and last included
    pick = [0, 37, 63, 64 + 21, 127, 128 + 5, 191, 192 + 50, 255]
    rg = ref.graph(gcsr(g))
    res, rsd, rs = rg.power_push_batch([int(src[i]) for i in pick], ALPHA, LAM, THREADS, keep=True)
    for j, i in enumerate(pick):
        est = dres[i].cpu().numpy()
        assert abs(float(drsd[i].sum().item()) - outs[i].achieved_r_sum) <= 1e-12
        assert_high_precision(est, outs[i].achieved_r_sum, res[j], rs[j], LAM,
                              f"configs[2] query {i} (block {i // 64}, column {i % 64})")


# ---- configs[3]: SpeedPPR with the walk index on Chung-Lu 2^22 ---------------------
def test_config3_speedppr_epsilon(P, oracle, ref):
    n_raw = 1 << 22
    g = P.generate_chung_lu(n_raw, 146 * n_raw // 4, 4)
    n = g.n()
    src = P.sample_sources(np.diff(g.out_offsets()), 1024, 4)
    idx = P.build_index(g, ALPHA, 4)
    sub = src[:64]  # one full 64-column SpeedPPR batch
    outs, _ = P.speedppr_batch(g, sub, P.QueryConfig(epsilon=0.5, seed=4), idx)
    truth, _ = P.ground_truth_batch(g, sub, ALPHA)
    mu = 1.0 / n
    worst = []
    for c in range(len(sub)):
        assert truth[c].achieved_r_sum <= P.GROUND_TRUTH_LAMBDA
        est = outs[c].estimates
        assert abs(float(est.sum()) - 1.0) <= 1e-9  # test_speedppr.cpp:61-72
        rep = oracle.compare_to_truth(est, truth[c].estimates, mu, 0.5)
        assert rep.violations == 0, (c, int(sub[c]), rep.violations, rep.max_rel_above_mu)
        worst.append(rep.max_rel_above_mu)
    assert max(worst) <= 0.5
    # the truth itself against the reference library's power_push at lambda = 1e-12
    rg = ref.graph(gcsr(g))
    res, _, rs = rg.power_push_batch([int(s) for s in sub[:2]], ALPHA, 1e-12, 2, keep=True)
    for j in range(2):
        d = np.abs(truth[j].estimates - res[j])
        assert float(d.max()) <= 1e-12 + SLACK
        assert float(d.sum()) <= rs[j] + 1e-15


# ---- configs[4]: scale-25 single source, one GPU and vertex-partitioned -------------
@pytest.mark.slow
def test_config4_scale25_power_push(P, ref):
    from paper_2101_03652_b200.partition import run_virtual_parts
    g = P.generate_rmat(25, 32, 5)
    s = int(P.sample_sources(np.diff(g.out_offsets()), 8, 5)[0])
    got = P.power_push(g, s, ALPHA, LAM)
    rg = ref.graph(gcsr(g))
    want = rg.power_push(s, ALPHA, LAM)  # ~3 min on one host core
    assert_high_precision(got.estimates, got.achieved_r_sum, want.estimates,
                          want.r_sum, LAM, "configs[4] single GPU")
    del got
    # the 8-part vertex partition with the fused peer-store exchange, parts run in turn
    res, rsd, rs, sweeps, parts = run_virtual_parts(g, 8, [s], ALPHA, LAM, fused=True)
    for p in parts:
        p.close()
    assert_high_precision(res[0], float(rs[0]), want.estimates, want.r_sum, LAM,
                          "configs[4] 8 parts, fused exchange")
    assert float(rsd[0].min()) >= 0.0
