"""The delta sweeps (csrc/delta_sweep.cuh: explicit residues, 16-bit per-sweep
shares, lagged waves) forced on for graphs far below their automatic
threshold: parity against the CPU oracle and against the k_sweeps path, exact
mass conservation, non-negative residues, the wave / lag / task-size knobs."""
import os

import numpy as np
import pytest

from oracle.pyoracle import CSR
from test_gpu_fuzz import hub_graph

pytestmark = pytest.mark.gpu
ALPHA = 0.2


@pytest.fixture(scope="module")
def P():
    import paper_2101_03652_b200 as P
    P.load_library()
    return P


@pytest.fixture()
def delta(monkeypatch):
    """PPRG_DELTA / PPRG_DS_* are read per call (delta_on) or once (plan sizes)."""
    def set_mode(v):
        monkeypatch.setenv("PPRG_DELTA", str(v))
    set_mode(1)
    return set_mode


def check(o, ref, lam):
    assert o.achieved_r_sum <= lam
    assert np.max(np.abs(o.estimates - ref.estimates)) <= lam
    # mass: reserve + residue == 1 to fp64 rounding (a share is added exactly
    # once by every out-neighbour, the rounding remainder stays a residue)
    assert abs(o.estimates.sum() + o.residues.sum() - 1.0) < 1e-12
    assert abs(o.residues.sum() - o.achieved_r_sum) < 1e-13
    assert np.all(o.residues >= 0.0)


CASES = [(300, 1, 3000, 2), (2000, 3, 9000, 3), (5000, 2, 20000, 4), (3000, 4, 700, 5),
         (20000, 6, 1500, 6)]


@pytest.mark.parametrize("n,hubs,hub_deg,seed", CASES)
@pytest.mark.parametrize("k", [17, 32, 64, 100])
def test_delta_power_push_vs_oracle(P, oracle, delta, n, hubs, hub_deg, seed, k):
    rng = np.random.default_rng(seed)
    g = hub_graph(n, hubs, hub_deg, rng)
    d = P.Graph(g.offsets, g.neighbors)
    src = rng.integers(0, g.n, size=k)
    src[1] = src[0]                                   # a duplicated source
    dead = np.flatnonzero(np.diff(g.offsets.astype(np.int64)) == 0)
    if len(dead):
        src[2] = dead[0]                              # a dead-end source
    indeg = np.bincount(g.neighbors, minlength=g.n)
    noin = np.flatnonzero((indeg == 0) & (np.diff(g.offsets.astype(np.int64)) > 0))
    if len(noin):
        src[3] = noin[0]                              # a source without in-edges
    lam = 1e-9
    # queue limit 0: no local phase beyond the seed, every push happens in the sweeps
    for thr in (None, 0):
        kw = {} if thr is None else {"scan_threshold": thr}
        outs, cs = P.power_push_batch(d, src, ALPHA, lam, **kw)
        assert cs.max_sweeps > 0
        for q in sorted({0, 1, 2, 3, k // 2, k - 1}):
            check(outs[q], oracle.power_push(g, int(src[q]), ALPHA, lam), lam)


def test_delta_matches_sweeps_path(P, delta):
    g = P.generate_rmat(15, 12, 7)
    src = P.sample_sources(np.diff(g.out_offsets()), 64, 7)
    lam = 1e-8
    a, ca = P.power_push_batch(g, src, ALPHA, lam)
    delta(0)
    b, cb = P.power_push_batch(g, src, ALPHA, lam)
    assert ca.kernel_launches != cb.kernel_launches or ca.max_sweeps != cb.max_sweeps  # two engines
    for q in range(64):
        assert a[q].achieved_r_sum <= lam and b[q].achieved_r_sum <= lam
        # both are within r_sum of the exact vector, from below
        assert np.max(np.abs(a[q].estimates - b[q].estimates)) <= lam
        assert abs(a[q].estimates.sum() + a[q].residues.sum() - 1.0) < 1e-12


def test_delta_all_dead_end_graph(P, oracle, delta):
    # a star into dead ends: every push of a leaf returns its mass to the source
    n = 200
    off = np.zeros(n + 1, np.uint64)
    off[1:] = n - 1
    nbr = np.arange(1, n, dtype=np.uint32)
    g = CSR(off, nbr)
    d = P.Graph(g.offsets, g.neighbors)
    src = np.zeros(40, np.uint32)
    src[5:] = np.arange(5, 40)
    outs, _ = P.power_push_batch(d, src, ALPHA, 1e-10, scan_threshold=0)
    for q in (0, 7, 39):
        check(outs[q], oracle.power_push(g, int(src[q]), ALPHA, 1e-10), 1e-10)


def test_delta_small_blocks_keep_the_sweeps_path(P, delta):
    # fewer than 17 sources round to <= 16 columns: not a delta block
    g = P.generate_rmat(12, 8, 3)
    src = P.sample_sources(np.diff(g.out_offsets()), 8, 3)
    a, _ = P.power_push_batch(g, src, ALPHA, 1e-8)
    delta(0)
    b, _ = P.power_push_batch(g, src, ALPHA, 1e-8)
    for q in range(8):
        assert np.max(np.abs(a[q].estimates - b[q].estimates)) <= 1e-8


def test_delta_on_the_chung_lu_graph_of_configs3(P, monkeypatch):
    """A second graph family at full size (the 2^22-node Chung-Lu graph of
    configs[3]: power-law in- and out-degrees, 124M edges): the automatic choice
    is the delta sweeps, and they agree with k_sweeps (which the configs tests pin
    to the reference) within lambda, with exact mass."""
    import torch
    n = 1 << 22
    g = P.generate_chung_lu(n, 146 * n // 4, 4)
    src = P.sample_sources(np.diff(g.out_offsets()), 64, 4)
    lam = 1e-8
    monkeypatch.delenv("PPRG_DELTA", raising=False)
    assert g.uses_delta_sweeps(64)
    k, nn = len(src), g.n()
    a = torch.empty((2, k, nn), dtype=torch.float64, device="cuda:0")
    b = torch.empty((2, k, nn), dtype=torch.float64, device="cuda:0")
    oa, ca = P.power_push_batch(g, src, ALPHA, lam, device_out=(a[0].data_ptr(), a[1].data_ptr()))
    monkeypatch.setenv("PPRG_DELTA", "0")
    assert not g.uses_delta_sweeps(64)
    ob, cb = P.power_push_batch(g, src, ALPHA, lam, device_out=(b[0].data_ptr(), b[1].data_ptr()))
    assert float((a[0] - b[0]).abs().max().item()) <= lam
    mass = a[0].sum(dim=1) + a[1].sum(dim=1)
    assert float((mass - 1.0).abs().max().item()) < 1e-11
    assert float(a[1].min().item()) >= 0.0
    for q in range(k):
        assert oa[q].achieved_r_sum <= lam and ob[q].achieved_r_sum <= lam
        assert abs(float(a[1][q].sum().item()) - oa[q].achieved_r_sum) <= 1e-12
