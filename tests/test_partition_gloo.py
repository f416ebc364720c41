"""The vertex-partitioned exchange protocol (paper_2101_03652_b200.partition,
SURVEY 8(e)) at world size 2 over gloo on CPU.

Each rank drives a numpy part — a row-by-row restatement of the pull sweep
over its own destination rows (test infrastructure, not the product) —
through the same `run_partitioned` the GPU ranks use, with the library's host
epoch rule (pprg_epoch_init / pprg_epoch_advance, no GPU needed). The
assembled reserve must match the oracle's power_push within lambda and the
exact r_sum must be <= lambda (the north-star bound)."""
import os
import socket

import numpy as np
import pytest

from oracle.pyoracle import CSR

ALPHA = 0.2


class NumpyPart:
    """Part interface of partition.GpuPart over a host CSR. Rows [lo, hi) are
    cut on in-edges; the queue phase is skipped (scan_threshold 0), so the
    global phase starts from the unit residue at the source."""

    def __init__(self, csr: CSR, nparts: int, part: int, sources, lam: float, epoch_num=8):
        from paper_2101_03652_b200.partition import EpochRule
        self.n = csr.n
        self.off = csr.offsets.astype(np.int64)
        nbr = csr.neighbors.astype(np.int64)
        self.deg = np.diff(self.off)
        src_of = np.repeat(np.arange(self.n), self.deg)
        order = np.lexsort((src_of, nbr))  # transpose, in-neighbours ascending
        self.in_nbr = src_of[order]
        self.in_off = np.concatenate([[0], np.cumsum(np.bincount(nbr, minlength=self.n))])
        cum = self.in_off + np.arange(self.n + 1)  # +1 per row so empty rows count
        cuts = [0] + [int(np.searchsorted(cum, cum[-1] * p / nparts)) for p in range(1, nparts)] \
            + [self.n]
        self.lo, self.hi = cuts[part], cuts[part + 1]
        self.src = list(sources)
        self.k = len(self.src)
        self.columns = self.k
        self.m_eff = float(len(nbr) + np.count_nonzero(self.deg == 0))
        self.rule = EpochRule(self.k, lam, epoch_num, ALPHA)
        self.thr = self.rule.lam / self.m_eff
        self.x = np.zeros((self.n, self.k))
        self.y = np.zeros(self.n * self.k)
        self.cnt = np.zeros(5 * self.k)

    def begin(self):
        return np.zeros(128)

    def x_view(self):  # the adopted local-phase state (zero here: no queue phase)
        import torch
        return torch.from_numpy(self.x.reshape(-1))

    def resum(self):
        out = np.zeros(128)
        xs = self.x[self.lo:self.hi]
        out[:self.k] = xs.sum(axis=0)
        out[64:64 + self.k] = xs[self.deg[self.lo:self.hi] == 0].sum(axis=0)
        return out

    def start(self, summed):
        return self.rule.init(summed[:64], summed[64:128])

    def y_view(self):
        import torch
        return torch.from_numpy(self.y)

    def counters_view(self):
        import torch
        return torch.from_numpy(self.cnt)

    def sweep(self):
        K = self.k
        y = self.y.reshape(self.n, K)
        self.cnt[:] = 0.0
        for c in range(K):
            st = self.rule.state(c)
            if st.done:
                continue
            thr = self.thr[st.epoch]
            for u in range(self.lo, self.hi):
                inflow = y[self.in_nbr[self.in_off[u]:self.in_off[u + 1]], c].sum()
                if u == self.src[c]:
                    inflow += 1.0 + st.D
                d = self.deg[u]
                r = inflow - self.x[u, c]
                if r > max(d, 1) * thr:
                    self.x[u, c] = inflow
                    if d:
                        y[u, c] = (1 - ALPHA) * inflow / d
                    self.cnt[c] += r
                    self.cnt[K + c] += max(d, 1)
                    self.cnt[2 * K + c] += 1
                    self.cnt[4 * K + c] += d
                if d == 0:
                    self.cnt[3 * K + c] += (1 - ALPHA) * self.x[u, c]

    def advance(self, summed):
        return self.rule.advance(summed)

    def finish(self):
        K = self.k
        y = self.y.reshape(self.n, K)
        self.residue = np.zeros((self.n, K))
        for c in range(K):
            D = self.rule.state(c).D
            for u in range(self.lo, self.hi):
                inflow = y[self.in_nbr[self.in_off[u]:self.in_off[u + 1]], c].sum()
                if u == self.src[c]:
                    inflow += 1.0 + D
                self.residue[u, c] = max(inflow - self.x[u, c], 0.0)
        return self.residue[self.lo:self.hi].sum(axis=0)


def _worker(rank, world, port, csr_arrays, sources, lam, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2101_03652_b200.partition import run_partitioned
        part = NumpyPart(CSR(*csr_arrays), world, rank, sources, lam)
        r = run_partitioned(part)
        # assemble the reserve of every rank's rows on all ranks
        res = torch.zeros(part.n * part.k, dtype=torch.float64)
        res.view(part.n, part.k)[part.lo:part.hi] = torch.from_numpy(
            ALPHA * part.x[part.lo:part.hi])
        dist.all_reduce(res)
        if rank == 0:
            np.savez(out_path, reserve=res.numpy().reshape(part.n, part.k), r_sum=r.r_sum,
                     sweeps=r.sweeps, bounds=np.array(r.bounds))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("sources", [[3], [0, 17, 42]])
def test_partitioned_protocol_gloo_world2(oracle, tmp_path, sources):
    import torch.multiprocessing as mp
    g = oracle.random_graph(120, 0, 5, 7)  # dead ends included
    lam = 1e-7
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), (g.offsets, g.neighbors), sources, lam, out),
             nprocs=2, join=True)
    r = np.load(out)
    lo0, hi0 = r["bounds"][0]
    lo1, hi1 = r["bounds"][1]
    assert lo0 == 0 and hi0 == lo1 and hi1 == g.n
    assert int(r["sweeps"]) > 0
    for c, s in enumerate(sources):
        ref = oracle.power_push(g, s, ALPHA, lam)
        assert r["r_sum"][c] <= lam
        assert np.max(np.abs(r["reserve"][:, c] - ref.estimates)) <= lam
        assert abs(r["reserve"][:, c].sum() + r["r_sum"][c] - 1.0) < 1e-9


def test_epoch_rule_matches_reference_thresholds():
    """Host epoch rule: lambda_i = lambda^(i/E) (push.cpp:176-178); an epoch
    ends at r_sum <= lambda_i or at a fixpoint (no pushes in a sweep)."""
    from paper_2101_03652_b200.partition import EpochRule
    r = EpochRule(1, 1e-8, 8, ALPHA)
    assert np.allclose(r.lam, [1e-8 ** (i / 8) for i in range(1, 9)])
    assert r.init(np.zeros(1), np.zeros(1))
    st = r.state(0)
    assert st.r_sum == 1.0 and st.epoch == 0 and not st.done
    # a sweep pushing mass 4 from r_sum 1: r_sum = 1 - 0.2 * 4 = 0.2 -> epoch 1 (0.1) still open
    s = np.zeros(5)
    s[0], s[1] = 4.0, 10.0
    assert not r.advance(s)
    st = r.state(0)
    assert abs(st.r_sum - 0.2) < 1e-15 and st.epoch == 0 and st.sweeps == 1 and st.pushes == 10
    # fixpoint: no pushes moves to the next epoch
    assert not r.advance(np.zeros(5))
    assert r.state(0).epoch == 1
    # r_sum below every lambda ends the phase
    s[0] = 1.0
    assert r.advance(s)
    assert r.state(0).done
