"""Concurrent queries on one graph handle from many host threads (SURVEY 8(b):
"each graph handle is safe for concurrent queries from many host threads;
each call uses its own stream and scratch"). Narrow calls (1-2 columns) run
on the graph's lanes concurrently, wide column blocks and index builds take
the whole device; every result must still meet the parity bar against the
oracle (ctypes releases the GIL, so the threads do overlap)."""
import threading

import numpy as np
import pytest

from oracle.pyoracle import CSR

pytestmark = pytest.mark.gpu

ALPHA, LAM = 0.2, 1e-8


@pytest.fixture(scope="module")
def P():
    import paper_2101_03652_b200 as P
    P.load_library()
    return P


def run_threads(fns):
    errors = []

    def wrap(fn):
        try:
            fn()
        except Exception as e:  # noqa: BLE001 - collected and re-raised below
            errors.append(e)

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]


def test_concurrent_mixed_queries_meet_parity(P, oracle):
    g = P.generate_rmat(13, 8, 7)
    csr = CSR(g.out_offsets().copy(), g.out_neighbors().copy())
    deg = np.diff(g.out_offsets())
    singles = [int(s) for s in P.sample_sources(deg, 12, 3)]
    block = P.sample_sources(deg, 64, 4)
    idx = P.build_index(g, ALPHA, 2)
    refs = {s: oracle.power_push(csr, s, ALPHA, LAM).estimates for s in singles}
    got = {}
    lock = threading.Lock()

    def singles_worker(part):
        def fn():
            for _ in range(3):
                for s in part:
                    outs, _ = P.power_push_batch(g, [s], ALPHA, LAM)
                    assert outs[0].achieved_r_sum <= LAM
                    with lock:
                        got[s] = outs[0].estimates
        return fn

    wide = {}

    def wide_worker():
        outs, _ = P.power_push_batch(g, block, ALPHA, LAM)
        wide["outs"] = outs

    spp = {}

    def spp_worker():
        o, _ = P.speedppr_batch(g, singles[:2], P.QueryConfig(epsilon=0.5, seed=3), idx)
        spp["outs"] = o

    fifo = {}

    def fifo_worker():
        fifo["o"] = P.fifo_forward_push(g, singles[0], ALPHA, 1e-9 / csr.m_eff)

    run_threads([singles_worker(singles[i::4]) for i in range(4)] + [wide_worker, spp_worker, fifo_worker])
    for s in singles:
        assert float(np.max(np.abs(got[s] - refs[s]))) <= LAM
    for i in (0, 63):
        ref = oracle.power_push(csr, int(block[i]), ALPHA, LAM)
        assert float(np.max(np.abs(wide["outs"][i].estimates - ref.estimates))) <= LAM
    for o in spp["outs"]:
        assert abs(o.estimates.sum() - 1.0) < 1e-6
    ref = oracle.fifo_forward_push(csr, singles[0], ALPHA, 1e-9 / csr.m_eff)
    assert float(np.max(np.abs(fifo["o"].estimates - ref.estimates))) <= 1e-9


def test_concurrent_deterministic_reruns(P):
    # deterministic mode under concurrency: every thread's rerun is bit-identical
    g = P.generate_rmat(13, 8, 8)
    srcs = [int(s) for s in P.sample_sources(np.diff(g.out_offsets()), 4, 1)]
    res = {}

    def worker(s):
        def fn():
            a, _ = P.power_push_batch(g, [s], ALPHA, LAM)
            b, _ = P.power_push_batch(g, [s], ALPHA, LAM)
            res[s] = (a[0].estimates, b[0].estimates)
        return fn

    with P.deterministic():
        run_threads([worker(s) for s in srcs])
    for s in srcs:
        a, b = res[s]
        assert a.tobytes() == b.tobytes()
