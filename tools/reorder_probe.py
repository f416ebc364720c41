"""Exploration: does a degree-sorted node order change the sweep's L2 reuse?
Builds configs[2]'s R-MAT as is and relabeled by descending out-degree (an
isomorphic graph), runs one 64-source block on each and prints the timings."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P  # noqa: E402

g, edges = P.generate_rmat(22, 16, 3, return_edges=True)
src_ids, dst_ids = edges[:, 0], edges[:, 1]
uniq = np.unique(np.concatenate([src_ids, dst_ids]))
s = np.searchsorted(uniq, src_ids)
d = np.searchsorted(uniq, dst_ids)
n = len(uniq)
for name, key in (("in-degree", np.bincount(d, minlength=n)), ("out-degree", np.bincount(s, minlength=n))):
    perm = np.empty(n, np.int64)
    perm[np.argsort(-key, kind="stable")] = np.arange(n)
    pairs = np.stack([perm[s], perm[d]], axis=1).astype(np.uint64)
    g2 = P.build_graph_from_edges(pairs)
    for label, gg in (("original", g), (f"sorted by {name}", g2)):
        srcs = P.sample_sources(np.diff(gg.out_offsets()), 64, 3)
        P.power_push_batch(gg, srcs, 0.2, 1e-8, keep=False)
        t0 = time.perf_counter()
        outs, cs = P.power_push_batch(gg, srcs, 0.2, 1e-8, keep=False)
        dt = time.perf_counter() - t0
        print(f"{label:22s} n={gg.n()} m={gg.m()} wall {dt*1e3:7.1f} ms sweep {cs.sweep_ms:7.1f} ms "
              f"sweeps {cs.max_sweeps}", flush=True)
