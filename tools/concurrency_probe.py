"""Throughput of concurrent single-source PowerPush queries from T host
threads on one graph handle (the lanes of SURVEY 8(b)). configs[0]'s graph
(R-MAT 17/8 seed 1), 1-source calls. Prints one JSON line."""
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_03652_b200 as P  # noqa: E402

g = P.generate_rmat(17, 8, 1)
srcs = [int(s) for s in P.sample_sources(np.diff(g.out_offsets()), 64, 9)]
Q = 32
rec = {"env": {k: v for k, v in os.environ.items() if k.startswith("PPRG_")}}
P.power_push_batch(g, srcs[:1], 0.2, 1e-8, keep=False)
for T in (1, 2, 4, 8):
    def worker(t):
        for q in range(Q):
            P.power_push_batch(g, [srcs[(t * Q + q) % len(srcs)]], 0.2, 1e-8, keep=False)
    ths = [threading.Thread(target=worker, args=(t,)) for t in range(T)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    rec[f"threads_{T}"] = {"queries": T * Q, "s": dt, "queries_per_s": T * Q / dt}
print(json.dumps(rec))
