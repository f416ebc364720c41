"""CPU baseline of BASELINE configs[4]: the reference
library's own power_push (compiled unchanged, oracle/_ref) on the scale-25
R-MAT: single-thread latency of one source, then the 8 sources of the config
concurrently on 8 host threads, beside the GPU's single-query time for the
same sources. Test/measurement infrastructure (imports the oracle package).

python tools/config5_cpu.py [--single 1] [--concurrent 8]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_03652_b200 as P  # noqa: E402
from oracle.pyoracle import CSR, Ref  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--single", type=int, default=1)
ap.add_argument("--concurrent", type=int, default=8)
a = ap.parse_args()
g = P.generate_rmat(25, 32, 5)
src = P.sample_sources(np.diff(g.out_offsets()), 8, 5)
gpu = []
for s in src[: max(a.single, 1)]:
    P.power_push_batch(g, [s], 0.2, 1e-8, keep=False)
    t0 = time.perf_counter()
    outs, cs = P.power_push_batch(g, [s], 0.2, 1e-8, keep=False)
    gpu.append({"source": int(s), "wall_s": time.perf_counter() - t0, "device_ms": cs.device_ms,
                "sweeps": outs[0].sweeps})
off, nbr = g.out_offsets().copy(), g.out_neighbors().copy()
n, m = g.n(), g.m()
del g
rg = Ref().graph(CSR(off, nbr))
single = []
for s in src[: a.single]:
    t0 = time.perf_counter()
    r = rg.power_push(int(s), 0.2, 1e-8)
    single.append({"source": int(s), "s": time.perf_counter() - t0})
conc = None
if a.concurrent:
    t0 = time.perf_counter()
    rg.power_push_batch(src[: a.concurrent], 0.2, 1e-8, a.concurrent)
    dt = time.perf_counter() - t0
    conc = {"sources": a.concurrent, "threads": a.concurrent, "wall_s": dt,
            "queries_per_s": a.concurrent / dt}
print(json.dumps({"config": "configs[4] CPU baseline: reference power_push, R-MAT 25/32 seed 5",
                  "n": n, "m": m, "host_threads": os.cpu_count(), "gpu_single_query": gpu,
                  "cpu_single_thread": single, "cpu_concurrent": conc}))
