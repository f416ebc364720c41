"""Quick GPU timing of the query paths (no CPU reference): configs[0] latency,
configs[2] one 64-source block with its phase split, configs[3] SpeedPPR 256
queries with its phase split. A/B helper: run under different PPRG_* env."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_03652_b200 as P  # noqa: E402

ALPHA, LAM = 0.2, 1e-8
if os.environ.get("AB_DET"):
    P.set_deterministic(True)
which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["0", "2", "3"]
rec = {"env": {k: v for k, v in os.environ.items() if k.startswith(("PPRG_", "AB_"))}}


def split(cs, k):
    return {"device_ms": cs.device_ms / k, "local_ms": cs.local_ms / k, "sweep_ms": cs.sweep_ms / k,
            "final_ms": cs.final_ms / k, "launches": cs.kernel_launches, "max_sweeps": cs.max_sweeps}


if "0" in which:
    g = P.generate_rmat(17, 8, 1)
    s = P.sample_sources(np.diff(g.out_offsets()), 1, 1)
    P.power_push_batch(g, s, ALPHA, LAM, keep=False)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        outs, cs = P.power_push_batch(g, s, ALPHA, LAM, keep=False)
        ts.append(time.perf_counter() - t0)
    rec["configs[0]"] = {"ms_median": 1e3 * float(np.median(ts)), **split(cs, 1)}
if "1" in which:
    g = P.generate_rmat(17, 8, 1)
    s = P.sample_sources(np.diff(g.out_offsets()), 64, 2)
    P.power_push_batch(g, s, ALPHA, LAM, keep=False)
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        outs, cs = P.power_push_batch(g, s, ALPHA, LAM, keep=False)
        ts.append(time.perf_counter() - t0)
    rec["configs[1]"] = {"ms_median": 1e3 * float(np.median(ts)), **split(cs, 1)}
if "2" in which:
    g = P.generate_rmat(22, 16, 3)
    s = P.sample_sources(np.diff(g.out_offsets()), 256, 3)[:64]
    P.power_push_batch(g, s, ALPHA, LAM, keep=False)
    t0 = time.perf_counter()
    outs, cs = P.power_push_batch(g, s, ALPHA, LAM, keep=False)
    rec["configs[2] 64-block"] = {"wall_ms": 1e3 * (time.perf_counter() - t0), **split(cs, 1),
                                  "levels_col0": outs[0].local_levels}
if "3" in which:
    n = 1 << 22
    g = P.generate_chung_lu(n, 146 * n // 4, 4)
    s = P.sample_sources(np.diff(g.out_offsets()), 1024, 4)
    idx = P.build_index(g, ALPHA, 4)
    cfg = P.QueryConfig(epsilon=0.5, seed=4)
    P.speedppr_batch(g, s[256:320], cfg, idx, keep=False)
    t0 = time.perf_counter()
    outs, cs = P.speedppr_batch(g, s[:256], cfg, idx, keep=False)
    dt = time.perf_counter() - t0
    rec["configs[3]"] = {"queries_per_s": 256 / dt, **split(cs, 256)}
print(json.dumps(rec))
