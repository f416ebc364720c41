"""Secondary measurements of the BASELINE.json configs other than the bench's
configs[2] (bench.py). One JSON record per config, GPU beside the reference
CPU library (oracle/_ref) on the same CSR and sources. Not the driver's bench.

python tools/bench_configs.py [--configs 1,2,4,5] [--out profiles/r01_configs.json]
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

ALPHA, LAM = 0.2, 1e-8


def ref_graph(g):
    from oracle.pyoracle import CSR, Ref
    return Ref().graph(CSR(g.out_offsets().copy(), g.out_neighbors().copy()))


def timed(fn, reps=1):
    fn()  # warm
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return (time.perf_counter() - t0) / reps, out


def config1(threads):
    g = P.generate_rmat(17, 8, 1)
    s = P.sample_sources(np.diff(g.out_offsets()), 1, 1)
    dt, (outs, cs) = timed(lambda: P.power_push_batch(g, s, ALPHA, LAM), reps=10)
    rg = ref_graph(g)
    t0 = time.perf_counter()
    ref = rg.power_push(int(s[0]), ALPHA, LAM)
    cpu = time.perf_counter() - t0
    err = float(np.max(np.abs(outs[0].estimates - ref.estimates)))
    return {"config": "configs[0]: PowerPush 1 source, R-MAT 17/8 seed 1", "n": g.n(), "m": g.m(),
            "source": int(s[0]), "gpu_ms_per_query": dt * 1e3, "gpu_device_ms": cs.device_ms,
            "sweeps": outs[0].sweeps, "cpu_ms_per_query_1thread": cpu * 1e3,
            "max_abs_diff_vs_reference": err, "r_sum": outs[0].achieved_r_sum}


def config2(threads):
    g = P.generate_rmat(17, 8, 1)
    s = P.sample_sources(np.diff(g.out_offsets()), 64, 2)
    rec = {"config": "configs[1]: 64 sources as one 64-column block, R-MAT 17/8", "n": g.n(),
           "m": g.m()}
    for name, fn in (("powerpush", lambda: P.power_push_batch(g, s, ALPHA, LAM, keep=False)),
                     ("powitr", lambda: P.power_iteration_batch(g, s, ALPHA, LAM, keep=False))):
        dt, (outs, cs) = timed(fn, reps=5)
        rec[f"gpu_{name}_queries_per_s"] = 64 / dt
        rec[f"gpu_{name}_sweeps"] = cs.max_sweeps
        rec[f"gpu_{name}_alg_GBps"] = cs.alg_bytes / max(cs.sweep_ms, 1e-9) / 1e6
    rg = ref_graph(g)
    for name, pw in (("powerpush", False), ("powitr", True)):
        t0 = time.perf_counter()
        rg.power_push_batch(list(s), ALPHA, LAM, threads, powitr=pw)
        rec[f"cpu_{name}_queries_per_s_{threads}threads"] = 64 / (time.perf_counter() - t0)
    return rec


def config4(threads):
    n = 1 << 22
    t0 = time.perf_counter()
    g = P.generate_chung_lu(n, 146 * n // 4, 4)  # ~146M draws -> ~120M cleaned edges
    gen = time.perf_counter() - t0
    s = P.sample_sources(np.diff(g.out_offsets()), 1024, 4)
    t0 = time.perf_counter()
    idx = P.build_index(g, ALPHA, 4)
    build = time.perf_counter() - t0
    cfg = P.QueryConfig(epsilon=0.5, seed=4)
    sub = s[:256]
    P.speedppr_batch(g, s[256:320], cfg, idx, keep=False)  # warm-up: transpose, plans, workspaces
    t0 = time.perf_counter()
    outs, cs = P.speedppr_batch(g, sub, cfg, idx, keep=False)
    dt = time.perf_counter() - t0
    rec = {"config": "configs[3]: SpeedPPR eps=0.5 with index, Chung-Lu 2^22", "n": g.n(),
           "m": g.m(), "generate_s": gen, "gpu_index_build_s": build,
           "gpu_queries_per_s": len(sub) / dt, "queries_timed": int(len(sub)),
           "walks_per_query": float(np.mean([o.walks for o in outs])),
           "pushes_per_query_over_m": float(np.mean([o.pushes for o in outs])) / g.m(),
           "gpu_ms_per_query_device": cs.device_ms / len(sub),
           "gpu_ms_per_query_local": cs.local_ms / len(sub),
           "gpu_ms_per_query_sweeps": cs.sweep_ms / len(sub),
           "gpu_ms_per_query_final": cs.final_ms / len(sub),
           "gpu_ms_per_query_mc_and_rest": (cs.device_ms - cs.local_ms - cs.sweep_ms - cs.final_ms) / len(sub)}
    rg = ref_graph(g)
    k = threads
    t0 = time.perf_counter()
    rg.speedppr_batch(list(s[:k]), ALPHA, 0.5, 4, threads)
    rec[f"cpu_queries_per_s_{threads}threads_indexfree"] = k / (time.perf_counter() - t0)
    ends = idx.endpoints()
    t0 = time.perf_counter()
    rg.speedppr_batch(list(s[:k]), ALPHA, 0.5, 4, threads, index=ends, index_seed=4)
    rec[f"cpu_queries_per_s_{threads}threads_with_index"] = k / (time.perf_counter() - t0)
    return rec


def config5(threads):
    t0 = time.perf_counter()
    g = P.generate_rmat(25, 32, 5)
    gen = time.perf_counter() - t0
    s = P.sample_sources(np.diff(g.out_offsets()), 8, 5)
    times = []
    for src in s:
        t0 = time.perf_counter()
        outs, cs = P.power_push_batch(g, [src], ALPHA, LAM, keep=False)
        times.append(time.perf_counter() - t0)
    return {"config": "configs[4] on ONE GPU (graph fits in 180 GB; vertex partition not exercised)",
            "n": g.n(), "m": g.m(), "generate_s": gen, "gpu_s_per_query": times,
            "sweeps_last": outs[0].sweeps, "alg_GBps_last": cs.alg_bytes / max(cs.sweep_ms, 1e-9) / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_configs.json"))
    a = ap.parse_args()
    threads = os.cpu_count() or 1
    res = {"host_threads": threads}
    for c in a.configs.split(","):
        fn = {"1": config1, "2": config2, "4": config4, "5": config5}[c]
        try:
            res[f"config{c}"] = fn(threads)
        except Exception as e:  # recorded, not fatal
            res[f"config{c}"] = {"error": repr(e)}
        print(json.dumps({f"config{c}": res[f"config{c}"]}), flush=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
