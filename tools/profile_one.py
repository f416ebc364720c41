"""Short PowerPush workload for ncu / timing breakdowns (not the bench).

python tools/profile_one.py [--scale 22] [--ef 16] [--queries 4] [--columns K]
Runs one warm-up batch and one measured batch on the configs[2] graph and
prints per-call counters (device ms, sweep ms, algorithmic GB/s, sweeps).
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_03652_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--seed", type=int, default=3)
ap.add_argument("--queries", type=int, default=4)
ap.add_argument("--engine", default="powerpush", choices=["powerpush", "powitr", "speedppr"])
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--epochs", type=int, default=8)
a = ap.parse_args()
g = P.generate_rmat(a.scale, a.ef, a.seed)
src = P.sample_sources(np.diff(g.out_offsets()), a.queries, a.seed)
print(f"n={g.n()} m={g.m()} dead={len(g.dead_ends())}")


def run():
    if a.engine == "powerpush":
        return P.power_push_batch(g, src, 0.2, 1e-8, epoch_num=a.epochs, keep=False)
    if a.engine == "powitr":
        return P.power_iteration_batch(g, src, 0.2, 1e-8, keep=False)
    return P.speedppr_batch(g, src, P.QueryConfig(epsilon=0.5, seed=4), keep=False)


run()
for _ in range(a.reps):
    t0 = time.perf_counter()
    outs, cs = run()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"wall {wall:.2f} ms  device {cs.device_ms:.2f} ms  sweeps_kernel {cs.sweep_ms:.2f} ms  "
          f"alg {cs.alg_bytes / 1e9:.2f} GB  {cs.alg_bytes / max(cs.sweep_ms, 1e-9) / 1e6:.1f} GB/s  "
          f"local {cs.local_ms:.2f} ms final {cs.final_ms:.2f} ms "
          f"max_sweeps {cs.max_sweeps} launches {cs.kernel_launches}  "
          f"r_sum_max {max(o.achieved_r_sum for o in outs):.3e} "
          f"levels {outs[0].local_levels} pushes/m {outs[0].pushes / g.m():.2f}")
