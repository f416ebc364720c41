"""BASELINE configs[4]: PowerPush on R-MAT scale 25 / ef 32 (seed 5), 8
sources (seed 5) one at a time, vertex-partitioned over P parts.

Two modes:
  virtual (default, one GPU): the P parts run one after another on the same
      GPU each sweep (partition.run_virtual_parts), so the partitioned
      kernels, the cut and the sweep count are real; reported beside the
      unpartitioned single-GPU query on the same source, with the max |diff|.
      The per-part sweep times give the compute time of the slowest part;
      the exchange volume per sweep is n * 8 bytes gathered per rank.
  dist (torchrun, one rank per GPU): partition.run_partitioned over NCCL;
      wall time per query is the max over ranks.

python tools/config5_partitioned.py [--parts 8] [--queries 2] [--scale 25]
torchrun --nproc-per-node N tools/config5_partitioned.py --mode dist
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
from paper_2101_03652_b200.partition import GpuPart, run_partitioned, run_virtual_parts  # noqa: E402

ALPHA, LAM = 0.2, 1e-8


def virtual(a):
    t0 = time.perf_counter()
    g = P.generate_rmat(a.scale, a.ef, 5)
    gen = time.perf_counter() - t0
    src = P.sample_sources(np.diff(g.out_offsets()), 8, 5)
    n = g.n()
    recs = []
    for s in src[:a.queries]:
        t0 = time.perf_counter()
        outs, cs = P.power_push_batch(g, [s], ALPHA, LAM)
        single = time.perf_counter() - t0
        t0 = time.perf_counter()
        res, rsd, rs, sweeps, parts = run_virtual_parts(g, a.parts, [s], ALPHA, LAM,
                                                        fused=a.fused)
        virt = time.perf_counter() - t0
        per = [p.stats()[1] for p in parts]
        recs.append({
            "source": int(s), "single_gpu_s": single, "single_gpu_sweeps": outs[0].sweeps,
            "single_gpu_sweep_ms": cs.sweep_ms,
            "partitioned_sweeps": sweeps, "partitioned_r_sum": float(rs[0]),
            "max_abs_diff_vs_single_gpu": float(np.max(np.abs(res[0] - outs[0].estimates))),
            "part_rows": [p.hi - p.lo for p in parts],
            "part_sweep_ms": [c.sweep_ms for c in per],
            "slowest_part_sweep_ms": max(c.sweep_ms for c in per),
            "sum_part_sweep_ms": sum(c.sweep_ms for c in per),
            "exchange_bytes_per_sweep_per_rank": 8 * n,
            "virtual_wall_s": virt})
        for p in parts:
            p.close()
        print(json.dumps(recs[-1]), flush=True)
    return {"config": f"configs[4] vertex-partitioned into {a.parts} parts, run as virtual parts "
                      f"on one GPU ({'fused P2P-style y stores' if a.fused else 'y all-gather'} "
                      "exchange)", "n": n, "m": g.m(), "generate_s": gen, "queries": recs}


def dist_mode(a):
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    g = P.generate_rmat(a.scale, a.ef, 5, device=local)
    src = P.sample_sources(np.diff(g.out_offsets()), 8, 5)
    times, sweeps = [], []
    for s in src[:a.queries]:
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part = GpuPart(g, world, rank, [s], ALPHA, LAM)
        r = run_partitioned(part, comm_device=f"cuda:{local}", fused=a.fused and world > 1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
        sweeps.append(r.sweeps)
        assert r.r_sum[0] <= LAM
        part.close()
    if rank == 0:
        print(json.dumps({"config": f"configs[4] over {world} GPUs (NCCL)", "n": g.n(), "m": g.m(),
                          "s_per_query_max_over_ranks": times, "sweeps": sweeps}), flush=True)
    dist.destroy_process_group()
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="virtual", choices=["virtual", "dist"])
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--queries", type=int, default=2)
    ap.add_argument("--scale", type=int, default=25)
    ap.add_argument("--ef", type=int, default=32)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fused", action="store_true", help="fused exchange (y stores into peers)")
    a = ap.parse_args()
    rec = virtual(a) if a.mode == "virtual" else dist_mode(a)
    if rec is not None and a.out:
        with open(a.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
