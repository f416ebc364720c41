"""Benchmark: PowerPush SSPPR queries/s at lambda = 1e-8 (BASELINE.json `metric`).

Workload (BASELINE.json configs[2]): directed R-MAT scale 22, edge factor 16,
a=0.57 b=0.19 c=0.19 d=0.05, self-loops and duplicates removed (graph seed 3),
256 sources drawn uniformly from nodes with out-degree > 0 (seed 3), fp64,
alpha = 0.2, lambda = 1e-8, epoch_num 8, scan threshold n/4. The graph is
replicated on every GPU and the 256 sources are sharded across ranks (strong
scaling). A step = the rank's shard of the 256 queries.

  value : queries/s with the graph resident in HBM and results left in HBM
          (device time, max over ranks)
  e2e   : the same through the public API with host buffers: sources copied
          in and every query's reserve + residue vectors copied back to pinned
          host memory inside the timed region
  roofline: algorithmic bytes of the global PowerPush sweeps
          over the persistent sweep kernel's CUDA-event time, against the
          measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline: the reference library (oracle/_ref, compiled unchanged from
          /root/reference) running power_push on the same CSR and sources on
          the host cores (rank 0, N = 1 only)

--impl reference runs only the reference CPU arm (all host threads) and prints
its own line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PowerPush SSPPR queries/s at lambda=1e-8"
UNIT = "queries/s"
CFG = dict(scale=22, edge_factor=16, graph_seed=3, sources=256, source_seed=3, alpha=0.2,
           lam=1e-8)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None
        self.t0, self.t1 = 0.0, float("inf")

    def mark_start(self):  # samples before this (nvidia-smi start-up, warm-up) are dropped
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time()

    @staticmethod
    def _t(stamp: str) -> float:
        import datetime
        try:
            return datetime.datetime.strptime(stamp, "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return -1.0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        # rows carry nvidia-smi's own timestamp (host local time): keep the timed region's
        rows = [r[1:] for r in self.rows if r and self.t0 <= self._t(r[0]) <= self.t1 + 0.25]
        sm = [float(r[0]) for r in rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_for(workload: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(workload)
    return None


def ceiling_for(workload: str):
    p = os.path.join(ROOT, "profiles", "ceilings.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(workload)
    return None


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def make_graph(P, device):
    t0 = time.time()
    g = P.generate_rmat(CFG["scale"], CFG["edge_factor"], CFG["graph_seed"], device=device)
    srcs = P.sample_sources(np.diff(g.out_offsets()), CFG["sources"], CFG["source_seed"])
    log(f"graph: n={g.n()} m={g.m()} dead={len(g.dead_ends())} built in {time.time() - t0:.1f}s")
    return g, srcs


def cpu_reference_run(g_off, g_nbr, sources, threads, budget_s=20.0):
    """Reference power_push (oracle/_ref) on host threads; returns (q/s, sample, cores)."""
    from oracle.pyoracle import CSR, Ref
    ref = Ref()
    rg = ref.graph(CSR(g_off, g_nbr))
    t0 = time.time()
    sample = list(sources[:threads])
    rg.power_push_batch(sample, CFG["alpha"], CFG["lam"], threads)
    dt = time.time() - t0
    done = len(sample)
    while dt < budget_s * 0.5 and done < len(sources):
        more = list(sources[done:done + threads])
        t1 = time.time()
        rg.power_push_batch(more, CFG["alpha"], CFG["lam"], threads)
        dt += time.time() - t1
        done += len(more)
    return done / dt, done, dt


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    import paper_2101_03652_b200 as P
    threads = os.cpu_count() or 1
    # input data only: the R-MAT CSR comes from our generator (as for our arm);
    # the timed region is the reference's own power_push on its own Graph.
    g, srcs = make_graph(P, 0)
    off, nbr = g.out_offsets().copy(), g.out_neighbors().copy()
    cfg = workload_config(P, g, g.block_columns(len(srcs)))
    del g
    from oracle.pyoracle import CSR, Ref
    ref = Ref()
    rg = ref.graph(CSR(off, nbr))
    per_step = max(threads, 1)
    times = []
    q = 0
    for i in range(args.warmup + args.steps):
        sample = [srcs[(i * per_step + j) % len(srcs)] for j in range(per_step)]
        t0 = time.time()
        rg.power_push_batch(sample, CFG["alpha"], CFG["lam"], threads)
        dt = time.time() - t0
        if i >= args.warmup:
            times.append(dt)
            q += len(sample)
    total = sum(times)
    value = q / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * total / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": f"{per_step} power_push queries per step on {threads} "
                                       f"threads (reference libppr_core, -O3)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(P, g, K):
    return {"workload": "BASELINE configs[2]: PowerPush high-precision batch, R-MAT scale 22 "
                        "ef 16 (a=.57 b=.19 c=.19), 256 sources seed 3, graph replicated, "
                        "sources sharded",
            "graph": "rmat-22-16-seed3", "n": None if g is None else g.n(),
            "m": None if g is None else g.m(), "sources": CFG["sources"],
            "alpha": CFG["alpha"], "lambda": CFG["lam"], "epoch_num": 8,
            "columns_per_block": K, "parallelism": "source-sharded replicas",
            "l2": "inputs larger than L2 (CSR + transpose ~560 MB vs 126 MB L2)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return
    import torch

    import paper_2101_03652_b200 as P
    torch.cuda.set_device(local)
    g, srcs = make_graph(P, local)
    mine = srcs[rank::world]
    n = g.n()
    k = len(mine)
    # warm the transpose / tiles outside the timed region
    P.power_push_batch(g, mine[:1], CFG["alpha"], CFG["lam"], keep=False)

    dev_res = torch.empty((k, n), dtype=torch.float64, device=f"cuda:{local}")
    dev_rsd = torch.empty((k, n), dtype=torch.float64, device=f"cuda:{local}")

    def step_device():
        return P.power_push_batch(g, mine, CFG["alpha"], CFG["lam"],
                                  device_out=(dev_res.data_ptr(), dev_rsd.data_ptr()))

    clk = ClockSampler(local)
    clk.__enter__()  # nvidia-smi starts before the warm-up; only timed-region samples count
    for _ in range(args.warmup):
        step_device()
    barrier(world)
    torch.cuda.synchronize()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sweep_ms = dev_ms = 0.0
    alg = launches = sweep_launches = 0
    sweeps = []
    with clk:
        clk.mark_start()
        start.record()
        for _ in range(args.steps):
            outs, cs = step_device()
            sweep_ms += cs.sweep_ms
            dev_ms += cs.device_ms
            alg += cs.alg_bytes
            launches += cs.kernel_launches
            sweep_launches += cs.sweep_launches
            sweeps.append(cs.max_sweeps)
        stop.record()
        torch.cuda.synchronize()
        clk.mark_stop()
    barrier(world)
    ms = start.elapsed_time(stop)
    ms = max_over_ranks(world, ms)
    total_q = sum_over_ranks(world, float(k * args.steps))
    value = total_q / (ms / 1000.0)
    r_sums = [o.achieved_r_sum for o in outs]
    assert max(r_sums) <= CFG["lam"], "a query missed lambda"

    # ---- e2e: host buffers through the public API ---------------------------
    pin_res = torch.empty((k, n), dtype=torch.float64).pin_memory()
    pin_rsd = torch.empty((k, n), dtype=torch.float64).pin_memory()
    pin_src = torch.from_numpy(mine.astype(np.int64)).pin_memory()
    e2e_steps = args.e2e_steps or args.steps

    import ctypes
    L = P.load_library()
    L.pprg_graph_sync.argtypes = [ctypes.c_void_p]

    def step_e2e():
        # PPRG_ASYNC_HOST: a step returns once computed; its last result copies
        # land while the next step computes (pprg_graph_sync below waits for all)
        src = pin_src.numpy().astype(np.uint32)
        q = (P._abi.QStats * k)()
        c = P._abi.CStats()
        P._abi._check(L.pprg_power_push(g.handle, src.ctypes.data, k, CFG["alpha"], CFG["lam"],
                                        8, -1, pin_res.data_ptr(), pin_rsd.data_ptr(), 2, q,
                                        ctypes.byref(c), None))
        return c

    step_e2e()
    P._abi._check(L.pprg_graph_sync(g.handle))
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_launches = 0
    for _ in range(e2e_steps):
        c = step_e2e()
        e2e_launches += c.kernel_launches
    P._abi._check(L.pprg_graph_sync(g.handle))  # every step's results are on the host
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1000.0
    e2e_ms = max_over_ranks(world, e2e_ms)
    e2e_value = sum_over_ranks(world, float(k * e2e_steps)) / (e2e_ms / 1000.0)

    peak, peak_kind = peaks()
    achieved = alg / (sweep_ms / 1000.0) / 1e9 if sweep_ms > 0 else 0.0
    traffic = traffic_for("config3")
    launch_s = sweep_ms / max(sweep_launches, 1) / 1000.0
    dram_rate = traffic / launch_s / 1e9 if (traffic and launch_s > 0) else None
    # measured ms per sweep (a launch runs one block's sweeps) against the
    # gather-pattern ceiling microbenchmark (profiles/ceilings.json)
    ceil = ceiling_for("config3")
    ms_sweep = launch_s * 1000.0 / max(sweeps[-1], 1)
    gather_ceiling = None
    if ceil:
        gather_ceiling = {"ms_per_sweep": ms_sweep,
                          "ceiling_ms_per_sweep": ceil["gather_state_ms_per_sweep"],
                          "frac": ceil["gather_state_ms_per_sweep"] / ms_sweep,
                          "l2_resident_ms_per_sweep": ceil["l2_resident_gather_ms_per_sweep"],
                          "source": "profiles/ceilings.json"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(P, g, g.block_columns(k)),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 4 * k,
                    "d2h_bytes_per_step": 16 * k * n},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel": "k_sweeps<K,POWERPUSH>",
                         "alg_bytes_per_step": alg / args.steps,
                         "alg_bytes_per_launch": alg / max(sweep_launches, 1),
                         "achieved_whole_step_GBps": alg / args.steps / (ms / args.steps / 1e3) / 1e9,
                         # ncu DRAM bytes per launch over the live launch time: the rate the
                         # kernel actually moves (gather misses included), vs the same peak
                         "dram_traffic_GBps": dram_rate,
                         "dram_traffic_frac": dram_rate / peak if dram_rate else None,
                         "sweep_ms_per_step": sweep_ms / args.steps,
                         "device_ms_per_step": dev_ms / args.steps,
                         "sweeps_per_block": sweeps[-1],
                         # the sweep is bound by its y-row gathers (L2 sectors + gather
                         # misses), which the algorithmic bytes do not count: fraction of
                         # a minimal kernel with the same gathers and state traffic
                         "gather_ceiling": gather_ceiling},
            "clocks": clk.summary()}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            v, done, dt = cpu_reference_run(g.out_offsets(), g.out_neighbors(), mine, threads)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads,
                                    "kind": "reference",
                                    "sample": f"{done} power_push queries of this workload on "
                                              f"{threads} host threads in {dt:.1f}s"}
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
