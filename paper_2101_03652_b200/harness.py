"""Accuracy metrics, PPR csv files and the parameter-sweep harness — the
reference's metrics.hpp, csv.hpp and sweep.hpp (core/src/metrics.cpp,
csv.cpp, sweep.cpp) over the GPU engines.

Checkpoints (the reference's CheckpointRecorder, sweep.cpp:25-38) come from
the engine's per-step progress series (`pprg_run_traced`): one point per
global sweep, iteration or frontier level rather than per push, filtered with
the reference's cadence rule (a checkpoint when the cumulative edge pushes
reach the next multiple of the cadence, default 4m).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import PPRVector, QStats, QueryConfig, _check, default_lambda, default_mu, load_library

ALGO_POWITR = "powitr"            # sweep.hpp:15-19
ALGO_FIFO = "fwdpush-fifo"
ALGO_SIMFWD = "simfwdpush"
ALGO_POWERPUSH = "powerpush"
ALGO_SPEEDPPR = "speedppr"
_ALGO_ID = {ALGO_POWITR: 0, ALGO_SIMFWD: 1, ALGO_FIFO: 2, ALGO_POWERPUSH: 3}


def is_high_precision_algo(name: str) -> bool:  # sweep.cpp:16-19
    return name in _ALGO_ID


def is_known_algo(name: str) -> bool:  # sweep.cpp:21-23
    return is_high_precision_algo(name) or name == ALGO_SPEEDPPR


# ---- metrics.hpp ----------------------------------------------------------------
def l1_error(estimate, truth) -> float:  # metrics.cpp:11-18
    estimate, truth = np.asarray(estimate), np.asarray(truth)
    if estimate.shape != truth.shape:
        raise _abi.InvalidArgument("l1_error: vector lengths differ")
    return float(np.abs(estimate - truth).sum())


@dataclass
class ErrorReport:  # metrics.hpp:17-22
    l1: float = 0.0
    max_rel_above_mu: float = 0.0
    nodes_above_mu: int = 0
    violations: int = 0


def compare_to_truth(estimate, truth, mu: float, epsilon: float) -> ErrorReport:  # metrics.cpp:27-42
    estimate, truth = np.asarray(estimate, np.float64), np.asarray(truth, np.float64)
    if estimate.shape != truth.shape:
        raise _abi.InvalidArgument("compare_to_truth: vector lengths differ")
    diff = np.abs(estimate - truth)
    above = truth >= mu
    rel = diff[above] / truth[above]
    return ErrorReport(float(diff.sum()), float(rel.max()) if rel.size else 0.0,
                       int(above.sum()), int((rel > epsilon).sum()))


# ---- csv.hpp --------------------------------------------------------------------
def format_double(v: float) -> str:  # csv.cpp:9-13
    return "%.17g" % v


def write_ppr_csv(path: str, values) -> None:  # csv.cpp:15-22
    try:
        with open(path, "w") as f:
            f.write("node,ppr\n")
            f.writelines(f"{v},{format_double(x)}\n" for v, x in enumerate(np.asarray(values)))
    except OSError:
        raise _abi.DataError("cannot open for writing: " + path)


def read_ppr_csv(path: str) -> np.ndarray:  # csv.cpp:24-43
    try:
        f = open(path)
    except OSError:
        raise _abi.DataError("cannot open: " + path)
    with f:
        if f.readline().rstrip("\n") != "node,ppr":
            raise _abi.DataError(path + ": missing node,ppr header")
        vals = []
        for line in f:
            line = line.rstrip("\n")
            if not line:
                continue
            if "," not in line:
                raise _abi.DataError(path + ": malformed row: " + line)
            a, b = line.split(",", 1)
            if int(a) != len(vals):
                raise _abi.DataError(path + ": node ids must be consecutive from 0")
            vals.append(float(b))
    return np.asarray(vals, np.float64)


# ---- sweep.hpp ------------------------------------------------------------------
@dataclass
class Checkpoint:  # sweep.hpp:25-29
    pushes: int = 0
    r_sum: float = 0.0
    time_ns: int = 0


class _CPoint(C.Structure):
    _fields_ = [("pushes", C.c_uint64), ("r_sum", C.c_double), ("time_ns", C.c_uint64)]


def _lib():
    L = load_library()
    if not getattr(L, "_harness_bound", False):
        L.pprg_run_traced.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_double, C.c_double,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                      C.POINTER(C.c_uint32)]
        L._harness_bound = True
    return L


def run_traced(g: _abi.Graph, algo: str, s: int, alpha: float, lam: float, capacity: int = 1 << 16):
    """run_high_precision (sweep.cpp:50-61) with its per-step progress series.
    Returns (PPRVector without residues, list[Checkpoint] of every step)."""
    if not is_high_precision_algo(algo):
        raise _abi.InvalidArgument("unknown algorithm: " + algo)
    est = np.empty(g.n(), np.float64)
    q = QStats()
    pts = (_CPoint * capacity)()
    cnt = C.c_uint32()
    _check(_lib().pprg_run_traced(g.handle, _ALGO_ID[algo], int(s), alpha, lam, est.ctypes.data,
                                  C.byref(q), pts, capacity, C.byref(cnt)))
    out = PPRVector(est, None, int(s), alpha, q.achieved_r_sum, q.pushes, q.walks, q.sweeps,
                    q.local_levels, bool(q.used_scan_phase))
    return out, [Checkpoint(p.pushes, p.r_sum, p.time_ns) for p in pts[:cnt.value]]


def cadence_filter(points: Sequence[Checkpoint], cadence: int) -> List[Checkpoint]:
    """CheckpointRecorder::on_push (sweep.cpp:30-38) applied to step points."""
    cadence = cadence or 1
    nxt, out = cadence, []
    for p in points:
        if p.pushes < nxt:
            continue
        out.append(p)
        while nxt <= p.pushes:
            nxt += cadence
    return out


@dataclass
class SweepPlan:  # sweep.hpp:48-56
    algorithms: List[str] = field(default_factory=list)
    lambdas: List[float] = field(default_factory=list)
    epsilons: List[float] = field(default_factory=list)
    seeds: List[int] = field(default_factory=lambda: [0])
    alpha: float = 0.2
    mu: Optional[float] = None
    checkpoint_every: int = 0


@dataclass
class SweepRow:  # sweep.hpp:58-67
    source: int = 0
    algo: str = ""
    param: float = 0.0
    wall_time_ns: int = 0
    edge_pushes: int = 0
    walks: int = 0
    l1_error: float = 0.0
    max_rel_error: float = 0.0


@dataclass
class SweepCell:
    row: SweepRow
    checkpoints: List[Checkpoint] = field(default_factory=list)


@dataclass
class SweepResult:
    cells: List[SweepCell] = field(default_factory=list)


def run_sweep(g: _abi.Graph, sources: Sequence[int], plan: SweepPlan,
              index: Optional[_abi.WalkIndex] = None) -> SweepResult:  # sweep.cpp:64-118
    for a in plan.algorithms:
        if not is_known_algo(a):
            raise _abi.InvalidArgument("unknown algorithm: " + a)
    cadence = plan.checkpoint_every or 4 * g.m()
    mu = plan.mu if plan.mu is not None else default_mu(g.n())
    res = SweepResult()
    for s in sources:
        truth = _abi.ground_truth(g, int(s), plan.alpha).estimates
        for algo in plan.algorithms:
            if is_high_precision_algo(algo):
                for lam in plan.lambdas:
                    t0 = time.perf_counter_ns()
                    got, pts = run_traced(g, algo, int(s), plan.alpha, lam)
                    wall = time.perf_counter_ns() - t0
                    rep = compare_to_truth(got.estimates, truth, mu, 0.0)
                    res.cells.append(SweepCell(
                        SweepRow(int(s), algo, lam, wall, got.pushes, got.walks, rep.l1,
                                 rep.max_rel_above_mu), cadence_filter(pts, cadence)))
            else:
                for eps in plan.epsilons:
                    for seed in plan.seeds:
                        cfg = QueryConfig(alpha=plan.alpha, epsilon=eps, mu=plan.mu, seed=seed)
                        t0 = time.perf_counter_ns()
                        got = _abi.speedppr_query(g, int(s), cfg, index)
                        wall = time.perf_counter_ns() - t0
                        rep = compare_to_truth(got.estimates, truth, mu, eps)
                        res.cells.append(SweepCell(
                            SweepRow(int(s), algo, eps, wall, got.pushes, got.walks, rep.l1,
                                     rep.max_rel_above_mu)))
    return res


def write_sweep_csv(result: SweepResult, directory: str, graph_name: str) -> None:  # sweep.cpp:120-140
    os.makedirs(directory, exist_ok=True)
    try:
        summary = open(os.path.join(directory, graph_name + "_sweep.csv"), "w")
    except OSError:
        raise _abi.DataError("cannot write sweep summary")
    with summary:
        summary.write("source,algo,param,wall_time_ns,edge_pushes,walks,l1_error,max_rel_error\n")
        for cell in result.cells:
            r = cell.row
            summary.write(f"{r.source},{r.algo},{format_double(r.param)},{r.wall_time_ns},"
                          f"{r.edge_pushes},{r.walks},{format_double(r.l1_error)},"
                          f"{format_double(r.max_rel_error)}\n")
            if cell.checkpoints:
                name = f"{graph_name}_{r.algo}_{'%g' % r.param}.csv"
                with open(os.path.join(directory, name), "w") as f:
                    f.write("pushes,r_sum,time_ns\n")
                    for c in cell.checkpoints:
                        f.write(f"{c.pushes},{format_double(c.r_sum)},{c.time_ns}\n")


def sample_sources_uniform(n: int, count: int, seed: int) -> np.ndarray:
    """sample_sources (sweep.cpp:142-147): Rng(seed).below(n), count times."""
    from .sources import Mt19937_64
    rng = Mt19937_64(seed)
    return np.asarray([rng.below(n) for _ in range(count)], np.uint32)
