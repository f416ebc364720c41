"""Command-line front end over the GPU engines — the reference's `ppr` tool
(tools/ppr_main.cpp) with the same subcommands, flags, output formats and
exit codes (0 success, 1 usage error, 2 data error):

    python -m paper_2101_03652_b200 clean --graph G [--undirected] --out G.pprg
    python -m paper_2101_03652_b200 query --graph G --algo A (--source S | --random-sources N)
                                          [--lambda L] [--epsilon E] [--mu M] [--seed X]
                                          [--epochs 8] [--scan-threshold T] [--index I] [--out F]
    python -m paper_2101_03652_b200 build-index --graph G [--seed X] --out I.pprw
    python -m paper_2101_03652_b200 groundtruth --graph G --source S --out F.csv
    python -m paper_2101_03652_b200 bench --graph G --algo A [--algo B ...] [--lambda L ...]
                                          [--epsilon E ...] (--source S | --random-sources N)
                                          [--checkpoint-every P] [--out DIR] [--name NAME]
"""
from __future__ import annotations

import argparse
import sys
import time
from typing import List, Optional

from . import _abi, formats, harness

EXIT_OK, EXIT_USAGE, EXIT_DATA = 0, 1, 2


class UsageError(RuntimeError):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit with the usage code
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def load_graph(path: str, undirected: bool) -> _abi.Graph:  # ppr_main.cpp:30-33
    if formats.is_graph_cache(path):
        return formats.load_graph_cache(path)
    return formats.undirected_to_directed(path) if undirected else formats.load_edge_list(path)


def _common(p):
    p.add_argument("--graph", required=True, help="edge list or .pprg cache")
    p.add_argument("--undirected", action="store_true",
                   help="treat each input pair as two directed edges")
    p.add_argument("--alpha", type=float, default=0.2, help="stop probability in [0,1)")


def resolve_sources(g, source: Optional[int], random_sources: int, seed: int):  # ppr_main.cpp:75-84
    if source is not None and random_sources:
        raise UsageError("--source and --random-sources are mutually exclusive")
    if source is not None:
        if source >= g.n():
            raise _abi.DataError("--source is out of range")
        return [source]
    if random_sources:
        return [int(v) for v in harness.sample_sources_uniform(g.n(), random_sources, seed)]
    raise UsageError("one of --source or --random-sources is required")


def run_clean(a) -> int:  # ppr_main.cpp:52-58
    g = load_graph(a.graph, a.undirected)
    formats.save_graph_cache(g, a.out)
    print(f"n={g.n()} m={g.m()} dead_ends={len(g.dead_ends())}")
    return EXIT_OK


def run_query(a) -> int:  # ppr_main.cpp:98-152
    if not harness.is_known_algo(a.algo):
        raise UsageError("unknown --algo (expected powitr, fwdpush-fifo, simfwdpush, "
                         "powerpush or speedppr)")
    if a.algo == harness.ALGO_SPEEDPPR and a.epsilon is None:
        raise UsageError("speedppr requires --epsilon")
    if a.source is not None and a.random_sources:
        raise UsageError("--source and --random-sources are mutually exclusive")
    g = load_graph(a.graph, a.undirected)
    cfg = _abi.QueryConfig(alpha=a.alpha, lam=a.lam, epsilon=a.epsilon, mu=a.mu, seed=a.seed,
                           epoch_num=a.epochs, scan_threshold=a.scan_threshold)
    cfg.validate()
    sources = resolve_sources(g, a.source, a.random_sources, a.seed)
    index = None
    if a.index:
        index = formats.load_index(a.index, g)
        if index.alpha() != cfg.alpha:
            raise _abi.DataError("walk index was built for a different alpha")
    lam = cfg.lambda_for(g.m())
    print("algorithm,param,edge_pushes,wall_time_ns,achieved_r_sum")
    for s in sources:
        t0 = time.perf_counter_ns()
        if a.algo == harness.ALGO_POWITR:
            r = _abi.power_iteration(g, s, cfg.alpha, lam)
        elif a.algo == harness.ALGO_SIMFWD:
            r = _abi.sim_forward_push(g, s, cfg.alpha, lam)
        elif a.algo == harness.ALGO_FIFO:
            r = _abi.fifo_forward_push(g, s, cfg.alpha, lam / float(g.m() + len(g.dead_ends())))
        elif a.algo == harness.ALGO_POWERPUSH:
            r = _abi.power_push(g, s, cfg.alpha, lam, cfg)
        else:
            r = _abi.speedppr_query(g, s, cfg, index)
        wall = time.perf_counter_ns() - t0
        param = cfg.epsilon if a.algo == harness.ALGO_SPEEDPPR else lam
        print(f"{a.algo},{harness.format_double(param)},{r.pushes},{wall},"
              f"{harness.format_double(r.achieved_r_sum)}")
        if a.out:
            path = a.out if len(sources) == 1 else f"{a.out}.{s}"
            harness.write_ppr_csv(path, r.estimates)
    return EXIT_OK


def run_build_index(a) -> int:  # ppr_main.cpp:154-161
    g = load_graph(a.graph, a.undirected)
    idx = _abi.build_index(g, a.alpha, a.seed)
    formats.save_index(idx, a.out)
    print(f"endpoints={idx.endpoint_count()}")
    return EXIT_OK


def run_groundtruth(a) -> int:  # ppr_main.cpp:163-171
    g = load_graph(a.graph, a.undirected)
    if a.source >= g.n():
        raise _abi.DataError("--source is out of range")
    harness.write_ppr_csv(a.out, _abi.ground_truth(g, a.source, a.alpha).estimates)
    return EXIT_OK


def run_bench(a) -> int:  # ppr_main.cpp:186-221
    for algo in a.algo:
        if not harness.is_known_algo(algo):
            raise UsageError("unknown algorithm: " + algo)
    g = load_graph(a.graph, a.undirected)
    if a.source is not None:
        if a.source >= g.n():
            raise _abi.DataError("--source is out of range")
        sources = [a.source]
    elif a.random_sources:
        sources = [int(v) for v in harness.sample_sources_uniform(g.n(), a.random_sources, a.seed)]
    else:
        raise UsageError("one of --source or --random-sources is required")
    plan = harness.SweepPlan(algorithms=list(a.algo),
                             lambdas=list(a.lam) if a.lam else [_abi.default_lambda(g.m())],
                             epsilons=list(a.epsilon or []), alpha=a.alpha, mu=a.mu,
                             checkpoint_every=a.checkpoint_every)
    res = harness.run_sweep(g, sources, plan)
    harness.write_sweep_csv(res, a.out, a.name)
    print(f"cells={len(res.cells)}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="ppr", description="single-source personalized PageRank engine (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    c = sub.add_parser("clean", help="parse, clean and cache a graph")
    _common(c)
    c.add_argument("--out", required=True, help="output .pprg path")
    q = sub.add_parser("query", help="run one single-source query")
    _common(q)
    q.add_argument("--algo", required=True)
    q.add_argument("--lambda", dest="lam", type=float, help="l1-error threshold (default min(1/m,1e-8))")
    q.add_argument("--epsilon", type=float, help="relative error (speedppr)")
    q.add_argument("--mu", type=float, help="PPR threshold (default 1/n)")
    q.add_argument("--source", type=int)
    q.add_argument("--random-sources", type=int, default=0)
    q.add_argument("--seed", type=int, default=0)
    q.add_argument("--epochs", type=int, default=8)
    q.add_argument("--scan-threshold", type=int)
    q.add_argument("--index", default="", help="walk index path (speedppr)")
    q.add_argument("--out", default="", help="result csv path")
    b = sub.add_parser("build-index", help="precompute the walk index")
    _common(b)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--out", required=True)
    t = sub.add_parser("groundtruth", help="reference answer at lambda=1e-17")
    _common(t)
    t.add_argument("--source", type=int, required=True)
    t.add_argument("--out", required=True)
    s = sub.add_parser("bench", help="parameter sweep with csv output")
    _common(s)
    s.add_argument("--algo", action="append", required=True, help="algorithm (repeatable)")
    s.add_argument("--lambda", dest="lam", type=float, action="append", help="lambda grid (repeatable)")
    s.add_argument("--epsilon", type=float, action="append", help="epsilon grid (repeatable)")
    s.add_argument("--source", type=int)
    s.add_argument("--random-sources", type=int, default=0)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--mu", type=float)
    s.add_argument("--checkpoint-every", type=int, default=0,
                   help="edge pushes between checkpoints (default 4m)")
    s.add_argument("--out", default=".", help="output directory")
    s.add_argument("--name", default="graph", help="prefix for csv files")
    return ap


def main(argv: Optional[List[str]] = None) -> int:  # ppr_main.cpp:223-296
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code in (0, None) else EXIT_USAGE
    run = {"clean": run_clean, "query": run_query, "build-index": run_build_index,
           "groundtruth": run_groundtruth, "bench": run_bench}[a.cmd]
    if a.cmd != "bench":
        # SPEC.md: identical argv -> identical result files for every subcommand
        _abi.set_deterministic(True)
    try:
        return run(a)
    except (UsageError, _abi.InvalidArgument) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE
    except Exception as e:  # data errors and the rest
        sys.stderr.write(f"error: {e}\n")
        return EXIT_DATA
