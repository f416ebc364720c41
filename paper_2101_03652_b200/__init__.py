"""B200-native single-source Personalized PageRank (PowerPush / PowItr / SpeedPPR).

Python mirror of the reference's C++ core API (/root/reference/proj/core/
include/ppr/*.hpp) over the engine's C ABI (include/pprg.h, lib/libpprg.so).
Same names, argument meaning and error behaviour:

    Graph(offsets, neighbors)              graph.hpp:18
    build_graph_from_edges(pairs)          graph.hpp:92
    power_iteration(g, s, alpha, lam)      push.hpp:80
    sim_forward_push / fifo_forward_push   push.hpp:86-95
    power_push(g, s, alpha, lam, cfg)      push.hpp:105
    build_index / speedppr_query           walk_index.hpp:50, speedppr.hpp:37
    compute_walk_budget                    speedppr.hpp:17
    ground_truth                           metrics.hpp:41

Every query runs on the GPU; there is no CPU fallback — the module raises if
the CUDA library is missing or no device is visible.
"""
from ._abi import (PPRVector, QueryConfig, Graph, WalkIndex, CallStats, PowerPushTrace,
                   build_graph_from_edges, generate_rmat, generate_chung_lu, power_iteration,
                   sim_forward_push, fifo_forward_push, power_push, power_push_batch,
                   power_iteration_batch, speedppr_query, speedppr_batch, build_index,
                   compute_walk_budget, walk_terminals, ground_truth, ground_truth_batch, refine, monte_carlo_phase, pinned_empty,
                   GROUND_TRUTH_LAMBDA, default_lambda, default_mu,
                   default_scan_threshold, load_library, lib_path, PPRGError, InvalidArgument,
                   DataError, LogicError, KINDEX_TAG, RNG_ID_PHILOX, set_deterministic,
                   deterministic)
from .formats import save_graph_cache, load_graph_cache, save_index, load_index, is_graph_cache
from .sources import sample_sources

__all__ = [n for n in dir() if not n.startswith("_")]
