"""ctypes binding of include/pprg.h and the reference-shaped Python API."""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.abspath(os.environ.get("PPRG_LIB") or "") if os.environ.get("PPRG_LIB") else os.path.join(_HERE, "lib", "libpprg.so")

KINDEX_TAG = 0xFFFFFFFF
RNG_ID_PHILOX = 2
OUT_DEVICE = 1


class PPRGError(RuntimeError):
    pass


class InvalidArgument(PPRGError, ValueError):
    """std::invalid_argument in the reference (PPRG_EINVAL)."""


class DataError(PPRGError):
    """std::runtime_error in the reference (PPRG_EDATA)."""


class LogicError(PPRGError):
    """std::logic_error in the reference (PPRG_EINTERNAL)."""


_ERR = {1: InvalidArgument, 2: DataError, 3: LogicError}


class QStats(C.Structure):
    _fields_ = [("achieved_r_sum", C.c_double), ("pushes", C.c_uint64), ("walks", C.c_uint64),
                ("sweeps", C.c_uint32), ("local_levels", C.c_uint32),
                ("used_scan_phase", C.c_int32), ("reserved", C.c_int32)]


class CStats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("sweep_ms", C.c_double), ("local_ms", C.c_double),
                ("final_ms", C.c_double), ("alg_bytes", C.c_uint64),
                ("sweep_launches", C.c_uint64), ("max_sweeps", C.c_uint32),
                ("kernel_launches", C.c_uint32)]


@dataclass
class CallStats:
    device_ms: float = 0.0
    sweep_ms: float = 0.0
    local_ms: float = 0.0
    final_ms: float = 0.0
    alg_bytes: int = 0
    sweep_launches: int = 0
    max_sweeps: int = 0
    kernel_launches: int = 0

    @classmethod
    def of(cls, c: CStats) -> "CallStats":
        return cls(c.device_ms, c.sweep_ms, c.local_ms, c.final_ms, c.alg_bytes,
                   c.sweep_launches, c.max_sweeps, c.kernel_launches)


_lib = None
vp = C.c_void_p
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


def load_library(path: str = lib_path):
    """Load lib/libpprg.so. Raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise PPRGError(f"{path} not built: run `make -C paper_2101_03652_b200` "
                        "(or __graft_entry__.build())")
    L = C.CDLL(path)
    L.pprg_last_error.restype = C.c_char_p
    L.pprg_graph_create.argtypes = [vp, vp, C.c_uint64, C.c_int, C.POINTER(vp)]
    L.pprg_graph_build_from_edges.argtypes = [vp, C.c_uint64, C.c_int, C.POINTER(vp)]
    L.pprg_graph_generate_rmat.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                           C.c_uint64, C.c_int, vp, u64p, C.POINTER(vp)]
    L.pprg_graph_generate_chung_lu.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                               C.c_int, vp, u64p, C.POINTER(vp)]
    L.pprg_graph_info.argtypes = [vp, u64p, u64p, u64p]
    L.pprg_graph_export.argtypes = [vp, vp, vp, vp]
    L.pprg_graph_export_transpose.argtypes = [vp, vp, vp]
    L.pprg_graph_destroy.argtypes = [vp]
    L.pprg_graph_destroy.restype = None
    eng = [vp, vp, C.c_uint32, C.c_double, C.c_double, vp, vp, C.c_uint32, vp, vp]
    L.pprg_power_iteration.argtypes = eng
    L.pprg_sim_forward_push.argtypes = eng
    L.pprg_fifo_forward_push.argtypes = [vp, vp, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                         vp, vp, C.c_uint32, vp, vp]
    L.pprg_power_push.argtypes = [vp, vp, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                                  C.c_int64, vp, vp, C.c_uint32, vp, vp, vp]
    L.pprg_walk_budget.argtypes = [C.c_uint64, C.c_double, C.c_double, u64p]
    L.pprg_graph_load_cache.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
    L.pprg_graph_save_cache.argtypes = [vp, C.c_char_p]
    L.pprg_index_load.argtypes = [vp, C.c_char_p, C.POINTER(vp)]
    L.pprg_index_save.argtypes = [vp, C.c_char_p]
    L.pprg_monte_carlo.argtypes = [vp, vp, C.c_uint32, C.c_double, C.c_uint64, C.c_uint64, vp, vp,
                                   vp, u64p]
    L.pprg_refine.argtypes = [vp, vp, C.c_uint32, C.c_double, C.c_double, vp, vp, C.c_uint32, vp,
                              vp]
    L.pprg_ground_truth.argtypes = [vp, vp, C.c_uint32, C.c_double, vp, C.c_uint32, vp, vp]
    L.pprg_block_columns.argtypes = [vp, C.c_uint32, C.POINTER(C.c_uint32)]
    L.pprg_uses_delta_sweeps.argtypes = [vp, C.c_uint32, C.POINTER(C.c_int)]
    L.pprg_index_build.argtypes = [vp, C.c_double, C.c_uint64, C.POINTER(vp)]
    L.pprg_index_from_host.argtypes = [vp, C.c_double, C.c_uint64, vp, C.POINTER(vp)]
    L.pprg_index_export.argtypes = [vp, vp]
    L.pprg_index_destroy.argtypes = [vp]
    L.pprg_index_destroy.restype = None
    L.pprg_speedppr.argtypes = [vp, vp, vp, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                C.c_uint64, vp, C.c_uint32, vp, vp]
    L.pprg_walk_terminals.argtypes = [vp, vp, vp, vp, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_double, C.c_uint64, vp]
    L.pprg_device_count.argtypes = [C.POINTER(C.c_int)]
    L.pprg_host_alloc.argtypes = [C.c_uint64, C.POINTER(vp)]
    L.pprg_graph_sync.argtypes = [vp]
    L.pprg_host_free.argtypes = [vp]
    L.pprg_device_alloc.argtypes = [C.c_int, C.c_uint64, C.POINTER(vp)]
    L.pprg_device_free.argtypes = [C.c_int, vp]
    if hasattr(L, "pprg_set_deterministic"):  # (older builds loaded through PPRG_LIB lack it)
        L.pprg_set_deterministic.argtypes = [C.c_int]
    _lib = L
    return L


def set_deterministic(on: bool = True) -> None:
    """Process-wide PPRG_DETERMINISTIC (include/pprg.h): every later query returns
    bitwise-identical results for identical inputs (the reference's rerun
    guarantee), at the cost of more sweeps. Off by default."""
    _check(load_library().pprg_set_deterministic(1 if on else 0))


class deterministic:
    """Context manager: deterministic queries inside the block."""

    def __init__(self, on: bool = True):
        self.on = on

    def __enter__(self):
        set_deterministic(self.on)
        return self

    def __exit__(self, *exc):
        set_deterministic(False)
        return False


def _check(rc):
    if rc:
        msg = _lib.pprg_last_error().decode(errors="replace")
        raise _ERR.get(rc, PPRGError)(msg)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _default_device() -> int:
    for key in ("PPRG_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


# ---- types.hpp ---------------------------------------------------------------
def default_lambda(m: int) -> float:  # types.hpp:17-19
    return min(1.0 / float(m), 1e-8)


def default_mu(n: int) -> float:  # types.hpp:22
    return 1.0 / float(n)


def default_scan_threshold(n: int) -> int:  # types.hpp:25
    return n // 4


@dataclass
class QueryConfig:  # types.hpp:27-53
    alpha: float = 0.2
    lam: Optional[float] = None
    epsilon: Optional[float] = None
    mu: Optional[float] = None
    seed: int = 0
    epoch_num: int = 8
    scan_threshold: Optional[int] = None

    def validate(self):
        if not (0.0 <= self.alpha < 1.0):
            raise InvalidArgument("alpha must be in [0,1)")
        if self.lam is not None and not (0.0 < self.lam <= 1.0):
            raise InvalidArgument("lambda must be in (0,1]")
        if self.epsilon is not None and not (self.epsilon > 0.0):
            raise InvalidArgument("epsilon must be positive")
        if self.mu is not None and not (0.0 < self.mu <= 1.0):
            raise InvalidArgument("mu must be in (0,1]")
        if self.epoch_num == 0:
            raise InvalidArgument("epoch_num must be positive")

    def lambda_for(self, m):
        return self.lam if self.lam is not None else default_lambda(m)

    def mu_for(self, n):
        return self.mu if self.mu is not None else default_mu(n)

    def scan_threshold_for(self, n):
        return self.scan_threshold if self.scan_threshold is not None else default_scan_threshold(n)


@dataclass
class PPRVector:  # types.hpp:57-65
    estimates: np.ndarray
    residues: np.ndarray
    source: int = 0
    alpha: float = 0.2
    achieved_r_sum: float = 0.0
    pushes: int = 0
    walks: int = 0
    sweeps: int = 0
    local_levels: int = 0
    used_scan_phase: bool = False


@dataclass
class PowerPushTrace:  # push.hpp:97-100
    used_scan_phase: bool = False
    epoch_r_max: list = field(default_factory=list)


# ---- graph.hpp -----------------------------------------------------------------
class Graph:
    """Device-resident immutable CSR graph (graph.hpp:16-55)."""

    def __init__(self, out_offsets=None, out_neighbors=None, device: Optional[int] = None,
                 _handle=None):
        L = load_library()
        self.device = _default_device() if device is None else device
        self._h = vp()
        if _handle is not None:
            self._h = _handle
        else:
            off = np.ascontiguousarray(out_offsets, dtype=np.uint64)
            nbr = np.ascontiguousarray(out_neighbors, dtype=np.uint32)
            if off.size == 0:
                raise DataError("graph: offsets array must have length n+1")  # graph.cpp:15-16
            if int(off[-1]) != nbr.size:
                raise DataError("graph: offsets must end at m")
            _check(L.pprg_graph_create(_ptr(off), _ptr(nbr) if nbr.size else None, off.size - 1,
                                       self.device, C.byref(self._h)))
        n, m, d = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(L.pprg_graph_info(self._h, C.byref(n), C.byref(m), C.byref(d)))
        self._n, self._m, self._nd = n.value, m.value, d.value
        self._off = self._nbr = self._dead = None

    def __del__(self):
        try:
            if self._h:
                _lib.pprg_graph_destroy(self._h)
                self._h = vp()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def n(self) -> int:
        return self._n

    def m(self) -> int:
        return self._m

    def _export(self):
        if self._off is None:
            off = np.zeros(self._n + 1, np.uint64)
            nbr = np.zeros(max(self._m, 1), np.uint32)
            dead = np.zeros(max(self._nd, 1), np.uint32)
            _check(_lib.pprg_graph_export(self._h, _ptr(off), _ptr(nbr), _ptr(dead)))
            self._off, self._nbr, self._dead = off, nbr[: self._m], dead[: self._nd]

    def out_offsets(self) -> np.ndarray:
        self._export()
        return self._off

    def out_neighbors(self) -> np.ndarray:
        self._export()
        return self._nbr

    def dead_ends(self) -> np.ndarray:
        self._export()
        return self._dead

    def block_columns(self, k: int) -> int:
        """Columns per device block the engines use for a k-source call."""
        out = C.c_uint32()
        _check(load_library().pprg_block_columns(self.handle, k, C.byref(out)))
        return out.value

    def uses_delta_sweeps(self, k: int) -> bool:
        """True if a k-source power_push call runs its global phase as delta sweeps."""
        out = C.c_int()
        _check(load_library().pprg_uses_delta_sweeps(self.handle, k, C.byref(out)))
        return bool(out.value)

    def out_degree(self, v: int) -> int:
        off = self.out_offsets()
        return int(off[v + 1] - off[v])

    def is_dead_end(self, v: int) -> bool:
        return self.out_degree(v) == 0

    def neighbors(self, v: int) -> np.ndarray:
        off = self.out_offsets()
        return self.out_neighbors()[int(off[v]): int(off[v + 1])]

    def effective_edge_count(self) -> int:
        return self._m + self._nd

    def transpose(self):
        ioff = np.zeros(self._n + 1, np.uint64)
        inbr = np.zeros(max(self._m, 1), np.uint32)
        _check(_lib.pprg_graph_export_transpose(self._h, _ptr(ioff), _ptr(inbr)))
        return ioff, inbr[: self._m]


def effective_degree(g: Graph, v: int) -> int:  # graph.hpp:83-86
    d = g.out_degree(v)
    return d if d else 1


def build_graph_from_edges(edges, device: Optional[int] = None) -> Graph:
    """graph.cpp:36-63 on the GPU (bit-exact relabel and input-order scatter)."""
    L = load_library()
    pairs = np.ascontiguousarray(np.asarray(edges, dtype=np.uint64).reshape(-1, 2))
    dev = _default_device() if device is None else device
    h = vp()
    _check(L.pprg_graph_build_from_edges(_ptr(pairs) if len(pairs) else None, len(pairs), dev,
                                         C.byref(h)))
    return Graph(device=dev, _handle=h)


def generate_rmat(scale: int, edge_factor: int, seed: int, a=0.57, b=0.19, c=0.19,
                  device: Optional[int] = None, return_edges=False):
    """Directed R-MAT, cleaned; Philox keyed (seed, edge index)."""
    L = load_library()
    dev = _default_device() if device is None else device
    h = vp()
    cnt = C.c_uint64()
    edges = np.zeros(edge_factor << scale, np.uint64) if return_edges else None
    _check(L.pprg_graph_generate_rmat(scale, edge_factor, a, b, c, seed, dev, _ptr(edges),
                                      C.byref(cnt), C.byref(h)))
    g = Graph(device=dev, _handle=h)
    if return_edges:
        e = edges[: cnt.value]
        return g, np.stack([e >> np.uint64(32), e & np.uint64(0xFFFFFFFF)], axis=1)
    return g


def generate_chung_lu(n: int, draws: int, seed: int, beta=2.1, device: Optional[int] = None,
                      return_edges=False):
    L = load_library()
    dev = _default_device() if device is None else device
    h = vp()
    cnt = C.c_uint64()
    edges = np.zeros(draws, np.uint64) if return_edges else None
    _check(L.pprg_graph_generate_chung_lu(n, draws, beta, seed, dev, _ptr(edges), C.byref(cnt),
                                          C.byref(h)))
    g = Graph(device=dev, _handle=h)
    if return_edges:
        e = edges[: cnt.value]
        return g, np.stack([e >> np.uint64(32), e & np.uint64(0xFFFFFFFF)], axis=1)
    return g


# ---- engines (push.hpp) --------------------------------------------------------
def _sources(sources) -> np.ndarray:
    return np.ascontiguousarray(np.atleast_1d(np.asarray(sources, dtype=np.uint32)))


class _Pinned:
    """Owner of a page-locked host allocation (pprg_host_alloc)."""

    def __init__(self, nbytes: int):
        self.p = vp()
        _check(load_library().pprg_host_alloc(max(nbytes, 1), C.byref(self.p)))

    def __del__(self):
        try:
            if self.p:
                _lib.pprg_host_free(self.p)
                self.p = vp()
        except Exception:
            pass


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (freed with the array)."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape))
    owner = _Pinned(n * dt.itemsize)
    buf = (C.c_char * max(n * dt.itemsize, 1)).from_address(owner.p.value)
    arr = np.frombuffer(buf, dtype=dt, count=n).reshape(shape)
    arr_owner = _PinnedArray(arr, owner)
    return arr_owner.view


class _PinnedArray:
    def __init__(self, arr, owner):
        self.view = arr.view(_PinnedNd)
        self.view._owner = owner


class _PinnedNd(np.ndarray):
    """ndarray subclass that keeps its page-locked allocation alive."""

    def __array_finalize__(self, obj):
        self._owner = getattr(obj, "_owner", None)


def _outs(g: Graph, k: int, keep: bool, device_out, host_out=None):
    if device_out is not None:
        return None, None, device_out[0], device_out[1], OUT_DEVICE
    if host_out is not None:  # caller's arrays, e.g. pinned_empty((k, n)) reused across calls
        res, rsd = host_out
        for a in (res, rsd):
            if a is not None and (a.dtype != np.float64 or a.shape != (k, g.n())
                                  or not a.flags.c_contiguous):
                raise InvalidArgument("host_out arrays must be C-contiguous float64 (k, n)")
        return (res, rsd, res.ctypes.data if res is not None else None,
                rsd.ctypes.data if rsd is not None else None, 0)
    if not keep:
        return None, None, None, None, 0
    res = np.empty((k, g.n()), np.float64)
    rsd = np.empty((k, g.n()), np.float64)
    return res, rsd, res.ctypes.data, rsd.ctypes.data, 0


def _vectors(src, res, rsd, q, alpha):
    out = []
    for i, s in enumerate(src):
        out.append(PPRVector(res[i] if res is not None else None,
                             rsd[i] if rsd is not None else None, int(s), alpha,
                             q[i].achieved_r_sum, q[i].pushes, q[i].walks, q[i].sweeps,
                             q[i].local_levels, bool(q[i].used_scan_phase)))
    return out


def power_push_batch(g: Graph, sources, alpha: float, lam: float, epoch_num: int = 8,
                     scan_threshold: Optional[int] = None, keep: bool = True, device_out=None,
                     host_out=None):
    """k independent power_push queries as one column block per <= 64 sources.
    host_out = (reserve, residue) caller arrays (k, n) — page-locked ones from
    pinned_empty() make the result copies overlap the next block's compute.
    Returns (list[PPRVector], CallStats)."""
    load_library()
    src = _sources(sources)
    res, rsd, rp, dp, flags = _outs(g, len(src), keep, device_out, host_out)
    q = (QStats * max(len(src), 1))()
    cs = CStats()
    _check(_lib.pprg_power_push(g.handle, _ptr(src), len(src), alpha, lam, epoch_num,
                                -1 if scan_threshold is None else scan_threshold, rp, dp, flags,
                                q, C.byref(cs), None))
    return _vectors(src, res, rsd, q, alpha), CallStats.of(cs)


def power_iteration_batch(g: Graph, sources, alpha: float, lam: float, keep=True, device_out=None,
                          simultaneous=False):
    load_library()
    src = _sources(sources)
    res, rsd, rp, dp, flags = _outs(g, len(src), keep, device_out)
    q = (QStats * max(len(src), 1))()
    cs = CStats()
    fn = _lib.pprg_sim_forward_push if simultaneous else _lib.pprg_power_iteration
    _check(fn(g.handle, _ptr(src), len(src), alpha, lam, rp, dp, flags, q, C.byref(cs)))
    return _vectors(src, res, rsd, q, alpha), CallStats.of(cs)


def power_iteration(g: Graph, s: int, alpha: float, lam: float) -> PPRVector:
    """push.hpp:80-81 (push.cpp:81-108)."""
    return power_iteration_batch(g, [s], alpha, lam)[0][0]


def sim_forward_push(g: Graph, s: int, alpha: float, lam: float) -> PPRVector:
    """push.hpp:86-87 (push.cpp:110-138)."""
    return power_iteration_batch(g, [s], alpha, lam, simultaneous=True)[0][0]


def fifo_forward_push(g: Graph, s: int, alpha: float, r_max: float,
                      lambda_stop: Optional[float] = None) -> PPRVector:
    """push.hpp:92-94 (push.cpp:140-149)."""
    load_library()
    src = _sources([s])
    res, rsd, rp, dp, flags = _outs(g, 1, True, None)
    q = (QStats * 1)()
    cs = CStats()
    _check(_lib.pprg_fifo_forward_push(g.handle, _ptr(src), 1, alpha, r_max,
                                       lambda_stop if lambda_stop is not None else -1.0, rp, dp,
                                       flags, q, C.byref(cs)))
    return _vectors(src, res, rsd, q, alpha)[0]


def refine(g: Graph, s: int, alpha: float, r_max: float, state: PPRVector) -> PPRVector:
    """refine (push.hpp:118-119, push.cpp:208-222) of a push state given as a
    PPRVector (estimates = reserve, residues); returns the refined state."""
    load_library()
    if not (r_max > 0.0):
        raise InvalidArgument("refine: r_max must be positive")
    src = _sources([s])
    res = np.ascontiguousarray(state.estimates, np.float64).copy().reshape(1, -1)
    rsd = np.ascontiguousarray(state.residues, np.float64).copy().reshape(1, -1)
    q = (QStats * 1)()
    _check(_lib.pprg_refine(g.handle, _ptr(src), 1, alpha, r_max, res.ctypes.data, rsd.ctypes.data,
                            0, q, None))
    out = _vectors(src, res, rsd, q, alpha)[0]
    out.pushes = state.pushes + q[0].pushes
    return out


def monte_carlo_phase(g: Graph, s: int, alpha: float, state: PPRVector, walk_budget: int,
                      seed: int, index: Optional["WalkIndex"] = None) -> PPRVector:
    """monte_carlo_phase (speedppr.hpp:24-30, speedppr.cpp:23-72) on a refined
    push state (estimates = reserve, residues); Philox walks keyed by seed."""
    load_library()
    res = np.ascontiguousarray(state.estimates, np.float64)
    rsd = np.ascontiguousarray(state.residues, np.float64)
    out = np.empty(g.n(), np.float64)
    walks = C.c_uint64()
    _check(_lib.pprg_monte_carlo(g.handle, index._h if index is not None else None, int(s), alpha,
                                 int(walk_budget), int(seed), res.ctypes.data, rsd.ctypes.data,
                                 out.ctypes.data, C.byref(walks)))
    return PPRVector(out, np.zeros(g.n()), int(s), alpha, 0.0, state.pushes, int(walks.value))


GROUND_TRUTH_LAMBDA = 1e-17  # kGroundTruthLambda, metrics.hpp:10


def ground_truth_batch(g: Graph, sources, alpha: float):
    """ground_truth for k sources (metrics.cpp:44-55): reserve with r_sum <= 1e-17.
    Returns (list[PPRVector] without residues, CallStats)."""
    load_library()
    src = _sources(sources)
    res = np.empty((len(src), g.n()), np.float64)
    q = (QStats * max(len(src), 1))()
    cs = CStats()
    _check(_lib.pprg_ground_truth(g.handle, _ptr(src), len(src), alpha, res.ctypes.data, 0, q,
                                  C.byref(cs)))
    return _vectors(src, res, None, q, alpha), CallStats.of(cs)


def ground_truth(g: Graph, s: int, alpha: float) -> PPRVector:
    """metrics.hpp:41 (metrics.cpp:44-55)."""
    return ground_truth_batch(g, [s], alpha)[0][0]


def power_push(g: Graph, s: int, alpha: float, lam: float, cfg: Optional[QueryConfig] = None,
               trace: Optional[PowerPushTrace] = None) -> PPRVector:
    """push.hpp:105-107 (push.cpp:151-206)."""
    cfg = cfg or QueryConfig()
    load_library()
    src = _sources([s])
    res, rsd, rp, dp, flags = _outs(g, 1, True, None)
    q = (QStats * 1)()
    cs = CStats()
    ep = np.zeros(max(cfg.epoch_num, 1), np.float64)
    _check(_lib.pprg_power_push(g.handle, _ptr(src), 1, alpha, lam, cfg.epoch_num,
                                -1 if cfg.scan_threshold is None else cfg.scan_threshold, rp, dp,
                                flags, q, C.byref(cs), _ptr(ep)))
    out = _vectors(src, res, rsd, q, alpha)[0]
    if trace is not None:
        trace.used_scan_phase = out.used_scan_phase
        trace.epoch_r_max = list(ep[: cfg.epoch_num]) if out.used_scan_phase else []
    return out


# ---- SpeedPPR (speedppr.hpp / walk_index.hpp) ----------------------------------------
def compute_walk_budget(n: int, epsilon: float, mu: float) -> int:
    load_library()
    out = C.c_uint64()
    _check(_lib.pprg_walk_budget(n, epsilon, mu, C.byref(out)))
    return out.value


class WalkIndex:
    """Device-resident walk index (walk_index.hpp:21-46); rng-id 2 (Philox)."""

    def __init__(self, g: Graph, alpha: float, seed: int, handle):
        self.graph, self._alpha, self._seed, self._h = g, alpha, seed, handle

    def __del__(self):
        try:
            if self._h:
                _lib.pprg_index_destroy(self._h)
                self._h = vp()
        except Exception:
            pass

    def alpha(self):
        return self._alpha

    def seed(self):
        return self._seed

    def rng_id(self):
        return RNG_ID_PHILOX

    def node_count(self):
        return self.graph.n()

    def endpoint_count(self):
        return self.graph.m()

    def endpoints(self) -> np.ndarray:
        out = np.zeros(max(self.graph.m(), 1), np.uint32)
        _check(_lib.pprg_index_export(self._h, _ptr(out)))
        return out[: self.graph.m()]

    def endpoints_of(self, v: int) -> np.ndarray:
        off = self.graph.out_offsets()
        return self.endpoints()[int(off[v]): int(off[v + 1])]

    def check_compatible(self, g: Graph):
        if g.n() != self.graph.n() or g.m() != self.graph.m() or not np.array_equal(
                g.out_offsets(), self.graph.out_offsets()):
            raise DataError("walk index does not match the graph shape")

    @classmethod
    def from_endpoints(cls, g: Graph, alpha: float, seed: int, endpoints) -> "WalkIndex":
        load_library()
        ep = np.ascontiguousarray(endpoints, np.uint32)
        if ep.size != g.m():
            raise DataError("walk index does not match the graph shape")
        h = vp()
        _check(_lib.pprg_index_from_host(g.handle, alpha, seed, _ptr(ep) if ep.size else None,
                                         C.byref(h)))
        return cls(g, alpha, seed, h)


def build_index(g: Graph, alpha: float, seed: int) -> WalkIndex:
    load_library()
    h = vp()
    _check(_lib.pprg_index_build(g.handle, alpha, seed, C.byref(h)))
    return WalkIndex(g, alpha, seed, h)


def speedppr_batch(g: Graph, sources, cfg: QueryConfig, index: Optional[WalkIndex] = None,
                   keep=True, device_out=None, host_out=None):
    load_library()
    cfg.validate()
    if cfg.epsilon is None:
        raise InvalidArgument("speedppr: epsilon is required")
    src = _sources(sources)
    if index is not None:
        index.check_compatible(g)
        if index.alpha() != cfg.alpha:
            raise DataError("walk index was built for a different alpha")
    k = len(src)
    est = None
    ep = None
    flags = 0
    if device_out is not None:
        ep, flags = device_out, OUT_DEVICE
    elif host_out is not None:  # e.g. pinned_empty((k, n)), reused across calls
        est = host_out
        if est.dtype != np.float64 or est.shape != (k, g.n()) or not est.flags.c_contiguous:
            raise InvalidArgument("host_out must be a C-contiguous float64 (k, n) array")
        ep = est.ctypes.data
    elif keep:
        est = np.empty((k, g.n()), np.float64)
        ep = est.ctypes.data
    q = (QStats * max(k, 1))()
    cs = CStats()
    _check(_lib.pprg_speedppr(g.handle, index._h if index is not None else None, _ptr(src), k,
                              cfg.alpha, cfg.epsilon, cfg.mu if cfg.mu is not None else -1.0,
                              cfg.seed, ep, flags, q, C.byref(cs)))
    zeros = np.zeros((k, g.n())) if (keep or host_out is not None) else None
    return _vectors(src, est, zeros, q, cfg.alpha), CallStats.of(cs)


def speedppr_query(g: Graph, s: int, cfg: QueryConfig, index: Optional[WalkIndex] = None):
    """speedppr.hpp:37-38 (speedppr.cpp:74-111)."""
    if s >= g.n():
        raise InvalidArgument("speedppr: source out of range")
    return speedppr_batch(g, [s], cfg, index)[0][0]


def walk_terminals(g: Graph, starts, ks, vs, source: int, tag: int, alpha: float, seed: int):
    load_library()
    s = np.ascontiguousarray(starts, np.uint32)
    k = np.ascontiguousarray(ks, np.uint32)
    v = np.ascontiguousarray(vs, np.uint32)
    out = np.zeros(max(len(s), 1), np.uint32)
    _check(_lib.pprg_walk_terminals(g.handle, _ptr(s), _ptr(k), _ptr(v), len(s), source, tag, alpha,
                                    seed, _ptr(out)))
    return out[: len(s)]
