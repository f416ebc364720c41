"""TEST INFRASTRUCTURE ONLY: numpy/ctypes views of the two CPU checkers.

* ``Oracle``  -> oracle/liboracle.so, our plain-C restatement (oracle.c).
* ``Ref``     -> oracle/_ref/libppr_ref.so, the reference library compiled
  unchanged from /root/reference (see oracle/Makefile) behind ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` arm may import this module, and only as the checker or
the measured CPU baseline; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libppr_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
vp = C.c_void_p


class OracleError(RuntimeError):
    pass


class InvalidArgument(OracleError, ValueError):
    """status 1: std::invalid_argument in the reference"""


class DataError(OracleError):
    """status 2: std::runtime_error in the reference"""


class LogicError(OracleError):
    """status 3: std::logic_error in the reference"""


_ERR = {1: InvalidArgument, 2: DataError, 3: LogicError}


def _check(rc, msg=""):
    if rc:
        raise _ERR.get(rc, OracleError)(f"status {rc} {msg}")


class OgStats(C.Structure):
    _fields_ = [("r_sum", C.c_double), ("pushes", C.c_uint64), ("iterations", C.c_uint32),
                ("used_scan_phase", C.c_int), ("local_node_pushes", C.c_uint64)]


class OgErrorReport(C.Structure):
    _fields_ = [("l1", C.c_double), ("max_rel_above_mu", C.c_double),
                ("nodes_above_mu", C.c_uint64), ("violations", C.c_uint64)]


@dataclass
class PPRResult:
    estimates: np.ndarray
    residues: np.ndarray
    r_sum: float
    pushes: int
    iterations: int = 0
    used_scan_phase: bool = False
    epoch_r_max: np.ndarray | None = None
    walks: int = 0


@dataclass
class CSR:
    offsets: np.ndarray  # uint64[n+1]
    neighbors: np.ndarray  # uint32[m]

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def m(self) -> int:
        return int(self.offsets[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)

    def dead_ends(self) -> np.ndarray:
        return np.nonzero(self.degrees() == 0)[0].astype(np.uint32)

    @property
    def m_eff(self) -> int:
        return self.m + int((self.degrees() == 0).sum())


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.og_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.og_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.og_philox_walk.argtypes = [u64p, u32p, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                     C.c_uint32, C.c_uint32, C.c_uint32]
        L.og_philox_walk.restype = C.c_uint32
        L.og_philox_build_index.argtypes = [u64p, u32p, C.c_uint64, C.c_double, C.c_uint64, u32p]
        L.og_build_graph_from_edges.argtypes = [u64p, C.c_uint64, u64p, u32p, C.POINTER(C.c_uint64)]
        L.og_generate_rmat.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                       C.c_uint64, C.c_int, vp, vp, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]
        L.og_random_graph.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, vp, vp,
                                      C.POINTER(C.c_uint64)]
        L.og_push_once.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double, f64p, f64p,
                                   C.POINTER(OgStats), C.c_uint32]
        L.og_power_iteration.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                                         f64p, f64p, C.POINTER(OgStats), vp, C.c_uint32]
        L.og_sim_forward_push.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double,
                                          C.c_double, f64p, f64p, C.POINTER(OgStats)]
        L.og_fifo_forward_push.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double,
                                           C.c_double, C.c_double, f64p, f64p, C.POINTER(OgStats)]
        L.og_power_push.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                                    C.c_uint32, C.c_int64, f64p, f64p, C.POINTER(OgStats), vp]
        L.og_refine.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double, C.c_double, f64p,
                                f64p, C.POINTER(OgStats)]
        L.og_exact_ppr.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double, f64p]
        L.og_compare_to_truth.argtypes = [f64p, f64p, C.c_uint64, C.c_double, C.c_double,
                                          C.POINTER(OgErrorReport)]
        L.og_walk_budget_real.argtypes = [C.c_uint64, C.c_double, C.c_double]
        L.og_walk_budget_real.restype = C.c_double
        L.og_compute_walk_budget.argtypes = [C.c_uint64, C.c_double, C.c_double,
                                             C.POINTER(C.c_uint64)]
        L.og_build_index.argtypes = [u64p, u32p, C.c_uint64, C.c_double, C.c_uint64, u32p]
        L.og_speedppr_query.argtypes = [u64p, u32p, C.c_uint64, C.c_uint32, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, vp, f64p, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64)]

    # ---- rng ----------------------------------------------------------------
    def rng_draws(self, seed, count, bound=0):
        out = np.zeros(count, np.uint64)
        self.L.og_rng_draws(seed, count, bound, out)
        return out

    def philox(self, ctr, key):
        out = np.zeros(4, np.uint32)
        self.L.og_philox4x32_10(np.asarray(ctr, np.uint32), np.asarray(key, np.uint32), out)
        return out

    def philox_walk(self, g: CSR, start, source, alpha, seed, k, v, tag):
        return int(self.L.og_philox_walk(g.offsets, g.neighbors, start, source, alpha, seed, k, v,
                                         tag))

    def philox_build_index(self, g: CSR, alpha, seed):
        out = np.zeros(max(g.m, 1), np.uint32)
        self.L.og_philox_build_index(g.offsets, g.neighbors, g.n, alpha, seed, out)
        return out[: g.m]

    # ---- graphs -------------------------------------------------------------
    def build_graph_from_edges(self, pairs) -> CSR:
        pairs = np.ascontiguousarray(np.asarray(pairs, np.uint64).reshape(-1, 2))
        cnt = len(pairs)
        if cnt == 0:
            raise DataError("graph is empty after cleaning")
        off = np.zeros(2 * cnt + 1, np.uint64)
        nbr = np.zeros(cnt, np.uint32)
        n = C.c_uint64()
        _check(self.L.og_build_graph_from_edges(pairs.reshape(-1), cnt, off, nbr, C.byref(n)))
        return CSR(off[: n.value + 1].copy(), nbr)

    def generate_rmat(self, scale, edge_factor, seed, a=0.57, b=0.19, c=0.19, threads=None) -> CSR:
        """Host restatement of pprg_graph_generate_rmat (bit-exact; see oracle.c)."""
        threads = threads or os.cpu_count() or 1
        off = np.zeros((1 << scale) + 1, np.uint64)
        nbr = np.empty(max(edge_factor << scale, 1), np.uint32)
        n, m = C.c_uint64(), C.c_uint64()
        _check(self.L.og_generate_rmat(scale, edge_factor, a, b, c, seed, threads, off.ctypes.data,
                                       nbr.ctypes.data, C.byref(n), C.byref(m)),
               "rmat generation")
        return CSR(off[: n.value + 1].copy(), nbr[: m.value].copy())

    def random_graph(self, n, min_out, max_out, seed) -> CSR:
        m = C.c_uint64()
        _check(self.L.og_random_graph(n, min_out, max_out, seed, None, None, C.byref(m)))
        off = np.zeros(n + 1, np.uint64)
        nbr = np.zeros(max(m.value, 1), np.uint32)
        _check(self.L.og_random_graph(n, min_out, max_out, seed, off.ctypes.data,
                                      nbr.ctypes.data, C.byref(m)))
        return CSR(off, nbr[: m.value])

    # ---- engines ------------------------------------------------------------
    def _vecs(self, g):
        return np.zeros(g.n, np.float64), np.zeros(g.n, np.float64), OgStats()

    def push_once(self, g, s, alpha, reserve, residue, stats, v):
        self.L.og_push_once(g.offsets, g.neighbors, g.n, s, alpha, reserve, residue,
                            C.byref(stats), v)

    def power_iteration(self, g: CSR, s, alpha, lam, trace_cap=0):
        res, rsd, st = self._vecs(g)
        tr = np.zeros(max(trace_cap, 1), np.float64)
        _check(self.L.og_power_iteration(g.offsets, g.neighbors, g.n, s, alpha, lam, res, rsd,
                                         C.byref(st), tr.ctypes.data if trace_cap else None,
                                         trace_cap))
        out = PPRResult(res, rsd, st.r_sum, st.pushes, st.iterations)
        out.trace = tr[: min(st.iterations, trace_cap)]
        return out

    def sim_forward_push(self, g, s, alpha, lam):
        res, rsd, st = self._vecs(g)
        _check(self.L.og_sim_forward_push(g.offsets, g.neighbors, g.n, s, alpha, lam, res, rsd,
                                          C.byref(st)))
        return PPRResult(res, rsd, st.r_sum, st.pushes, st.iterations)

    def fifo_forward_push(self, g, s, alpha, r_max, lambda_stop=None):
        res, rsd, st = self._vecs(g)
        _check(self.L.og_fifo_forward_push(g.offsets, g.neighbors, g.n, s, alpha, r_max,
                                           lambda_stop if lambda_stop else -1.0, res, rsd,
                                           C.byref(st)))
        return PPRResult(res, rsd, st.r_sum, st.pushes)

    def power_push(self, g, s, alpha, lam, epoch_num=8, scan_threshold=None):
        res, rsd, st = self._vecs(g)
        ep = np.zeros(max(epoch_num, 1), np.float64)
        _check(self.L.og_power_push(g.offsets, g.neighbors, g.n, s, alpha, lam, epoch_num,
                                    -1 if scan_threshold is None else scan_threshold, res, rsd,
                                    C.byref(st), ep.ctypes.data))
        return PPRResult(res, rsd, st.r_sum, st.pushes, st.iterations, bool(st.used_scan_phase),
                         ep[:epoch_num] if st.used_scan_phase else ep[:0])

    def power_push_refine(self, g, s, alpha, lam, r_max):
        r = self.power_push(g, s, alpha, lam)
        st = OgStats(r.r_sum, r.pushes, r.iterations, int(r.used_scan_phase), 0)
        _check(self.L.og_refine(g.offsets, g.neighbors, g.n, s, alpha, r_max, r.estimates,
                                r.residues, C.byref(st)))
        return PPRResult(r.estimates, r.residues, st.r_sum, st.pushes)

    def exact_ppr(self, g, s, alpha):
        pi = np.zeros(g.n, np.float64)
        _check(self.L.og_exact_ppr(g.offsets, g.neighbors, g.n, s, alpha, pi))
        return pi

    def compare_to_truth(self, est, truth, mu, eps):
        rep = OgErrorReport()
        self.L.og_compare_to_truth(np.ascontiguousarray(est, np.float64),
                                   np.ascontiguousarray(truth, np.float64), len(est), mu, eps,
                                   C.byref(rep))
        return rep

    def walk_budget_real(self, n, eps, mu):
        w = self.L.og_walk_budget_real(n, eps, mu)
        if w < 0:
            raise InvalidArgument("walk budget")
        return w

    def compute_walk_budget(self, n, eps, mu):
        out = C.c_uint64()
        _check(self.L.og_compute_walk_budget(n, eps, mu, C.byref(out)), "walk budget")
        return out.value

    def build_index(self, g, alpha, seed):
        out = np.zeros(max(g.m, 1), np.uint32)
        self.L.og_build_index(g.offsets, g.neighbors, g.n, alpha, seed, out)
        return out[: g.m]

    def speedppr_query(self, g, s, alpha, eps, seed, mu=None, index=None):
        est = np.zeros(g.n, np.float64)
        walks, pushes = C.c_uint64(), C.c_uint64()
        idx = None if index is None else np.ascontiguousarray(index, np.uint32)
        _check(self.L.og_speedppr_query(g.offsets, g.neighbors, g.n, s, alpha, eps,
                                        -1.0 if mu is None else mu, seed,
                                        None if idx is None else idx.ctypes.data, est,
                                        C.byref(walks), C.byref(pushes)))
        return PPRResult(est, np.zeros(g.n), 0.0, pushes.value, walks=walks.value)


class Ref:
    """The reference library itself (compiled unchanged), for pinning."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_graph_from_edges.argtypes = [u64p, C.c_uint64, C.POINTER(vp)]
        L.ref_graph_from_csr.argtypes = [u64p, u32p, C.c_uint64, C.POINTER(vp)]
        L.ref_random_graph.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.POINTER(vp)]
        L.ref_load_graph_cache.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_save_graph_cache.argtypes = [vp, C.c_char_p]
        L.ref_load_edge_list.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        L.ref_graph_free.argtypes = [vp]
        for f in ("ref_graph_n", "ref_graph_m", "ref_graph_dead_end_count"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = C.c_uint64
        L.ref_graph_export.argtypes = [vp, vp, vp, vp]
        L.ref_power_iteration.argtypes = [vp, C.c_uint32, C.c_double, C.c_double, f64p, f64p,
                                          C.POINTER(C.c_double), C.POINTER(C.c_uint64), vp,
                                          C.c_uint32, C.POINTER(C.c_uint32)]
        L.ref_sim_forward_push.argtypes = [vp, C.c_uint32, C.c_double, C.c_double, f64p, f64p,
                                           C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        L.ref_fifo_forward_push.argtypes = [vp, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                            f64p, f64p, C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint64)]
        L.ref_power_push.argtypes = [vp, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                                     C.c_int64, f64p, f64p, C.POINTER(C.c_double),
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_int), vp]
        L.ref_power_push_refine.argtypes = [vp, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                            f64p, f64p, C.POINTER(C.c_double),
                                            C.POINTER(C.c_uint64)]
        L.ref_power_push_batch.argtypes = [vp, u32p, C.c_uint32, C.c_double, C.c_double,
                                           C.c_uint32, vp, vp, vp, C.c_int]
        L.ref_walk_budget_real.argtypes = [C.c_uint64, C.c_double, C.c_double]
        L.ref_walk_budget_real.restype = C.c_double
        L.ref_compute_walk_budget.argtypes = [C.c_uint64, C.c_double, C.c_double,
                                              C.POINTER(C.c_uint64)]
        L.ref_build_index.argtypes = [vp, C.c_double, C.c_uint64, C.POINTER(vp)]
        L.ref_index_free.argtypes = [vp]
        L.ref_index_export.argtypes = [vp, u32p]
        L.ref_index_from_arrays.argtypes = [C.c_double, C.c_uint64, C.c_uint8, u64p, C.c_uint64,
                                            u32p, C.POINTER(vp)]
        L.ref_save_index.argtypes = [vp, C.c_char_p]
        L.ref_load_index.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.ref_speedppr_query.argtypes = [vp, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                         C.c_uint64, vp, f64p, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.ref_speedppr_batch.argtypes = [vp, u32p, C.c_uint32, C.c_double, C.c_double, C.c_uint64,
                                         vp, C.c_uint32]
        L.ref_exact_ppr.argtypes = [vp, C.c_uint32, C.c_double, f64p]
        L.ref_ground_truth.argtypes = [vp, C.c_uint32, C.c_double, f64p]
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]

    def _chk(self, rc):
        if rc:
            raise _ERR.get(rc, OracleError)(self.L.ref_last_error().decode())

    # graphs are held as RefGraph handles
    def graph(self, g: CSR) -> "RefGraph":
        h = vp()
        self._chk(self.L.ref_graph_from_csr(g.offsets, g.neighbors, g.n, C.byref(h)))
        return RefGraph(self, h)

    def graph_from_edges(self, pairs) -> "RefGraph":
        pairs = np.ascontiguousarray(np.asarray(pairs, np.uint64).reshape(-1))
        h = vp()
        self._chk(self.L.ref_graph_from_edges(pairs, len(pairs) // 2, C.byref(h)))
        return RefGraph(self, h)

    def random_graph(self, n, min_out, max_out, seed) -> "RefGraph":
        h = vp()
        self._chk(self.L.ref_random_graph(n, min_out, max_out, seed, C.byref(h)))
        return RefGraph(self, h)

    def load_graph_cache(self, path) -> "RefGraph":
        h = vp()
        self._chk(self.L.ref_load_graph_cache(path.encode(), C.byref(h)))
        return RefGraph(self, h)

    def rng_draws(self, seed, count, bound=0):
        out = np.zeros(count, np.uint64)
        self.L.ref_rng_draws(seed, count, bound, out)
        return out

    def compute_walk_budget(self, n, eps, mu):
        out = C.c_uint64()
        self._chk(self.L.ref_compute_walk_budget(n, eps, mu, C.byref(out)))
        return out.value


class RefGraph:
    def __init__(self, ref: Ref, h):
        self.ref, self.h, self.L = ref, h, ref.L

    def __del__(self):
        try:
            self.L.ref_graph_free(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return int(self.L.ref_graph_n(self.h))

    @property
    def m(self):
        return int(self.L.ref_graph_m(self.h))

    def csr(self) -> CSR:
        off = np.zeros(self.n + 1, np.uint64)
        nbr = np.zeros(max(self.m, 1), np.uint32)
        self.L.ref_graph_export(self.h, off.ctypes.data, nbr.ctypes.data, None)
        return CSR(off, nbr[: self.m])

    def dead_ends(self):
        c = int(self.L.ref_graph_dead_end_count(self.h))
        out = np.zeros(max(c, 1), np.uint32)
        self.L.ref_graph_export(self.h, None, None, out.ctypes.data)
        return out[:c]

    def save(self, path):
        self.ref._chk(self.L.ref_save_graph_cache(self.h, path.encode()))

    def _out(self):
        n = self.n
        return np.zeros(n), np.zeros(n), C.c_double(), C.c_uint64()

    def power_iteration(self, s, alpha, lam, trace_cap=0):
        res, rsd, rs, pu = self._out()
        tr = np.zeros(max(trace_cap, 1))
        it = C.c_uint32()
        self.ref._chk(self.L.ref_power_iteration(self.h, s, alpha, lam, res, rsd, C.byref(rs),
                                                 C.byref(pu), tr.ctypes.data, trace_cap,
                                                 C.byref(it)))
        out = PPRResult(res, rsd, rs.value, pu.value, it.value)
        out.trace = tr[: min(it.value, trace_cap)]
        return out

    def sim_forward_push(self, s, alpha, lam):
        res, rsd, rs, pu = self._out()
        self.ref._chk(self.L.ref_sim_forward_push(self.h, s, alpha, lam, res, rsd, C.byref(rs),
                                                  C.byref(pu)))
        return PPRResult(res, rsd, rs.value, pu.value)

    def fifo_forward_push(self, s, alpha, r_max, lambda_stop=None):
        res, rsd, rs, pu = self._out()
        self.ref._chk(self.L.ref_fifo_forward_push(self.h, s, alpha, r_max,
                                                   lambda_stop if lambda_stop else -1.0, res, rsd,
                                                   C.byref(rs), C.byref(pu)))
        return PPRResult(res, rsd, rs.value, pu.value)

    def power_push(self, s, alpha, lam, epoch_num=8, scan_threshold=None):
        res, rsd, rs, pu = self._out()
        used = C.c_int()
        ep = np.zeros(max(epoch_num, 1))
        self.ref._chk(self.L.ref_power_push(self.h, s, alpha, lam, epoch_num,
                                            -1 if scan_threshold is None else scan_threshold, res,
                                            rsd, C.byref(rs), C.byref(pu), C.byref(used),
                                            ep.ctypes.data))
        return PPRResult(res, rsd, rs.value, pu.value, 0, bool(used.value),
                         ep[:epoch_num] if used.value else ep[:0])

    def power_push_refine(self, s, alpha, lam, r_max):
        res, rsd, rs, pu = self._out()
        self.ref._chk(self.L.ref_power_push_refine(self.h, s, alpha, lam, r_max, res, rsd,
                                                   C.byref(rs), C.byref(pu)))
        return PPRResult(res, rsd, rs.value, pu.value)

    def power_push_batch(self, sources, alpha, lam, threads, keep=False, powitr=False):
        src = np.ascontiguousarray(sources, np.uint32)
        k, n = len(src), self.n
        res = np.zeros((k, n)) if keep else None
        rsd = np.zeros((k, n)) if keep else None
        rs = np.zeros(k)
        self.ref._chk(self.L.ref_power_push_batch(
            self.h, src, k, alpha, lam, threads, None if res is None else res.ctypes.data,
            None if rsd is None else rsd.ctypes.data, rs.ctypes.data, int(powitr)))
        return res, rsd, rs

    def exact_ppr(self, s, alpha):
        pi = np.zeros(self.n)
        self.ref._chk(self.L.ref_exact_ppr(self.h, s, alpha, pi))
        return pi

    def ground_truth(self, s, alpha):
        pi = np.zeros(self.n)
        self.ref._chk(self.L.ref_ground_truth(self.h, s, alpha, pi))
        return pi

    def build_index(self, alpha, seed):
        h = vp()
        self.ref._chk(self.L.ref_build_index(self.h, alpha, seed, C.byref(h)))
        out = np.zeros(max(self.m, 1), np.uint32)
        self.L.ref_index_export(h, out)
        self.L.ref_index_free(h)
        return out[: self.m]

    def speedppr_query(self, s, alpha, eps, seed, mu=None, index=None, rng_id=1, index_seed=0):
        est = np.zeros(self.n)
        walks, pushes = C.c_uint64(), C.c_uint64()
        ih = None
        if index is not None:
            ih = vp()
            off = self.csr().offsets
            self.ref._chk(self.L.ref_index_from_arrays(alpha, index_seed, rng_id, off, self.n,
                                                       np.ascontiguousarray(index, np.uint32),
                                                       C.byref(ih)))
        try:
            self.ref._chk(self.L.ref_speedppr_query(self.h, s, alpha, eps,
                                                    -1.0 if mu is None else mu, seed, ih, est,
                                                    C.byref(walks), C.byref(pushes)))
        finally:
            if ih is not None:
                self.L.ref_index_free(ih)
        return PPRResult(est, np.zeros(self.n), 0.0, pushes.value, walks=walks.value)

    def speedppr_batch(self, sources, alpha, eps, seed, threads, index=None, index_seed=0):
        ih = None
        if index is not None:
            ih = vp()
            self.ref._chk(self.L.ref_index_from_arrays(alpha, index_seed, 1, self.csr().offsets,
                                                       self.n, np.ascontiguousarray(index, np.uint32),
                                                       C.byref(ih)))
        try:
            src = np.ascontiguousarray(sources, np.uint32)
            self.ref._chk(self.L.ref_speedppr_batch(self.h, src, len(src), alpha, eps, seed, ih,
                                                    threads))
        finally:
            if ih is not None:
                self.L.ref_index_free(ih)


def five_node_edges():
    """testutil.hpp:18-24, the paper's Figure-1 running example."""
    return [(0, 1), (0, 2), (1, 0), (1, 2), (1, 3), (1, 4), (2, 1), (2, 3), (3, 0), (3, 1),
            (3, 2), (4, 1), (4, 2)]


FIVE_NODE_PI0 = np.array([0.29366106080206994, 0.27166882276843485, 0.23285899094437276,
                          0.1474773609314361, 0.054333764553686985])  # testutil.hpp:28-33
