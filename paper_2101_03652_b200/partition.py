"""Vertex-partitioned PowerPush over torch.distributed (BASELINE configs[4],
SURVEY 8(e)): one process per GPU, each holding the graph and owning a
contiguous range of pull-sweep rows (cut at row-aligned tiles so every part
holds ~m/P in-edges). The engine's per-part primitives are the C-ABI
pprg_part_* sessions (include/pprg.h); this module is the exchange between
them, over NCCL on GPUs (or gloo for the CPU protocol tests):

    begin  -> broadcast part 0's local-phase x, resum
           -> all_reduce(sum x, sum dead-end x)   -> start (identical epoch state)
    sweep loop:  broadcast every part's y row slice (all-gather-v of y)
                 -> sweep own rows -> all_reduce(sweep counters) -> advance
    finish -> all_reduce(residue sums) = exact r_sum per source

The epoch decisions (push.cpp:168-197) use only all-reduced values, so every
rank advances identically; remote y is at most one sweep stale, which only
under-estimates inflow, and r_sum = 1 - alpha * sum(x) is exact regardless,
so the results obey the reference's lambda bounds.

`run_partitioned(part)` is the protocol for any object with the part
interface (`GpuPart` here; the CPU tests drive a numpy part through the same
function and the library's host epoch rule). `run_virtual_parts` runs P parts
one after another on one GPU, copying the slices itself (no collectives, no
part waits on another) — the single-GPU check of the partitioned kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _abi
from ._abi import CStats, CallStats, QStats, _check, load_library

KMAX = 64


class _DeviceArray:
    """Zero-copy view of an engine device buffer for torch.as_tensor."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3}


def _device_view(ptr: int, count: int, device: int):
    import torch
    return torch.as_tensor(_DeviceArray(ptr, count), device=f"cuda:{device}")


def _bind(L):
    if getattr(L, "_part_bound", False):
        return
    vp, f64p = C.c_void_p, C.POINTER(C.c_double)
    L.pprg_part_begin.argtypes = [vp, C.c_uint32, C.c_uint32, vp, C.c_uint32, C.c_double,
                                  C.c_double, C.c_uint32, C.c_int64, vp, C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint64), C.POINTER(vp)]
    L.pprg_part_start.argtypes = [vp, vp, C.POINTER(C.c_int)]
    L.pprg_part_buffers.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_uint32), C.POINTER(vp)]
    L.pprg_part_sweep.argtypes = [vp, vp]
    L.pprg_part_local_x.argtypes = [vp, C.POINTER(vp)]
    L.pprg_part_resum.argtypes = [vp, vp]
    L.pprg_part_advance.argtypes = [vp, vp, C.POINTER(C.c_int)]
    L.pprg_part_finish.argtypes = [vp, vp, vp, C.c_uint32, vp]
    L.pprg_part_stats.argtypes = [vp, vp, vp]
    L.pprg_part_destroy.argtypes = [vp]
    L.pprg_part_destroy.restype = None
    L.pprg_part_set_peers.argtypes = [vp, vp, C.c_uint32]
    L.pprg_part_ipc_handle.argtypes = [vp, vp]
    L.pprg_ipc_open.argtypes = [C.c_int, vp, C.POINTER(vp)]
    L.pprg_ipc_close.argtypes = [C.c_int, vp]
    L.pprg_epoch_init.argtypes = [vp, C.c_uint32, vp, vp, vp, C.c_uint32, C.c_double,
                                  C.POINTER(C.c_int)]
    L.pprg_epoch_advance.argtypes = [vp, C.c_uint32, vp, vp, C.c_uint32, C.c_double,
                                     C.POINTER(C.c_int)]
    L._part_bound = True


def _lib():
    L = load_library()
    _bind(L)
    return L


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


class ColumnState(C.Structure):
    """pprg_column_state (include/pprg.h)."""
    _fields_ = [("r_sum", C.c_double), ("D", C.c_double), ("epoch", C.c_int32),
                ("done", C.c_int32), ("sweeps", C.c_uint32), ("pushes", C.c_uint64)]


def epoch_lambdas(lam: float, epoch_num: int) -> np.ndarray:
    """lambda^(i/epoch_num), i = 1..epoch_num (push.cpp:176-178)."""
    return np.array([lam ** ((e + 1) / epoch_num) for e in range(epoch_num)], np.float64)


class EpochRule:
    """The library's host epoch rule (pprg_epoch_init / pprg_epoch_advance)
    over per-column state; used by parts that keep their state in Python."""

    def __init__(self, columns: int, lam: float, epoch_num: int, alpha: float):
        self.columns, self.E, self.alpha = columns, epoch_num, alpha
        self.lam = epoch_lambdas(lam, epoch_num)
        self.cols = (ColumnState * columns)()

    def init(self, sum_x: np.ndarray, sum_dead_x: np.ndarray) -> bool:
        need = C.c_int()
        sx = np.ascontiguousarray(sum_x[:self.columns], np.float64)
        sd = np.ascontiguousarray(sum_dead_x[:self.columns], np.float64)
        _check(_lib().pprg_epoch_init(C.addressof(self.cols), self.columns, _p(sx), _p(sd),
                                      _p(self.lam), self.E, self.alpha, C.byref(need)))
        return bool(need.value)

    def advance(self, summed: np.ndarray) -> bool:
        done = C.c_int()
        s = np.ascontiguousarray(summed[:5 * self.columns], np.float64)
        _check(_lib().pprg_epoch_advance(C.addressof(self.cols), self.columns, _p(s), _p(self.lam),
                                         self.E, self.alpha, C.byref(done)))
        return bool(done.value)

    def state(self, c: int) -> ColumnState:
        return self.cols[c]


class GpuPart:
    """One vertex part of a k-source power_push on this process's GPU
    (pprg_part_* session over a resident Graph)."""

    def __init__(self, g: _abi.Graph, nparts: int, part: int, sources: Sequence[int], alpha: float,
                 lam: float, epoch_num: int = 8, scan_threshold: Optional[int] = None):
        self.g, self.nparts, self.part = g, nparts, part
        self.src = np.ascontiguousarray(sources, np.uint32)
        self.k = len(self.src)
        self.alpha, self.lam, self.E = alpha, lam, epoch_num
        self.scan_threshold = -1 if scan_threshold is None else scan_threshold
        self.h = None
        self.n = g.n()

    # -- the part interface ---------------------------------------------------
    def begin(self) -> np.ndarray:
        L = _lib()
        partial = np.zeros(2 * KMAX, np.float64)
        lo, hi, h = C.c_uint64(), C.c_uint64(), C.c_void_p()
        _check(L.pprg_part_begin(self.g.handle, self.nparts, self.part, _p(self.src), self.k,
                                 self.alpha, self.lam, self.E, self.scan_threshold, _p(partial),
                                 C.byref(lo), C.byref(hi), C.byref(h)))
        self.h, self.lo, self.hi = h, lo.value, hi.value
        y, cols, cnt = C.c_void_p(), C.c_uint32(), C.c_void_p()
        _check(L.pprg_part_buffers(self.h, C.byref(y), C.byref(cols), C.byref(cnt)))
        self.columns, self._y, self._cnt = cols.value, y.value, cnt.value
        return partial

    def x_view(self):
        """This part's local-phase state x [n * columns] (device)."""
        x = C.c_void_p()
        _check(_lib().pprg_part_local_x(self.h, C.byref(x)))
        return _device_view(x.value, self.n * self.columns, self.g.device)

    def resum(self) -> np.ndarray:
        """Partial sums of this part after x was overwritten (adopted local phase)."""
        partial = np.zeros(2 * KMAX, np.float64)
        _check(_lib().pprg_part_resum(self.h, _p(partial)))
        return partial

    def start(self, summed: np.ndarray) -> bool:
        need = C.c_int()
        s = np.ascontiguousarray(summed, np.float64)
        _check(_lib().pprg_part_start(self.h, _p(s), C.byref(need)))
        return bool(need.value)

    def set_peers(self, ptrs: Sequence[int]):
        """Fused exchange: this part's sweeps store pushed y rows into these
        device buffers (other parts' y) instead of a per-sweep all-gather."""
        arr = (C.c_void_p * max(len(ptrs), 1))(*ptrs)
        _check(_lib().pprg_part_set_peers(self.h, arr, len(ptrs)))
        self.fused = len(ptrs) > 0

    def y_ptr(self) -> int:
        return self._y

    def ipc_handle(self) -> bytes:
        buf = (C.c_ubyte * 64)()
        _check(_lib().pprg_part_ipc_handle(self.h, buf))
        return bytes(buf)

    def y_view(self):
        return _device_view(self._y, self.n * self.columns, self.g.device)

    def counters_view(self):
        return _device_view(self._cnt, 5 * self.columns, self.g.device)

    def sweep(self, local: Optional[np.ndarray] = None):
        _check(_lib().pprg_part_sweep(self.h, None if local is None else _p(local)))

    def advance(self, summed: np.ndarray) -> bool:
        done = C.c_int()
        s = np.ascontiguousarray(summed, np.float64)
        _check(_lib().pprg_part_advance(self.h, _p(s), C.byref(done)))
        return bool(done.value)

    def finish(self, reserve_ptr=None, residue_ptr=None, on_device=False) -> np.ndarray:
        rs = np.zeros(KMAX, np.float64)
        _check(_lib().pprg_part_finish(self.h, reserve_ptr, residue_ptr,
                                       _abi.OUT_DEVICE if on_device else 0, _p(rs)))
        return rs[:self.k]

    def stats(self) -> Tuple[list, CallStats]:
        q = (QStats * self.k)()
        c = CStats()
        _check(_lib().pprg_part_stats(self.h, q, C.byref(c)))
        return list(q), CallStats.of(c)

    def close(self):
        if self.h:
            _lib().pprg_part_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PartitionResult:
    r_sum: np.ndarray           # exact final r_sum per source (all parts)
    sweeps: int
    node_range: Tuple[int, int]  # this rank's rows
    bounds: List[Tuple[int, int]]
    local_stats: object = None


def _open_peer_buffers(part, group, dev):
    """IPC-map every other rank's y buffer on this GPU (fused exchange)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = torch.tensor(list(part.ipc_handle()), dtype=torch.uint8, device=dev)
    allh = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allh, mine, group=group)
    L = _lib()
    ptrs = []
    for r in range(world):
        if r == rank:
            continue
        h = bytes(allh[r].cpu().numpy().tolist())
        p = C.c_void_p()
        _check(L.pprg_ipc_open(part.g.device, h, C.byref(p)))
        ptrs.append(p.value)
    return ptrs


def ranks_of(group, world):
    import torch.distributed as dist
    return [dist.get_global_rank(group, p) if group is not None else p for p in range(world)]


def run_partitioned(part, group=None, comm_device=None, finish_kwargs=None,
                    fused: bool = False) -> PartitionResult:
    """Drive one part through the exchange protocol with torch.distributed.
    `part` exposes begin/start/y_view/counters_view/sweep/advance/finish and
    lo/hi/columns; tensors live on `comm_device` (cuda for NCCL, cpu for gloo).
    fused=True (GPU parts, one GPU per rank): the sweeps store pushed y rows
    straight into the peers' IPC-mapped y buffers, and the per-sweep y
    all-gather is skipped."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = torch.device(comm_device) if comm_device is not None else torch.device("cpu")
    on_gpu = dev.type == "cuda"

    def allreduce_np(a: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64)).to(dev)
        dist.all_reduce(t, group=group)
        return t.cpu().numpy()

    partial = part.begin()
    if world > 1:
        # one local phase for all parts: rank 0's x (the level-synchronous
        # queue phase need not stop in the same state on every rank)
        x = part.x_view()
        if on_gpu:
            dist.broadcast(x, src=ranks_of(group, world)[0], group=group)
        else:
            xc = x.cpu()
            dist.broadcast(xc, src=ranks_of(group, world)[0], group=group)
            x.copy_(xc)
        partial = part.resum()
    peers = _open_peer_buffers(part, group, dev) if fused else []
    if fused:
        part.set_peers(peers)
    need = part.start(allreduce_np(partial))
    mine = torch.tensor([part.lo, part.hi], dtype=torch.int64, device=dev)
    allb = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allb, mine, group=group)
    bounds = [(int(b[0]), int(b[1])) for b in allb]
    ranks = ranks_of(group, world)
    Cw = part.columns
    y = part.y_view()

    def exchange():  # all-gather-v of the y row slices; the final pass needs it too
        if fused or world == 1:
            return
        for p, (lo, hi) in enumerate(bounds):
            if hi > lo:
                dist.broadcast(y[lo * Cw:hi * Cw], src=ranks[p], group=group)
        if on_gpu:
            torch.cuda.current_stream(dev).synchronize()

    exchange()
    sweeps = 0
    while need:
        part.sweep()
        cnt = part.counters_view()
        if not on_gpu and cnt.is_cuda:  # gloo: reduce a host copy
            cnt = cnt.cpu()
        dist.all_reduce(cnt, group=group)
        need = not part.advance(cnt.cpu().numpy())
        exchange()
        sweeps += 1
    rs = allreduce_np(part.finish(**(finish_kwargs or {})))
    if fused:
        dist.barrier(group=group)  # every rank's final pass has read the peers' y
        for p in peers:
            _check(_lib().pprg_ipc_close(part.g.device, p))
    return PartitionResult(rs, sweeps, (part.lo, part.hi), bounds)


def run_virtual_parts(g: _abi.Graph, nparts: int, sources: Sequence[int], alpha: float, lam: float,
                      epoch_num: int = 8, scan_threshold: Optional[int] = None,
                      fused: bool = False):
    """P parts of one query block on ONE GPU, run one after another each sweep;
    the exchange is device copies between the parts' y buffers (or, fused,
    each part's sweep storing its pushed rows into the others' buffers) and
    host sums of their counters. Returns (reserve [k, n], residue [k, n],
    r_sum [k], sweeps, parts). No part ever waits on another."""
    import torch
    parts = [GpuPart(g, nparts, p, sources, alpha, lam, epoch_num, scan_threshold)
             for p in range(nparts)]
    for p in parts:
        p.begin()
    x0 = parts[0].x_view()
    for p in parts[1:]:  # one local phase for all parts (see run_partitioned)
        p.x_view().copy_(x0)
    partial = sum(p.resum() for p in parts)
    if fused:
        for p in parts:
            p.set_peers([q.y_ptr() for q in parts if q is not p])
    need = [p.start(partial) for p in parts]
    assert len(set(need)) == 1
    need = need[0]
    Cw = parts[0].columns
    ys = [p.y_view() for p in parts]

    def exchange():
        if fused:
            torch.cuda.synchronize(g.device)
            return
        for src in parts:
            if src.hi > src.lo:
                sl = slice(src.lo * Cw, src.hi * Cw)
                for dst, yd in zip(parts, ys):
                    if dst is not src:
                        yd[sl].copy_(ys[src.part][sl])
        torch.cuda.synchronize(g.device)

    exchange()
    sweeps = 0
    while need:
        for p in parts:
            p.sweep()
        summed = sum(p.counters_view().cpu().numpy() for p in parts)
        done = [p.advance(summed) for p in parts]
        assert len(set(done)) == 1
        need = not done[0]
        exchange()
        sweeps += 1
    k, n = len(sources), g.n()
    reserve = np.zeros((k, n))
    residue = np.zeros((k, n))
    rs = np.zeros(k)
    for p in parts:
        rs += p.finish(reserve.ctypes.data, residue.ctypes.data, False)
    return reserve, residue, rs, sweeps, parts
