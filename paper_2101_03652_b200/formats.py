"""On-disk formats shared with the reference, little-endian, bit-exact.

PPRG graph cache (graph.hpp:102-106, graph.cpp:115-149):
    magic "PPRG", version u8 = 1, n u64, m u64, offsets (n+1) x u64, neighbors m x u32
PPRW walk index (walk_index.hpp:52-56, walk_index.cpp:57-104):
    magic "PPRW", version u8 = 1, rng-id u8, alpha f64, seed u64, n u64, m u64,
    offsets (n+1) x u64, endpoints m x u32
Our index files carry rng-id 2 (Philox4x32-10); the reference loader accepts
only 1 (walk_index.cpp:91-93) by design.
"""
from __future__ import annotations

import numpy as np

from ._abi import DataError, Graph, RNG_ID_PHILOX, WalkIndex

_G_MAGIC, _W_MAGIC, _VERSION = b"PPRG", b"PPRW", 1


def save_graph_cache(g: Graph, path: str) -> None:
    """graph.cpp:115-125, written from device memory (pprg_graph_save_cache)."""
    from ._abi import _check, load_library
    _check(load_library().pprg_graph_save_cache(g.handle, path.encode()))


def write_graph_cache(path: str, offsets, neighbors) -> None:
    """The same PPRG bytes from host arrays (tests, tools)."""
    with open(path, "wb") as f:
        f.write(_G_MAGIC)
        f.write(bytes([_VERSION]))
        f.write(np.array([len(offsets) - 1, len(neighbors)], "<u8").tobytes())
        f.write(np.asarray(offsets).astype("<u8").tobytes())
        f.write(np.asarray(neighbors).astype("<u4").tobytes())


def is_graph_cache(path: str) -> bool:
    try:
        with open(path, "rb") as f:
            return f.read(4) == _G_MAGIC
    except OSError:
        return False


def read_graph_cache(path: str):
    """(offsets, neighbors) host arrays of a PPRG file, with the reference's checks."""
    try:
        f = open(path, "rb")
    except OSError:
        raise DataError(f"cannot open graph cache: {path}")
    with f:
        if f.read(4) != _G_MAGIC:
            raise DataError(f"{path}: not a graph cache (bad magic)")
        v = f.read(1)
        if len(v) != 1 or v[0] != _VERSION:
            raise DataError(f"{path}: unsupported graph cache version")
        hdr = f.read(16)
        if len(hdr) != 16:
            raise DataError(f"{path}: truncated graph cache")
        n, m = (int(x) for x in np.frombuffer(hdr, "<u8"))
        off = np.frombuffer(f.read(8 * (n + 1)), "<u8")
        nbr = np.frombuffer(f.read(4 * m), "<u4")
        if off.size != n + 1 or nbr.size != m:
            raise DataError(f"{path}: truncated graph cache")
    return off.astype(np.uint64), nbr.astype(np.uint32)


def load_graph_cache(path: str, device=None) -> Graph:
    """graph.cpp:127-143, streamed straight into device memory (pprg_graph_load_cache)."""
    import ctypes as C
    from ._abi import _check, _default_device, load_library
    dev = _default_device() if device is None else device
    h = C.c_void_p()
    _check(load_library().pprg_graph_load_cache(path.encode(), dev, C.byref(h)))
    return Graph(device=dev, _handle=h)


def load_graph_cache_host(path: str, device=None) -> Graph:
    off, nbr = read_graph_cache(path)
    return Graph(off, nbr, device=device)


def save_index(index: WalkIndex, path: str) -> None:
    """walk_index.cpp:61-81 from device memory (pprg_index_save)."""
    from ._abi import _check, load_library
    _check(load_library().pprg_index_save(index._h, path.encode()))


def write_index_host(index: WalkIndex, path: str) -> None:
    g = index.graph
    with open(path, "wb") as f:
        f.write(_W_MAGIC)
        f.write(bytes([_VERSION, index.rng_id()]))
        f.write(np.array([index.alpha()], "<f8").tobytes())
        f.write(np.array([index.seed(), g.n(), g.m()], "<u8").tobytes())
        f.write(g.out_offsets().astype("<u8").tobytes())
        f.write(index.endpoints().astype("<u4").tobytes())


def read_index(path: str):
    try:
        f = open(path, "rb")
    except OSError:
        raise DataError(f"cannot open walk index: {path}")
    with f:
        if f.read(4) != _W_MAGIC:
            raise DataError(f"{path}: not a walk index (bad magic)")
        b = f.read(2)
        if len(b) != 2 or b[0] != _VERSION:
            raise DataError(f"{path}: unsupported walk index version")
        if b[1] != RNG_ID_PHILOX:
            raise DataError(f"{path}: unknown generator id")
        hdr = f.read(32)
        if len(hdr) != 32:
            raise DataError(f"{path}: truncated walk index")
        alpha = float(np.frombuffer(hdr[:8], "<f8")[0])
        seed, n, m = (int(x) for x in np.frombuffer(hdr[8:], "<u8"))
        off = np.frombuffer(f.read(8 * (n + 1)), "<u8")
        ep = np.frombuffer(f.read(4 * m), "<u4")
        if off.size != n + 1 or ep.size != m:
            raise DataError(f"{path}: truncated walk index")
    return alpha, seed, off.astype(np.uint64), ep.astype(np.uint32)


def load_index(path: str, g: Graph) -> WalkIndex:
    """walk_index.cpp:83-104 + check_compatible, streamed into device memory."""
    import ctypes as C
    from ._abi import _check, load_library
    L = load_library()
    h = C.c_void_p()
    _check(L.pprg_index_load(g.handle, path.encode(), C.byref(h)))
    alpha, seed = _index_header(path)
    return WalkIndex(g, alpha, seed, h)


def _index_header(path: str):
    with open(path, "rb") as f:
        hdr = f.read(22)
    return float(np.frombuffer(hdr[6:14], "<f8")[0]), int(np.frombuffer(hdr[14:22], "<u8")[0])


def load_index_host(path: str, g: Graph) -> WalkIndex:
    alpha, seed, off, ep = read_index(path)
    if off.size != g.n() + 1 or ep.size != g.m() or not np.array_equal(off, g.out_offsets()):
        raise DataError("walk index does not match the graph shape")
    return WalkIndex.from_endpoints(g, alpha, seed, ep)


# ---- edge-list text files (graph.cpp:66-101) --------------------------------------
def parse_edge_list(path: str, undirected: bool = False) -> np.ndarray:
    """Pairs (src, dst) as uint64 [count, 2], with the reference's rules and
    messages: blank lines and '#' comments skipped, two non-negative integers
    per line separated by spaces/tabs, nothing after them; `undirected` adds
    the reverse of every pair right after it."""
    try:
        f = open(path, "rb")
    except OSError:
        raise DataError("cannot open graph file: " + path)
    out = []
    with f:
        for line_no, raw in enumerate(f, 1):
            line = raw.rstrip(b"\n")
            p, end = 0, len(line)

            def fail(what):
                raise DataError(f"{path}:{line_no}: {what}")

            while p < end and line[p] in b" \t\r":
                p += 1
            if p == end or line[p:p + 1] == b"#":
                continue
            vals = []
            for what in ("expected non-negative integer source id",
                         "expected non-negative integer target id"):
                q = p
                while q < end and 48 <= line[q] <= 57:
                    q += 1
                if q == p:
                    fail(what)
                v = int(line[p:q])
                if v >= 1 << 64:
                    fail(what)
                vals.append(v)
                p = q
                while p < end and line[p] in b" \t\r":
                    p += 1
            if p != end:
                fail("trailing content after edge pair")
            out.append(vals)
            if undirected:
                out.append(vals[::-1])
    if not out:
        raise DataError(path + ": graph is empty after cleaning")
    return np.asarray(out, dtype=np.uint64)


def load_edge_list(path: str, device=None) -> Graph:  # graph.hpp:97
    from ._abi import build_graph_from_edges
    return build_graph_from_edges(parse_edge_list(path), device=device)


def undirected_to_directed(path: str, device=None) -> Graph:  # graph.hpp:100
    from ._abi import build_graph_from_edges
    return build_graph_from_edges(parse_edge_list(path, undirected=True), device=device)
