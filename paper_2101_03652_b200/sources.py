"""Query-source sampling for the benchmark configs.

The reference samples uniformly over [0, n) with its mt19937_64 Rng
(sweep.cpp:141-146, rng.hpp:14-39). The BASELINE configs require
out-degree > 0, so draws landing on a dead-end are rejected (with
replacement otherwise, as the reference). mt19937_64 and Lemire's bounded
draw are restated here so source lists are identical to Rng(seed).below(n).
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


class Mt19937_64:
    def __init__(self, seed: int):
        mt = [0] * 312
        mt[0] = seed & _MASK
        for i in range(1, 312):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self.mt, self.i = mt, 312

    def next(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _MASK

    def below(self, bound: int) -> int:  # rng.hpp:24-35
        product = self.next() * bound
        low = product & _MASK
        if low < bound:
            threshold = (-bound % (1 << 64)) % bound
            while low < threshold:
                product = self.next() * bound
                low = product & _MASK
        return product >> 64


def sample_sources(out_degree: np.ndarray, count: int, seed: int) -> np.ndarray:
    """`count` sources from Rng(seed).below(n), rejecting dead-ends."""
    n = len(out_degree)
    if not np.any(out_degree > 0):
        raise ValueError("graph has no node with out-degree > 0")
    rng = Mt19937_64(seed)
    out = []
    while len(out) < count:
        v = rng.below(n)
        if out_degree[v] > 0:
            out.append(v)
    return np.asarray(out, dtype=np.uint32)
