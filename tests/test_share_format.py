"""The 16-bit share format of the delta sweeps (csrc/delta_sweep.cuh:
share_field / share_value / value_b / add_shares), restated in numpy integer
arithmetic: the contract the kernel's exactness rests on. A row that wants to
give each out-neighbour the raw share q publishes a field whose decoded value
never exceeds q (so the mass it deducts, value * deg / (1 - alpha), never
exceeds its residue), an odd column's value includes its even neighbour's bits
exactly as every reader will decode them, and the rounding loss is bounded."""
import numpy as np

EXP = 769  # value = raw * 2^769 (DS_EXP)


def hi_word(q):
    return (np.asarray(q, np.float64).view(np.uint64) >> np.uint64(32)).astype(np.uint64)


def share_field(q, odd):
    """e8m8 field of the wanted raw share q, rounded down (one more step for odd
    columns); 0 = below the format."""
    h = hi_word(q) >> np.uint64(12)
    h = np.minimum(h, np.uint64(0xFFFF))
    if odd:
        return np.where(h >= 257, h - np.uint64(1), np.uint64(0))
    return np.where(h >= 256, h, np.uint64(0))


def value_a(w):
    """even column: fp64 bits (w << 16 truncated to 32 bits) * 2^28"""
    lo16 = (w.astype(np.uint64) << np.uint64(16)) & np.uint64(0xFFFFFFFF)
    return (lo16 * np.uint64(1 << 28)).view(np.float64)


def value_b(w):
    """odd column: fp64 bits w * 2^28 (carries the even column's field below its mantissa)"""
    return (w.astype(np.uint64) * np.uint64(1 << 28)).view(np.float64)


def clean(h):
    return (h.astype(np.uint64) << np.uint64(44)).view(np.float64)


def raw_shares(rng, n):
    # raw shares: true shares in [1e-40, 2) scaled by 2^-769 (normal doubles far from the edges)
    true = np.exp(rng.uniform(np.log(1e-40), np.log(2.0), size=n))
    return np.ldexp(true, -EXP)


def test_decoded_values_never_exceed_the_wanted_share():
    rng = np.random.default_rng(1)
    qa, qb = raw_shares(rng, 200000), raw_shares(rng, 200000)
    # exactly representable wants too (power-of-two degrees, residue 1): the worst case
    qa[:1000] = np.ldexp(1.0 + rng.integers(0, 256, 1000) / 256.0, rng.integers(-120, 0, 1000) - EXP)
    qb[:1000] = np.ldexp(1.0 + rng.integers(0, 256, 1000) / 256.0, rng.integers(-120, 0, 1000) - EXP)
    ha, hb = share_field(qa, False), share_field(qb, True)
    w = ha | (hb << np.uint64(16))
    va, vb = value_a(w), value_b(w)
    assert np.all(va <= qa) and np.all(vb[hb > 0] <= qb[hb > 0])
    # the even column is clean (its value is its field alone), the odd one is not
    assert np.array_equal(va, clean(ha))
    assert np.all(vb >= clean(hb)) and np.any(vb > clean(hb))
    # rounding loss: < 2^-8 of the share (even), < 2^-7 (odd)
    assert np.all(va[ha > 0] >= qa[ha > 0] * (1 - 2.0 ** -8))
    assert np.all(vb[hb > 0] >= qb[hb > 0] * (1 - 2.0 ** -7))


def test_empty_halves():
    rng = np.random.default_rng(2)
    q = raw_shares(rng, 10000)
    ha = share_field(q, False)
    hb = share_field(q, True)
    # odd half empty: the even value is untouched, the odd one decodes to a subnormal
    w = ha
    assert np.array_equal(value_a(w), clean(ha))
    junk = value_b(w)
    assert np.all(junk < np.finfo(np.float64).tiny)             # < 2^-1022 raw
    assert np.all(np.ldexp(junk, EXP) < 2.0 ** -252)           # < 1.4e-76 as a share
    # even half empty: exact zero for the even column, the odd value is clean
    w = hb << np.uint64(16)
    assert np.all(value_a(w) == 0.0)
    assert np.array_equal(value_b(w), clean(hb))
    # nothing published: both zero
    assert value_a(np.zeros(1, np.uint64))[0] == 0.0 and value_b(np.zeros(1, np.uint64))[0] == 0.0


def test_range_and_monotonicity():
    # fields are float bit patterns: order-preserving, 2^-253 .. just under 4 as true shares
    h = np.arange(256, 0x10000, dtype=np.uint64)
    v = np.ldexp(clean(h), EXP)
    assert np.all(np.diff(v) > 0)
    assert v[0] == 2.0 ** -253 and v[-1] == 4.0 - 2.0 ** -7
    # below the format: no push; above: clamped to the largest field
    assert share_field(np.ldexp(2.0 ** -254, -EXP), False) == 0
    assert share_field(np.ldexp(2.0 ** -253, -EXP), False) == 256
    assert share_field(np.ldexp(2.0 ** -253, -EXP), True) == 0          # (one step down would leave the format)
    assert share_field(np.ldexp(1000.0, -EXP), False) == 0xFFFF
    # sums of decoded shares scale exactly: sum(raw) * 2^769 == sum(raw * 2^769)
    rng = np.random.default_rng(3)
    hs = rng.integers(256 + 120 * 256, 256 + 250 * 256, size=4096).astype(np.uint64)
    raw = clean(hs)
    assert np.ldexp(raw.sum(), EXP) == np.ldexp(raw, EXP).sum()
