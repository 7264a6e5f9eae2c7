"""CPU model of the exact accumulators (paper_2512_13796_b200/csrc/nx_xacc.cuh) in Python
integers: the chunking of fp32 / fp64 addends into 32-bit pieces of one fixed-point
number (lsb 2^-128) added to 6 int64 words with wrap-around, the carry normalisation and
the read-back. Checks the design claims the GPU results rely on: the words (hence the
value) do not depend on the order of the addends; the sum is exact for every bit of
the addends at or above 2^-128 (fp64 addends above 2^-75 and fp32 addends above 2^-104
keep all their bits; smaller ones lose the bits below 2^-128), compared with
fractions.Fraction; and the read-back is within a couple of ulp of that sum.
The GPU side is covered by tests/test_gpu_backward.py::test_backward_is_bit_reproducible."""
import math
import random
import struct
from fractions import Fraction

WORDS, E0 = 6, -128
MASK64 = (1 << 64) - 1


def chunks_f32(v):
    b = struct.unpack("<I", struct.pack("<f", v))[0]
    ex, neg = (b >> 23) & 0xFF, b >> 31
    m = b & 0x7FFFFF
    if ex:
        m |= 0x800000
    if ex == 0xFF or m == 0:
        return []
    s = (ex if ex else 1) - 150 - E0
    if s < 0:
        if s <= -24:
            return []
        m >>= -s
        s = 0
    k, r = s >> 5, s & 31
    assert k + 1 < WORDS
    y = m << r
    out = [(k, y & 0xFFFFFFFF), (k + 1, y >> 32)]
    return [(kk, (-c) & MASK64 if neg else c) for kk, c in out if c]


def chunks_f64(v):
    b = struct.unpack("<Q", struct.pack("<d", v))[0]
    ex, neg = (b >> 52) & 0x7FF, b >> 63
    m = b & ((1 << 52) - 1)
    if ex:
        m |= 1 << 52
    if ex == 0x7FF or m == 0:
        return []
    s = (ex if ex else 1) - 1075 - E0
    if s < 0:
        if s <= -53:
            return []
        m >>= -s
        s = 0
    k, r = s >> 5, s & 31
    lo, hi = (m << r) & MASK64, (m >> (64 - r)) if r else 0
    out = [(k, lo & 0xFFFFFFFF), (k + 1, lo >> 32), (k + 2, hi)]
    assert max(kk for kk, c in out if c) < WORDS
    return [(kk, (-c) & MASK64 if neg else c) for kk, c in out if c]


def accumulate(addends, f64):
    w = [0] * WORDS
    for v in addends:
        for k, c in (chunks_f64(v) if f64 else chunks_f32(v)):
            w[k] = (w[k] + c) & MASK64  # integer atomicAdd on the word
    return w


def signed(x):
    return x - (1 << 64) if x >> 63 else x


def exact_value(w):
    return sum(Fraction(signed(x)) * Fraction(2) ** (E0 + 32 * k) for k, x in enumerate(w))


def take(w):
    """xacc_take: carry-normalise to 32-bit digits + signed top, then sum from the top."""
    d, c = [], 0
    for x in w:
        t = signed(x) + c
        d.append(t & 0xFFFFFFFF)
        c = (t - (t & 0xFFFFFFFF)) >> 32
    neg = c < 0
    if neg:
        carry = 1
        for i in range(WORDS):
            t = (~d[i] & 0xFFFFFFFF) + carry
            d[i] = t & 0xFFFFFFFF
            carry = t >> 32
        c = ~c + carry
    r = float(c) * 2.0 ** 64
    for k in range(WORDS - 1, -1, -1):
        r += float(d[k]) * 2.0 ** (E0 + 32 * k)
    return -r if neg else r


def on_grid(x):
    """x with the bits below 2^E0 dropped (toward zero), as the chunking does."""
    q = Fraction(2) ** E0
    f = Fraction(x)
    n = abs(f) // q
    return n * q if f >= 0 else -n * q


def _addends(rng, n, f64):
    out = []
    for _ in range(n):
        mag = 10.0 ** rng.uniform(-30, 12)
        v = rng.choice([-1, 1]) * mag * rng.random()
        out.append(v if f64 else struct.unpack("<f", struct.pack("<f", v))[0])
    return out


def test_order_independent_and_exact_fp32():
    rng = random.Random(1)
    for trial in range(40):
        xs = _addends(rng, 200, f64=False)
        w = accumulate(xs, False)
        ys = xs[:]
        rng.shuffle(ys)
        assert accumulate(ys, False) == w  # the words are order-independent
        exact = sum(on_grid(x) for x in xs)
        assert exact_value(w) == exact  # the fixed-point sum is exact
        got = take(w)
        if exact != 0:
            assert abs(Fraction(got) - exact) <= abs(exact) * Fraction(2) ** -51


def test_order_independent_and_exact_fp64_with_cancellation():
    rng = random.Random(2)
    for trial in range(40):
        xs = _addends(rng, 100, f64=True)
        xs += [-x for x in xs[:50]]  # heavy cancellation
        w = accumulate(xs, True)
        ys = xs[:]
        rng.shuffle(ys)
        assert accumulate(ys, True) == w
        exact = sum(on_grid(x) for x in xs)
        assert exact_value(w) == exact
        got = take(w)
        if exact != 0:
            assert abs(Fraction(got) - exact) <= abs(exact) * Fraction(2) ** -51
        else:
            assert got == 0.0


def test_negative_totals_and_tiny_addends():
    w = accumulate([-1.5, 0.25, -2.0 ** -120, 3.0e10, -3.0e10], True)
    assert exact_value(w) == Fraction(-1.25) - Fraction(2) ** -120
    assert take(w) == -1.25
    assert accumulate([2.0 ** -140], True) == [0] * WORDS  # below 2^E0: dropped
    # addends above 2^-75 keep every bit: exact; below, the bits under 2^-128 go
    assert take(accumulate([3.0e-20] * 1000, True)) == float(Fraction(3.0e-20) * 1000)
    assert math.isclose(take(accumulate([1e-30] * 1000, True)), 1e-27, rel_tol=1e-8)
