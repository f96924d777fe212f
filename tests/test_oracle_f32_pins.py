"""Pins for the binary32 oracle (oracle.exact.round_decimal32; -m "not gpu").

Each test checks it against something other than itself:
  * round trip: every finite binary32 printed with 9 significant digits (or
    more, or its exact expansion) parses back to itself (PAPER.md L120-121:
    "If we serialize a 32-bit number using 9 digits, we can always parse it
    back exactly");
  * Clinger's fast path for binary32: for w <= 2^24 and
    -10 <= q <= 10 the nearest binary32 to w * 10^q is ONE correctly rounded
    IEEE single-precision multiplication or division of exact operands --
    numpy float32 arithmetic, an independent library routine;
  * brute force: argmin over all binary32 values of tiny windows, exact
    Fraction distances, ties to the even significand;
  * ties and near-ties constructed from exact midpoints,
    the overflow threshold 2^128 - 2^103 and half the smallest subnormal;
  * no double rounding: a value just above a binary32 midpoint that
    binary64 rounds onto the midpoint must still round up.
A wrong bias, precision, subnormal or overflow limit or tie rule in
round_decimal32 fails at least one of these.
"""
import random
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle

INF32 = 0x7F800000
SIGN32 = 1 << 31


def parse32(s):
    return oracle.parse_record(s.encode() if isinstance(s, str) else s, "f32")


def f32_of_bits(b):
    return struct.unpack("<f", struct.pack("<I", b))[0]


def f32_fraction(b):
    """exact value of finite binary32 bits (IEEE 754 decoding)."""
    sign = -1 if b >> 31 else 1
    ef, fr = (b >> 23) & 0xFF, b & ((1 << 23) - 1)
    assert ef != 0xFF
    m, e = (fr, -149) if ef == 0 else (fr | (1 << 23), ef - 150)
    return sign * Fraction(m) * Fraction(2) ** e


def exact_dec(fr):
    """exact decimal expansion of a dyadic Fraction n / 2^k, scientific notation:
    n / 2^k = n * 5^k * 10^-k."""
    neg = fr < 0
    fr = abs(fr)
    n, d = fr.numerator, fr.denominator
    k = d.bit_length() - 1
    assert d == 1 << k and n > 0
    D, q = str(n * 5 ** k), -k
    while len(D) > 1 and D[-1] == "0":
        D, q = D[:-1], q + 1
    s = D[0] + ("." + D[1:] if len(D) > 1 else "")
    return ("-" if neg else "") + s + "e%d" % (q + len(D) - 1)


def random_finite_bits(rng):
    while True:
        b = rng.getrandbits(32)
        if (b >> 23) & 0xFF != 0xFF:
            return b


def test_round_trip_9_digits():
    rng = random.Random(32)
    for _ in range(20000):
        b = random_finite_bits(rng)
        x = float(f32_of_bits(b))  # exact: a binary32 is a binary64
        for fmt in ("%.9g", "%.8e", "%.12e", "%.30e"):
            got, st = parse32(fmt % x)
            assert got == b, (hex(b), fmt % x, hex(got))
            assert st == oracle.STATUS_OK


def test_round_trip_exact_expansions():
    rng = random.Random(33)
    for _ in range(2000):
        b = random_finite_bits(rng)
        if b & 0x7FFFFFFF == 0:
            continue
        assert parse32(exact_dec(f32_fraction(b)))[0] == b


def test_clinger_fast_path_single_precision():
    # w <= 2^24, -10 <= q <= 10: w and 10^|q| are exact
    # binary32 values, so one IEEE operation gives the correctly rounded result
    rng = random.Random(34)
    for _ in range(20000):
        w = rng.randrange(0, (1 << 24) + 1)
        q = rng.randrange(-10, 11)
        fw = np.float32(w)
        p = np.float32(10 ** abs(q))
        assert int(fw) == w and int(p) == 10 ** abs(q)
        r = fw * p if q >= 0 else fw / p
        want = int(np.array([r], dtype=np.float32).view(np.uint32)[0])
        s = "%de%d" % (w, q)
        got, st = parse32(s)
        if want & 0x7FFFFFFF == INF32:
            assert st == oracle.STATUS_OVERFLOW
        assert got == want, (s, hex(got), hex(want))


def brute(fr, lo, hi):
    """nearest binary32 bits in [lo, hi] (positive, consecutive bit patterns) to Fraction fr,
    ties to the even significand; hi may be 0x7F800000 standing for 2^128."""
    best = None
    for b in range(lo, hi + 1):
        v = Fraction(2) ** 128 if b == INF32 else f32_fraction(b)
        d = abs(v - fr)
        if best is None or d < best[0] or (d == best[0] and b % 2 == 0):
            best = (d, b)
    return best[1]


@pytest.mark.parametrize("name,lo,count", [
    ("subnormal", 0x00000000, 96),
    ("subnormal-normal", 0x007FFFD0, 96),
    ("around-one", 0x3F7FFFD0, 96),
    ("top", 0x7F7FFFA0, 96),
])
def test_brute_force_window(name, lo, count):
    rng = random.Random(hash(name) & 0xFFFF)
    hi = lo + count - 1
    if name == "top":
        hi = INF32
    a, z = f32_fraction(lo + 1), f32_fraction(hi - 1) if hi != INF32 else f32_fraction(INF32 - 1)
    for _ in range(300):
        # a random decimal of 6..14 significant digits inside the window
        fr = a + (z - a) * Fraction(rng.randrange(10 ** 6), 10 ** 6)
        digits = rng.randrange(6, 15)
        s = "%.*e" % (digits - 1, float(fr))
        dec = Fraction(s)  # the exact value of the printed string
        if not (f32_fraction(lo) <= dec <= (f32_fraction(hi) if hi != INF32 else Fraction(2) ** 128)):
            continue
        want = brute(dec, lo, hi)
        got, _ = parse32(s)
        assert got == want, (name, s, hex(got), hex(want))


def test_ties_and_neighbours():
    rng = random.Random(35)
    for _ in range(3000):
        b = random_finite_bits(rng) & 0x7FFFFFFF
        if b >= 0x7F7FFFFF:
            continue
        lo, hi = f32_fraction(b), f32_fraction(b + 1)
        mid = (lo + hi) / 2
        s = exact_dec(mid)
        even = b if b % 2 == 0 else b + 1
        assert parse32(s)[0] == even, (s, hex(b))
        # one unit in the last printed digit above / below the midpoint
        mant, ex = s.split("e")
        nd = len(mant.replace(".", "")) - 1
        ulp = Fraction(10) ** (int(ex) - nd)
        if 2 * ulp >= hi - lo:  # a short expansion: one unit may pass the next midpoint
            continue
        for dv, want in ((ulp, b + 1), (-ulp, b)):
            v = mid + dv
            if v <= 0:
                continue
            got = parse32("%s" % exact_fraction_dec(v, nd + 1, int(ex)))[0]
            assert got == want, (s, dv, hex(got), hex(want))


def exact_fraction_dec(v, ndig, ex):
    """v (an exact multiple of 10^(ex-ndig+1)) printed with those digits."""
    scale = Fraction(10) ** (ex - ndig + 1)
    n = v / scale
    assert n.denominator == 1
    return "%de%d" % (n.numerator, ex - ndig + 1)


def test_thresholds():
    # overflow: 2^128 - 2^103 is the midpoint of FLT_MAX (odd significand) and 2^128 -> inf
    mid = Fraction(2) ** 128 - Fraction(2) ** 103
    s = exact_dec(mid)
    assert parse32(s) == (INF32, oracle.STATUS_OVERFLOW)
    assert parse32("-" + s) == (SIGN32 | INF32, oracle.STATUS_OVERFLOW)
    below = str(mid.numerator - 1)
    assert parse32(below) == (0x7F7FFFFF, oracle.STATUS_OK)
    # half the smallest subnormal: tie between 0 (even) and 2^-149 -> 0, underflow
    half = exact_dec(Fraction(1, 2 ** 150))
    assert parse32(half) == (0, oracle.STATUS_UNDERFLOW)
    assert parse32("-" + half) == (SIGN32, oracle.STATUS_UNDERFLOW)
    mant, ex = half.split("e")
    assert parse32(mant + "1e" + ex)[0] == 1  # a hair above the midpoint
    # the smallest normal and the largest subnormal
    assert parse32(exact_dec(Fraction(1, 2 ** 126)))[0] == 0x00800000
    assert parse32(exact_dec(Fraction(2 ** 23 - 1, 2 ** 149)))[0] == 0x007FFFFF
    assert parse32("1e39")[1] == oracle.STATUS_OVERFLOW
    assert parse32("1e-46") == (0, oracle.STATUS_UNDERFLOW)


def test_no_double_rounding():
    # x = M + 2^(e-41) just above the binary32 midpoint M = (2k+1) * 2^(e-1),
    # k even: binary64 rounds x onto M (the perturbation is far below half a
    # binary64 ulp of M), and M then ties to k.  Rounded once, x goes up to k+1.
    rng = random.Random(36)
    for _ in range(500):
        k = (1 << 23) + 2 * rng.randrange(1 << 22)  # even significand
        e = rng.randrange(-120, 100)
        M = Fraction(2 * k + 1) * Fraction(2) ** (e - 1)
        x = M + Fraction(2) ** (e - 41)
        s = exact_dec(x)
        assert float(Fraction(s)) == float(M)  # binary64 rounds it onto the midpoint
        got, _ = parse32(s)
        want = ((e + 150) << 23) | ((k + 1) - (1 << 23))
        assert got == want, (s, hex(got), hex(want))


def test_specials_and_grammar():
    assert parse32("inf") == (INF32, 0)
    assert parse32("-Infinity") == (SIGN32 | INF32, 0)
    assert parse32("nan") == (0x7FC00000, 0)
    assert parse32("-nan") == (SIGN32 | 0x7FC00000, 0)
    assert parse32("") == (0x7FC00000, oracle.STATUS_EMPTY)
    assert parse32("1x") == (0x7FC00000, oracle.STATUS_INVALID)
    assert parse32("-0") == (SIGN32, 0)
    assert parse32("0.1") == (0x3DCCCCCD, 0)  # the textbook binary32 of 0.1
