"""Pins for the grammar options of the oracle (-m "not gpu").

Hexadecimal floats (GRAMMAR_HEX):
  * the paper's two worked examples: 0x1.ff973cafa8p+52 = 9000000000000000 and
    0x1.3c27b13272fb6p+82 = 5.972e24 (L1497);
  * CPython float.fromhex -- an independent correctly rounded library routine --
    on random hex strings of 1-30 nibbles, any point position and exponents
    spanning subnormals and overflow;
  * binary32: exact values (<= 24 significant bits, where one rounding
    from binary64 is exact), constructed ties, brute-force windows.
JSON (GRAMMAR_JSON; RFC 8259 number grammar):
  * the paper's invalid examples "+1", "01", "1.e1", plus the RFC's other rules;
  * every JSON-valid record gives the same result as the default grammar.
"""
import random
import struct
from fractions import Fraction

import pytest

import oracle
from oracle import GRAMMAR_HEX, GRAMMAR_JSON

INF = 0x7FF0000000000000
QNAN = 0x7FF8000000000000


def hexparse(s, fmt="f64"):
    return oracle.parse_record(s.encode() if isinstance(s, str) else s, fmt, GRAMMAR_HEX)


def fbits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def test_paper_hex_examples():
    # "9000000000000000 can be written as 0x1.ff973cafa8p+52.
    # The mass of the Earth in kilogram (5.972e24) is 0x1.3c27b13272fb6p+82."
    assert hexparse("0x1.ff973cafa8p+52") == (fbits(9000000000000000.0), 0)
    assert hexparse("0x1.3c27b13272fb6p+82") == (fbits(5.972e24), 0)
    # the same values through the decimal grammar (cross-check of both paths)
    assert oracle.parse_record(b"9000000000000000")[0] == hexparse("0x1.ff973cafa8p+52")[0]
    assert oracle.parse_record(b"5.972e24")[0] == hexparse("0x1.3c27b13272fb6p+82")[0]


def _rand_hex(rng):
    nib = rng.randrange(1, 31)
    digs = "".join(rng.choice("0123456789abcdefABCDEF") for _ in range(nib))
    pt = rng.randrange(0, nib + 1)
    body = digs[:pt] + ("." if rng.random() < 0.7 else "") + digs[pt:]
    e = rng.randrange(-1200, 1100)
    s = ("-" if rng.random() < 0.3 else "") + rng.choice(["0x", "0X"]) + body
    if rng.random() < 0.9:
        s += rng.choice("pP") + ("%+d" % e if rng.random() < 0.5 else "%d" % e)
    return s


def test_against_float_fromhex():
    rng = random.Random(1497)
    n = 0
    while n < 20000:
        s = _rand_hex(rng)
        if s.lstrip("-")[2:] in (".", ""):
            continue
        n += 1
        bits, st = hexparse(s)
        try:
            x = float.fromhex(s)
        except OverflowError:
            assert (bits & ~(1 << 63), st) == (INF, oracle.STATUS_OVERFLOW), s
            continue
        assert bits == fbits(x), (s, hex(bits), x.hex())
        nonzero = int(s.lstrip("-")[2:].split("p")[0].split("P")[0].replace(".", "") or "0", 16) != 0
        if x == 0.0 and nonzero:
            assert st == oracle.STATUS_UNDERFLOW, s
        elif abs(x) != float("inf"):
            assert st == oracle.STATUS_OK, s


def test_hex_grammar():
    for bad in ["0x", "0x.", "0xp3", "0x1p", "0x1p+", "0x1g", "0x1.8q3", "0x1p3x", "x1p3", "0x 1"]:
        assert hexparse(bad) == (QNAN, oracle.STATUS_INVALID), bad
    assert hexparse("0x1p3\r\n")[0] == fbits(8.0)
    assert hexparse("-0x0p0") == (1 << 63, 0)
    assert hexparse("+0X.8P1") == (fbits(1.0), 0)
    assert hexparse("0x10") == (fbits(16.0), 0)  # exponent optional (reading H2)
    # without the option hex strings stay invalid (default grammar unchanged)
    assert oracle.parse_record(b"0x1p3") == (QNAN, oracle.STATUS_INVALID)


def _f32_fraction(b):
    ef, fr = (b >> 23) & 0xFF, b & ((1 << 23) - 1)
    m, e = (fr, -149) if ef == 0 else (fr | (1 << 23), ef - 150)
    return Fraction(m) * Fraction(2) ** e


def test_hex_binary32():
    rng = random.Random(1498)
    for _ in range(5000):
        # exact: a 24-bit significand and an exponent inside the binary32 range
        m = rng.randrange(1 << 23, 1 << 24)
        e = rng.randrange(-149 - 0, 104)
        if e < -149:
            continue
        s = "0x%xp%d" % (m, e)
        want = struct.unpack("<I", struct.pack("<f", float.fromhex(s)))[0] if e + 23 < 128 else None
        got, st = hexparse(s, "f32")
        if want is not None and _f32_fraction(want) == Fraction(m) * Fraction(2) ** e:
            assert got == want, s
    # ties: 1 + 2^-24 is the midpoint of 1 and 1 + 2^-23 -> 1 (even); a hair above -> up
    assert hexparse("0x1.000001p0", "f32")[0] == 0x3F800000
    assert hexparse("0x1.0000010000000001p0", "f32")[0] == 0x3F800001
    assert hexparse("0x1.000003p0", "f32")[0] == 0x3F800002  # midpoint of odd 0x..1 and 0x..2 -> even
    # overflow midpoint (2^128 - 2^103) and half the smallest subnormal
    assert hexparse("0x1.ffffffp127", "f32") == (0x7F800000, oracle.STATUS_OVERFLOW)
    assert hexparse("0x1.fffffefffp127", "f32") == (0x7F7FFFFF, 0)
    assert hexparse("0x1p-150", "f32") == (0, oracle.STATUS_UNDERFLOW)
    assert hexparse("0x1.000001p-150", "f32") == (1, 0)


@pytest.mark.parametrize("lo", [0x00000000, 0x007FFFF0, 0x3F7FFFF0])
def test_hex_binary32_brute_force(lo):
    rng = random.Random(lo)
    hi = lo + 40
    a, z = _f32_fraction(lo), _f32_fraction(hi)
    for _ in range(300):
        v = a + (z - a) * Fraction(rng.randrange(1 << 30), 1 << 30)
        # v is dyadic: print it exactly in hex
        n, d = v.numerator, v.denominator
        k = d.bit_length() - 1
        s = "0x%xp-%d" % (n, k)
        best = None
        for b in range(lo, hi + 1):
            dist = abs(_f32_fraction(b) - v)
            if best is None or dist < best[0] or (dist == best[0] and b % 2 == 0):
                best = (dist, b)
        assert hexparse(s, "f32")[0] == best[1], s


def jparse(s):
    return oracle.parse_record(s.encode(), "f64", GRAMMAR_JSON)


def test_json_invalid():
    # "in JSON, the following strings are invalid numbers: +1, 01, 1.e1"
    for bad in ["+1", "01", "1.e1", ".5", "5.", "00", "-01.5", "-", "1e", "1e+", "inf", "-Infinity",
                "nan", "0x1p3", "1.5.", "--1", "1E5x"]:
        assert jparse(bad) == (QNAN, oracle.STATUS_INVALID), bad
    assert jparse("") == (QNAN, oracle.STATUS_EMPTY)


def test_json_valid_matches_default():
    rng = random.Random(8259)
    for _ in range(20000):
        ip = "0" if rng.random() < 0.2 else str(rng.randrange(1, 10)) + "".join(
            str(rng.randrange(10)) for _ in range(rng.randrange(0, 25)))
        s = ("-" if rng.random() < 0.4 else "") + ip
        if rng.random() < 0.6:
            s += "." + "".join(str(rng.randrange(10)) for _ in range(rng.randrange(1, 25)))
        if rng.random() < 0.5:
            s += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.randrange(0, 400))
        assert jparse(s) == oracle.parse_record(s.encode()), s
        assert jparse(s)[1] in (0, 1, 2)
