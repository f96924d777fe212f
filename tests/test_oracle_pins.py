"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself:
  * values PAPER.md prints for worked examples (tests/golden/paper_examples.tsv);
  * the 17-digit round trip of every binary64;
  * brute force: argmin over all candidate doubles of a tiny window, with
    exact rational distances (Fractions) and ties to the even significand;
  * CPython float(), an independent correctly rounded library routine;
  * invariants (sign symmetry, zero padding, "D e Q" == "D0 e Q-1", monotonicity);
  * ties and near-ties known by construction (workloads config 5).
A dropped term, wrong sign, wrong tie rule, wrong subnormal or overflow
threshold in oracle/exact.py fails at least one of these.
"""
import os
import random
from fractions import Fraction

import pytest

import oracle
from oracle import (STATUS_OK, STATUS_OVERFLOW, STATUS_UNDERFLOW, STATUS_INVALID, STATUS_EMPTY,
                    QNAN_BITS)
from tests.pins import (value_to_bits, bits_to_fraction, exact_decimal, float_bits, bits_float,
                        hexfloat_bits, load_paper_examples)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_examples.tsv")
INF = 0x7FF0000000000000
SIGN = 1 << 63


def parse(s):
    return oracle.parse_record(s.encode() if isinstance(s, str) else s)


# ----------------------------------------------------------------------------
# worked examples printed in the paper
@pytest.mark.parametrize("row", load_paper_examples(GOLDEN), ids=lambda r: r[0][:30] + "|" + r[1][:12])
def test_paper_examples(row):
    inp, exp, cite = row
    bits, st = parse(inp)
    assert st == STATUS_OK, cite
    kind, val = exp.split(":", 1)
    if kind == "me":
        M, E = (int(v) for v in val.split(","))
        assert bits == value_to_bits(M, E), cite
    elif kind == "hex":
        assert bits == hexfloat_bits(val), cite
    elif kind == "int":
        assert bits_to_fraction(bits) == int(val), cite
    elif kind == "m":
        assert (bits & ((1 << 52) - 1)) | (1 << 52) == int(val), cite
    else:
        raise AssertionError(kind)


def test_paper_subnormal_examples():
    # (2^53-1) x 2^-1076 -> 2^51 x 2^-1074 (subnormal)
    b, st = parse(exact_decimal((1 << 53) - 1, -1076))
    assert (b, st) == (value_to_bits(1 << 51, -1074), STATUS_OK)
    # (2^53-1) x 2^-1075 -> 2^52 x 2^-1074, the smallest normal
    b, st = parse(exact_decimal((1 << 53) - 1, -1075))
    assert (b, st) == (0x0010000000000000, STATUS_OK)


def test_paper_768_digit_tie():
    # 2^-1022 + 2^-1074 + 2^-1075 needs 768 digits and rounds
    # (tie, to even) up to 2^-1022 + 2^-1073; any truncation is closer to the lower value.
    s = exact_decimal((1 << 53) + 3, -1075)
    mant = s.split("e")[0].replace(".", "")
    assert len(mant) == 768
    assert parse(s) == (value_to_bits((1 << 52) + 2, -1074), STATUS_OK)
    exp10 = int(s.split("e")[1])
    for keep in (17, 19, 40, 300, 767):
        t = mant[0] + "." + mant[1:keep] + "e%d" % exp10
        assert parse(t) == (value_to_bits((1 << 52) + 1, -1074), STATUS_OK), keep


def test_paper_bracket_example():
    # 1383425612993491676e-298 and ...677e-298 map to the same double
    a = parse("1383425612993491676e-298")
    b = parse("1383425612993491677e-298")
    assert a == b and a[1] == STATUS_OK


def test_paper_exactness_examples():
    # 1e22 exact, 1e23 not exact
    assert bits_to_fraction(parse("1e22")[0]) == 10 ** 22
    assert bits_to_fraction(parse("1e23")[0]) != 10 ** 23


# ----------------------------------------------------------------------------
# round trip of printed binary64 values (17 significant digits
# always parse back exactly; more digits are closer still)
def _random_finite_bits(rng):
    while True:
        b = rng.getrandbits(64)
        if (b >> 52) & 0x7FF != 0x7FF:
            return b


@pytest.mark.parametrize("fmt", ["%.16e", "%.17g", "%.17e", "%.25e", "%.40e"])
def test_round_trip(fmt):
    rng = random.Random(55 + len(fmt))
    specials = [0, 1, 2, 0x000FFFFFFFFFFFFF, 0x0010000000000000, 0x0010000000000001,
                0x7FEFFFFFFFFFFFFF, 0x7FEFFFFFFFFFFFFE, 0x3FF0000000000000, 0x433FFFFFFFFFFFFF]
    cases = specials + [s | SIGN for s in specials] + [_random_finite_bits(rng) for _ in range(6000)]
    for b in cases:
        s = fmt % bits_float(b)
        assert parse(s) == (b, STATUS_OK), s


def test_round_trip_exact_expansions():
    # %.767e prints the exact value of any double (<= 767 significant digits)
    rng = random.Random(767)
    for _ in range(300):
        b = _random_finite_bits(rng)
        s = "%.767e" % bits_float(b)
        assert parse(s) == (b, STATUS_OK)


# ----------------------------------------------------------------------------
# brute force over tiny windows of consecutive doubles
def _window(lo_bits, count):
    return [lo_bits + k for k in range(count)]


def _brute_nearest(x, cand_bits, top_is_inf):
    """argmin |x - c| over candidates (exact), ties to even significand."""
    best = None
    for i, b in enumerate(cand_bits):
        if top_is_inf and i == len(cand_bits) - 1:
            c = Fraction(2) ** 1024          # stands for +inf (IEEE)
        else:
            c = bits_to_fraction(b)
        d = abs(x - c)
        if best is None or d < best[0] or (d == best[0] and (b & 1) == 0):
            best = (d, b)
    return best[1]


def _decimal_in(lo, hi, rng):
    """a random decimal string (1-40 significant digits) with value in [lo, hi)."""
    t = lo + (hi - lo) * Fraction(rng.getrandbits(80), 1 << 80)
    nd = rng.randint(1, 40)
    # scientific digits of t truncated to nd digits (integer arithmetic)
    e10 = len(str(t.numerator // t.denominator)) - 1 if t >= 1 else -1
    while Fraction(10) ** e10 > t:
        e10 -= 1
    while Fraction(10) ** (e10 + 1) <= t:
        e10 += 1
    D = int(t / Fraction(10) ** (e10 - nd + 1))
    s = str(D)
    return s[0] + "." + s[1:] + "e%d" % e10 if len(s) > 1 else s + "e%d" % e10


@pytest.mark.parametrize("name,lo_bits,count,top_inf", [
    ("subnormal", 0x0, 192, False),
    ("subnormal-normal", 0x0010000000000000 - 96, 192, False),
    ("around-one", 0x3FF0000000000000 - 96, 192, False),
    ("overflow", 0x7FF0000000000000 - 160, 161, True),
])
def test_brute_force_window(name, lo_bits, count, top_inf):
    rng = random.Random(hash(name) & 0xFFFF)
    cands = _window(lo_bits, count)
    lo = bits_to_fraction(cands[0])
    hi_b = cands[-1]
    hi = Fraction(2) ** 1024 if top_inf else bits_to_fraction(hi_b)
    done = 0
    while done < 250:
        s = _decimal_in(lo, hi + (hi - lo) / 8 if top_inf else hi, rng)
        x = Fraction(s.split("e")[0]) * Fraction(10) ** int(s.split("e")[1])
        # the argmin over the window is the global argmin only inside [c_0, c_last]
        if x < lo or (x > hi and not top_inf):
            continue
        done += 1
        want = _brute_nearest(x, cands, top_inf)
        st = STATUS_OK
        if top_inf and want == cands[-1]:
            want, st = INF, STATUS_OVERFLOW
        if want == 0 and x != 0:
            st = STATUS_UNDERFLOW
        assert parse(s) == (want, st), s


def test_subnormal_ties_even():
    # ties in the subnormal range round to even (G3): k*2^-1074 + 2^-1075
    for k in range(0, 64):
        s = exact_decimal(2 * k + 1, -1075)
        want = k + (k & 1)
        st = STATUS_UNDERFLOW if want == 0 else STATUS_OK
        assert parse(s) == (want, st), s


def test_binade_carry():
    # rounding up out of the top of a binade: the tie between (2^53-1)*2^f and
    # 2^53*2^f goes to the even 2^(53+f); just above it too, just below it not.
    for f in (-1074, -1060, -200, -53, 0, 7, 300, 969):
        mid = ((1 << 54) - 1) * 2 ** 0, f - 1
        want = value_to_bits(1, 53 + f)
        below = value_to_bits((1 << 53) - 1, f)
        assert parse(exact_decimal(*mid)) == (want, STATUS_OK), f
        up = exact_decimal(((1 << 54) - 1) * (1 << 30) + 1, f - 31)
        assert parse(up) == (want, STATUS_OK), f
        dn = exact_decimal(((1 << 54) - 1) * (1 << 30) - 1, f - 31)
        assert parse(dn) == (below, STATUS_OK), f


def test_overflow_threshold():
    # midpoint of DBL_MAX and 2^1024 is 2^1024 - 2^970; IEEE rounds the tie to inf (G12)
    mid = exact_decimal((1 << 54) - 1, 970)
    assert parse(mid) == (INF, STATUS_OVERFLOW)
    below = exact_decimal(((1 << 54) - 1) * (1 << 20) - 1, 950)
    assert parse(below) == (0x7FEFFFFFFFFFFFFF, STATUS_OK)


# ----------------------------------------------------------------------------
# CPython float(): a correctly rounded library conversion, used as a witness
def _random_decimal(rng):
    nd = rng.choice([1, 2, 5, 10, 15, 16, 17, 18, 19, 20, 21, 25, 30, 40, 60, 120])
    digits = "".join(rng.choice("0123456789") for _ in range(nd))
    point = rng.randint(0, nd)
    s = digits[:point] + ("." + digits[point:] if point < nd else "")
    if not s or s == ".":
        s = "0"
    if rng.random() < 0.8:
        s += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.randint(0, 420))
    if rng.random() < 0.5:
        s = "-" + s
    return s


def test_against_cpython_float():
    rng = random.Random(2101)
    for _ in range(20000):
        s = _random_decimal(rng)
        f = float(s)
        want = float_bits(f)
        digits_nonzero = any(ch in "123456789" for ch in s.split("e")[0].split("E")[0])
        st = STATUS_OK
        if f in (float("inf"), float("-inf")):
            st = STATUS_OVERFLOW
        elif f == 0.0 and digits_nonzero:
            st = STATUS_UNDERFLOW
        assert parse(s) == (want, st), s


# ----------------------------------------------------------------------------
# invariants
def test_invariants():
    rng = random.Random(11408)
    for _ in range(3000):
        digits = str(rng.randint(1, 10 ** rng.randint(1, 30)))
        q = rng.randint(-360, 330)
        base = parse("%se%d" % (digits, q))
        # sign symmetry (negative numbers flip the sign bit)
        neg = parse("-%se%d" % (digits, q))
        assert neg == (base[0] | SIGN, base[1])
        # leading/trailing zero padding and D e Q == D0 e Q-1
        assert parse("000%s.000e%d" % (digits, q)) == base
        assert parse("%s0e%d" % (digits, q - 1)) == base
        assert parse("0.%se%d" % (digits, q + len(digits))) == base


def test_monotone():
    rng = random.Random(7)
    vals = []
    for _ in range(2000):
        D = rng.randint(1, 10 ** 25)
        q = rng.randint(-340, 300)
        vals.append((Fraction(D) * Fraction(10) ** q, "%de%d" % (D, q)))
    vals.sort()
    prev = -1
    for _, s in vals:
        b, _st = parse(s)
        v = b if b != INF else (0x7FF << 52)
        assert v >= prev, s
        prev = v


# ----------------------------------------------------------------------------
# ties and near-ties known by construction (PAPER.md L45-46 generalised)
def test_constructed_ties_and_neighbours():
    import workloads
    w = workloads.generate(5, 600, impl="py")
    data = bytes(w.data)
    offs = list(w.offsets) + [len(data)]
    checked = 0
    for i in range(w.n):
        if not w.known[i]:
            continue
        rec = data[offs[i]:offs[i + 1]]
        assert parse(rec) == (int(w.exp_bits[i]), int(w.exp_status[i])), rec[:60]
        checked += 1
    assert checked > 400


# ----------------------------------------------------------------------------
# grammar and boundary vectors (numeric values
# cross-checked with CPython float() above)
GRAMMAR = [
    (b"", QNAN_BITS, STATUS_EMPTY), (b"\n", QNAN_BITS, STATUS_EMPTY), (b",", QNAN_BITS, STATUS_EMPTY),
    (b"\r\n", QNAN_BITS, STATUS_EMPTY),
    (b".", QNAN_BITS, STATUS_INVALID), (b"+", QNAN_BITS, STATUS_INVALID),
    (b"-", QNAN_BITS, STATUS_INVALID), (b"e5", QNAN_BITS, STATUS_INVALID),
    (b".e5", QNAN_BITS, STATUS_INVALID), (b"1e", QNAN_BITS, STATUS_INVALID),
    (b"1e+", QNAN_BITS, STATUS_INVALID), (b" 1", QNAN_BITS, STATUS_INVALID),
    (b"1 ", QNAN_BITS, STATUS_INVALID), (b"1,2", QNAN_BITS, STATUS_INVALID),
    (b"0x1p3", QNAN_BITS, STATUS_INVALID), (b"infinit", QNAN_BITS, STATUS_INVALID),
    (b"nan(1)", QNAN_BITS, STATUS_INVALID), (b"--1", QNAN_BITS, STATUS_INVALID),
    (b"1..2", QNAN_BITS, STATUS_INVALID), (b"1e5.", QNAN_BITS, STATUS_INVALID),
    (b"1.", 0x3FF0000000000000, STATUS_OK), (b".5", 0x3FE0000000000000, STATUS_OK),
    (b"01", 0x3FF0000000000000, STATUS_OK), (b"+.5", 0x3FE0000000000000, STATUS_OK),
    (b"-0", 0x8000000000000000, STATUS_OK), (b"0e99999", 0, STATUS_OK),
    (b"1\r\n", 0x3FF0000000000000, STATUS_OK), (b"1,", 0x3FF0000000000000, STATUS_OK),
    (b"inf", INF, STATUS_OK), (b"-Infinity", INF | SIGN, STATUS_OK),
    (b"NAN", QNAN_BITS, STATUS_OK), (b"-nan", QNAN_BITS | SIGN, STATUS_OK),
    (b"+InF\r", INF, STATUS_OK),
    (b"1e400", INF, STATUS_OVERFLOW), (b"-1e-400", SIGN, STATUS_UNDERFLOW),
    (b"1e-99999999999999999999", 0, STATUS_UNDERFLOW),
    (b"1e+99999999999999999999", INF, STATUS_OVERFLOW),
    (b"0." + b"0" * 399 + b"1e400", 0x3FF0000000000000, STATUS_OK),
]


@pytest.mark.parametrize("rec,bits,st", GRAMMAR, ids=lambda v: repr(v)[:24])
def test_grammar_vectors(rec, bits, st):
    assert parse(rec) == (bits, st)


# ----------------------------------------------------------------------------
# record bounds
def test_split_records():
    sr = oracle.split_records
    assert sr(b"", 0) == []
    assert sr(b"\n", 0) == [(0, 0)]
    assert sr(b"1\n2", 0) == [(0, 1), (2, 3)]
    assert sr(b"1\n2\n", 0) == [(0, 1), (2, 3)]
    assert sr(b"1,2\n\n3", 0) == [(0, 1), (2, 3), (4, 4), (5, 6)]
    assert sr(b"1,2\n", 1) == [(0, 3)]
    assert sr(b"1,2\n", 2) == [(0, 1), (2, 4)]


def test_batch_bounds():
    from oracle.api import batch_bounds
    assert batch_bounds(5, [0, 2, 4]) == [(0, 2), (2, 4), (4, 5)]
    assert batch_bounds(5, [0, 6, 4]) == [None, None, (4, 5)]
    assert batch_bounds(5, [3, 1]) == [None, (1, 5)]
    assert batch_bounds(5, [-1, 5]) == [None, (5, 5)]
