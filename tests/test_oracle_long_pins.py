"""Pins for the oracle's long-input branches and its multiprocess runners (-m "not gpu").

* int_of_digits (oracle/exact.py) folds 4000-digit chunks for significands
  CPython's int(str) refuses (> 4300 digits).  Pinned against int(str) with the
  limit lifted (a library routine), against 10^n, and through round_decimal on
  strings of 4001-12000 significant digits against CPython float() (correctly
  rounded and not subject to the int limit) -- PAPER.md L972-973 (long inputs
  must be honoured exactly), L986-987 ("it has to be exact").
* Exponents of any length (oracle/lexer.py, reading G9): values
  fixed by arithmetic ("1e" + 5000 zeros + "5" is 1e5), the 0/finite/inf class of
  huge exponents, and the compensating form 0.<N zeros>1e<N+1> == 1.
* oracle/api.py's static partition (_run with procs > 1, rebased bounds,
  out-of-range batch records) and parse_split_pool (chunks cut at separators)
  must equal the single-process evaluation record for record.
"""
import contextlib
import random
import sys

import pytest

import oracle
from oracle.exact import int_of_digits, round_decimal
from tests.pins import exact_decimal, float_bits, bits_to_fraction

INF = 0x7FF0000000000000
SIGN = 1 << 63


def parse(s):
    return oracle.parse_record(s.encode() if isinstance(s, str) else s)


@contextlib.contextmanager
def unlimited_int_str():
    old = sys.get_int_max_str_digits()
    sys.set_int_max_str_digits(0)
    try:
        yield
    finally:
        sys.set_int_max_str_digits(old)


# ----------------------------------------------------------------------------
# int_of_digits, > 4000 digits
@pytest.mark.parametrize("n", [1, 17, 3999, 4000, 4001, 4300, 4301, 8000, 8001, 12345, 20001])
def test_int_of_digits_matches_library_int(n):
    rng = random.Random(n)
    s = "".join(rng.choice("0123456789") for _ in range(n))
    with unlimited_int_str():
        want = int(s)
    assert int_of_digits(s) == want


@pytest.mark.parametrize("n", [4000, 4001, 7999, 8000, 8001, 15000])
def test_int_of_digits_powers_and_suffix(n):
    # 1 followed by n zeros is 10^n; the last k digits are the value mod 10^k
    assert int_of_digits("1" + "0" * n) == 10 ** n
    rng = random.Random(7 * n)
    s = "".join(rng.choice("0123456789") for _ in range(n))
    v = int_of_digits(s)
    assert v % 10 ** 1000 == int(s[-1000:])
    assert v // 10 ** (n - 1000) == int(s[:1000])


def _float_witness(s):
    f = float(s)  # correctly rounded, no digit limit
    st = oracle.STATUS_OK
    mant = s.lower().split("e")[0]
    if f in (float("inf"), float("-inf")):
        st = oracle.STATUS_OVERFLOW
    elif f == 0.0 and any(c in "123456789" for c in mant):
        st = oracle.STATUS_UNDERFLOW
    return float_bits(f), st


def test_long_significands_against_cpython_float():
    rng = random.Random(4001)
    for _ in range(60):
        n = rng.randint(4001, 12000)
        digits = str(rng.randint(1, 9)) + "".join(rng.choice("0123456789") for _ in range(n - 1))
        q = rng.randint(-n - 340, -n + 320)
        pos = rng.randint(1, n)  # where the point goes
        s = digits[:pos] + "." + digits[pos:] + "e%d" % (q + n - pos)
        if rng.random() < 0.5:
            s = "-" + s
        assert parse(s) == _float_witness(s), s[:40]


def test_long_midpoints_by_construction():
    # the exact decimal of the midpoint of b and b+ is a tie (-> the even one);
    # 4100 zeros and a 1 appended lift it just above (-> b+); the 4100-zero
    # padding alone changes nothing.  The 1.(4100 zeros)1 case: just above 1.
    rng = random.Random(4100)
    for _ in range(40):
        b = rng.randrange(1, 0x7FEFFFFFFFFFFFFF)
        x = bits_to_fraction(b)
        y = bits_to_fraction(b + 1)
        mid = (x + y) / 2
        M, E = mid.numerator, 0
        den = mid.denominator
        while den > 1:
            den //= 2
            E -= 1
        s = exact_decimal(M, E)
        mant, ex = s.split("e")
        if "." not in mant:
            mant += "."
        even = b if b % 2 == 0 else b + 1
        assert parse(s) == (even, oracle.STATUS_OK)
        assert parse(mant + "0" * 4100 + "e" + ex) == (even, oracle.STATUS_OK)
        assert parse(mant + "0" * 4100 + "1e" + ex) == (b + 1, oracle.STATUS_OK)
    assert parse("1." + "0" * 4100 + "1") == (0x3FF0000000000000, oracle.STATUS_OK)
    assert parse("9" * 4500) == (INF, oracle.STATUS_OVERFLOW)
    assert parse("0." + "0" * 4500 + "1") == (0, oracle.STATUS_UNDERFLOW)
    assert round_decimal(False, "1" + "0" * 5000, -5000) == (0x3FF0000000000000, oracle.STATUS_OK)


# ----------------------------------------------------------------------------
# exponents of any length (reading G9: the exact value)
@pytest.mark.parametrize("ndig", [13, 25, 4300, 4301, 5000, 9000])
def test_long_exponents(ndig):
    z = "0" * (ndig - 1)
    assert parse("1e" + z + "5") == (float_bits(1e5), 0)
    assert parse("1e-" + z + "5") == (float_bits(1e-5), 0)
    assert parse("-2.5E+" + z + "1") == (float_bits(-25.0), 0)
    nines = "9" * ndig
    assert parse("1e" + nines) == (INF, oracle.STATUS_OVERFLOW)
    assert parse("-1e" + nines) == (INF | SIGN, oracle.STATUS_OVERFLOW)
    assert parse("1e-" + nines) == (0, oracle.STATUS_UNDERFLOW)
    assert parse("0e" + nines) == (0, oracle.STATUS_OK)
    assert parse("-0.000e-" + nines) == (SIGN, oracle.STATUS_OK)
    assert parse("1e" + nines + "x") == (oracle.QNAN_BITS, oracle.STATUS_INVALID)


@pytest.mark.parametrize("N", [10, 400, 5000, 100_000])
def test_compensating_exponent(N):
    # 0.<N zeros>1 e(N+1) == 1 and 1<N zeros> e-N == 1, exactly
    assert parse("0." + "0" * N + "1e" + str(N + 1)) == (0x3FF0000000000000, 0)
    assert parse("1" + "0" * N + "e-" + str(N)) == (0x3FF0000000000000, 0)
    assert parse("0." + "0" * N + "15e" + str(N + 1)) == (float_bits(1.5), 0)


def test_long_hex_exponent():
    assert oracle.parse_record(b"0x1p" + b"0" * 5000 + b"3", "f64", oracle.GRAMMAR_HEX) == (float_bits(8.0), 0)
    assert oracle.parse_record(b"0x1p-" + b"9" * 5000, "f64", oracle.GRAMMAR_HEX) == (0, oracle.STATUS_UNDERFLOW)


# ----------------------------------------------------------------------------
# the multiprocess runners equal the single-process evaluation
def _mixed_buffer(n, seed):
    rng = random.Random(seed)
    recs = []
    for _ in range(n):
        k = rng.random()
        if k < 0.6:
            recs.append("%.17g" % rng.random())
        elif k < 0.8:
            recs.append("%d.%de%d" % (rng.randint(0, 99999), rng.randint(0, 10 ** 12), rng.randint(-330, 310)))
        elif k < 0.9:
            recs.append(rng.choice(["", "inf", "-nan", "1e", "x", ".", "1e400", "-1e-400"]))
        else:
            recs.append(str(rng.randint(1, 9)) + "".join(rng.choice("0123456789") for _ in range(rng.randint(19, 60))))
    return ("\n".join(recs) + "\n").encode()


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_run_partition_equals_single_process_batch(fmt):
    from oracle.api import parse_batch
    data = _mixed_buffer(12000, 1)
    offs = [0] + [i + 1 for i, c in enumerate(data) if c == 10][:-1]
    # out-of-range and decreasing bounds spread through every partition
    rng = random.Random(5)
    for i in rng.sample(range(len(offs)), 60):
        offs[i] = rng.choice([-3, len(data) + 7, offs[i - 1] - 1 if i else -1])
    one = parse_batch(data, offs, procs=1, fmt=fmt)
    many = parse_batch(data, offs, procs=8, fmt=fmt)
    assert len(one) == len(offs) and one == many
    assert sum(1 for b, st in one if st == oracle.STATUS_INVALID) >= 60


def test_run_partition_equals_single_process_split():
    data = _mixed_buffer(11000, 2).replace(b"\n", b",", 3000)
    offs1, r1 = oracle.parse_split(data, 0, procs=1)
    offs8, r8 = oracle.parse_split(data, 0, procs=8)
    assert offs1 == offs8 and r1 == r8 and len(r1) >= 11000


def test_parse_split_pool_equals_single_process():
    import multiprocessing as mp
    from oracle.api import parse_split_pool
    data = _mixed_buffer(10000, 3)
    _offs, ref = oracle.parse_split(data, 1)
    with mp.get_context("fork").Pool(4) as pool:
        for nchunks in (1, 7, 64):
            bits, st = parse_split_pool(data, 1, pool, nchunks)
            assert [(int(b), int(s)) for b, s in zip(bits, st)] == ref


@pytest.mark.parametrize("h", ["0x1p-1074", "0x1p-1075", "0x1.0000000000001p-1075", "0x1.8p-1076", "0x1p-1076",
                               "0x1.fffffffffffffp-1076", "0x1p1023", "0x1.fffffffffffff7p1023",
                               "0x1.fffffffffffff8p1023", "0x1p1024", "0x0.0000000000001p-1022", "0x8p-1078"])
def test_hex_range_thresholds_against_fromhex(h):
    # the cheap range decisions of _round_dyadic sit exactly at these thresholds;
    # float.fromhex is a correctly rounded library routine (ties to even)
    try:
        f = float.fromhex(h)
        want = float_bits(f)
        st = oracle.STATUS_UNDERFLOW if f == 0.0 else oracle.STATUS_OK
    except OverflowError:
        want, st = INF, oracle.STATUS_OVERFLOW
    assert oracle.parse_record(h.encode(), "f64", oracle.GRAMMAR_HEX) == (want, st)
