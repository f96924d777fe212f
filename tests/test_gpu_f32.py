"""GPU parity for the binary32 entry points (parse_f32_batch / parse_f32_split,
SURVEY.md 8(f) f1) against the binary32 oracle (oracle.round_decimal32),
bit-exact IEEE bits plus status, through the C ABI.

Inputs: the paper's workload shapes (configs 1-5 at small sizes: the same
strings read as binary32, as PAPER.md Table tab:mfloatsamd32 does), and
binary32-specific cases -- exact midpoints of adjacent binary32 values and
their +-1 neighbours (ties only for q in [-17, 10]),
the subnormal / normal / overflow thresholds, 9-digit round trips (L120-121)
and long significands that need the w / w+1 bracket or the exact slow path.
"""
import random
import struct
from fractions import Fraction

import numpy as np
import pytest

import workloads
from tests.gpu_helpers import gpu_batch, gpu_split, oracle_batch, oracle_split, assert_same

pytestmark = pytest.mark.gpu


def _buffer(recs, sep=b"\n"):
    offs, pos, parts = [], 0, []
    for r in recs:
        offs.append(pos)
        parts.append(r + sep)
        pos += len(r) + len(sep)
    return b"".join(parts), np.array(offs, dtype=np.int64)


def _check(data, offsets, sep_mask, what):
    gb, gs = gpu_batch(data, offsets, fmt="f32")
    wb, ws = oracle_batch(data, offsets, fmt="f32")
    assert_same(gb, gs, wb, ws, data, offsets, what + " [f32 batch]")
    n, sb, ss, so = gpu_split(data, sep_mask, fmt="f32")
    wo, wb2, ws2 = oracle_split(data, sep_mask, fmt="f32")
    assert n == len(wo), (what, n, len(wo))
    assert np.array_equal(so, wo), what + " [f32 split offsets]"
    assert_same(sb, ss, wb2, ws2, data, wo, what + " [f32 split]")


@pytest.mark.parametrize("cfg,n", [(1, 60_000), (3, 30_000), (4, 40_000), (5, 4_000)])
def test_configs_f32(cuda_lib, cfg, n):
    w = workloads.generate(cfg, n)
    _check(w.data, w.offsets, w.sep_mask, "config %d" % cfg)


def _f32_fraction(b):
    ef, fr = (b >> 23) & 0xFF, b & ((1 << 23) - 1)
    m, e = (fr, -149) if ef == 0 else (fr | (1 << 23), ef - 150)
    return Fraction(m) * Fraction(2) ** e


def _exact_dec(fr):
    n, d = fr.numerator, fr.denominator
    k = d.bit_length() - 1
    D, q = str(n * 5 ** k), -k
    while len(D) > 1 and D[-1] == "0":
        D, q = D[:-1], q + 1
    return (D[0] + ("." + D[1:] if len(D) > 1 else "") + "e%d" % (q + len(D) - 1)).encode()


def _rand_bits(rng, lo_e=0, hi_e=254):
    return (rng.randrange(lo_e, hi_e + 1) << 23) | rng.getrandbits(23)


def test_ties_and_neighbours_f32(cuda_lib):
    rng = random.Random(320)
    recs = []
    for i in range(6000):
        # exponent fields spread over the whole range, denser near 2^0 where
        # short (<= 19-digit) ties exist
        b = _rand_bits(rng, 100, 160) if i % 2 else _rand_bits(rng, 0, 253)
        mid = (_f32_fraction(b) + _f32_fraction(b + 1)) / 2
        s = _exact_dec(mid)
        sign = b"-" if rng.random() < 0.5 else b""
        recs.append(sign + s)
        mant, ex = s.split(b"e")
        digits = mant.replace(b".", b"")
        v = int(digits) + (1 if rng.random() < 0.5 else -1)
        if v > 0:
            recs.append(sign + b"%de%d" % (v, int(ex) - (len(digits) - 1)))
    data, offs = _buffer(recs)
    _check(data, offs, 1, "binary32 ties")


def test_thresholds_f32(cuda_lib):
    recs = [
        _exact_dec(Fraction(2) ** 128 - Fraction(2) ** 103),       # overflow tie -> inf
        b"340282356779733661637539395458142568447",                # just below it -> FLT_MAX
        b"3.4028234663852886e38", b"3.4028235e38", b"3.4028236e38", b"1e39", b"-1e39",
        _exact_dec(Fraction(1, 2 ** 150)),                           # half the smallest subnormal -> 0
        b"1.4012984643248171e-45", b"1e-45", b"7e-46", b"7.1e-46", b"1e-46",
        b"1.17549435e-38", b"1.1754942e-38", b"1.1754943508222875e-38",
        b"16777216", b"16777217", b"16777218", b"16777219", b"33554433", b"9007199254740993",
        b"0.1", b"-0", b"0e10", b"inf", b"-nan", b"1x", b"", b"1e", b".5", b"5.", b"+.5e-3",
        b"1.000000059604644775390625", b"1.00000005960464477539062500000000001",
        b"0.000000000000000000000000000000000000000000001401298464324817070923729583289916131280",
    ]
    data, offs = _buffer(recs)
    _check(data, offs, 1, "binary32 thresholds")


def test_round_trip_and_long_f32(cuda_lib):
    rng = random.Random(321)
    recs = []
    for i in range(20000):
        b = _rand_bits(rng, 0, 254)
        x = struct.unpack("<f", struct.pack("<I", b))[0]
        recs.append((("%.9g", "%.8e", "%.12e", "%.25e")[i % 4] % x).encode())
        # long significands: 20-40 random digits (bracket, slow path)
        nd = rng.randrange(20, 41)
        d = str(rng.randrange(1, 10)) + "".join(str(rng.randrange(10)) for _ in range(nd - 1))
        recs.append(("%s.%se%d" % (d[0], d[1:], rng.randrange(-50, 40))).encode())
    data, offs = _buffer(recs)
    _check(data, offs, 1, "binary32 round trip + long")


def test_queue_overflow_marks_f32(cuda_lib):
    # overlapping offsets overflow the batch queue: the status-scan fallback
    # rebuilds the candidate (and its flags) from out[] and the mark
    rec = b"1.2345678901234567890123456789e-30\n"
    tie = b"16777217.000000000000000000000000000000000000000000000000000000000000001\n"
    data = rec + tie
    offs = []
    for k in range(3000):
        offs += [0, len(rec), len(rec) + 5, 0] if k % 2 else [len(rec), len(data), 3]
    gb, gs = gpu_batch(data, offs, fmt="f32")
    wb, ws = oracle_batch(data, offs, fmt="f32")
    assert_same(gb, gs, wb, ws, what="f32 queue overflow")
