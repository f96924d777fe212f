"""GPU parity for the grammar options through the *_ex C ABI
calls: C99 hexadecimal floats (FPP_GRAMMAR_HEX) and RFC
8259 JSON numbers (FPP_GRAMMAR_JSON), binary64 and binary32,
split and batch, against the oracle's grammar options bit for bit.
"""
import random

import numpy as np
import pytest

import workloads
from tests.gpu_helpers import gpu_batch, gpu_split, oracle_batch, oracle_split, assert_same

pytestmark = pytest.mark.gpu

HEX, JSON = 1, 2


def _buffer(recs, sep=b"\n"):
    offs, pos, parts = [], 0, []
    for r in recs:
        offs.append(pos)
        parts.append(r + sep)
        pos += len(r) + len(sep)
    return b"".join(parts), np.array(offs, dtype=np.int64)


def _check(data, offsets, sep_mask, grammar, fmt, what):
    gb, gs = gpu_batch(data, offsets, fmt=fmt, grammar=grammar)
    wb, ws = oracle_batch(data, offsets, fmt=fmt, grammar=grammar)
    assert_same(gb, gs, wb, ws, data, offsets, "%s [%s batch]" % (what, fmt))
    n, sb, ss, so = gpu_split(data, sep_mask, fmt=fmt, grammar=grammar)
    wo, wb2, ws2 = oracle_split(data, sep_mask, fmt=fmt, grammar=grammar)
    assert n == len(wo)
    assert np.array_equal(so, wo)
    assert_same(sb, ss, wb2, ws2, data, wo, "%s [%s split]" % (what, fmt))


def _hex_records(rng, n):
    recs = []
    for i in range(n):
        nib = rng.randrange(1, 40 if i % 5 == 0 else 18)
        digs = "".join(rng.choice("0123456789abcdefABCDEF") for _ in range(nib))
        pt = rng.randrange(0, nib + 1)
        body = digs[:pt] + ("." if rng.random() < 0.7 else "") + digs[pt:]
        e = rng.choice([rng.randrange(-1200, 1100), rng.randrange(-160, 140), rng.randrange(-20, 20)])
        s = rng.choice(["", "-", "+"]) + rng.choice(["0x", "0X"]) + body
        if rng.random() < 0.9:
            s += rng.choice("pP") + ("%+d" % e if rng.random() < 0.5 else "%d" % e)
        recs.append(s.encode())
    recs += [b"0x1.ff973cafa8p+52", b"0x1.3c27b13272fb6p+82", b"0x1p-1074", b"0x1p-1075", b"0x1.8p-1075",
             b"0x1.fffffffffffff8p1023", b"0x1.fffffffffffff7ffp1023", b"0x1.000001p0", b"0x1.ffffffp127",
             b"0x1p-150", b"0x", b"0xp3", b"0x1p", b"0x1g", b"0x.", b"-0x0p0", b"0x1p3\r", b"1.5", b"inf",
             b"0x" + b"0" * 70 + b"1p0", b"0x1." + b"0" * 80 + b"1p0"]
    return recs


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_hex_floats(cuda_lib, fmt):
    rng = random.Random(1497 if fmt == "f64" else 1498)
    data, offs = _buffer(_hex_records(rng, 8000))
    _check(data, offs, 1, HEX, fmt, "hex")


def _json_records(rng, n):
    recs = []
    for _ in range(n):
        ip = "0" if rng.random() < 0.2 else str(rng.randrange(1, 10)) + "".join(
            str(rng.randrange(10)) for _ in range(rng.randrange(0, 25)))
        s = ("-" if rng.random() < 0.4 else "") + ip
        if rng.random() < 0.6:
            s += "." + "".join(str(rng.randrange(10)) for _ in range(rng.randrange(1, 25)))
        if rng.random() < 0.5:
            s += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.randrange(0, 400))
        r = rng.random()
        if r < 0.1:
            s = "+" + s              # invalid in JSON
        elif r < 0.2:
            s = "0" + s.lstrip("-")  # leading zero (or "00")
        elif r < 0.25:
            s = s.replace(".", "") + "."
        elif r < 0.3:
            s = "." + s.lstrip("-0123456789").lstrip(".") if "." in s else "." + s
        recs.append(s.encode())
    recs += [b"+1", b"01", b"1.e1", b".5", b"5.", b"inf", b"nan", b"-0", b"0", b"0e0", b"-0.0e-0",
             b"1" * 60, b"0." + b"1" * 70, b"-" + b"9" * 40 + b".5e-3"]
    return recs


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_json_strict(cuda_lib, fmt):
    rng = random.Random(8259)
    data, offs = _buffer(_json_records(rng, 20000))
    _check(data, offs, 1, JSON, fmt, "json")


def test_json_on_workloads(cuda_lib):
    # configs 3 and 4 are valid JSON numbers apart from config 4's inf / nan
    for cfg, n in ((3, 30000), (4, 30000)):
        w = workloads.generate(cfg, n)
        _check(w.data, w.offsets, w.sep_mask, JSON, "f64", "json config %d" % cfg)


def test_bad_grammar_value(cuda_lib):
    import torch
    from paper_2101_11408_b200 import native
    d = torch.zeros(4, dtype=torch.uint8, device="cuda")
    with pytest.raises(native.FppError):
        native.parse_f64_split(d, 1, grammar=3)
