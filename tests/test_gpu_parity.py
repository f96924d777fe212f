"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Bits and status bytes must be identical for every record (SURVEY.md 8d
"Bit-exact gate").  Sizes span many tiles and ragged tails; the full-size
configs are in test_gpu_fullsize.py.
"""
import random

import numpy as np
import pytest
import torch

import workloads
from tests.gpu_helpers import gpu_batch, gpu_split, oracle_batch, oracle_split, assert_same, to_dev

pytestmark = pytest.mark.gpu


def _records_to_buffer(recs, sep=b"\n"):
    offs, pos, parts = [], 0, []
    for r in recs:
        offs.append(pos)
        parts.append(r + sep)
        pos += len(r) + len(sep)
    return b"".join(parts), np.array(offs, dtype=np.int64)


def _check_both(data, offsets, sep_mask, what):
    gb, gs = gpu_batch(data, offsets)
    wb, ws = oracle_batch(data, offsets)
    assert_same(gb, gs, wb, ws, data, offsets, what + " [batch]")
    n, sb, ss, so = gpu_split(data, sep_mask)
    wo, wb2, ws2 = oracle_split(data, sep_mask)
    assert n == len(wo), (what, n, len(wo))
    assert np.array_equal(so, wo), what + " [split offsets]"
    assert_same(sb, ss, wb2, ws2, data, wo, what + " [split]")


@pytest.mark.parametrize("cfg,n", [(1, 100_000), (3, 40_000), (4, 60_000), (5, 6_000), (6, 100_000),
                                   (7, 20_000)])
def test_configs_vs_oracle(cuda_lib, cfg, n):
    w = workloads.generate(cfg, n)
    _check_both(w.data, w.offsets, w.sep_mask, "config %d" % cfg)
    # construction (known answers) agrees too
    gb, gs = gpu_batch(w.data, w.offsets)
    k = w.known.astype(bool)
    assert np.array_equal(gb[k], w.exp_bits[k]) and np.array_equal(gs[k], w.exp_status[k])


def test_random_w_q(cuda_lib):
    # Algorithm 1 over random (w, q) pairs across the whole table range
    rng = random.Random(1)
    recs = []
    for _ in range(60_000):
        w = rng.randint(0, 10 ** rng.randint(1, 19))
        q = rng.randint(-360, 330)
        recs.append(("%de%d" % (w, q)).encode())
    data, offs = _records_to_buffer(recs)
    _check_both(data, offs, 1, "random w,q")


ABORT_INPUTS = [  # Algorithm 1 "Abort" inputs (exhaustive list, early-stop form)
    "9495784171365944765e-329", "9734559530549076843e-224", "9313446463250210747e-188",
    "9266852287701459753e-169", "9797296344114496101e-160", "9801065208877838037e-156",
    "9342708520487353745e-130", "9782740569521650461e-121", "9847830601098862761e-115",
    "9283354611594685709e-89", "9280786500547668979e-67", "9586467486297153595e-46",
    "9792353653691471313e270", "9854224025956197963e276", "9724429689633648307e292",
    "6670407195648763069e-167", "9393790170148263134e-161", "6816081804757785610e-55",
]


def test_abort_inputs(cuda_lib):
    recs = [s.encode() for s in ABORT_INPUTS] + [("-" + s).encode() for s in ABORT_INPUTS]
    data, offs = _records_to_buffer(recs)
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    gb, gs = gpu_batch(data, offs, stats=stats)
    wb, ws = oracle_batch(data, offs)
    assert_same(gb, gs, wb, ws, data, offs, "abort inputs")
    assert stats[4].item() >= 30  # FPP_STAT_ABORT: the early-stop form aborts on them


def _fuzz_record(rng):
    alpha = b"0123456789.eE+-infatyINFATY\n,\rx "
    kind = rng.random()
    if kind < 0.5:
        L = rng.choice([0, 1, 2, 3, 5, 8, 17, 20, 40, 120, 300, 1000])
        return bytes(rng.choice(alpha) for _ in range(rng.randint(0, L)))
    if kind < 0.8:
        nd = rng.choice([1, 5, 17, 19, 20, 25, 60, 200, 800])
        digs = "".join(rng.choice("0123456789") for _ in range(nd))
        p = rng.randint(0, nd)
        s = digs[:p] + "." + digs[p:] if rng.random() < 0.7 else digs
        if rng.random() < 0.6:
            s += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.randint(0, 400))
        if rng.random() < 0.3:
            s = rng.choice("+-") + s
        return s.encode() + rng.choice([b"", b"\r", b",", b"\r\r"])
    return rng.choice([b"inf", b"-Infinity", b"nan", b"NaN", b"+inf\r", b"infinit", b"nan(1)", b"",
                       b"\r", b",", b"-0", b"0e99999", b".5", b"1.", b".", b"-", b"1e", b"1e+"])


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_grammar_fuzz(cuda_lib, seed):
    rng = random.Random(seed)
    recs = [_fuzz_record(rng) for _ in range(6000)]
    # batch: records include arbitrary bytes (separators too)
    data, offs = _records_to_buffer(recs, sep=b"")
    gb, gs = gpu_batch(data, offs)
    wb, ws = oracle_batch(data, offs)
    assert_same(gb, gs, wb, ws, data, offs, "fuzz batch")
    # split: the same text under each separator mask
    for mask in (0, 1, 2, 3):
        n, sb, ss, so = gpu_split(data, mask)
        wo, wb2, ws2 = oracle_split(data, mask)
        assert n == len(wo) and np.array_equal(so, wo)
        assert_same(sb, ss, wb2, ws2, data, wo, "fuzz split mask %d" % mask)


@pytest.mark.parametrize("shift", [1, 3, 7, 15])
def test_unaligned_and_ragged(cuda_lib, shift):
    w = workloads.generate(4, 30_000)
    raw = np.concatenate([np.zeros(shift, np.uint8), w.data, np.frombuffer(b"1.25", np.uint8)])
    dev = to_dev(raw)[shift:]                     # bytes pointer not 16-byte aligned
    data = raw[shift:]
    assert dev.data_ptr() % 16 == shift % 16
    from paper_2101_11408_b200 import native
    out, st, offs, n_out = native.parse_f64_split(dev, 1, want_offsets=True)
    torch.cuda.synchronize()
    n = int(n_out.item())
    wo, wb, ws = oracle_split(data, 1)
    assert n == len(wo) == w.n + 1
    assert_same(out[:n].cpu().numpy().view(np.uint64), st[:n].cpu().numpy(), wb, ws, data, wo, "unaligned split")
    o = to_dev(wo)
    out2, st2 = native.parse_f64_batch(dev, o)
    torch.cuda.synchronize()
    assert_same(out2.cpu().numpy().view(np.uint64), st2.cpu().numpy(), wb, ws, data, wo, "unaligned batch")


def test_long_records_straddle_tiles(cuda_lib):
    # records far longer than the staged halo, crossing many 8 KiB tiles
    rng = random.Random(5)
    recs = []
    for k in range(300):
        nd = rng.choice([30, 200, 900, 5000, 20000])
        digs = str(rng.randint(1, 9)) + "".join(rng.choice("0123456789") for _ in range(nd))
        recs.append((digs[:3] + "." + digs[3:] + "e-%d" % rng.randint(0, 340)).encode())
        recs.append(b"0." + b"0" * rng.choice([10, 500, 9000]) + b"1e%d" % rng.randint(0, 9400))
    data, offs = _records_to_buffer(recs)
    _check_both(data, offs, 1, "long records")


def test_edge_cases(cuda_lib):
    from paper_2101_11408_b200 import native
    # empty input: no records
    n, sb, ss, so = gpu_split(b"", 0)
    assert n == 0
    # separators only: each separator ends one EMPTY record; no record after the last
    n, sb, ss, so = gpu_split(b"\n\n,\n", 0)
    assert n == 4 and (ss == 4).all()
    # no trailing separator; single record
    n, sb, ss, so = gpu_split(b"0.5", 0)
    assert n == 1 and sb[0] == 0x3FE0000000000000 and ss[0] == 0
    # capacity smaller than the record count: first `capacity` written, n_out true count
    data = b"1\n2\n3\n4\n5\n"
    n, sb, ss, so = gpu_split(data, 1, capacity=3)
    assert n == 5 and sb.size == 3 and sb[2] == 0x4008000000000000
    # bad offsets: out of range / decreasing records are INVALID, never read
    d = b"1.5\n2.5\n"
    gb, gs = gpu_batch(d, [0, 100, 4, -3])
    wb, ws = oracle_batch(d, [0, 100, 4, -3])
    assert_same(gb, gs, wb, ws, what="bad offsets")
    # argument errors
    lib = native.load()
    assert lib.parse_f64_batch(None, 10, None, 1, None, None, None) == native.FPP_EARG
    assert lib.parse_f64_batch(None, 0, None, -1, None, None, None) == native.FPP_EARG
    assert lib.parse_f64_split(None, 5, 0, None, 0, None, None, None, None) == native.FPP_EARG


def test_overlapping_offsets_queue_overflow(cuda_lib):
    # zig-zag offsets make valid records overlap: the slow queue (sized from
    # len) can overflow; the status-scan fallback must still be exact
    rec = b"1.2345678901234567890123456789e-300\n"
    tie = b"9007199254740993.000000000000000000000000000001\n"
    data = rec + tie
    offs = []
    for k in range(3000):
        offs += [0, len(rec), len(rec) + 5, 0] if k % 2 else [len(rec), len(data), 3]
    gb, gs = gpu_batch(data, offs)
    wb, ws = oracle_batch(data, offs)
    assert_same(gb, gs, wb, ws, what="queue overflow")


def test_determinism_and_stats(cuda_lib):
    w = workloads.generate(2, 200_000)
    s1 = torch.zeros(8, dtype=torch.int64, device="cuda")
    a = gpu_split(w.data, 1, stats=s1)
    b = gpu_split(w.data, 1)
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    st = s1.cpu().numpy()
    assert st[0] == w.n                      # records
    assert st[3] == 0 and st[4] == 0         # no slow path, no abort on uniform %.17g
    rate = st[1] / w.n                       # two multiplications: 0.66% in the paper
    assert 0.002 < rate < 0.015, rate
    assert np.array_equal(a[1], w.exp_bits)  # round trip


def test_capacity_with_slow_and_long_records(cuda_lib):
    # records past `capacity` are counted but never written, also when they are
    # queued for the slow kernel (by (tile, j)) or are long (> 64 B)
    w = workloads.generate(5, 6000)
    data = bytes(w.data)
    wo, wb, ws = oracle_split(data, 1)
    for cap in (0, 1, 37, 2999, 5999):
        n, sb, ss, so = gpu_split(data, 1, capacity=cap)
        assert n == len(wo) and sb.size == min(cap, n)
        assert_same(sb, ss, wb[:cap], ws[:cap], data, wo, "capacity %d" % cap)
        assert np.array_equal(so, wo[:cap])


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_split_host_streaming(cuda_lib, fmt):
    # host-buffer streaming call: small chunks so that many chunk boundaries
    # (including ones at empty records and before long records) are crossed
    from paper_2101_11408_b200 import native
    parts = [bytes(workloads.generate(c, 3000).data) for c in (1, 3, 4, 5)]
    data = b"".join(parts) + b"\n\n,1.5\n" + b"7" * 500 + b"\n0.25"
    text = torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy()).pin_memory()
    fn = native.parse_f64_split_host if fmt == "f64" else native.parse_f32_split_host
    offs = torch.empty(len(data) + 1, dtype=torch.int64).pin_memory()
    for chunk in (1 << 12, 1 << 16, 0):
        out, st, o, n = fn(text, 3, offsets_out=offs, chunk_bytes=chunk)
        wo, wb, ws = oracle_split(data, 3, fmt=fmt)
        assert n == len(wo)
        u = np.uint64 if fmt == "f64" else np.uint32
        assert_same(out[:n].numpy().view(u), st[:n].numpy(), wb, ws, data, wo, "host chunk %d" % chunk)
        assert np.array_equal(o[:n].numpy(), wo)
    # capacity below the record count
    out, st, _, n = fn(text, 3, capacity=100, chunk_bytes=1 << 12)
    assert n == len(wo) and out.numel() == 100


def test_dense_tiles(cuda_lib):
    # records of 0-5 bytes: more than 512 record starts per 4 KiB tile, so the
    # kernel's dense path (lanes parse their own starts) runs; long records in
    # between end in later lanes, in the halo or in the next tile
    rng = random.Random(77)
    recs = []
    for i in range(200_000):
        r = rng.random()
        if r < 0.3:
            recs.append(str(rng.randrange(10)).encode())
        elif r < 0.5:
            recs.append(b"")
        elif r < 0.7:
            recs.append(("-%d" % rng.randrange(100)).encode())
        elif r < 0.9:
            recs.append(("%d.%d" % (rng.randrange(10), rng.randrange(10))).encode())
        elif r < 0.999:
            recs.append(b"1e5")
        else:
            recs.append(("%.17g" % rng.random()).encode() * rng.choice([1, 3, 40]))
    data = b"".join(r + rng.choice([b"\n", b","]) for r in recs)
    offs = []
    pos = 0
    for r in recs:
        offs.append(pos)
        pos += len(r) + 1
    _check_both(data, np.array(offs, dtype=np.int64), 3, "dense tiles")


def _fixed_len_record(rng, L):
    """A decimal record of exactly L bytes (L >= 3): "d.ddd..." with an optional sign."""
    s = ("-" if rng.random() < 0.3 else "") + str(rng.randrange(1, 10)) + "."
    return (s + "".join(str(rng.randrange(10)) for _ in range(L - len(s)))).encode()


@pytest.mark.parametrize("mix", ["long", "eight", "long_then_short", "slow_mixed"])
def test_result_buffering_paths(cuda_lib, mix):
    # k_split buffers a tile's results in the parsed front of its staged text
    # when every later round starts far enough in (records of ~9+ bytes), and
    # otherwise writes after the second round: exercise both, tiles that
    # switch from long to short records (the up-front check fails late), and
    # slow-path records and a capacity cut inside buffered tiles
    rng = random.Random({"long": 91, "eight": 92, "long_then_short": 93, "slow_mixed": 94}[mix])
    recs = []
    if mix == "long":
        recs = [_fixed_len_record(rng, rng.randrange(9, 30)) for _ in range(60_000)]
    elif mix == "eight":
        recs = [_fixed_len_record(rng, 7) for _ in range(80_000)]
    elif mix == "long_then_short":
        while len(recs) < 80_000:
            recs += [_fixed_len_record(rng, 25) for _ in range(rng.randrange(20, 120))]
            recs += [_fixed_len_record(rng, rng.randrange(3, 6)) for _ in range(rng.randrange(50, 400))]
    else:
        for _ in range(50_000):
            r = rng.random()
            if r < 0.02:  # more than 19 digits: bracket / slow path
                recs.append(_fixed_len_record(rng, rng.randrange(22, 60)))
            elif r < 0.025:  # long record (> 64 bytes): queued unscanned
                recs.append(_fixed_len_record(rng, rng.randrange(70, 300)))
            else:
                recs.append(_fixed_len_record(rng, rng.randrange(10, 20)))
    data, offs = _records_to_buffer(recs)
    _check_both(data, offs, 1, "buffering " + mix)
    if mix == "slow_mixed":  # capacity cut in the middle of a tile
        n, sb, ss, so = gpu_split(data, 1, capacity=len(recs) // 2 + 17)
        wo, wb, ws = oracle_split(data, 1)
        m = len(recs) // 2 + 17
        assert n == len(wo) and len(sb) == m
        assert np.array_equal(so, wo[:m])
        assert_same(sb, ss, wb[:m], ws[:m], data, wo[:m], "buffering capacity")


def _midpoint_digits(x):
    """(digits, exp10) with the midpoint of x and its successor = int(digits) * 10**exp10, exactly."""
    import math
    from fractions import Fraction
    m = (Fraction(x) + Fraction(math.nextafter(x, math.inf))) / 2
    k = 0
    while m.denominator != 1:  # denominator is a power of two: scale by 10 until integral
        m *= 10
        k += 1
    return str(m.numerator), -k


@pytest.mark.parametrize("seed", [11, 12])
def test_slow_path_limb_geometry(cuda_lib, seed):
    # exact midpoints (ties), and one unit above / below in the last digit,
    # printed with the decimal point at every offset modulo the 9-digit limb
    # grid, with leading zeros on either side of the point, and padded with
    # trailing zeros to lengths around the slow kernel's 2048-byte staging
    # limit: the comparison limbs straddle the point, the first nonzero digit
    # and the end of the digits in every way
    import math
    rng = random.Random(seed)
    recs = []
    for i in range(3000):
        kind = rng.random()
        if kind < 0.2:
            x = math.ldexp(rng.randrange(1, 1 << 52), -1074)         # subnormal region
        elif kind < 0.3:
            x = math.ldexp(1.0 + rng.random(), rng.randrange(1000, 1023))  # near overflow
        else:
            x = math.ldexp(1.0 + rng.random(), rng.randrange(-1000, 1000))
        digs, e10 = _midpoint_digits(x)
        tweak = rng.randrange(3)
        if tweak == 1:
            digs = str(int(digs) + 1)
        elif tweak == 2:
            digs = str(int(digs) - 1)
        pt = rng.randrange(0, min(len(digs), 40) + 1)  # digits before the point
        lead = "0" * rng.choice([0, 0, 1, 5, 13])
        pad = "0" * rng.choice([0, 0, 3, 17])
        if i % 50 == 0:  # around the staging limit
            pad = "0" * max(0, rng.randrange(2030, 2060) - len(digs) - 12)
        body = lead + digs[:pt] + "." + digs[pt:] + pad
        exp = e10 + len(digs) - pt
        recs.append(("%se%d" % (body, exp)).encode())
        if i % 7 == 0:  # the same value as 0.000ddd (no exponent when it stays short)
            z = rng.randrange(1, 30)
            recs.append(("0." + "0" * z + digs + "e%d" % (e10 + len(digs) + z)).encode())
    data, offs = _records_to_buffer(recs)
    _check_both(data, offs, 1, "slow-path limb geometry")


@pytest.mark.parametrize("edge", [-2, -1, 0, 1, 2, 30, 31, 32, 33])
def test_separators_at_tile_edges(cuda_lib, edge):
    # k_split's tiles own kWarpStride = 5088 bytes each and classify 32 more
    # (the halo): put separators at and around the ownership edge and the halo
    # end of the first few tiles, with short records (the fast parser) on both
    # sides, so the last record of a tile ends in the halo, at its first byte,
    # or just past it
    stride = 5088
    rng = random.Random(1000 + edge)
    parts, pos = [], 0
    for t in range(1, 5):
        o = t * stride + edge  # a separator at byte o
        while o - pos > 40:
            r = ("%.*f" % (rng.randrange(1, 8), rng.random() * 100)).encode()
            parts.append(r + b"\n")
            pos += len(r) + 1
        n = o - pos  # the record [pos, o): "d." and digits, then the separator at o
        r = (b"7." + b"".join(str(rng.randrange(10)).encode() for _ in range(n - 2))) if n >= 3 else b"7" * n
        parts.append(r + b"\n")
        pos += len(r) + 1
        assert pos == o + 1
    parts.append(b"0.5\n1e3")
    data = b"".join(parts)
    n, sb, ss, so = gpu_split(data, 1)
    wo, wb, ws = oracle_split(data, 1)
    assert n == len(wo)
    assert np.array_equal(so, wo)
    assert_same(sb, ss, wb, ws, data, wo, "tile edge %d" % edge)


def _many_digit_record(rng):
    """20 or more significant digits in at most ~70 bytes: the SWAR many-digit
    scanner (fastscan.cuh many_scan) -- the point anywhere, leading zeros in
    either part, exponents of 1-5 digits, trailing zeros (tnz false) and a
    lone nonzero digit far behind the 19th (tnz true)."""
    ni = rng.choice([0, 1, 1, 2, 5, 19, 20, 25, 40])
    nf = rng.choice([0, 1, 5, 18, 19, 20, 30, 45])
    lz = rng.choice([0, 0, 1, 3, 10])
    body = "".join(rng.choice("0123456789") for _ in range(ni + nf))
    shape = rng.random()
    if shape < 0.2:  # exact: 19 digits then zeros
        body = body[:19] + "0" * max(0, len(body) - 19)
    elif shape < 0.35:  # a lone nonzero digit far behind
        body = body[:19] + "0" * max(0, len(body) - 20) + ("1" if len(body) > 19 else "")
    ip, fp = body[:ni], body[ni:]
    if rng.random() < 0.5:
        ip = "0" * lz + ip
    else:
        fp = "0" * lz + fp
    s = ip + ("." + fp if (fp or rng.random() < 0.3) else "")
    if not any(c.isdigit() for c in s):
        s = "0" + s
    if rng.random() < 0.5:
        s += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.choice([0, 7, 45, 300, 330, 999, 12345]))
    if rng.random() < 0.4:
        s = rng.choice("+-") + s
    return s.encode() + rng.choice([b"", b"", b"\r"])


@pytest.mark.parametrize("seed", [21, 22])
def test_many_digit_records(cuda_lib, seed):
    rng = random.Random(seed)
    recs = [_many_digit_record(rng) for _ in range(20000)]
    assert sum(1 for r in recs if 20 <= len(r) <= 64) > 8000
    data, offs = _records_to_buffer(recs)
    _check_both(data, offs, 1, "many digits")


def _frac0_stream(rng, n, other_rate):
    """Mostly "0.ddd" records (the shape of config 2: %.17g of [1e-4, 1)), so
    most tiles' round 0 takes the "0.ddd" tile loop (k_split.cuh, fast_frac0),
    with fraction lengths 1-20, leading zeros, 20 digits with and without a
    leading zero (exact only with one), zeros, and records of other shapes
    mixed in (each lane's fallback to the general parse)."""
    others = [b"1.5e-05", b"-0.5", b"0.5e3", b"0.", b"00.5", b"0.1x", b"+0.25", b"0.123456789012345678901",
              b"0e5", b".5", b"0.5\r", b"1", b"12.5", b"0.00000000000000000001", b"0.99999999999999999999"]
    recs = []
    for _ in range(n):
        if rng.random() < other_rate:
            recs.append(rng.choice(others))
            continue
        nf = rng.choice([1, 2, 5, 9, 15, 16, 17, 17, 17, 18, 19, 20, 20])
        lz = rng.choice([0, 0, 0, 1, 2, 5]) if nf > 1 else 0
        digs = "0" * lz + "".join(rng.choice("0123456789") for _ in range(nf - lz))
        if rng.random() < 0.02:
            digs = "0" * nf
        recs.append(b"0." + digs.encode())
    return recs


@pytest.mark.parametrize("other_rate", [0.02, 0.3])
def test_frac0_tile_lane_fallbacks(cuda_lib, other_rate):
    """The tile-level "0.ddd" test (k_split.cuh FPP_F0_TILE: every non-digit of
    the tile is a separator or the byte after a record start) holds for these
    streams, so the tile loop runs, and the records of another shape -- another
    leading digit, another byte after it, too short, too long, 20 digits that
    are not exact -- take each lane's fallback to the general parse."""
    rng = random.Random(int(other_rate * 1000) + 77)
    others = [b"1.5", b"9.25", b"0e5", b"0.", b"0", b"7", b"0x5", b"5.", b"0a5", b"0.123456789012345678901",
              b"0.1234567890123456789012345", b"0.99999999999999999999", b"1e5", b"3.00000000000000000001",
              b"0.0", b"0,5", b"0.00000000000000000000"]
    recs = []
    for _ in range(50000):
        if rng.random() < other_rate:
            recs.append(rng.choice(others))
        else:
            nf = rng.choice([1, 3, 12, 15, 16, 17, 17, 18, 19, 20])
            lz = rng.choice([0, 0, 1, 4]) if nf > 4 else 0
            recs.append(b"0." + b"0" * lz + "".join(rng.choice("0123456789") for _ in range(nf - lz)).encode())
    data, offs = _records_to_buffer(recs)
    for fmt in ("f64", "f32"):
        n, sb, ss, so = gpu_split(data, 1, fmt=fmt)
        wo, wb, ws = oracle_split(data, 1, fmt=fmt)
        assert n == len(wo) and np.array_equal(so, wo)
        assert_same(sb, ss, wb, ws, data, wo, "frac0 lane fallbacks %s %.2f" % (fmt, other_rate))


@pytest.mark.parametrize("other_rate", [0.0, 0.003, 0.05])
def test_frac0_tiles(cuda_lib, other_rate):
    rng = random.Random(int(other_rate * 1000) + 5)
    recs = _frac0_stream(rng, 60000, other_rate)
    data, offs = _records_to_buffer(recs)
    for fmt in ("f64", "f32"):
        n, sb, ss, so = gpu_split(data, 1, fmt=fmt)
        wo, wb, ws = oracle_split(data, 1, fmt=fmt)
        assert n == len(wo) and np.array_equal(so, wo)
        assert_same(sb, ss, wb, ws, data, wo, "frac0 tiles %s %.3f" % (fmt, other_rate))
