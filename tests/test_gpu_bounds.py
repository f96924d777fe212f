"""Memory-safety checks of our own (compute-sanitizer is closed on this GPU pool).

PAPER.md L167: "The parser must not access characters outside the string
range"; fpparse.h: nothing at or beyond bytes[len] (or before bytes[0]) is
read, and nothing outside out[0, capacity) / status / offsets_out is written.

* Reads: the same records are parsed inside differently filled guard zones
  (4 KiB before and after the text: digits, separators, 0xFF, '.', 'e') at
  every alignment; a read outside [0, len) that influenced a result would make
  the runs disagree with each other and with the oracle.
* Writes: out / status / offsets_out live inside larger allocations whose
  guard elements hold a sentinel; after the call the guards are unchanged,
  also when capacity cuts the output short.
"""
import random

import numpy as np
import pytest
import torch

import workloads
from tests.gpu_helpers import oracle_split, oracle_batch, assert_same

pytestmark = pytest.mark.gpu

GUARD = 4096
FILLS = [b"9", b"\n", b"\xff", b".", b"e", b"0"]


def _inputs():
    rng = random.Random(167)
    yield "c1", bytes(workloads.generate(1, 4000).data)
    yield "c3", bytes(workloads.generate(3, 4000).data)
    yield "c5", bytes(workloads.generate(5, 600).data)
    yield "c7", bytes(workloads.generate(7, 600).data)
    # records that end exactly at len (no trailing separator), long first and
    # last records, digits at both edges
    yield "edges", b"1" * 70 + b"\n" + bytes(workloads.generate(4, 800).data) + b"9" * 90
    yield "short", b"\n".join(str(rng.randrange(100)).encode() for _ in range(5000)) + b"\n7"
    yield "tail_e", bytes(workloads.generate(2, 500).data) + b"1.5e"
    yield "tail_dot", bytes(workloads.generate(2, 500).data) + b"12."


def _embedded(data, shift, fill):
    total = GUARD + shift + len(data) + GUARD
    raw = np.frombuffer(fill * total, dtype=np.uint8)[:total].copy()
    raw[GUARD + shift:GUARD + shift + len(data)] = np.frombuffer(data, dtype=np.uint8)
    dev = torch.from_numpy(raw).cuda()
    return dev[GUARD + shift:GUARD + shift + len(data)]


@pytest.mark.parametrize("name,data", list(_inputs()), ids=lambda v: v if isinstance(v, str) else "")
def test_reads_stay_inside(cuda_lib, name, data):
    from paper_2101_11408_b200 import native
    wo, wb, ws = oracle_split(data, 3 if name == "c3" else 1)
    sep = 3 if name == "c3" else 1
    offs = torch.from_numpy(np.asarray(wo, dtype=np.int64)).cuda()
    for shift in (0, 1, 7, 13):
        for fill in FILLS:
            dev = _embedded(data, shift, fill)
            out, st, _, n_out = native.parse_f64_split(dev, sep)
            out2, st2 = native.parse_f64_batch(dev, offs)
            torch.cuda.synchronize()
            n = int(n_out.item())
            assert n == len(wo), (name, shift, fill)
            what = "%s shift %d fill %r" % (name, shift, fill)
            assert_same(out[:n].cpu().numpy().view(np.uint64), st[:n].cpu().numpy(), wb, ws, data, wo, what)
            assert_same(out2.cpu().numpy().view(np.uint64), st2.cpu().numpy(), wb, ws, data, wo, what + " batch")


def _guarded(n, dtype, sentinel):
    full = torch.full((n + 2 * 64,), sentinel, dtype=dtype, device="cuda")
    return full, full[64:64 + n]


@pytest.mark.parametrize("fmt", ["f64", "f32"])
def test_writes_stay_inside(cuda_lib, fmt):
    from paper_2101_11408_b200 import native
    data = bytes(workloads.generate(5, 3000).data) + bytes(workloads.generate(1, 3000).data)
    wo, wb, ws = oracle_split(data, 1, fmt=fmt)
    dev = torch.from_numpy(np.frombuffer(data, dtype=np.uint8).copy()).cuda()
    vt = torch.int64 if fmt == "f64" else torch.int32
    fn = native.parse_f64_split if fmt == "f64" else native.parse_f32_split
    for cap in (len(wo), len(wo) - 1, 2999, 1, 0):
        fo, out = _guarded(cap, vt, -0x1234567)
        fs, st = _guarded(cap, torch.uint8, 0xA5)
        fofs, ofs = _guarded(cap, torch.int64, -7)
        o2, s2, _, n_out = fn(dev, 1, capacity=cap, out=out.view(torch.float64 if fmt == "f64" else torch.float32),
                              status=st, offsets_out=ofs)
        torch.cuda.synchronize()
        assert int(n_out.item()) == len(wo)
        for full, sentinel in ((fo, -0x1234567), (fs, 0xA5), (fofs, -7)):
            g = torch.cat([full[:64], full[-64:]]).cpu()
            assert bool((g == sentinel).all()), ("guard written", fmt, cap)
        u = np.uint64 if fmt == "f64" else np.uint32
        got = out.cpu().numpy().view(u)
        assert_same(got, st.cpu().numpy(), wb[:cap], ws[:cap], data, wo, "guarded cap %d" % cap)
        assert np.array_equal(ofs.cpu().numpy(), np.asarray(wo[:cap]))
    # batch: exactly n outputs between guards
    offs = torch.from_numpy(np.asarray(wo, dtype=np.int64)).cuda()
    fo, out = _guarded(len(wo), vt, -0x1234567)
    fs, st = _guarded(len(wo), torch.uint8, 0xA5)
    bf = native.parse_f64_batch if fmt == "f64" else native.parse_f32_batch
    bf(dev, offs, out=out.view(torch.float64 if fmt == "f64" else torch.float32), status=st)
    torch.cuda.synchronize()
    for full, sentinel in ((fo, -0x1234567), (fs, 0xA5)):
        g = torch.cat([full[:64], full[-64:]]).cpu()
        assert bool((g == sentinel).all()), ("batch guard written", fmt)
