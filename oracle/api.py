"""Whole-buffer oracle entry points (test infrastructure only).

Record semantics:
  batch: record i = bytes[offsets[i], end_i), end_i = offsets[i+1] (i < n-1)
         or len; a record whose bounds are decreasing or outside [0, len] is
         INVALID (never read outside the string).
  split: records are the maximal segments between separator bytes selected by
         sep_mask (bit0 '\\n', bit1 ','; 0 means both); the segment after a
         final trailing separator is not a record; len == 0 gives no record.

Per record: lex (lexer.py), then exact rounding (exact.py).  INVALID and EMPTY
records yield +qNaN 0x7FF8000000000000; "inf" -> +-inf, "nan" -> qNaN with the
sign bit for "-nan" (G10, G11).
"""
import os

from .exact import (STATUS_OK, STATUS_INVALID, STATUS_EMPTY, QNAN_BITS, INF_BITS,
                    SIGN_BIT, round_decimal, QNAN32_BITS, INF32_BITS, SIGN32_BIT, round_decimal32,
                    round_hex, round_hex32)
from .lexer import lex_record, GRAMMAR_DEFAULT, GRAMMAR_HEX, GRAMMAR_JSON


# per output format: (rounding, quiet NaN, infinity, sign bit)
_FORMATS = {
    "f64": (round_decimal, QNAN_BITS, INF_BITS, SIGN_BIT, round_hex),
    "f32": (round_decimal32, QNAN32_BITS, INF32_BITS, SIGN32_BIT, round_hex32),
}


def parse_record(rec, fmt="f64", grammar=GRAMMAR_DEFAULT):
    """(bits, status) for one record (bytes-like); fmt "f64" or "f32";
    grammar: lexer.GRAMMAR_* option."""
    rnd, qnan, inf, sgn, rhex = _FORMATS[fmt]
    lx = lex_record(rec, grammar)
    kind = lx[0]
    if kind == "num":
        return rnd(lx[1], lx[2], lx[3])
    if kind == "hex":
        return rhex(lx[1], lx[2], lx[3])
    if kind == "empty":
        return qnan, STATUS_EMPTY
    if kind == "invalid":
        return qnan, STATUS_INVALID
    sign = sgn if lx[1] else 0
    if kind == "inf":
        return sign | inf, STATUS_OK
    return sign | qnan, STATUS_OK  # nan


def sep_bytes(sep_mask):
    if sep_mask == 0:
        sep_mask = 3
    s = b""
    if sep_mask & 1:
        s += b"\n"
    if sep_mask & 2:
        s += b","
    return s


def split_records(data, sep_mask=0):
    """List of (start, end) record bounds for the split variant."""
    seps = sep_bytes(sep_mask)
    n = len(data)
    out = []
    start = 0
    for i in range(n):
        if data[i] in seps:
            out.append((start, i))
            start = i + 1
    if start < n:
        out.append((start, n))
    return out


def batch_bounds(length, offsets):
    """Record bounds for the batch variant; None marks an out-of-range record."""
    n = len(offsets)
    out = []
    for i in range(n):
        s = int(offsets[i])
        e = int(offsets[i + 1]) if i + 1 < n else length
        if s < 0 or s > length or e < s or e > length:
            out.append(None)
        else:
            out.append((s, e))
    return out


def _parse_bounds(args):
    data, bounds = args[0], args[1]
    fmt = args[2] if len(args) > 2 else "f64"
    grammar = args[3] if len(args) > 3 else GRAMMAR_DEFAULT
    mv = memoryview(data)
    res = []
    for b in bounds:
        if b is None:
            res.append((_FORMATS[fmt][1], STATUS_INVALID))
        else:
            res.append(parse_record(bytes(mv[b[0]:b[1]]), fmt, grammar))
    return res


def _run(data, bounds, procs, fmt="f64", grammar=GRAMMAR_DEFAULT):
    """Evaluate records, optionally over a process pool (static partition)."""
    if procs is None:
        procs = 1
    if procs <= 1 or len(bounds) < 2048:
        return _parse_bounds((data, bounds, fmt, grammar))
    import multiprocessing as mp
    chunk = (len(bounds) + procs - 1) // procs
    parts = []
    for k in range(procs):
        bs = bounds[k * chunk:(k + 1) * chunk]
        if not bs:
            continue
        lo = min((b[0] for b in bs if b is not None), default=0)
        hi = max((b[1] for b in bs if b is not None), default=0)
        rb = [None if b is None else (b[0] - lo, b[1] - lo) for b in bs]
        parts.append((bytes(data[lo:hi]), rb, fmt, grammar))
    ctx = mp.get_context("fork")
    with ctx.Pool(len(parts)) as pool:
        out = pool.map(_parse_bounds, parts)
    res = []
    for r in out:
        res.extend(r)
    return res


def parse_batch(data, offsets, procs=None, fmt="f64", grammar=GRAMMAR_DEFAULT):
    """Oracle for parse_f64_batch (fmt "f32": parse_f32_batch; grammar: the
    *_ex calls' option): list of (bits, status)."""
    return _run(data, batch_bounds(len(data), offsets), procs, fmt, grammar)


def parse_split(data, sep_mask=0, procs=None, fmt="f64", grammar=GRAMMAR_DEFAULT):
    """Oracle for parse_f64_split (fmt "f32": parse_f32_split; grammar: the
    *_ex calls' option): (offsets list, list of (bits, status))."""
    bounds = split_records(data, sep_mask)
    return [b[0] for b in bounds], _run(data, bounds, procs, fmt, grammar)


def default_procs():
    return os.cpu_count() or 1


# ----------------------------------------------------------------------------
# timing harness for the cpu_baseline / --impl reference legs of bench.py:
# the same oracle, run over chunks of the buffer cut at separators.
def _split_chunk(args):
    data, sep_mask = args
    offs, res = parse_split(data, sep_mask)
    import numpy as np
    return (np.array([r[0] for r in res], dtype=np.uint64), np.array([r[1] for r in res], dtype=np.uint8))


def chunk_at_separators(data, sep_mask, nchunks):
    """Cut data into <= nchunks pieces, each ending right after a separator."""
    seps = sep_bytes(sep_mask)
    L = len(data)
    cuts = [0]
    for k in range(1, nchunks):
        p = L * k // nchunks
        while p < L and data[p - 1] not in seps:
            p += 1
        if p > cuts[-1] and p < L:
            cuts.append(p)
    cuts.append(L)
    return [data[cuts[i]:cuts[i + 1]] for i in range(len(cuts) - 1)]


def parse_split_pool(data, sep_mask, pool, nchunks):
    """Oracle over `data` on a multiprocessing pool; returns (bits, status) arrays."""
    import numpy as np
    parts = pool.map(_split_chunk, [(c, sep_mask) for c in chunk_at_separators(data, sep_mask, nchunks)])
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
