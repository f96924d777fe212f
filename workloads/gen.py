"""Workload generators: C (threaded, full sizes) and a pure-Python twin.

generate(cfg, n) -> Workload with
  data        uint8[len]  newline (and for config 3 comma) separated text
  offsets     int64[n]    start of each record (batch variant input)
  sep_mask    separators the split variant should use (1 '\\n', 3 '\\n' and ',')
  exp_bits    uint64[n]   answer where known by construction, else 0
  exp_status  uint8[n]
  known       uint8[n]    1 where exp_bits/exp_status are known by construction:
                          configs 1, 2, 4 by the 17-digit round trip
                          (PAPER.md L55), config 6 (integers < 2^32 are
                          exact binary64), config 5 ties/near-ties by
                          construction; config 3 and the
                          random-digit quarter of config 5, config 7: 0
                          (oracle decides)

The per-record stream is counter based (SplitMix64, see csrc/fpgen.c), so the C
and Python generators agree byte for byte (tests/test_workloads.py).
"""
import ctypes
import os
import struct
import subprocess
from dataclasses import dataclass

import numpy as np

# configs 1-5: BASELINE.json; 6 "integer" and 7 "many digits": the paper's
# other synthetic datasets
# 8: config 2's values as C99 hexadecimal floats (grammar option HEX, 8(f) f4)
CONFIG_N = {1: 100_000, 2: 100_000_000, 3: 50_000_000, 4: 100_000_000, 5: 10_000_000,
            6: 100_000_000, 7: 10_000_000, 8: 100_000_000}
CONFIG_SEP_MASK = {1: 1, 2: 1, 3: 3, 4: 1, 5: 1, 6: 1, 7: 1, 8: 1}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "fpgen.c")
_LIB = os.path.join(_HERE, "libfpgen.so")

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
SIGN = 1 << 63
PINF = 0x7FF0000000000000
QNAN = 0x7FF8000000000000


@dataclass
class Workload:
    cfg: int
    data: np.ndarray
    offsets: np.ndarray
    sep_mask: int
    exp_bits: np.ndarray
    exp_status: np.ndarray
    known: np.ndarray

    @property
    def n(self):
        return int(self.offsets.shape[0])


# --------------------------------------------------------------------------
# C generator
def build_lib(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_lib())
        lib.fpgen_begin.restype = ctypes.c_void_p
        lib.fpgen_begin.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
        lib.fpgen_finish.restype = None
        lib.fpgen_finish.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def _generate_c(cfg, n, seed, threads):
    lib = _load()
    offsets = np.empty(n, dtype=np.int64)
    exp_bits = np.zeros(n, dtype=np.uint64)
    exp_status = np.zeros(n, dtype=np.uint8)
    known = np.zeros(n, dtype=np.uint8)
    total = ctypes.c_uint64(0)
    h = lib.fpgen_begin(cfg, n, seed, threads, offsets.ctypes.data, exp_bits.ctypes.data,
                        exp_status.ctypes.data, known.ctypes.data, ctypes.byref(total))
    data = np.empty(total.value, dtype=np.uint8)
    lib.fpgen_finish(h, data.ctypes.data)
    return Workload(cfg, data, offsets, CONFIG_SEP_MASK[cfg], exp_bits, exp_status, known)


# --------------------------------------------------------------------------
# pure-Python twin (small n)
def _mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


class _Rng:
    __slots__ = ("s",)

    def __init__(self, key, i):
        self.s = _mix64((key + (i + 1) * GAMMA) & MASK64)

    def next(self):
        self.s = (self.s + GAMMA) & MASK64
        return _mix64(self.s)


def _b2d(b):
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def _d2b(d):
    return struct.unpack("<Q", struct.pack("<d", d))[0]


_C4_FIXED = [0x0, 0x1, 0x2, 0x000FFFFFFFFFFFFF, 0x0010000000000000, 0x0010000000000001,
             0x7FEFFFFFFFFFFFFE, 0x7FEFFFFFFFFFFFFF]


def _emit_sci(neg, D, q):
    while len(D) > 1 and D[-1] == "0":
        D = D[:-1]
        q += 1
    s = "-" if neg else ""
    s += D[0]
    if len(D) > 1:
        s += "." + D[1:]
    return s + "e%+d" % (q + len(D) - 1)


def _midpoint_digits(bits):
    ef = (bits >> 52) & 0x7FF
    fr = bits & ((1 << 52) - 1)
    if ef == 0:
        m, e = fr, -1074
    else:
        m, e = fr | (1 << 52), ef - 1075
    f = e - 1
    if f < 0:
        return str((2 * m + 1) * 5 ** (-f)), f
    return str((2 * m + 1) << f), 0


def _py_record(cfg, key, i):
    """(text, exp_bits, exp_status, known) for record i."""
    r = _Rng(key, i)
    if cfg in (1, 2):
        x = (r.next() >> 11) * 2.0 ** -53
        return "%.17g\n" % x, _d2b(x), 0, 1
    if cfg == 3:
        u = (r.next() >> 11) * 2.0 ** -53
        s = 6 + r.next() % 11
        x = -90.0 + 180.0 * u if (i & 1) else -180.0 + 360.0 * u
        ax = abs(x)
        if ax >= 1.0:
            prec = max(s - len(str(int(ax))), 0)
        else:
            lz, y = 0, ax
            while 0.0 < y < 0.1 and lz < 30:
                y = y * 10.0
                lz += 1
            prec = s + lz
        return ("%.*f" % (prec, x)) + ("\n" if (i & 1) else ","), 0, 0, 0
    if cfg == 4:
        if i < 16:
            bits = _C4_FIXED[i >> 1] | (SIGN if (i & 1) else 0)
        else:
            r0 = r.next()
            if r0 % 1000 == 0:
                k = r.next() % 3
                return ["inf", "-inf", "nan"][k] + "\n", [PINF, PINF | SIGN, QNAN][k], 0, 1
            bits = r.next()
            while ((bits >> 52) & 0x7FF) == 0x7FF:
                bits = r.next()
        return "%.17e\n" % _b2d(bits), bits, 0, 1
    if cfg == 6:
        u = r.next() >> 32
        return "%u\n" % u, _d2b(float(u)), 0, 1
    if cfg == 8:
        x = (r.next() >> 11) * 2.0 ** -53
        b = _d2b(x)
        if b == 0:
            t = "0x0p+0"
        else:
            e = ((b >> 52) & 0x7FF) - 1023
            fr = b & ((1 << 52) - 1)
            nn = 13
            while nn > 0 and (fr & 15) == 0:
                fr >>= 4
                nn -= 1
            t = ("0x1.%0*xp%+d" % (nn, fr, e)) if nn else ("0x1p%+d" % e)
        return t + "\n", b, 0, 1
    if cfg == 7:
        a, b, d = r.next(), r.next(), r.next()
        return "%d%d%d\n" % (a, b, d), 0, 0, 0
    # cfg 5
    kind = r.next() & 3
    neg = r.next() & 1
    if i < 5:
        neg = 0
        kind = 0 if i in (0, 2) else (2 if i in (1, 3) else 4)
    if kind == 3:
        nd = 20 + r.next() % 21
        D = chr(ord("1") + r.next() % 9)
        for _ in range(1, nd):
            D += chr(ord("0") + r.next() % 10)
        E = -330 + r.next() % 641
        return _emit_sci(neg, D, E - (nd - 1)) + "\n", 0, 0, 0
    if i in (0, 1):
        bits = 0x7FEFFFFFFFFFFFFF
    elif 2 <= i < 5:
        bits = 0
    else:
        bits = r.next() & ~SIGN
        while ((bits >> 52) & 0x7FF) == 0x7FF:
            bits = r.next() & ~SIGN
    D, q = _midpoint_digits(bits)
    lo, hi = bits, bits + 1
    if kind <= 1:
        up = lo & 1
    else:
        plus = (kind == 2) if i < 5 else (r.next() & 1)
        if plus:
            D = str(int(D) + 1)
            up = 1
        else:
            D = str(int(D) - 1)
            up = 0
    res = hi if up else lo
    st = 1 if res == PINF else (2 if res == 0 else 0)
    return _emit_sci(neg, D, q) + "\n", res | (SIGN if neg else 0), st, 1


def _generate_py(cfg, n, seed):
    key = _mix64(((seed * GAMMA) & MASK64) ^ cfg)
    parts, offs, eb, es, kn = [], [], [], [], []
    pos = 0
    for i in range(n):
        t, b, s, k = _py_record(cfg, key, i)
        tb = t.encode()
        offs.append(pos)
        pos += len(tb)
        parts.append(tb)
        eb.append(b)
        es.append(s)
        kn.append(k)
    data = np.frombuffer(b"".join(parts), dtype=np.uint8).copy()
    return Workload(cfg, data, np.array(offs, dtype=np.int64), CONFIG_SEP_MASK[cfg],
                    np.array(eb, dtype=np.uint64), np.array(es, dtype=np.uint8),
                    np.array(kn, dtype=np.uint8))


def generate(cfg, n=None, seed=None, threads=None, impl="auto"):
    """Generate config cfg (1-5) with n records (default: the config's size).

    seed defaults to the config number.  impl: "c", "py", "auto".
    """
    if n is None:
        n = CONFIG_N[cfg]
    if seed is None:
        seed = cfg
    if impl == "auto":
        impl = "py" if n <= 2000 else "c"
    if impl == "py":
        return _generate_py(cfg, n, seed)
    if threads is None:
        threads = os.cpu_count() or 1
    return _generate_c(cfg, n, seed, threads)
