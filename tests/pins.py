"""Textbook helpers for the pins (no conversion arithmetic of the method).

value_to_bits packs an *exactly representable* value M * 2^E into binary64
bits (IEEE 754 encoding); exact_decimal prints M * 2^E as
its exact decimal expansion with integer arithmetic.  Neither rounds
anything: they raise if the value is not representable.
"""
import struct
from fractions import Fraction


def value_to_bits(M, E, neg=False):
    """binary64 bits of M * 2^E (M > 0 integer); must be exactly representable."""
    if M == 0:
        return (1 << 63) if neg else 0
    while M % 2 == 0:
        M //= 2
        E += 1
    # now M odd: normalise to 53 bits
    shift = 53 - M.bit_length()
    if shift < 0:
        raise ValueError("not representable (too many bits)")
    m, e = M << shift, E - shift          # m in [2^52, 2^53)
    if e < -1074:                          # subnormal: need e == -1074 after denormalising
        k = -1074 - e
        if m % (1 << k):
            raise ValueError("not representable (below subnormal grid)")
        bits = m >> k                      # < 2^52: biased exponent field 0
    else:
        if e + 52 > 1023:
            raise ValueError("overflow")
        bits = ((e + 1075) << 52) | (m - (1 << 52))
    return bits | ((1 << 63) if neg else 0)


def bits_to_fraction(bits):
    """Exact value of finite binary64 bits as a Fraction."""
    sign = -1 if bits >> 63 else 1
    ef = (bits >> 52) & 0x7FF
    fr = bits & ((1 << 52) - 1)
    if ef == 0x7FF:
        raise ValueError("not finite")
    if ef == 0:
        m, e = fr, -1074
    else:
        m, e = fr | (1 << 52), ef - 1075
    return sign * (Fraction(m) * (Fraction(2) ** e))


def exact_decimal(M, E):
    """Exact decimal expansion (scientific, no trailing zeros) of M * 2^E."""
    if E >= 0:
        D, q = str(M << E), 0
    else:
        D, q = str(M * 5 ** (-E)), E
    while len(D) > 1 and D[-1] == "0":
        D = D[:-1]
        q += 1
    s = D[0] + ("." + D[1:] if len(D) > 1 else "")
    return s + "e%d" % (q + len(D) - 1)


def float_bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def bits_float(b):
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def hexfloat_bits(h):
    """bits of a C99 hex float literal (library routine float.fromhex)."""
    return float_bits(float.fromhex(h))


def load_paper_examples(path):
    rows = []
    with open(path) as f:
        for line in f:
            if not line.strip() or line.startswith("#"):
                continue
            inp, exp, cite = line.rstrip("\n").split("\t")
            rows.append((inp, exp, cite))
    return rows
