"""Exact correctly rounded decimal -> binary64 (test infrastructure only).

This is the plain definition of what arXiv 2101.11408 computes: "the nearest
binary floating-point value" to a decimal number, ties to even
(notation table: "round(x) is an integer value nearest
to x, with ties broken by rounding to the nearest even integer").  The paper's
Algorithm 1 (L223-260) plus its long-number bracket and exact fallback
(L968-987) reach exactly this result, only faster.

Binary64 facts used (table tab:commmonieee L123-135):
normal values m*2^e with m in [2^52, 2^53), unbiased exponent e+52 in
[-1022, 1023], bias 1023; subnormals m*2^-1074 with m in [0, 2^52); values at
or beyond the midpoint 2^1024 - 2^970 round to infinity (IEEE; G12).

Everything is Python integer arithmetic; no float is used anywhere.
Steps follow SURVEY.md 8(c) 2-7 (the plain definition written out).
"""

STATUS_OK = 0
STATUS_OVERFLOW = 1
STATUS_UNDERFLOW = 2
STATUS_INVALID = 3
STATUS_EMPTY = 4

QNAN_BITS = 0x7FF8000000000000
INF_BITS = 0x7FF0000000000000
SIGN_BIT = 1 << 63

_TWO52 = 1 << 52
_TWO53 = 1 << 53


def int_of_digits(s):
    """int(s) for a decimal digit string of any length (CPython limits int(str)
    to 4300 digits; fold 4000-digit chunks instead: plain Horner in base 10^4000)."""
    if len(s) <= 4000:
        return int(s)
    v = 0
    for i in range(0, len(s), 4000):
        part = s[i:i + 4000]
        v = v * 10 ** len(part) + int(part)
    return v


def floor_log2_ratio(N, D):
    """floor(log2(N/D)) for positive integers N, D, exactly.

    N/D lies in [2^(t-1), 2^(t+1)) with t = bitlen(N) - bitlen(D); one
    comparison decides which of t, t-1 it is.
    """
    t = N.bit_length() - D.bit_length()
    if t >= 0:
        ge = N >= (D << t)
    else:
        ge = (N << (-t)) >= D
    return t if ge else t - 1


def round_decimal(neg, digits, Q):
    """Nearest binary64 to (-1)^neg * int(digits) * 10^Q, ties to even.

    digits: str of ASCII decimal digits (may have leading/trailing zeros, may be
    empty); Q: int (unbounded).  Returns (bits, status).

    status: OK, OVERFLOW (finite decimal rounds to +-inf), UNDERFLOW (nonzero
    decimal rounds to +-0).  Subnormal results are OK (G11).
    """
    sign = SIGN_BIT if neg else 0
    # Step 2 (zero): strip leading zeros; no significant digit -> +-0.
    s = digits.lstrip("0")
    if not s:
        return sign, STATUS_OK
    # Step 3 (cheap range decisions): strip trailing zeros into Q.
    t = s.rstrip("0")
    Q = Q + (len(s) - len(t))
    k = len(t)
    # x >= 10^(Q+k-1) >= 10^309 > 2^1024  -> infinity
    if Q + k - 1 >= 309:
        return sign | INF_BITS, STATUS_OVERFLOW
    # x < 10^(Q+k) <= 10^-325 < 2^-1075 (half the smallest subnormal) -> zero
    if Q + k <= -325:
        return sign, STATUS_UNDERFLOW
    # Step 4 (exact rational): x = N / D
    c = int_of_digits(t)
    if Q >= 0:
        N, D = c * 10 ** Q, 1
    else:
        N, D = c, 10 ** (-Q)
    # Step 5 (scale): e = max(floor(log2 x) - 52, -1074); m = floor(x / 2^e)
    e = max(floor_log2_ratio(N, D) - 52, -1074)
    if e <= 0:
        num, den = N << (-e), D
    else:
        num, den = N, D << e
    m, rem = divmod(num, den)
    # Step 6 (midpoint comparison): x vs (m + 1/2) * 2^e  <=>  2*rem vs den
    twice = 2 * rem
    if twice > den or (twice == den and (m & 1)):
        m += 1
    # Step 7 (finish)
    if m == _TWO53:
        m = _TWO52
        e += 1
    if m >= _TWO52 and e + 52 > 1023:
        return sign | INF_BITS, STATUS_OVERFLOW
    if m == 0:
        return sign, STATUS_UNDERFLOW
    if m < _TWO52:
        # subnormal (here e == -1074): biased exponent field 0
        return sign | m, STATUS_OK
    return sign | ((e + 1075) << 52) | (m - _TWO52), STATUS_OK


# ----------------------------------------------------------------------------
# binary32.  Binary32 facts (table
# tab:commmonieee L123-135): normal values m*2^e with m in [2^23, 2^24),
# unbiased exponent e+23 in [-126, 127], bias 127; subnormals m*2^-149 with m
# in [0, 2^23); values at or beyond the midpoint 2^128 - 2^103 round to
# infinity (IEEE, as G12 for binary64).  The same plain definition as
# round_decimal, written out again with these constants: the result is
# rounded once, from the exact decimal, never through binary64 (no
# double rounding).

QNAN32_BITS = 0x7FC00000
INF32_BITS = 0x7F800000
SIGN32_BIT = 1 << 31

_TWO23 = 1 << 23
_TWO24 = 1 << 24


def round_decimal32(neg, digits, Q):
    """Nearest binary32 to (-1)^neg * int(digits) * 10^Q, ties to even.

    Same arguments and status codes as round_decimal; returns (bits, status)
    with 32-bit IEEE bits.
    """
    sign = SIGN32_BIT if neg else 0
    s = digits.lstrip("0")
    if not s:
        return sign, STATUS_OK
    t = s.rstrip("0")
    Q = Q + (len(s) - len(t))
    k = len(t)
    # x >= 10^(Q+k-1) >= 10^39 > 2^128  -> infinity
    if Q + k - 1 >= 39:
        return sign | INF32_BITS, STATUS_OVERFLOW
    # x < 10^(Q+k) <= 10^-46 < 2^-150 (half the smallest subnormal) -> zero
    if Q + k <= -46:
        return sign, STATUS_UNDERFLOW
    c = int_of_digits(t)
    if Q >= 0:
        N, D = c * 10 ** Q, 1
    else:
        N, D = c, 10 ** (-Q)
    # e = max(floor(log2 x) - 23, -149); m = floor(x / 2^e)
    e = max(floor_log2_ratio(N, D) - 23, -149)
    if e <= 0:
        num, den = N << (-e), D
    else:
        num, den = N, D << e
    m, rem = divmod(num, den)
    twice = 2 * rem
    if twice > den or (twice == den and (m & 1)):
        m += 1
    if m == _TWO24:
        m = _TWO23
        e += 1
    if m >= _TWO23 and e + 23 > 127:
        return sign | INF32_BITS, STATUS_OVERFLOW
    if m == 0:
        return sign, STATUS_UNDERFLOW
    if m < _TWO23:
        return sign | m, STATUS_OK
    return sign | ((e + 150) << 23) | (m - _TWO23), STATUS_OK


# ----------------------------------------------------------------------------
# hexadecimal floats: the value
# c * 2^E2 is a dyadic rational; its nearest binary64 / binary32 follows the
# same plain definition (exact scale, compare with the midpoint, ties to even).

def _round_dyadic(neg, c, E2, prec, emin, emax, inf_bits, sign_bit):
    """Nearest value with prec-bit significands, exponents [emin, emax] (of the
    leading bit), subnormals, to (-1)^neg * c * 2^E2; (bits, status)."""
    sign = sign_bit if neg else 0
    if c == 0:
        return sign, STATUS_OK
    # floor(log2 x) = bitlen(c) - 1 + E2 exactly
    lg = c.bit_length() - 1 + E2
    # cheap range decisions (as steps 3 of round_decimal; E2 is unbounded,
    # reading G9): x < 2^(lg+1) <= 2^(emin-prec), half the smallest subnormal,
    # rounds to zero; x >= 2^lg >= 2^(emax+1) is beyond every finite value
    if lg <= emin - prec - 1:
        return sign, STATUS_UNDERFLOW
    if lg >= emax + 1:
        return sign | inf_bits, STATUS_OVERFLOW
    e = max(lg - (prec - 1), emin - (prec - 1))   # weight of the last significand bit
    if e <= E2:
        m, rem2, den2 = c << (E2 - e), 0, 1
    else:
        sh = e - E2
        m, r = c >> sh, c & ((1 << sh) - 1)
        rem2, den2 = 2 * r, 1 << sh
    if rem2 > den2 or (rem2 == den2 and (m & 1)):
        m += 1
    if m == 1 << prec:
        m >>= 1
        e += 1
    if m >= 1 << (prec - 1) and e + prec - 1 > emax:
        return sign | inf_bits, STATUS_OVERFLOW
    if m == 0:
        return sign, STATUS_UNDERFLOW
    if m < 1 << (prec - 1):
        return sign | m, STATUS_OK   # subnormal
    bias = emax
    return sign | ((e + prec - 1 + bias) << (prec - 1)) | (m - (1 << (prec - 1))), STATUS_OK


def round_hex(neg, hexdigits, E2):
    """Nearest binary64 to (-1)^neg * int(hexdigits, 16) * 2^E2, ties to even."""
    return _round_dyadic(neg, int(hexdigits, 16) if hexdigits else 0, E2, 53, -1022, 1023, INF_BITS, SIGN_BIT)


def round_hex32(neg, hexdigits, E2):
    """Nearest binary32 to (-1)^neg * int(hexdigits, 16) * 2^E2, ties to even."""
    return _round_dyadic(neg, int(hexdigits, 16) if hexdigits else 0, E2, 24, -126, 127, INF32_BITS, SIGN32_BIT)
