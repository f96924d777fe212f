// scan.cuh -- per-record scanner: bytes -> (sign, w, q, truncation flag, kind).
//
// Follows the string-parsing strategy of PAPER.md "Parsing the String"
// (L158-185) and the pseudo-code of Appendix D (L1502-1530): explicit bounds
// (never read p[L] or beyond, L167), optional sign (L169), digits with an
// optional '.', at least one digit (L171), running significand w = 10w + d
// over at most 19 significant digits -- leading zeros, including "0.000", do
// not count (L181) -- then an optional exponent with saturation (L179), then
// terminators only.  The number of fraction
// digits and of dropped digits fold into the decimal exponent q, so that the
// record's value is w * 10^q exactly when tnz == false and lies in
// [w * 10^q, (w+1) * 10^q) otherwise.
#pragma once
#include "common.cuh"

namespace fpp {

struct Scan {
  uint64_t w;    // first <= 19 significant digits
  int32_t q;     // decimal exponent of w (clamped to +-2^30; |q| > 400 decides 0 / inf)
  int32_t kind;  // K_NUM / K_INF / K_NAN / K_INVALID / K_EMPTY
  bool neg;
  bool tnz;      // a nonzero digit was dropped beyond the 19th significant digit
};

__device__ __forceinline__ uint32_t lower(uint32_t c) { return c | 0x20u; }

// specials "inf" / "infinity" / "nan" (ASCII case-insensitive), then terminators
__device__ __noinline__ Scan scan_special(const uint8_t* p, uint32_t i, uint32_t L, Scan s) {
  uint32_t rem = L - i;
  uint32_t j = i;
  int kind = K_INVALID;
  if (rem >= 3 && lower(p[i]) == 'i' && lower(p[i + 1]) == 'n' && lower(p[i + 2]) == 'f') {
    kind = K_INF;
    j = i + 3;
    if (rem >= 8 && lower(p[i + 3]) == 'i' && lower(p[i + 4]) == 'n' && lower(p[i + 5]) == 'i' &&
        lower(p[i + 6]) == 't' && lower(p[i + 7]) == 'y')
      j = i + 8;
  } else if (rem >= 3 && lower(p[i]) == 'n' && lower(p[i + 1]) == 'a' && lower(p[i + 2]) == 'n') {
    kind = K_NAN;
    j = i + 3;
  }
  for (; j < L; j++)
    if (!is_term(p[j])) kind = K_INVALID;
  s.kind = kind;
  return s;
}

__device__ __forceinline__ uint32_t hexval(uint32_t c) {  // 16 if not a hex digit
  if (c - '0' < 10u) return c - '0';
  const uint32_t l = lower(c);
  return l - 'a' < 6u ? l - 'a' + 10 : 16u;
}

// C99 hexadecimal float after its "0x" (grammar option G_HEX, PAPER.md
// L1486-1497): w = the first 16 significant nibbles, q = binary exponent of
// w's last bit, tnz = a nonzero nibble was dropped (reading H1: a hex point
// divides by 16 per fraction nibble; H2: the 'p' exponent is optional).
__device__ __noinline__ Scan scan_hex(const uint8_t* p, uint32_t i, uint32_t L, Scan s) {
  uint64_t w = 0;
  int nsig = 0, nint = 0, nfrac = 0;
  int64_t dropped = 0;
  bool tnz = false;
  for (; i < L && hexval(p[i]) < 16u; i++, nint++) {
    const uint32_t d = hexval(p[i]);
    if (nsig < 16) { w = (w << 4) | d; nsig += (w != 0); }
    else { dropped++; tnz |= (d != 0); }
  }
  if (i < L && p[i] == '.') {
    for (i++; i < L && hexval(p[i]) < 16u; i++, nfrac++) {
      const uint32_t d = hexval(p[i]);
      if (nsig < 16) { w = (w << 4) | d; nsig += (w != 0); }
      else { dropped++; tnz |= (d != 0); }
    }
  }
  if (nint == 0 && nfrac == 0) return s;  // INVALID: no hex digit
  int64_t e = 0;
  if (i < L && lower(p[i]) == 'p') {
    i++;
    bool en = false;
    if (i < L && (p[i] == '+' || p[i] == '-')) { en = (p[i] == '-'); i++; }
    const uint32_t eb = i;
    for (; i < L && is_digit(p[i]); i++)
      if (e < (1ll << 40)) e = e * 10 + (p[i] - '0');  // saturation (reading G9)
    if (i == eb) return s;  // INVALID: exponent without digits
    if (en) e = -e;
  }
  for (; i < L; i++)
    if (!is_term(p[i])) return s;
  // nibbles after the 16 kept ones: dropped, 4 bits each; fraction nibbles: -4 each
  int64_t q = e - 4 * (int64_t)nfrac + 4 * dropped;
  q = q < -(1ll << 30) ? -(1ll << 30) : (q > (1ll << 30) ? (1ll << 30) : q);
  s.w = w;
  s.q = (int32_t)q;
  s.tnz = tnz;
  s.kind = K_HEX;
  return s;
}

// grammar: 0, or G_HEX / G_JSON (common.cuh)
__device__ __forceinline__ Scan scan_record(const uint8_t* __restrict__ p, uint32_t L, uint32_t grammar = 0) {
  Scan s;
  s.w = 0;
  s.q = 0;
  s.kind = K_INVALID;
  s.neg = false;
  s.tnz = false;
  if (L == 0) { s.kind = K_EMPTY; return s; }
  uint32_t c = p[0];
  uint32_t i = 0;
  if (is_term(c)) {  // EMPTY iff terminator bytes only
    for (i = 1; i < L; i++)
      if (!is_term(p[i])) return s;
    s.kind = K_EMPTY;
    return s;
  }
  const bool json = (grammar & G_JSON) != 0;
  if (c == '-' || (c == '+' && !json)) { s.neg = (c == '-'); i = 1; }
  if (i < L && !json) {
    uint32_t lc = lower(p[i]);
    if (lc == 'i' || lc == 'n') return scan_special(p, i, L, s);
    if ((grammar & G_HEX) && p[i] == '0' && i + 1 < L && lower(p[i + 1]) == 'x') return scan_hex(p, i + 2, L, s);
  }
  uint64_t w = 0;
  int nsig = 0;
  int64_t dropped = 0;
  bool tnz = false;
  const uint32_t ib = i;
  while (i < L && is_digit(p[i])) {
    uint32_t d = p[i] - '0';
    if (nsig < 19) { w = w * 10 + d; nsig += (w != 0); }
    else { dropped++; tnz |= (d != 0); }
    i++;
  }
  const uint32_t nint = i - ib;
  uint32_t nfrac = 0;
  bool dot = false;
  if (i < L && p[i] == '.') {
    dot = true;
    i++;
    const uint32_t fb = i;
    while (i < L && is_digit(p[i])) {
      uint32_t d = p[i] - '0';
      if (nsig < 19) { w = w * 10 + d; nsig += (w != 0); }
      else { dropped++; tnz |= (d != 0); }
      i++;
    }
    nfrac = i - fb;
  }
  if (nint == 0 && nfrac == 0) return s;  // INVALID: no digit
  // JSON: int := '0' | [1-9] digit*, frac := '.' digit+ 
  if (json && (nint == 0 || (nint > 1 && p[ib] == '0') || (dot && nfrac == 0))) return s;
  int64_t e = 0;
  if (i < L && lower(p[i]) == 'e') {
    i++;
    bool en = false;
    if (i < L && (p[i] == '+' || p[i] == '-')) { en = (p[i] == '-'); i++; }
    const uint32_t eb = i;
    while (i < L && is_digit(p[i])) {
      if (e < (1ll << 40)) e = e * 10 + (p[i] - '0');  // saturation (reading G9)
      i++;
    }
    if (i == eb) return s;  // INVALID: exponent without digits (reading G7)
    if (en) e = -e;
  }
  for (; i < L; i++)
    if (!is_term(p[i])) return s;  // INVALID: trailing garbage
  int64_t q = e - (int64_t)nfrac + dropped;
  q = q < -(1ll << 30) ? -(1ll << 30) : (q > (1ll << 30) ? (1ll << 30) : q);
  s.w = w;
  s.q = (int32_t)q;
  s.tnz = tnz;
  s.kind = K_NUM;
  return s;
}

}  // namespace fpp
