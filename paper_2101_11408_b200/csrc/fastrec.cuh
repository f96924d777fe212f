// fastrec.cuh -- the fast kernels' common-case record parser: few
// instructions, few branches.
//
// Covers the records that make up the paper's workloads (PAPER.md L1018-1024:
// random numbers printed with 17 digits, coordinates, scientific notation):
//
//     [sign] d{0,4} ['.' d*] [(e|E) [sign] d{1,4}]     at most 30 bytes,
//
// at least one digit, and at most 19 significant digits -- or, after an
// integer part of zeros, a fraction of up to 20 digits whose first is a zero
// ("0.000ddd..": %.17g of values below 0.001).  Anything else returns
// false and goes to the general scanner (fastscan.cuh / scan.cuh), which
// accepts the whole grammar.  On this subset the significand is exact, so the
// result is Algorithm 1 on (w, q) with no w/w+1 bracket.
//
// Structure comes from the tile's non-digit mask word (one bit per byte):
// the integer run ends at the first non-digit after the sign, the fraction run
// at the next one, and the exponent must end exactly at the record's end.
// Digits are converted 4 per 32-bit word with dp2a (fastscan.cuh), read from
// the END of each run with '0' fill, so no lane diverges on the digit count.
//
// Algorithm 1 runs straight through for the common case -- w != 0, q inside
// the table, a normal result, no abort -- and every other case (zero, q out
// of range, subnormal, possible overflow, the abort of line 6) is sent by one
// branch to the general decision (decide.cuh), which recomputes it.  The
// rounded significand m (implicit bit included) is added to (p + 1022) << 52,
// so a rounding carry into the exponent (Algorithm 1 line 20, reading L20 in
// DESIGN.md) falls out of the addition.  Only the second multiplication
// (~0.6% of records) and the tie test (q in [-4, 23],
// L287-333) sit behind branches of their own.
#pragma once
#include "decide.cuh"
#include "fastscan.cuh"

namespace fpp {

#ifndef FPP_CLINGER
#define FPP_CLINGER 0  // 1: Clinger's fast path first, 2: the same after a warp vote (SURVEY 8(f) f3 ablation)
#endif

// Clinger's fast path: for w <= 2^53 and
// |q| <= 22 (binary32: w <= 2^24, |q| <= 10) both w and 10^|q| are exact
// floating-point values, so one correctly rounded IEEE multiplication or
// division gives the nearest value.  Returns false outside that range.
__device__ const double kClingerP10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                           1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
template <bool F32>
__device__ __forceinline__ bool clinger(uint64_t w, int q, uint64_t& bits) {
  if (F32) {
    if (w > (1ull << 24) || (uint32_t)(q + 10) > 20u) return false;
    const float p = (float)__ldg(&kClingerP10[q < 0 ? -q : q]);  // exact for |q| <= 10
    const float x = (float)(uint32_t)w;                          // exact for w <= 2^24
    bits = (uint32_t)__float_as_uint(q < 0 ? __fdiv_rn(x, p) : __fmul_rn(x, p));
  } else {
    if (w > (1ull << 53) || (uint32_t)(q + 22) > 44u) return false;
    const double p = __ldg(&kClingerP10[q < 0 ? -q : q]);
    const double x = __ull2double_rn(w);  // exact for w <= 2^53
    bits = (uint64_t)__double_as_longlong(q < 0 ? __ddiv_rn(x, p) : __dmul_rn(x, p));
  }
  return true;
}

// position of the lowest set bit (32 when x == 0)
__device__ __forceinline__ uint32_t low_bit(uint32_t x) { return __clz(__brev(x)); }
// the same for x != 0 (BREV + FLO.SH; 0xFFFFFFFF when x == 0): callers
// guarantee a set bit, or reject the result
__device__ __forceinline__ uint32_t ctz_nz(uint32_t x) {
  uint32_t r;
  asm("{\n .reg .b32 t;\n brev.b32 t, %1;\n bfind.shiftamt.u32 %0, t;\n}" : "=r"(r) : "r"(x));
  return r;
}
// value of 4 bytes holding digit values 0..9 (byte 0 most significant)
__device__ __forceinline__ uint32_t dig4v(uint32_t v) {
  const int t = dp2a_hi(0x0001000A, (int)v, 0);   // 10 b2 + b3
  return (uint32_t)dp2a_lo(0x006403E8, (int)v, t);  // + 1000 b0 + 100 b1
}
// the last k of a word's 4 ASCII bytes as digit values, the others 0, for
// k in [0, 4]; k > 4 is treated as 0 (s = 8 (4 - k) > 32 clamps)
__device__ __forceinline__ uint32_t last_digits(uint32_t x, uint32_t k) {
  const uint32_t keep = __funnelshift_lc(0u, 0xFFFFFFFFu, 32u - 8u * k);
  return (x ^ 0x30303030u) & keep;
}

// T[q] for q clamped to the table range (qc); q != qc is rare
__device__ __forceinline__ ulonglong2 pow5_entry(int q, int& qc) {
  qc = min(max(q, -342), 308);
  return __ldg(reinterpret_cast<const ulonglong2*>(&kPow5_128[2 * (qc + 342)]));
}

// Algorithm 1 on (w, q) for the common case: w != 0, q in the table range,
// a normal result (no overflow) and no abort.  Returns false (any result
// left undefined) when the case is not common; the caller then runs the
// general decision (decide.cuh).  fl gets F_TWO.
// NORANGE: the caller guarantees q == qc and a value far inside the normal
// range (fast_frac0_tile: q in [-20, 2], w < 2^64), so only w == 0 and the
// abort are rare.
template <bool F32, bool NORANGE = false>
__device__ __forceinline__ bool alg1_common(uint64_t w, int q, int qc, const ulonglong2 t, uint64_t& bits,
                                            uint32_t& fl) {
  using F = Fmt<F32>;
  constexpr uint64_t kCutMask = (1ull << F::kCut) - 1;
  // lines 3-4: normalise (w | 1 keeps clz defined; w == 0 is rare)
  const int l = __clzll((long long)(w | 1ull));
  const uint64_t wn = w << l;
  // line 5: truncated product (t = T[qc], qc = q clamped to the table, loaded
  // by the caller ahead of the digit conversion), second multiplication when
  // the high word's bits below the exact ones are all ones
  uint64_t hi = __umul64hi(wn, t.x);
  uint64_t lo = wn * t.x;
  const bool two = F32 ? ((hi & kCutMask) == kCutMask) : (((uint32_t)hi & (uint32_t)kCutMask) == (uint32_t)kCutMask);
  if (two) {
    const uint64_t add = __umul64hi(wn, t.y);
    lo += add;
    hi += (lo < add);
    fl |= F_TWO;
  }
  // lines 7-9: significand with one extra bit, binary exponent
  const int u = (int)(hi >> 63);
  uint64_t m = hi >> (u + F::kCut);
  const int p = ((217706 * qc) >> 16) + 63 - l + u;
  // rare: w == 0, q out of range, subnormal or zero (p < kEmin, G1), a
  // possible overflow (p >= kEmax), the abort of line 6 (lo all ones)
  const bool rare = (((uint32_t)(w >> 32) | (uint32_t)w) == 0u) |
                    (!NORANGE && ((q != qc) | ((uint32_t)(p - F::kEmin) >= (uint32_t)(F::kEmax - F::kEmin)))) |
                    (((uint32_t)(lo >> 32) & (uint32_t)lo) == 0xFFFFFFFFu);
  // lines 16-18: ties to even (only for q in [kTieLo, kTieHi]): lo <= 1,
  // m odd by one ((m & 3) == 1) and no bit of hi below m (G4)
  if ((uint32_t)(qc - F::kTieLo) <= (uint32_t)(F::kTieHi - F::kTieLo)) {
    bool below0;
    if (F32) below0 = (m << (u + F::kCut)) == hi;
    else below0 = ((uint32_t)hi & ((0x200u << u) - 1u)) == 0u;
    if (lo <= 1 && ((uint32_t)m & 3u) == 1u && below0) m -= 1;
  }
  // lines 19-21: round half up on the extra bit ((m + (m & 1)) >> 1 equals
  // (m + 1) >> 1); the rounded m (implicit bit included) is added to
  // (p + bias - 1) << kFracBits so that a carry out of the significand moves
  // into the exponent (reading L20)
  m = (m + 1) >> 1;
  bits = ((uint64_t)(uint32_t)(p + F::kEmax - 1) << F::kFracBits) + m;
  return !rare;
}

// Parse the record text[ts, ts+L) of the common subset (see above).  Returns
// false, leaving r untouched, when the record is outside it.  TERM: the
// record may end with one terminator byte (batch records keep their
// separator; split records never include it).  JSON: grammar option G_JSON --
// no '+', no empty integer part, no leading zero, a '.' needs fraction digits.
template <bool TERM, bool F32, bool JSON = false>
__device__ __forceinline__ bool fast_record(const uint8_t* text, uint32_t ts, uint32_t L, uint32_t ndw,
                                            const uint64_t* __restrict__ p10, Res& r) {
  if (TERM && L > 0) L -= is_term(text[ts + L - 1]) ? 1u : 0u;
  // structure: bytes at and past L count as non-digits (L < 32 below, so
  // every ctz_nz operand has a set bit)
  const uint32_t nd = ndw | __funnelshift_lc(0u, 0xFFFFFFFFu, L);
  const uint32_t c0 = text[ts];
  const bool neg = c0 == '-';
  const uint32_t p = (((c0 - '+') & ~2u) == 0u) ? 1u : 0u;   // '+' or '-'
  const uint32_t nd1 = nd & ~p;                       // sign bit cleared
  const uint32_t i1 = ctz_nz(nd1);                    // end of the integer run
  const bool dot = (text[ts + i1] == '.') && (i1 < L);
  const uint32_t nd2 = dot ? (nd1 & (nd1 - 1)) : nd1; // dot bit cleared
  const uint32_t f1 = ctz_nz(nd2);                    // end of the fraction run
  const uint32_t ni = i1 - p;
  const uint32_t nf = f1 - i1 - (dot ? 1u : 0u);
  bool ok = (L - 1u) < 30u && ni <= 4u && ni + nf != 0u;
  if (JSON) {  // RFC 8259: int := '0' | [1-9] digit*, frac := '.' digit+
    ok = ok && c0 != '+' && ni != 0u && (ni == 1u || text[ts + p] != '0') && (!dot || nf != 0u);
  }
  int32_t ex = 0;
  if (f1 < L) {  // exponent: (e|E) [sign] 1-4 digits, ending the record
    const uint32_t ce = text[ts + f1];
    const uint32_t cs = text[ts + f1 + 1];
    const bool eneg = cs == '-';
    const uint32_t es = ((((cs - '+') & ~2u) == 0u) && f1 + 1 < L) ? 1u : 0u;
    uint32_t nd3 = nd2 & (nd2 - 1);                   // 'e' bit cleared
    if (es) nd3 &= nd3 - 1;                           // exponent sign bit cleared
    const uint32_t ke = ctz_nz(nd3);
    const uint32_t ne = ke - (f1 + 1 + es);
    ok = ok && (ce | 0x20u) == 'e' && ke == L && ne - 1u < 4u;
    const int32_t ev = (int32_t)dig4v(last_digits(lds4(text, ts + ke - 4), ne));
    ex = eneg ? -ev : ev;
  }
  // the decimal exponent is known before the digits: T[q]'s load is issued
  // here so that the digit conversion hides its latency
  const int q = ex - (int)nf;
  int qc;
  const ulonglong2 t = pow5_entry(q, qc);
  // integer part: <= 4 digits, the word ending at the point
  const uint32_t I = dig4v(last_digits(lds4(text, ts + i1 - 4), ni));
  // fraction: the nf <= 20 digits ending at f1, five words read from the end
  // (bytes before the run count as 0); 20 digits only with a leading zero
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(text);
  const uint32_t E = ts + f1, a = E - 20, wi = a >> 2, sh = (a & 3) * 8;
  const uint32_t w0 = wd[wi], w1 = wd[wi + 1], w2 = wd[wi + 2], w3 = wd[wi + 3], w4 = wd[wi + 4],
                 w5 = wd[wi + 5];
  uint32_t c = __funnelshift_r(w0, w1, sh);   // [E-20, E-16)
  uint32_t b0 = __funnelshift_r(w1, w2, sh);  // [E-16, E-12)
  uint32_t b1 = __funnelshift_r(w2, w3, sh);  // [E-12, E-8)
  uint32_t a0 = __funnelshift_r(w3, w4, sh);  // [E-8, E-4)
  uint32_t a1 = __funnelshift_r(w4, w5, sh);  // [E-4, E)
  const int n = (int)nf;
  if (n < 16) {  // 17-digit printing fills only the top word
    a1 = fill_word(a1, 4 - n);
    a0 = fill_word(a0, 8 - n);
    b1 = fill_word(b1, 12 - n);
    b0 = fill_word(b0, 16 - n);
  }
  const uint32_t C = dig4v(last_digits(c, nf - 16u));  // nf < 16: no digit (the shift clamps)
  const uint32_t A = dig4(a0) * 10000u + dig4(a1);
  const uint32_t B = dig4(b0) * 10000u + dig4(b1);
  // exact significand: <= 19 digits in all, or an integer part of zeros and
  // a fraction of <= 20 digits whose value is below 10^19
  ok = ok && nf <= 20u && C < 1000u && (ni + nf <= 19u || I == 0u);
  if (!ok) return false;
  uint64_t w = ((uint64_t)C * 100000000ull + B) * 100000000ull + A;
  if (I != 0) w += (uint64_t)I * p10[min(nf, 19u)];  // "0.ddd": skipped
  uint64_t bits;
  uint32_t fl = 0;
#if FPP_CLINGER == 2
  // warp vote: Clinger only when every active lane's record is eligible, so
  // the FP64 path never diverges from the integer one
  const bool elig = F32 ? (w <= (1ull << 24) && (uint32_t)(q + 10) <= 20u)
                        : (w <= (1ull << 53) && (uint32_t)(q + 22) <= 44u);
  if (__all_sync(__activemask(), elig)) {
    clinger<F32>(w, q, bits);
    r.bits = bits | (neg ? Fmt<F32>::kSign : 0ull);
    r.info = ST_OK;
    return true;
  }
#elif FPP_CLINGER
  if (clinger<F32>(w, q, bits)) {
    r.bits = bits | (neg ? Fmt<F32>::kSign : 0ull);
    r.info = ST_OK;  // |q| <= 22: never overflows or underflows; w == 0 gives +-0
    return true;
  }
#endif
  if (!alg1_common<F32>(w, q, qc, t, bits, fl)) {
    r = decide_num_ni<F32>(w, q, neg);  // zero, range, subnormal, overflow, abort (out of line)
    r.info |= fl & F_TWO;
    return true;
  }
  r.bits = bits | (neg ? Fmt<F32>::kSign : 0ull);
  r.info = fl;
  return true;
}

// The "0.ddd" shape: an integer part "0", the point, and 1-20 fraction digits
// ending the record (%.17g of values in [1e-4, 1): config 2).  The caller has
// checked the shape (frac0_shape) for every lane of the warp, so the structure
// needs no search and the integer part no conversion; the digits and
// Algorithm 1 are fast_record's.  False: not exact in 19 digits (20 digits
// without a leading zero), the caller takes the general path.
__device__ __forceinline__ bool frac0_shape(const uint8_t* text, uint32_t ts, uint32_t L, uint32_t ndw) {
  return (L - 3u <= 19u) && text[ts] == '0' && text[ts + 1] == '.' && (ndw & ((1u << L) - 1u)) == 2u;
}
template <bool F32>
__device__ __forceinline__ bool fast_frac0(const uint8_t* text, uint32_t ts, uint32_t L, Res& r) {
  const uint32_t nf = L - 2;
  const int q = -(int)nf;
  int qc;
  const ulonglong2 t = pow5_entry(q, qc);
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(text);
  const uint32_t E = ts + L, a = E - 20, wi = a >> 2, sh = (a & 3) * 8;
  const uint32_t w0 = wd[wi], w1 = wd[wi + 1], w2 = wd[wi + 2], w3 = wd[wi + 3], w4 = wd[wi + 4],
                 w5 = wd[wi + 5];
  uint32_t c = __funnelshift_r(w0, w1, sh);
  uint32_t b0 = __funnelshift_r(w1, w2, sh);
  uint32_t b1 = __funnelshift_r(w2, w3, sh);
  uint32_t a0 = __funnelshift_r(w3, w4, sh);
  uint32_t a1 = __funnelshift_r(w4, w5, sh);
  const int n = (int)nf;
  if (n < 16) {
    a1 = fill_word(a1, 4 - n);
    a0 = fill_word(a0, 8 - n);
    b1 = fill_word(b1, 12 - n);
    b0 = fill_word(b0, 16 - n);
  }
  const uint32_t C = dig4v(last_digits(c, nf - 16u));
  const uint32_t A = dig4(a0) * 10000u + dig4(a1);
  const uint32_t B = dig4(b0) * 10000u + dig4(b1);
  // no early exit before Algorithm 1: an exit here lets the compiler sink
  // T[q]'s load past it, next to its use (exposed L1 latency)
  const bool ok = C < 1000u;  // else 20 digits without a leading zero: not exact
  const uint64_t w = ((uint64_t)C * 100000000ull + B) * 100000000ull + A;
  uint64_t bits;
  uint32_t fl = 0;
  if (!alg1_common<F32>(w, q, qc, t, bits, fl) && ok) {
    r = decide_num_ni<F32>(w, q, false);  // zero, subnormal, abort (out of line)
    r.info |= fl & F_TWO;
    return true;
  }
  r.bits = bits;
  r.info = fl;
  return ok;
}

// The same for a tile whose non-digit mask has been checked as a whole
// (k_split: every non-digit byte of the tile is a separator or the byte after
// a record start), so that a record of L >= 3 bytes is d X d* with X a
// non-digit: the shape needs only the two bytes "0." and the length, with no
// branch before the digit loads and no mask word.  L is clamped for the
// addresses (a record that runs past the window has a huge L).
#ifndef FPP_F0_FILL
#define FPP_F0_FILL 3  // 3: the rare fill out of line (a real branch); 1: inline (the compiler predicates it)
#endif
#ifndef FPP_F0_NORANGE
#define FPP_F0_NORANGE 1  // 1: Algorithm 1 without the range tests (q in [-20, 2] is always normal)
#endif
// '0' fill of the four low fraction words of a run of n < 16 digits, out of line
__device__ __noinline__ uint4 fill4_ni(uint4 x, int n) {
  return make_uint4(fill_word(x.x, 16 - n), fill_word(x.y, 12 - n), fill_word(x.z, 8 - n), fill_word(x.w, 4 - n));
}
template <bool F32>
__device__ __forceinline__ bool fast_frac0_tile(const uint8_t* text, uint32_t ts, uint32_t L, Res& r) {
  const uint32_t c0 = text[ts], c1 = text[ts + 1];
  const uint32_t Lc = min(L, 22u);
  const uint32_t nf = Lc - 2;
  const int q = 2 - (int)Lc;
  int qc;
  const ulonglong2 t = pow5_entry(q, qc);
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(text);
  const uint32_t E = ts + Lc, a = E - 20, wi = a >> 2, sh = (a & 3) * 8;
  const uint32_t w0 = wd[wi], w1 = wd[wi + 1], w2 = wd[wi + 2], w3 = wd[wi + 3], w4 = wd[wi + 4],
                 w5 = wd[wi + 5];
  uint32_t c = __funnelshift_r(w0, w1, sh);
  uint32_t b0 = __funnelshift_r(w1, w2, sh);
  uint32_t b1 = __funnelshift_r(w2, w3, sh);
  uint32_t a0 = __funnelshift_r(w3, w4, sh);
  uint32_t a1 = __funnelshift_r(w4, w5, sh);
  const int n = (int)nf;
#if FPP_F0_FILL == 3
  // a call keeps the rare fill behind a real branch (the compiler predicates
  // the inline form: 16 issue slots in every round)
  if (n < 16) {
    const uint4 f = fill4_ni(make_uint4(b0, b1, a0, a1), n);
    b0 = f.x;
    b1 = f.y;
    a0 = f.z;
    a1 = f.w;
  }
#else
  if (n < 16) {
    a1 = fill_word(a1, 4 - n);
    a0 = fill_word(a0, 8 - n);
    b1 = fill_word(b1, 12 - n);
    b0 = fill_word(b0, 16 - n);
  }
#endif
  const uint32_t C = dig4v(last_digits(c, nf - 16u));
  const uint32_t A = dig4(a0) * 10000u + dig4(a1);
  const uint32_t B = dig4(b0) * 10000u + dig4(b1);
  // C >= 1000: 20 digits without a leading zero, not exact in 64 bits
  const bool ok = (L - 3u <= 19u) & (c0 == '0') & (c1 == '.') & (C < 1000u);
  const uint64_t w = ((uint64_t)C * 100000000ull + B) * 100000000ull + A;
  uint64_t bits;
  uint32_t fl = 0;
  if (!alg1_common<F32, FPP_F0_NORANGE != 0>(w, q, qc, t, bits, fl) && ok) {
    r = decide_num_ni<F32>(w, q, false);  // zero, subnormal, abort (out of line)
    r.info |= fl & F_TWO;
    return true;
  }
  r.bits = bits;
  r.info = fl;
  return ok;
}

// --------------------------------------------------------------------------
// Hexadecimal floats (grammar option G_HEX): the common
// shapes [sign] 0x H [. F{0,15}] [p [sign] d{1,4}] and [sign] 0x H{1,16}
// [p [sign] d{1,4}] in at most 30 bytes, by SWAR: the run of nibbles is read
// as four words from its end ('0' fill), checked to be hex digits, turned into
// nibble values ((b & 15) + 9 * bit 6) and packed four per word with two dp2a
// (weights 4096, 256 / 16, 1).  The structure comes from the tile's
// non-decimal-digit mask: the exponent is the decimal run after the last
// non-digit.  The value w * 2^E2 is then rounded exactly (round_hex).

// flags (bit 7 of each byte) of bytes that are hex digits
__device__ __forceinline__ uint32_t hexdigit80(uint32_t w) {
  const uint32_t dig = ~nondigit80(w) & 0x80808080u;
  const uint32_t x = (w | 0x20202020u) & 0x7F7F7F7Fu;  // lower case, bit 7 clear
  const uint32_t ge_a = (x + 0x1F1F1F1Fu) & 0x80808080u;  // >= 'a'
  const uint32_t ge_g = (x + 0x19191919u) & 0x80808080u;  // >= 'g'
  return dig | (ge_a & ~ge_g & ~w);
}
// value of 4 hex digit bytes, first byte most significant
__device__ __forceinline__ uint32_t nib4(uint32_t w) {
  const uint32_t v = (w & 0x0F0F0F0Fu) + 9u * ((w >> 6) & 0x01010101u);
  const int t = dp2a_hi(0x00010010, (int)v, 0);    // 16 b2 + b3
  return (uint32_t)dp2a_lo(0x01001000, (int)v, t);  // + 4096 b0 + 256 b1
}

// false: not a common-shape hex float (the byte scanner decides it)
template <bool F32>
__device__ __forceinline__ bool fast_hex(const uint8_t* text, uint32_t ts, uint32_t L, uint32_t ndw, Res& r) {
  if (L > 0 && is_term(text[ts + L - 1])) L--;  // one trailing terminator (batch records)
  if (L - 3u > 27u) return false;               // 3 <= L <= 30
  const uint32_t c0 = text[ts];
  const uint32_t p = (((c0 - '+') & ~2u) == 0u) ? 1u : 0u;
  if (text[ts + p] != '0' || (text[ts + p + 1] | 0x20u) != 'x') return false;
  const uint32_t m0 = p + 2;  // first mantissa byte
  // exponent: the decimal digits after the last non-digit byte
  const uint32_t nd = ndw & ((1u << L) - 1u);
  const uint32_t k = 31u - __clz(nd);  // last non-digit (the 'x' at least)
  uint32_t pp = L;                     // end of the mantissa
  int32_t ex = 0;
  const uint32_t bk = text[ts + k];
  if (k + 1 < L && k >= m0) {  // decimal digits follow a non-digit of the mantissa region
    const bool sgn = bk == '+' || bk == '-';
    const uint32_t kp = sgn ? k - 1 : k;  // k >= m0 >= 2
    if ((text[ts + kp] | 0x20u) == 'p') {
      const uint32_t ne = L - k - 1;
      if (ne > 4u) return false;
      ex = (int32_t)dig4(fill_word(lds4(text, ts + L - 4), 4 - (int)ne));
      if (bk == '-') ex = -ex;
      pp = kp;
    } else if (sgn) {
      return false;  // a sign not after 'p'
    }
    // else: no exponent; the trailing decimal digits are mantissa nibbles
  } else if ((bk | 0x20u) == 'p') {
    return false;  // 'p' without digits
  }
  if (pp <= m0) return false;
  // shape A (a point after one nibble) or B (no point)
  const bool dot = pp > m0 + 1 && text[ts + m0 + 1] == '.';
  const uint32_t rb = dot ? m0 + 2 : m0;  // the run converted below: [rb, pp)
  const uint32_t n = pp - rb;
  if (n > (dot ? 15u : 16u) || (!dot && n == 0)) return false;
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(text);
  const uint32_t E = ts + pp, a = E - 16, wi = a >> 2, sh = (a & 3) * 8;
  const uint32_t w0 = wd[wi], w1 = wd[wi + 1], w2 = wd[wi + 2], w3 = wd[wi + 3], w4 = wd[wi + 4];
  uint32_t x0 = fill_word(__funnelshift_r(w0, w1, sh), 16 - (int)n);
  uint32_t x1 = fill_word(__funnelshift_r(w1, w2, sh), 12 - (int)n);
  uint32_t x2 = fill_word(__funnelshift_r(w2, w3, sh), 8 - (int)n);
  uint32_t x3 = fill_word(__funnelshift_r(w3, w4, sh), 4 - (int)n);
  if ((hexdigit80(x0) & hexdigit80(x1) & hexdigit80(x2) & hexdigit80(x3)) != 0x80808080u) return false;
  uint64_t w = ((uint64_t)((nib4(x0) << 16) | nib4(x1)) << 32) | ((nib4(x2) << 16) | nib4(x3));
  int E2 = ex;
  if (dot) {
    const uint32_t h = hexval(text[ts + m0]);
    if (h > 15u) return false;
    w |= (n < 16 ? (uint64_t)h << (4 * n) : 0ull);
    E2 -= 4 * (int)n;
  }
  uint32_t fl = 0;
  r.bits = round_hex<F32>(w, E2, false, fl) | ((c0 == '-') ? Fmt<F32>::kSign : 0ull);
  r.info = fl;
  return true;
}

// the general path for records fast_record() declines, out of line
// (grammar options other than the default: the byte scanner alone)
template <bool F32>
__device__ __noinline__ Res parse_general(const uint8_t* text, uint32_t ts, uint32_t L, uint32_t ndw,
                                          const uint64_t* p10, uint32_t grammar) {
  if (grammar & G_HEX) {
    Res r;
    if (fast_hex<F32>(text, ts, L, ndw, r)) return r;
  }
  if (grammar != 0) return decide<F32>(scan_record(text + ts, L, grammar));
  // plain integers of 5-19 digits (the paper's "integer" dataset, L1024):
  // one run conversion, q = 0
  const uint32_t nd = ndw | __funnelshift_lc(0u, 0xFFFFFFFFu, L);
  if (L - 5u < 15u && (nd & ((1u << L) - 1u)) == 0u) return decide_num<F32>(run19(text, ts + L, (int)L), 0, false);
  // plain integers of 20-64 digits without a leading zero (the paper's "many
  // digits", L1290): w = the first 19 digits, q = L - 19, and the truncation
  // flag from a SWAR scan of the rest; Algorithm 1 with the w / w+1 bracket
  // (L968-983) decides, else the slow kernel
  if (L - 20u <= 44u && (ndw & (L >= 32u ? 0xFFFFFFFFu : ((1u << L) - 1u))) == 0u && text[ts] != '0') {
    uint32_t nondig = 0, nz = 0;
    for (uint32_t k = 32; k < L; k += 4) {  // bytes [32, L) (the mask word covered [0, 32)): digits?
      uint32_t x = lds4(text, ts + k);
      if (L - k < 4) {  // bytes past L count as digits
        const uint32_t keep = 0xFFFFFFFFu >> (8 * (4 - (L - k)));
        x = (x & keep) | (0x30303030u & ~keep);
      }
      nondig |= nondigit80(x);
    }
    if (nondig == 0) {
      for (uint32_t k = 19; k < L; k += 4) {  // a nonzero digit after the 19th?
        uint32_t x = lds4(text, ts + k) ^ 0x30303030u;
        if (L - k < 4) x &= 0xFFFFFFFFu >> (8 * (4 - (L - k)));
        nz |= x;
      }
      Scan sc;
      sc.w = run19(text, ts + 19, 19);
      sc.q = (int32_t)(L - 19);
      sc.kind = K_NUM;
      sc.neg = false;
      sc.tnz = nz != 0;
      return decide<F32>(sc);
    }
  }
  const Scan sc = fast_scan(text, ts, L, ndw, p10);
  if (sc.kind == K_SLOWSCAN) return decide<F32>(scan_record(text + ts, L));
  return decide_num<F32>(sc.w, sc.q, sc.neg);
}

}  // namespace fpp
