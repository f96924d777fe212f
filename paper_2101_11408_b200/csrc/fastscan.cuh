// fastscan.cuh -- SWAR record scanner over shared memory (the common case).
//
// The paper parses 8 digits at a time with SWAR (Appendix D
// L1534-1553: is_made_of_eight_digits / parse_eight_digits on a 64-bit
// little-endian word).  Re-derived here for 32-bit GPU lanes:
//   * the tile kernel classifies every staged byte once (32 bytes per thread)
//     into a bit mask of non-digit bytes (nondigit80, k_common.cuh pack_byte), so a
//     record's structure -- sign, integer run, '.', fraction run, 'e' exponent
//     -- is found with a funnel shift and find-first-set;
//   * digit runs are converted 4 digits per 32-bit word with two dp2a
//     instructions (16-bit weights 1000,100 / 10,1 against the 4 bytes; the
//     ASCII '0' offset folded into the accumulator), 8 digits per word pair,
//     runs taken from their END so the weights are fixed and missing leading
//     digits are filled with '0' (run19, fill_word).
// Records this path does not cover (longer than 30 bytes, more than 19
// significant digits, specials, trailing terminators beyond one, exponents of
// more than 4 digits) return K_SLOWSCAN and are rescanned byte by byte
// (scan.cuh).
#pragma once
#include "scan.cuh"

namespace fpp {

constexpr int K_SLOWSCAN = 99;

// 4 bytes at shared byte offset a (any alignment), little endian
__device__ __forceinline__ uint32_t lds4(const uint8_t* base, uint32_t a) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
  const uint32_t lo = w[a >> 2], hi = w[(a >> 2) + 1];
  return __funnelshift_r(lo, hi, (a & 3) * 8);
}
__device__ __forceinline__ int dp2a_lo(int a, int b, int c) {
  int r;
  asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ int dp2a_hi(int a, int b, int c) {
  int r;
  asm("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// value of the 4 ASCII digits in w (byte 0 = first = most significant)
__device__ __forceinline__ uint32_t dig4(uint32_t w) {
  const int t = dp2a_hi(0x0001000A, (int)w, -48 * 1111);  // 10 b2 + b3 - 48 (1000+100+10+1)
  return (uint32_t)dp2a_lo(0x006403E8, (int)w, t);        // + 1000 b0 + 100 b1
}

// value of the n (1..4) digits ending at shared offset e (one word, '0' fill)
__device__ __forceinline__ uint32_t dig_tail4(const uint8_t* base, uint32_t e, uint32_t n) {
  uint32_t x = lds4(base, e - 4);
  const uint32_t keep = n >= 4 ? 0xFFFFFFFFu : (0xFFFFFFFFu << (8 * (4 - n)));
  x = (x & keep) | (0x30303030u & ~keep);
  return dig4(x);
}

// keep masks for a 4-byte word whose first k bytes (k may exceed 4) read as '0'
__device__ __forceinline__ uint32_t fill_word(uint32_t x, int k) {
  // keep = ~0 << 8k for k in [0, 4] (0 for k >= 4): one clamped funnel shift
  const uint32_t keep = __funnelshift_lc(0u, 0xFFFFFFFFu, (uint32_t)(8 * max(k, 0)));
  return (x & keep) | (0x30303030u & ~keep);
}

// Branch-free value of the n (0..19) digits ending at shared offset e: three
// windows [e-20, e-16), [e-16, e-8), [e-8, e) read once (6 words), bytes
// before the run read as '0'.  Reads up to 20 bytes before e (callers keep a
// pad in front of the buffer).  Uniform across lanes whatever n is.
__device__ __forceinline__ uint64_t run19(const uint8_t* base, uint32_t e, int n) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
  const uint32_t a = e - 20, i = a >> 2, sh = (a & 3) * 8;
  const uint32_t w0 = w[i], w1 = w[i + 1], w2 = w[i + 2], w3 = w[i + 3], w4 = w[i + 4], w5 = w[i + 5];
  uint32_t c = __funnelshift_r(w0, w1, sh);   // [e-20, e-16)
  uint32_t b0 = __funnelshift_r(w1, w2, sh);  // [e-16, e-12)
  uint32_t b1 = __funnelshift_r(w2, w3, sh);  // [e-12, e-8)
  uint32_t a0 = __funnelshift_r(w3, w4, sh);  // [e-8, e-4)
  uint32_t a1 = __funnelshift_r(w4, w5, sh);  // [e-4, e)
  // digits present in each word, counted from the end of the run; 16..19
  // digits (17-digit printing, the common case) only fill the top word
  if (n < 16) {
    a1 = fill_word(a1, 4 - n);
    a0 = fill_word(a0, 8 - n);
    b1 = fill_word(b1, 12 - n);
    b0 = fill_word(b0, 16 - n);
  }
  c = fill_word(c, 20 - n);
  const uint32_t A = dig4(a0) * 10000u + dig4(a1);
  const uint32_t B = dig4(b0) * 10000u + dig4(b1);
  return ((uint64_t)dig4(c) * 100000000ull + B) * 100000000ull + A;
}

// three-input logic op (LOP3) with an explicit truth table: f(0xF0, 0xCC, 0xAA)
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return r;
}
constexpr uint32_t LUT_XOR_AND = (0xF0 ^ 0xCC) & 0xAA;     // (a ^ b) & c
constexpr uint32_t LUT_OR_AND = (0xF0 | 0xCC) & 0xAA;      // (a | b) & c
constexpr uint32_t LUT_NOR_AND = (~(0xF0 | 0xCC)) & 0xAA;  // ~(a | b) & c

// non-digit flags (bit 7 of each byte) of a little-endian word, exact per byte
// (3 instructions: digits map to 0..9 and stay below 0x80 after + 0x76)
__device__ __forceinline__ uint32_t nondigit80(uint32_t v) {
  const uint32_t x = lop3<LUT_XOR_AND>(v, 0x30303030u, 0x7F7F7F7Fu);
  return lop3<LUT_OR_AND>(x + 0x76767676u, v, 0x80808080u);
}
// separator flags (bit 7 of each byte): exact zero-byte test of v ^ sep
template <uint32_t SEPS>
__device__ __forceinline__ uint32_t sep80(uint32_t v) {
  uint32_t hit = 0;
  if (SEPS & 1u) {
    const uint32_t x = lop3<LUT_XOR_AND>(v, 0x0A0A0A0Au, 0x7F7F7F7Fu);
    hit |= lop3<LUT_NOR_AND>(x + 0x7F7F7F7Fu, v, 0x80808080u);
  }
  if (SEPS & 2u) {
    const uint32_t x = lop3<LUT_XOR_AND>(v, 0x2C2C2C2Cu, 0x7F7F7F7Fu);
    hit |= lop3<LUT_NOR_AND>(x + 0x7F7F7F7Fu, v, 0x80808080u);
  }
  return hit;
}
// Fast scan of the record text[s, s+L) (shared memory), given its non-digit
// mask word ndw (bit i set iff byte s+i is not a digit, i < 32).
// Covers [sign] digits* ['.' digits*] [(e|E) [sign] 1-4 digits] [terminator].
__device__ __forceinline__ Scan fast_scan(const uint8_t* text, uint32_t s, uint32_t L, uint32_t ndw,
                                          const uint64_t* __restrict__ p10) {
  Scan r;
  r.w = 0;
  r.q = 0;
  r.kind = K_SLOWSCAN;
  r.neg = false;
  r.tnz = false;
  if (L == 0 || L > 30) return r;
  const uint32_t nd = ndw | (0xFFFFFFFFu << L);  // bytes past the record read as non-digits
  const uint32_t c0 = text[s];
  const uint32_t p = (c0 == '-' || c0 == '+') ? 1u : 0u;
  r.neg = (c0 == '-');
  const uint32_t i1 = __ffs(nd >> p) - 1 + p;  // end of the integer run
  // i1 <= L <= 30: the byte is inside the staged buffer even at i1 == L
  const bool dot = (text[s + i1] == '.') & (i1 < L);
  const uint32_t fb = i1 + (dot ? 1u : 0u);
  const uint32_t f1 = dot ? __ffs(nd >> fb) - 1 + fb : i1;
  const uint32_t ni = i1 - p;
  uint32_t nf = f1 - fb;
  if (ni + nf == 0) return r;  // specials / invalid: byte scanner
  int32_t e = 0;
  uint32_t end = f1;
  if (f1 < L && (text[s + f1] | 0x20) == 'e') {
    uint32_t k = f1 + 1;
    const uint32_t cs = k < L ? (uint32_t)text[s + k] : 0u;
    const bool eneg = cs == '-';
    k += (cs == '-' || cs == '+') ? 1u : 0u;
    const uint32_t ke = __ffs(nd >> k) - 1 + k;
    const uint32_t ne = ke - k;
    if (ne == 0 || ne > 4) return r;
    e = (int32_t)dig_tail4(text, s + ke, ne);
    if (eneg) e = -e;
    end = ke;
  }
  // one trailing terminator allowed here; anything else goes to the byte scanner
  if (end != L && (end + 1 != L || !is_term(text[s + end]))) return r;
  // integer part: one uniform 4-byte window for up to 4 digits (the common case)
  uint64_t I;
  if (ni <= 4) {
    I = dig4(fill_word(lds4(text, s + i1 - 4), 4 - (int)ni));
  } else {
    if (ni > 19) return r;
    I = run19(text, s + i1, (int)ni);
  }
  const int32_t q = e - (int32_t)nf;
  if (ni + nf > 19) {
    // only "0.000ddd..."-like records: skip the fraction's leading zeros
    if (I != 0 || nf > 27) return r;
    const uint64_t z = ((uint64_t)lds4(text, s + fb + 4) << 32 | lds4(text, s + fb)) ^ 0x3030303030303030ull;
    const uint32_t lz = z ? (__ffsll((long long)z) - 1) >> 3 : 8u;
    if (nf - lz > 19) return r;
    nf -= lz;
  }
  // fraction: branch-free for any length 0..19 (no divergence between lanes)
  r.w = run19(text, s + f1, (int)nf);
  if (I != 0) r.w += I * p10[nf];
  r.q = q;
  r.kind = K_NUM;
  return r;
}

}  // namespace fpp
