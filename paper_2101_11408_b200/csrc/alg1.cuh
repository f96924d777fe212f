// alg1.cuh -- the paper's Algorithm 1 on the GPU.
//
// Computes the binary64 nearest to w * 10^q for w in (0, 10^19] from the
// 128-bit table T[q] (generated, tables/pow5_128.inc; Appendix B)
// with one or two 64x64->128 multiplications (__umul64hi + low product).
// Readings: G1 subnormal iff p <= -1023 with s = -1022 - p (the
// printed "p <= -1022, s = -1022 - p + 1" treats p = -1022, a normal, as
// subnormal); G2 zero iff p <= -1086 (keeps every shift < 64); G4 "(z/2^64)/m
// is a power of two" == ((m << (9+u)) == hi); G5 m = hi >> (9+u); reading L20:
// the carry test after rounding is m == 2^53 (the printed 2^54 cannot occur
// after the halving) -- folded into the packing: the exponent gains m >> 53
// and the stored fraction is m mod 2^52.
// The rare tests (second multiplication, abort, tie, subnormal, overflow) sit
// behind branches on cheap 32-bit conditions so the common path stays short.
#pragma once
#include "common.cuh"

namespace fpp {

// T[q] as {hi, lo} pairs, index 2*(q+342)
__device__ const __align__(16) uint64_t kPow5_128[1302] = {
#include "tables/pow5_128.inc"
};

// flags reported through `fl` (the low byte carries the status of the result)
constexpr uint32_t F_TWO = 1u << 9;     // second multiplication used
constexpr uint32_t F_ABORT = 1u << 11;  // line 6: fall back

// positive result bits for w * 10^q, w != 0 (lines 1-2 early exits included);
// fl |= ST_OVERFLOW / ST_UNDERFLOW when the result is +inf / +0.  F32: the
// binary32 column of Algorithm 1 (26 exact bits, 25-bit m, subnormal below
// 2^-126, ties for q in [-17, 10], overflow above 127), same readings.
template <bool F32>
__device__ __forceinline__ uint64_t alg1(uint64_t w, int q, uint32_t& fl) {
  using F = Fmt<F32>;
  constexpr uint64_t kCutMask = (1ull << F::kCut) - 1;
  if ((uint32_t)(q + 342) > 650u) {
    fl |= q < 0 ? ST_UNDERFLOW : ST_OVERFLOW;
    return q < 0 ? 0ull : F::kInf;
  }
  // lines 3-4: normalise w into [2^63, 2^64)
  const int l = __clzll((long long)w);
  w <<= l;
  // line 5: truncated product z = (T[q] * w) / 2^64, stopping after one
  // multiplication unless the high word's bits below the exact ones are all
  // ones; T[q] through the read-only path (L1-resident, 10 KiB)
  const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(&kPow5_128[2 * (q + 342)]));
  uint64_t hi = __umul64hi(w, t.x);
  uint64_t lo = w * t.x;
  if ((hi & kCutMask) == kCutMask) {
    const uint64_t add = __umul64hi(w, t.y);
    lo += add;
    hi += (lo < add);
    fl |= F_TWO;
  }
  // line 6: abort when the second word is all ones outside [-27, 55]
  if ((uint32_t)(lo >> 32) == 0xFFFFFFFFu) {
    if ((uint32_t)lo == 0xFFFFFFFFu && (uint32_t)(q + 27) > 82u) fl |= F_ABORT;
  }
  // lines 7-9: significand with one extra bit, exponent formula
  const int u = (int)(hi >> 63);
  uint64_t m = hi >> (u + F::kCut);
  const int p = ((217706 * q) >> 16) + 63 - l + u;
  // lines 10-15: zero (G2) and subnormals (G1); half-up is exact here (L909)
  if (p <= F::kEmin - 1) {
    if (p <= F::kEmin - 64) { fl |= ST_UNDERFLOW; return 0; }
    m >>= (F::kEmin - p);
    m = (m + (m & 1)) >> 1;  // 2^kFracBits encodes the smallest normal
    if (m == 0) fl |= ST_UNDERFLOW;
    return m;
  }
  // lines 16-18: ties to even, only possible for q in [kTieLo, kTieHi] (L287-333)
  if ((uint32_t)(q - F::kTieLo) <= (uint32_t)(F::kTieHi - F::kTieLo)) {
    if (lo <= 1 && ((uint32_t)m & 3u) == 1u && (m << (u + F::kCut)) == hi) m -= 1;
  }
  // lines 19-21: round, carry, overflow, pack
  m = (m + (m & 1)) >> 1;
  const int pe = p + (int)(m >> (F::kFracBits + 1));
  if (pe > F::kEmax) { fl |= ST_OVERFLOW; return F::kInf; }
  return ((uint64_t)(pe + F::kEmax) << F::kFracBits) | (m & ((1ull << F::kFracBits) - 1));
}

}  // namespace fpp
