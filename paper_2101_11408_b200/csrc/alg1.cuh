// alg1.cuh -- the paper's Algorithm 1 on the GPU.
//
// Computes the binary64 nearest to w * 10^q for w in [0, 10^19] from the
// 128-bit table T[q] (generated, tables/pow5_128.inc; Appendix B)
// with one or two 64x64->128 multiplications (__umul64hi + low product).
// Readings: G1 subnormal iff p <= -1023 with s = -1022 - p (the
// printed "p <= -1022, s = -1022 - p + 1" treats p = -1022, a normal, as
// subnormal); G2 zero iff p <= -1086 (keeps every shift < 64); G4 "(z/2^64)/m
// is a power of two" == ((m << (9+u)) == hi); G5 m = hi >> (9+u); G-line17:
// the carry test after rounding is m == 2^53 (the printed 2^54 cannot occur
// after the halving).
#pragma once
#include "common.cuh"

namespace fpp {

// T[q] as {hi, lo} pairs, index 2*(q+342)
__device__ const uint64_t kPow5_128[1302] = {
#include "tables/pow5_128.inc"
};

struct A1Out {
  uint64_t bits;  // positive result bits
  bool abort;     // Algorithm 1 line 6: fall back
  bool two;       // second multiplication used
};

// T: the 1302-word table (shared or global memory)
__device__ __forceinline__ A1Out alg1(uint64_t w, int q, const uint64_t* __restrict__ T) {
  A1Out r;
  r.abort = false;
  r.two = false;
  // lines 1-2: early exits
  if (w == 0 || q < -342) { r.bits = 0; return r; }
  if (q > 308) { r.bits = kInf; return r; }
  // lines 3-4: normalise w into [2^63, 2^64)
  const int l = __clzll((long long)w);
  w <<= l;
  // line 5: truncated product z = (T[q] * w) / 2^64, stopping after one
  // multiplication unless the low 9 bits of the high word are all ones
  const uint64_t th = T[2 * (q + 342)];
  uint64_t hi = __umul64hi(w, th);
  uint64_t lo = w * th;
  if ((hi & 0x1FF) == 0x1FF) {
    const uint64_t tl = T[2 * (q + 342) + 1];
    const uint64_t add = __umul64hi(w, tl);
    lo += add;
    hi += (lo < add);
    r.two = true;
  }
  // line 6: abort when the second word is all ones outside [-27, 55]
  if (lo == ~0ull && (q < -27 || q > 55)) r.abort = true;
  // lines 7-9: 54-bit significand, exponent formula
  const int u = (int)(hi >> 63);
  uint64_t m = hi >> (u + 9);
  int p = ((217706 * q) >> 16) + 63 - l + u;
  // line 10: certainly zero (G2)
  if (p <= -1086) { r.bits = 0; return r; }
  // lines 11-15: subnormals (G1), half-up rounding is exact here
  if (p <= -1023) {
    const int s = -1022 - p;
    m >>= s;
    m += (m & 1);
    m >>= 1;
    r.bits = m;  // m == 2^52 encodes the smallest normal
    return r;
  }
  // lines 16-18: ties to even, only possible for q in [-4, 23]
  if (lo <= 1 && q >= -4 && q <= 23 && (m & 3) == 1 && (m << (u + 9)) == hi) m -= 1;
  // line 19: round
  m += (m & 1);
  m >>= 1;
  // line 20: carry out of the top bit
  if (m == (1ull << 53)) { m >>= 1; p += 1; }
  // line 21: overflow
  if (p > 1023) { r.bits = kInf; return r; }
  r.bits = ((uint64_t)(p + 1023) << 52) | (m & ((1ull << 52) - 1));
  return r;
}

}  // namespace fpp
