// decide.cuh -- scanner result -> (bits, status) or a slow-path candidate.
//
// Number records: Algorithm 1 on (w, q).  With more than
// 19 significant digits and a nonzero dropped digit (tnz) the value lies in
// [w*10^q, (w+1)*10^q) and Algorithm 1 runs on both ends: equal results decide
// the record; otherwise, or when Algorithm 1 aborts
// (line 6, L232), the record goes to the exact slow path with candidate
// r0 = Alg1(w, q) (the un-aborted product when aborting: within one ulp).
#pragma once
#include "alg1.cuh"
#include "scan.cuh"

namespace fpp {

constexpr uint64_t kCandNoLower = 1ull << 63;  // candidate flag: also check the lower neighbour
// long records (more than kLongRec bytes, or running past a fast kernel's
// staged text) are not scanned by the fast kernels at all: they go to the
// slow kernel, which lexes them with the whole warp, with this candidate
constexpr uint64_t kCandUnknown = ~0ull;
constexpr int64_t kLongRec = 64;
constexpr uint32_t F_PENDING = 1u << 8;        // decided by the slow kernel
constexpr uint32_t F_BRACKET = 1u << 10;       // w / w+1 bracket evaluated

// Result of the fast path.  bits: final bits with sign, or (F_PENDING) the
// slow-path candidate.  info: status in the low byte, F_* flags above.
struct Res {
  uint64_t bits;
  uint32_t info;
};

// nearest value to (w + d) * 2^q, d = 0 (tnz false) or some d in (0, 1)
// (tnz true): a hexadecimal float's kept nibbles and dropped sticky part.
// Exact: round to nearest on the bits below the significand, ties to even,
// subnormals by shifting further (sticky kept), overflow to infinity.
template <bool F32>
__device__ __forceinline__ uint64_t round_hex(uint64_t w, int q, bool tnz, uint32_t& fl) {
  using F = Fmt<F32>;
  constexpr int P = F::kFracBits + 1;  // significand bits
  if (w == 0) return 0;
  const int l = __clzll((long long)w);
  const uint64_t m64 = w << l;                   // leading bit at 63
  const int64_t lead = (int64_t)q - l + 63;      // exponent of the leading bit
  // bits of m64 below the significand: 64 - P normally, more for subnormals
  int64_t drop = 64 - P;
  if (lead < F::kEmin) drop += F::kEmin - lead;
  if (lead > F::kEmax) { fl |= ST_OVERFLOW; return F::kInf; }
  uint64_t m, half, rest;
  bool sticky = tnz;
  if (drop >= 64) {
    m = 0;
    half = drop == 64 ? (m64 >> 63) : 0;
    sticky |= drop == 64 ? (m64 << 1) != 0 : m64 != 0;
  } else {
    m = m64 >> drop;
    half = (m64 >> (drop - 1)) & 1;
    rest = drop >= 2 ? (m64 & ((1ull << (drop - 1)) - 1)) : 0;
    sticky |= rest != 0;
  }
  if (half && (sticky || (m & 1))) m++;
  // m < 2^P (normal, biased exponent lead + bias) or subnormal (< 2^(P-1));
  // a carry to 2^P moves into the exponent through the addition below
  uint64_t bits;
  if (lead < F::kEmin) bits = m;  // subnormal: exponent field 0 (2^(P-1) -> smallest normal)
  else bits = ((uint64_t)(lead + F::kEmax - 1) << F::kFracBits) + m;
  if (bits >= F::kInf) { fl |= ST_OVERFLOW; return F::kInf; }
  if (bits == 0) fl |= ST_UNDERFLOW;
  return bits;
}

template <bool F32>
__device__ __forceinline__ Res decide(const Scan& s) {
  using F = Fmt<F32>;
  Res r;
  const uint64_t sg = s.neg ? F::kSign : 0;
  if (s.kind == K_HEX) {
    uint32_t fl = 0;
    r.bits = sg | round_hex<F32>(s.w, s.q, s.tnz, fl);
    r.info = fl;
    return r;
  }
  if (s.kind != K_NUM) {
    if (s.kind == K_INF) { r.bits = sg | F::kInf; r.info = ST_OK; }
    else if (s.kind == K_NAN) { r.bits = sg | F::kQNaN; r.info = ST_OK; }
    else { r.bits = F::kQNaN; r.info = (s.kind == K_EMPTY) ? ST_EMPTY : ST_INVALID; }
    return r;
  }
  if (s.w == 0) { r.bits = sg; r.info = ST_OK; return r; }  // +-0 (reading G13)
  uint32_t fl = 0;
  const uint64_t a = alg1<F32>(s.w, s.q, fl);
  if (s.tnz) {
    uint32_t fl2 = 0;
    const uint64_t b = alg1<F32>(s.w + 1, s.q, fl2);  // w + 1 <= 10^19 < 2^64
    fl |= F_BRACKET | (fl2 & F_TWO);
    if (a != b || ((fl | fl2) & F_ABORT)) fl |= F_PENDING;
  } else if (fl & F_ABORT) {
    fl |= F_PENDING;
  }
  if (fl & F_PENDING) {
    r.bits = a | ((fl & F_ABORT) ? kCandNoLower : 0);
    r.info = fl & ~0xFFu;  // status OK until the slow kernel decides
    return r;
  }
  r.bits = sg | a;
  r.info = fl;  // alg1 put ST_OVERFLOW / ST_UNDERFLOW in the low byte
  return r;
}

// Fast-path decision for a number the SWAR scanner produced: at most 19
// significant digits (no truncation, so no bracket), kind K_NUM.
template <bool F32>
__device__ __forceinline__ Res decide_num(uint64_t w, int q, bool neg) {
  Res r;
  const uint64_t sg = neg ? Fmt<F32>::kSign : 0;
  if (w == 0) { r.bits = sg; r.info = ST_OK; return r; }
  uint32_t fl = 0;
  const uint64_t a = alg1<F32>(w, q, fl);
  if (fl & F_ABORT) {  // line 6: the exact slow path decides, candidate within one ulp
    r.bits = a | kCandNoLower;
    r.info = (fl | F_PENDING) & ~0xFFu;
    return r;
  }
  r.bits = sg | a;
  r.info = fl;
  return r;
}

// the same out of line: the fast parsers' rare branch (zero, q outside the
// table, subnormal, overflow, abort), kept out of their hot loops' code
template <bool F32>
__device__ __noinline__ Res decide_num_ni(uint64_t w, int q, bool neg) {
  return decide_num<F32>(w, q, neg);
}

}  // namespace fpp
