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

template <bool F32>
__device__ __forceinline__ uint32_t status_of(uint64_t pos_bits) {
  return pos_bits == Fmt<F32>::kInf ? ST_OVERFLOW : (pos_bits == 0 ? ST_UNDERFLOW : ST_OK);
}

template <bool F32>
__device__ __forceinline__ Res decide(const Scan& s) {
  using F = Fmt<F32>;
  Res r;
  const uint64_t sg = s.neg ? F::kSign : 0;
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

}  // namespace fpp
