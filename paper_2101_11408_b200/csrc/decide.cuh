// decide.cuh -- scanner result -> (bits, status) or a slow-path candidate.
//
// Number records: Algorithm 1 on (w, q).  With more than
// 19 significant digits and a nonzero dropped digit (tnz) the value lies in
// [w*10^q, (w+1)*10^q) and Algorithm 1 runs on both ends: equal results decide
// the record; otherwise, or when Algorithm 1 aborts
// (line 6, L232), the record goes to the exact slow path with candidate
// r0 = Alg1(w, q) (or the un-aborted product when aborting).
#pragma once
#include "alg1.cuh"
#include "scan.cuh"

namespace fpp {

constexpr uint64_t kCandNoLower = 1ull << 63;  // candidate flag: also check the lower neighbour

struct Decision {
  uint64_t bits;  // final bits incl. sign (when !pending)
  uint64_t cand;  // slow-path candidate (when pending)
  uint8_t st;
  bool pending;
  bool two;
  bool bracket;
  bool abort;
};

__device__ __forceinline__ uint8_t status_of(uint64_t pos_bits) {
  return pos_bits == kInf ? ST_OVERFLOW : (pos_bits == 0 ? ST_UNDERFLOW : ST_OK);
}

__device__ __forceinline__ Decision decide(const Scan& s, const uint64_t* __restrict__ T) {
  Decision d;
  d.pending = false;
  d.two = false;
  d.bracket = false;
  d.abort = false;
  d.cand = 0;
  const uint64_t sg = s.neg ? kSign : 0;
  if (s.kind != K_NUM) {
    if (s.kind == K_INF) { d.bits = sg | kInf; d.st = ST_OK; }
    else if (s.kind == K_NAN) { d.bits = sg | kQNaN; d.st = ST_OK; }
    else { d.bits = kQNaN; d.st = (s.kind == K_EMPTY) ? ST_EMPTY : ST_INVALID; }
    return d;
  }
  if (s.w == 0) { d.bits = sg; d.st = ST_OK; return d; }  // +-0 (reading G13)
  A1Out a = alg1(s.w, s.q, T);
  d.two = a.two;
  d.abort = a.abort;
  if (!s.tnz) {
    if (a.abort) { d.pending = true; d.cand = a.bits | kCandNoLower; }
    d.bits = sg | a.bits;
    d.st = status_of(a.bits);
    return d;
  }
  d.bracket = true;
  A1Out b = alg1(s.w + 1, s.q, T);  // w + 1 <= 10^19 < 2^64
  d.abort |= b.abort;
  if (!a.abort && !b.abort && a.bits == b.bits) {
    d.bits = sg | a.bits;
    d.st = status_of(a.bits);
    return d;
  }
  d.pending = true;
  d.cand = a.bits | (a.abort ? kCandNoLower : 0);
  d.bits = sg | a.bits;
  d.st = status_of(a.bits);
  return d;
}

}  // namespace fpp
