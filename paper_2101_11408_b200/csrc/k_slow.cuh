// k_slow.cuh -- exact slow path.
//
// One warp per queued record.  The paper falls back on an exact
// higher-precision conversion when the 19-digit bracket w / w+1 disagrees or
// Algorithm 1 aborts ("its performance is secondary. However, it has to be
// exact", L986-987).  Here: the value x of the whole digit string lies in
// [w*10^q, (w+1)*10^q), an interval far narrower than one ulp, so by
// monotonicity the result is the candidate r0 = Alg1(w, q) or its successor
// (when Algorithm 1 aborted, the un-aborted product is within one ulp and both
// neighbours are checked).  The warp decides by comparing x exactly with the
// midpoint
//     M = (2m+1) * 2^(e-1),   r0 = m * 2^e,
// whose decimal digits (2m+1) * 5^(1-e)  (e < 1)  or  (2m+1) * 2^(e-1)  it
// forms in base-1e9 limbs from exact power tables (tables/declimbs.inc), one
// limb per lane, carries resolved with a ballot carry-lookahead, then compares
// limb by limb against the record's digits: x < M -> r0, x > M -> successor,
// x == M -> the one with the even significand (ties to even, also for
// subnormals and at the overflow threshold 2^1024 - 2^970; readings G3, G12).
#pragma once
#include "decide.cuh"
#include "fastscan.cuh"
#include "tables/declimbs_meta.h"
#include "k_common.cuh"

namespace fpp {

__device__ const uint32_t kDecLimbs[FPP_DECLIMBS_N] = {
#include "tables/declimbs.inc"
};
// (offset << 8) | limb count, for 5^k and 2^k
__device__ const uint32_t kPow5Index[FPP_POW5_KMAX + 1] = {
#include "tables/pow5_index.inc"
};
__device__ const uint32_t kPow2Index[FPP_POW2_KMAX + 1] = {
#include "tables/pow2_index.inc"
};

constexpr uint32_t kBase = 1000000000u;
constexpr int kSlowThreads = 128;

// The record's digit string as the warp sees it: integer digits at
// [ib, ib+nI), fraction digits at [fb, fb+nF) (the '.' skipped).
struct DigitStream {
  const uint8_t* bytes;
  int64_t ib, nI, fb, nF, N;
  int64_t z;   // stream index of the first nonzero digit
  int64_t Ex;  // decimal exponent of that digit: x in [10^Ex, 10^(Ex+1))
  __device__ __forceinline__ uint32_t digit(int64_t u) const {
    const int64_t pos = u < nI ? ib + u : fb + (u - nI);
    return (uint32_t)bytes[pos] - '0';
  }
};

// first stream index in [from, to) holding a nonzero digit (to if none)
__device__ __forceinline__ int64_t warp_first_nonzero(const DigitStream& ds, int64_t from, int64_t to) {
  const int lane = threadIdx.x & 31;
  for (int64_t u0 = from; u0 < to; u0 += 32) {
    const int64_t u = u0 + lane;
    const unsigned m = __ballot_sync(0xffffffffu, u < to && ds.digit(u) != 0);
    if (m) return u0 + __ffs(m) - 1;
  }
  return to;
}

// first position in [from, to) whose byte satisfies PRED (to if none)
template <typename PRED>
__device__ __forceinline__ int64_t warp_find(const uint8_t* b, int64_t from, int64_t to, PRED pred) {
  const int lane = threadIdx.x & 31;
  for (int64_t p0 = from; p0 < to; p0 += 32) {
    const int64_t p = p0 + lane;
    const unsigned m = __ballot_sync(0xffffffffu, p < to && pred((uint32_t)b[p]));
    if (m) return p0 + __ffs(m) - 1;
  }
  return to;
}

// first position in [from, to) whose byte is not a digit
__device__ __forceinline__ int64_t warp_find_nondigit(const uint8_t* b, int64_t from, int64_t to) {
  return warp_find(b, from, to, [](uint32_t c) { return !is_digit(c); });
}

// the same over the warp's staged copy (4-byte aligned): one word per lane,
// 128 bytes per step, a SWAR digit test (fastscan.cuh nondigit80)
__device__ __forceinline__ int warp_find_nondigit_w(const uint8_t* b, int from, int to) {
  const uint32_t* wd = reinterpret_cast<const uint32_t*>(b);
  const int lane = threadIdx.x & 31;
  for (int w0 = from >> 2; (w0 << 2) < to; w0 += 32) {
    const int wi = w0 + lane, pw = wi << 2;
    uint32_t f = 0;
    if (pw < to) {
      f = nondigit80(wd[wi]);
      if (pw < from) f &= 0xFFFFFFFFu << (8 * (from - pw));
      if (pw + 4 > to) f &= 0xFFFFFFFFu >> (8 * (pw + 4 - to));
    }
    const unsigned m = __ballot_sync(0xffffffffu, f != 0);
    if (m) {
      const int l = __ffs(m) - 1;
      return ((w0 + l) << 2) + ((__ffs(__shfl_sync(0xffffffffu, f, l)) - 1) >> 3);
    }
  }
  return to;
}

__device__ __forceinline__ int64_t warp_find_sep(const uint8_t* b, int64_t from, int64_t to, uint32_t seps) {
  return warp_find(b, from, to, [seps](uint32_t c) { return is_sep(c, seps); });
}

// number of decimal digits of v
__device__ __forceinline__ int ndigits_u32(uint32_t v) {
  return 1 + (v >= 10u) + (v >= 100u) + (v >= 1000u) + (v >= 10000u) + (v >= 100000u) + (v >= 1000000u) +
         (v >= 10000000u) + (v >= 100000000u) + (v >= 1000000000u);
}

// value of the 9 stream digits [u0, u0 + 9) (digits outside [z, N) read as 0):
// one run of contiguous bytes unless the window touches the ends or the '.'
__device__ __forceinline__ uint32_t limb_digits(const DigitStream& ds, int64_t u0) {
  uint32_t X = 0;
  if (u0 >= ds.N || u0 + 9 <= ds.z) return 0u;  // all outside the digits
  const bool inI = u0 >= ds.z && u0 + 9 <= ds.nI;
  const bool inF = u0 >= ds.nI && u0 >= ds.z && u0 + 9 <= ds.N;
  if (inI || inF) {
    const uint8_t* q = ds.bytes + (inI ? ds.ib + u0 : ds.fb + (u0 - ds.nI));
#pragma unroll
    for (int t = 0; t < 9; t++) X = X * 10 + ((uint32_t)q[t] - '0');
  } else {
    for (int t = 0; t < 9; t++) {
      const int64_t u = u0 + t;
      X = X * 10 + ((u >= ds.z && u < ds.N) ? ds.digit(u) : 0u);
    }
  }
  return X;
}

// Staged records: the value of the k (0..9) digit bytes ending at offset E
// of buf (readable from E - 12), '0'-filled before them -- three words read
// from the end, 4 digits per dp2a pair (fastscan.cuh)
__device__ __forceinline__ uint32_t digits_before(const uint8_t* buf, int64_t E, int k) {
  const uint8_t* padded = buf - 16;
  const uint32_t e = (uint32_t)E + 16u;
  const uint32_t w0 = lds4(padded, e - 12), w1 = lds4(padded, e - 8), w2 = lds4(padded, e - 4);
  return dig4(fill_word(w0, 12 - k)) * 100000000u + dig4(fill_word(w1, 8 - k)) * 10000u + dig4(fill_word(w2, 4 - k));
}

// floor(t / 1e9) for t < 2^60 without a division (Granlund-Montgomery:
// m = floor(2^90 / 1e9) + 1 and 2^90 <= m 1e9 <= 2^90 + 2^30, so
// floor(t m / 2^90) = floor(t / 1e9) for every t < 2^60)
__device__ __forceinline__ uint32_t div1e9_60(uint64_t t) {
  return (uint32_t)(__umul64hi(t, 1237940039285380275ull) >> 26);
}

// The midpoint M = a * 2^f (a odd, a < 2^54, f in [-1075, 970]) in base-1e9
// limbs, one per lane in three groups (limb j = lane + 32 g): M = a * 5^-f *
// 10^f (f < 0) or a * 2^f; F = decimal exponent of limb 0's lowest digit,
// J = the most significant nonzero limb, EM = M's leading decimal exponent.
struct MidLimbs {
  uint32_t Fl[3];
  int J;
  int64_t F, EM;
};
__device__ __forceinline__ void mid_limbs(uint64_t a, int f, MidLimbs& L) {
  const int lane = threadIdx.x & 31;
  uint32_t idx;
  if (f < 0) { idx = kPow5Index[-f]; L.F = f; }
  else { idx = kPow2Index[f]; L.F = 0; }
  const uint32_t* P = kDecLimbs + (idx >> 8);
  const int nP = (int)(idx & 0xFF);
  const uint64_t a1 = div1e9_60(a), a0 = a - a1 * kBase;
  // limb j of a * P, before carries: t_j = a0 P_j + a1 P_(j-1) < 1.02e18 < 2^60;
  // the product has at most nP + 2 limbs, so groups past that are zero
  const int ng = (nP + 2 + 31) >> 5;
  uint32_t hi[3], lo[3];
#pragma unroll
  for (int g = 0; g < 3; g++) {
    hi[g] = lo[g] = 0u;
    if (g < ng) {  // warp-uniform
      const int j = 32 * g + lane;
      const uint64_t pj = j < nP ? __ldg(P + j) : 0u;
      const uint64_t pm = (j >= 1 && j - 1 < nP) ? __ldg(P + j - 1) : 0u;
      const uint64_t t = a0 * pj + a1 * pm;
      hi[g] = div1e9_60(t);
      lo[g] = (uint32_t)(t - (uint64_t)hi[g] * kBase);
    }
  }
  // R_j = lo_j + hi_(j-1)  (< 2.02e9),  c_j = R_j / 1e9 in {0,1,2}
  uint32_t r[3], c[3];
#pragma unroll
  for (int g = 0; g < 3; g++) {
    uint32_t hp = __shfl_up_sync(0xffffffffu, hi[g], 1);
    const uint32_t hl = g ? __shfl_sync(0xffffffffu, hi[g ? g - 1 : 0], 31) : 0u;
    if (lane == 0) hp = hl;
    const uint32_t R = lo[g] + hp;
    c[g] = R / kBase;
    r[g] = R - c[g] * kBase;
  }
  // S_j = r_j + c_(j-1) <= 1e9 + 1; carry-lookahead over generate / propagate
  uint32_t S[3], G[3], Pp[3];
#pragma unroll
  for (int g = 0; g < 3; g++) {
    uint32_t cp = __shfl_up_sync(0xffffffffu, c[g], 1);
    const uint32_t cl = g ? __shfl_sync(0xffffffffu, c[g ? g - 1 : 0], 31) : 0u;
    if (lane == 0) cp = cl;
    S[g] = r[g] + cp;
    G[g] = __ballot_sync(0xffffffffu, S[g] >= kBase);
    Pp[g] = __ballot_sync(0xffffffffu, S[g] == kBase - 1);
  }
  // carries into each limb: (X + Y) ^ X ^ Y with X = G, Y = G | P (96-bit)
  const uint64_t s0 = (uint64_t)G[0] + (G[0] | Pp[0]);
  const uint64_t s1 = (uint64_t)G[1] + (G[1] | Pp[1]) + (s0 >> 32);
  const uint64_t s2 = (uint64_t)G[2] + (G[2] | Pp[2]) + (s1 >> 32);
  const uint32_t CIN[3] = {(uint32_t)s0 ^ G[0] ^ (G[0] | Pp[0]), (uint32_t)s1 ^ G[1] ^ (G[1] | Pp[1]),
                           (uint32_t)s2 ^ G[2] ^ (G[2] | Pp[2])};
  unsigned nz[3];
#pragma unroll
  for (int g = 0; g < 3; g++) {
    uint32_t v = S[g] + ((CIN[g] >> lane) & 1u);
    if (v >= kBase) v -= kBase;
    L.Fl[g] = v;
    nz[g] = __ballot_sync(0xffffffffu, v != 0);
  }
  L.J = nz[2] ? 64 + 31 - __clz(nz[2]) : (nz[1] ? 32 + 31 - __clz(nz[1]) : 31 - __clz(nz[0]));
  const uint32_t top = __shfl_sync(0xffffffffu, L.Fl[L.J >> 5], L.J & 31);
  L.EM = L.F + 9 * (int64_t)L.J + ndigits_u32(top) - 1;
}

// sign(x - M): x's digit stream has its first nonzero digit at stream index z,
// of decimal exponent Ex; limbx(u0) = the value of stream digits [u0, u0 + 9)
// (0 outside the digits); tailnz(u) = a nonzero digit at stream index >= u
template <typename LimbX, typename TailNZ>
__device__ __forceinline__ int cmp_limbs(const MidLimbs& L, int64_t z, int64_t Ex, LimbX limbx, TailNZ tailnz) {
  const int lane = threadIdx.x & 31;
  if (Ex != L.EM) return Ex > L.EM ? 1 : -1;
  // x's digits in the same base-1e9 grid: limb j covers 10^(F+9j) .. 10^(F+9j+8)
  unsigned diff[3];
  int res[3];
#pragma unroll
  for (int g = 0; g < 3; g++) {
    diff[g] = 0u;
    res[g] = 0;
    if (32 * g <= L.J) {  // warp-uniform: groups above M's top limb hold nothing to compare
      const int j = 32 * g + lane;
      // limb j's most significant digit has weight 10^(F + 9j + 8)
      const int64_t u0 = z + (Ex - (L.F + 9 * (int64_t)j + 8));
      const uint32_t X = j <= L.J ? limbx(u0) : 0u;
      diff[g] = __ballot_sync(0xffffffffu, j <= L.J && X != L.Fl[g]);
      res[g] = X > L.Fl[g] ? 1 : -1;
    }
  }
  if (diff[2] | diff[1] | diff[0]) {
    const int D = diff[2] ? 64 + 31 - __clz(diff[2]) : (diff[1] ? 32 + 31 - __clz(diff[1]) : 31 - __clz(diff[0]));
    return __shfl_sync(0xffffffffu, res[D >> 5], D & 31);
  }
  // all of M's digits matched: x > M iff x has a nonzero digit of weight < 10^F
  const int64_t from = z + (Ex - L.F) + 1;
  return tailnz(from < 0 ? 0 : from) ? 1 : 0;
}

// sign(x - a 2^f) for the global-memory digit stream
__device__ int cmp_mid(const DigitStream& ds, uint64_t a, int f) {
  MidLimbs L;
  mid_limbs(a, f, L);
  return cmp_limbs(
      L, ds.z, ds.Ex, [&](int64_t u0) { return limb_digits(ds, u0); },
      [&](int64_t u) { return warp_first_nonzero(ds, u, ds.N) < ds.N; });
}

// midpoint between finite bits b and b+1 as a * 2^f (binary64, or binary32)
template <bool F32>
__device__ __forceinline__ void mid_of(uint64_t b, uint64_t& a, int& f) {
  using F = Fmt<F32>;
  const uint64_t ef = b >> F::kFracBits, fr = b & ((1ull << F::kFracBits) - 1);
  uint64_t m;
  int e;
  if (ef == 0) { m = fr; e = F::kEmin - F::kFracBits; }
  else { m = fr | (1ull << F::kFracBits); e = (int)ef - (F::kEmax + F::kFracBits); }
  a = 2 * m + 1;
  f = e - 1;
}

// true if some byte in [from, to) is not a terminator
__device__ __forceinline__ bool warp_any_nonterm(const uint8_t* b, int64_t from, int64_t to) {
  return warp_find(b, from, to, [](uint32_t c) { return !is_term(c); }) < to;
}

__device__ const uint64_t kSlowPow10[19] = {
    1ull, 10ull, 100ull, 1000ull, 10000ull, 100000ull, 1000000ull, 10000000ull, 100000000ull,
    1000000000ull, 10000000000ull, 100000000000ull, 1000000000000ull, 10000000000000ull,
    100000000000000ull, 1000000000000000ull, 10000000000000000ull, 100000000000000000ull,
    1000000000000000000ull};

template <bool F32>
__device__ __forceinline__ void put_result(int64_t idx, uint64_t bits, uint32_t st, void* out, uint8_t* status) {
  if ((threadIdx.x & 31) == 0) {
    if (F32) reinterpret_cast<uint32_t*>(out)[idx] = (uint32_t)bits;
    else reinterpret_cast<unsigned long long*>(out)[idx] = bits;
    status[idx] = (uint8_t)st;
  }
}

// The result from candidate cand (bit 63: kCandNoLower) by at most two exact
// comparisons, cmp(a, f) = sign(x - a 2^f), through one inlined copy:
//   mode 0: x against the midpoint above c      (> or an odd tie: c + 1)
//   mode 1: x against the midpoint below c      (< or an odd tie: c - 1)
//   mode 2: c = inf, x against the overflow threshold 2^(emax+1) - 2^(emax-p)
//           ((2^(p+1) - 1) * 2^(emax - p); a tie stays at inf, the even one)
template <bool F32, typename Cmp>
__device__ __forceinline__ uint64_t resolve_cand(uint64_t cand, Cmp cmp_fn) {
  using F = Fmt<F32>;
  const bool chk_low = (cand & kCandNoLower) != 0;
  const uint64_t c = cand & ~kCandNoLower;
  uint64_t r = c;
  int mode = -1;
  uint64_t a = 0;
  int f = 0;
  if (c != F::kInf) {
    mid_of<F32>(c, a, f);
    mode = 0;
  } else if (chk_low) {
    a = (1ull << (F::kFracBits + 2)) - 1;
    f = F::kEmax - F::kFracBits - 1;
    mode = 2;
  }
  while (mode >= 0) {
    const int cmp = cmp_fn(a, f);
    if (mode == 0) {
      if (cmp > 0 || (cmp == 0 && (c & 1))) {
        r = c + 1;
      } else if (chk_low && c != 0) {
        mid_of<F32>(c - 1, a, f);
        mode = 1;
        continue;
      }
    } else if (mode == 1) {
      if (cmp < 0 || (cmp == 0 && (c & 1))) r = c - 1;
    } else if (cmp < 0) {
      r = F::kInf - 1;
    }
    break;
  }
  return r;
}

// Decide one record [s, e) of `bytes` (global memory or the warp's staged
// copy) from candidate `cand`; writes out[idx] and status[idx].
// Warp-collective.  cand == kCandUnknown: a long record the fast kernel did
// not scan -- lexed and checked here (the grammar of scan.cuh), its first 19
// significant digits give (w, q, tnz) and the fast path's decision (Algorithm
// 1 with the w / w+1 bracket, decide.cuh); only an undecided record goes on
// to the exact comparison.  Anything but a well-formed number (specials,
// invalid, empty) is left to the sequential scanner on lane 0.
template <bool F32>
__device__ __noinline__ void slow_record_global(const uint8_t* bytes, int64_t s, int64_t e, uint64_t cand,
                                                int64_t idx, void* out, uint8_t* status, uint32_t grammar) {
  using F = Fmt<F32>;
  const int lane = threadIdx.x & 31;
  const uint32_t c0 = s < e ? bytes[s] : 0u;
  const bool neg = c0 == '-';
  const int64_t p = s + ((c0 == '+' || c0 == '-') ? 1 : 0);
  DigitStream ds;
  ds.bytes = bytes;
  const int64_t ie = warp_find_nondigit(bytes, p, e);
  int64_t fb = ie, fe = ie;
  if (ie < e && bytes[ie] == '.') {
    fb = ie + 1;
    fe = warp_find_nondigit(bytes, fb, e);
  }
  int64_t exp10 = 0, tail = fe;
  bool number = (ie - p) + (fe - fb) > 0;  // at least one digit
  if (fe < e && (bytes[fe] | 0x20) == 'e') {
    int64_t k = fe + 1;
    bool en = false;
    if (k < e && (bytes[k] == '+' || bytes[k] == '-')) { en = bytes[k] == '-'; k++; }
    const int64_t ke = warp_find_nondigit(bytes, k, e);
    number = number && ke > k;
    if (lane == 0) {
      for (int64_t t = k; t < ke; t++)
        if (exp10 < 1000000000000000ll) exp10 = exp10 * 10 + (bytes[t] - '0');  // reading G9
      if (en) exp10 = -exp10;
    }
    exp10 = __shfl_sync(0xffffffffu, exp10, 0);
    tail = ke;
  }
  ds.ib = p;
  ds.nI = ie - p;
  ds.fb = fb;
  ds.nF = fe - fb;
  ds.N = ds.nI + ds.nF;
  if (cand == kCandUnknown) {
    number = number && !warp_any_nonterm(bytes, tail, e);
    if (grammar & G_JSON)  // RFC 8259: no '+', int := '0' | [1-9] digit*, frac := '.' digit+
      number = number && c0 != '+' && ds.nI != 0 && (ds.nI == 1 || bytes[p] != '0') && !(fb > ie && ds.nF == 0);
    if (!number) {  // specials, invalid, empty (never undecided)
      if (lane == 0) {
        Scan sc;
        if (e - s >= (1ll << 31)) {
          sc.kind = K_INVALID; sc.neg = false; sc.tnz = false; sc.w = 0; sc.q = 0;
        } else {
          sc = scan_record(bytes + s, (uint32_t)(e - s), grammar);
        }
        const Res r = decide<F32>(sc);
        if (F32) reinterpret_cast<uint32_t*>(out)[idx] = (uint32_t)r.bits;
        else reinterpret_cast<unsigned long long*>(out)[idx] = r.bits;
        status[idx] = (uint8_t)(r.info & 0xFF);
      }
      return;
    }
    ds.z = warp_first_nonzero(ds, 0, ds.N);
    if (ds.z == ds.N) {  // all digits zero: +-0 (reading G13)
      put_result<F32>(idx, neg ? F::kSign : 0ull, ST_OK, out, status);
      return;
    }
    // w = the first (up to) 19 significant digits, one per lane; the rest
    // only tells whether a nonzero digit was dropped
    const int64_t cnt = min((int64_t)19, ds.N - ds.z);
    uint64_t w = lane < cnt ? (uint64_t)ds.digit(ds.z + lane) * kSlowPow10[cnt - 1 - lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    Scan sc;
    sc.w = w;
    const int64_t q = exp10 + ds.nI - ds.z - cnt;  // weight of the last digit taken
    sc.q = (int32_t)max((int64_t)-(1 << 30), min((int64_t)(1 << 30), q));
    sc.kind = K_NUM;
    sc.neg = neg;
    sc.tnz = warp_first_nonzero(ds, ds.z + cnt, ds.N) < ds.N;
    const Res r = decide<F32>(sc);
    if (!(r.info & F_PENDING)) {
      put_result<F32>(idx, r.bits, r.info & 0xFF, out, status);
      return;
    }
    cand = r.bits;
  } else {
    ds.z = warp_first_nonzero(ds, 0, ds.N);
  }
  ds.Ex = exp10 - ds.nF + (ds.N - ds.z) - 1;

  const uint64_t r = resolve_cand<F32>(cand, [&](uint64_t a, int f) { return cmp_mid(ds, a, f); });
  put_result<F32>(idx, r | (neg ? F::kSign : 0ull), r == F::kInf ? ST_OVERFLOW : (r == 0 ? ST_UNDERFLOW : ST_OK),
                  out, status);
}

// ---------------------------------------------------------------------------
// Staged records (the common case): the record is buf[s, e) in the warp's
// shared buffer (s < 16, e <= kSlowStage), with 32 writable bytes on either
// side.  The warp classifies the record once into two bit masks -- non-digit
// bytes and nonzero digits -- and every structural question (end of the
// integer / fraction / exponent runs, first nonzero digit, a nonzero digit
// past the 19th) becomes a search of those words, 32 words per warp step.
// The digits are then made one contiguous stream (the integer digits moved
// one byte up onto the '.'), '0'-padded on both sides, so a base-1e9 limb of
// x is one 9-byte window (no per-limb position arithmetic around the point).

constexpr int kSlowStage = 2048;  // record bytes staged in shared memory per warp
constexpr int kSlowMaskWords = kSlowStage / 32 + 2;

// flags (bit 7 of each byte) of digits other than '0', given the word's non-digit flags
__device__ __forceinline__ uint32_t nzdigit80(uint32_t v, uint32_t nd80) {
  const uint32_t t = lop3<LUT_XOR_AND>(v, 0x30303030u, 0x7F7F7F7Fu);       // (v ^ '0'), bit 7 cleared
  const uint32_t nonzero = lop3<LUT_OR_AND>(t + 0x7F7F7F7Fu, v, 0x80808080u);  // byte != '0'
  return nonzero & ~nd80;
}

// nd / nz masks of buf[0, e) (bit i of word g: byte 32 g + i); bytes at and
// past e count as non-digits, so every nd search ends by e
__device__ __forceinline__ void classify_record(const uint8_t* buf, int e, uint32_t* nd, uint32_t* nz) {
  const int lane = threadIdx.x & 31;
  const int ng = (e + 31) >> 5;
  for (int g = lane; g <= ng; g += 32) {
    uint32_t mn = 0xFFFFFFFFu, mz = 0u;
    if (g < ng) {
      const uint4 A = *reinterpret_cast<const uint4*>(buf + 32 * g);
      const uint4 B = *reinterpret_cast<const uint4*>(buf + 32 * g + 16);
      const uint32_t w[8] = {A.x, A.y, A.z, A.w, B.x, B.y, B.z, B.w};
      mn = 0u;
#pragma unroll
      for (int k = 6; k >= 0; k -= 2) {
        const uint32_t n0 = nondigit80(w[k]), n1 = nondigit80(w[k + 1]);
        mn = pack_byte(mn, n0, n1);
        mz = pack_byte(mz, nzdigit80(w[k], n0), nzdigit80(w[k + 1], n1));
      }
      const int rem = e - 32 * g;  // record bytes in this group
      if (rem < 32) {
        mn |= 0xFFFFFFFFu << rem;
        mz &= ~(0xFFFFFFFFu << rem);
      }
    }
    nd[g] = mn;
    nz[g] = mz;
  }
  __syncwarp();
}

// lowest set bit position in [x, lim) of mask words m (lim if none): the
// first word by every lane alike, then 32 words (1 KiB of record) per warp step
__device__ __forceinline__ int warp_next_set(const uint32_t* m, int x, int lim) {
  if (x >= lim) return lim;
  const int lane = threadIdx.x & 31;
  int r = lim;
  const uint32_t v = m[x >> 5] & (0xFFFFFFFFu << (x & 31));
  if (v) {
    r = (x & ~31) + __ffs(v) - 1;
  } else {
    for (int w0 = (x >> 5) + 1; (w0 << 5) < lim; w0 += 32) {
      const int wi = w0 + lane;
      const uint32_t u = (wi << 5) < lim ? m[wi] : 0u;
      const unsigned b = __ballot_sync(0xffffffffu, u != 0u);
      if (b) {
        const int l = __ffs(b) - 1;
        r = ((w0 + l) << 5) + __ffs(__shfl_sync(0xffffffffu, u, l)) - 1;
        break;
      }
    }
  }
  return r < lim ? r : lim;
}

// the fast path's decision for a long record's (w, q, tnz): with a nonzero
// dropped digit, Algorithm 1 on w and w + 1 runs on two
// lanes at once (decide.cuh's logic, one evaluation's instructions)
template <bool F32>
__device__ __forceinline__ Res slow_decide(const Scan& sc) {
  if (!sc.tnz) return decide<F32>(sc);
  const int lane = threadIdx.x & 31;
  uint32_t fl = 0;
  const uint64_t v = alg1<F32>(sc.w + (uint64_t)(lane & 1), sc.q, fl);  // w + 1 <= 10^19 < 2^64
  const uint64_t a = __shfl_sync(0xffffffffu, v, 0), b = __shfl_sync(0xffffffffu, v, 1);
  const uint32_t fa = __shfl_sync(0xffffffffu, fl, 0), fb = __shfl_sync(0xffffffffu, fl, 1);
  uint32_t f = fa | F_BRACKET | (fb & F_TWO);
  if (a != b || ((fa | fb) & F_ABORT)) f |= F_PENDING;
  Res r;
  if (f & F_PENDING) {
    r.bits = a | ((f & F_ABORT) ? kCandNoLower : 0ull);
    r.info = f & ~0xFFu;
  } else {
    r.bits = (sc.neg ? Fmt<F32>::kSign : 0ull) | a;
    r.info = f;
  }
  return r;
}

// Decide the staged record buf[s, e) from candidate cand (kCandUnknown: not
// scanned by the fast kernel); writes out[idx], status[idx].  Warp-collective.
template <bool F32>
__device__ void slow_record_staged(uint8_t* buf, uint32_t* nd, uint32_t* nz, int s, int e, uint64_t cand,
                                   int64_t idx, void* out, uint8_t* status, uint32_t grammar) {
  using F = Fmt<F32>;
  const int lane = threadIdx.x & 31;
  classify_record(buf, e, nd, nz);
  const uint32_t c0 = s < e ? buf[s] : 0u;
  const bool neg = c0 == '-';
  const int p = s + ((c0 == '+' || c0 == '-') ? 1 : 0);
  // structure: digits, '.', digits, (e|E) [sign] digits, terminators
  const int ie = warp_next_set(nd, p, e);
  const bool dot = ie < e && buf[ie] == '.';
  const int fb = dot ? ie + 1 : ie;
  const int fe = dot ? warp_next_set(nd, fb, e) : ie;
  bool number = (ie - p) + (fe - fb) > 0;  // at least one digit
  int64_t exp10 = 0;
  int tail = fe;
  if (fe < e && (buf[fe] | 0x20) == 'e') {
    int k = fe + 1;
    bool en = false;
    if (k < e && (buf[k] == '+' || buf[k] == '-')) {
      en = buf[k] == '-';
      k++;
    }
    const int ke = warp_next_set(nd, k, e);
    number = number && ke > k;
    const int kz = warp_next_set(nz, k, ke);  // leading zeros of the exponent do not count
    const int ne = ke - kz;
    if (ne > 15) exp10 = 1000000000000000ll;  // reading G9: saturated beyond any record's reach
    else if (ne > 9) exp10 = (int64_t)digits_before(buf, ke - 9, ne - 9) * 1000000000ll + digits_before(buf, ke, 9);
    else exp10 = digits_before(buf, ke, ne);
    if (en) exp10 = -exp10;
    tail = ke;
  }
  const int nI = ie - p, nF = fe - fb, N = nI + nF;
  if (cand == kCandUnknown) {
    number = number && !warp_any_nonterm(buf, tail, e);
    if (grammar & G_JSON)  // RFC 8259: no '+', int := '0' | [1-9] digit*, frac := '.' digit+
      number = number && c0 != '+' && nI != 0 && (nI == 1 || buf[p] != '0') && !(dot && nF == 0);
    if (!number) {  // specials, invalid, empty (never undecided): the byte scanner on lane 0
      if (lane == 0) {
        const Res r = decide<F32>(scan_record(buf + s, (uint32_t)(e - s), grammar));
        if (F32) reinterpret_cast<uint32_t*>(out)[idx] = (uint32_t)r.bits;
        else reinterpret_cast<unsigned long long*>(out)[idx] = r.bits;
        status[idx] = (uint8_t)(r.info & 0xFF);
      }
      return;
    }
  }
  // first nonzero digit (the '.' is no digit, so the search crosses it)
  const int zb = warp_next_set(nz, p, fe);
  if (zb >= fe) {  // all digits zero: +-0 (reading G13)
    put_result<F32>(idx, neg ? F::kSign : 0ull, ST_OK, out, status);
    return;
  }
  const int uz = zb < ie ? zb - p : nI + (zb - fb);  // its stream index
  bool tnz = false;
  if (cand == kCandUnknown) {  // a nonzero digit after the first 19 significant ones
    const int u19 = uz + 19;
    tnz = u19 < N && warp_next_set(nz, u19 < nI ? p + u19 : fb + (u19 - nI), fe) < fe;
  }
  // the digit stream: integer digits moved one byte up onto the '.', so that
  // stream index u is byte S + u; '0' on both sides of it (16 bytes)
  if (dot && nI > 0) {
    for (int t0 = (nI - 1) & ~31; t0 >= 0; t0 -= 32) {  // top chunk first: nothing is overwritten unread
      const int t = t0 + lane;
      const uint32_t v = t < nI ? buf[p + t] : 0u;
      __syncwarp();
      if (t < nI) buf[p + t + 1] = (uint8_t)v;
      __syncwarp();
    }
  }
  const int S = dot ? p + 1 : p;
  buf[lane < 16 ? S - 16 + lane : S + N + (lane - 16)] = '0';
  __syncwarp();
  const uint8_t* pb = buf - 32;  // word-aligned base with every read offset >= 0
  if (cand == kCandUnknown) {  // (w, q): the first <= 19 significant digits
    const int cnt = min(19, N - uz);
    Scan sc;
    sc.w = run19(pb, (uint32_t)(32 + S + uz + cnt), cnt);
    const int64_t q = exp10 + nI - uz - cnt;  // weight of the last digit taken
    sc.q = (int32_t)max((int64_t)-(1 << 30), min((int64_t)(1 << 30), q));
    sc.kind = K_NUM;
    sc.neg = neg;
    sc.tnz = tnz;
    const Res r = slow_decide<F32>(sc);
    if (!(r.info & F_PENDING)) {
      put_result<F32>(idx, r.bits, r.info & 0xFF, out, status);
      return;
    }
    cand = r.bits;
  }
  const int64_t Ex = exp10 - nF + (N - uz) - 1;  // decimal exponent of the first nonzero digit
  auto limbx = [&](int64_t u0) -> uint32_t {
    if (u0 >= N || u0 + 9 <= 0) return 0u;
    const uint32_t b = 32u + (uint32_t)(S + (int)u0);
    return ((uint32_t)pb[b] - '0') * 100000000u + dig4(lds4(pb, b + 1)) * 10000u + dig4(lds4(pb, b + 5));
  };
  auto tailnz = [&](int64_t u) -> bool {  // the masks describe the original layout
    if (u >= N) return false;
    const int ui = (int)u;
    return warp_next_set(nz, ui < nI ? p + ui : fb + (ui - nI), fe) < fe;
  };
  const uint64_t r = resolve_cand<F32>(cand, [&](uint64_t a, int f) {
    MidLimbs L;
    mid_limbs(a, f, L);
    return cmp_limbs(L, (int64_t)uz, Ex, limbx, tailnz);
  });
  put_result<F32>(idx, r | (neg ? F::kSign : 0ull), r == F::kInf ? ST_OVERFLOW : (r == 0 ? ST_UNDERFLOW : ST_OK),
                  out, status);
}

struct SlowArgs {
  const uint8_t* bytes;
  int64_t len;
  const int64_t* offsets;  // batch variant: for the ST_PENDING overflow scan; NULL for split
  int64_t n;
  uint32_t seps;
  void* out;  // double[] or (F32) float[]
  uint8_t* status;
  WsHeader* hdr;
  const SlowEntry* queue;
  uint64_t qcap;
  const uint64_t* desc;  // split: the fast kernel's per-tile descriptors (inclusive prefixes)
  int64_t capacity;      // split: output slots
  uint32_t grammar;      // 0 or G_HEX / G_JSON
  int64_t* n_out;        // split: the record count; set to -FPP_ECAPACITY if the queue overflowed
};

#ifndef FPP_SLOW_MINB
#define FPP_SLOW_MINB 8  // 64 registers: 8 CTAs per SM (the register-limited 7 ran 5% slower)
#endif
template <bool F32>
__global__ void __launch_bounds__(kSlowThreads, FPP_SLOW_MINB) k_slow(SlowArgs a) {
  // per warp: 32 pad bytes, kSlowStage bytes, 32 pad bytes (the staged
  // path's '0' padding and 12-byte read-behind windows), and the record's masks
  constexpr int kWarpBuf = kSlowStage + 64;
  __shared__ __align__(16) uint8_t stage[(kSlowThreads / 32) * kWarpBuf];
  __shared__ uint32_t masks[kSlowThreads / 32][2][kSlowMaskWords];
  const int lane = threadIdx.x & 31;
  uint8_t* buf = stage + 32 + (threadIdx.x >> 5) * kWarpBuf;
  uint32_t* nd = masks[threadIdx.x >> 5][0];
  uint32_t* nz = masks[threadIdx.x >> 5][1];
  const unsigned long long qcount = *(volatile unsigned long long*)&a.hdr->qcount;
  const unsigned long long qn = qcount < a.qcap ? qcount : a.qcap;
  const int64_t head = (int64_t)(reinterpret_cast<uintptr_t>(a.bytes) & 15);
  while (true) {
    unsigned int i = 0;
    if (lane == 0) i = atomicAdd(&a.hdr->slow_ctr, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= qn) break;
    const SlowEntry en = a.queue[i];
    int64_t idx = en.idx;
    if (idx < 0) {  // split entry: (tile, j) -> exclusive prefix of the tile + j
      const uint64_t k = ~(uint64_t)idx;
      const int64_t t = (int64_t)(k >> kSplitJBits);
      idx = (int64_t)(k & ((1u << kSplitJBits) - 1));
      if (t > 0) idx += (int64_t)(a.desc[t - 1] & ((1ull << 62) - 1));
      if (idx >= a.capacity) continue;  // counted in n_out, no output slot
    }
    int64_t end = en.end;
    if (end < 0) end = warp_find_sep(a.bytes, en.start, a.len, a.seps);
    // stage the record (16-byte chunks on the absolute 16-byte grid) when it
    // fits: the lexing and digit reads below then hit shared memory
    const int64_t p_al = en.start - ((en.start + head) & 15);
    if (end - p_al <= kSlowStage) {
      const int nch = (int)((end - p_al + 15) >> 4);
      for (int c = lane; c < nch; c += 32) {
        const int64_t q = p_al + 16 * c;
        uint4 v;
        if (q >= 0 && q + 16 <= a.len) {
          v = __ldg(reinterpret_cast<const uint4*>(a.bytes + q));
        } else {  // the buffer's unaligned head or tail: bytes outside [0, len) read as 0
          uint32_t w[4] = {0, 0, 0, 0};
          for (int k = 0; k < 16; k++)
            if (q + k >= 0 && q + k < a.len) w[k >> 2] |= (uint32_t)a.bytes[q + k] << (8 * (k & 3));
          v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        *reinterpret_cast<uint4*>(buf + 16 * c) = v;
      }
      __syncwarp();
      slow_record_staged<F32>(buf, nd, nz, (int)(en.start - p_al), (int)(end - p_al), en.cand, idx, a.out,
                              a.status, a.grammar);
      __syncwarp();
    } else {
      slow_record_global<F32>(a.bytes, en.start, end, en.cand, idx, a.out, a.status, a.grammar);
    }
  }
  // The split queue cannot overflow (every queued
  // record is at least 20 bytes long); should it ever, the dropped records'
  // results are wrong, so the call fails loudly: *n_out = -3 (-FPP_ECAPACITY)
  if (qcount > a.qcap && a.offsets == nullptr && a.n_out != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    *a.n_out = -3;
  if (qcount > a.qcap && a.offsets != nullptr) {  // batch queue overflow: scan for marks
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = wid; r < a.n; r += nw) {
      const uint8_t mk = a.status[r];
      if (mk < ST_PENDING_UNK) continue;
      const int64_t s = a.offsets[r];
      const int64_t e = r + 1 < a.n ? a.offsets[r + 1] : a.len;
      uint64_t cand = F32 ? (uint64_t)reinterpret_cast<const uint32_t*>(a.out)[r]
                          : (uint64_t)reinterpret_cast<const unsigned long long*>(a.out)[r];
      if (mk == ST_PENDING_LOW) cand |= kCandNoLower;
      if (mk == ST_PENDING_UNK) cand = kCandUnknown;
      slow_record_global<F32>(a.bytes, s, e, cand, r, a.out, a.status, a.grammar);
    }
  }
}

}  // namespace fpp
