// k_slow.cuh -- exact slow path.
//
// The paper falls back on an exact higher-precision conversion when the
// 19-digit bracket w / w+1 disagrees or Algorithm 1 aborts ("its performance
// is secondary. However, it has to be exact", L986-987).  Here the fast
// kernels queue those records (and every record longer than 64 bytes,
// unscanned), and two kernels decide them:
//   k_slow_scan  a THREAD per queued record: structure (SWAR over global
//                memory), the first 19 significant digits, the fast path's
//                decision; undecided records become descriptors in place;
//   k_slow       a WARP per undecided record: the value x of the whole digit
//                string lies in [w*10^q, (w+1)*10^q), an interval far narrower
//                than one ulp, so by monotonicity the result is the candidate
//                r0 = Alg1(w, q) or its successor (when Algorithm 1 aborted,
//                the un-aborted product is within one ulp and both neighbours
//                are checked).  The warp compares x exactly with the midpoint
//                    M = (2m+1) * 2^(e-1),   r0 = m * 2^e,
//                whose decimal digits (2m+1) * 5^(1-e) (e < 1) or
//                (2m+1) * 2^(e-1) it forms in base-1e9 limbs from exact power
//                tables (tables/declimbs.inc), one limb per lane, carries
//                resolved with a ballot carry-lookahead, then limb by limb:
//                x < M -> r0, x > M -> successor, x == M -> the one with the
//                even significand (ties to even, also for subnormals and at the
//                overflow threshold 2^1024 - 2^970; readings G3, G12).
// slow_record_global (one warp, global memory) serves the batch variant's
// queue-overflow marks.
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

constexpr int kSlowStage = 2048;  // record bytes staged in shared memory per warp

// flags (bit 7 of each byte) of digits other than '0', given the word's non-digit flags
__device__ __forceinline__ uint32_t nzdigit80(uint32_t v, uint32_t nd80) {
  const uint32_t t = lop3<LUT_XOR_AND>(v, 0x30303030u, 0x7F7F7F7Fu);       // (v ^ '0'), bit 7 cleared
  const uint32_t nonzero = lop3<LUT_OR_AND>(t + 0x7F7F7F7Fu, v, 0x80808080u);  // byte != '0'
  return nonzero & ~nd80;
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
  SlowEntry* queue;       // rewritten in place by k_slow_scan (two-phase slow path)
  uint64_t qcap;
  const uint64_t* desc;  // split: the fast kernel's per-tile descriptors (inclusive prefixes)
  int64_t capacity;      // split: output slots
  uint32_t grammar;      // 0 or G_HEX / G_JSON
  int64_t* n_out;        // split: the record count; set to -FPP_ECAPACITY if the queue overflowed
};

// ---------------------------------------------------------------------------
// Two-phase slow path (round 2).  Phase A, k_slow_scan: every queued record
// goes to ONE THREAD, which finds its structure with 16-byte SWAR steps over
// global memory, takes the first 19 significant digits and runs the fast
// path's decision (Algorithm 1 with the w / w+1 bracket);
// specials and invalid records go to the byte scanner.  A decided record is
// written and its queue entry marked done; an undecided one is rewritten in
// place as a descriptor of its digit stream.  Phase B, k_slow: one WARP per
// undecided record for the exact midpoint comparison (the limb arithmetic is
// the part that needs 32 lanes).  The scalar work of a record -- about 800 of
// the 1177 warp instructions the one-warp-per-record kernel spent -- thus
// runs once per record instead of once per lane.
//
// Descriptor (SlowEntry rewritten in place):
//   idx   -1 (done), else (output index << 24) | (Ex + 2^23) (Ex clamped to
//         +-(2^23 - 1): only compared with the midpoint's exponent, |EM| < 400)
//   start position of the first integer digit (ib), bits 0..46; bits 47..63:
//         the stream index of the first nonzero digit (saturated at 2^17 - 1)
//   end   (nI << 33) | (nF << 2) | (dot << 1) | neg
//   cand  candidate (bit 63: kCandNoLower)

// 16-bit flag mask of the 16 bytes v (bit i: byte i)
template <typename F>
__device__ __forceinline__ uint32_t chunk_mask16(const uint4 v, F flag80) {
  uint32_t m = pack_byte(0u, flag80(v.z), flag80(v.w));
  return pack_byte(m, flag80(v.x), flag80(v.y)) & 0xFFFFu;
}

// first position in [from, to) whose byte's flag is set (to if none);
// per thread, 16 bytes per step on the buffer's 16-byte grid (head = bytes % 16)
template <typename F>
__device__ __forceinline__ int64_t thr_find(const uint8_t* bytes, int64_t len, int64_t head, int64_t from, int64_t to,
                                           F flag80) {
  if (from >= to) return to;
  for (int64_t c = from - ((from + head) & 15); c < to; c += 16) {
    uint32_t m = chunk_mask16(load_chunk(bytes, len, c), flag80);
    if (c < from) m &= 0xFFFFu << (int)(from - c);
    if (m) {
      const int64_t r = c + __ffs(m) - 1;
      return r < to ? r : to;
    }
  }
  return to;
}

// bytes equal to c (exact zero-byte test of v ^ c...c)
__device__ __forceinline__ uint32_t eq80(uint32_t v, uint32_t c4) {
  const uint32_t x = v ^ c4;
  const uint32_t t = x & 0x7F7F7F7Fu;
  return lop3<LUT_NOR_AND>(t + 0x7F7F7F7Fu, x, 0x80808080u);
}
// separators of the split variant (seps: bit0 '\n', bit1 ','), a runtime mask
__device__ __forceinline__ uint32_t sep80v(uint32_t v, uint32_t seps) {
  uint32_t h = 0;
  if (seps & 1u) h |= eq80(v, 0x0A0A0A0Au);
  if (seps & 2u) h |= eq80(v, 0x2C2C2C2Cu);
  return h;
}
// bytes that are not terminators ('\n', '\r', ',')
__device__ __forceinline__ uint32_t nonterm80(uint32_t v) {
  return ~(eq80(v, 0x0A0A0A0Au) | eq80(v, 0x0D0D0D0Du) | eq80(v, 0x2C2C2C2Cu)) & 0x80808080u;
}

template <bool F32>
__device__ __forceinline__ void thr_put(int64_t idx, uint64_t bits, uint32_t st, void* out, uint8_t* status) {
  if (F32) reinterpret_cast<uint32_t*>(out)[idx] = (uint32_t)bits;
  else reinterpret_cast<unsigned long long*>(out)[idx] = bits;
  status[idx] = (uint8_t)st;
}

template <bool F32>
__global__ void __launch_bounds__(kSlowThreads) k_slow_scan(SlowArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned long long qcount = *(volatile unsigned long long*)&a.hdr->qcount;
  const unsigned long long qn = qcount < a.qcap ? qcount : a.qcap;
  const int64_t head = (int64_t)(reinterpret_cast<uintptr_t>(a.bytes) & 15);
  const uint8_t* B = a.bytes;
  const int64_t len = a.len;
  auto nondig = [](uint32_t v) { return nondigit80(v); };
  auto nzdig = [](uint32_t v) { return nzdigit80(v, nondigit80(v)); };
  while (true) {
    unsigned int b0 = 0;
    if (lane == 0) b0 = atomicAdd(&a.hdr->scan_ctr, 32u);
    b0 = __shfl_sync(0xffffffffu, b0, 0);
    if (b0 >= qn) break;
    const unsigned long long qi = b0 + lane;
    if (qi >= qn) continue;
    SlowEntry& E = a.queue[qi];
    const SlowEntry en = E;
    int64_t idx = en.idx;
    if (idx < 0) {  // split entry: (tile, j) -> exclusive prefix of the tile + j
      const uint64_t k = ~(uint64_t)idx;
      const int64_t t = (int64_t)(k >> kSplitJBits);
      idx = (int64_t)(k & ((1u << kSplitJBits) - 1));
      if (t > 0) idx += (int64_t)(a.desc[t - 1] & ((1ull << 62) - 1));
      if (idx >= a.capacity) {  // counted in n_out, no output slot
        E.idx = -1;
        continue;
      }
    }
    const int64_t s = en.start;
    int64_t e = en.end;
    if (e < 0) e = thr_find(B, len, head, s, len, [&](uint32_t v) { return sep80v(v, a.seps); });
    // the record's cache lines requested at once (its searches then hit L1
    // instead of waiting on one line after the other)
    for (int64_t l = s & ~(int64_t)127; l < e && l < s + 2048; l += 128)
      asm volatile("prefetch.global.L1 [%0];" ::"l"(B + (l > s ? l : s)));
    uint64_t cand = en.cand;
    if (e - s >= (1ll << 31)) {  // records of 2^31 bytes or more are unsupported (R2): INVALID
      thr_put<F32>(idx, Fmt<F32>::kQNaN, ST_INVALID, a.out, a.status);
      E.idx = -1;
      continue;
    }
    // structure
    const uint32_t c0 = s < e ? B[s] : 0u;
    const bool neg = c0 == '-';
    const int64_t p = s + ((c0 == '+' || c0 == '-') ? 1 : 0);
    const int64_t ie = thr_find(B, len, head, p, e, nondig);
    const bool dot = ie < e && B[ie] == '.';
    const int64_t fb = dot ? ie + 1 : ie;
    const int64_t fe = dot ? thr_find(B, len, head, fb, e, nondig) : ie;
    bool number = (ie - p) + (fe - fb) > 0;
    int64_t exp10 = 0, tail = fe;
    if (fe < e && (B[fe] | 0x20) == 'e') {
      int64_t k = fe + 1;
      bool en2 = false;
      if (k < e && (B[k] == '+' || B[k] == '-')) {
        en2 = B[k] == '-';
        k++;
      }
      const int64_t ke = thr_find(B, len, head, k, e, nondig);
      number = number && ke > k;
      const int64_t kz = thr_find(B, len, head, k, ke, nzdig);  // leading zeros do not count
      if (ke - kz > 15) {
        exp10 = 1000000000000000ll;  // reading G9: saturated beyond any record's reach
      } else {
        for (int64_t t = kz; t < ke; t++) exp10 = exp10 * 10 + (B[t] - '0');
      }
      if (en2) exp10 = -exp10;
      tail = ke;
    }
    const int64_t nI = ie - p, nF = fe - fb, N = nI + nF;
    if (cand == kCandUnknown) {
      if (number) number = thr_find(B, len, head, tail, e, [](uint32_t v) { return nonterm80(v); }) >= e;
      if (a.grammar & G_JSON)  // RFC 8259: no '+', int := '0' | [1-9] digit*, frac := '.' digit+
        number = number && c0 != '+' && nI != 0 && (nI == 1 || B[p] != '0') && !(dot && nF == 0);
      if (!number) {  // specials, invalid, empty: the byte scanner
        Scan sc;
        if (e - s >= (1ll << 31)) {
          sc.kind = K_INVALID; sc.neg = false; sc.tnz = false; sc.w = 0; sc.q = 0;
        } else {
          sc = scan_record(B + s, (uint32_t)(e - s), a.grammar);
        }
        const Res r = decide<F32>(sc);
        thr_put<F32>(idx, r.bits, r.info & 0xFF, a.out, a.status);
        E.idx = -1;
        continue;
      }
    }
    // first nonzero digit (the '.' is no digit, so the search crosses it)
    const int64_t zb = thr_find(B, len, head, p, fe, nzdig);
    if (zb >= fe) {  // all digits zero: +-0 (reading G13)
      thr_put<F32>(idx, neg ? Fmt<F32>::kSign : 0ull, ST_OK, a.out, a.status);
      E.idx = -1;
      continue;
    }
    const int64_t uz = zb < ie ? zb - p : nI + (zb - fb);  // its stream index
    const int64_t Ex = exp10 - nF + (N - uz) - 1;          // its decimal exponent
    if (cand == kCandUnknown) {  // (w, q, tnz): the first <= 19 significant digits
      const int64_t cnt = min((int64_t)19, N - uz);
      uint64_t w = 0;
      int64_t u = uz, pos = zb;
      for (int t = 0; t < (int)cnt; t++) {
        if (pos == ie && dot) pos++;  // skip the point
        w = w * 10 + (B[pos] - '0');
        pos++;
        u++;
      }
      Scan sc;
      sc.w = w;
      const int64_t q = exp10 + nI - uz - cnt;  // weight of the last digit taken
      sc.q = (int32_t)max((int64_t)-(1 << 30), min((int64_t)(1 << 30), q));
      sc.kind = K_NUM;
      sc.neg = neg;
      sc.tnz = false;
      if (u < N) {  // a nonzero digit after the 19th significant one
        if (pos == ie && dot) pos++;
        sc.tnz = thr_find(B, len, head, pos, fe, nzdig) < fe;
      }
      const Res r = decide<F32>(sc);
      if (!(r.info & F_PENDING)) {
        thr_put<F32>(idx, r.bits, r.info & 0xFF, a.out, a.status);
        E.idx = -1;
        continue;
      }
      cand = r.bits;
    }
    const int64_t Exc = max((int64_t)-(1 << 23) + 1, min((int64_t)(1 << 23) - 1, Ex));
    SlowEntry d;
    d.idx = (idx << 24) | (int64_t)((Exc + (1 << 23)) & 0xFFFFFF);
    d.start = p | ((uz < (1 << 17) - 1 ? uz : (int64_t)((1 << 17) - 1)) << 47);  // uz saturated: recomputed
    d.end = (int64_t)(((uint64_t)nI << 33) | ((uint64_t)nF << 2) | ((dot ? 1ull : 0ull) << 1) | (neg ? 1ull : 0ull));
    d.cand = cand;
    E = d;
  }
}

#ifndef FPP_SLOW_MINB
#define FPP_SLOW_MINB 8  // 64 registers: 8 CTAs per SM
#endif

// Phase B: one warp per record k_slow_scan left undecided (descriptor, above):
// the exact comparison of x with the midpoint(s) of the candidate.  (Tried:
// static striding with the next record copied by cp.async into a second
// buffer during the comparison: 6.05 ms against 5.47 ms on config 5 -- the
// next entry's load still stalled, and two buffers per warp cost occupancy.)
template <bool F32>
__global__ void __launch_bounds__(kSlowThreads, FPP_SLOW_MINB) k_slow(SlowArgs a) {
  // per warp: 32 pad bytes, kSlowStage bytes, 32 pad bytes
  // ('0' padding and the 9-byte windows around the digit stream)
  constexpr int kWarpBuf = kSlowStage + 64;
  __shared__ __align__(16) uint8_t stage_mem[(kSlowThreads / 32) * kWarpBuf];
  const int lane = threadIdx.x & 31;
  uint8_t* const buf0 = stage_mem + 32 + (threadIdx.x >> 5) * kWarpBuf;
  const unsigned long long qcount = *(volatile unsigned long long*)&a.hdr->qcount;
  const long long qn = (long long)(qcount < a.qcap ? qcount : a.qcap);
  const int64_t head = (int64_t)(reinterpret_cast<uintptr_t>(a.bytes) & 15);

  // copy an entry's record into buf; true if it is staged
  auto stage = [&](const SlowEntry& en, uint8_t* b) -> bool {
    const int64_t ib = en.start & ((1ll << 47) - 1), uzs = en.start >> 47;
    const uint64_t pk = (uint64_t)en.end;
    const int64_t e = ib + (int64_t)(pk >> 33) + (int64_t)((pk >> 1) & 1ull) + (int64_t)((pk >> 2) & 0x7FFFFFFFull);
    const int64_t p_al = ib - ((ib + head) & 15);
    if (e - p_al > kSlowStage || uzs >= (1 << 17) - 1) return false;
    const int nch = (int)((e - p_al + 15) >> 4);
    for (int c = lane; c < nch; c += 32)
      *reinterpret_cast<uint4*>(b + 16 * c) = load_chunk(a.bytes, a.len, p_al + 16 * c);
    __syncwarp();
    return true;
  };

#ifndef FPP_SLOW_CTRS
#define FPP_SLOW_CTRS 8  // claim counters: one counter's same-address atomics queued at ~1.5 G/s
#endif
  // warp w claims from counter w mod G, which hands out entries g, g + G, ...
  const int g = (int)((((unsigned)blockIdx.x * blockDim.x + threadIdx.x) >> 5) % FPP_SLOW_CTRS);
  unsigned int* const ctr = FPP_SLOW_CTRS > 1 ? slow_ctr_g(a.hdr, g) : &a.hdr->slow_ctr;
  while (true) {
    unsigned long long i = 0;
    if (lane == 0) i = (unsigned long long)atomicAdd(ctr, 1u) * FPP_SLOW_CTRS + (FPP_SLOW_CTRS > 1 ? g : 0);
    i = __shfl_sync(0xffffffffu, i, 0);
    if ((long long)i >= qn) break;
    const SlowEntry cur = a.queue[i];
    if (cur.idx < 0) continue;  // decided by k_slow_scan (or no output slot)
    const bool cur_st = stage(cur, buf0);
    {
      uint8_t* buf = buf0;
      const int64_t oidx = cur.idx >> 24;
      const uint64_t pk = (uint64_t)cur.end;
      const int64_t ib = cur.start & ((1ll << 47) - 1), uzs = cur.start >> 47;
      const int64_t nI = (int64_t)(pk >> 33), nF = (int64_t)((pk >> 2) & 0x7FFFFFFFull);
      const int dot = (int)((pk >> 1) & 1ull);
      const int64_t fb = ib + nI + dot, N = nI + nF;
      const int64_t Ex = (int64_t)(cur.idx & 0xFFFFFF) - (1 << 23);
      const bool neg = (pk & 1ull) != 0;
      uint64_t r;
      if (cur_st) {
        // the digits made one '0'-padded stream (the integer digits moved
        // onto the '.'): stream digit u is byte S + u, a limb one 9-byte window
        const int p = (int)((ib + head) & 15), nIi = (int)nI, Ni = (int)N;
        if (dot && nIi > 0) {
          for (int t0 = (nIi - 1) & ~31; t0 >= 0; t0 -= 32) {  // top chunk first: nothing overwritten unread
            const int t = t0 + lane;
            const uint32_t v = t < nIi ? buf[p + t] : 0u;
            __syncwarp();
            if (t < nIi) buf[p + t + 1] = (uint8_t)v;
            __syncwarp();
          }
        }
        const int S = p + dot;
        buf[lane < 16 ? S - 16 + lane : S + Ni + (lane - 16)] = '0';
        __syncwarp();
        const uint8_t* pb = buf - 32;
        auto limbx = [&](int64_t u0) -> uint32_t {
          if (u0 >= Ni || u0 + 9 <= 0) return 0u;
          const uint32_t b = 32u + (uint32_t)(S + (int)u0);
          return ((uint32_t)pb[b] - '0') * 100000000u + dig4(lds4(pb, b + 1)) * 10000u + dig4(lds4(pb, b + 5));
        };
        auto tailnz = [&](int64_t u) -> bool {  // a nonzero digit at stream index >= u
          for (int64_t u0 = u; u0 < Ni; u0 += 32) {
            const int64_t uu = u0 + lane;
            if (__ballot_sync(0xffffffffu, uu < Ni && buf[S + (int)uu] != '0')) return true;
          }
          return false;
        };
        r = resolve_cand<F32>((uint64_t)cur.cand, [&](uint64_t aa, int ff) {
          MidLimbs L;
          mid_limbs(aa, ff, L);
          return cmp_limbs(L, uzs, Ex, limbx, tailnz);
        });
      } else {  // too long to stage: the digits read from global memory
        DigitStream ds;
        ds.bytes = a.bytes;
        ds.ib = ib;
        ds.nI = nI;
        ds.nF = nF;
        ds.fb = fb;
        ds.N = N;
        ds.z = warp_first_nonzero(ds, 0, ds.N);
        ds.Ex = Ex;
        r = resolve_cand<F32>((uint64_t)cur.cand, [&](uint64_t aa, int ff) { return cmp_mid(ds, aa, ff); });
      }
      put_result<F32>(oidx, r | (neg ? Fmt<F32>::kSign : 0ull),
                      r == Fmt<F32>::kInf ? ST_OVERFLOW : (r == 0 ? ST_UNDERFLOW : ST_OK), a.out, a.status);
    }
    __syncwarp();  // done with the buffer before it is refilled
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
