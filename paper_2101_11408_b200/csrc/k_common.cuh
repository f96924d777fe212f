// k_common.cuh -- helpers shared by the fast kernels (k_split.cuh, k_batch.cuh):
// byte staging, SWAR classification into bit masks, the warp-aggregated slow
// queue push, the decoupled look-back over published tile counts, and the
// per-record parse (common-case parser -> general scanner -> Algorithm 1).
#pragma once
#include "fastrec.cuh"

namespace fpp {

constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

struct StatAcc {
  uint32_t v[NSTATS];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < NSTATS; i++) v[i] = 0;
  }
};

__device__ __forceinline__ void flush_stats(StatAcc& acc, uint64_t* stats) {
#pragma unroll
  for (int i = 0; i < NSTATS; i++) {
    uint32_t x = acc.v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd((unsigned long long*)&stats[i], (unsigned long long)x);
  }
}

template <bool STATS>
__device__ __forceinline__ void count_stats(StatAcc& acc, const Res& r, bool global) {
  if (!STATS) return;
  acc.v[STAT_RECORDS]++;
  acc.v[STAT_TWO_MULT] += (r.info & F_TWO) ? 1u : 0u;
  acc.v[STAT_BRACKET] += (r.info & F_BRACKET) ? 1u : 0u;
  acc.v[STAT_ABORT] += (r.info & F_ABORT) ? 1u : 0u;
  acc.v[STAT_SLOW] += (r.info & F_PENDING) ? 1u : 0u;
  const uint32_t st = r.info & 0xFF;
  acc.v[STAT_BAD] += (st == ST_INVALID || st == ST_EMPTY) ? 1u : 0u;
  acc.v[STAT_GLOBAL] += global ? 1u : 0u;
}

// 16 bytes at position p (absolute-aligned), zero outside [0, len)
__device__ __forceinline__ uint4 load_chunk(const uint8_t* __restrict__ bytes, int64_t len, int64_t p) {
  if (p >= 0 && p + 16 <= len) return __ldg(reinterpret_cast<const uint4*>(bytes + p));
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 16; k++) {
    int64_t q = p + k;
    uint32_t b = (q >= 0 && q < len) ? bytes[q] : 0u;
    w[k >> 2] |= b << (8 * (k & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// masks for 32 staged bytes (two 16-byte words): non-digit and separator bits.
// Two words' flags are packed per multiply: f = flags(w1) + flags(w0) >> 4
// puts w0's at bits 3, 11, 19, 27 and w1's at 7, 15, 23, 31; times 0x00204081
// (no carries: the twenty partial-product bits are distinct) gathers them
// into the top byte as w0 byte 0..3, w1 byte 0..3.
__device__ __forceinline__ uint32_t pack_byte(uint32_t acc, uint32_t f80_lo, uint32_t f80_hi) {
  return __funnelshift_l((f80_hi + (f80_lo >> 4)) * 0x00204081u, acc, 8);
}
#ifndef FPP_PACK
#define FPP_PACK 2  // 2: flags gathered by dp4a (weights 1, 2, 4, ..., 128 per pair of words); 1: the multiply gather
#endif
__device__ __forceinline__ uint32_t dp4a_uu(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
// the 32-bit mask of eight words' flags (0x80 per byte): each pair of words
// gives its 8 bits times 128 by two dp4a, the four pairs are joined by
// multiply-adds
__device__ __forceinline__ uint32_t pack32_dp(const uint32_t* f) {
  uint32_t r[4];
#pragma unroll
  for (int p = 0; p < 4; p++) r[p] = dp4a_uu(f[2 * p + 1], 0x80402010u, dp4a_uu(f[2 * p], 0x08040201u, 0u));
  uint32_t t = r[3] * 256u + r[2];
  t = t * 256u + r[1];
  return t * 2u + (r[0] >> 7);
}
template <uint32_t SEPS>
__device__ __forceinline__ void classify32(const uint4 a, const uint4 b, uint32_t& nd, uint32_t& sp) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#if FPP_PACK == 2
  uint32_t fn[8], fs[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    fn[k] = nondigit80(w[k]);
    fs[k] = SEPS ? sep80<SEPS>(w[k]) : 0u;
  }
  nd = pack32_dp(fn);
  sp = SEPS ? pack32_dp(fs) : 0u;
  return;
#endif
  nd = 0;
  sp = 0;
#pragma unroll
  for (int k = 6; k >= 0; k -= 2) {
    nd = pack_byte(nd, nondigit80(w[k]), nondigit80(w[k + 1]));
    if (SEPS) sp = pack_byte(sp, sep80<SEPS>(w[k]), sep80<SEPS>(w[k + 1]));
  }
}

__device__ __forceinline__ uint32_t mask_at(const uint32_t* m, uint32_t x) {
  return __funnelshift_r(m[x >> 5], m[(x >> 5) + 1], x & 31);
}

// warp-aggregated push onto the slow queue (all lanes call); false if full
__device__ __forceinline__ bool queue_push(bool want, WsHeader* hdr, SlowEntry* q, uint64_t qcap,
                                           const SlowEntry& e) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (m == 0) return true;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&hdr->qcount, (unsigned long long)__popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (!want) return true;
  const unsigned long long slot = base + __popc(m & ((1u << lane) - 1));
  if (slot >= qcap) return false;
  q[slot] = e;
  return true;
}

// push from the lanes that are active here (a rare, divergent branch): they
// aggregate their slots with one atomicAdd
__device__ __forceinline__ void queue_push_active(WsHeader* hdr, SlowEntry* q, uint64_t qcap, const SlowEntry& e) {
  const unsigned m = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&hdr->qcount, (unsigned long long)__popc(m));
  base = __shfl_sync(m, base, leader);
  const unsigned long long slot = base + __popc(m & ((1u << lane) - 1));
  if (slot < qcap) q[slot] = e;
}

// the same out of line (rare: keeps the caller's hot loop small)
__device__ __noinline__ void queue_push_cold(WsHeader* hdr, SlowEntry* q, uint64_t qcap, SlowEntry e) {
  queue_push_active(hdr, q, qcap, e);
}

// decoupled look-back (one warp); the tile's aggregate was published earlier.
// Returns the exclusive prefix and publishes the inclusive one.
// Forward progress: a predecessor that stays unpublished for kSpinLimit
// polls (its tile may not be claimed yet: its claim counter's CTAs are not
// resident, e.g. another kernel holds the SMs) gets its aggregate computed
// here from global memory (count(t), all lanes) and published by CAS, so no
// warp ever waits on a tile that is not running.
#ifndef FPP_SPIN_LIMIT
#define FPP_SPIN_LIMIT 2048  // a test build sets 1: every wait takes the fallback at once
#endif
constexpr int kSpinLimit = FPP_SPIN_LIMIT;
#ifndef FPP_LB_DIAG
#define FPP_LB_DIAG 0  // experiment: count look-back windows / spins in the stats (STAT_GLOBAL / STAT_BAD)
#endif
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// hook: called once the first window's descriptor loads are issued (and after
// every re-read), before their values are used -- work that overlaps the L2
// round trip (k_split: the next tile's claim and L2 prefetch)
template <typename CountFn, typename Hook = NoHook>
__device__ __forceinline__ int64_t lookback(uint64_t* desc, int64_t tile, uint64_t agg, CountFn count,
                                            uint32_t* diag = nullptr, Hook hook = Hook()) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;  // published as inclusive at count time
  uint64_t excl = 0;
  int64_t look = tile - 1;
  int spins = 0;
#ifndef FPP_LB_K
#define FPP_LB_K 2  // windows of 32 predecessors read per L2 round trip (0: the round-1 loop)
#endif
#if FPP_LB_K >= 1
  // K windows per round trip, used nearest first; a window with an
  // unpublished predecessor (before the first inclusive one) is re-read
  while (true) {
    uint64_t dk[FPP_LB_K];
#pragma unroll
    for (int h = 0; h < FPP_LB_K; h++) {
      const int64_t t = look - 32 * h - lane;
      dk[h] = (t >= 0) ? ld_relaxed_u64(&desc[t]) : kFlagInc;
    }
    hook();
    bool done = false;
#pragma unroll
    for (int h = 0; h < FPP_LB_K; h++) {
      const uint64_t d = dk[h];
      const unsigned inc = __ballot_sync(0xffffffffu, (d >> 62) == 2);
      const unsigned zero = __ballot_sync(0xffffffffu, (d >> 62) == 0);
      const unsigned upto = inc ? ((inc & (0u - inc)) << 1) - 1 : 0xffffffffu;
      if (FPP_LB_DIAG && diag) diag[0]++;
      if (zero & upto) {
        if (FPP_LB_DIAG && diag) diag[1]++;
        if (++spins < kSpinLimit) {
          __nanosleep(100);
        } else {
          const int64_t u = look - (__ffs(zero & upto) - 1);
          const uint64_t c = (uint64_t)count(u);
          if (lane == 0)
            atomicCAS(reinterpret_cast<unsigned long long*>(&desc[u]), 0ull, (unsigned long long)(kFlagAgg | c));
          __syncwarp();
        }
        break;  // re-read from look
      }
      // aggregates (tile counts, < 2^13) of the lanes before the first
      // inclusive prefix, plus that prefix (64-bit) from its lane
      const unsigned before = upto & ~inc;
      excl += __reduce_add_sync(0xffffffffu, ((before >> lane) & 1) ? (unsigned)(d & kValMask) : 0u);
      if (inc) excl += __shfl_sync(0xffffffffu, d & kValMask, __ffs(inc) - 1);
      look -= 32;
      if (inc) {
        done = true;
        break;
      }
    }
    if (done) break;
  }
#else
  while (true) {
    const int64_t t = look - lane;
    const uint64_t d = (t >= 0) ? ld_relaxed_u64(&desc[t]) : kFlagInc;
    const unsigned inc = __ballot_sync(0xffffffffu, (d >> 62) == 2);
    const unsigned zero = __ballot_sync(0xffffffffu, (d >> 62) == 0);
    const unsigned upto = inc ? ((inc & (0u - inc)) << 1) - 1 : 0xffffffffu;  // lanes <= first inclusive
    if (FPP_LB_DIAG && diag) diag[0]++;
    if (zero & upto) {  // a predecessor has not published yet: back off, re-read
      if (FPP_LB_DIAG && diag) diag[1]++;
      if (++spins < kSpinLimit) {
        __nanosleep(100);
      } else {  // rare: compute the nearest unpublished predecessor's aggregate ourselves
        const int64_t u = look - (__ffs(zero & upto) - 1);
        const uint64_t c = (uint64_t)count(u);
        if (lane == 0)
          atomicCAS(reinterpret_cast<unsigned long long*>(&desc[u]), 0ull, (unsigned long long)(kFlagAgg | c));
        __syncwarp();
      }
      continue;
    }
    uint64_t v = ((upto >> lane) & 1) ? (d & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    look -= 32;
  }
#endif
  if (lane == 0) st_relaxed_u64(&desc[tile], kFlagInc | (excl + agg));
  return (int64_t)excl;
}

// scan + decide one record whose bytes are text[ts, ts+L) in shared memory:
// the common-case parser, else the general one (fastrec.cuh).  TERM: a
// trailing terminator byte may be part of the record (batch offsets).
// G: the grammar option the kernel is instantiated for (0 default, G_HEX:
// hex floats tried first, G_JSON: the JSON checks in the common-case parser)
template <bool TERM, bool F32, int G = 0>
__device__ __forceinline__ Res parse_staged(const uint8_t* text, uint32_t ts, uint32_t L, uint32_t ndw,
                                            const uint64_t* p10, uint32_t grammar) {
  Res r;
  if (G == (int)G_HEX && fast_hex<F32>(text, ts, L, ndw, r)) return r;
  if (!fast_record<TERM, F32, G == (int)G_JSON>(text, ts, L, ndw, p10, r))
    r = parse_general<F32>(text, ts, L, ndw, p10, grammar);
  return r;
}

// a long record: queued for the slow kernel with no candidate
__device__ __forceinline__ Res long_record() {
  Res r;
  r.bits = kCandUnknown;
  r.info = F_PENDING;
  return r;
}

template <bool F32>
__device__ __noinline__ Res parse_global(const uint8_t* bytes, int64_t s, int64_t e, uint32_t grammar) {
  Scan sc;
  if (e - s >= (1ll << 31)) {
    sc.kind = K_INVALID; sc.neg = false; sc.tnz = false; sc.w = 0; sc.q = 0;
  } else {
    sc = scan_record(bytes + s, (uint32_t)(e - s), grammar);
  }
  return decide<F32>(sc);
}

}  // namespace fpp
