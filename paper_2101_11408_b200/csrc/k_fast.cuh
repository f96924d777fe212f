// k_fast.cuh -- the fast kernels: record splitter + scanner + Algorithm 1.
//
// k_split (parse_f64_split), persistent CTAs of 256 threads, 16 KiB tiles
// claimed in order (atomicAdd), each thread owning 64 bytes of a tile:
//   1. stage: the NEXT tile is prefetched by one TMA bulk copy
//      (cp.async.bulk + mbarrier) into the other half of a double buffer while
//      this one is processed (byte loads only for the ragged first/last tiles);
//   2. classify: each thread reads its 64 bytes once and packs two bit masks,
//      separators (record starts) and non-digits (record structure);
//   3. split: popc + block exclusive scan compact the record starts; thread 0
//      publishes the tile's record count for the decoupled look-back;
//   4. parse: warp 0 first resolves the tile's global record index (look-back)
//      while all warps parse one record per thread -- SWAR scanner
//      (fastscan.cuh) + Algorithm 1 (+ the 19-digit bracket) -- into a
//      shared-memory result buffer;
//   5. write out coalesced; undecided records go to the slow queue with a
//      warp-aggregated atomicAdd.
// Tiles with more than kStartsCap records (records < 4 bytes on average) take
// a dense path: look-back first, then each thread parses the records starting
// in its own 64 bytes and writes them directly.
// k_batch (parse_f64_batch): tiles of 512 records; the covered text span is
// staged by TMA when the tile's offsets are well formed; same classify/parse.
#pragma once
#include "decide.cuh"
#include "fastscan.cuh"

namespace fpp {

constexpr int kBytesPerThread = 64;
constexpr int kSplitHalo = 128;                 // bytes staged beyond the tile

constexpr int kBatchThreads = 256;
constexpr int kBatchRecs = 512;                 // records per tile
constexpr int kBatchText = 16384;               // staged text capacity per tile
constexpr int kBatchMaskWords = kBatchText / 32;

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

// masks for 32 staged bytes (two 16-byte words): non-digit and separator bits
template <uint32_t SEPS>
__device__ __forceinline__ void classify32(const uint4 a, const uint4 b, uint32_t& nd, uint32_t& sp) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  nd = 0;
  sp = 0;
#pragma unroll
  for (int k = 7; k >= 0; k--) {
    nd = pack_nibble(nd, nondigit80(w[k]));
    if (SEPS) sp = pack_nibble(sp, sep80<SEPS>(w[k]));
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

// decoupled look-back (one warp); the tile's aggregate was published earlier.
// Returns the exclusive prefix and publishes the inclusive one.
__device__ __forceinline__ int64_t lookback(uint64_t* desc, int64_t tile, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;  // published as inclusive at count time
  uint64_t excl = 0;
  int64_t look = tile - 1;
  while (true) {
    const int64_t t = look - lane;
    const uint64_t d = (t >= 0) ? ld_relaxed_u64(&desc[t]) : kFlagInc;
    const unsigned inc = __ballot_sync(0xffffffffu, (d >> 62) == 2);
    const unsigned zero = __ballot_sync(0xffffffffu, (d >> 62) == 0);
    const unsigned upto = inc ? ((inc & (0u - inc)) << 1) - 1 : 0xffffffffu;  // lanes <= first inclusive
    if (zero & upto) continue;  // a predecessor has not published yet: re-read
    uint64_t v = ((upto >> lane) & 1) ? (d & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    look -= 32;
  }
  if (lane == 0) st_relaxed_u64(&desc[tile], kFlagInc | (excl + agg));
  return (int64_t)excl;
}

// scan + decide one record whose bytes are text[ts, ts+L) in shared memory
__device__ __forceinline__ Res parse_staged(const uint8_t* text, uint32_t ts, uint32_t L, uint32_t ndw,
                                            const uint64_t* p10) {
  Scan sc = fast_scan(text, ts, L, ndw, p10);
  if (sc.kind == K_SLOWSCAN) sc = scan_record(text + ts, L);
  return decide(sc);
}

__device__ __noinline__ Res parse_global(const uint8_t* bytes, int64_t s, int64_t e) {
  Scan sc;
  if (e - s >= (1ll << 31)) {
    sc.kind = K_INVALID; sc.neg = false; sc.tnz = false; sc.w = 0; sc.q = 0;
  } else {
    sc = scan_record(bytes + s, (uint32_t)(e - s));
  }
  return decide(sc);
}

// ============================================================================
// k_split: warp-level agents.  Every warp independently claims 2 KiB tiles in
// order, stages them with its own TMA double buffer, classifies 64 bytes per
// lane, compacts record starts with a warp scan, parses one record per lane,
// resolves its global record index by decoupled look-back and writes out.
// There is no CTA-wide barrier: a warp never waits for another warp's parse.
constexpr int kWarpTile = 32 * kBytesPerThread;                 // 2 KiB
constexpr int kWarpStage = 16 + kWarpTile + kSplitHalo;         // 2192 = 137 x 16
constexpr int kWarpStageAlloc = kWarpStage + 112;
constexpr int kWarpMaskWords = (kWarpTile + kSplitHalo) / 32;   // 68
constexpr int kWarpStartsCap = 512;                              // compacted path
constexpr int kWarpRcap = 192;                                   // results buffered per tile
constexpr int kSplitWarps = 4;                                   // warps per CTA

struct SplitArgs {
  const uint8_t* bytes;
  int64_t len;
  int64_t head;      // bytes % 16: tile t covers positions [t*TILE - head, (t+1)*TILE - head)
  int64_t ntiles;
  int64_t* offsets_out;
  int64_t capacity;
  int64_t* n_out;
  double* out;
  uint8_t* status;
  WsHeader* hdr;
  uint64_t* desc;
  SlowEntry* queue;
  uint64_t qcap;
  uint64_t* stats;
};

struct __align__(128) WarpSmem {
  uint8_t text[2][kWarpStageAlloc];           // double buffer; tile at text[b][16 ..]
  uint64_t res_bits[kWarpRcap];               // buffered results
  uint32_t ndm[kWarpMaskWords + 2];           // non-digit masks, tile coordinates
  uint32_t spm[kWarpMaskWords + 2];           // separator masks, tile coordinates
  uint16_t starts[kWarpStartsCap];            // record starts (tile coordinates)
  uint8_t res_st[kWarpRcap];
  unsigned long long bar[2];
};

struct __align__(128) SplitSmem {
  WarpSmem w[kSplitWarps];
  uint64_t p10[20];                           // powers of ten for the scanner
};

__device__ __forceinline__ bool split_interior(const SplitArgs& a, int64_t tile) {
  const int64_t base = tile * kWarpTile - a.head;
  return tile < a.ntiles && base - 16 >= 0 && base + kWarpTile + kSplitHalo <= a.len;
}

template <uint32_t SEPS, bool STATS>
__global__ void __launch_bounds__(32 * kSplitWarps) k_split(SplitArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SplitSmem& SS = *reinterpret_cast<SplitSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& S = SS.w[warp];
  if (threadIdx.x < 20) {
    uint64_t p = 1;
    for (int k = 0; k < (int)threadIdx.x; k++) p *= 10;
    SS.p10[threadIdx.x] = p;
  }
  const uint64_t* p10 = SS.p10;
  int64_t tile = 0;
  if (lane == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    S.ndm[kWarpMaskWords] = S.ndm[kWarpMaskWords + 1] = 0xFFFFFFFFu;
    S.spm[kWarpMaskWords] = S.spm[kWarpMaskWords + 1] = 0xFFFFFFFFu;
    tile = (int64_t)atomicAdd(&a.hdr->tile_ctr, 1u);
    if (split_interior(a, tile))
      tma_load_1d(S.text[0], a.bytes + (tile * kWarpTile - a.head - 16), kWarpStage, &S.bar[0]);
  }
  __syncthreads();  // p10, mbarrier init (the only CTA barrier)
  tile = __shfl_sync(0xffffffffu, tile, 0);
  StatAcc acc;
  acc.zero();
  uint32_t phase = 0;  // bit b: parity of buffer b's next completion
  int b = 0;

  while (tile < a.ntiles) {
    const int64_t base = tile * kWarpTile - a.head;  // position of text[b][16]
    uint8_t* text = S.text[b];
    // ---- 1. prefetch the next tile into the other buffer; wait for this one --
    int64_t next = 0;
    if (lane == 0) {
      next = (int64_t)atomicAdd(&a.hdr->tile_ctr, 1u);
      if (split_interior(a, next))
        tma_load_1d(S.text[b ^ 1], a.bytes + (next * kWarpTile - a.head - 16), kWarpStage, &S.bar[b ^ 1]);
    }
    next = __shfl_sync(0xffffffffu, next, 0);
    if (split_interior(a, tile)) {
      mbar_wait(&S.bar[b], (phase >> b) & 1);
      phase ^= 1u << b;
    } else {  // ragged first / last tiles: byte-exact loads, zero outside [0, len)
      for (int c = lane; c < kWarpStage / 16; c += 32)
        *reinterpret_cast<uint4*>(&text[16 * c]) = load_chunk(a.bytes, a.len, base - 16 + 16 * c);
      __syncwarp();
    }
    // ---- 2. classify 64 bytes per lane (+ the 128-byte halo by lanes 0-3) ---
    const int x0 = kBytesPerThread * lane;
    uint32_t nd0, sp0, nd1, sp1;
    classify32<SEPS>(*reinterpret_cast<const uint4*>(&text[16 + x0]),
                     *reinterpret_cast<const uint4*>(&text[32 + x0]), nd0, sp0);
    classify32<SEPS>(*reinterpret_cast<const uint4*>(&text[48 + x0]),
                     *reinterpret_cast<const uint4*>(&text[64 + x0]), nd1, sp1);
    *reinterpret_cast<uint2*>(&S.ndm[2 * lane]) = make_uint2(nd0, nd1);
    *reinterpret_cast<uint2*>(&S.spm[2 * lane]) = make_uint2(sp0, sp1);
    if (lane < kWarpMaskWords - 64) {
      const int xh = kWarpTile + 32 * lane;
      uint32_t ndh, sph;
      classify32<SEPS>(*reinterpret_cast<const uint4*>(&text[16 + xh]),
                       *reinterpret_cast<const uint4*>(&text[32 + xh]), ndh, sph);
      S.ndm[64 + lane] = ndh;
      S.spm[64 + lane] = sph;
    }
    // ---- 3. record starts: a separator at x-1 (or position 0) starts a record at x
    const uint32_t up = __shfl_up_sync(0xffffffffu, sp1, 1);
    const uint32_t prev = (lane == 0) ? (is_sep(text[15], SEPS) ? 1u : 0u) : (up >> 31);
    uint32_t s0 = (sp0 << 1) | prev;
    uint32_t s1 = (sp1 << 1) | (sp0 >> 31);
    const int64_t p0 = base + x0;
    if (p0 < 64 || p0 + 64 > a.len) {  // only near the ends of the input
      uint64_t m = ((uint64_t)s1 << 32) | s0;
      if (p0 <= 0 && p0 + 64 > 0) m |= 1ull << (int)(-p0);  // position 0 starts record 0
      if (p0 < 0) m &= (p0 <= -64) ? 0ull : (~0ull << (int)(-p0));
      if (p0 + 64 > a.len) m &= (p0 >= a.len) ? 0ull : (~0ull >> (int)(p0 + 64 - a.len));
      s0 = (uint32_t)m;
      s1 = (uint32_t)(m >> 32);
    }
    const int cnt = __popc(s0) + __popc(s1);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - cnt;
    if (lane == 0) st_relaxed_u64(&a.desc[tile], (tile == 0 ? kFlagInc : kFlagAgg) | (uint64_t)total);
    if (STATS) acc.v[STAT_TILES] += (lane == 0);

    // first separator at or after tile position s within the staged window
    // (or len); -1 if the record runs past the window
    auto sep_end = [&](int s) -> int {
      constexpr int win = kWarpTile + kSplitHalo;
      const int lim = (a.len - base < (int64_t)win) ? (int)(a.len - base) : win;
      int x = s;
      while (true) {  // the padding mask words past the window are all ones: terminates
        const uint32_t m = mask_at(S.spm, (uint32_t)x);
        if (m) {
          const int e = x + __ffs(m) - 1;
          return e < lim ? e : (lim < win ? lim : -1);
        }
        x += 32;
        if (x >= lim) return lim < win ? lim : -1;
      }
    };
    // parse the record starting at s whose end (tile coordinates) is e (-1: past the window)
    auto parse_at = [&](int s, int e, int64_t& re, bool& global) -> Res {
      if (e >= 0) {
        re = base + e;
        global = false;
        return parse_staged(text, 16u + (uint32_t)s, (uint32_t)(e - s), mask_at(S.ndm, (uint32_t)s), p10);
      }
      int64_t p = base + kWarpTile + kSplitHalo;  // long record: find its end in global memory
      while (p < a.len && !is_sep(a.bytes[p], SEPS)) p++;
      re = p;
      global = true;
      return parse_global(a.bytes, base + s, re);
    };

    if (total <= kWarpStartsCap) {
      // ---- compacted path: record starts -> shared list ---------------------
      int o = excl;
      for (uint32_t m = s0; m; m &= m - 1) S.starts[o++] = (uint16_t)(x0 + __ffs(m) - 1);
      for (uint32_t m = s1; m; m &= m - 1) S.starts[o++] = (uint16_t)(x0 + 32 + __ffs(m) - 1);
      __syncwarp();
      // ---- 4. parse into the buffer, then look back -------------------------
      const int nbuf = min(total, kWarpRcap);
      int64_t last_end = 0;
      for (int j = lane; j < nbuf; j += 32) {
        const int s = S.starts[j];
        const int e = (j + 1 < total) ? S.starts[j + 1] - 1 : sep_end(s);
        int64_t re;
        bool global;
        const Res r = parse_at(s, e, re, global);
        count_stats<STATS>(acc, r, global);
        S.res_bits[j] = r.bits;
        S.res_st[j] = (r.info & F_PENDING) ? ST_PENDING : (uint8_t)r.info;
        if (j == total - 1) last_end = re;
      }
      const int64_t prefix = lookback(a.desc, tile, (uint64_t)total);
      if (lane == 0 && tile == a.ntiles - 1) *a.n_out = prefix + total;
      last_end = __shfl_sync(0xffffffffu, last_end, (total - 1) & 31);
      __syncwarp();
      // ---- 5. write out -----------------------------------------------------
      for (int j = lane; j < ((total + 31) & ~31); j += 32) {
        const bool have = j < total;
        const int64_t gidx = prefix + j;
        const bool live = have && gidx < a.capacity;
        uint64_t bits = 0;
        uint32_t st = 0;
        int64_t re = 0;
        if (have && j >= kWarpRcap) {  // tiles with very many records: parse now
          const int s = S.starts[j];
          const int e = (j + 1 < total) ? S.starts[j + 1] - 1 : sep_end(s);
          bool global;
          const Res r = parse_at(s, e, re, global);
          count_stats<STATS>(acc, r, global);
          bits = r.bits;
          st = (r.info & F_PENDING) ? ST_PENDING : (r.info & 0xFF);
        } else if (have) {
          bits = S.res_bits[j];
          st = S.res_st[j];
        }
        const bool pend = live && st == ST_PENDING;
        if (live) {
          a.out[gidx] = __longlong_as_double((long long)(pend ? (bits & ~kCandNoLower) : bits));
          a.status[gidx] = pend ? (uint8_t)ST_OK : (uint8_t)st;
          if (a.offsets_out) a.offsets_out[gidx] = base + S.starts[j];
        }
        if (__any_sync(0xffffffffu, pend)) {
          SlowEntry en;
          en.idx = gidx;
          en.start = have ? base + S.starts[j] : 0;
          if (pend && j < kWarpRcap) re = (j + 1 < total) ? base + S.starts[j + 1] - 1 : last_end;
          en.end = re;
          en.cand = bits;
          queue_push(pend, a.hdr, a.queue, a.qcap, en);  // the split queue cannot overflow
        }
      }
    } else {
      // ---- dense path (records shorter than 4 bytes on average) -------------
      const int64_t prefix = lookback(a.desc, tile, (uint64_t)total);
      if (lane == 0 && tile == a.ntiles - 1) *a.n_out = prefix + total;
      int k = 0;
      uint64_t m = ((uint64_t)s1 << 32) | s0;
      const int rounds = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
      for (int r_ = 0; r_ < rounds; r_++) {
        const bool have = m != 0;
        const int64_t gidx = prefix + excl + k;
        int64_t re = 0;
        int s = 0;
        Res r;
        r.bits = 0;
        r.info = 0;
        if (have) {
          s = x0 + __ffsll((long long)m) - 1;
          m &= m - 1;
          bool global;
          r = parse_at(s, sep_end(s), re, global);
          count_stats<STATS>(acc, r, global);
        }
        const bool live = have && gidx < a.capacity;
        const bool pend = live && (r.info & F_PENDING);
        if (live) {
          a.out[gidx] = __longlong_as_double((long long)(pend ? (r.bits & ~kCandNoLower) : r.bits));
          a.status[gidx] = pend ? (uint8_t)ST_OK : (uint8_t)(r.info & 0xFF);
          if (a.offsets_out) a.offsets_out[gidx] = base + s;
        }
        SlowEntry en;
        en.idx = gidx;
        en.start = base + s;
        en.end = re;
        en.cand = r.bits;
        queue_push(pend, a.hdr, a.queue, a.qcap, en);
        k++;
      }
    }
    __syncwarp();
    tile = next;
    b ^= 1;
  }
  if (STATS) flush_stats(acc, a.stats);
}

// ============================================================================
struct BatchArgs {
  const uint8_t* bytes;
  int64_t len;
  int64_t head;  // bytes % 16
  const int64_t* offsets;
  int64_t n;
  int64_t ntiles;
  double* out;
  uint8_t* status;
  WsHeader* hdr;
  SlowEntry* queue;
  uint64_t qcap;
  uint64_t* stats;
};

struct __align__(128) BatchSmem {
  uint8_t text[kBatchText + 64];
  uint64_t p10[20];
  int64_t offs[kBatchRecs + 1];
  uint32_t ndm[kBatchMaskWords + 2];
  unsigned long long bar;
  int64_t tile;
};

template <bool STATS>
__global__ void __launch_bounds__(kBatchThreads) k_batch(BatchArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  BatchSmem& S = *reinterpret_cast<BatchSmem*>(smem_raw);
  const int tid = threadIdx.x;
  if (tid < 20) {
    uint64_t p = 1;
    for (int k = 0; k < tid; k++) p *= 10;
    S.p10[tid] = p;
  }
  if (tid == 0) mbar_init(&S.bar, 1);
  StatAcc acc;
  acc.zero();
  uint32_t phase = 0;
  __syncthreads();

  while (true) {
    if (tid == 0) S.tile = (int64_t)atomicAdd(&a.hdr->tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = S.tile;
    if (tile >= a.ntiles) break;
    const int64_t r0 = tile * kBatchRecs;
    const int cnt = (int)min((int64_t)kBatchRecs, a.n - r0);
    for (int k = tid; k <= cnt; k += kBatchThreads)
      S.offs[k] = (r0 + k < a.n) ? a.offsets[r0 + k] : a.len;
    __syncthreads();
    const int64_t lo = S.offs[0], hi = S.offs[cnt];
    const int64_t p_al = lo - ((lo + a.head) & 15);  // absolute 16-byte aligned
    const bool staged = lo >= 0 && lo <= hi && hi <= a.len && hi - p_al <= kBatchText;
    const int nbytes = staged ? (int)(((hi - p_al) + 15) & ~15ll) : 0;
    if (staged) {
      if (p_al >= 0 && p_al + nbytes <= a.len) {
        if (tid == 0) tma_load_1d(S.text, a.bytes + p_al, (uint32_t)nbytes, &S.bar);
        mbar_wait(&S.bar, phase);
        phase ^= 1;
      } else {
        for (int c = tid; c < nbytes / 16; c += kBatchThreads)
          *reinterpret_cast<uint4*>(&S.text[16 * c]) = load_chunk(a.bytes, a.len, p_al + 16 * c);
        __syncthreads();
      }
      for (int c = tid; c < (nbytes + 31) / 32; c += kBatchThreads) {
        uint32_t nd, sp;
        classify32<0>(*reinterpret_cast<const uint4*>(&S.text[32 * c]),
                      *reinterpret_cast<const uint4*>(&S.text[32 * c + 16]), nd, sp);
        S.ndm[c] = nd;
      }
      if (tid == 0) S.ndm[(nbytes + 31) / 32] = S.ndm[(nbytes + 31) / 32 + 1] = 0xFFFFFFFFu;
      __syncthreads();
    }
    if (STATS) acc.v[STAT_TILES] += (tid == 0);
    for (int j = tid; j < ((cnt + 31) & ~31); j += kBatchThreads) {
      const bool have = j < cnt;
      Res r;
      r.bits = 0;
      r.info = 0;
      int64_t s = 0, e = 0;
      if (have) {
        s = S.offs[j];
        e = S.offs[j + 1];
        if (s < 0 || s > a.len || e < s || e > a.len) {
          r.bits = kQNaN;
          r.info = ST_INVALID;
          count_stats<STATS>(acc, r, false);
        } else if (staged && s >= lo && e <= hi) {
          const uint32_t ts = (uint32_t)(s - p_al);
          r = parse_staged(S.text, ts, (uint32_t)(e - s), mask_at(S.ndm, ts), S.p10);
          count_stats<STATS>(acc, r, false);
        } else {
          r = parse_global(a.bytes, s, e);
          count_stats<STATS>(acc, r, true);
        }
      }
      const bool pend = have && (r.info & F_PENDING);
      bool ok = true;
      if (__any_sync(0xffffffffu, pend)) {
        SlowEntry ent;
        ent.idx = r0 + j;
        ent.start = s;
        ent.end = e;
        ent.cand = r.bits;
        ok = queue_push(pend, a.hdr, a.queue, a.qcap, ent);
      }
      if (have) {
        // queue overflow (only with overlapping offsets): leave the candidate
        // in out[] and mark the record for the slow kernel's status scan
        const bool mark = pend && !ok;
        a.out[r0 + j] = __longlong_as_double((long long)(pend ? (mark ? r.bits : r.bits & ~kCandNoLower) : r.bits));
        a.status[r0 + j] = mark ? (uint8_t)ST_PENDING : (uint8_t)(pend ? ST_OK : (r.info & 0xFF));
      }
    }
    __syncthreads();
  }
  if (STATS) flush_stats(acc, a.stats);
}

}  // namespace fpp
