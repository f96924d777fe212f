// k_split.cuh -- parse_f64_split's fast kernel: record splitter + scanner +
// Algorithm 1, organised as independent warp-level agents.
//
// Every warp claims 5 KiB tiles in order (atomicAdd on one of eight counters)
// and, for each tile:
//   1. stages it with one TMA bulk copy (cp.async.bulk + its own mbarrier);
//      byte-exact loads only for the ragged first and last tiles;
//   2. classifies 160 bytes per lane into two bit masks -- separators (record
//      starts, kept in registers) and non-digits (record structure, kept in
//      shared memory);
//   3. counts record starts (popc), warp-scans them, publishes the tile's
//      count for the decoupled look-back and compacts the starts into a list
//      (dense tiles: each lane keeps its own starts);
//   4. parses one record per lane per round -- the common-case parser
//      (fastrec.cuh), else the general scanner, then Algorithm 1 with the
//      19-digit bracket -- and queues undecided and long records for the slow
//      kernel at once, named by (tile, index in tile);
//   5. once the tile is parsed (its results buffered in the parsed front of
//      the staged text), resolves the tile's first global record index by
//      decoupled look-back over the tiles' published counts (single pass,
//      SURVEY.md 8a a1) and copies the results out (consecutive records ->
//      consecutive lanes: coalesced).  Tiles of short records, where the
//      buffer would overlap unparsed text, look back after the second round
//      and write straight from registers.
// A tile owns the records starting in its first kWarpStride bytes; the last
// 32 classified bytes overlap the next tile and serve as the halo that ends
// the tile's last record (longer records go to the slow kernel).
// There is no CTA-wide barrier after start-up: a warp only ever waits for its
// own data and for its predecessors' published counts.
#pragma once
#include "k_common.cuh"

#ifndef FPP_ABLATE
#define FPP_ABLATE 0  // 0 = the product; 1 = splitting only, 3 = no look-back (timing experiments only)
#endif

namespace fpp {

constexpr int kLaneWords = 5;  // 32-byte words classified per lane (5 KiB tiles)
constexpr int kSplitLaneBytes = 32 * kLaneWords;
constexpr int kWarpTile = 32 * kSplitLaneBytes;                 // 5 KiB classified per tile
constexpr int kWarpStride = kWarpTile - 32;                     // 5088 = 318 x 16 owned
constexpr int kWarpStage = 16 + kWarpTile;                      // 5136 = 321 x 16 staged
constexpr int kWarpStageAlloc = kWarpStage + 48;                // slack for word reads just past the window
constexpr int kWarpMaskWords = kWarpTile / 32;                  // 160
constexpr int kWarpStartsCap = 512;                             // compacted path (records >= 9.9 B)
constexpr int kSplitWarps = 4;                                  // warps per CTA

struct SplitArgs {
  const uint8_t* bytes;
  int64_t len;
  int64_t head;      // bytes % 16: tile t covers positions [t*STRIDE - head, ...)
  int64_t ntiles;
  int64_t* offsets_out;
  int64_t capacity;
  int64_t* n_out;
  void* out;  // double[capacity] or (F32) float[capacity]
  uint8_t* status;
  WsHeader* hdr;
  uint64_t* desc;
  SlowEntry* queue;
  uint64_t qcap;
  uint64_t* stats;
  uint32_t grammar;  // 0 or G_HEX / G_JSON (also the template argument G)
  int nctr;          // tile counters in use, min(kTileCtrs, grid)
  int last_interior; // tiles 1 .. last_interior are staged by one bulk copy (0: none)
};

struct __align__(128) WarpSmem {
  uint8_t pad[32];                            // digit windows may read up to 20 bytes before text
  uint8_t text[kWarpStageAlloc];              // tile at text[16 ..]; text[0..16) precedes it
  __align__(16) uint32_t ndm[kWarpMaskWords + 4];  // non-digit masks, tile coordinates (+ padding)
  uint16_t starts[kWarpStartsCap + 2];        // record starts (tile coordinates), then end + 1 of the last
  unsigned long long bar;
};

struct __align__(128) SplitSmem {
  WarpSmem w[kSplitWarps];
  uint64_t p10[20];                           // powers of ten for the scanner
};

// tile t's window [t * kWarpStride - head - 16, + kWarpStage) lies inside
// [0, len): 1 <= t <= last_interior (host: fpparse.cu split_last_interior)
__device__ __forceinline__ bool split_interior(const SplitArgs& a, int tile) {
  return (unsigned)(tile - 1) < (unsigned)a.last_interior;
}

// record starts in tile t's owned bytes [t * kWarpStride - head, + kWarpStride)
// counted from global memory (the look-back's forward-progress fallback; the
// same count the tile's owner publishes): position 0, and every position x
// in (0, len) after a separator
template <uint32_t SEPS>
__device__ __forceinline__ int count_tile_starts(const uint8_t* bytes, int64_t len, int64_t head, int64_t t) {
  const int lane = threadIdx.x & 31;
  const int64_t lo = t * kWarpStride - head, hi = lo + kWarpStride;
  int c = 0;
  for (int64_t x = lo + lane; x < hi; x += 32) {
    if (x < 0 || x >= len) continue;
    c += (x == 0 || is_sep(bytes[x - 1], SEPS)) ? 1 : 0;
  }
  return __reduce_add_sync(0xffffffffu, (unsigned)c);
}

// atomicAdd from one lane without the compiler's warp-aggregation code
__device__ __forceinline__ unsigned atom_add_u32(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}

// start bits of the word covering positions [p, p+32): only positions in
// [0, len) start records, and position 0 always does
__device__ __forceinline__ uint32_t fix_start_word(uint32_t m, int64_t p, int64_t len) {
  if (p <= 0 && p + 32 > 0) m |= 1u << (int)(-p);
  if (p < 0) m &= (p <= -32) ? 0u : (0xffffffffu << (int)(-p));
  if (p + 32 > len) m &= (p >= len) ? 0u : (0xffffffffu >> (int)(p + 32 - len));
  return m;
}

// scan + Algorithm 1 for the record [s, e) of a staged tile (tile coordinates;
// e < 0: the record runs past the staged window; long records go to the slow
// kernel unscanned)
template <bool F32, int G>
__device__ __forceinline__ Res split_parse(const uint8_t* text, const uint32_t* ndm, int s, int e,
                                           const uint64_t* p10, uint32_t grammar) {
  Res r;
#if FPP_ABLATE == 1 || FPP_ABLATE == 4  // experiment: splitting only (no scan, no Algorithm 1)
  r.bits = (uint64_t)(uint32_t)s << 32 | (uint32_t)e;
  r.info = 0;
  return r;
#endif
  if (G == (int)G_HEX) {
    if (e >= 0 && e - s <= kLongRec) {
      r = parse_staged<false, F32, G>(text, 16u + (uint32_t)s, (uint32_t)(e - s), mask_at(ndm, (uint32_t)s), p10,
                                      grammar);
    } else {  // long: the slow path scans it (k_slow_scan; it finds the end if e < 0)
      r = long_record();
    }
    return r;
  }
  // The common-case parser runs on every lane (a long record, or e < 0,
  // gives a length it rejects; its reads stay inside the staged buffer),
  // the branch is only on its rare failure
  const uint32_t ts = 16u + (uint32_t)s, L = (uint32_t)(e - s), ndw = mask_at(ndm, (uint32_t)s);
  if (!fast_record<false, F32, G == (int)G_JSON>(text, ts, L, ndw, p10, r)) {
    if (e >= 0 && e - s <= kLongRec)
      r = parse_general<F32>(text, ts, L, ndw, p10, grammar);
    else  // long: the slow path scans it (k_slow_scan; it finds the end if e < 0)
      r = long_record();
  }
  return r;
}
template <bool F32, int G>
__device__ __noinline__ Res split_parse_ni(const uint8_t* text, const uint32_t* ndm, int s, int e,
                                           const uint64_t* p10, uint32_t grammar) {
  return split_parse<F32, G>(text, ndm, s, e, p10, grammar);
}

#ifndef FPP_SHAPE
#define FPP_SHAPE 1  // 0: no "0.ddd" tile loop
#endif
#ifndef FPP_F0_TILE
#define FPP_F0_TILE 1  // 1: the "0.ddd" shape checked once per tile on the masks; 0: per record (round 0 votes)
#endif
#ifndef FPP_PF_DIST
#define FPP_PF_DIST 0  // > 0: L2 prefetch of the tile this many claims ahead on the warp's counter (experiment)
#endif
#ifndef FPP_EARLY_CLAIM
#define FPP_EARLY_CLAIM 1  // 1: the next tile claimed and requested into L2 during the look-back; 2: claimed only; 3: claimed after the look-back; 0: claimed at the top of the loop
#endif
#ifndef FPP_COMPACT
#define FPP_COMPACT 2  // 2: two predicated stores per word behind one vote; 1: per-word loops
#endif
#ifndef FPP_SPLIT_OWN
#define FPP_SPLIT_OWN 0  // 1: every lane parses the records starting in its own bytes (no starts list)
#endif
#ifndef FPP_SPLIT_MINB
#define FPP_SPLIT_MINB 8  // CTAs per SM the register allocation must allow (shared memory allows 8)
#endif
template <uint32_t SEPS, bool STATS, bool F32, int G>
__global__ void __launch_bounds__(32 * kSplitWarps, FPP_SPLIT_MINB) k_split(SplitArgs a) {
  using OutT = typename std::conditional<F32, uint32_t, unsigned long long>::type;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  SplitSmem& SS = *reinterpret_cast<SplitSmem*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem& S = SS.w[warp];
  if (threadIdx.x < 20) {
    uint64_t p = 1;
    for (int k = 0; k < (int)threadIdx.x; k++) p *= 10;
    SS.p10[threadIdx.x] = p;
  }
  if (lane == 0) {
    mbar_init(&S.bar, 1);
    S.ndm[kWarpMaskWords] = S.ndm[kWarpMaskWords + 1] = 0xFFFFFFFFu;
  }
  __syncthreads();  // p10 and the mbarriers (the only CTA barrier)
  const uint64_t* p10 = SS.p10;
  uint8_t* text = S.text;
  StatAcc acc;
  acc.zero();
  uint32_t phase = 0;
  const int g = (int)(blockIdx.x % (unsigned)a.nctr);
  unsigned* const ctr = split_ctr(a.hdr, g);

#ifndef FPP_STATIC_TILES
#define FPP_STATIC_TILES 0  // 1: experiment only -- static tile striding (needs every CTA resident)
#endif
#if FPP_STATIC_TILES
  int static_next = (int)blockIdx.x * kSplitWarps + warp;
#endif
#if FPP_EARLY_CLAIM
  int nxt = -1;  // lane 0: the tile claimed during the previous tile's look-back (-1: none)
#endif
  while (true) {
    // ---- 1. claim and stage a tile -------------------------------------------
    int tile = 0;
    if (lane == 0) {
#if FPP_STATIC_TILES
      tile = static_next;
      static_next += (int)gridDim.x * kSplitWarps;
#elif FPP_EARLY_CLAIM
      tile = nxt >= 0 ? nxt : (int)atom_add_u32(ctr, 1u) * a.nctr + g;
      nxt = -1;
#else
      // G counters, CTA b on counter b mod G: one global counter serialised
      // the claims (same-address atomics, ~2 ns each: 1 ms for 2 GB of 4 KiB
      // tiles); each counter's claims stay in time order, so tile t's
      // predecessors are claimed about when t is (a predecessor that is not
      // claimed in time is counted by the look-back's fallback)
      tile = (int)atom_add_u32(ctr, 1u) * a.nctr + g;
#endif
      // (the buffer's generic writes were fenced for the async proxy at the
      // end of the previous tile)
      if (split_interior(a, tile))
        tma_load_1d_nf(text, a.bytes + ((int64_t)tile * kWarpStride - a.head - 16), kWarpStage, &S.bar);
    }
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= a.ntiles) break;
    const int64_t base = (int64_t)tile * kWarpStride - a.head;  // position of text[16]
    if (split_interior(a, tile)) {
      mbar_wait(&S.bar, phase);
      phase ^= 1u;
    } else {  // ragged first / last tiles: byte-exact loads, zero outside [0, len)
      for (int c = lane; c < kWarpStage / 16; c += 32)
        *reinterpret_cast<uint4*>(&text[16 * c]) = load_chunk(a.bytes, a.len, base - 16 + 16 * c);
      __syncwarp();
    }
#if FPP_ABLATE == 6  // experiment: claim + staging only
    if (lane == 0 && tile == a.ntiles - 1) *a.n_out = 0;
    __syncwarp();
    continue;
#endif
    // ---- 2. classify kSplitLaneBytes (160) bytes per lane -----------------------
    const int x0 = kSplitLaneBytes * lane;
    constexpr int W = kLaneWords;
    uint32_t sp[W];
#if FPP_F0_TILE
    uint32_t ndr[W];
#endif
    {
      // Lanes 160 bytes apart read their 32-byte words in the same order, the
      // lanes l with bit 2 set taking the word's second 16 bytes first: the 8
      // lanes of each LDS.128 wavefront then cover all 8 16-byte bank groups
      // (16 x l + 2 k + half, mod 8), so the loads are conflict-free; the two
      // 16-bit halves of those lanes' masks are swapped back
      static_assert(kLaneWords == 5, "bank-group schedule for 160-byte lanes");
      const int swp = (lane >> 2) & 1;
#pragma unroll
      for (int k = 0; k < W; k++) {
        uint32_t nd, sw;
        classify32<SEPS>(*reinterpret_cast<const uint4*>(&text[16 + x0 + 32 * k + 16 * swp]),
                         *reinterpret_cast<const uint4*>(&text[32 + x0 + 32 * k - 16 * swp]), nd, sw);
        nd = __funnelshift_l(nd, nd, 16 * swp);
        S.ndm[W * lane + k] = nd;
#if FPP_F0_TILE
        ndr[k] = nd;
#endif
        sp[k] = __funnelshift_l(sw, sw, 16 * swp);
      }
    }
    // ---- 3. record starts: a separator at x-1 (or position 0) starts a record at x
    const uint32_t up = __shfl_up_sync(0xffffffffu, sp[W - 1], 1);
    uint32_t st[W];
    st[0] = (sp[0] << 1) | ((lane == 0) ? (is_sep(text[15], SEPS) ? 1u : 0u) : (up >> 31));
#pragma unroll
    for (int k = 1; k < W; k++) st[k] = (sp[k] << 1) | (sp[k - 1] >> 31);
#if FPP_F0_TILE
    // "0.ddd" tiles: every non-digit byte
    // of the tile is a separator or the byte after a record start.  (Lane 0's
    // bit 0 belongs to a record of the previous tile.  The starts are the
    // ones before the data-end fix: position 0 and bytes past the data fail
    // the test, and the tile takes the general loop.)
    bool tile_f0 = false;
    if (FPP_SHAPE && G == 0) {
      const uint32_t ups = __shfl_up_sync(0xffffffffu, st[W - 1], 1);
      uint32_t bad = (ndr[0] ^ (sp[0] | __funnelshift_l(ups, st[0], 1))) & (lane == 0 ? ~1u : ~0u);
#pragma unroll
      for (int k = 1; k < W; k++) bad |= ndr[k] ^ (sp[k] | __funnelshift_l(st[k - 1], st[k], 1));
      tile_f0 = __all_sync(0xffffffffu, bad == 0u);
    }
#endif
    const int64_t p0 = base + x0;
    if (p0 < kSplitLaneBytes || p0 + kSplitLaneBytes > a.len) {  // only near the ends
#pragma unroll
      for (int k = 0; k < W; k++) st[k] = fix_start_word(st[k], p0 + 32 * k, a.len);
    }
    // [kWarpStride, kWarpTile) is the halo: its starts belong to the next
    // tile, but the first of them ends this tile's last record (bit b:
    // separator at kWarpStride - 1 + b)
    const uint32_t halo = __shfl_sync(0xffffffffu, st[W - 1], 31);
    if (lane == 31) st[W - 1] = 0u;
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < W; k++) cnt += __popc(st[k]);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    const int excl = incl - cnt;
    if (lane == 0) st_relaxed_u64(&a.desc[tile], (tile == 0 ? kFlagInc : kFlagAgg) | (uint64_t)total);
#if FPP_SPLIT_OWN
    const bool compact = false;
#else
    const bool compact = total <= kWarpStartsCap;
#endif
#if FPP_COMPACT == 2
    if (compact) {
      // no word of the tile with a third start (records of 16 bytes or more
      // never have one): two predicated stores per word and no branch; else
      // a loop over every word's starts
      uint32_t third = 0;
#pragma unroll
      for (int k = 0; k < W; k++) {
        const uint32_t m1 = st[k] & (st[k] - 1);
        third |= m1 & (m1 - 1);
      }
      uint16_t* sq = S.starts + excl;
      if (!__any_sync(0xffffffffu, third != 0u)) {
#pragma unroll
        for (int k = 0; k < W; k++) {
          const uint32_t m0 = st[k], m1 = m0 & (m0 - 1);
          if (m0) sq[0] = (uint16_t)(x0 + 32 * k + __popc(~m0 & (m0 - 1)));
          if (m1) sq[1] = (uint16_t)(x0 + 32 * k + __popc(~m1 & (m1 - 1)));
          sq += __popc(m0);
        }
      } else {
#pragma unroll
        for (int k = 0; k < W; k++)
          for (uint32_t m = st[k]; m; m &= m - 1) *sq++ = (uint16_t)(x0 + 32 * k + low_bit(m));
      }
    }
#else
    if (compact) {
      // two starts per 32-byte word without a loop (predicated: records of 16
      // bytes or more never have a third), the rest in a loop
      int o = excl;
#pragma unroll
      for (int k = 0; k < W; k++) {
        const uint32_t m0 = st[k], m1 = m0 & (m0 - 1);
        if (m0) S.starts[o] = (uint16_t)(x0 + 32 * k + low_bit(m0));
        if (m1) S.starts[o + 1] = (uint16_t)(x0 + 32 * k + low_bit(m1));
        o += min(__popc(m0), 2);
        for (uint32_t m = m1 & (m1 - 1); m; m &= m - 1) S.starts[o++] = (uint16_t)(x0 + 32 * k + low_bit(m));
      }
    }
#endif
    if (STATS) acc.v[STAT_TILES] += (lane == 0);
    __syncwarp();  // starts / masks visible to the whole warp

    // first separator at or after tile position s within the staged window
    // (or len); -1 if the record runs past the window.  Candidates are the
    // non-digit bytes (a separator is one); their bytes are checked in turn.
    auto sep_end = [&](int s) -> int {
      constexpr int win = kWarpTile;
      const int lim = (a.len - base < (int64_t)win) ? (int)(a.len - base) : win;
      int x = s;
      while (true) {  // the padding mask words past the window are all ones: terminates
        for (uint32_t m = mask_at(S.ndm, (uint32_t)x); m; m &= m - 1) {
          const int e = x + __ffs(m) - 1;
          if (e >= lim) return lim < win ? lim : -1;
          if (is_sep(text[16 + e], SEPS)) return e;
        }
        x += 32;
        if (x >= lim) return lim < win ? lim : -1;
      }
    };
    // scan + Algorithm 1 for the record [s, e) (tile coordinates; e < 0: the
    // record runs past the staged window; long records go to the slow kernel).
    // Inlined only in the common (deferred) round loop; the rare paths (short
    // records, dense tiles) call one out-of-line copy, which keeps the hot
    // code small (instruction fetch)
    auto parse = [&](int s, int e) -> Res {
      return split_parse<F32, G>(text, S.ndm, s, e, p10, a.grammar);
    };
    auto parse_ni = [&](int s, int e) -> Res {
      return split_parse_ni<F32, G>(text, S.ndm, s, e, p10, a.grammar);
    };
    // bookkeeping for record j of the tile right after its parse: counters,
    // and the slow-queue entry of an undecided record.  The entry names the
    // record by (tile, j); the slow kernel turns that into the output index
    // from the published inclusive prefixes, so no entry waits for the
    // look-back (split_queue_idx, k_slow.cuh).
    auto account = [&](int j, int s, int e, const Res& r) {
      count_stats<STATS>(acc, r, e < 0);
      if (r.info & F_PENDING) {  // rare: lanes aggregate among themselves
        SlowEntry en;
        en.idx = split_queue_idx(tile, j);
        en.start = base + s;
        en.end = e >= 0 ? base + e : -1;
        en.cand = r.bits;
        // out of line: rare, and inlined it made the round loop's code larger
        // (config 2 +2%, config 7 +5%); the split queue cannot overflow
        queue_push_cold(a.hdr, a.queue, a.qcap, en);
      }
    };
    // ---- 4. global index of the tile's first record, 5. write out -------------
    int64_t prefix = 0;
    int live_n = 0;  // records j < live_n have an output slot (capacity, snprintf-like)
    OutT* outp = nullptr;
    uint8_t* stp = nullptr;
    auto resolve = [&]() {
#if FPP_ABLATE == 3 || FPP_ABLATE == 4  // experiment: no look-back (output positions wrong; timing only)
      prefix = min((int64_t)tile * 200, a.capacity > 512 ? a.capacity - 512 : 0);
#else
#if FPP_PF_DIST > 0
      // L2 prefetch of a tile this counter hands out soon (FPP_PF_DIST claims
      // ahead of its current value), issued while the look-back's descriptor
      // loads are in flight: the claims of one counter are FPP_PF_DIST apart
      // in time by about that many claim intervals, so whoever claims that
      // tile finds it in L2
      bool pf_done = false;
      auto pf = [&]() {
        if (lane == 0 && !pf_done) {
          pf_done = true;
          unsigned c;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory");
          const int pt = (int)(c + FPP_PF_DIST) * a.nctr + g;
          if (split_interior(a, pt))
            prefetch_l2_bulk(a.bytes + ((int64_t)pt * kWarpStride - a.head - 16), kWarpStage);
        }
      };
      prefix = lookback(a.desc, tile, (uint64_t)total,
                        [&](int64_t u) { return count_tile_starts<SEPS>(a.bytes, a.len, a.head, u); },
                        (FPP_LB_DIAG && STATS && lane == 0) ? &acc.v[STAT_GLOBAL] : nullptr, pf);
      pf();
#elif FPP_EARLY_CLAIM == 3
      // the next tile claimed right after the look-back: the claim's round trip
      // overlaps the copy-out
      prefix = lookback(a.desc, tile, (uint64_t)total,
                        [&](int64_t u) { return count_tile_starts<SEPS>(a.bytes, a.len, a.head, u); },
                        (FPP_LB_DIAG && STATS && lane == 0) ? &acc.v[STAT_GLOBAL] : nullptr);
      if (lane == 0) nxt = (int)atom_add_u32(ctr, 1u) * a.nctr + g;
#elif FPP_EARLY_CLAIM
      // the next tile is claimed here, and its bytes requested into L2, while
      // this tile's look-back waits for its descriptors: the claim's round
      // trip and most of the next tile's DRAM latency overlap the look-back
      // and the copy-out (the staging copy itself needs the buffer, which
      // holds this tile's results until they are copied out)
      unsigned claimed = 0;
      if (lane == 0) claimed = atom_add_u32(ctr, 1u);
      auto take = [&]() {
        if (lane == 0 && nxt < 0) {
          nxt = (int)claimed * a.nctr + g;
          if (FPP_EARLY_CLAIM == 1 && split_interior(a, nxt))
            prefetch_l2_bulk(a.bytes + ((int64_t)nxt * kWarpStride - a.head - 16), kWarpStage);
        }
      };
      prefix = lookback(a.desc, tile, (uint64_t)total,
                        [&](int64_t u) { return count_tile_starts<SEPS>(a.bytes, a.len, a.head, u); },
                        (FPP_LB_DIAG && STATS && lane == 0) ? &acc.v[STAT_GLOBAL] : nullptr, take);
      take();  // tile 0 has no look-back
#else
      prefix = lookback(a.desc, tile, (uint64_t)total,
                        [&](int64_t u) { return count_tile_starts<SEPS>(a.bytes, a.len, a.head, u); },
                        (FPP_LB_DIAG && STATS && lane == 0) ? &acc.v[STAT_GLOBAL] : nullptr);
#endif
#endif
      if (lane == 0 && tile == a.ntiles - 1) *a.n_out = prefix + total;
      live_n = (int)max((int64_t)0, min((int64_t)total, a.capacity - prefix));
      outp = reinterpret_cast<OutT*>(a.out) + prefix;
      stp = a.status + prefix;
    };
    // pending records: the candidate and OK until the slow kernel decides
    auto write = [&](int j, int s, const Res& r) {
      if (j < live_n) {  // implies j < total
        outp[j] = (OutT)r.bits;
        stp[j] = (uint8_t)r.info;
        if (a.offsets_out) a.offsets_out[prefix + j] = base + s;
      }
    };
    if (compact) {
      // end of the tile's last record, decided once for the warp (so that the
      // lane holding it does not diverge from the others): the first halo
      // separator, else a search of the separator mask (long records, data end)
#if FPP_ABLATE == 5  // experiment: no rounds (claim, staging, classification, scan, compaction)
      if (lane == 0 && tile == a.ntiles - 1) *a.n_out = total;
      __syncwarp();
      continue;
#endif
      int e_last = 0;
      if (total > 0) e_last = halo ? (kWarpStride - 2) + __ffs(halo) : sep_end(S.starts[total - 1]);
      // sentinel: record j ends at starts[j + 1] - 1 for every j < total
      if (lane == 0) S.starts[total] = (uint16_t)(e_last + 1);
      __syncwarp();
      // One record per lane per round; in the last round the lanes past the
      // end parse the last record again and write nothing, so the parse
      // needs no branch on the lane.  The look-back waits for the
      // predecessors' counts and goes to L2, so it runs as late as possible:
      // after the whole tile (results buffered, below), else after the
      // second round with the first round's results held in registers.
      if (total == 0) {
        resolve();  // publishes the tile's (empty) inclusive prefix
      } else {
        const int rounds = (total + 31) >> 5;
        // Deferred look-back: round r's results (32 values and 32 status
        // bytes) wait in the already parsed front of the text buffer, at
        // text + 288 r, when that region ends before every later round's
        // records (and their 20-byte read-behind windows).  The look-back then
        // runs once the whole tile is parsed, when the predecessors have long
        // published inclusive prefixes, and the results are copied out.
        constexpr int kRoundBuf = 288;  // values and status bytes per round in the text front
#ifdef FPP_NO_DEFER
        bool defer = false;
#else
        bool defer = rounds > 1 && kRoundBuf * rounds <= kWarpStageAlloc;
#endif
        if (defer) {
          const int rr = lane + 1;
          defer = __all_sync(0xffffffffu, rr >= rounds || kRoundBuf * rr + 32 <= 16 + (int)S.starts[32 * rr]);
        }
        if (defer) {
          uint8_t* rb = text;  // round rd's results at text + 288 rd
          // "0.ddd" tiles (config 2's shape, %.17g of values in [1e-4, 1)):
          // when round 0's 32 records all have it, the tile runs a loop of
          // fast_frac0 -- no structure search, no integer part -- each lane
          // falling back to the general parse (out of line) for a record of
          // another shape.  Other tiles run the general loop, having paid one
          // vote.
          bool f0 = false;
#if FPP_F0_TILE
          f0 = tile_f0;
          if (f0) {
            for (int rd = 0; rd < rounds; rd++) {
              const int j = (rd << 5) + lane;
              const int jc = min(j, total - 1);
              const int s = S.starts[jc];
              const int e = (int)S.starts[jc + 1] - 1;
              Res r;
              if (!fast_frac0_tile<F32>(text, 16u + (uint32_t)s, (uint32_t)(e - s), r)) r = parse_ni(s, e);
              if (j < total) account(j, s, e, r);
              __syncwarp();  // every lane is done reading this round's text
              reinterpret_cast<unsigned long long*>(rb)[lane] = r.bits;
              rb[256 + lane] = (uint8_t)r.info;
              rb += 288;
            }
          } else
#else
          if (FPP_SHAPE && G == 0) {
            const int s0 = S.starts[min(lane, total - 1)];
            const int e0 = (int)S.starts[min(lane, total - 1) + 1] - 1;
            f0 = __all_sync(0xffffffffu,
                            frac0_shape(text, 16u + (uint32_t)s0, (uint32_t)(e0 - s0), mask_at(S.ndm, (uint32_t)s0)));
          }
          if (f0) {
            for (int rd = 0; rd < rounds; rd++) {
              const int j = (rd << 5) + lane;
              const int jc = min(j, total - 1);
              const int s = S.starts[jc];
              const int e = (int)S.starts[jc + 1] - 1;
              const uint32_t ts = 16u + (uint32_t)s, L = (uint32_t)(e - s);
              Res r;
              if (!(frac0_shape(text, ts, L, mask_at(S.ndm, (uint32_t)s)) && fast_frac0<F32>(text, ts, L, r)))
                r = parse_ni(s, e);
              if (j < total) account(j, s, e, r);
              __syncwarp();  // every lane is done reading this round's text
              reinterpret_cast<unsigned long long*>(rb)[lane] = r.bits;
              rb[256 + lane] = (uint8_t)r.info;
              rb += 288;
            }
          } else
#endif
          for (int rd = 0; rd < rounds; rd++) {
            const int j = (rd << 5) + lane;
            const int jc = min(j, total - 1);
            const int s = S.starts[jc];
            const int e = (int)S.starts[jc + 1] - 1;
            const Res r = parse(s, e);
            if (j < total) account(j, s, e, r);
            __syncwarp();  // every lane is done reading this round's text
            reinterpret_cast<unsigned long long*>(rb)[lane] = r.bits;
            rb[256 + lane] = (uint8_t)r.info;
            rb += 288;
          }
          __syncwarp();
          resolve();
          {
            const uint8_t* rb = text;
            OutT* o = outp + lane;
            uint8_t* so = stp + lane;
            for (int j = lane; j < live_n; j += 32, rb += 288, o += 32, so += 32) {
              *o = (OutT)reinterpret_cast<const unsigned long long*>(rb)[lane];
              *so = rb[256 + lane];
            }
          }
          if (a.offsets_out)
            for (int j = lane; j < live_n; j += 32) a.offsets_out[prefix + j] = base + S.starts[j];
        } else {
        // round 0, peeled: its results wait in registers for the look-back
        int s0;
        Res r0;
        {
          const int jc = min(lane, total - 1);
          s0 = S.starts[jc];
          const int e = (int)S.starts[jc + 1] - 1;
          r0 = parse_ni(s0, e);
          if (lane < total) account(lane, s0, e, r0);
        }
        if (rounds == 1) {
          resolve();
          write(lane, s0, r0);
        }
        for (int rd = 1; rd < rounds; rd++) {
          const int j = (rd << 5) + lane;
          const int jc = min(j, total - 1);
          const int s = S.starts[jc];
          const int e = (int)S.starts[jc + 1] - 1;
          const Res r = parse_ni(s, e);
          if (j < total) account(j, s, e, r);
          if (rd == 1) {  // warp-uniform
            resolve();
            write(lane, s0, r0);
          }
          write(j, s, r);
        }
        }
      }
    } else {
      // Own starts: every lane parses the records starting in its own bytes,
      // k-th record of lane l = record excl_l + k.  A record ends one byte
      // before the next start: the lane's next start bit, else the first
      // start of a later lane (suffix minimum over the warp, the halo's first
      // start standing after lane 31), else a search (long records, data end).
      constexpr int kNone = 1 << 20;
      uint64_t mlo = ((uint64_t)st[1] << 32) | st[0], mhi = ((uint64_t)st[3] << 32) | st[2];
      uint32_t mtop = W > 4 ? st[W > 4 ? 4 : 0] : 0u;  // bits 128..159 (5-word lanes)
      // lowest start of the lane at or after the bits still set (kNone if none)
      auto lane_first = [&]() -> int {
        return mlo ? x0 + __ffsll((long long)mlo) - 1
                   : (mhi ? x0 + 64 + __ffsll((long long)mhi) - 1 : (mtop ? x0 + 128 + __ffs(mtop) - 1 : kNone));
      };
      const int fs = lane_first();
      const int hf = halo ? (kWarpStride - 1) + __ffs(halo) : kNone;  // the halo's first start
      int suf = lane == 31 ? min(fs, hf) : fs;            // min of fs over lanes >= lane (and the halo)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_down_sync(0xffffffffu, suf, o);
        if (lane + o < 32) suf = min(suf, y);
      }
      int ns = __shfl_down_sync(0xffffffffu, suf, 1);  // first start after this lane
      if (lane == 31) ns = hf;
      const int rounds = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
      Res held;
      held.bits = 0;
      held.info = 0;
      int held_s = 0;
      bool resolved = false;
      for (int k = 0; k < (rounds == 0 ? 1 : rounds); k++) {
        int s = 0;
        Res r;
        r.bits = 0;
        r.info = 0;
        const bool have = k < cnt;
        if (have) {
          s = lane_first();  // have: some bit is still set
          if (mlo) mlo &= mlo - 1;
          else if (mhi) mhi &= mhi - 1;
          else mtop &= mtop - 1;
          const int nl = lane_first();
          const int nx = nl < kNone ? nl : ns;
          const int e = nx < kNone ? nx - 1 : sep_end(s);
          r = parse_ni(s, e);
          account(excl + k, s, e, r);
        }
        if (!resolved) {  // warp-uniform: look back after the second round
          if (k == 0 && rounds > 1) {
            held = r;
            held_s = s;
            continue;
          }
          resolve();
          resolved = true;
          if (k == 1) write(0 < cnt ? excl : (1 << 30), held_s, held);
        }
        write(have ? excl + k : (1 << 30), s, r);
      }
    }
    // the buffered results (and the ragged tiles' byte loads) were generic
    // writes to the buffer the next tile's bulk copy fills
    fence_proxy_async_smem();
    __syncwarp();
  }
  if (STATS) flush_stats(acc, a.stats);
}

}  // namespace fpp
