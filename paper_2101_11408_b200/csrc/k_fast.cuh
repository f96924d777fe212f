// k_fast.cuh -- the fast kernels: record splitter + scanner + Algorithm 1.
//
// k_split (parse_f64_split): persistent CTAs claim byte tiles in order
// (atomicAdd), stage tile + halo in shared memory with 16-byte loads, find the
// separators with SWAR byte compares, count record starts with popc and a block
// scan, obtain the tile's first global record index from a decoupled
// look-back over the tiles' counts, then parse one record per thread from
// shared memory.  Records running past the staged halo are read from global
// memory.  Undecided records (bracket failed / Algorithm 1 abort) are pushed to
// the slow-path queue with a warp-aggregated atomicAdd.
//
// k_batch (parse_f64_batch): persistent CTAs claim tiles of R records, load
// their offsets, stage the covered text span in shared memory when the offsets
// are well formed, and parse one record per thread.
#pragma once
#include "decide.cuh"

namespace fpp {

constexpr int kSplitThreads = 256;
constexpr int kSplitTile = 32 * kSplitThreads;  // 8 KiB of text per tile, 32 B per thread
constexpr int kSplitHalo = 128;                 // bytes staged beyond the tile
constexpr int kSplitStage = 16 + kSplitTile + kSplitHalo;

constexpr int kBatchThreads = 256;
constexpr int kBatchRecs = 512;                 // records per tile
constexpr int kBatchText = 16384;               // staged text capacity per tile

constexpr uint64_t kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = (1ull << 62) - 1;

struct StatAcc {
  uint32_t v[NSTATS];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < NSTATS; i++) v[i] = 0;
  }
};

__device__ __forceinline__ void flush_stats(StatAcc& acc, uint64_t* stats) {
  if (stats == nullptr) return;
#pragma unroll
  for (int i = 0; i < NSTATS; i++) {
    uint32_t x = acc.v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd((unsigned long long*)&stats[i], (unsigned long long)x);
  }
}

// stage 16-byte chunk `c` of a window starting at absolute-aligned position p
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

// 4-bit mask of separator bytes in a little-endian word
__device__ __forceinline__ uint32_t sep_nibble(uint32_t v, uint32_t seps) {
  uint32_t hit = 0;
  if (seps & 1u) {
    uint32_t x = v ^ 0x0A0A0A0Au;
    hit |= ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
  }
  if (seps & 2u) {
    uint32_t x = v ^ 0x2C2C2C2Cu;
    hit |= ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
  }
  return (((hit >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// warp-aggregated push onto the slow queue; returns false if the queue is full
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

// decoupled look-back (warp 0 of the CTA); returns the exclusive prefix
__device__ __forceinline__ int64_t lookback(uint64_t* desc, int64_t tile, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(&desc[0], kFlagInc | agg);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(&desc[tile], kFlagAgg | agg);
  uint64_t excl = 0;
  int64_t look = tile - 1;
  while (true) {
    const int64_t t = look - lane;
    uint64_t d = (t >= 0) ? ld_relaxed_u64(&desc[t]) : kFlagInc;
    const unsigned inc = __ballot_sync(0xffffffffu, (d >> 62) == 2);
    const unsigned zero = __ballot_sync(0xffffffffu, (d >> 62) == 0);
    const unsigned upto = inc ? ((inc & (0u - inc)) << 1) - 1 : 0xffffffffu;  // lanes <= first inclusive
    if (zero & upto) continue;  // a predecessor has not published yet: re-read
    uint64_t v = (upto >> lane) & 1 ? (d & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc) break;
    look -= 32;
  }
  if (lane == 0) st_relaxed_u64(&desc[tile], kFlagInc | (excl + agg));
  return (int64_t)excl;
}

struct SplitArgs {
  const uint8_t* bytes;
  int64_t len;
  int64_t head;      // bytes % 16: tile t covers positions [t*TILE - head, (t+1)*TILE - head)
  int64_t ntiles;
  uint32_t seps;
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

__global__ void __launch_bounds__(kSplitThreads) k_split(SplitArgs a) {
  __shared__ __align__(16) uint8_t text[kSplitStage];
  __shared__ uint16_t starts[kSplitTile];
  __shared__ uint64_t T[1302];
  __shared__ int warp_tot[kSplitThreads / 32];
  __shared__ int64_t s_prefix;
  __shared__ int64_t s_tile;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 1302; i += kSplitThreads) T[i] = kPow5_128[i];
  StatAcc acc;
  acc.zero();

  while (true) {
    if (tid == 0) s_tile = (int64_t)atomicAdd(&a.hdr->tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= a.ntiles) break;
    const int64_t base = tile * kSplitTile - a.head;  // position of text[16]
    // ---- stage [base - 16, base + TILE + HALO) -------------------------------
    for (int c = tid; c < kSplitStage / 16; c += kSplitThreads)
      *reinterpret_cast<uint4*>(&text[16 * c]) = load_chunk(a.bytes, a.len, base - 16 + 16 * c);
    __syncthreads();
    // ---- record starts in [32*tid, 32*tid + 32) ------------------------------
    const int x0 = 32 * tid;
    const uint4 v0 = *reinterpret_cast<const uint4*>(&text[16 + x0]);
    const uint4 v1 = *reinterpret_cast<const uint4*>(&text[32 + x0]);
    uint32_t msep = sep_nibble(v0.x, a.seps) | (sep_nibble(v0.y, a.seps) << 4) |
                    (sep_nibble(v0.z, a.seps) << 8) | (sep_nibble(v0.w, a.seps) << 12) |
                    (sep_nibble(v1.x, a.seps) << 16) | (sep_nibble(v1.y, a.seps) << 20) |
                    (sep_nibble(v1.z, a.seps) << 24) | (sep_nibble(v1.w, a.seps) << 28);
    const uint32_t prev = is_sep(text[15 + x0], a.seps) ? 1u : 0u;
    uint32_t smask = (msep << 1) | prev;  // bit b: a record starts at x0 + b
    const int64_t p0 = base + x0;
    if (p0 <= 0 && p0 + 32 > 0) smask |= 1u << (int)(-p0);  // position 0 starts record 0
    // keep positions in [0, len)
    if (p0 < 0) smask &= (p0 <= -32) ? 0u : (0xffffffffu << (int)(-p0));
    if (p0 + 32 > a.len) smask &= (p0 >= a.len) ? 0u : (0xffffffffu >> (int)(p0 + 32 - a.len));
    const int cnt = __popc(smask);
    // ---- block exclusive scan of counts --------------------------------------
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kSplitThreads / 32; w++) {
      int t = warp_tot[w];
      wbase += (w < warp) ? t : 0;
      total += t;
    }
    int o = wbase + incl - cnt;
    for (uint32_t m = smask; m; m &= m - 1) starts[o++] = (uint16_t)(x0 + __ffs(m) - 1);
    // ---- decoupled look-back -------------------------------------------------
    if (warp == 0) {
      int64_t pre = lookback(a.desc, tile, (uint64_t)total);
      if (lane == 0) {
        s_prefix = pre;
        if (tile == a.ntiles - 1) *a.n_out = pre + total;
      }
    }
    __syncthreads();
    const int64_t prefix = s_prefix;
    acc.v[STAT_TILES] += (tid == 0);
    // ---- parse: one record per thread ----------------------------------------
    for (int j = tid; j < ((total + 31) & ~31); j += kSplitThreads) {
      const bool have = j < total;
      int64_t gidx = prefix + j;
      bool live = have && gidx < a.capacity;
      Decision d;
      d.pending = false;
      int64_t rs = 0, re = 0;
      if (live) {
        const int s = starts[j];
        int e = -1;
        if (j + 1 < total) {
          e = starts[j + 1] - 1;
        } else {
          for (int x = s; x < kSplitTile + kSplitHalo; x++) {
            if (base + x >= a.len || is_sep(text[16 + x], a.seps)) { e = x; break; }
          }
        }
        rs = base + s;
        const uint8_t* ptr;
        if (e >= 0) {
          re = base + e;
          ptr = &text[16 + s];
        } else {  // long record: continue the separator search in global memory
          int64_t p = base + kSplitTile + kSplitHalo;
          while (p < a.len && !is_sep(a.bytes[p], a.seps)) p++;
          re = p;
          ptr = a.bytes + rs;
          acc.v[STAT_GLOBAL]++;
        }
        const int64_t L = re - rs;
        Scan sc;
        if (L >= (1ll << 31)) { sc.kind = K_INVALID; sc.neg = false; sc.tnz = false; sc.w = 0; sc.q = 0; }
        else sc = scan_record(ptr, (uint32_t)L);
        d = decide(sc, T);
        a.out[gidx] = __longlong_as_double((long long)d.bits);
        a.status[gidx] = d.st;
        if (a.offsets_out) a.offsets_out[gidx] = rs;
        acc.v[STAT_RECORDS]++;
        acc.v[STAT_TWO_MULT] += d.two;
        acc.v[STAT_BRACKET] += d.bracket;
        acc.v[STAT_ABORT] += d.abort;
        acc.v[STAT_SLOW] += d.pending;
        acc.v[STAT_BAD] += (d.st == ST_INVALID || d.st == ST_EMPTY);
      }
      SlowEntry e;
      e.idx = gidx;
      e.start = rs;
      e.end = re;
      e.cand = d.cand;
      queue_push(live && d.pending, a.hdr, a.queue, a.qcap, e);  // split queue cannot overflow
    }
    __syncthreads();
  }
  flush_stats(acc, a.stats);
}

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

__global__ void __launch_bounds__(kBatchThreads) k_batch(BatchArgs a) {
  __shared__ __align__(16) uint8_t text[kBatchText + 32];
  __shared__ int64_t offs[kBatchRecs + 1];
  __shared__ uint64_t T[1302];
  __shared__ int64_t s_tile;

  const int tid = threadIdx.x;
  for (int i = tid; i < 1302; i += kBatchThreads) T[i] = kPow5_128[i];
  StatAcc acc;
  acc.zero();

  while (true) {
    if (tid == 0) s_tile = (int64_t)atomicAdd(&a.hdr->tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= a.ntiles) break;
    const int64_t r0 = tile * kBatchRecs;
    const int cnt = (int)min((int64_t)kBatchRecs, a.n - r0);
    for (int k = tid; k <= cnt; k += kBatchThreads)
      offs[k] = (r0 + k < a.n) ? a.offsets[r0 + k] : a.len;
    __syncthreads();
    const int64_t lo = offs[0], hi = offs[cnt];
    // stage the text span when the tile's offsets are well formed
    const int64_t p_al = lo - ((lo + a.head) & 15);  // absolute 16-byte aligned
    const bool staged = lo >= 0 && lo <= hi && hi <= a.len && hi - p_al <= kBatchText;
    if (staged) {
      const int nch = (int)((hi - p_al + 15) >> 4);
      for (int c = tid; c < nch; c += kBatchThreads)
        *reinterpret_cast<uint4*>(&text[16 * c]) = load_chunk(a.bytes, a.len, p_al + 16 * c);
    }
    __syncthreads();
    acc.v[STAT_TILES] += (tid == 0);
    for (int j = tid; j < ((cnt + 31) & ~31); j += kBatchThreads) {
      const bool have = j < cnt;
      Decision d;
      d.pending = false;
      int64_t s = 0, e = 0;
      if (have) {
        s = offs[j];
        e = offs[j + 1];
        if (s < 0 || s > a.len || e < s || e > a.len || e - s >= (1ll << 31)) {
          d.bits = kQNaN;
          d.st = ST_INVALID;
        } else {
          const uint8_t* ptr;
          if (staged && s >= lo && e <= hi) ptr = &text[s - p_al];
          else { ptr = a.bytes + s; acc.v[STAT_GLOBAL]++; }
          Scan sc = scan_record(ptr, (uint32_t)(e - s));
          d = decide(sc, T);
          acc.v[STAT_TWO_MULT] += d.two;
          acc.v[STAT_BRACKET] += d.bracket;
          acc.v[STAT_ABORT] += d.abort;
          acc.v[STAT_SLOW] += d.pending;
        }
        acc.v[STAT_RECORDS]++;
        acc.v[STAT_BAD] += (d.st == ST_INVALID || d.st == ST_EMPTY);
      }
      SlowEntry ent;
      ent.idx = r0 + j;
      ent.start = s;
      ent.end = e;
      ent.cand = d.cand;
      const bool ok = queue_push(have && d.pending, a.hdr, a.queue, a.qcap, ent);
      if (have) {
        // queue overflow (only with overlapping offsets): leave the candidate
        // in out[] and mark the record for the slow kernel's status scan
        const bool mark = d.pending && !ok;
        a.out[r0 + j] = __longlong_as_double((long long)(mark ? d.cand : d.bits));
        a.status[r0 + j] = mark ? ST_PENDING : d.st;
      }
    }
    __syncthreads();
  }
  flush_stats(acc, a.stats);
}

}  // namespace fpp
