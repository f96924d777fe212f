// k_batch.cuh -- parse_f64_batch's fast kernel: records given by offsets.
//
// Persistent CTAs of 256 threads claim tiles of 512 records (atomicAdd), load
// their offsets, stage the covered text span in shared memory with one TMA
// bulk copy when the offsets are well formed (monotone, in range, <= 16 KiB),
// classify it into a non-digit bit mask and parse one record per thread with
// the SWAR scanner + Algorithm 1 (+ bracket).  Records outside the staged span
// (malformed offsets, long records) are read from global memory.  Undecided
// records are pushed to the slow queue; if the queue (sized from len) is full
// -- possible only with overlapping offsets -- the record is marked ST_PENDING
// in status[] for the slow kernel's fallback scan.
#pragma once
#include "k_common.cuh"

namespace fpp {

constexpr int kBatchThreads = 256;
constexpr int kBatchRecs = 512;                 // records per tile
constexpr int kBatchText = 16384;               // staged text capacity per tile
constexpr int kBatchMaskWords = kBatchText / 32;

// ============================================================================
struct BatchArgs {
  const uint8_t* bytes;
  int64_t len;
  int64_t head;  // bytes % 16
  const int64_t* offsets;
  int64_t n;
  int64_t ntiles;
  void* out;  // double[n] or (F32) float[n]
  uint8_t* status;
  WsHeader* hdr;
  SlowEntry* queue;
  uint64_t qcap;
  uint64_t* stats;
  uint32_t grammar;  // 0 or G_HEX / G_JSON
};

struct __align__(128) BatchSmem {
  uint8_t pad[32];  // digit windows may read up to 20 bytes before text
  uint8_t text[kBatchText + 64];
  uint64_t p10[20];
  int64_t offs[kBatchRecs + 1];
  uint32_t ndm[kBatchMaskWords + 2];
  unsigned long long bar;
  int64_t tile;
};

#ifndef FPP_BATCH_MINB
#define FPP_BATCH_MINB 8  // 32 registers: 8 CTAs of 256 threads per SM (the compiler's free choice, 40, allows 6)
#endif
template <bool STATS, bool F32, int G>
__global__ void __launch_bounds__(kBatchThreads, FPP_BATCH_MINB) k_batch(BatchArgs a) {
  using OutT = typename std::conditional<F32, uint32_t, unsigned long long>::type;
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
          r.bits = Fmt<F32>::kQNaN;
          r.info = ST_INVALID;
          count_stats<STATS>(acc, r, false);
        } else if (e - s > kLongRec) {  // the slow path scans it (k_slow_scan)
          r = long_record();
          count_stats<STATS>(acc, r, false);
        } else if (staged && s >= lo && e <= hi) {
          const uint32_t ts = (uint32_t)(s - p_al);
          r = parse_staged<true, F32, G>(S.text, ts, (uint32_t)(e - s), mask_at(S.ndm, ts), S.p10, a.grammar);
          count_stats<STATS>(acc, r, false);
        } else {
          r = parse_global<F32>(a.bytes, s, e, a.grammar);
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
        // in out[] and mark the record for the slow kernel's status scan (the
        // mark also says whether to check the lower neighbour, or that there
        // is no candidate yet)
        const bool mark = pend && !ok;
        const uint64_t cand = r.bits == kCandUnknown ? 0ull : (r.bits & ~kCandNoLower);
        reinterpret_cast<OutT*>(a.out)[r0 + j] = (OutT)(pend ? cand : r.bits);
        const uint8_t mk = r.bits == kCandUnknown ? (uint8_t)ST_PENDING_UNK
                           : ((r.bits & kCandNoLower) ? (uint8_t)ST_PENDING_LOW : (uint8_t)ST_PENDING);
        a.status[r0 + j] = mark ? mk : (uint8_t)(pend ? ST_OK : (r.info & 0xFF));
      }
    }
    fence_proxy_async_smem();  // ragged tiles' generic writes to the text the next bulk copy fills
    __syncthreads();
  }
  if (STATS) flush_stats(acc, a.stats);
}

}  // namespace fpp
