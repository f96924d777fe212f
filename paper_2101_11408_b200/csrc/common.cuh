// common.cuh -- constants and byte classes shared by the fpparse kernels.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace fpp {

constexpr uint64_t kQNaN = 0x7FF8000000000000ull;  // canonical quiet NaN (G10/G11)
constexpr uint64_t kInf = 0x7FF0000000000000ull;
constexpr uint64_t kSign = 1ull << 63;

// Output formats (PAPER.md table tab:commmonieee L123-135; Algorithm 1 gives
// both cases, L223-260): binary64 (F32 = false) and binary32 (F32 = true,
// SURVEY.md 8(f) f1).  Bits travel as uint64_t in both cases.
template <bool F32>
struct Fmt {
  static constexpr uint64_t kInf = 0x7FF0000000000000ull;
  static constexpr uint64_t kQNaN = 0x7FF8000000000000ull;
  static constexpr uint64_t kSign = 1ull << 63;
  static constexpr int kFracBits = 52;  // stored significand bits
  static constexpr int kCut = 9;        // 64 - 55: the high word's low bits below the 55 exact ones (L231)
  static constexpr int kEmin = -1022, kEmax = 1023;
  static constexpr int kTieLo = -4, kTieHi = 23;  // q range of possible ties (L287-333)
};
template <>
struct Fmt<true> {
  static constexpr uint64_t kInf = 0x7F800000ull;
  static constexpr uint64_t kQNaN = 0x7FC00000ull;
  static constexpr uint64_t kSign = 1ull << 31;
  static constexpr int kFracBits = 23;
  static constexpr int kCut = 38;  // 64 - 26 (L231, L757-760)
  static constexpr int kEmin = -126, kEmax = 127;
  static constexpr int kTieLo = -17, kTieHi = 10;
};

enum : uint8_t { ST_OK = 0, ST_OVERFLOW = 1, ST_UNDERFLOW = 2, ST_INVALID = 3, ST_EMPTY = 4,
                 // internal marks (batch queue overflow), resolved by the slow kernel, never returned:
                 // candidate in out[]; the same, also check the lower neighbour; no candidate yet
                 ST_PENDING = 0xFE, ST_PENDING_LOW = 0xFD, ST_PENDING_UNK = 0xFC };

enum : int { STAT_RECORDS = 0, STAT_TWO_MULT, STAT_BRACKET, STAT_SLOW, STAT_ABORT, STAT_GLOBAL,
             STAT_BAD, STAT_TILES, NSTATS };

// record kinds produced by the scanner (K_HEX: w * 2^q, tnz = nonzero nibbles dropped)
enum : int { K_NUM = 0, K_INF = 1, K_NAN = 2, K_INVALID = 3, K_EMPTY = 4, K_HEX = 5 };

// grammar options (include/fpparse.h FPP_GRAMMAR_*)
constexpr uint32_t G_HEX = 1u;   // also C99 hexadecimal floats
constexpr uint32_t G_JSON = 2u;  // RFC 8259 numbers only

__device__ __forceinline__ bool is_digit(uint32_t c) { return c - '0' < 10u; }
// terminators allowed after a number
__device__ __forceinline__ bool is_term(uint32_t c) { return c == '\n' || c == '\r' || c == ','; }
// separator test for the split variant; seps: bit0 '\n', bit1 ','
__device__ __forceinline__ bool is_sep(uint32_t c, uint32_t seps) {
  return ((seps & 1u) && c == '\n') || ((seps & 2u) && c == ',');
}

// Slow-path queue entry: the record, its output slot and the
// fast path's candidate.  cand bit 63 set = candidate not proven to be a lower
// bound (Algorithm 1 aborted) -> check both neighbours.
struct SlowEntry {
  int64_t idx;    // output index (>= 0), or split_queue_idx(tile, j) (< 0)
  int64_t start;  // absolute byte position of the record
  int64_t end;    // absolute end (exclusive), -1: find the next separator
  uint64_t cand;  // candidate bits (positive) | flag
};

// split-kernel queue entries name their record by (tile, index in tile): the
// output index is the tile's exclusive prefix (the predecessor's published
// inclusive count) plus j, resolved by the slow kernel.  Negative, so batch
// entries (plain output indices) are told apart.
constexpr int kSplitJBits = 13;  // j < 4064 records per tile
__device__ __forceinline__ int64_t split_queue_idx(int64_t tile, int j) {
  return ~((tile << kSplitJBits) | (int64_t)j);
}

// workspace header (zeroed per call)
// k_split's tile counters: counter g hands out tiles g, g + G, g + 2G, ...
// Each sits in its own 256-byte block after the header (its own L2 line and,
// by the address hash, its own L2 slice), so their atomics do not queue on
// one slice.
constexpr int kTileCtrs = 8;
constexpr int kTileCtrStride = 256;
struct WsHeader {
  unsigned int tile_ctr;      // dynamic tile claims (k_batch)
  unsigned int slow_ctr;      // slow-kernel work claims
  unsigned long long qcount;  // queue fill (may exceed qcap: overflow -> ST_PENDING scan)
  unsigned int scan_ctr;      // slow path phase A (k_slow_scan) claims
  unsigned int pad0;
  unsigned long long pad[5];
};
static_assert(sizeof(WsHeader) <= 256, "the workspace header is 256 bytes");
__device__ __forceinline__ unsigned int* split_ctr(WsHeader* hdr, int g) {
  return reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(hdr) + 256 + kTileCtrStride * g);
}
// the slow kernel's claim counters, one per block too (a different 128-byte line)
__device__ __forceinline__ unsigned int* slow_ctr_g(WsHeader* hdr, int g) {
  return reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(hdr) + 256 + kTileCtrStride * g + 128);
}

// ---- TMA bulk copy global -> shared with an mbarrier (sm_90+; UBLKCP in SASS) ----
__device__ __forceinline__ uint32_t cvta_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(cvta_smem(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// every thread that wrote (generic proxy) to a buffer a later bulk copy
// (async proxy) overwrites: order those writes before the copy (then a
// warp / CTA barrier, then the issuing thread's own fence in tma_load_1d)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// issue (one thread): expect `bytes` and start the bulk copy; src/dst 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cvta_smem(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          cvta_smem(dst)),
      "l"(src), "r"(bytes), "r"(cvta_smem(bar))
      : "memory");
}
// the same without the fence (the caller fenced its generic writes already)
__device__ __forceinline__ void tma_load_1d_nf(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(cvta_smem(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          cvta_smem(dst)),
      "l"(src), "r"(bytes), "r"(cvta_smem(bar))
      : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (one thread; 16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(cvta_smem(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace fpp
