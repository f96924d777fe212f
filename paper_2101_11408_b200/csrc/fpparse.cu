// fpparse.cu -- C ABI (include/fpparse.h) and launch logic.
//
// parse_f{64,32}_split:  memset(workspace header + look-back descriptors)
//                        -> k_split (persistent) -> k_slow (persistent)
// parse_f{64,32}_batch:  memset(workspace header) -> k_batch -> k_slow
// The binary32 entry points run the same kernels instantiated with F32 =
// true (Fmt<true>, common.cuh).  All work is enqueued on the caller's stream;
// no host synchronisation.
#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <cstring>
#include <mutex>

#include "../../include/fpparse.h"
#include "k_batch.cuh"
#include "k_split.cuh"
#include "k_slow.cuh"

using namespace fpp;

namespace {

constexpr size_t kHdrBytes = 256 + kTileCtrs * kTileCtrStride;  // header + the split tile counters

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// a queued split record is at least 20 bytes plus its separator (DESIGN.md
// "Data layout"), so len / 20 entries always suffice
inline uint64_t split_qcap(size_t len) { return (uint64_t)(len / 20) + 1024; }
inline int64_t split_ntiles(size_t len, int64_t head) {
  return (int64_t)((len + (size_t)head + kWarpStride - 1) / kWarpStride);
}
inline uint64_t batch_qcap(size_t len, int64_t n) {
  uint64_t c = (uint64_t)(len / 16) + 1024;
  return (uint64_t)n < c ? (uint64_t)n : c;
}

struct DevInfo {
  int sms = 0;
  int occ_split = 0, occ_batch = 0, occ_slow = 0, occ_scan = 0;
};

DevInfo g_dev[64];
std::mutex g_dev_mu[64];                 // first-call initialisation, per device
std::atomic<bool> g_dev_ready[64];       // published after g_dev[dev] is complete

// profiling hook (fpp_set_profile_events): events recorded around the kernels
std::atomic<cudaEvent_t> g_ev_before_fast{nullptr}, g_ev_after_fast{nullptr}, g_ev_after_slow{nullptr};

inline void rec(const std::atomic<cudaEvent_t>& e, cudaStream_t st) {
  cudaEvent_t ev = e.load(std::memory_order_acquire);
  if (ev) cudaEventRecord(ev, st);
}

// occupancy and SM count of the current device, computed once (thread-safe:
// a mutex per device for the first call, then an acquire load)
bool dev_info(DevInfo& di) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  DevInfo& d = g_dev[dev];
  if (g_dev_ready[dev].load(std::memory_order_acquire)) {
    di = d;
    return true;
  }
  std::lock_guard<std::mutex> lock(g_dev_mu[dev]);
  if (!g_dev_ready[dev].load(std::memory_order_relaxed)) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return false;
    int o1 = 0, o2 = 0, o3 = 0;
    const int ss = (int)sizeof(SplitSmem), bs = (int)sizeof(BatchSmem);
    const void* ks[36] = {
        (const void*)k_split<1, false, false, 0>,
        (const void*)k_split<2, false, false, 0>,
        (const void*)k_split<3, false, false, 0>,
        (const void*)k_split<1, true, false, 0>,
        (const void*)k_split<2, true, false, 0>,
        (const void*)k_split<3, true, false, 0>,
        (const void*)k_split<1, false, true, 0>,
        (const void*)k_split<2, false, true, 0>,
        (const void*)k_split<3, false, true, 0>,
        (const void*)k_split<1, true, true, 0>,
        (const void*)k_split<2, true, true, 0>,
        (const void*)k_split<3, true, true, 0>,
        (const void*)k_split<1, false, false, 1>,
        (const void*)k_split<2, false, false, 1>,
        (const void*)k_split<3, false, false, 1>,
        (const void*)k_split<1, true, false, 1>,
        (const void*)k_split<2, true, false, 1>,
        (const void*)k_split<3, true, false, 1>,
        (const void*)k_split<1, false, true, 1>,
        (const void*)k_split<2, false, true, 1>,
        (const void*)k_split<3, false, true, 1>,
        (const void*)k_split<1, true, true, 1>,
        (const void*)k_split<2, true, true, 1>,
        (const void*)k_split<3, true, true, 1>,
        (const void*)k_split<1, false, false, 2>,
        (const void*)k_split<2, false, false, 2>,
        (const void*)k_split<3, false, false, 2>,
        (const void*)k_split<1, true, false, 2>,
        (const void*)k_split<2, true, false, 2>,
        (const void*)k_split<3, true, false, 2>,
        (const void*)k_split<1, false, true, 2>,
        (const void*)k_split<2, false, true, 2>,
        (const void*)k_split<3, false, true, 2>,
        (const void*)k_split<1, true, true, 2>,
        (const void*)k_split<2, true, true, 2>,
        (const void*)k_split<3, true, true, 2>};
    for (const void* k : ks)
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ss) != cudaSuccess) return false;
    const void* kb[12] = {
        (const void*)k_batch<false, false, 0>,
        (const void*)k_batch<true, false, 0>,
        (const void*)k_batch<false, true, 0>,
        (const void*)k_batch<true, true, 0>,
        (const void*)k_batch<false, false, 1>,
        (const void*)k_batch<true, false, 1>,
        (const void*)k_batch<false, true, 1>,
        (const void*)k_batch<true, true, 1>,
        (const void*)k_batch<false, false, 2>,
        (const void*)k_batch<true, false, 2>,
        (const void*)k_batch<false, true, 2>,
        (const void*)k_batch<true, true, 2>};
    for (const void* k : kb)
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bs) != cudaSuccess) return false;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_split<1, false, false, 0>, 32 * kSplitWarps, ss) != cudaSuccess)
      return false;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_batch<false, false, 0>, kBatchThreads, bs) != cudaSuccess)
      return false;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, k_slow<false>, kSlowThreads, 0) != cudaSuccess) return false;
    int o4 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, k_slow_scan<false>, kSlowThreads, 0) != cudaSuccess)
      return false;
    d.occ_scan = o4 > 0 ? o4 : 1;
    d.occ_split = o1 > 0 ? o1 : 1;
    d.occ_batch = o2 > 0 ? o2 : 1;
    d.occ_slow = o3 > 0 ? o3 : 1;
    d.sms = sms;
    g_dev_ready[dev].store(true, std::memory_order_release);
  }
  di = d;
  return true;
}

template <bool F32>
int launch_slow(const uint8_t* bytes, int64_t len, const int64_t* offsets, int64_t n, uint32_t seps,
                void* out, uint8_t* status, WsHeader* hdr, SlowEntry* queue, uint64_t qcap,
                const uint64_t* desc, int64_t capacity, uint32_t grammar, const DevInfo& di, cudaStream_t st,
                int64_t* n_out = nullptr) {
  SlowArgs a;
  a.bytes = bytes;
  a.len = len;
  a.offsets = offsets;
  a.n = n;
  a.seps = seps;
  a.out = out;
  a.status = status;
  a.hdr = hdr;
  a.queue = queue;
  a.qcap = qcap;
  a.desc = desc;
  a.capacity = capacity;
  a.grammar = grammar;
  a.n_out = n_out;
  k_slow_scan<F32><<<di.sms * di.occ_scan, kSlowThreads, 0, st>>>(a);
  k_slow<F32><<<di.sms * di.occ_slow, kSlowThreads, 0, st>>>(a);
  rec(g_ev_after_slow, st);
  return cudaGetLastError() == cudaSuccess ? FPP_SUCCESS : FPP_ECUDA;
}

}  // namespace

extern "C" {

size_t fpp_workspace_bytes_split(size_t len) {
  const int64_t nt = split_ntiles(len, 15);
  return kHdrBytes + align256((size_t)nt * 8) + align256(split_qcap(len) * sizeof(SlowEntry));
}

size_t fpp_workspace_bytes_batch(size_t len, int64_t n) {
  if (n < 0) n = 0;
  return kHdrBytes + align256(batch_qcap(len, n) * sizeof(SlowEntry));
}

}  // extern "C"

namespace {

template <bool F32, int G>
void launch_split(const SplitArgs& a, uint32_t seps, bool stats, int grid, cudaStream_t st) {
  const size_t ss = sizeof(SplitSmem);
  if (!stats) {
    if (seps == 1) k_split<1, false, F32, G><<<grid, 32 * kSplitWarps, ss, st>>>(a);
    else if (seps == 2) k_split<2, false, F32, G><<<grid, 32 * kSplitWarps, ss, st>>>(a);
    else k_split<3, false, F32, G><<<grid, 32 * kSplitWarps, ss, st>>>(a);
  } else {
    if (seps == 1) k_split<1, true, F32, G><<<grid, 32 * kSplitWarps, ss, st>>>(a);
    else if (seps == 2) k_split<2, true, F32, G><<<grid, 32 * kSplitWarps, ss, st>>>(a);
    else k_split<3, true, F32, G><<<grid, 32 * kSplitWarps, ss, st>>>(a);
  }
}

inline bool grammar_ok(uint32_t g) { return g <= 2u; }  // FPP_GRAMMAR_HEX and _JSON exclude each other

template <bool F32>
int split_ws(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out, int64_t capacity,
             int64_t* n_out, void* out, uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats,
             void* stream, uint32_t grammar = 0) {
  if (!grammar_ok(grammar)) return FPP_EARG;
  if ((bytes == nullptr && len > 0) || capacity < 0 || n_out == nullptr || sep_mask > 3 ||
      ((out == nullptr || status == nullptr) && capacity > 0) || ws == nullptr)
    return FPP_EARG;
  if (ws_bytes < fpp_workspace_bytes_split(len)) return FPP_ECAPACITY;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return FPP_EARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (len == 0) {
    return cudaMemsetAsync(n_out, 0, sizeof(int64_t), st) == cudaSuccess ? FPP_SUCCESS : FPP_ECUDA;
  }
  DevInfo di;
  if (!dev_info(di)) return FPP_ECUDA;
  const int64_t head = (int64_t)(reinterpret_cast<uintptr_t>(bytes) & 15);
  const int64_t ntiles = split_ntiles(len, head);
  if (ntiles > (int64_t)0x7FFFFFF0) return FPP_EARG;  // tile indices are 32-bit (inputs up to ~10 TB)
  uint8_t* w = static_cast<uint8_t*>(ws);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(w);
  uint64_t* desc = reinterpret_cast<uint64_t*>(w + kHdrBytes);
  SlowEntry* queue = reinterpret_cast<SlowEntry*>(w + kHdrBytes + align256((size_t)split_ntiles(len, 15) * 8));
  if (cudaMemsetAsync(w, 0, kHdrBytes + (size_t)ntiles * 8, st) != cudaSuccess) return FPP_ECUDA;
  SplitArgs a;
  a.bytes = reinterpret_cast<const uint8_t*>(bytes);
  a.len = (int64_t)len;
  a.head = head;
  a.ntiles = ntiles;
  const uint32_t a_seps = sep_mask == 0 ? 3u : sep_mask;
  a.offsets_out = offsets_out;
  a.capacity = capacity;
  a.n_out = n_out;
  a.out = out;
  a.status = status;
  a.hdr = hdr;
  a.desc = desc;
  a.queue = queue;
  a.qcap = split_qcap(len);
  a.stats = stats;
  int grid = di.sms * di.occ_split;
  if ((int64_t)grid > ntiles) grid = (int)ntiles;
  rec(g_ev_before_fast, st);
  a.grammar = grammar;
  a.nctr = grid < kTileCtrs ? grid : kTileCtrs;  // every counter has CTAs draining it
  {
    // interior tiles: 1 <= t and t * kWarpStride - head + kWarpTile <= len
    const int64_t li = ((int64_t)len + head - kWarpTile) / kWarpStride;
    a.last_interior = (int)(li < 0 ? 0 : (li > ntiles - 1 ? ntiles - 1 : li));
  }
  if (grammar & G_JSON) launch_split<F32, 2>(a, a_seps, stats != nullptr, grid, st);
  else if (grammar & G_HEX) launch_split<F32, 1>(a, a_seps, stats != nullptr, grid, st);
  else launch_split<F32, 0>(a, a_seps, stats != nullptr, grid, st);
  rec(g_ev_after_fast, st);
  if (cudaGetLastError() != cudaSuccess) return FPP_ECUDA;
  return launch_slow<F32>(a.bytes, a.len, nullptr, 0, a_seps, out, status, hdr, queue, a.qcap, desc, capacity,
                          grammar, di, st, n_out);
}

template <bool F32>
int batch_ws(const char* bytes, size_t len, const int64_t* offsets, int64_t n, void* out, uint8_t* status,
             void* ws, size_t ws_bytes, uint64_t* stats, void* stream, uint32_t grammar = 0) {
  if (!grammar_ok(grammar)) return FPP_EARG;
  if (n < 0 || (bytes == nullptr && len > 0) ||
      ((offsets == nullptr || out == nullptr || status == nullptr) && n > 0) || ws == nullptr)
    return FPP_EARG;
  if (ws_bytes < fpp_workspace_bytes_batch(len, n)) return FPP_ECAPACITY;
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return FPP_EARG;
  if (n == 0) return FPP_SUCCESS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  DevInfo di;
  if (!dev_info(di)) return FPP_ECUDA;
  uint8_t* w = static_cast<uint8_t*>(ws);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(w);
  SlowEntry* queue = reinterpret_cast<SlowEntry*>(w + kHdrBytes);
  if (cudaMemsetAsync(w, 0, kHdrBytes, st) != cudaSuccess) return FPP_ECUDA;
  BatchArgs a;
  a.bytes = reinterpret_cast<const uint8_t*>(bytes);
  a.len = (int64_t)len;
  a.head = (int64_t)(reinterpret_cast<uintptr_t>(bytes) & 15);
  a.offsets = offsets;
  a.n = n;
  a.ntiles = (n + kBatchRecs - 1) / kBatchRecs;
  a.out = out;
  a.status = status;
  a.hdr = hdr;
  a.queue = queue;
  a.qcap = batch_qcap(len, n);
  a.stats = stats;
  int grid = di.sms * di.occ_batch;
  if ((int64_t)grid > a.ntiles) grid = (int)a.ntiles;
  rec(g_ev_before_fast, st);
  a.grammar = grammar;
  const size_t bs = sizeof(BatchSmem);
  if (grammar & G_JSON) {
    if (stats == nullptr) k_batch<false, F32, 2><<<grid, kBatchThreads, bs, st>>>(a);
    else k_batch<true, F32, 2><<<grid, kBatchThreads, bs, st>>>(a);
  } else if (grammar & G_HEX) {
    if (stats == nullptr) k_batch<false, F32, 1><<<grid, kBatchThreads, bs, st>>>(a);
    else k_batch<true, F32, 1><<<grid, kBatchThreads, bs, st>>>(a);
  } else {
    if (stats == nullptr) k_batch<false, F32, 0><<<grid, kBatchThreads, bs, st>>>(a);
    else k_batch<true, F32, 0><<<grid, kBatchThreads, bs, st>>>(a);
  }
  rec(g_ev_after_fast, st);
  if (cudaGetLastError() != cudaSuccess) return FPP_ECUDA;
  return launch_slow<F32>(a.bytes, a.len, offsets, n, 3u, out, status, hdr, queue, a.qcap, nullptr, n, grammar, di,
                          st);
}

template <bool F32>
int split_alloc(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out, int64_t capacity,
                int64_t* n_out, void* out, uint8_t* status, void* stream) {
  if ((bytes == nullptr && len > 0) || capacity < 0 || n_out == nullptr || sep_mask > 3 ||
      ((out == nullptr || status == nullptr) && capacity > 0))
    return FPP_EARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t wsb = fpp_workspace_bytes_split(len);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, wsb, st) != cudaSuccess) return FPP_ECUDA;
  int rc = split_ws<F32>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, ws, wsb, nullptr, stream);
  if (cudaFreeAsync(ws, st) != cudaSuccess && rc == FPP_SUCCESS) rc = FPP_ECUDA;
  return rc;
}

template <bool F32>
int batch_alloc(const char* bytes, size_t len, const int64_t* offsets, int64_t n, void* out, uint8_t* status,
                void* stream) {
  if (n < 0 || (bytes == nullptr && len > 0) ||
      ((offsets == nullptr || out == nullptr || status == nullptr) && n > 0))
    return FPP_EARG;
  if (n == 0) return FPP_SUCCESS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t wsb = fpp_workspace_bytes_batch(len, n);
  void* ws = nullptr;
  if (cudaMallocAsync(&ws, wsb, st) != cudaSuccess) return FPP_ECUDA;
  int rc = batch_ws<F32>(bytes, len, offsets, n, out, status, ws, wsb, nullptr, stream);
  if (cudaFreeAsync(ws, st) != cudaSuccess && rc == FPP_SUCCESS) rc = FPP_ECUDA;
  return rc;
}

template <bool F32>
int split_ex(const char* bytes, size_t len, uint32_t sep_mask, uint32_t grammar, int64_t* offsets_out,
             int64_t capacity, int64_t* n_out, void* out, uint8_t* status, void* ws, size_t ws_bytes,
             uint64_t* stats, void* stream) {
  if (ws != nullptr)
    return split_ws<F32>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, ws, ws_bytes, stats,
                         stream, grammar);
  if (!grammar_ok(grammar)) return FPP_EARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t wsb = fpp_workspace_bytes_split(len);
  void* w = nullptr;
  if (cudaMallocAsync(&w, wsb, st) != cudaSuccess) return FPP_ECUDA;
  int rc = split_ws<F32>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, w, wsb, stats, stream,
                         grammar);
  if (cudaFreeAsync(w, st) != cudaSuccess && rc == FPP_SUCCESS) rc = FPP_ECUDA;
  return rc;
}

template <bool F32>
int batch_ex(const char* bytes, size_t len, const int64_t* offsets, int64_t n, uint32_t grammar, void* out,
             uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream) {
  if (ws != nullptr) return batch_ws<F32>(bytes, len, offsets, n, out, status, ws, ws_bytes, stats, stream, grammar);
  if (!grammar_ok(grammar)) return FPP_EARG;
  if (n == 0) return FPP_SUCCESS;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t wsb = fpp_workspace_bytes_batch(len, n);
  void* w = nullptr;
  if (cudaMallocAsync(&w, wsb, st) != cudaSuccess) return FPP_ECUDA;
  int rc = batch_ws<F32>(bytes, len, offsets, n, out, status, w, wsb, stats, stream, grammar);
  if (cudaFreeAsync(w, st) != cudaSuccess && rc == FPP_SUCCESS) rc = FPP_ECUDA;
  return rc;
}

// ---------------------------------------------------------------------------
// Host-buffer streaming (parse_f{64,32}_split_host): the text is cut into
// chunks that end right after a separator (so no record spans two chunks and
// the record sequence equals the whole buffer's), and a pipeline of kSlots
// device slots overlaps, per chunk, the host->device copy, the split parse
// (k_split + k_slow on the caller's stream) and the device->host copy of the
// previous chunk's results.  Copies in both directions run on their own
// streams, so PCIe carries text in and results out at the same time.  The host
// waits only for each chunk's record count, one chunk behind the GPU.
constexpr int kSlots = 3;

__global__ void k_add_base(int64_t* p, int64_t n, int64_t base) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] += base;
}

struct HostSlot {
  char* text = nullptr;
  void* out = nullptr;
  uint8_t* status = nullptr;
  int64_t* offs = nullptr;
  int64_t* n_out = nullptr;    // device alias of n_host (mapped pinned memory)
  int64_t* n_host = nullptr;   // the record count, written by the kernels, read after `parsed`
  void* ws = nullptr;
  size_t ws_bytes = 0;
  cudaEvent_t in_done = nullptr, parsed = nullptr, out_done = nullptr;
  int64_t base_rec = 0, base_byte = 0, nrec = 0;
  bool busy = false;
};

// end of the chunk that starts at `start`: the first separator at or after
// start + chunk - 1, plus one (or len)
inline size_t chunk_end(const char* h, size_t len, size_t start, size_t chunk, uint32_t seps) {
  size_t e = start + chunk;
  if (e >= len) return len;
  e -= 1;
  while (e < len) {
    const unsigned char c = (unsigned char)h[e];
    if (((seps & 1u) && c == '\n') || ((seps & 2u) && c == ',')) return e + 1;
    e++;
  }
  return len;
}

// device slots, copy streams and events of the streaming call, kept per device
// across calls (allocating ~2 GB per call would cost more than the parse);
// one call at a time per device (the mutex)
struct HostCtx {
  std::mutex mu;
  HostSlot sl[kSlots];
  cudaStream_t sin = nullptr, sout = nullptr;
  size_t cap = 0;
  bool with_offs = false;
  size_t ob = 0;
};
HostCtx g_host[64];

void free_slots(HostCtx& c) {
  for (auto& x : c.sl) {
    if (x.text) { cudaFree(x.text); cudaFree(x.out); cudaFree(x.status); cudaFree(x.ws); }
    if (x.n_host) cudaFreeHost(x.n_host);
    x.n_host = nullptr;
    x.n_out = nullptr;
    if (x.offs) cudaFree(x.offs);
    x.text = nullptr;
    x.offs = nullptr;
  }
  c.cap = 0;
}

bool alloc_slots(HostCtx& c, size_t bytes, size_t ob, bool offs) {
  free_slots(c);
  for (auto& x : c.sl) {
    const size_t recs = bytes + 1;
    x.ws_bytes = fpp_workspace_bytes_split(bytes);
    if (cudaMalloc(&x.text, bytes + 16) != cudaSuccess || cudaMalloc(&x.out, recs * ob) != cudaSuccess ||
        cudaMalloc(&x.status, recs) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void**>(&x.n_host), 8, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&x.n_out), x.n_host, 0) != cudaSuccess ||
        cudaMalloc(&x.ws, x.ws_bytes) != cudaSuccess)
      return false;
    if (offs && cudaMalloc(&x.offs, recs * 8) != cudaSuccess) return false;
  }
  c.cap = bytes;
  c.ob = ob;
  c.with_offs = offs;
  return true;
}

template <bool F32>
int split_host(const char* host, size_t len, uint32_t sep_mask, uint32_t grammar, int64_t* offs_host,
               int64_t capacity, int64_t* n_out_host, void* out_host, uint8_t* status_host, size_t chunk,
               void* stream) {
  if ((host == nullptr && len > 0) || capacity < 0 || n_out_host == nullptr || sep_mask > 3 ||
      ((out_host == nullptr || status_host == nullptr) && capacity > 0) || !grammar_ok(grammar))
    return FPP_EARG;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return FPP_ECUDA;
  HostCtx& c = g_host[dev];
  std::lock_guard<std::mutex> lock(c.mu);
  const uint32_t seps = sep_mask == 0 ? 3u : sep_mask;
  const size_t ob = F32 ? 4 : 8;
  if (chunk == 0) chunk = (size_t)64 << 20;
  if (chunk > len) chunk = len > 0 ? len : 1;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (c.sin == nullptr) {
    if (cudaStreamCreateWithFlags(&c.sin, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c.sout, cudaStreamNonBlocking) != cudaSuccess)
      return FPP_ECUDA;
    for (auto& x : c.sl)
      if (cudaEventCreateWithFlags(&x.in_done, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&x.parsed, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&x.out_done, cudaEventDisableTiming) != cudaSuccess)
        return FPP_ECUDA;
  }
  cudaStream_t sin = c.sin, sout = c.sout;
  HostSlot* sl = c.sl;
  for (int i = 0; i < kSlots; i++) sl[i].busy = false;
  int rc = FPP_SUCCESS;
  int64_t total = 0;
  auto fail = [&](int code) { if (rc == FPP_SUCCESS) rc = code; };
  // results of a parsed slot to the host (after its count is known)
  auto drain = [&](HostSlot& x) -> bool {
    if (!x.busy) return true;
    if (cudaEventSynchronize(x.parsed) != cudaSuccess) return false;
    // the count was written by the kernels straight into mapped host memory:
    // no copy that could queue behind the next chunk's parse on a legacy stream
    const int64_t n = *reinterpret_cast<volatile int64_t*>(x.n_host);
    if (n < 0) return false;  // internal queue overflow (never expected, k_slow.cuh)
    x.nrec = n;
    const int64_t room = capacity - x.base_rec;
    const int64_t m = room <= 0 ? 0 : (n < room ? n : room);
    if (m > 0) {
      if (cudaMemcpyAsync(static_cast<char*>(out_host) + (size_t)x.base_rec * ob, x.out, (size_t)m * ob,
                          cudaMemcpyDeviceToHost, sout) != cudaSuccess ||
          cudaMemcpyAsync(status_host + x.base_rec, x.status, (size_t)m, cudaMemcpyDeviceToHost, sout) != cudaSuccess)
        return false;
      if (offs_host) {  // chunk-relative starts + the chunk's position in the buffer
        k_add_base<<<(unsigned)((m + 255) / 256), 256, 0, sout>>>(x.offs, m, x.base_byte);
        if (cudaMemcpyAsync(offs_host + x.base_rec, x.offs, (size_t)m * 8, cudaMemcpyDeviceToHost, sout) != cudaSuccess)
          return false;
      }
    }
    if (cudaEventRecord(x.out_done, sout) != cudaSuccess) return false;
    x.busy = false;
    return true;
  };
  size_t start = 0;
  int k = 0, prev = -1;
  while (start < len && rc == FPP_SUCCESS) {
    const size_t end = chunk_end(host, len, start, chunk, seps);
    const size_t nb = end - start;
    if (nb > c.cap || ob > c.ob || (offs_host && !c.with_offs)) {  // (re)allocate after draining
      if (prev >= 0 && !drain(sl[prev])) { fail(FPP_ECUDA); break; }
      if (cudaDeviceSynchronize() != cudaSuccess) { fail(FPP_ECUDA); break; }
      if (!alloc_slots(c, nb > chunk ? nb : chunk, ob > c.ob ? ob : c.ob, offs_host != nullptr || c.with_offs)) {
        free_slots(c);
        fail(FPP_ECUDA);
        break;
      }
    }
    HostSlot& x = sl[k % kSlots];
    if (x.busy && !drain(x)) { fail(FPP_ECUDA); break; }
    // the slot's buffers are free once its previous results have left
    if (cudaStreamWaitEvent(sin, x.out_done, 0) != cudaSuccess ||
        cudaMemcpyAsync(x.text, host + start, nb, cudaMemcpyHostToDevice, sin) != cudaSuccess ||
        cudaEventRecord(x.in_done, sin) != cudaSuccess || cudaStreamWaitEvent(cs, x.in_done, 0) != cudaSuccess) {
      fail(FPP_ECUDA);
      break;
    }
    const int r = split_ws<F32>(x.text, nb, seps, offs_host ? x.offs : nullptr, (int64_t)nb + 1, x.n_out, x.out,
                                x.status, x.ws, x.ws_bytes, nullptr, cs, grammar);
    if (r != FPP_SUCCESS) { fail(r); break; }
    if (cudaEventRecord(x.parsed, cs) != cudaSuccess) { fail(FPP_ECUDA); break; }
    x.busy = true;
    x.base_byte = (int64_t)start;
    // the previous chunk's count gives this chunk's output base: wait for it,
    // one chunk behind (this chunk's copy and parse are already queued)
    if (prev >= 0 && sl[prev].busy && !drain(sl[prev])) { fail(FPP_ECUDA); break; }
    x.base_rec = prev >= 0 ? sl[prev].base_rec + sl[prev].nrec : 0;
    prev = k % kSlots;
    start = end;
    k++;
  }
  if (rc == FPP_SUCCESS && prev >= 0) {
    if (!drain(sl[prev])) fail(FPP_ECUDA);
    total = sl[prev].base_rec + sl[prev].nrec;
  }
  if (cudaStreamSynchronize(sout) != cudaSuccess) fail(FPP_ECUDA);
  if (rc == FPP_SUCCESS) *n_out_host = total;
  return rc;
}

}  // namespace

extern "C" {

int parse_f64_split_ws(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                       int64_t capacity, int64_t* n_out, double* out, uint8_t* status, void* ws,
                       size_t ws_bytes, uint64_t* stats, void* stream) {
  return split_ws<false>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, ws, ws_bytes, stats,
                         stream);
}
int parse_f32_split_ws(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                       int64_t capacity, int64_t* n_out, float* out, uint8_t* status, void* ws,
                       size_t ws_bytes, uint64_t* stats, void* stream) {
  return split_ws<true>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, ws, ws_bytes, stats,
                        stream);
}
int parse_f64_split(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                    int64_t capacity, int64_t* n_out, double* out, uint8_t* status, void* stream) {
  return split_alloc<false>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, stream);
}
int parse_f32_split(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                    int64_t capacity, int64_t* n_out, float* out, uint8_t* status, void* stream) {
  return split_alloc<true>(bytes, len, sep_mask, offsets_out, capacity, n_out, out, status, stream);
}
int parse_f64_batch_ws(const char* bytes, size_t len, const int64_t* offsets, int64_t n, double* out,
                       uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream) {
  return batch_ws<false>(bytes, len, offsets, n, out, status, ws, ws_bytes, stats, stream);
}
int parse_f32_batch_ws(const char* bytes, size_t len, const int64_t* offsets, int64_t n, float* out,
                       uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream) {
  return batch_ws<true>(bytes, len, offsets, n, out, status, ws, ws_bytes, stats, stream);
}
int parse_f64_batch(const char* bytes, size_t len, const int64_t* offsets, int64_t n, double* out,
                    uint8_t* status, void* stream) {
  return batch_alloc<false>(bytes, len, offsets, n, out, status, stream);
}
int parse_f32_batch(const char* bytes, size_t len, const int64_t* offsets, int64_t n, float* out,
                    uint8_t* status, void* stream) {
  return batch_alloc<true>(bytes, len, offsets, n, out, status, stream);
}


int parse_f64_split_ex(const char* bytes, size_t len, uint32_t sep_mask, uint32_t grammar, int64_t* offsets_out,
                       int64_t capacity, int64_t* n_out, double* out, uint8_t* status, void* ws, size_t ws_bytes,
                       uint64_t* stats, void* stream) {
  return split_ex<false>(bytes, len, sep_mask, grammar, offsets_out, capacity, n_out, out, status, ws, ws_bytes,
                         stats, stream);
}
int parse_f32_split_ex(const char* bytes, size_t len, uint32_t sep_mask, uint32_t grammar, int64_t* offsets_out,
                       int64_t capacity, int64_t* n_out, float* out, uint8_t* status, void* ws, size_t ws_bytes,
                       uint64_t* stats, void* stream) {
  return split_ex<true>(bytes, len, sep_mask, grammar, offsets_out, capacity, n_out, out, status, ws, ws_bytes,
                        stats, stream);
}
int parse_f64_batch_ex(const char* bytes, size_t len, const int64_t* offsets, int64_t n, uint32_t grammar,
                       double* out, uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream) {
  return batch_ex<false>(bytes, len, offsets, n, grammar, out, status, ws, ws_bytes, stats, stream);
}
int parse_f32_batch_ex(const char* bytes, size_t len, const int64_t* offsets, int64_t n, uint32_t grammar,
                       float* out, uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream) {
  return batch_ex<true>(bytes, len, offsets, n, grammar, out, status, ws, ws_bytes, stats, stream);
}

int parse_f64_split_host(const char* host_bytes, size_t len, uint32_t sep_mask, uint32_t grammar,
                         int64_t* offsets_out, int64_t capacity, int64_t* n_out, double* out, uint8_t* status,
                         size_t chunk_bytes, void* stream) {
  return split_host<false>(host_bytes, len, sep_mask, grammar, offsets_out, capacity, n_out, out, status,
                           chunk_bytes, stream);
}
int parse_f32_split_host(const char* host_bytes, size_t len, uint32_t sep_mask, uint32_t grammar,
                         int64_t* offsets_out, int64_t capacity, int64_t* n_out, float* out, uint8_t* status,
                         size_t chunk_bytes, void* stream) {
  return split_host<true>(host_bytes, len, sep_mask, grammar, offsets_out, capacity, n_out, out, status,
                          chunk_bytes, stream);
}

void fpp_set_profile_events(void* before_fast, void* after_fast, void* after_slow) {
  g_ev_before_fast.store(reinterpret_cast<cudaEvent_t>(before_fast), std::memory_order_release);
  g_ev_after_fast.store(reinterpret_cast<cudaEvent_t>(after_fast), std::memory_order_release);
  g_ev_after_slow.store(reinterpret_cast<cudaEvent_t>(after_slow), std::memory_order_release);
}

const char* fpp_version(void) {
  return "fpparse-b200 0.1 (sm_100a; Algorithm 1 of arXiv 2101.11408 + exact on-GPU slow path)";
}

}  // extern "C"
