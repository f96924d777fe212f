/*
 * fpparse.h -- C ABI of the B200 batched decimal -> binary64 / binary32 parser
 * (arXiv 2101.11408, "Number Parsing at a Gigabyte per Second").
 *
 * Operation (PAPER.md abstract L4-15, Introduction L40-46): every record is an
 * ASCII decimal number; its result is the binary64 value nearest to the
 * decimal, ties to even (notation table), computed with the paper's
 * Algorithm 1 (L223-260) over the 128-bit power-of-five table (Appendix B,
 * L1453-1484), the 19-digit w / w+1 bracket for long significands (L968-983)
 * and an exact fallback (L985-987), all on the GPU.
 *
 * Conventions common to every entry point
 *   - Pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless
 *     the parameter says "host".  The caller owns every buffer; the library
 *     keeps no pointer after returning.  bytes needs no alignment or padding.
 *   - Calls are asynchronous on `stream` (a cudaStream_t passed as void*; NULL
 *     is the legacy default stream).  Results are valid after the caller
 *     synchronizes the stream.  Calls on different streams are independent
 *     provided each uses its own workspace (the *_ws variants).  The plain
 *     variants are the convenience form: they allocate a per-call workspace
 *     with cudaMallocAsync/cudaFreeAsync on `stream` (the stream-ordered pool;
 *     no host synchronisation).  The hot path -- the paper's "no heap
 *     allocation" -- is the *_ws form with a reused workspace,
 *     which is what bench.py times.
 *   - The library is thread-safe: its only global state is per-device
 *     occupancy data initialised once under a lock, and the profiling hook.
 *   - Kernels never wait on work that is not running: the split variant's
 *     tile look-back counts an unpublished predecessor itself after a bounded
 *     wait, so partial residency (other kernels, concurrent calls) cannot
 *     deadlock.
 *   - Nothing at or beyond bytes[len] is read ("The parser must
 *     not access characters outside the string range").
 *   - Per-record problems are data, never call errors: they go to status[i]
 *     (FPP_ST_*).  out[i] then holds the value named below.
 *   - Return value: FPP_SUCCESS, FPP_EARG (bad arguments, nothing enqueued),
 *     FPP_ECUDA (a CUDA call or launch failed), FPP_ECAPACITY (*_ws variants:
 *     ws_bytes smaller than fpp_workspace_bytes_*; nothing enqueued).
 *
 * Record grammar (C locale):
 *     record  := [sign] ( decimal [exp] | special ) terminator*
 *     decimal := digit+ [ '.' digit* ] | '.' digit+
 *     exp     := ('e'|'E') [sign] digit+
 *     special := "inf" | "infinity" | "nan"    (ASCII case-insensitive)
 *     terminator := '\n' | '\r' | ','
 *   No whitespace; any number of digits (values exact).
 *
 * Per-record results
 *   FPP_ST_OK         finite or subnormal value; "inf" -> +-inf; "nan" -> quiet
 *                     NaN 0x7FF8000000000000 (sign bit set for "-nan")
 *   FPP_ST_OVERFLOW   finite decimal that rounds to +-inf; out = +-inf
 *   FPP_ST_UNDERFLOW  nonzero decimal that rounds to +-0; out = +-0
 *   FPP_ST_INVALID    grammar violation or bad record bounds; out = +qNaN
 *   FPP_ST_EMPTY      record of terminator bytes only (or zero length); +qNaN
 */
#ifndef FPPARSE_H_
#define FPPARSE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* per-record status codes (uint8_t status[i]) */
enum { FPP_ST_OK = 0, FPP_ST_OVERFLOW = 1, FPP_ST_UNDERFLOW = 2, FPP_ST_INVALID = 3, FPP_ST_EMPTY = 4 };

/* call return codes */
enum { FPP_SUCCESS = 0, FPP_EARG = 1, FPP_ECUDA = 2, FPP_ECAPACITY = 3 };

/* path counters accumulated into the optional `stats` array (uint64_t[FPP_NSTATS], device) */
enum {
  FPP_STAT_RECORDS = 0,    /* records parsed by the fast kernel                        */
  FPP_STAT_TWO_MULT = 1,   /* Algorithm 1 runs that needed the second multiplication   */
  FPP_STAT_BRACKET = 2,    /* >19 significant digits with a nonzero dropped digit      */
  FPP_STAT_SLOW = 3,       /* records decided by the exact slow path (bracket failed   */
                           /* or Algorithm 1 aborted)          */
  FPP_STAT_ABORT = 4,      /* Algorithm 1 aborts (line 6)                              */
  FPP_STAT_GLOBAL = 5,     /* records read from global memory (beyond the staged tile) */
  FPP_STAT_BAD = 6,        /* INVALID + EMPTY records                                  */
  FPP_STAT_TILES = 7,      /* tiles processed                                          */
  FPP_NSTATS = 8
};

/* Workspace bytes needed by the *_ws variants for an input of `len` bytes and
 * (batch variant) `n` records; n is ignored by the split variant (pass 0).
 * The workspace is scratch (tile descriptors, counters, slow-path queue); it
 * must be 256-byte aligned device memory and not shared by concurrent calls. */
size_t fpp_workspace_bytes_batch(size_t len, int64_t n);
size_t fpp_workspace_bytes_split(size_t len);

/* parse_f64_batch -- records given by their start offsets.
 *   bytes[len]   text (device, any alignment)
 *   offsets[n]   int64 record starts (device); record i is bytes[offsets[i],
 *                end_i) with end_i = offsets[i+1] (i < n-1) or len.  The
 *                number must occupy a prefix of the record; the rest may only
 *                hold terminators, so offsets may include or exclude separators.
 *                A record with start or end outside [0, len] or end < start is
 *                INVALID and is never read.
 *   out[n]       double results (device), status[n] uint8 (device).
 * Errors: FPP_EARG if n < 0, bytes == NULL with len > 0, or offsets/out/status
 * NULL with n > 0. */
int parse_f64_batch(const char* bytes, size_t len, const int64_t* offsets, int64_t n,
                    double* out, uint8_t* status, void* stream);
int parse_f64_batch_ws(const char* bytes, size_t len, const int64_t* offsets, int64_t n,
                       double* out, uint8_t* status, void* ws, size_t ws_bytes,
                       uint64_t* stats, void* stream);

/* parse_f64_split -- the library finds the records itself (record splitter).
 *   sep_mask     separator bytes: bit0 '\n', bit1 ','; 0 means both.  Records
 *                are the maximal segments between separators; an empty segment
 *                is an EMPTY record, except the one after a final trailing
 *                separator, which is no record.  len == 0 gives no record.
 *   offsets_out  nullable; int64 start of each record (device)
 *   capacity     length of out / status / offsets_out
 *   n_out        int64 (device) receives the true record count.  If it
 *                exceeds capacity only the first `capacity` records are
 *                written (snprintf-like); the count is only known once the
 *                stream has run, so callers compare *n_out with capacity after
 *                synchronizing.  A negative *n_out (-FPP_ECAPACITY) reports an
 *                internal slow-path queue overflow, which the queue's sizing
 *                rules out; results are then invalid.
 * Errors: FPP_EARG if bytes == NULL with len > 0, capacity < 0, n_out NULL,
 * out/status NULL with capacity > 0, or sep_mask > 3. */
int parse_f64_split(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                    int64_t capacity, int64_t* n_out, double* out, uint8_t* status, void* stream);
int parse_f64_split_ws(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                       int64_t capacity, int64_t* n_out, double* out, uint8_t* status,
                       void* ws, size_t ws_bytes, uint64_t* stats, void* stream);

/* parse_f32_batch / parse_f32_split -- the same operations with binary32
 * results: every record rounds ONCE, from its exact
 * decimal value, to the nearest binary32, ties to even -- never through
 * binary64 (no double rounding).  Algorithm 1's binary32 column (PAPER.md
 * L223-260: 26 exact bits, 25-bit m, subnormals below 2^-126, ties only for
 * q in [-17, 10] (L287-333), overflow above exponent 127) with the same table,
 * bracket and exact fallback; format facts at L117-121.
 *   out[]        float results (device).  Specials as for binary64 with the
 *                binary32 encodings: +-inf 0x7F800000, quiet NaN 0x7FC00000.
 * Everything else -- arguments, record semantics, status codes, workspace
 * (the same fpp_workspace_bytes_* sizes), errors -- as the binary64 calls. */
int parse_f32_batch(const char* bytes, size_t len, const int64_t* offsets, int64_t n,
                    float* out, uint8_t* status, void* stream);
int parse_f32_batch_ws(const char* bytes, size_t len, const int64_t* offsets, int64_t n,
                       float* out, uint8_t* status, void* ws, size_t ws_bytes,
                       uint64_t* stats, void* stream);
int parse_f32_split(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                    int64_t capacity, int64_t* n_out, float* out, uint8_t* status, void* stream);
int parse_f32_split_ws(const char* bytes, size_t len, uint32_t sep_mask, int64_t* offsets_out,
                       int64_t capacity, int64_t* n_out, float* out, uint8_t* status,
                       void* ws, size_t ws_bytes, uint64_t* stats, void* stream);

/* Grammar options, for the *_ex calls:
 *   FPP_GRAMMAR_DEFAULT  the record grammar above
 *   FPP_GRAMMAR_HEX      also C99 hexadecimal floats:
 *                          [sign] ('0x'|'0X') hexdigit* ['.' hexdigit*] [('p'|'P') [sign] digit+]
 *                        with at least one hex digit; value = hexdigits * 2^(p - 4 * fraction
 *                        nibbles) rounded once to the nearest value, ties to even (H1-H3)
 *   FPP_GRAMMAR_JSON     RFC 8259 numbers only ("+1, 01, 1.e1" are invalid):
 *                          ['-'] ('0' | [1-9] digit*) ['.' digit+] [('e'|'E') [sign] digit+]
 *                        no '+', no specials, no hex; terminators as above.  Anything else
 *                        is FPP_ST_INVALID.
 * HEX and JSON together are FPP_EARG. */
enum { FPP_GRAMMAR_DEFAULT = 0, FPP_GRAMMAR_HEX = 1, FPP_GRAMMAR_JSON = 2 };

/* parse_{f64,f32}_{split,batch}_ex -- the *_ws calls with a grammar option.
 * ws may be NULL: a workspace is then allocated on `stream` (ws_bytes ignored).
 * Errors as the *_ws calls, plus FPP_EARG for an unknown grammar value. */
int parse_f64_split_ex(const char* bytes, size_t len, uint32_t sep_mask, uint32_t grammar,
                       int64_t* offsets_out, int64_t capacity, int64_t* n_out, double* out,
                       uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream);
int parse_f32_split_ex(const char* bytes, size_t len, uint32_t sep_mask, uint32_t grammar,
                       int64_t* offsets_out, int64_t capacity, int64_t* n_out, float* out,
                       uint8_t* status, void* ws, size_t ws_bytes, uint64_t* stats, void* stream);
int parse_f64_batch_ex(const char* bytes, size_t len, const int64_t* offsets, int64_t n,
                       uint32_t grammar, double* out, uint8_t* status, void* ws, size_t ws_bytes,
                       uint64_t* stats, void* stream);
int parse_f32_batch_ex(const char* bytes, size_t len, const int64_t* offsets, int64_t n,
                       uint32_t grammar, float* out, uint8_t* status, void* ws, size_t ws_bytes,
                       uint64_t* stats, void* stream);

/* parse_{f64,f32}_split_host -- parse_*_split_ex on HOST buffers, streamed:
 * the text is cut into chunks of about chunk_bytes (0: 64 MiB) that end right
 * after a separator, and each chunk's host->device copy, parse and
 * device->host copy of results overlap with the neighbouring chunks' (three
 * device slots, copy streams in both directions).  Same records and results
 * as the device call on the whole buffer.
 *   host_bytes, offsets_out (nullable), out, status, n_out: HOST pointers;
 *   page-locked (cudaHostAlloc / cudaHostRegister) memory is needed for the
 *   copies to overlap -- pageable memory works but serialises them.
 *   stream: the parse runs on it; the call returns when all results are in
 *   host memory (synchronous).  The device slots are allocated on first use
 *   and kept per device; concurrent host calls on one device run one after
 *   the other.
 * Errors: as parse_*_split_ex; FPP_ECUDA if device memory for the slots
 * (about 3 x (chunk x 10 B)) cannot be allocated. */
int parse_f64_split_host(const char* host_bytes, size_t len, uint32_t sep_mask, uint32_t grammar,
                         int64_t* offsets_out, int64_t capacity, int64_t* n_out, double* out,
                         uint8_t* status, size_t chunk_bytes, void* stream);
int parse_f32_split_host(const char* host_bytes, size_t len, uint32_t sep_mask, uint32_t grammar,
                         int64_t* offsets_out, int64_t capacity, int64_t* n_out, float* out,
                         uint8_t* status, size_t chunk_bytes, void* stream);

/* Profiling hook (not thread safe; used by bench.py): when non-NULL, the
 * cudaEvent_t handles are recorded on the call's stream immediately before and
 * after the fast kernel (k_split / k_batch) and after the slow kernel, so the
 * dominant kernel's duration can be timed live with CUDA events on its own
 * stream.  Pass NULLs to disable. */
void fpp_set_profile_events(void* before_fast, void* after_fast, void* after_slow);

/* Human-readable library / build description (static string). */
const char* fpp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FPPARSE_H_ */
