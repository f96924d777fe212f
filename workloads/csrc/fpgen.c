/* Seeded synthetic workloads for configs 1-5 (BASELINE.json "configs") and
 * the paper's two other synthetic datasets (PAPER.md
 * L1024, L1290): 6 "integer" (random 32-bit unsigned integers, %u) and
 * 7 "many digits" (three random 64-bit unsigned integers printed in sequence);
 * and 8: config 2's values printed as C99 hexadecimal floats (grammar option
 * FPP_GRAMMAR_HEX).
 *
 * Input generation only: binary64 -> decimal text.  Holds none of the
 * method's arithmetic (decimal -> binary64).  Shared by the oracle tests and
 * the GPU tests / bench; workloads/gen.py holds a pure-Python twin that must
 * produce identical bytes (tests/test_workloads.py).
 *
 * Randomness: SplitMix64 (public textbook generator).  Record i of a config
 * owns its own stream: state_i = mix(key + (i+1)*GAMMA), key = mix(seed *
 * GAMMA ^ cfg), draws are mix(state_i += GAMMA).  Counter-based, so any
 * thread partition gives the same bytes.
 *
 * Formatting uses glibc snprintf (%.17g, %.17e, %.*f print exact correctly
 * rounded decimals) and, for config 5, exact big-integer (base 1e9) printing of
 * the midpoints between adjacent doubles.  Recipes: DESIGN.md "Inputs".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ull

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;
static inline uint64_t rng_next(rng_t* r) { r->s += GAMMA; return mix64(r->s); }

static inline rng_t rng_record(uint64_t key, uint64_t i) {
  rng_t r; r.s = mix64(key + (i + 1) * GAMMA); return r;
}

static inline double bits_to_double(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }

/* ------------------------------------------------------------------------ */
/* big unsigned integers in base 1e9, little-endian limbs                    */
#define BIG_LIMBS 140
typedef struct { int n; uint32_t l[BIG_LIMBS]; } big_t;

static void big_set_u64(big_t* b, uint64_t v) {
  b->n = 0;
  do { b->l[b->n++] = (uint32_t)(v % 1000000000u); v /= 1000000000u; } while (v);
}
static void big_mul_small(big_t* b, uint32_t m) {
  uint64_t carry = 0;
  for (int i = 0; i < b->n; i++) {
    uint64_t t = (uint64_t)b->l[i] * m + carry;
    b->l[i] = (uint32_t)(t % 1000000000u);
    carry = t / 1000000000u;
  }
  while (carry) { b->l[b->n++] = (uint32_t)(carry % 1000000000u); carry /= 1000000000u; }
}
/* decimal digits, most significant first; returns length */
static int big_to_str(const big_t* b, char* out) {
  int len = sprintf(out, "%u", b->l[b->n - 1]);
  for (int i = b->n - 2; i >= 0; i--) len += sprintf(out + len, "%09u", b->l[i]);
  return len;
}

/* digit string D (no leading zero), value D * 10^q -> "[-]d.ddde+E" with
 * trailing zeros of D folded into q first. */
static int emit_sci(char* dst, int neg, char* D, int len, long q) {
  while (len > 1 && D[len - 1] == '0') { len--; q++; }
  int o = 0;
  if (neg) dst[o++] = '-';
  dst[o++] = D[0];
  if (len > 1) { dst[o++] = '.'; memcpy(dst + o, D + 1, len - 1); o += len - 1; }
  o += sprintf(dst + o, "e%+ld", q + len - 1);
  return o;
}

/* exact midpoint of b (finite, positive pattern) and its successor:
 * (2m+1) * 2^(e-1); digits -> D, returns len, *q = decimal exponent */
static int midpoint_digits(uint64_t bits, char* D, long* q) {
  uint64_t ef = (bits >> 52) & 0x7FF, fr = bits & 0xFFFFFFFFFFFFFull;
  uint64_t m; long e;
  if (ef == 0) { m = fr; e = -1074; } else { m = fr | (1ull << 52); e = (long)ef - 1075; }
  big_t b; big_set_u64(&b, 2 * m + 1);
  long f = e - 1;
  if (f < 0) {
    long k = -f;
    while (k >= 13) { big_mul_small(&b, 1220703125u); k -= 13; }
    uint32_t p = 1; while (k-- > 0) p *= 5;
    if (p > 1) big_mul_small(&b, p);
    *q = f;
  } else {
    long k = f;
    while (k >= 29) { big_mul_small(&b, 1u << 29); k -= 29; }
    if (k > 0) big_mul_small(&b, 1u << k);
    *q = 0;
  }
  return big_to_str(&b, D);
}

/* D +- 1 on a decimal string in place (D has room for one more digit) */
static int dec_add_one(char* D, int len) {
  int i = len - 1;
  while (i >= 0 && D[i] == '9') { D[i] = '0'; i--; }
  if (i >= 0) { D[i]++; return len; }
  memmove(D + 1, D, len); D[0] = '1'; return len + 1;
}
static int dec_sub_one(char* D, int len) {
  int i = len - 1;
  while (i >= 0 && D[i] == '0') { D[i] = '9'; i--; }
  D[i]--;
  int z = 0; while (z < len - 1 && D[z] == '0') z++;
  if (z) { memmove(D, D + z, len - z); len -= z; }
  return len;
}

/* ------------------------------------------------------------------------ */
/* one record: writes text (with its trailing separator) into dst, returns
 * bytes; expected bits/status/known filled where known by construction.     */
typedef struct {
  int cfg; uint64_t key;
} gen_ctx;

static const uint64_t C4_FIXED[8] = {
  0x0000000000000000ull, 0x0000000000000001ull, 0x0000000000000002ull, 0x000FFFFFFFFFFFFFull,
  0x0010000000000000ull, 0x0010000000000001ull, 0x7FEFFFFFFFFFFFFEull, 0x7FEFFFFFFFFFFFFFull};

#define QNAN 0x7FF8000000000000ull
#define PINF 0x7FF0000000000000ull
#define SIGN (1ull << 63)

static int gen_record(const gen_ctx* c, uint64_t i, char* dst, uint64_t* exp_bits,
                      uint8_t* exp_status, uint8_t* known) {
  rng_t r = rng_record(c->key, i);
  *known = 0; *exp_bits = 0; *exp_status = 0;
  if (c->cfg == 1 || c->cfg == 2) {
    uint64_t u = rng_next(&r) >> 11;
    double x = (double)u * 0x1p-53;
    int o = snprintf(dst, 64, "%.17g", x);
    dst[o++] = '\n';
    memcpy(exp_bits, &x, 8); *known = 1;
    return o;
  }
  if (c->cfg == 3) {
    double u = (double)(rng_next(&r) >> 11) * 0x1p-53;
    int s = 6 + (int)(rng_next(&r) % 11);
    double x = (i & 1) ? -90.0 + 180.0 * u : -180.0 + 360.0 * u;
    double ax = fabs(x);
    int prec;
    if (ax >= 1.0) {
      long long ip = (long long)ax; int nd = 0;
      while (ip) { nd++; ip /= 10; }
      prec = s - nd; if (prec < 0) prec = 0;
    } else {
      int lz = 0; double y = ax;
      while (y > 0.0 && y < 0.1 && lz < 30) { y = y * 10.0; lz++; }
      prec = s + lz;
    }
    int o = snprintf(dst, 96, "%.*f", prec, x);
    dst[o++] = (i & 1) ? '\n' : ',';
    return o;
  }
  if (c->cfg == 4) {
    uint64_t bits;
    int o;
    if (i < 16) {
      bits = C4_FIXED[i >> 1] | ((i & 1) ? SIGN : 0);
    } else {
      uint64_t r0 = rng_next(&r);
      if (r0 % 1000 == 0) {
        uint64_t k = rng_next(&r) % 3;
        static const char* sp[3] = {"inf", "-inf", "nan"};
        static const uint64_t sb[3] = {PINF, PINF | SIGN, QNAN};
        o = sprintf(dst, "%s", sp[k]);
        dst[o++] = '\n';
        *exp_bits = sb[k]; *known = 1;
        return o;
      }
      do { bits = rng_next(&r); } while (((bits >> 52) & 0x7FF) == 0x7FF);
    }
    o = snprintf(dst, 64, "%.17e", bits_to_double(bits));
    dst[o++] = '\n';
    *exp_bits = bits; *known = 1;
    return o;
  }
  if (c->cfg == 6) {  /* random 32-bit integers: exact in binary64 */
    uint32_t u = (uint32_t)(rng_next(&r) >> 32);
    int o = sprintf(dst, "%u", u);
    dst[o++] = '\n';
    double x = (double)u;
    memcpy(exp_bits, &x, 8); *known = 1;
    return o;
  }
  if (c->cfg == 8) {  /* uniform [0,1) as "0x1.<13 nibbles, trailing zeros cut>p<exp>" */
    uint64_t u = rng_next(&r) >> 11;
    double x = (double)u * 0x1p-53;
    uint64_t b; memcpy(&b, &x, 8);
    int o;
    if (b == 0) {
      o = sprintf(dst, "0x0p+0");
    } else {
      int e = (int)((b >> 52) & 0x7FF) - 1023;  /* uniform01: always normal */
      uint64_t fr = b & ((1ull << 52) - 1);
      int nn = 13;
      while (nn > 0 && (fr & 15) == 0) { fr >>= 4; nn--; }
      if (nn) o = sprintf(dst, "0x1.%0*llxp%+d", nn, (unsigned long long)fr, e);
      else o = sprintf(dst, "0x1p%+d", e);
    }
    dst[o++] = '\n';
    memcpy(exp_bits, &x, 8); *known = 1;
    return o;
  }
  if (c->cfg == 7) {  /* three random 64-bit integers serialized in sequence (oracle decides) */
    uint64_t a = rng_next(&r), b = rng_next(&r), d = rng_next(&r);
    int o = sprintf(dst, "%llu%llu%llu", (unsigned long long)a, (unsigned long long)b, (unsigned long long)d);
    dst[o++] = '\n';
    return o;
  }
  /* cfg 5 */
  char D[1400];
  uint64_t kind = rng_next(&r) & 3;     /* 0,1: tie; 2: tie +-1; 3: random digits */
  int neg = (int)(rng_next(&r) & 1);
  int o;
  /* records 0-4 are fixed: DBL_MAX tie, DBL_MAX tie+1, 0 tie, 0 tie+1, 0 tie-1 */
  if (i < 5) { neg = 0; kind = (i == 0 || i == 2) ? 0 : (i == 1 || i == 3) ? 2 : 4; }
  if (kind == 3) {
    int nd = 20 + (int)(rng_next(&r) % 21);
    D[0] = (char)('1' + rng_next(&r) % 9);
    for (int j = 1; j < nd; j++) D[j] = (char)('0' + rng_next(&r) % 10);
    long E = -330 + (long)(rng_next(&r) % 641);
    o = emit_sci(dst, neg, D, nd, E - (nd - 1));
    dst[o++] = '\n';
    return o;
  }
  uint64_t bits;
  if (i == 0 || i == 1) bits = 0x7FEFFFFFFFFFFFFFull;      /* DBL_MAX: midpoint 2^1024-2^970 */
  else if (i >= 2 && i < 5) bits = 0;                      /* +0: midpoint 2^-1075 */
  else { do { bits = rng_next(&r) & ~SIGN; } while (((bits >> 52) & 0x7FF) == 0x7FF); }
  long q; int len = midpoint_digits(bits, D, &q);
  uint64_t lo = bits, hi = bits + 1;  /* b, b+ (hi may be +inf) */
  uint64_t sg = neg ? SIGN : 0;
  int up;
  if (kind <= 1) {                        /* exact tie: even one of b, b+ */
    up = (int)(lo & 1);
  } else {
    /* kind 2 / 4: +1 (b+), kind 2 with odd step or special kind 4: -1 (b) */
    int plus = (i < 5) ? (kind == 2) : (int)(rng_next(&r) & 1);
    if (plus) { len = dec_add_one(D, len); up = 1; }
    else { len = dec_sub_one(D, len); up = 0; }
  }
  o = emit_sci(dst, neg, D, len, q);
  dst[o++] = '\n';
  uint64_t res = up ? hi : lo;
  *exp_bits = res | sg; *known = 1;
  *exp_status = (res == PINF) ? 1 : (res == 0) ? 2 : 0;
  return o;
}

/* ------------------------------------------------------------------------ */
typedef struct {
  gen_ctx c; uint64_t i0, i1;
  char* buf; size_t cap, len;
  int64_t* rec_off;  /* relative starts, later made absolute */
  uint64_t* exp_bits; uint8_t* exp_status; uint8_t* known;
} job_t;

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  char tmp[2048];
  for (uint64_t i = j->i0; i < j->i1; i++) {
    uint64_t k = i - j->i0;
    int o = gen_record(&j->c, i, tmp, &j->exp_bits[i], &j->exp_status[i], &j->known[i]);
    if (j->len + (size_t)o > j->cap) {
      size_t nc = j->cap * 2 + 4096;
      j->buf = (char*)realloc(j->buf, nc); j->cap = nc;
    }
    memcpy(j->buf + j->len, tmp, (size_t)o);
    j->rec_off[k] = (int64_t)j->len;
    j->len += (size_t)o;
  }
  return NULL;
}

typedef struct { int nj; job_t* jobs; size_t total; } handle_t;

/* Phase 1: generate n records of config cfg with seed on nthreads threads.
 * offsets / exp_bits / exp_status / known: caller arrays of length n.
 * Returns an opaque handle; *total_len receives the text size. */
void* fpgen_begin(int cfg, uint64_t n, uint64_t seed, int nthreads, int64_t* offsets,
                  uint64_t* exp_bits, uint8_t* exp_status, uint8_t* known, uint64_t* total_len) {
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > n / 1024 + 1) nthreads = (int)(n / 1024 + 1);
  handle_t* h = (handle_t*)calloc(1, sizeof(handle_t));
  h->nj = nthreads;
  h->jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  gen_ctx c; c.cfg = cfg; c.key = mix64(seed * GAMMA ^ (uint64_t)cfg);
  uint64_t per = (n + (uint64_t)nthreads - 1) / (uint64_t)nthreads;
  for (int t = 0; t < nthreads; t++) {
    job_t* j = &h->jobs[t];
    j->c = c; j->i0 = per * (uint64_t)t; j->i1 = j->i0 + per;
    if (j->i0 > n) j->i0 = n;
    if (j->i1 > n) j->i1 = n;
    j->cap = (size_t)(j->i1 - j->i0) * 24 + 4096;
    j->buf = (char*)malloc(j->cap);
    j->rec_off = offsets + j->i0;
    j->exp_bits = exp_bits; j->exp_status = exp_status; j->known = known;
    pthread_create(&th[t], NULL, run_job, j);
  }
  size_t total = 0;
  for (int t = 0; t < nthreads; t++) {
    pthread_join(th[t], NULL);
    job_t* j = &h->jobs[t];
    for (uint64_t k = 0; k < j->i1 - j->i0; k++) j->rec_off[k] += (int64_t)total;
    total += j->len;
  }
  free(th);
  h->total = total;
  *total_len = total;
  return h;
}

typedef struct { job_t* j; char* dst; } copy_t;
static void* run_copy(void* p) { copy_t* c = (copy_t*)p; memcpy(c->dst, c->j->buf, c->j->len); return NULL; }

/* Phase 2: copy the text into dst (total_len bytes) and free the handle. */
void fpgen_finish(void* hp, char* dst) {
  handle_t* h = (handle_t*)hp;
  pthread_t* th = (pthread_t*)calloc((size_t)h->nj, sizeof(pthread_t));
  copy_t* cs = (copy_t*)calloc((size_t)h->nj, sizeof(copy_t));
  size_t pos = 0;
  for (int t = 0; t < h->nj; t++) {
    cs[t].j = &h->jobs[t]; cs[t].dst = dst + pos; pos += h->jobs[t].len;
    pthread_create(&th[t], NULL, run_copy, &cs[t]);
  }
  for (int t = 0; t < h->nj; t++) { pthread_join(th[t], NULL); free(h->jobs[t].buf); }
  free(th); free(cs); free(h->jobs); free(h);
}
