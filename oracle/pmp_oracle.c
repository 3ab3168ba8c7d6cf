/*
 * pmp_oracle.c -- the PM+ oracle.  TEST INFRASTRUCTURE ONLY (see
 * pmp_oracle.h): only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  Shares no code with the
 * CUDA path.
 *
 * Every function transcribes the paper's definition literally:
 *   - Eq. (1): f(s) = (b + sum a_i s_i) mod p, with `% p` after every
 *     product (P:602 allows one modulo per m products; the oracle does not
 *     use that freedom).
 *   - Algorithm 1, with level arrays materialised (the "first level
 *     entirely as a first step" formulation of P:451).
 *   - P:456: bytes -> n-bit words, "pad with a 1-byte and zeros".
 *   - P:585-588: result mod 2^n; the mixing step.
 *
 * Overflow note: with acc < p and t = (a*x) % p < p, acc + t < 2p < 2^66, so
 * no u128 step overflows (a*x <= (2^64-12)(2^64+12) < 2^128 by the kappa
 * constraint, reading Q7).  Adding a*x to acc *before* reducing
 * could exceed 2^128, so the product is reduced first.
 */
#include "pmp_oracle.h"
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static u128 mk(uint64_t lo, uint64_t hi) { return ((u128)hi << 64) | lo; }

int pmpo_params(int bits, uint64_t *p_lo, uint64_t *p_hi, uint64_t *k,
                uint64_t *kappa, uint64_t *a_max) {
  /* Table 2, and Table 1. */
  u128 p;
  uint64_t kk, kap;
  if (bits == 64) {
    kk = 13; kap = 24;
    p = ((u128)1 << 64) + kk;
  } else if (bits == 32) {
    kk = 15; kap = 28;
    p = ((u128)1 << 32) + kk;
  } else {
    return -1;
  }
  if (p_lo) *p_lo = (uint64_t)p;
  if (p_hi) *p_hi = (uint64_t)(p >> 64);
  if (k) *k = kk;
  if (kappa) *kappa = kap;
  /* keys a in (0, p - kappa): largest admissible key is p - kappa - 1. */
  if (a_max) *a_max = (uint64_t)(p - kap - 1);
  return 0;
}

/* ---- key generation (reading Q12) ---- */
static uint64_t splitmix64_next(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
static uint64_t xoshiro_next(uint64_t s[4]) {
  uint64_t result = rotl64(s[1] * 5, 7) * 9;
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

/* The raw generator streams keygen draws from, exported so that tests can pin
 * them to the published reference outputs (tests/golden/prng.txt). */
void pmpo_splitmix64_stream(uint64_t state, uint64_t n, uint64_t *out) {
  for (uint64_t i = 0; i < n; i++) out[i] = splitmix64_next(&state);
}
void pmpo_xoshiro256ss_stream(const uint64_t s_in[4], uint64_t n, uint64_t *out) {
  uint64_t s[4] = {s_in[0], s_in[1], s_in[2], s_in[3]};
  for (uint64_t i = 0; i < n; i++) out[i] = xoshiro_next(s);
}

int pmpo_keygen(uint64_t seed, int bits, uint64_t *b, uint64_t *a) {
  uint64_t a_max;
  if (pmpo_params(bits, NULL, NULL, NULL, NULL, &a_max) != 0) return -1;
  uint64_t sm = seed, st[4];
  for (int i = 0; i < 4; i++) st[i] = splitmix64_next(&sm);
  for (int j = 0; j < PMPO_L; j++) {
    uint64_t x = xoshiro_next(st);
    b[j] = bits == 64 ? x : (x >> 32); /* b in [0, 2^n), reading Q11 */
    for (int i = 0; i < PMPO_M; i++) {
      for (;;) {
        x = xoshiro_next(st);
        if (bits == 32) x >>= 32;
        if (x >= 1 && x <= a_max) break; /* non-zero, < p - kappa */
      }
      a[j * PMPO_M + i] = x;
    }
  }
  return 0;
}

/* ---- mixing step, P:722-734 ---- */
uint64_t pmpo_mix(int bits, uint64_t z) {
  if (bits == 64) {
    z = z ^ (z >> 33);
    z = z * 0xc4ceb9fe1a85ec53ULL;
    z = z ^ (z >> 33);
    return z;
  }
  uint32_t y = (uint32_t)z;
  y = y ^ (y >> 13);
  y = y * 0xab3be54fU;
  y = y ^ (y >> 16);
  return y;
}

/* Inverse, "These transformations are invertible".  x ^= x >> s is
 * undone by repeated xor-shifts; multiplication by an odd constant by its
 * inverse mod 2^n (Newton iteration x <- x(2 - c x)). */
static uint64_t inv_odd64(uint64_t c) {
  uint64_t x = c; /* correct to 3 bits */
  for (int i = 0; i < 6; i++) x *= 2 - c * x;
  return x;
}
static uint64_t unxorshift(uint64_t z, int s, int bits) {
  uint64_t mask = bits == 64 ? ~0ULL : 0xffffffffULL;
  uint64_t x = z & mask;
  for (int i = 0; i < bits / s + 1; i++) x = (z ^ (x >> s)) & mask;
  return x;
}
uint64_t pmpo_unmix(int bits, uint64_t z) {
  if (bits == 64) {
    z = unxorshift(z, 33, 64);
    z = z * inv_odd64(0xc4ceb9fe1a85ec53ULL);
    z = unxorshift(z, 33, 64);
    return z;
  }
  z &= 0xffffffffULL;
  z = unxorshift(z, 16, 32);
  z = (z * inv_odd64(0xab3be54fULL)) & 0xffffffffULL;
  z = unxorshift(z, 13, 32);
  return z;
}

/* ---- bytes -> sigma words, P:456 ---- */
uint64_t pmpo_num_words(int bits, uint64_t len) { return len / (uint64_t)(bits / 8) + 1; }

uint64_t pmpo_sigma_word(int bits, const uint8_t *bytes, uint64_t len, uint64_t t) {
  int w = bits / 8;
  uint64_t v = 0;
  for (int k = 0; k < w; k++) {
    uint64_t pos = t * (uint64_t)w + (uint64_t)k;
    uint64_t byte = pos < len ? bytes[pos] : (pos == len ? 1u : 0u);
    v |= byte << (8 * k); /* little-endian, reading Q3 */
  }
  return v;
}

/* ---- Eq. (1), P:543 ---- */
static u128 block_u128(u128 p, int m, uint64_t b, const uint64_t *a, const u128 *x) {
  u128 acc = (u128)b % p;
  for (int i = 0; i < m; i++) {
    u128 prod = ((u128)a[i] * x[i]) % p; /* x[i] < p, a[i] < p - kappa */
    acc = (acc + prod) % p;
  }
  return acc;
}

void pmpo_block(uint64_t p_lo, uint64_t p_hi, int m, uint64_t b,
                const uint64_t *a, const uint64_t *x_lo, const uint64_t *x_hi,
                uint64_t *out) {
  u128 p = mk(p_lo, p_hi);
  u128 *x = (u128 *)malloc(sizeof(u128) * (size_t)m);
  for (int i = 0; i < m; i++) x[i] = mk(x_lo[i], x_hi ? x_hi[i] : 0);
  u128 r = block_u128(p, m, b, a, x);
  free(x);
  out[0] = (uint64_t)r;
  out[1] = (uint64_t)(r >> 64);
}

/* Algorithm 1 loop (lines 5-9) applied to the array x[0..T),
 * starting at level index j (0-based).  Consumes/replaces x.  Returns the
 * number of levels applied or -1. */
static int alg1_loop(u128 p, int m, int L, int j, const uint64_t *b,
                     const uint64_t *a, u128 **px, uint64_t T, u128 *out) {
  u128 *x = *px;
  int applied = 0;
  while (T > 1) {                  /* while |sigma| > 1 */
    if (j >= L) {                  /* more than L levels: string too long */
      *px = x;
      return -1;
    }
    uint64_t nb = (T + (uint64_t)m - 1) / (uint64_t)m;
    u128 *y = (u128 *)malloc(sizeof(u128) * (size_t)nb);
    u128 *blk = (u128 *)malloc(sizeof(u128) * (size_t)m);
    for (uint64_t q = 0; q < nb; q++) {
      for (int r = 0; r < m; r++) {  /* append zeros to a multiple of m */
        uint64_t idx = q * (uint64_t)m + (uint64_t)r;
        blk[r] = idx < T ? x[idx] : 0;
      }
      y[q] = block_u128(p, m, b[j], a + (size_t)j * (size_t)m, blk);
    }
    free(blk);
    free(x);
    x = y;
    T = nb;
    j++;
    applied++;
  }
  *out = x[0];
  *px = x;
  return applied;
}

int pmpo_tree_generic(uint64_t p_lo, uint64_t p_hi, int m, int L, int j0,
                      const uint64_t *b, const uint64_t *a,
                      const uint64_t *x_lo, const uint64_t *x_hi, uint64_t T,
                      uint64_t *out) {
  u128 p = mk(p_lo, p_hi);
  if (T == 0) return -1;
  u128 *x = (u128 *)malloc(sizeof(u128) * (size_t)T);
  for (uint64_t i = 0; i < T; i++) x[i] = mk(x_lo[i], x_hi ? x_hi[i] : 0);
  u128 r = 0;
  int lv = alg1_loop(p, m, L, j0, b, a, &x, T, &r);
  free(x);
  out[0] = (uint64_t)r;
  out[1] = (uint64_t)(r >> 64);
  return lv;
}

/* ---- production tree over bytes ---- */
typedef struct {
  int bits;
  u128 p;
  const uint64_t *b, *a;
  const uint8_t *bytes;
  uint64_t len, T, c_begin, c_end;
  u128 *y;
} l1_job;

static void *l1_worker(void *arg) {
  l1_job *jb = (l1_job *)arg;
  u128 blk[PMPO_M];
  for (uint64_t c = jb->c_begin; c < jb->c_end; c++) {
    for (int r = 0; r < PMPO_M; r++) {
      uint64_t t = c * PMPO_M + (uint64_t)r;
      blk[r] = t < jb->T ? pmpo_sigma_word(jb->bits, jb->bytes, jb->len, t) : 0;
    }
    jb->y[c] = block_u128(jb->p, PMPO_M, jb->b[0], jb->a, blk);
  }
  return NULL;
}

static int tree_value_u128(int bits, const uint64_t *b, const uint64_t *a,
                           const uint8_t *bytes, uint64_t len, int nthreads,
                           u128 *V) {
  uint64_t plo, phi;
  if (pmpo_params(bits, &plo, &phi, NULL, NULL, NULL) != 0) return -1;
  u128 p = mk(plo, phi);
  uint64_t T = pmpo_num_words(bits, len);
  if (T == 1) { /* Alg. 1 loop never runs: the sole value is sigma_0 (reading Q2) */
    *V = pmpo_sigma_word(bits, bytes, len, 0);
    return 0;
  }
  uint64_t n1 = (T + PMPO_M - 1) / PMPO_M; /* level 1: zero-pad, map f_1 */
  l1_job one;
  memset(&one, 0, sizeof(one));
  one.bits = bits; one.p = p; one.b = b; one.a = a;
  one.bytes = bytes; one.len = len; one.T = T;
  one.c_begin = 0; one.c_end = n1;
  if (n1 == 1) { /* a single level-1 block: its value is the tree value (no heap) */
    u128 y0 = 0;
    one.y = &y0;
    l1_worker(&one);
    *V = y0;
    return 1;
  }
  u128 *y = (u128 *)malloc(sizeof(u128) * (size_t)n1);
  one.y = y;
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > n1) nthreads = (int)n1;
  if (nthreads == 1) {
    l1_worker(&one);
  } else {
    l1_job *jobs = (l1_job *)calloc((size_t)nthreads, sizeof(l1_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; i++) {
      jobs[i] = one;
      jobs[i].c_begin = n1 * (uint64_t)i / (uint64_t)nthreads;
      jobs[i].c_end = n1 * (uint64_t)(i + 1) / (uint64_t)nthreads;
      pthread_create(&th[i], NULL, l1_worker, &jobs[i]);
    }
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    free(jobs);
    free(th);
  }
  int lv = alg1_loop(p, PMPO_M, PMPO_L, 1, b, a, &y, n1, V); /* levels 2.. */
  free(y);
  return lv < 0 ? -1 : lv + 1;
}

int pmpo_tree_value(int bits, const uint64_t *b, const uint64_t *a,
                    const uint8_t *bytes, uint64_t len, int nthreads,
                    uint64_t *out) {
  u128 V = 0;
  int lv = tree_value_u128(bits, b, a, bytes, len, nthreads, &V);
  out[0] = (uint64_t)V;
  out[1] = (uint64_t)(V >> 64);
  return lv;
}

static uint64_t digest_of(int bits, u128 V) {
  /* h(s) mod 2^n, then mix */
  uint64_t z = bits == 64 ? (uint64_t)V : (uint64_t)(V & 0xffffffffu);
  return pmpo_mix(bits, z);
}

uint64_t pmpo_hash(int bits, const uint64_t *b, const uint64_t *a,
                   const uint8_t *bytes, uint64_t len) {
  u128 V = 0;
  tree_value_u128(bits, b, a, bytes, len, 1, &V);
  return digest_of(bits, V);
}

uint64_t pmpo_hash_long(int bits, const uint64_t *b, const uint64_t *a,
                        const uint8_t *bytes, uint64_t len, int nthreads) {
  u128 V = 0;
  tree_value_u128(bits, b, a, bytes, len, nthreads, &V);
  return digest_of(bits, V);
}

typedef struct {
  int bits;
  const uint64_t *b, *a, *offsets;
  const uint8_t *bytes;
  uint64_t i0, i1;
  uint64_t *out;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *jb = (batch_job *)arg;
  for (uint64_t i = jb->i0; i < jb->i1; i++) {
    uint64_t o0 = jb->offsets[i], o1 = jb->offsets[i + 1];
    jb->out[i] = pmpo_hash(jb->bits, jb->b, jb->a, jb->bytes + o0, o1 - o0);
  }
  return NULL;
}

void pmpo_hash_batch(int bits, const uint64_t *b, const uint64_t *a,
                     const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                     uint64_t *out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (n == 0) return;
  if ((uint64_t)nthreads > n) nthreads = (int)n;
  batch_job *jobs = (batch_job *)calloc((size_t)nthreads, sizeof(batch_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; i++) {
    batch_job *jb = &jobs[i];
    jb->bits = bits; jb->b = b; jb->a = a; jb->offsets = offsets;
    jb->bytes = bytes; jb->out = out;
    jb->i0 = n * (uint64_t)i / (uint64_t)nthreads;
    jb->i1 = n * (uint64_t)(i + 1) / (uint64_t)nthreads;
    if (nthreads == 1) batch_worker(jb);
    else pthread_create(&th[i], NULL, batch_worker, jb);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
  free(jobs);
  free(th);
}

/* ---- Two-level variant (reading Q19 in DESIGN.md) ----
 * "only the first level uses Multilinear, while the second level uses a
 * polynomial hash family":
 *   v_c = f_1(chunk c)            c = 0 .. C-1, C = ceil(T / 128) (Eq. (1), as the tree)
 *   h = 0; for c: h = (h + v_c) * r mod p      (Horner: h = sum_c v_c r^(C-c))
 *   V = (h + beta) mod p,  r = a_{2,1}, beta = b_2 (keys of the same schedule)
 *   digest = mix(V mod 2^n).
 * Every string, including T == 1, goes through both levels. */

/* x * y mod p for x, y < p < 2^66: shift-and-add over the bits of y (every
 * intermediate < 2p < 2^67). */
static u128 mulmod_u128(u128 x, u128 y, u128 p) {
  u128 r = 0;
  for (int i = 127; i >= 0; i--) {
    r = (r << 1) % p;
    if ((y >> i) & 1) r = (r + x) % p;
  }
  return r;
}

void pmpo_mulmod(uint64_t p_lo, uint64_t p_hi, uint64_t x_lo, uint64_t x_hi,
                 uint64_t y_lo, uint64_t y_hi, uint64_t *out) {
  u128 r = mulmod_u128(mk(x_lo, x_hi), mk(y_lo, y_hi), mk(p_lo, p_hi));
  out[0] = (uint64_t)r;
  out[1] = (uint64_t)(r >> 64);
}

static int hash2_value_u128(int bits, const uint64_t *b, const uint64_t *a,
                            const uint8_t *bytes, uint64_t len, int nthreads, u128 *V) {
  uint64_t plo, phi;
  if (pmpo_params(bits, &plo, &phi, NULL, NULL, NULL) != 0) return -1;
  u128 p = mk(plo, phi);
  uint64_t T = pmpo_num_words(bits, len);
  uint64_t C = (T + PMPO_M - 1) / PMPO_M; /* chunks, last one zero-padded */
  u128 *y = (u128 *)malloc(sizeof(u128) * (size_t)C);
  if (nthreads < 1) nthreads = 1;
  if ((uint64_t)nthreads > C) nthreads = (int)C;
  l1_job *jobs = (l1_job *)calloc((size_t)nthreads, sizeof(l1_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; i++) {
    l1_job *jb = &jobs[i];
    jb->bits = bits; jb->p = p; jb->b = b; jb->a = a;
    jb->bytes = bytes; jb->len = len; jb->T = T; jb->y = y;
    jb->c_begin = C * (uint64_t)i / (uint64_t)nthreads;
    jb->c_end = C * (uint64_t)(i + 1) / (uint64_t)nthreads;
    if (nthreads == 1) l1_worker(jb);
    else pthread_create(&th[i], NULL, l1_worker, jb);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
  free(jobs);
  free(th);
  const u128 r = a[PMPO_M]; /* a_{2,1} */
  const u128 beta = b[1];   /* b_2 */
  u128 h = 0;
  for (uint64_t c = 0; c < C; c++) h = mulmod_u128((h + y[c]) % p, r, p);
  free(y);
  *V = (h + beta) % p;
  return 0;
}

int pmpo_hash2_value(int bits, const uint64_t *b, const uint64_t *a,
                     const uint8_t *bytes, uint64_t len, int nthreads, uint64_t *out) {
  u128 V = 0;
  int rc = hash2_value_u128(bits, b, a, bytes, len, nthreads, &V);
  out[0] = (uint64_t)V;
  out[1] = (uint64_t)(V >> 64);
  return rc;
}

uint64_t pmpo_hash2(int bits, const uint64_t *b, const uint64_t *a,
                    const uint8_t *bytes, uint64_t len, int nthreads) {
  u128 V = 0;
  hash2_value_u128(bits, b, a, bytes, len, nthreads, &V);
  return digest_of(bits, V);
}

typedef struct {
  int bits;
  const uint64_t *b, *a, *offsets;
  const uint8_t *bytes;
  uint64_t i0, i1;
  uint64_t *out;
} batch2_job;

static void *batch2_worker(void *arg) {
  batch2_job *jb = (batch2_job *)arg;
  for (uint64_t i = jb->i0; i < jb->i1; i++) {
    uint64_t o0 = jb->offsets[i], o1 = jb->offsets[i + 1];
    jb->out[i] = pmpo_hash2(jb->bits, jb->b, jb->a, jb->bytes + o0, o1 - o0, 1);
  }
  return NULL;
}

void pmpo_hash2_batch(int bits, const uint64_t *b, const uint64_t *a,
                      const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                      uint64_t *out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (n == 0) return;
  if ((uint64_t)nthreads > n) nthreads = (int)n;
  batch2_job *jobs = (batch2_job *)calloc((size_t)nthreads, sizeof(batch2_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; i++) {
    batch2_job *jb = &jobs[i];
    jb->bits = bits; jb->b = b; jb->a = a; jb->offsets = offsets;
    jb->bytes = bytes; jb->out = out;
    jb->i0 = n * (uint64_t)i / (uint64_t)nthreads;
    jb->i1 = n * (uint64_t)(i + 1) / (uint64_t)nthreads;
    if (nthreads == 1) batch2_worker(jb);
    else pthread_create(&th[i], NULL, batch2_worker, jb);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
  free(jobs);
  free(th);
}
