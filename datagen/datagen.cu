// datagen.cu -- seeded synthetic input generators (no PM+ arithmetic here).
// See pmp_datagen.h for the stream contract.
#include "pmp_datagen.h"

#include <cuda_runtime.h>
#include <math.h>

#define HD __host__ __device__ __forceinline__

namespace {

HD uint64_t sm64(uint64_t *s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
HD uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
struct Xo {
  uint64_t s0, s1, s2, s3;
  HD void seed(uint64_t seed, uint64_t id) {
    uint64_t x = seed ^ (id * 0x9E3779B97F4A7C15ULL);
    s0 = sm64(&x); s1 = sm64(&x); s2 = sm64(&x); s3 = sm64(&x);
  }
  HD uint64_t next() {
    uint64_t r = rotl(s1 * 5, 7) * 9;
    uint64_t t = s1 << 17;
    s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = rotl(s3, 45);
    return r;
  }
};

__global__ void k_fill(uint64_t seed, uint8_t *dev, uint64_t nbytes, uint64_t npages, uint64_t page0) {
  uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npages) return;
  Xo g;
  g.seed(seed, 2 + page0 + q);
  uint64_t base = q * PMPD_PAGE;
  uint64_t end = base + PMPD_PAGE < nbytes ? base + PMPD_PAGE : nbytes;
  if (end - base == PMPD_PAGE) {
    ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(dev + base);
#pragma unroll 4
    for (int r = 0; r < (int)(PMPD_PAGE / 16); r++) {
      ulonglong2 v;
      v.x = g.next();
      v.y = g.next();
      dst[r] = v;
    }
  } else {
    for (uint64_t pos = base; pos < end; pos += 8) {
      uint64_t x = g.next();
      for (int k = 0; k < 8 && pos + k < end; k++) dev[pos + k] = (uint8_t)(x >> (8 * k));
    }
  }
}

}  // namespace

extern "C" void pmpd_lengths(int kind, uint64_t seed, uint64_t n, uint64_t lo, uint64_t hi,
                             uint64_t *lengths) {
  Xo g;
  g.seed(seed, 1);
  double lg = hi > 1 ? log2((double)hi) : 0.0;
  for (uint64_t i = 0; i < n; i++) {
    uint64_t x = g.next();
    uint64_t v;
    if (kind == PMPD_LEN_FIXED) {
      v = lo;
    } else if (kind == PMPD_LEN_UNIFORM) {
      v = lo + (uint64_t)(((unsigned __int128)(x >> 32) * (hi - lo + 1)) >> 32);
    } else {
      double u = (double)(x >> 11) * 0x1.0p-53;
      v = (uint64_t)floor(exp2(u * lg));
      if (v < lo) v = lo;
      if (v > hi) v = hi;
    }
    lengths[i] = v;
  }
}

// Raw generator streams, exported so the tests can pin them to published
// reference outputs (tests/golden/prng.txt).
extern "C" void pmpd_splitmix64_stream(uint64_t state, uint64_t n, uint64_t *out) {
  for (uint64_t i = 0; i < n; i++) out[i] = sm64(&state);
}
extern "C" void pmpd_xoshiro256ss_stream(const uint64_t *s, uint64_t n, uint64_t *out) {
  Xo g;
  g.s0 = s[0]; g.s1 = s[1]; g.s2 = s[2]; g.s3 = s[3];
  for (uint64_t i = 0; i < n; i++) out[i] = g.next();
}
extern "C" void pmpd_stream(uint64_t seed, uint64_t id, uint64_t n, uint64_t *out) {
  Xo g;
  g.seed(seed, id);
  for (uint64_t i = 0; i < n; i++) out[i] = g.next();
}

extern "C" uint64_t pmpd_offsets(const uint64_t *lengths, uint64_t n, uint64_t *offsets) {
  uint64_t acc = 0;
  offsets[0] = 0;
  for (uint64_t i = 0; i < n; i++) {
    acc += lengths[i];
    offsets[i + 1] = acc;
  }
  return acc;
}

extern "C" void pmpd_fill_host(uint64_t seed, uint64_t start, uint64_t nbytes, uint8_t *out) {
  uint64_t end = start + nbytes;
  uint64_t pos = start;
  while (pos < end) {
    uint64_t q = pos / PMPD_PAGE;
    Xo g;
    g.seed(seed, 2 + q);
    uint64_t off = pos - q * PMPD_PAGE;
    uint64_t r0 = off / 8;
    for (uint64_t r = 0; r < r0; r++) g.next();
    uint64_t page_end = (q + 1) * PMPD_PAGE < end ? (q + 1) * PMPD_PAGE : end;
    uint64_t wpos = q * PMPD_PAGE + r0 * 8;
    while (wpos < page_end) {
      uint64_t x = g.next();
      for (int k = 0; k < 8; k++) {
        uint64_t b = wpos + (uint64_t)k;
        if (b >= pos && b < page_end) out[b - start] = (uint8_t)(x >> (8 * k));
      }
      wpos += 8;
    }
    pos = page_end;
  }
}

extern "C" int pmpd_fill_device_at(uint64_t seed, uint8_t *dev, uint64_t nbytes, uint64_t page0,
                                   void *stream) {
  if (nbytes == 0) return 0;
  uint64_t npages = (nbytes + PMPD_PAGE - 1) / PMPD_PAGE;
  unsigned threads = 128;
  unsigned blocks = (unsigned)((npages + threads - 1) / threads);
  k_fill<<<blocks, threads, 0, (cudaStream_t)stream>>>(seed, dev, nbytes, npages, page0);
  return (int)cudaGetLastError();
}

extern "C" int pmpd_fill_device(uint64_t seed, uint8_t *dev, uint64_t nbytes, void *stream) {
  return pmpd_fill_device_at(seed, dev, nbytes, 0, stream);
}
