// pmp_kernels.cuh -- PM+ hot-path kernels for sm_100a.
//
// Layout of the work:
//   k_short   thread per string for strings <= kShortMax bytes (one level-1
//             block, T <= 16 / 32 words).  A warp stages the contiguous byte
//             span of its 32 strings into shared memory with coalesced 16-byte
//             loads, then each lane walks its own string.  Strings longer than
//             kShortMax are appended to a work list for k_wstring.
//   k_wstring warp per string (from the work list): chunk-parallel level 1 with
//             8 lanes per chunk, fused level 2, streaming upper levels.
//   k_node    warp per level-2 node of one long string (pmp_hash_long*):
//             partial level-2 sums s2 = sum_r a_{2,r} v1 over the caller's chunks.
//   k_level   warp per node of level j >= 3 over partial sums.
//   k_combine sums the rank partials + the key-only constant, finalises.
//
// Citations: P:n = PAPER.md line n.  Eq. (1); Algorithm 1 P:427-443;
// byte packing P:456; reduction P:659-709; finaliser P:722-734.
#pragma once
#include <stdint.h>
#include "pmp_arith.cuh"

namespace pmp {

constexpr uint32_t kShortMax = 127;      // bytes; k_short handles B <= kShortMax
constexpr uint32_t kBigBytes = 1u << 16; // work-list class "big" (processed first)
#ifndef PMP_SHORT_WARPS
#define PMP_SHORT_WARPS 16
#endif
#ifndef PMP_SHORT_RING_KB
#define PMP_SHORT_RING_KB 64
#endif
constexpr int kShortWarps = PMP_SHORT_WARPS;  // consumer warps per k_short block (+1 producer)
constexpr int kWWarps = 4;               // warps per k_wstring / k_node block
constexpr uint32_t FULL = 0xffffffffu;
// k_short word-loop granularity (words between warp-uniform exit tests)
#ifndef PMP_SHORT_G64
#define PMP_SHORT_G64 4
#endif
#ifndef PMP_SHORT_G32
#define PMP_SHORT_G32 8
#endif
constexpr int kShortG64 = PMP_SHORT_G64, kShortG32 = PMP_SHORT_G32;

// level-1 keys 0..31 and b_1 passed by value: they live in the constant bank
// and become immediate operands of the multiply-adds in k_short.
struct ParamKeys {
  uint64_t a[32];
  uint64_t b;
  uint64_t r, b2;  // two-level variant (reading Q19): r = a_{2,1}, b_2
  // dual-width k_short: the 32-bit schedule's a_{1,0..31} and b_1 (a, b hold the 64-bit one)
  uint32_t a32[32];
  uint64_t b32;
  uint64_t r32, b2_32;  // and its two-level r = a_{2,1}, b_2
};

// ------------------------------------------------------------- helpers
PMP_DI uint4 ld_stream16(const void *p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
PMP_DI uint32_t ld_u32(const void *p) {
  uint32_t r;
  asm("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
PMP_DI uint32_t funnel(uint32_t lo, uint32_t hi, uint32_t sh) { return __funnelshift_r(lo, hi, sh); }
PMP_DI uint32_t lds_u32(uint32_t saddr) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(saddr));
  return r;
}

// ------------------------------------------------------------- width traits
template <int BITS> struct Tr;
template <> struct Tr<64> {
  using Acc = Acc5;
  using Fe = Fe64;
  using Key = uint64_t;
  static constexpr int W = 8;            // bytes per word
  static constexpr int CHUNK = 1024;     // bytes per level-1 block (128 words)
  static constexpr int CPG = 1;          // chunks per 1 KiB group block
};
template <> struct Tr<32> {
  using Acc = Acc3;
  using Fe = uint64_t;
  using Key = uint32_t;
  static constexpr int W = 4;
  static constexpr int CHUNK = 512;
  static constexpr int CPG = 2;
};

PMP_DI void acc_zero(Acc5 &x) { x.c0 = x.c1 = x.c2 = x.c3 = x.c4 = 0; }
PMP_DI void acc_zero(Acc3 &x) { x.c0 = x.c1 = x.c2 = 0; }
PMP_DI void acc_add(Acc5 &x, const Acc5 &y) { acc5_add(x, y); }
PMP_DI void acc_add(Acc3 &x, const Acc3 &y) { acc3_add(x, y); }
PMP_DI void acc_add_word(Acc5 &x, uint64_t v) { acc5_add_u64(x, v); }
PMP_DI void acc_add_word(Acc3 &x, uint64_t v) { acc3_add_u64(x, v); }
PMP_DI void acc_mac_fe(Acc5 &x, uint64_t a, const Fe64 &v) { acc5_mac_fe(x, a, v); }
PMP_DI void acc_mac_fe(Acc3 &x, uint64_t a, uint64_t v) { acc3_mac_fe(x, (uint32_t)a, v); }
PMP_DI void acc_add_fe(Acc5 &x, const Fe64 &v) {  // x += v (field element, < 2^65)
  acc5_add_u64(x, v.lo);
  Acc5 h = {0, 0, v.hi, 0, 0};
  acc5_add(x, h);
}
PMP_DI void acc_add_fe(Acc3 &x, uint64_t v) { acc3_add_u64(x, v); }
PMP_DI Acc5 acc_shfl_xor(const Acc5 &x, int m) { return acc5_shfl_xor(x, m); }
PMP_DI Acc3 acc_shfl_xor(const Acc3 &x, int m) { return acc3_shfl_xor(x, m); }
PMP_DI Fe64 acc_reduce(const Acc5 &x) { return reduce_acc5(x); }
PMP_DI uint64_t acc_reduce(const Acc3 &x) { return reduce_acc3(x); }
PMP_DI uint64_t acc_reduce_lo(const Acc5 &x) { return reduce_lo_acc5(x); }  // V mod 2^n only
PMP_DI uint64_t acc_reduce_lo(const Acc3 &x) { return reduce_lo_acc3(x); }
PMP_DI uint64_t fe_lo(const Fe64 &v) { return v.lo; }
PMP_DI uint64_t fe_lo(uint64_t v) { return (uint32_t)v; }
PMP_DI void fe_store(uint64_t *dst, const Fe64 &v) { dst[0] = v.lo; dst[1] = v.hi; }
PMP_DI void fe_store(uint64_t *dst, uint64_t v) { dst[0] = v; dst[1] = 0; }
PMP_DI void fe_load(const uint64_t *src, Fe64 &v) { v.lo = src[0]; v.hi = (uint32_t)src[1]; }
PMP_DI void fe_load(const uint64_t *src, uint64_t &v) { v = src[0]; }
// L2-coherent loads of values another block of the same launch just wrote
PMP_DI void fe_load_cg(const uint64_t *src, Fe64 &v) { v.lo = __ldcg(src); v.hi = (uint32_t)__ldcg(src + 1); }
PMP_DI void fe_load_cg(const uint64_t *src, uint64_t &v) { v = __ldcg(src); }
PMP_DI Fe64 fe_shfl(const Fe64 &v, int lane) {
  Fe64 r;
  r.lo = __shfl_sync(FULL, v.lo, lane);
  r.hi = __shfl_sync(FULL, v.hi, lane);
  return r;
}
PMP_DI uint64_t fe_shfl(uint64_t v, int lane) { return __shfl_sync(FULL, v, lane); }
PMP_DI Fe64 fe_from_word(uint64_t w, Fe64 *) { Fe64 r; r.lo = w; r.hi = 0; return r; }
PMP_DI uint64_t fe_from_word(uint64_t w, uint64_t *) { return w; }
PMP_DI uint32_t fe_hi(const Fe64 &v) { return v.hi; }
PMP_DI uint32_t fe_hi(uint64_t v) { return (uint32_t)(v >> 32); }
// x += v * 2^n (field element v; exact, the accumulators have headroom)
PMP_DI void acc_add_fe_shl(Acc5 &x, const Fe64 &v) {
  Acc5 h = {0, 0, (uint32_t)v.lo, (uint32_t)(v.lo >> 32), v.hi};
  acc5_add(x, h);
}
PMP_DI void acc_add_fe_shl(Acc3 &x, uint64_t v) {
  Acc3 h = {0, (uint32_t)v, (uint32_t)(v >> 32)};
  acc3_add(x, h);
}
// x += w * v for two field elements: (w mod 2^n) * v + [w >= 2^n] v 2^n (< 2^(2n+2))
PMP_DI void acc_mac_fe_full(Acc5 &x, const Fe64 &w, const Fe64 &v) {
  acc5_mac_fe(x, w.lo, v);
  if (w.hi) acc_add_fe_shl(x, v);
}
PMP_DI void acc_mac_fe_full(Acc3 &x, uint64_t w, uint64_t v) {
  acc3_mac_fe(x, (uint32_t)w, v);
  if (w >> 32) acc_add_fe_shl(x, v);
}
// w * v mod p (P:659-709 reduction of the exact product)
template <class Fe> PMP_DI Fe fe_mul(const Fe &w, const Fe &v) {
  if constexpr (sizeof(Fe) == 8) {
    Acc3 x = {0, 0, 0};
    acc_mac_fe_full(x, w, v);
    return reduce_acc3(x);
  } else {
    Acc5 x = {0, 0, 0, 0, 0};
    acc_mac_fe_full(x, w, v);
    return reduce_acc5(x);
  }
}

PMP_DI void load_acc(const uint32_t *w, Acc5 &x) { x.c0 = w[0]; x.c1 = w[1]; x.c2 = w[2]; x.c3 = w[3]; x.c4 = w[4]; }
PMP_DI void load_acc(const uint32_t *w, Acc3 &x) { x.c0 = w[0]; x.c1 = w[1]; x.c2 = w[2]; }
PMP_DI void store_acc(uint32_t *w, const Acc5 &x) { w[0] = x.c0; w[1] = x.c1; w[2] = x.c2; w[3] = x.c3; w[4] = x.c4; }
PMP_DI void store_acc(uint32_t *w, const Acc3 &x) { w[0] = x.c0; w[1] = x.c1; w[2] = x.c2; }
// chunk sum -> a_2-weighted contribution without Algorithm 2 (acc5/acc3_mac_v01)
PMP_DI void acc_mac_partial(Acc5 &acc, uint64_t a, const Acc5 &x) {
  uint64_t v0;
  uint32_t v1;
  reduce3to2_64(((uint64_t)x.c1 << 32) | x.c0, ((uint64_t)x.c3 << 32) | x.c2, x.c4, v0, v1);
  acc5_mac_v01(acc, a, v0, v1);
}
PMP_DI void acc_mac_partial(Acc3 &acc, uint64_t a, const Acc3 &x) {
  uint32_t v0, v1;
  reduce3to2_32(x.c0, x.c1, x.c2, v0, v1);
  acc3_mac_v01(acc, (uint32_t)a, v0, v1);
}
// the same for a field-element weight w (< p, the extra bit included):
// w (v0 + v1 2^n) = w_lo (v0 + v1 2^n) + [w >= 2^n] (v0 + v1 2^n) 2^n
PMP_DI void acc_mac_partial_fe(Acc5 &acc, const Fe64 &w, const Acc5 &x) {
  uint64_t v0;
  uint32_t v1;
  reduce3to2_64(((uint64_t)x.c1 << 32) | x.c0, ((uint64_t)x.c3 << 32) | x.c2, x.c4, v0, v1);
  acc5_mac_v01(acc, w.lo, v0, v1);
  if (w.hi) {
    const Acc5 h = {0, 0, (uint32_t)v0, (uint32_t)(v0 >> 32), v1};
    acc5_add(acc, h);
  }
}
PMP_DI void acc_mac_partial_fe(Acc3 &acc, uint64_t w, const Acc3 &x) {
  uint32_t v0, v1;
  reduce3to2_32(x.c0, x.c1, x.c2, v0, v1);
  acc3_mac_v01(acc, (uint32_t)w, v0, v1);
  if (w >> 32) {
    const Acc3 h = {0, v0, v1};
    acc3_add(acc, h);
  }
}
// levels of Algorithm 1 applied to T words: 0 if T == 1, else ceil(log_128 T)
PMP_HDI int levels_of(uint64_t T) {
  return (T > 1) + (T > (1ULL << 7)) + (T > (1ULL << 14)) + (T > (1ULL << 21)) + (T > (1ULL << 28)) +
         (T > (1ULL << 35)) + (T > (1ULL << 42)) + (T > (1ULL << 49));
}

// Where a batch digest goes: the digest itself (M == 0), or -- the hash-table
// consumer of SURVEY 8(f3) -- its bucket digest mod M (h mod M
// stays almost Delta-universal; it is 2-regular, regular when M | 2^n),
// optionally counted into a device histogram.
struct OutSpec {
  void *out;        // n digests (uint64/uint32) or n uint32 buckets
  uint32_t M;       // 0: digests
  uint32_t *counts; // M counters (atomically incremented) or nullptr
};

template <int BITS> PMP_DI void store_digest(void *out, uint64_t i, uint64_t lo);
template <> PMP_DI void store_digest<64>(void *out, uint64_t i, uint64_t lo) {
  reinterpret_cast<uint64_t *>(out)[i] = mix64(lo);
}
template <> PMP_DI void store_digest<32>(void *out, uint64_t i, uint64_t lo) {
  reinterpret_cast<uint32_t *>(out)[i] = mix32((uint32_t)lo);
}
template <int BITS> PMP_DI void emit(const OutSpec &os, uint64_t i, uint64_t lo) {
  if (os.M == 0) {
    store_digest<BITS>(os.out, i, lo);
    return;
  }
  const uint64_t d = BITS == 64 ? mix64(lo) : (uint64_t)mix32((uint32_t)lo);
  const uint32_t b = (uint32_t)(d % os.M);
  reinterpret_cast<uint32_t *>(os.out)[i] = b;
  if (os.counts) atomicAdd(&os.counts[b], 1u);
}

// ============================================================= k_short
// One short string (B <= kShortMax, so T = floor(B/w)+1 <= 16 / 32 words and
// the tree is a single f_1 block, or no block at all when T == 1).
// fetch(k) returns the k-th aligned 32-bit word of the region starting at the
// word containing the string's first byte; `sh` is that byte's bit offset.
// The loop runs to the warp's largest number of full words; a lane past its
// own full words multiplies zeros (a*0 adds nothing), so the multiply-adds are
// never branched around.  The marker word is done once per lane with
// its key read from shared memory.
// V2: the two-level variant (reading Q19): V = b_2 + r * v_0 with v_0 = f_1 of
// the single chunk (no |sigma| = 1 shortcut).
template <int BITS, bool V2, class Fetch>
PMP_DI uint64_t short_tree_lo(const ParamKeys &K, const uint64_t *__restrict__ skeys, uint32_t B, uint32_t sh,
                              int tfull_max, Fetch fetch) {
  if constexpr (BITS == 64) {
    const int tlast = (int)(B >> 3);
    const uint32_t r = B & 7;
    MacAcc64 A;
    macc_zero(A);
    uint32_t y0 = fetch(0);
#pragma unroll
    for (int tb = 0; tb < 16; tb += kShortG64) {
      if (tb >= tfull_max) break;                              // warp-uniform, once per kShortG64 words
#pragma unroll
      for (int j = 0; j < kShortG64; j++) {
        const int t = tb + j;
        if (t >= 15) break;                                    // compile-time
        const uint32_t y1 = fetch(2 * t + 1), y2 = fetch(2 * t + 2);
        uint32_t lo = funnel(y0, y1, sh), hi = funnel(y1, y2, sh);
        y0 = y2;
        if ((uint32_t)t >= (uint32_t)tlast) lo = hi = 0;       // past this lane's full words
        mac64(A, (uint32_t)K.a[t], (uint32_t)(K.a[t] >> 32), lo, hi);  // Eq. (1), lazy
      }
    }
    const uint32_t z0 = fetch(2 * tlast), z1 = fetch(2 * tlast + 1), z2 = fetch(2 * tlast + 2);
    const uint32_t zl = funnel(z0, z1, sh), zh = funnel(z1, z2, sh);
    // bytes || 0x01 || 0: mask the half holding byte r, keep / drop the other
    const uint32_t mb = 1u << (8 * (r & 3)), wh = (((r & 4) ? zh : zl) & (mb - 1)) | mb;
    const uint64_t w = (r & 4) ? ((uint64_t)wh << 32) | zl : (uint64_t)wh;
    if (!V2 && tlast == 0) return w;                           // |sigma| = 1: no f_j (reading Q2)
    mac64(A, skeys[tlast], w);
    Acc5 x = macc_normalize(A);
    acc5_add_u64(x, K.b);
    if constexpr (V2) {
      const Fe64 v0 = reduce_acc5(x);
      Acc5 y = {0, 0, 0, 0, 0};
      acc5_mac_fe(y, K.r, v0);
      acc5_add_u64(y, K.b2);
      return reduce_lo_acc5(y);
    }
    return reduce_lo_acc5(x);                                  // mod p, then mod 2^64
  } else {
    const int tlast = (int)(B >> 2);
    const uint32_t r = B & 3;
    Acc3 A = {0, 0, 0};
    uint32_t y0 = fetch(0);
#pragma unroll
    for (int tb = 0; tb < 32; tb += kShortG32) {
      if (tb >= tfull_max) break;                              // warp-uniform, once per kShortG32 words
#pragma unroll
      for (int j = 0; j < kShortG32; j++) {
        const int t = tb + j;
        if (t >= 31) break;
        const uint32_t y1 = fetch(t + 1);
        uint32_t w = funnel(y0, y1, sh);
        y0 = y1;
        if ((uint32_t)t >= (uint32_t)tlast) w = 0;
        mac32(A, (uint32_t)K.a[t], w);
      }
    }
    const uint32_t z0 = fetch(tlast), z1 = fetch(tlast + 1);
    uint32_t w = funnel(z0, z1, sh);
    w = (w & ((1u << (8 * r)) - 1)) | (1u << (8 * r));
    if (!V2 && tlast == 0) return w;
    mac32(A, (uint32_t)skeys[tlast], w);
    acc3_add_u64(A, K.b);
    if constexpr (V2) {
      const uint64_t v0 = reduce_acc3(A);
      Acc3 y = {0, 0, 0};
      acc3_mac_fe(y, (uint32_t)K.r, v0);
      acc3_add_u64(y, K.b2);
      return reduce_lo_acc3(y);
    }
    return reduce_lo_acc3(A);
  }
}

// Both digests of one short string in one pass (a 64-bit and a 32-bit key
// schedule: the two configs[1] outputs).  The 32-bit words of PM+32 are the
// halves of the 64-bit words of PM+64, so the loads, funnel shifts, masks and
// the loop over the full 64-bit words (warp maximum tfull_max) are shared;
// each width keeps its own marker word, exact sum and reduction.
// V2: the two-level variant (reading Q19) for both schedules: V = b_2 + r v_0,
// every string (no |sigma| = 1 shortcut).
template <bool V2, class Fetch>
PMP_DI void short_tree_dual(const ParamKeys &K, const uint64_t *__restrict__ skeys, const uint32_t *__restrict__ skeys32,
                            uint32_t B, uint32_t sh, int tfull_max, Fetch fetch, uint64_t &lo64, uint32_t &lo32) {
  const int tl64 = (int)(B >> 3), tl32 = (int)(B >> 2);
  MacAcc64 A;
  macc_zero(A);
  Acc3 C = {0, 0, 0};
  uint32_t y0 = fetch(0);
#pragma unroll
  for (int tb = 0; tb < 16; tb += kShortG64) {
    if (tb >= tfull_max) break;                              // warp-uniform
#pragma unroll
    for (int j = 0; j < kShortG64; j++) {
      const int t = tb + j;
      if (t >= 16) break;                                    // compile-time
      const uint32_t y1 = fetch(2 * t + 1), y2 = fetch(2 * t + 2);
      const uint32_t lo = funnel(y0, y1, sh), hi = funnel(y1, y2, sh);
      y0 = y2;
      // both halves of a full 64-bit word are full PM+32 words; the one PM+32
      // word beyond them (the low half at t = tl64 when B mod 8 >= 4) is added
      // with the markers below
      const bool f64 = t < tl64;
      const uint32_t lm = f64 ? lo : 0u, hm = f64 ? hi : 0u;
      if (t < 15) {
        mac64(A, (uint32_t)K.a[t], (uint32_t)(K.a[t] >> 32), lm, hm);  // Eq. (1)
        mac32(C, K.a32[2 * t], lm);
        mac32(C, K.a32[2 * t + 1], hm);
      }
    }
  }
  // marker words: the 8 bytes at 8 tl64, and its half holding byte 4 tl32
  const uint32_t z0 = fetch(2 * tl64), z1 = fetch(2 * tl64 + 1), z2 = fetch(2 * tl64 + 2);
  const uint32_t zl = funnel(z0, z1, sh), zh = funnel(z1, z2, sh);
  // the partial 32-bit word is the PM+32 marker word, and a half of the PM+64 one
  const bool up = (B & 4) != 0;                              // B mod 8 >= 4
  const uint32_t mb = 1u << (8 * (B & 3));
  const uint32_t w32 = ((up ? zh : zl) & (mb - 1)) | mb;
  const uint64_t w = up ? ((uint64_t)w32 << 32) | zl : (uint64_t)w32;
  if (up) mac32(C, skeys32[2 * tl64], zl);                   // the full PM+32 word 2 tl64
  if (!V2 && tl64 == 0) {
    lo64 = w;                                                // |sigma| = 1 (reading Q2)
  } else {
    mac64(A, skeys[tl64], w);
    Acc5 x = macc_normalize(A);
    acc5_add_u64(x, K.b);
    if constexpr (V2) {
      const Fe64 v0 = reduce_acc5(x);
      Acc5 y = {0, 0, 0, 0, 0};
      acc5_mac_fe(y, K.r, v0);
      acc5_add_u64(y, K.b2);
      lo64 = reduce_lo_acc5(y);
    } else {
      lo64 = reduce_lo_acc5(x);
    }
  }
  if (!V2 && tl32 == 0) {
    lo32 = w32;
  } else {
    mac32(C, skeys32[tl32], w32);
    acc3_add_u64(C, K.b32);
    if constexpr (V2) {
      const uint64_t v0 = reduce_acc3(C);
      Acc3 y = {0, 0, 0};
      acc3_mac_fe(y, (uint32_t)K.r32, v0);
      acc3_add_u64(y, K.b2_32);
      lo32 = reduce_lo_acc3(y);
    } else {
      lo32 = reduce_lo_acc3(C);
    }
  }
}

// ---- TMA bulk-copy / mbarrier helpers (cp.async.bulk -> UBLKCP in SASS)
PMP_DI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
PMP_DI void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
PMP_DI void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
}
PMP_DI void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
PMP_DI void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
PMP_DI void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "PMP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra PMP_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// (PMP_WAIT_HINT_NS > 0: try_wait with a suspend-time hint, so a waiting warp
// sleeps until the phase completes instead of re-issuing the probe)
#ifndef PMP_WAIT_HINT_NS
#define PMP_WAIT_HINT_NS 0
#endif
PMP_DI void mbar_wait_s(uint32_t bar_s, uint32_t parity) {
#if PMP_WAIT_HINT_NS
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "PMP_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
      "@!P bra PMP_WAITS_%=;\n}" ::"r"(bar_s),
      "r"(parity), "r"((uint32_t)PMP_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "PMP_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra PMP_WAITS_%=;\n}" ::"r"(bar_s),
      "r"(parity)
      : "memory");
#endif
}
PMP_DI void mbar_arrive_s(uint32_t bar_s) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_s) : "memory");
}
PMP_DI void lds_u32x2(uint32_t a, uint32_t &x, uint32_t &y) {  // 8-byte aligned
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
}
PMP_DI void lds_u64x2(uint32_t a, uint64_t &x, uint64_t &y) {  // two consecutive u64 (8-byte aligned)
  asm volatile("ld.shared.u64 %0, [%2];\n\tld.shared.u64 %1, [%2+8];" : "=l"(x), "=l"(y) : "r"(a));
}
PMP_DI void lds_hdr(uint32_t a, uint64_t &alo, uint32_t &pos, uint32_t &mode) {  // 16-byte TileHdr
  uint32_t x, y;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(pos), "=r"(mode) : "r"(a));
  alo = ((uint64_t)y << 32) | x;
}
PMP_DI uint32_t atoms_add(uint32_t a, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
  return r;
}
PMP_DI void sts_u32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
PMP_DI void sts_u16(uint32_t a, uint16_t v) { asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory"); }
PMP_DI uint32_t lds_u16(uint32_t a) {
  uint16_t r;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(a) : "memory");
  return r;
}
// named barrier among the consumer warps only (id 0 is __syncthreads)
PMP_DI void named_bar_sync(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }
PMP_DI void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// k_short: warp-specialised TMA pipeline.  A block = 1 producer warp + kShortWarps
// consumer warps, working on tiles of kTile = 32 * kShortWarps consecutive
// strings (grid-strided).  Shared memory holds
//   - an offsets ring (kRing slots): the kTile+1 offsets of tile k, one TMA bulk
//     copy issued kOffAhead tiles ahead;
//   - a byte ring (kByteRing bytes): the 16-byte aligned contiguous byte span of
//     each staged tile, one TMA bulk copy, packed back to back so the number of
//     tiles in flight adapts to the string lengths;
//   - a header per tile.
// The producer's work per tile is O(1) (the span is [offsets[first],
// offsets[last+1])), so one producer warp keeps many consumer warps fed.  A
// tile whose span exceeds kSpanMaxTile is "direct": consumers read its short
// strings from global.  Strings longer than kShortMax are appended by the
// consumers to the work list of k_wstring in either mode.
constexpr int kPasses = 1;                                     // strings per consumer lane per tile
constexpr int kTile = 32 * kShortWarps * kPasses;              // 384
#ifndef PMP_SHORT_SLOTS
#define PMP_SHORT_SLOTS 8
#endif
constexpr int kRing = PMP_SHORT_SLOTS, kOffAhead = PMP_SHORT_SLOTS / 2;  // tile slots (power of 2), offsets prefetch
constexpr uint32_t kByteRing = PMP_SHORT_RING_KB * 1024;
// Block-wide counting sort of each tile by word count before hashing
// (PMP_SHORT_SORT=1): removes most of the zero-padding multiply-adds but costs
// two named barriers per tile; measured 4-10% slower on configs[1]
// (profiles/r01_summary.md), so it is off.
#ifndef PMP_SHORT_SORT
#define PMP_SHORT_SORT 0
#endif
constexpr uint32_t kSpanMaxTile = kByteRing / 2 < 32 * 1024 ? kByteRing / 2 : 32 * 1024;  // larger spans go direct
constexpr int kOffBytes = ((kTile + 1) * 8 + 15) & ~15;        // 3088
constexpr int kSlack = 144;                                    // fetch() reads <= 136 B past a start
struct TileHdr {
  uint64_t alo;    // global address of staged byte 0
  uint32_t pos;    // ring position of staged byte 0
  uint32_t mode;   // 0 staged, 1 direct
};
constexpr size_t kShortSmem = 384 /* keys */ + kByteRing + kSlack + 16 + (size_t)kRing * kOffBytes +
                              (size_t)kRing * sizeof(TileHdr) +
                              (size_t)(3 * kRing) * 8 + (PMP_SHORT_SORT ? 256 /* sort histograms */ + 2 * kTile /* permutation */ : 0) + 128;

// DUAL: BITS = 64 and a second, 32-bit schedule in K.a32 / K.b32 whose digests go to os2
template <int BITS, bool V2 = false, bool DUAL = false>
__global__ void __launch_bounds__((kShortWarps + 1) * 32)
k_short(const ParamKeys K, const uint8_t *__restrict__ bytes, const uint64_t *__restrict__ offsets,
        uint64_t n, const OutSpec os, uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount,
        const OutSpec os2) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t *skeys = reinterpret_cast<uint64_t *>(smem);                       // a_{1,0..31}
  uint32_t *skeys32 = reinterpret_cast<uint32_t *>(smem + 256);               // DUAL: 32-bit a_{1,0..31}
  uint8_t *ring = smem + 384;                                                  // kByteRing (+ slack)
  uint64_t *offs = reinterpret_cast<uint64_t *>(ring + kByteRing + kSlack + 16);  // kRing x kOffBytes
  TileHdr *hdr = reinterpret_cast<TileHdr *>(reinterpret_cast<uint8_t *>(offs) + (size_t)kRing * kOffBytes);
  uint64_t *bar_off = reinterpret_cast<uint64_t *>(hdr + kRing);  // offsets landed (producer)
  uint64_t *bar_done = bar_off + kRing;                            // tile consumed (producer)
  uint64_t *bar_full = bar_done + kRing;                           // tile ready (consumers)
  if (threadIdx.x < 32) skeys[threadIdx.x] = K.a[threadIdx.x];
  if (DUAL && threadIdx.x < 32) skeys32[threadIdx.x] = K.a32[threadIdx.x];
#if PMP_SHORT_SORT
  uint32_t *s_hist = reinterpret_cast<uint32_t *>(bar_full + kRing);  // 2 x 32 class counters
  uint16_t *s_perm = reinterpret_cast<uint16_t *>(s_hist + 64);      // kTile sorted slots
  if (threadIdx.x < 64) s_hist[threadIdx.x] = 0;
#endif
  if (threadIdx.x == 0) {
    for (int q = 0; q < kRing; q++) {
      mbar_init(&bar_off[q], 1);
      mbar_init(&bar_done[q], kShortWarps);
      mbar_init(&bar_full[q], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const uint32_t ntiles = (uint32_t)((n + kTile - 1) / kTile);
  // tiles of this block: blockIdx.x + k * gridDim.x
  const uint32_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto tile_base = [&](uint32_t k) { return ((uint64_t)blockIdx.x + (uint64_t)k * gridDim.x) * kTile; };
  auto off_slot = [&](uint32_t k) { return offs + (size_t)(k & (kRing - 1)) * (kOffBytes / 8); };

  if (wib == kShortWarps) {
    // ------------------------------------------------------------ producer warp
    auto wait_done = [&](uint32_t k) {  // tile k fully consumed
      mbar_wait(&bar_done[k & (kRing - 1)], (k / kRing) & 1);
    };
    auto issue_offs = [&](uint32_t k) {
      if (k >= kRing) wait_done(k - kRing);  // slot reuse
      if (lane == 0) {
        const int q = (int)(k & (kRing - 1));
        const uint64_t base = tile_base(k);
        const uint64_t cnt = min((uint64_t)kTile + 1, n + 1 - base);
        const uint32_t nb = (uint32_t)((cnt * 8 + 15) & ~15ULL);
        mbar_arrive_tx(&bar_off[q], nb);
        bulk_g2s(off_slot(k), offsets + base, nb, &bar_off[q]);
      }
    };
    // byte-ring bookkeeping (identical in every lane): [tail, head) is in use;
    // tile k's bytes end at tend[k % kRing]; `oldest` is the first unreleased tile.
    uint32_t head = 0, tail = 0, oldest = 0;
    __shared__ uint32_t tend[kRing];
    for (uint32_t k = 0; k < (uint32_t)kOffAhead && k < my_tiles; k++) issue_offs(k);
    for (uint32_t k = 0; k < my_tiles; k++) {
      const int q = (int)(k & (kRing - 1));
      if (k + kOffAhead < my_tiles) issue_offs(k + kOffAhead);
      mbar_wait(&bar_off[q], (k / kRing) & 1);
      const uint64_t base = tile_base(k);
      const uint32_t nv = (uint32_t)min((uint64_t)kTile, n - base);  // strings in this tile
      const uint64_t *o = off_slot(k);
      // span of the tile and its place in the byte ring
      uint32_t mode = 1, nb = 0, pos = 0;
      uintptr_t alo = 0;
      {
        const uint64_t first = o[0], endo = o[nv];
        alo = (uintptr_t)(bytes + first) & ~(uintptr_t)15;
        const uintptr_t ahi = ((uintptr_t)(bytes + endo) + 15) & ~(uintptr_t)15;
        const uint64_t span = first < endo ? (uint64_t)(ahi - alo) : 0;
        if (span <= kSpanMaxTile) {
          mode = 0;
          nb = (uint32_t)span;
          uint32_t start = head;
          if ((start % kByteRing) + nb > kByteRing) start += kByteRing - (start % kByteRing);  // no wrap inside a span
          while (start + nb - tail > kByteRing) {  // release consumed tiles until the span fits
            wait_done(oldest);
            tail = tend[oldest & (kRing - 1)];
            oldest++;
          }
          pos = start % kByteRing;
          head = start + nb;
        }
      }
      // keep `oldest` within kRing of k so tend[] slots are not overwritten early
      while (k - oldest >= (uint32_t)kRing - 1) {
        wait_done(oldest);
        tail = tend[oldest & (kRing - 1)];
        oldest++;
      }
      __syncwarp();
      if (lane == 0) {
        tend[q] = head;
        hdr[q].alo = (uint64_t)alo;
        hdr[q].pos = pos;
        hdr[q].mode = mode;
        mbar_arrive_tx(&bar_full[q], nb);   // release: hdr and offsets visible to consumers
        if (nb) bulk_g2s(ring + pos, reinterpret_cast<const void *>(alo), nb, &bar_full[q]);
      }
      __syncwarp();
    }
    return;
  }
  // -------------------------------------------------------------- consumer warps
  // shared-window addresses computed once (the loop uses explicit ld.shared)
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t offs_s = smem_u32(offs) + 8u * (32u * wib + lane);
  const uint32_t hdr_s = smem_u32(hdr), full_s = smem_u32(bar_full), done_s = smem_u32(bar_done);
  const uint64_t tstride = (uint64_t)gridDim.x * kTile;
  const uint32_t ct = 32u * wib + lane;                 // consumer thread = string slot in the tile
#if PMP_SHORT_SORT
  const uint32_t offs0_s = smem_u32(offs), hist_s = smem_u32(s_hist), perm_s = smem_u32(s_perm);
#endif
  uint64_t ibase = (uint64_t)blockIdx.x * kTile;
  for (uint32_t k = 0; k < my_tiles; k++, ibase += tstride) {
    const uint32_t q = k & (kRing - 1);
    uint64_t i = ibase + ct;
    mbar_wait_s(full_s + 8 * q, (k / kRing) & 1);
    uint64_t ralo;
    uint32_t rpos, mode;
    lds_hdr(hdr_s + 16 * q, ralo, rpos, mode);
    bool valid = i < n;
    uint64_t o0, o1;
    lds_u64x2(offs_s + q * kOffBytes, o0, o1);      // offsets[i], offsets[i+1] (slot-local)
    const uint64_t Bl = valid ? o1 - o0 : 0;
    bool is_short = Bl <= kShortMax;                 // invalid lanes: an empty string, not stored
    const bool is_long = !is_short;
    uint32_t B = (uint32_t)Bl;
    const unsigned longmask = __ballot_sync(FULL, is_long);
    if (longmask) {
      // warp-aggregated append: big strings from the back, others from the front
      const bool big = is_long && Bl >= kBigBytes;
      const unsigned bigmask = __ballot_sync(FULL, big), midmask = longmask & ~bigmask;
      uint32_t mbase = 0, bbase = 0;
      if (lane == 0) {
        if (midmask) mbase = atomicAdd(&wcount[0], (uint32_t)__popc(midmask));
        if (bigmask) bbase = atomicAdd(&wcount[1], (uint32_t)__popc(bigmask));
      }
      mbase = __shfl_sync(FULL, mbase, 0);
      bbase = __shfl_sync(FULL, bbase, 0);
      const unsigned lt = (1u << lane) - 1;
      if (is_long && !big) wlist[mbase + __popc(midmask & lt)] = (uint32_t)i;
      if (big) wlist[n - 1 - (bbase + __popc(bigmask & lt))] = (uint32_t)i;
    }
#if PMP_SHORT_SORT
    // ---- counting sort of the tile's strings by word count (block-wide, two
    // named barriers): warp w then hashes sorted strings 32w..32w+31, whose
    // word counts differ by at most one class, so the word loop below runs
    // to (almost) every lane's own length instead of the longest string of
    // 32 random ones.  Long / past-n strings sort last and are skipped.
    {
      const uint32_t cls = is_short ? min(B / (uint32_t)(BITS / 8), 30u) : 31u;
      const uint32_t hb = hist_s + 128u * (k & 1);
      const uint32_t rank = atoms_add(hb + 4 * cls, 1u);
      named_bar_sync(1, kShortWarps * 32);
      const uint32_t h = lds_u32(hb + 4 * lane);
      uint32_t incl = h;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t start = __shfl_sync(FULL, incl - h, (int)cls);
      sts_u16(perm_s + 2 * (start + rank), (uint16_t)ct);
      named_bar_sync(1, kShortWarps * 32);
      if (ct < 32) sts_u32(hb + 4 * ct, 0u);
      const uint32_t j = lds_u16(perm_s + 2 * ct);
      uint64_t p0, p1;
      lds_u64x2(offs0_s + q * kOffBytes + 8 * j, p0, p1);
      i = ibase + j;
      valid = i < n;
      o0 = p0;
      const uint64_t Bj = valid ? p1 - p0 : 0;
      is_short = Bj <= kShortMax;
      B = (uint32_t)Bj;
    }
#endif
    // warp max of the number of full words (the marker word is handled apart)
    const int tfm = (int)__reduce_max_sync(FULL, is_short ? B / (BITS / 8) : 0u);
    if (is_short) {
      uint64_t lo;
      uint32_t lo32 = 0;
      if (mode == 0) {
        // (lanes past n read the tile's first bytes: in bounds, result not stored)
        const uint32_t sofs = rpos + (valid ? (uint32_t)((uintptr_t)(bytes + o0) - (uintptr_t)ralo) : 0u);
        const uint32_t pa = ring_s + (sofs & ~3u);
        auto fetch = [&](int kk) { return lds_u32(pa + 4 * kk); };
        if constexpr (DUAL) short_tree_dual<V2>(K, skeys, skeys32, B, 8 * (sofs & 3), tfm, fetch, lo, lo32);
        else lo = short_tree_lo<BITS, V2>(K, skeys, B, 8 * (sofs & 3), tfm, fetch);
      } else {
        // direct tile: read the string's aligned 32-bit words straight from global,
        // touching only words that overlap [start, end) (never past offsets[n]).
        const uintptr_t sa = (uintptr_t)(bytes + o0), se = sa + B;
        const uintptr_t pa = sa & ~(uintptr_t)3;
        auto fetch = [&](int kk) {
          const uintptr_t a = pa + 4 * (uintptr_t)kk;
          return (B > 0 && a < se) ? ld_u32(reinterpret_cast<const void *>(a)) : 0u;
        };
        if constexpr (DUAL) short_tree_dual<V2>(K, skeys, skeys32, B, 8 * (uint32_t)(sa & 3), tfm, fetch, lo, lo32);
        else lo = short_tree_lo<BITS, V2>(K, skeys, B, 8 * (uint32_t)(sa & 3), tfm, fetch);
      }
      if (valid) {
        emit<BITS>(os, i, lo);
        if constexpr (DUAL) emit<32>(os2, i, lo32);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(done_s + 8 * q);
  }
}

// ============================================================= warp chunk engine
// A warp walks a range of level-1 chunks of one string, 4 KiB per iteration:
// lane group g = lane/8 owns a 1 KiB group block (1 chunk for PM+64, 2 for
// PM+32), lane r = lane%8 loads units r, r+8, ..., r+56 of it (each load
// instruction covers four whole 128-byte lines).  Each lane multiply-adds its
// 16 words against 16 level-1 keys held in registers, the 8 lanes of a group
// combine their exact partial sums with 3 shuffle levels, add b_1, reduce mod p
// (v_1 of the chunk, Eq. (1)), and fold a_{2, c mod 128} * v_1 into the
// group's exact level-2 accumulator.
template <int BITS> struct LaneKeys;
template <> struct LaneKeys<64> {
  uint64_t k[16];
  PMP_DI void load(const uint64_t *a1, int r) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      k[2 * j] = a1[2 * (r + 8 * j)];
      k[2 * j + 1] = a1[2 * (r + 8 * j) + 1];
    }
  }
};
template <> struct LaneKeys<32> {
  uint32_t k[16];
  PMP_DI void load(const uint64_t *a1, int r) {
#pragma unroll
    for (int jj = 0; jj < 4; jj++)
#pragma unroll
      for (int h = 0; h < 4; h++) k[4 * jj + h] = (uint32_t)a1[4 * (r + 8 * jj) + h];
  }
};

struct StrView {
  const uint8_t *base;  // byte at global offset g0 of the string
  uint64_t g0;          // global byte offset of `base` (multiple of the chunk size)
  uint64_t avail_end;   // global offset one past the last byte readable from `base`
  uint64_t B;           // total string length (bytes)
  uint32_t delta;       // (uintptr)base & 15
};

PMP_DI uint4 realign16(const uint4 &c, const uint4 &n, uint32_t q, uint32_t sh) {
  const uint32_t y0 = q == 0 ? c.x : q == 1 ? c.y : q == 2 ? c.z : c.w;
  const uint32_t y1 = q == 0 ? c.y : q == 1 ? c.z : q == 2 ? c.w : n.x;
  const uint32_t y2 = q == 0 ? c.z : q == 1 ? c.w : q == 2 ? n.x : n.y;
  const uint32_t y3 = q == 0 ? c.w : q == 1 ? n.x : q == 2 ? n.y : n.z;
  const uint32_t y4 = q == 0 ? n.x : q == 1 ? n.y : q == 2 ? n.z : n.w;
  uint4 r;
  r.x = funnel(y0, y1, sh);
  r.y = funnel(y1, y2, sh);
  r.z = funnel(y2, y3, sh);
  r.w = funnel(y3, y4, sh);
  return r;
}

// Loads the 8 units of this lane for the group block starting at global byte
// offset `gofs`, realigned to the string's byte 0, zero where unavailable.
PMP_DI void load_group_block(const StrView &s, uint64_t gofs, int lane, uint4 (&U)[8]) {
  const int r = lane & 7;
  if (s.delta == 0) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint64_t off = gofs + 16 * (uint64_t)(r + 8 * j);
      U[j] = off < s.avail_end ? ld_stream16(s.base + (off - s.g0)) : make_uint4(0, 0, 0, 0);
    }
  } else {
    // aligned unit k covers string-relative bytes [16k - delta, 16k - delta + 16)
    const uint8_t *abase = s.base - s.delta;
    uint4 X[9];
#pragma unroll
    for (int j = 0; j < 9; j++) {
      const uint64_t off = gofs + 16 * (uint64_t)(r + 8 * j);
      const bool need = (j < 8) || (r == 0);
      X[j] = (need && off < s.avail_end + s.delta) ? ld_stream16(abase + (off - s.g0))
                                                   : make_uint4(0, 0, 0, 0);
    }
    const uint32_t q = s.delta >> 2, sh = 8 * (s.delta & 3);
    const int src = (lane & ~7) | ((r + 1) & 7);
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const uint4 send = r == 0 ? X[j + 1] : X[j];  // lane r needs aligned unit r+8j+1
      uint4 nx;
      nx.x = __shfl_sync(FULL, send.x, src);
      nx.y = __shfl_sync(FULL, send.y, src);
      nx.z = __shfl_sync(FULL, send.z, src);
      nx.w = __shfl_sync(FULL, send.w, src);
      U[j] = realign16(X[j], nx, q, sh);
    }
  }
}

// sigma word fix-up near the end of the string: word tlast carries the
// 0x01 marker after the last data byte; words past it are the zero padding.
template <int BITS>
PMP_DI void fixup_unit(uint4 &u, uint64_t t0, uint64_t tlast, uint32_t rbytes) {
  if constexpr (BITS == 64) {
    uint64_t w[2] = {((uint64_t)u.y << 32) | u.x, ((uint64_t)u.w << 32) | u.z};
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint64_t t = t0 + h;
      if (t == tlast) w[h] = (w[h] & ((1ULL << (8 * rbytes)) - 1)) | (1ULL << (8 * rbytes));
      else if (t > tlast) w[h] = 0;
    }
    u = make_uint4((uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32));
  } else {
    uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const uint64_t t = t0 + h;
      if (t == tlast) w[h] = (w[h] & ((1u << (8 * rbytes)) - 1)) | (1u << (8 * rbytes));
      else if (t > tlast) w[h] = 0;
    }
    u = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <int BITS> struct ChunkOut {
  typename Tr<BITS>::Acc acc2;  // sum over processed chunks of a_{2,c mod 128} * v_1(c)
  typename Tr<BITS>::Fe v1_first;  // v_1 of chunk cb (for the single-chunk tree)
};

// Processes chunks [cb, ce) (all inside one level-2 node).  Every lane returns
// the same values.
// POLY (two-level variant, reading Q19): a2 is a table of 128 field elements
// (lo, hi pairs) and chunk c is weighted by a2[(c + rot) mod 128].
// LANE: each lane folds a_{2,c} times its own 3->2-reduced partial
// of block c (lane r = 0 adds b_1 first) into a per-lane level-2 sum: since
// a_{2,c} v_1(c) = a_{2,c} (b_1 + sum_lanes P_lane) mod p, the 3 shuffle levels
// per block are replaced by one 5-level sum per call (v1_first is not set).
// Per lane and node: 32 products < 2^(2n+1.6) (POLY: weights W < p, products
// < 2^(2n+2.6)), so the 5- / 3-limb sums hold the whole warp's total.
#ifndef PMP_L2PF
#define PMP_L2PF 2   // warp_chunks: bulk L2 prefetch distance in 4 KiB tiles (0: off)
#endif
template <int BITS, bool POLY = false, bool LANE = false>
PMP_DI ChunkOut<BITS> warp_chunks(const StrView &s, uint64_t cb, uint64_t ce, const LaneKeys<BITS> &lk,
                                  uint64_t b1, const uint64_t *__restrict__ a2, int lane, uint32_t rot = 0) {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  constexpr int CPG = T::CPG, CPI = 4 * CPG, W = T::W;
  const int g = lane >> 3, r = lane & 7;
  const uint64_t tlast = s.B / W;             // index of the marker word, T - 1
  const uint32_t rbytes = (uint32_t)(s.B % W);
  ChunkOut<BITS> res;
  acc_zero(res.acc2);
  res.v1_first = Fe();
  for (uint64_t c0 = cb; c0 < ce; c0 += CPI) {
    const uint64_t gofs = (c0 + (uint64_t)g * CPG) * (uint64_t)T::CHUNK;  // group block start
#if PMP_L2PF
    // bulk L2 prefetch (TMA engine, no registers) of the tile PMP_L2PF ahead,
    // so that the register-fed loads below find their lines in L2
    if (lane == 0 && c0 + (uint64_t)PMP_L2PF * CPI < ce) {
      const uint64_t pf = (c0 + (uint64_t)PMP_L2PF * CPI) * (uint64_t)T::CHUNK;   // global offset
      const uint64_t pe = min(pf + 4096, s.avail_end);
      if (pe > pf) {
        const uintptr_t a = (uintptr_t)(s.base + (pf - s.g0)) & ~(uintptr_t)15;
        const uint32_t nb = (uint32_t)(((uintptr_t)(s.base + (pe - s.g0)) + 15 - a) & ~(uintptr_t)15);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(nb) : "memory");
      }
    }
#endif
    uint4 U[8];
    load_group_block(s, gofs, lane, U);
    const bool tail = tlast < (c0 + CPI) * 128;  // warp-uniform
    if (tail) {
#pragma unroll
      for (int j = 0; j < 8; j++) fixup_unit<BITS>(U[j], (gofs + 16 * (uint64_t)(r + 8 * j)) / W, tlast, rbytes);
    }
    // ---- level-1 multiply-accumulate (the hot loop) ----
    Acc part[CPG];
    if constexpr (BITS == 64) {
      MacAcc64 A;
      macc_zero(A);
#pragma unroll
      for (int j = 0; j < 8; j++) {
        mac64(A, (uint32_t)lk.k[2 * j], (uint32_t)(lk.k[2 * j] >> 32), U[j].x, U[j].y);
        mac64(A, (uint32_t)lk.k[2 * j + 1], (uint32_t)(lk.k[2 * j + 1] >> 32), U[j].z, U[j].w);
      }
      part[0] = macc_normalize(A);
    } else {
      Acc3 A[2] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int cs = j >> 2, kb = 4 * (j & 3);
        mac32(A[cs], lk.k[kb + 0], U[j].x);
        mac32(A[cs], lk.k[kb + 1], U[j].y);
        mac32(A[cs], lk.k[kb + 2], U[j].z);
        mac32(A[cs], lk.k[kb + 3], U[j].w);
      }
      part[0] = A[0];
      part[1] = A[1];
    }
    if constexpr (LANE) {
#pragma unroll
      for (int cs = 0; cs < CPG; cs++) {
        const uint64_t c = c0 + (uint64_t)g * CPG + cs;
        if (c < ce) {
          Acc x = part[cs];
          if (r == 0) acc_add_word(x, b1);
          if constexpr (POLY) {
            Fe w;
            fe_load(a2 + 2 * ((c + rot) & 127), w);
            acc_mac_partial_fe(res.acc2, w, x);
          } else {
            acc_mac_partial(res.acc2, a2[c & 127], x);
          }
        }
      }
    } else {
    // ---- combine the 8 lanes of each group, reduce, fold into level 2 ----
#pragma unroll
    for (int cs = 0; cs < CPG; cs++) {
      Acc x = part[cs];
#pragma unroll
      for (int m = 1; m < 8; m <<= 1) {
        Acc y = acc_shfl_xor(x, m);
        acc_add(x, y);
      }
      const uint64_t c = c0 + (uint64_t)g * CPG + cs;
      acc_add_word(x, b1);                      // Eq. (1): b_1 + sum a s
      const Fe v1 = acc_reduce(x);
      if (c == cb) res.v1_first = v1;
      if constexpr (POLY) {
        if (c < ce) {
          Fe w;
          fe_load(a2 + 2 * ((c + rot) & 127), w);
          acc_mac_fe_full(res.acc2, w, v1);
        }
      } else {
        if (c < ce) acc_mac_fe(res.acc2, a2[c & 127], v1);
      }
    }
    }
  }
  // sum the four groups' level-2 accumulators (LANE: all 32 lanes')
#pragma unroll
  for (int m = LANE ? 1 : 8; m < 32; m <<= 1) {
    Acc y = acc_shfl_xor(res.acc2, m);
    acc_add(res.acc2, y);
  }
  res.v1_first = fe_shfl(res.v1_first, 0);
  return res;
}

// Level sizes of Algorithm 1 for a string of T words: T_0 = T, T_j = ceil(T_{j-1}/128).
// L_eff = number of f_j applications (0 when T == 1).
struct Geom {
  uint64_t T[kL + 1];
  int leff;
};
PMP_HDI Geom make_geom(uint64_t Twords) {
  Geom gm;
  gm.T[0] = Twords;
  gm.leff = 0;
  uint64_t t = Twords;
  for (int j = 1; j <= (int)kL; j++) {
    if (t > 1) {
      t = (t + 127) / 128;
      gm.leff = j;
    }
    gm.T[j] = t;
  }
  return gm;
}

// ============================================================= k_wstring
// Warp per string from the work list (big strings first).  Each warp streams
// its strings through a private shared-memory ring of 4 KiB tiles fed by TMA
// bulk copies (one elected lane issues them), up to kWStages tiles ahead and
// across string boundaries, and hashes tile t while tiles t+1.. are in flight.
// The issue side is warp-uniform: every lane holds the same cursor (item,
// tile) in registers, so feeding a tile costs a few dozen instructions and no
// divergent single-lane code.  Work items: big strings (>= kBigBytes, listed
// from the back of the work list) are claimed dynamically through a small
// non-blocking claim pipeline (atomic -> work-list entry -> offsets, one
// stage per issued tile); mid strings are strided statically over the warps,
// their offsets fetched 32 at a time, one per lane, one batch ahead.
// A tile is 4 level-1 blocks (PM+64) / 8 (PM+32) of one string; its copy
// starts at the 16-byte aligned address at or below the string's byte 4096 t
// and carries 16 bytes of overlap, so a misaligned string is realigned from
// shared memory (3 loads + funnel shifts per 16 bytes) without shuffles.
// Level 2 is accumulated per lane group and closed every 128 blocks; levels
// >= 3 are streamed by lane 0 (bounded memory).
// POLY: the two-level variant (reading Q19): the same
// level-1 chunk values, combined by V = b_2 + sum_c v_c r^(C-c) instead of the
// tree.  With d = (-C) mod 128 virtual leading zero chunks, chunk c sits at
// position i = (c + d) mod 128 of virtual node q = (c + d) / 128 and
// r^(C-c) = W[i] R^(Q-1-q) (pmp_poly.cuh), so the pipeline is the tree's with
// a_{2,i} replaced by W[i], node boundaries shifted by d, and each closed node
// weighted by a power of R = r^128 and summed.
constexpr uint32_t kPolyW = kL + kL * kM;    // blob word offset of W[0..128) = r^(128-i) (lo, hi pairs)
constexpr uint32_t kPolyLadder = 48;         // R^(2^k), k < 48 (Q < 2^42 for T < 2^56)
constexpr uint32_t kPolyRP = kPolyW + 2 * kM;
constexpr uint32_t kBlobWords = kPolyRP + 2 * kPolyLadder;

// R^e from the square ladder RP[k] = R^(2^k) (same value in every lane)
template <int BITS>
PMP_DI typename Tr<BITS>::Fe poly_pow_R(const uint64_t *__restrict__ keys, uint64_t e) {
  using Fe = typename Tr<BITS>::Fe;
  Fe w = fe_from_word(1, (Fe *)nullptr);
  for (uint32_t k = 0; e; k++, e >>= 1) {
    if (e & 1) {
      Fe f;
      fe_load(keys + kPolyRP + 2 * k, f);
      w = fe_mul(w, f);
    }
  }
  return w;
}

constexpr int kWTile = 4096;
#ifndef PMP_W_STAGES
#define PMP_W_STAGES 2
#endif
constexpr int kWStages = PMP_W_STAGES;
constexpr int kWStageBytes = kWTile + 32;      // + 16 B overlap + 16 B read slack
constexpr int kWBlockWarps = 4;
struct WStack {      // lane 0's streaming state for levels 3..8
  uint64_t T[kL + 1];
  uint64_t pushed[kL - 2];
  uint32_t up[kL - 2][5];
};
struct WHdr {        // one per stage, written by the issuing lane
  uint64_t sa;       // address of the string's byte 0
  uint64_t B;        // string length
  uint32_t i;        // string index
  uint32_t tile;     // tile index within the string
  uint32_t nt;       // tiles | fold flag << 31
  uint32_t nb;       // bytes copied (0: the tile holds only a marker-only block)
};
constexpr size_t kWSmemPerWarpBig =
    ((size_t)kWStages * (kWStageBytes + sizeof(WHdr) + 8) + sizeof(WStack) + 15) & ~(size_t)15;
constexpr size_t kWSmemPerWarpMid =   // mid_phase's layout (kept in step with kMSmemPerWarp)
    ((size_t)2 * (4 * (1024 + 32) + 4 * 32 + 8) + 15) & ~(size_t)15;
constexpr size_t kWSmemPerWarp = kWSmemPerWarpBig > kWSmemPerWarpMid ? kWSmemPerWarpBig : kWSmemPerWarpMid;
// block region: a_{2,0..127} (POLY: W[0..127] lo words), b_1..8, the key-only
// values a_{2,r} * (b_1 + a_{1,0}) mod p (lo words, then hi bits) of a
// marker-only level-1 block at position r (POLY: lo words unused, hi words =
// W hi bits), a_{1,0..127}
constexpr size_t kWBlockRegion = 1024 + 64 + 1024 + 512 + 1024 /* a_{1,0..127} */;
constexpr size_t kWSmem = kWBlockRegion + kWBlockWarps * kWSmemPerWarp;

// Mid strings in 8-lane groups (mid_phase) instead of warp per string.
#ifndef PMP_MID_INLINE
#define PMP_MID_INLINE __forceinline__
#endif
#ifndef PMP_MID_GROUPS
#define PMP_MID_GROUPS 1
#endif
// ============================================================= mid strings (k_wstring, second phase)
// Mid strings (kShortMax < B < kBigBytes, listed at the front of the work
// list).  Such a string has T1 <= 128 level-1 blocks, so its tree is one block
// (L_eff = 1) or one level-2 node (L_eff = 2) and needs no level stack.  One
// 8-lane group hashes one string, four strings per warp: lane r of group g
// owns units r, r+8, ..., r+56 of the group's 1 KiB piece (one PM+64 block,
// two PM+32 blocks) per iteration, the 8 lanes combine their exact sums with 3
// in-group shuffle levels (every lane ends with the block value), and the
// level-2 sum is kept redundantly by all 8 lanes -- so closing a string needs
// no shuffle at all, and the per-string control (geometry, the level-2 close,
// the digest) is paid once per warp for four strings.
// Each iteration stages the four groups' 1 KiB pieces in one ring slot (four
// TMA bulk copies completing on one mbarrier).  Work: the warp claims batches
// of 32 strings (one atomic, one string per lane) and hands them to its
// groups as they finish, so a group that drew short strings takes more.
// POLY (reading Q19): C = T1 <= 128 gives Q = 1 virtual node, d = 128 - C,
// and chunk c weighs W[c + d] = r^(C - c); every string (T1 = 1 included)
// gets V = b_2 + sum.
constexpr int kMPiece = 1024;                  // bytes per group per iteration
constexpr int kMSlot = kMPiece + 32;           // + 16 B overlap + 16 B read slack
#ifndef PMP_M_STAGES
#define PMP_M_STAGES 2
#endif
constexpr int kMStages = PMP_M_STAGES;
struct MHdr {        // per stage and group, written by the group's leader
  uint64_t sa;       // address of the string's byte 0
  uint64_t B;        // length
  uint32_t i;        // string index
  uint32_t t;        // piece index within the string
  uint32_t nt;       // pieces | fold << 31 (0: group idle this iteration)
  uint32_t nb;       // bytes copied
};
constexpr size_t kMSmemPerWarp = ((size_t)kMStages * (4 * kMSlot + 4 * sizeof(MHdr) + 8) + 15) & ~(size_t)15;

// Runs after the warp has drained its big strings; uses the warp's shared
// region (wbase) with its own ring layout and barriers.
template <int BITS, bool POLY>
__device__ PMP_MID_INLINE void mid_phase(const uint64_t *__restrict__ keys, const uint8_t *__restrict__ bytes,
                                       const uint64_t *__restrict__ offsets, const OutSpec &os,
                                       const uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount,
                                       uint32_t nmid, const uint64_t *s_a2, const uint64_t *s_mklo,
                                       const uint32_t *s_mkhi, const uint64_t *s_a1, uint64_t b1, uint64_t b2,
                                       typename Tr<BITS>::Fe v1mk, uint8_t *wbase) {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  constexpr int CPG = T::CPG, W = T::W;
  const int lane = threadIdx.x & 31;
  const int g = lane >> 3, r = lane & 7;
  const bool leader = r == 0;
  MHdr *hdr = reinterpret_cast<MHdr *>(wbase + (size_t)kMStages * 4 * kMSlot);   // [stage][group]
  uint64_t *bar = reinterpret_cast<uint64_t *>(hdr + 4 * kMStages);
  if (nmid == 0) return;
  if (lane == 0) {
    for (int q = 0; q < kMStages; q++) mbar_init(&bar[q], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const uint32_t a1_s = smem_u32(s_a1);
  const uint32_t stg_s = smem_u32(wbase);

  // ---- work: batches of 32 strings per warp (lane e holds string e), two
  // batches in registers (cur is being handed out, nxt is in flight)
  uint32_t cur_i = 0, nxt_i = 0, bi = 0, cur_n = 0, nxt_n = 0;
  uint64_t cur_o0 = 0, cur_o1 = 0, nxt_o0 = 0, nxt_o1 = 0;
  auto fetch_batch = [&]() {  // -> nxt
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(&wcount[3], 32u);
    base = __shfl_sync(FULL, base, 0);
    nxt_n = base < nmid ? min(32u, nmid - base) : 0u;
    if ((uint32_t)lane < nxt_n) {
      nxt_i = wlist[base + lane];
      nxt_o0 = offsets[nxt_i];
      nxt_o1 = offsets[nxt_i + 1];
    }
  };
  fetch_batch();
  cur_i = nxt_i;
  cur_o0 = nxt_o0;
  cur_o1 = nxt_o1;
  cur_n = nxt_n;
  if (cur_n) fetch_batch();

  // ---- issue side: a cursor per group (replicated in its 8 lanes)
  uint64_t p_sa = 0, p_B = 0;
  uint32_t p_i = 0, p_t = 0, p_nt = 0;
  bool p_have = false, p_done = false;
  uint32_t issued = 0, consumed = 0, pq = 0;
  auto pieces_of = [&](uint64_t B) -> uint32_t {
    const uint64_t T1 = (B / W + 1 + 127) / 128;
    const uint32_t nt = (uint32_t)((T1 + CPG - 1) / CPG);
    // a trailing piece holding only the marker-only block is folded away
    const bool fold = nt > 1 && (uint64_t)(nt - 1) * kMPiece >= B;
    return fold ? (nt - 1) | 0x80000000u : nt;
  };
  auto produce = [&]() {
    while (!p_done && issued - consumed < (uint32_t)kMStages) {
      // groups that need a string take the next ones of the batch, in group order
      const bool need = !p_have || p_t == (p_nt & 0x7fffffffu);
      const unsigned needm = __ballot_sync(FULL, need && leader);
      if (needm) {
        const uint32_t rank = __popc(needm & ((1u << lane) - 1));  // meaningful in leaders
        const uint32_t nneed = __popc(needm);
        const uint32_t avail = cur_n > bi ? cur_n - bi : 0u;
        const uint32_t rk = __shfl_sync(FULL, rank, lane & ~7);     // the group's rank
        const bool from_cur = rk < avail;
        const int src = (int)(from_cur ? bi + rk : rk - avail);
        const uint64_t c0 = __shfl_sync(FULL, cur_o0, src & 31), c1 = __shfl_sync(FULL, cur_o1, src & 31);
        const uint64_t n0 = __shfl_sync(FULL, nxt_o0, src & 31), n1 = __shfl_sync(FULL, nxt_o1, src & 31);
        const uint32_t ci = __shfl_sync(FULL, cur_i, src & 31), ni = __shfl_sync(FULL, nxt_i, src & 31);
        if (need) {
          const bool ok = from_cur || (uint32_t)src < nxt_n;
          p_have = ok;
          if (ok) {
            const uint64_t o0 = from_cur ? c0 : n0, o1 = from_cur ? c1 : n1;
            p_sa = (uint64_t)(uintptr_t)(bytes + o0);
            p_B = o1 - o0;
            p_i = from_cur ? ci : ni;
            p_nt = pieces_of(p_B);
            p_t = 0;
          }
        }
        if (cur_n && nneed >= avail) {  // batch used up: rotate (nxt may be empty)
          bi = min(nneed - avail, nxt_n);
          cur_i = nxt_i;
          cur_o0 = nxt_o0;
          cur_o1 = nxt_o1;
          cur_n = nxt_n;
          if (cur_n) fetch_batch();
          else nxt_n = 0;
        } else if (cur_n) {
          bi += nneed;
        }
      }
      if (!__any_sync(FULL, p_have)) {
        p_done = true;
        break;
      }
      // stage pq: this group's piece p_t
      uint32_t nb = 0;
      const uint64_t A = p_sa & ~(uint64_t)15;
      const uint64_t off = (uint64_t)p_t * kMPiece;
      if (p_have) {
        const uint64_t nbytes = ((p_sa + p_B + 15) & ~(uint64_t)15) - A;
        nb = off < nbytes ? (uint32_t)min((uint64_t)(kMPiece + 16), nbytes - off) : 0u;
      }
      const uint32_t tot = __reduce_add_sync(FULL, leader ? nb : 0u);
      MHdr &h = hdr[pq * 4 + g];
      if (leader) {
        h.sa = p_sa;
        h.B = p_B;
        h.i = p_i;
        h.t = p_t;
        h.nt = p_have ? p_nt : 0u;
        h.nb = nb;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the slot
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_tx(&bar[pq], tot);
      __syncwarp();
      if (leader && nb)
        bulk_g2s(wbase + (size_t)(pq * 4 + g) * kMSlot, reinterpret_cast<const void *>(A + off), nb, &bar[pq]);
      if (p_have) p_t++;
      pq = pq + 1 == (uint32_t)kMStages ? 0u : pq + 1;
      issued++;
    }
  };
  produce();

  // ---- consumer: per group, the level-2 sum of the string being hashed
  Acc acc2;
  acc_zero(acc2);
  uint32_t cq = 0, cph = 0;
  while (consumed < issued) {
    const int q = (int)cq;
    mbar_wait(&bar[q], cph);
    if (++cq == (uint32_t)kMStages) {
      cq = 0;
      cph ^= 1;
    }
    const MHdr &h = hdr[q * 4 + g];
    const uint32_t ntf = h.nt, t = h.t, si = h.i;
    const uint64_t B = h.B;
    const uint32_t delta = (uint32_t)h.sa & 15u;
    const bool active = ntf != 0;
    const uint32_t nt = ntf & 0x7fffffffu;
    const bool last = active && t + 1 == nt;
    const bool fold = last && (ntf >> 31);
    const uint64_t tlast = B / W;                   // marker word index
    const uint32_t rbytes = (uint32_t)(B % W);
    const uint64_t T1 = (tlast + 1 + 127) / 128;
    // ---- this lane's 8 units of the group's piece, realigned to the string,
    // in two halves of 4 units (fewer live registers: PM+32 halves are its two
    // blocks), each multiply-added as soon as it is loaded
    const uint32_t ub = stg_s + (uint32_t)(q * 4 + g) * kMSlot + 16 * r;
    const bool aligned = __all_sync(FULL, delta == 0);
    const uint64_t tw0 = (uint64_t)t * (kMPiece / W);  // first word of the piece
    const bool has_marker = active && tlast < tw0 + kMPiece / W;
    const bool fix = __any_sync(FULL, has_marker || !active);
    Acc part[CPG];
    MacAcc64 A64;
    macc_zero(A64);
#pragma unroll
    for (int hp = 0; hp < 2; hp++) {
      uint4 U[4];
      if (aligned) {
#pragma unroll
        for (int j = 0; j < 4; j++)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(U[j].x), "=r"(U[j].y), "=r"(U[j].z), "=r"(U[j].w) : "r"(ub + 128 * (4 * hp + j)));
      } else {
        const uint32_t a0 = ub + (delta & ~3u), sh = 8 * (delta & 3);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t a = a0 + 128 * (4 * hp + j);
          const uint32_t y0 = lds_u32(a), y1 = lds_u32(a + 4), y2 = lds_u32(a + 8), y3 = lds_u32(a + 12),
                         y4 = lds_u32(a + 16);
          U[j] = make_uint4(funnel(y0, y1, sh), funnel(y1, y2, sh), funnel(y2, y3, sh), funnel(y3, y4, sh));
        }
      }
      if (fix) {
        if (!active) {
#pragma unroll
          for (int j = 0; j < 4; j++) U[j] = make_uint4(0, 0, 0, 0);
        } else if (has_marker) {
#pragma unroll
          for (int j = 0; j < 4; j++)
            fixup_unit<BITS>(U[j], tw0 + (uint64_t)(16 * (r + 8 * (4 * hp + j))) / W, tlast, rbytes);
        }
      }
      // ---- level-1 multiply-accumulate
      if constexpr (BITS == 64) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint4 kk;  // a_{1,2u}, a_{1,2u+1}, u = r + 8j
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(kk.x), "=r"(kk.y), "=r"(kk.z), "=r"(kk.w)
                       : "r"(a1_s + 16 * (r + 8 * (4 * hp + j))));
          mac64(A64, kk.x, kk.y, U[j].x, U[j].y);
          mac64(A64, kk.z, kk.w, U[j].z, U[j].w);
        }
        if (hp == 1) part[0] = macc_normalize(A64);
      } else {
        Acc3 A = {0, 0, 0};   // block hp of the piece
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint4 kk;  // a_{1,4u..4u+3}, u = r + 8 j, the same for both blocks
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(kk.x), "=r"(kk.y), "=r"(kk.z), "=r"(kk.w)
                       : "r"(a1_s + 16 * (r + 8 * j)));
          mac32(A, kk.x, U[j].x);
          mac32(A, kk.y, U[j].y);
          mac32(A, kk.z, U[j].z);
          mac32(A, kk.w, U[j].w);
        }
        part[hp < CPG ? hp : 0] = A;
      }
    }
    __syncwarp();
    consumed++;
    produce();                                      // the slot is free: refill it
    // ---- block values (in-group shuffles), level 2
    if (active && t == 0) acc_zero(acc2);
    // each lane folds its own 3->2-reduced partial of block c, times the
    // block's level-2 weight (tree: a_{2,c}, or 1 when the block is the whole
    // tree; POLY: W[c + 128 - C]), into its share of the string's sum; the
    // group adds the shares when the string ends
#pragma unroll
    for (int cs = 0; cs < CPG; cs++) {
      const uint64_t c = (uint64_t)t * CPG + cs;
      if (active && c < T1) {
        Acc x = part[cs];
        if (r == 0) acc_add_word(x, b1);
        if constexpr (POLY) {
          const uint32_t wi = (uint32_t)(c + 128 - T1);
          const uint64_t w2[2] = {s_a2[wi], s_mkhi[wi]};
          Fe w;
          fe_load(w2, w);
          acc_mac_partial_fe(acc2, w, x);
        } else {
          acc_mac_partial(acc2, T1 == 1 ? 1ull : s_a2[c], x);
        }
      }
    }
    if (__any_sync(FULL, last)) {
      Acc x = acc2;
#pragma unroll
      for (int m = 1; m < 8; m <<= 1) {
        Acc y = acc_shfl_xor(x, m);
        acc_add(x, y);
      }
      if (last) {
        if (fold) {                                 // marker-only block T1 - 1
          if constexpr (POLY) {                     // at position 127: W[127] v_1
            const uint64_t w2[2] = {s_a2[127], s_mkhi[127]};
            Fe w;
            fe_load(w2, w);
            acc_mac_fe_full(x, w, v1mk);
          } else {
            const uint64_t w2[2] = {s_mklo[T1 - 1], s_mkhi[T1 - 1]};
            Fe m;
            fe_load(w2, m);
            acc_add_fe(x, m);
          }
        }
        if (POLY || T1 > 1) acc_add_word(x, b2);    // b_2 (POLY: V = b_2 + sum, reading Q19)
        if (leader) emit<BITS>(os, si, acc_reduce_lo(x));
      }
    }
  }
}


#ifndef PMP_W_MINB
#define PMP_W_MINB 5
#endif
template <int BITS, bool POLY = false>
__global__ void __launch_bounds__(kWBlockWarps * 32, PMP_W_MINB)
k_wstring(const uint64_t *__restrict__ keys, const uint8_t *__restrict__ bytes,
          const uint64_t *__restrict__ offsets, uint64_t n, const OutSpec os,
          const uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount) {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  constexpr int CPG = T::CPG, CPI = 4 * CPG, W = T::W;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int g = lane >> 3, r = lane & 7;
  uint64_t *s_a2 = reinterpret_cast<uint64_t *>(smem);   // a_{2,0..127}
  uint64_t *s_b = s_a2 + kM;                              // b_1..b_8
  uint64_t *s_mklo = s_b + kL;                            // marker-only block terms (lo)
  uint32_t *s_mkhi = reinterpret_cast<uint32_t *>(s_mklo + kM);  // (hi bit)
  uint64_t *s_a1 = reinterpret_cast<uint64_t *>(s_mkhi + kM);    // a_{1,0..127} (u64 or packed u32)
  uint8_t *wbase = smem + kWBlockRegion + (size_t)wib * kWSmemPerWarp;
  uint8_t *stg = wbase;                                                   // kWStages x kWStageBytes
  WHdr *hdr = reinterpret_cast<WHdr *>(wbase + (size_t)kWStages * kWStageBytes);
  uint64_t *bar = reinterpret_cast<uint64_t *>(hdr + kWStages);
  WStack *stk = reinterpret_cast<WStack *>(bar + kWStages);
  const uint64_t *bk = keys;           // b_1..b_8
  const uint64_t *ak = keys + kL;      // a_{j,i} at ak[(j-1)*128 + i]
  const uint32_t nmid = wcount[0], nbig = wcount[1];
  if (nmid + nbig == 0) return;
  for (int k = threadIdx.x; k < (int)kM; k += blockDim.x) {
    if constexpr (POLY) {
      s_a2[k] = keys[kPolyW + 2 * k];
      s_mkhi[k] = (uint32_t)keys[kPolyW + 2 * k + 1];
      if constexpr (BITS == 64) s_a1[k] = ak[k];
      else reinterpret_cast<uint32_t *>(s_a1)[k] = (uint32_t)ak[k];
      continue;
    }
    s_a2[k] = ak[kM + k];
    // a marker-only level-1 block (sigma = 1, 0, ..., 0) has v_1 = b_1 + a_{1,0} mod p
    Acc x, y;
    acc_zero(x);
    acc_add_word(x, bk[0]);
    acc_add_word(x, ak[0]);
    acc_zero(y);
    acc_mac_fe(y, ak[kM + k], acc_reduce(x));
    Fe m = acc_reduce(y);
    uint64_t w2[2];
    fe_store(w2, m);
    s_mklo[k] = w2[0];
    s_mkhi[k] = (uint32_t)w2[1];
    if constexpr (BITS == 64) s_a1[k] = ak[k];
    else reinterpret_cast<uint32_t *>(s_a1)[k] = (uint32_t)ak[k];
  }
  if (threadIdx.x < kL) s_b[threadIdx.x] = bk[threadIdx.x];
  if (lane == 0) {
    for (int q = 0; q < kWStages; q++) mbar_init(&bar[q], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const uint64_t b1 = s_b[0], b2 = s_b[1], a10 = ak[0];
  Fe v1mk = Fe();  // POLY: v_1 of a marker-only chunk, b_1 + a_{1,0} mod p
  if constexpr (POLY) {
    Acc x;
    acc_zero(x);
    acc_add_word(x, b1);
    acc_add_word(x, a10);
    v1mk = acc_reduce(x);
  }
  const uint32_t a1_s = smem_u32(s_a1);
  const uint32_t stg_s = smem_u32(stg);

  // tile count of a string and whether its last tile is folded: a trailing
  // tile holding only a marker-only block (no data bytes) is folded into the
  // previous tile unless that block opens a level-2 node
  auto tiles_of = [&](uint64_t sa, uint64_t B) -> uint32_t {
    const uint64_t A = sa & ~(uint64_t)15;
    const uint64_t nbytes = ((sa + B + 15) & ~(uint64_t)15) - A;
    const uint64_t T1 = (B / W + 1 + 127) / 128;           // level-1 blocks
    uint32_t nt = (uint32_t)((T1 + CPI - 1) / CPI);
    // (POLY: the last chunk is at position 127 of its virtual node, never opening one)
    const bool fold = nt > 1 && (uint64_t)(nt - 1) * kWTile >= nbytes && (POLY || ((T1 - 1) & 127) != 0);
    return fold ? (nt - 1) | 0x80000000u : nt;
  };

  // ---- work-item source (warp-uniform state) ----
  const uint32_t gw = blockIdx.x * kWBlockWarps + wib, nw = gridDim.x * kWBlockWarps;
  // big strings: claim pipeline.  cl = 0 idle/exhausted, 1 atomic issued (lane 0),
  // 2 work-list entry loading, 3 offsets loading; each step consumes the
  // previous step's load, so it only stalls if that load is still in flight.
  uint32_t cl = 0, cl_item = 0, cl_bi = 0;
  uint64_t cl_o0 = 0, cl_o1 = 0;
  bool big_open = nbig > 0;
  auto claim_step = [&]() {
    if (cl == 1) {
      cl_item = __shfl_sync(FULL, cl_item, 0);
      if (cl_item < nbig) {
        cl_bi = wlist[n - 1 - cl_item];
        cl = 2;
      } else {
        cl = 0;
        big_open = false;
      }
    } else if (cl == 2) {
      cl_o0 = offsets[cl_bi];
      cl_o1 = offsets[cl_bi + 1];
      cl = 3;
    }
  };
  auto claim_start = [&]() {
    if (lane == 0) cl_item = atomicAdd(&wcount[2], 1u);
    cl = 1;
  };
  if (big_open) claim_start();
  // mid strings: item k of this warp = gw + k * nw; lane e holds item 32 b + e of
  // the current batch b (cur) and of the next one (nxt, loads in flight)
  uint32_t mk = 0;                                   // mid items taken
  uint32_t cur_i = 0, nxt_i = 0;
  uint64_t cur_o0 = 0, cur_o1 = 0, nxt_o0 = 0, nxt_o1 = 0;
  auto fetch_batch = [&](uint32_t kbase) {           // item kbase + lane -> nxt
    const uint32_t item = gw + (kbase + lane) * nw;
    if (item < nmid) {
      nxt_i = wlist[item];
      nxt_o0 = offsets[nxt_i];
      nxt_o1 = offsets[nxt_i + 1];
    }
  };
  if (!PMP_MID_GROUPS) fetch_batch(0);
  // next item into (sa, B, i); false when the warp's work is exhausted
  auto next_item = [&](uint64_t &sa, uint64_t &B, uint32_t &i) -> bool {
    while (big_open) {
      if (cl == 3) {
        sa = (uint64_t)(uintptr_t)(bytes + cl_o0);
        B = cl_o1 - cl_o0;
        i = cl_bi;
        claim_start();
        return true;
      }
      claim_step();                                   // (blocks on the pending load)
    }
    if (PMP_MID_GROUPS) return false;                 // mid strings: mid_phase
    const uint32_t item = gw + mk * nw;
    if (item >= nmid) return false;
    const int e = (int)(mk & 31);
    if (e == 0) {                                     // rotate: next batch becomes current
      cur_i = nxt_i;
      cur_o0 = nxt_o0;
      cur_o1 = nxt_o1;
      fetch_batch(mk + 32);
    }
    const uint64_t o0 = __shfl_sync(FULL, cur_o0, e), o1 = __shfl_sync(FULL, cur_o1, e);
    i = __shfl_sync(FULL, cur_i, e);
    sa = (uint64_t)(uintptr_t)(bytes + o0);
    B = o1 - o0;
    mk++;
    return true;
  };

  // ---- issue side (warp-uniform cursor) ----
  uint64_t p_sa = 0, p_B = 0;
  uint32_t p_i = 0, p_nt = 0, p_tile = 0;
  bool p_have = false, p_done = false;
  uint32_t issued = 0, consumed = 0, pq = 0;
  auto produce = [&]() {
    while (!p_done && issued - consumed < (uint32_t)kWStages) {
      if (!p_have || p_tile == (p_nt & 0x7fffffffu)) {
        if (!next_item(p_sa, p_B, p_i)) {
          p_done = true;
          break;
        }
        p_nt = tiles_of(p_sa, p_B);
        p_tile = 0;
        p_have = true;
      }
      const uint64_t A = p_sa & ~(uint64_t)15;
      const uint64_t nbytes = ((p_sa + p_B + 15) & ~(uint64_t)15) - A;
      const uint64_t off = (uint64_t)p_tile * kWTile;
      const uint32_t nb = off < nbytes ? (uint32_t)min((uint64_t)(kWTile + 16), nbytes - off) : 0u;
      if (lane == 0) {
        WHdr &h = hdr[pq];
        h.sa = p_sa;
        h.B = p_B;
        h.i = p_i;
        h.tile = p_tile;
        h.nt = p_nt;
        h.nb = nb;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the slot
        mbar_arrive_tx(&bar[pq], nb);
        if (nb) bulk_g2s(stg + (size_t)pq * kWStageBytes, reinterpret_cast<const void *>(A + off), nb, &bar[pq]);
      }
      pq = pq + 1 == (uint32_t)kWStages ? 0u : pq + 1;
      p_tile++;
      issued++;
      if (cl == 1 || cl == 2) claim_step();          // advance the big claim one step per tile
    }
  };
  produce();

  // ---- consumer state (whole warp): the string being hashed
  uint64_t tlast = 0, T1 = 0;
  uint32_t rbytes = 0;
  int leff = 0;
  Acc acc2;
  acc_zero(acc2);
  Fe root = Fe();
  Acc pacc, acc2b;                                 // POLY: sum of weighted node values;
  acc_zero(pacc);                                  //   next virtual node's level-2 sum
  acc_zero(acc2b);
  uint32_t dsh = 0;                                // POLY: d = (-C) mod 128
  uint64_t Qp = 0;                                 // POLY: number of virtual nodes
  uint32_t cq = 0, cph = 0;                        // consumer slot and phase
  while (consumed < issued) {
    const int q = (int)cq;
    mbar_wait(&bar[q], cph);
    if (++cq == (uint32_t)kWStages) {
      cq = 0;
      cph ^= 1;
    }
    const WHdr &h = hdr[q];
    const uint32_t si = h.i, t = h.tile, ntiles = h.nt & 0x7fffffffu;
    const uint32_t delta = (uint32_t)h.sa & 15u;
    const bool fold = (h.nt >> 31) && t + 1 == ntiles; // + the string's marker-only last block
    const bool nodata = h.nb == 0;                   // only the marker word (= 1) at word 128*c0
    if (t == 0) {                                    // a new string starts
      const uint64_t B = h.B;
      tlast = B / W;
      rbytes = (uint32_t)(B % W);
      T1 = (tlast + 1 + 127) / 128;
      leff = tlast == 0 ? 0 : T1 == 1 ? 1 : T1 <= 128 ? 2 : levels_of(tlast + 1);
      acc_zero(acc2);
      if constexpr (POLY) {
        dsh = (uint32_t)((128 - T1 % 128) % 128);
        Qp = (T1 + dsh) / 128;
        acc_zero(pacc);
        acc_zero(acc2b);
        leff = 2;                                    // (no level stack)
      }
      if (!POLY && leff >= 3 && lane == 0) {                  // streaming state for levels >= 3
        const Geom gm = make_geom(tlast + 1);
        for (int j = 0; j <= (int)kL; j++) stk->T[j] = gm.T[j];
        for (int j = 0; j < (int)kL - 2; j++) {
          stk->pushed[j] = 0;
          for (int l = 0; l < 5; l++) stk->up[j][l] = 0;
        }
      }
    }
    const uint32_t st_s = stg_s + (uint32_t)q * kWStageBytes;
    const uint64_t c0 = (uint64_t)t * CPI;          // first level-1 block of this tile
    // ---- this lane's 8 units, in two halves of 4 (fewer live registers; the
    // PM+32 halves are the group's two blocks), each multiply-added as loaded
    Acc part[CPG];
    const uint32_t ub = st_s + 1024 * g + 16 * r;    // this lane's unit j is at ub + 128 j (+ delta)
    const bool tailtile = tlast < (c0 + CPI) * 128;   // warp-uniform: the tile holds the marker word
    const uint64_t tw0 = (c0 + (uint64_t)g * CPG) * 128;
    MacAcc64 A64;
    macc_zero(A64);
#pragma unroll
    for (int hp = 0; hp < 2; hp++) {
      uint4 U[4];
      if (nodata) {
#pragma unroll
        for (int j = 0; j < 4; j++) U[j] = make_uint4(0, 0, 0, 0);
        // sigma of block c0 is (1, 0, ..., 0): its sum is a_{1,0} (added in lane 0 of group 0 below)
      } else if (delta == 0) {                       // warp-uniform: aligned string
#pragma unroll
        for (int j = 0; j < 4; j++)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(U[j].x), "=r"(U[j].y), "=r"(U[j].z), "=r"(U[j].w) : "r"(ub + 128 * (4 * hp + j)));
      } else {                                       // realign: 5 aligned words + funnel shifts
        const uint32_t a0 = ub + (delta & ~3u), sh = 8 * (delta & 3);
        if ((delta & 4) == 0) {                      // a0 is 8-byte aligned: (y0,y1) (y2,y3) y4
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t a = a0 + 128 * (4 * hp + j);
            uint32_t y0, y1, y2, y3;
            lds_u32x2(a, y0, y1);
            lds_u32x2(a + 8, y2, y3);
            const uint32_t y4 = lds_u32(a + 16);
            U[j] = make_uint4(funnel(y0, y1, sh), funnel(y1, y2, sh), funnel(y2, y3, sh), funnel(y3, y4, sh));
          }
        } else {                                     // a0 + 4 is 8-byte aligned: y0 (y1,y2) (y3,y4)
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const uint32_t a = a0 + 128 * (4 * hp + j);
            uint32_t y1, y2, y3, y4;
            const uint32_t y0 = lds_u32(a);
            lds_u32x2(a + 4, y1, y2);
            lds_u32x2(a + 12, y3, y4);
            U[j] = make_uint4(funnel(y0, y1, sh), funnel(y1, y2, sh), funnel(y2, y3, sh), funnel(y3, y4, sh));
          }
        }
      }
      if (!nodata && tailtile) {
#pragma unroll
        for (int j = 0; j < 4; j++)
          fixup_unit<BITS>(U[j], tw0 + (uint64_t)(16 * (r + 8 * (4 * hp + j))) / W, tlast, rbytes);
      }
      // ---- level-1 multiply-accumulate (the hot loop) ----
      if constexpr (BITS == 64) {
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint4 kk;  // a_{1,2u}, a_{1,2u+1} for this lane's unit u = r + 8j (block-shared copy)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(kk.x), "=r"(kk.y), "=r"(kk.z), "=r"(kk.w)
                       : "r"(a1_s + 16 * (r + 8 * (4 * hp + j))));
          mac64(A64, kk.x, kk.y, U[j].x, U[j].y);
          mac64(A64, kk.z, kk.w, U[j].z, U[j].w);
        }
        if (hp == 1) part[0] = macc_normalize(A64);
      } else {
        Acc3 A = {0, 0, 0};   // block hp of the group block
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uint4 kk;  // a_{1,4u..4u+3}, u = r + 8 j (packed u32 copy), same for both blocks
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(kk.x), "=r"(kk.y), "=r"(kk.z), "=r"(kk.w)
                       : "r"(a1_s + 16 * (r + 8 * j)));
          mac32(A, kk.x, U[j].x);
          mac32(A, kk.y, U[j].y);
          mac32(A, kk.z, U[j].z);
          mac32(A, kk.w, U[j].w);
        }
        part[hp < CPG ? hp : 0] = A;
      }
    }
    if (nodata && lane == 0) acc_add_word(part[0], a10);
    __syncwarp();
    // the slot is free: refill the ring before the reductions
    consumed++;
    produce();
    // POLY: virtual node of the tile's first chunk, and whether the tile crosses
    // into the next one (virtual node boundaries fall inside tiles when d > 0)
    const uint64_t qf = (c0 + dsh) >> 7;
    const bool cross = POLY && ((c0 + CPI - 1 + dsh) >> 7) != qf;
    // tree strings with a level 2: each lane folds a_{2,c} times its own
    // 3->2-reduced partial (lane r = 0 adds b_1) into its level-2 sum, which
    // the node close sums over all 32 lanes (see warp_chunks, LANE)
    const bool lane_sums = POLY || leff >= 2;
    if (lane_sums) {
#pragma unroll
      for (int cs = 0; cs < CPG; cs++) {
        const uint64_t c = c0 + (uint64_t)g * CPG + cs;
        if (c < T1) {
          Acc x = part[cs];
          if (r == 0) acc_add_word(x, b1);
          if constexpr (POLY) {                     // W[(c + d) mod 128] times the lane's share
            const uint32_t wi = (uint32_t)(c + dsh) & 127;
            const uint64_t w2[2] = {s_a2[wi], s_mkhi[wi]};
            Fe w;
            fe_load(w2, w);
            if (cross && ((c + dsh) >> 7) != qf) acc_mac_partial_fe(acc2b, w, x);
            else acc_mac_partial_fe(acc2, w, x);
          } else {
            acc_mac_partial(acc2, s_a2[c & 127], x);
          }
        }
      }
    }
    // ---- combine the 8 lanes of each group, fold into level 2 ----
#pragma unroll
    for (int cs = 0; cs < CPG; cs++) {
      if (lane_sums) break;
      Acc x = part[cs];
#pragma unroll
      for (int m = 1; m < 8; m <<= 1) {
        Acc y = acc_shfl_xor(x, m);
        acc_add(x, y);
      }
      const uint64_t c = c0 + (uint64_t)g * CPG + cs;
      acc_add_word(x, b1);                          // Eq. (1): b_1 + sum a s
      if constexpr (POLY) {
        if (c < T1) {                               // W[(c + d) mod 128] * v_1(c), v_1 reduced
          const uint32_t wi = (uint32_t)(c + dsh) & 127;
          const uint64_t w2[2] = {s_a2[wi], s_mkhi[wi]};
          Fe w;
          fe_load(w2, w);
          const Fe v1 = acc_reduce(x);
          if (cross && ((c + dsh) >> 7) != qf) acc_mac_fe_full(acc2b, w, v1);
          else acc_mac_fe_full(acc2, w, v1);
        }
      } else if (leff == 1) {
        if (c == 0) root = acc_reduce(x);           // the whole tree is one block
      } else if (c < T1) {
        acc_mac_partial(acc2, s_a2[c & 127], x);    // a_{2, c mod 128} * v_1(c), v_1 3->2-reduced
      }
    }
    if (fold && lane == 0) {
      // marker-only last block c = T1 - 1 (sigma = 1, 0, ..., 0): its term
      // a_{2,c mod 128} (b_1 + a_{1,0}) mod p is key-only, precomputed per block
      // (POLY: W[127] v_1, the chunk being at position 127)
      if constexpr (POLY) {
        const uint64_t w2[2] = {s_a2[127], s_mkhi[127]};
        Fe w;
        fe_load(w2, w);
        if (cross && ((T1 - 1 + dsh) >> 7) != qf) acc_mac_fe_full(acc2b, w, v1mk);
        else acc_mac_fe_full(acc2, w, v1mk);
      } else {
        const uint64_t w2[2] = {s_mklo[(T1 - 1) & 127], s_mkhi[(T1 - 1) & 127]};
        Fe m;
        fe_load(w2, m);
        acc_add_fe(acc2, m);
      }
    }
    // ---- close a level-2 node every 128 blocks and at the end of the string
    const uint64_t cend = fold ? T1 : c0 + CPI;
    if constexpr (POLY) {
      // virtual nodes completed by this tile: qf when cend + d reaches its end,
      // and qf + 1 too at the end of the string (cend + d = 128 Q there)
      const uint64_t cv = min(cend, T1) + dsh;
      for (uint64_t qn = qf; qn < Qp && cv >= 128 * (qn + 1); qn++) {
        Acc x = acc2;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {            // lane sums: all 32 lanes
          Acc y = acc_shfl_xor(x, m);
          acc_add(x, y);
        }
        acc2 = acc2b;
        acc_zero(acc2b);
        Fe nv = acc_reduce(x);                      // node sum, weighted by R^(Q-1-q)
        if (qn + 1 < Qp) nv = fe_mul(nv, poly_pow_R<BITS>(keys, Qp - 1 - qn));
        acc_add_fe(pacc, nv);
      }
      if (cend >= T1 && lane == 0) {
        acc_add_word(pacc, b2);                     // V = b_2 + sum (reading Q19)
        emit<BITS>(os, si, acc_reduce_lo(pacc));
      }
      continue;
    }
    if (leff >= 2 && ((cend & 127) == 0 || cend >= T1)) {
      Acc x = acc2;
#pragma unroll
      for (int m = 1; m < 32; m <<= 1) {             // lane sums (!POLY, leff >= 2): all 32 lanes
        Acc y = acc_shfl_xor(x, m);
        acc_add(x, y);
      }
      acc_zero(acc2);
      acc_add_word(x, b2);                          // b_2
      if (leff == 2) {
        if (lane == 0) emit<BITS>(os, si, acc_reduce_lo(x));  // V mod 2^n
        continue;
      }
      Fe v = acc_reduce(x);                         // v_{2,q}
      if (lane == 0) {
        // push v into level 3, carrying completed nodes upward
        for (int j = 3; j <= leff; j++) {
          const int li = j - 3;
          Acc u;
          load_acc(stk->up[li], u);
          acc_mac_fe(u, ak[(uint64_t)(j - 1) * kM + (stk->pushed[li] & 127)], v);
          const uint64_t pu = ++stk->pushed[li];
          if ((pu & 127) != 0 && pu != stk->T[j - 1]) {  // node still open
            store_acc(stk->up[li], u);
            break;
          }
          acc_add_word(u, s_b[j - 1]);
          v = acc_reduce(u);
          acc_zero(u);
          store_acc(stk->up[li], u);
          if (j == leff) root = v;
        }
      }
    }
    if (t + 1 == ntiles && leff != 2) {
      if (leff == 1) root = fe_shfl(root, 0);
      if (lane == 0) emit<BITS>(os, si, fe_lo(root));
    }
  }
#if PMP_MID_GROUPS
  static_assert(kWSmemPerWarp >= kMSmemPerWarp, "mid_phase layout");
  __syncwarp();
  if (lane == 0)   // the big phase's barriers sit in memory mid_phase reuses
    for (int q = 0; q < kWStages; q++) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar[q])) : "memory");
  __syncwarp();
  mid_phase<BITS, POLY>(keys, bytes, offsets, os, wlist, wcount, nmid, s_a2, s_mklo, s_mkhi, s_a1, b1, b2,
                        v1mk, wbase);
#endif
}

// ============================================================= long string
// Partial tree of one long string split across callers (ranks): every level-1
// chunk value v_1 includes b_1; every level >= 2 sums a_{j,r} * child over the
// children the caller owns, without b_j.  The key-only constant C (all v_1 = 0)
// is added once in k_combine, so V = C + sum over callers ("Long
// strings: affine split").
template <int BITS>
__global__ void __launch_bounds__(kWWarps * 32)
k_node(const uint64_t *__restrict__ keys, StrView s, uint64_t cb, uint64_t ce, uint64_t qb, uint64_t qe,
       int single, uint64_t *__restrict__ s2) {
  using T = Tr<BITS>;
  using Fe = typename T::Fe;
  const int lane = threadIdx.x & 31;
  const uint64_t *bk = keys, *ak = keys + kL;
  const uint64_t warp = (uint64_t)blockIdx.x * kWWarps + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kWWarps;
  if (single) {  // whole tree is one level-1 block (or no block at all)
    if (warp != 0) return;
    if (s.B < (uint64_t)T::W) {  // T == 1: the sole value is sigma_0 (reading Q2)
      if (lane == 0) {
        uint64_t w = 0;
        for (uint32_t k = 0; k < (uint32_t)s.B; k++) w |= (uint64_t)s.base[k] << (8 * k);
        w |= 1ULL << (8 * s.B);
        Fe v = fe_from_word(w, (Fe *)nullptr);
        fe_store(s2, v);
      }
      return;
    }
    LaneKeys<BITS> lk;
    lk.load(ak, lane & 7);
    ChunkOut<BITS> co = warp_chunks<BITS>(s, 0, 1, lk, bk[0], ak + kM, lane);
    if (lane == 0) fe_store(s2, co.v1_first);
    return;
  }
  if (warp >= qe - qb) return;
  LaneKeys<BITS> lk;
  lk.load(ak, lane & 7);
  for (uint64_t q = qb + warp; q < qe; q += nw) {
    const uint64_t lo = max(q * 128, cb), hi = min(q * 128 + 128, ce);
    ChunkOut<BITS> co = warp_chunks<BITS, false, true>(s, lo, hi, lk, bk[0], ak + kM, lane);
    const Fe v = acc_reduce(co.acc2);
    if (lane == 0) fe_store(s2 + 2 * (q - qb), v);
  }
}

// out node q (global index) = sum over owned children c in [128q, 128q+128) of
// a_{j, c mod 128} * in[c - in_lo]; children are field elements (lo, hi).
template <int BITS>
__global__ void __launch_bounds__(kWWarps * 32)
k_level(const uint64_t *__restrict__ keys, int j, const uint64_t *__restrict__ in, uint64_t in_lo,
        uint64_t in_cnt, uint64_t *__restrict__ outv, uint64_t out_lo, uint64_t out_cnt) {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  const int lane = threadIdx.x & 31;
  const uint64_t *aj = keys + kL + (uint64_t)(j - 1) * kM;
  const uint64_t warp = (uint64_t)blockIdx.x * kWWarps + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kWWarps;
  for (uint64_t qi = warp; qi < out_cnt; qi += nw) {
    const uint64_t q = out_lo + qi;
    Acc x;
    acc_zero(x);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint64_t c = q * 128 + lane + 32 * k;
      if (c >= in_lo && c < in_lo + in_cnt) {
        Fe v;
        fe_load(in + 2 * (c - in_lo), v);
        acc_mac_fe(x, aj[lane + 32 * k], v);
      }
    }
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
      Acc y = acc_shfl_xor(x, m);
      acc_add(x, y);
    }
    if (lane == 0) fe_store(outv + 2 * qi, acc_reduce(x));
  }
}

// ============================================================= streaming
// Device state of an incremental hash (the tree evaluated bottom-up
// with bounded memory).  Instead of buffering up to m values per level, every
// level keeps the exact running sum of its open node (sum_r a_{j,r} x_r, b_j
// added when the node closes) -- O(L) state, same arithmetic.
struct StreamState {
  uint32_t acc[kL + 1][5];   // open node sums of levels 2..8 (Acc5, or Acc3 in the first words)
  uint32_t cnt[kL + 1];      // children already in the open node of level j
  uint64_t last[kL + 1][2];  // last value emitted at level j (field element)
  uint64_t emitted[kL + 1];  // values emitted so far at level j (cnt[j+1] == emitted[j] mod 128)
  uint32_t blocks_done;      // k_stream_node: blocks finished in the current launch
};

template <int BITS> struct StreamOps {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  const uint64_t *bk, *ak;
  StreamState *st;
  PMP_DI void close(int j) {  // node of level j complete: emit it and push into level j+1
    for (;;) {
      Acc a;
      load_acc(st->acc[j], a);
      acc_add_word(a, bk[j - 1]);
      const Fe v = acc_reduce(a);
      fe_store(st->last[j], v);
      acc_zero(a);
      store_acc(st->acc[j], a);
      st->cnt[j] = 0;
      if (j + 1 > (int)kL) return;  // only reachable past the string's own top level
      if (!push(j + 1, v)) return;
      j++;
    }
  }
  // adds child v to level j's open node; true if that node is now full (the caller closes it)
  PMP_DI bool push(int j, const Fe &v) {
    Acc a;
    load_acc(st->acc[j], a);
    acc_mac_fe(a, ak[(uint64_t)(j - 1) * kM + st->cnt[j]], v);
    store_acc(st->acc[j], a);
    return ++st->cnt[j] == kM;
  }
};

// Sum of the P piece partials of one level-2 node, by one warp (lanes over
// pieces), result in every lane.
template <int BITS>
PMP_DI typename Tr<BITS>::Acc node_pieces_sum(const uint64_t *s2, uint64_t qi, int P, int lane) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  Acc x;
  acc_zero(x);
  if (lane < P) {
    Fe v;
    fe_load_cg(s2 + 2 * (qi * P + lane), v);
    acc_add_fe(x, v);
  }
#pragma unroll
  for (int mm = 1; mm < 32; mm <<= 1) {
    Acc y = acc_shfl_xor(x, mm);
    acc_add(x, y);
  }
  return x;
}

// Folds one update (level-1 blocks [c0, c0+N) = level-2 nodes qb .. qb+nq-1,
// P pieces each) into the stream state, on the one block that finished last.
// The grid has already written va[qi] = v_2 of every node the update completes
// except node qb when it was open before (its earlier children live in the
// state).  Here: that node, the open node at the end of the update, and levels
// >= 3 -- level by level, one warp per level-j node over its <= 128 new
// children (as k_level); complete nodes emit in parallel and only the open
// node of each level (first/last of the batch) meets the persistent state.
// The new open sum is staged in shared memory and committed after a barrier,
// so the warp reading the old one never races the warp replacing it.
// va/vb: values of two adjacent levels (>= nq each).
template <int BITS>
__device__ void stream_merge_block(const uint64_t *__restrict__ keys, StreamState *st,
                                   const uint64_t *__restrict__ s2, uint64_t qb, uint64_t nq, uint64_t c0,
                                   uint64_t N, int P, bool open0, uint64_t *__restrict__ va,
                                   uint64_t *__restrict__ vb) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  const uint64_t *bk = keys, *ak = keys + kL;
  __shared__ uint64_t s_m, s_e;
  __shared__ uint32_t s_open[5];
  __shared__ int s_has_open;
  // ---------------- level 2: the boundary nodes
  const uint64_t end = c0 + N;
  const uint64_t m2 = end / 128 - qb;               // nodes this update completes
  if (wid == 0 && open0 && m2 > 0) {                // node qb: earlier children + this update's
    Acc x = node_pieces_sum<BITS>(s2, 0, P, lane);
    if (lane == 0) {
      Acc o;
      load_acc(st->acc[2], o);
      acc_add(x, o);
      acc_add_word(x, bk[1]);
      fe_store(va, acc_reduce(x));
    }
  }
  if (wid == nwarps - 1 && lane == 0) s_has_open = 0;
  if (wid == nwarps - 1 && m2 < nq) {               // the update ends inside node qb + nq - 1
    Acc x = node_pieces_sum<BITS>(s2, nq - 1, P, lane);
    if (lane == 0) {
      if (m2 == 0) {                                // still node qb: keep its earlier children
        Acc o;
        load_acc(st->acc[2], o);
        acc_add(x, o);
      }
      store_acc(s_open, x);
      s_has_open = 1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    Acc o;
    if (s_has_open) load_acc(s_open, o);
    else acc_zero(o);
    store_acc(st->acc[2], o);
    st->cnt[2] = (uint32_t)(end % 128);
    s_e = st->emitted[2];
    st->emitted[2] += m2;
    if (m2) {
      Fe v;
      fe_load_cg(va + 2 * (m2 - 1), v);
      fe_store(&st->last[2][0], v);
    }
    s_m = m2;
    s_has_open = 0;
  }
  __syncthreads();
  // ---------------- levels 3..8: the new values of level j-1 join level-j nodes
  uint64_t *in = va, *outv = vb;
  for (int j = 3; j <= (int)kL; j++) {
    const uint64_t m_in = s_m, e_in = s_e;          // new values have level-(j-1) indices [e_in, e_in + m_in)
    if (m_in == 0) break;
    const uint64_t kf = e_in / 128, kl = (e_in + m_in - 1) / 128;
    const uint64_t m_out = (e_in + m_in) / 128 - kf; // level-j nodes completed by this batch
    const uint64_t *aj = ak + (uint64_t)(j - 1) * kM;
    const bool openj = st->cnt[j] != 0;
    for (uint64_t k = kf + wid; k <= kl; k += nwarps) {
      Acc x;
      acc_zero(x);
#pragma unroll
      for (int r0 = 0; r0 < 128; r0 += 32) {
        const uint64_t g = k * 128 + r0 + lane;
        if (g >= e_in && g < e_in + m_in) {
          Fe v;
          fe_load_cg(in + 2 * (g - e_in), v);
          acc_mac_fe(x, aj[r0 + lane], v);
        }
      }
#pragma unroll
      for (int mm = 1; mm < 32; mm <<= 1) {
        Acc y = acc_shfl_xor(x, mm);
        acc_add(x, y);
      }
      if (lane == 0) {
        if (k == kf && openj) {
          Acc o;
          load_acc(st->acc[j], o);
          acc_add(x, o);
        }
        if (k - kf < m_out) {                       // complete node: emit its value
          acc_add_word(x, bk[j - 1]);
          fe_store(outv + 2 * (k - kf), acc_reduce(x));
        } else {                                    // the batch ends inside it: it stays open
          store_acc(s_open, x);
          s_has_open = 1;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      Acc o;
      if (s_has_open) load_acc(s_open, o);
      else acc_zero(o);
      store_acc(st->acc[j], o);
      st->cnt[j] = (uint32_t)((e_in + m_in) % 128);
      s_e = st->emitted[j];
      st->emitted[j] += m_out;
      if (m_out) {
        Fe v;
        fe_load_cg(outv + 2 * (m_out - 1), v);
        fe_store(&st->last[j][0], v);
      }
      s_m = m_out;
      s_has_open = 0;
    }
    __syncthreads();
    uint64_t *t = in;
    in = outv;
    outv = t;
  }
}

// One update of a stream in one launch.  Warps compute the partial level-2
// sums of (node, piece) items, P pieces of 128/P level-1 blocks per node (as
// k_node); the warp that finishes a node's last piece (per-node counter,
// self-resetting) emits v_2 of every complete node the state has no share in;
// the block that finishes last runs stream_merge_block.
template <int BITS>
__global__ void __launch_bounds__(kWWarps * 32)
k_stream_node(const uint64_t *__restrict__ keys, StrView s, uint64_t c0, uint64_t N, uint64_t qb, uint64_t qe,
              int P, uint64_t *__restrict__ s2, uint32_t *__restrict__ node_cnt, StreamState *st,
              uint64_t *__restrict__ va, uint64_t *__restrict__ vb) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  const int lane = threadIdx.x & 31;
  const uint64_t *bk = keys, *ak = keys + kL;
  const uint64_t warp = (uint64_t)blockIdx.x * kWWarps + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kWWarps;
  const uint64_t nu = (qe - qb) * (uint64_t)P, span = 128 / P;
  const uint64_t m2 = (c0 + N) / 128 - qb;          // nodes the update completes
  const bool open0 = st->cnt[2] != 0;
  if (warp < nu) {
    LaneKeys<BITS> lk;
    lk.load(ak, lane & 7);
    for (uint64_t u = warp; u < nu; u += nw) {
      const uint64_t qi = u / P;
      const uint64_t c = (qb + qi) * 128 + (u % P) * span;
      const uint64_t lo = max(c, c0), hi = min(c + span, c0 + N);
      Acc x;
      if (lo < hi) {
        ChunkOut<BITS> co = warp_chunks<BITS, false, true>(s, lo, hi, lk, bk[0], ak + kM, lane);
        x = co.acc2;
      } else {
        acc_zero(x);
      }
      if (qi >= m2 || (qi == 0 && open0)) {         // boundary node: the merge sums its pieces
        if (lane == 0) fe_store(s2 + 2 * u, acc_reduce(x));
        continue;
      }
      bool last_piece = true;
      if (P > 1) {
        int done = 0;
        if (lane == 0) {
          fe_store(s2 + 2 * u, acc_reduce(x));
          __threadfence();
          done = atomicAdd(&node_cnt[qi], 1u) == (unsigned)P - 1;
        }
        last_piece = __shfl_sync(0xffffffffu, done, 0);
        if (!last_piece) continue;
        __threadfence();
        x = node_pieces_sum<BITS>(s2, qi, P, lane);
      }
      if (lane == 0) {
        if (P > 1) node_cnt[qi] = 0;
        acc_add_word(x, bk[1]);
        fe_store(va + 2 * qi, acc_reduce(x));
      }
    }
  }
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  stream_merge_block<BITS>(keys, st, s2, qb, qe - qb, c0, N, P, open0, va, vb);
  if (threadIdx.x == 0) st->blocks_done = 0;
}

// Final: fold the last level-1 block (partial sum in s2last), close every open
// node bottom-up through the top level leff, whose single value is the root
// (Algorithm 1's "while |sigma| > 1"); leff <= 1: s2last is the root.
template <int BITS>
__global__ void k_stream_final(const uint64_t *__restrict__ keys, StreamState *st, const uint64_t *__restrict__ s2last,
                               int leff, void *__restrict__ out) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Fe root;
  if (leff <= 1) {
    fe_load(s2last, root);
  } else {
    StreamOps<BITS> ops{keys, keys + kL, st};
    Fe v;
    fe_load(s2last, v);
    Acc a;
    load_acc(st->acc[2], a);
    acc_add_fe(a, v);
    store_acc(st->acc[2], a);
    if (++st->cnt[2] == kM) ops.close(2);
    for (int j = 2; j <= leff; j++) {
      if (st->cnt[j] == 0) continue;
      // close level j (zero padding) and push into j+1 unless j is the top
      Acc x;
      load_acc(st->acc[j], x);
      acc_add_word(x, keys[j - 1]);
      const Fe w = acc_reduce(x);
      fe_store(st->last[j], w);
      acc_zero(x);
      store_acc(st->acc[j], x);
      st->cnt[j] = 0;
      if (j < leff && ops.push(j + 1, w)) ops.close(j + 1);
    }
    fe_load(st->last[leff], root);
  }
  store_digest<BITS>(out, 0, fe_lo(root));
}

// V = C + sum_g P_g mod p; digest = mix(V mod 2^n)
template <int BITS>
__global__ void k_combine(const uint64_t *__restrict__ partials, int G, uint64_t c_lo, uint64_t c_hi,
                          void *__restrict__ out) {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Acc x;
  acc_zero(x);
  uint64_t cw[2] = {c_lo, c_hi};
  Fe c;
  fe_load(cw, c);
  acc_add_fe(x, c);
  for (int g = 0; g < G; g++) {
    Fe v;
    fe_load(partials + 2 * g, v);
    acc_add_fe(x, v);
  }
  store_digest<BITS>(out, 0, fe_lo(acc_reduce(x)));
}

// ============================================================= self-test hooks
// mode 0: reduce the exact value (w0 + w1 2^n + w2 2^2n) mod p through the
//         3->2 reduction + Algorithm 2; in = 3 words, out = (lo, hi).
// mode 1: one block f(s) = (b + sum a_i s_i) mod p with the hot-loop MAC;
//         in = [b, a_0..a_127, s_0..s_127], out = (lo, hi).
// mode 2: out = mix(in[0]).
// mode 3: as mode 0 but only (value mod p) mod 2^n (the digest input).
// Histogram of bucket ids (the hash-table consumer's counts):
// a separate pass over the n bucket ids, privatised per block in shared memory
// when M fits (one global atomic per non-empty bucket and block), so the
// hashing kernels never contend on a few hundred global counters.
constexpr uint32_t kHistSmemMax = 12288;     // counters per block (48 KB)
__global__ void __launch_bounds__(512)
k_histogram(const uint32_t *__restrict__ buckets, uint64_t n, uint32_t M, uint32_t *__restrict__ counts) {
  extern __shared__ uint32_t h[];
  const bool priv = M <= kHistSmemMax;
  if (priv) {
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) h[i] = 0;
    __syncthreads();
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t b = __ldcs(buckets + i);
    if (priv) atomicAdd(&h[b], 1u);
    else atomicAdd(&counts[b], 1u);
  }
  if (priv) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x)
      if (h[i]) atomicAdd(&counts[i], h[i]);
  }
}

template <int BITS>
__global__ void k_selftest(int mode, const uint64_t *__restrict__ in, uint64_t n, uint64_t *__restrict__ outv) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (mode == 0) {
    const uint64_t *w = in + 3 * t;
    if constexpr (BITS == 64) {
      Acc5 x = {(uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32), (uint32_t)w[2]};
      fe_store(outv + 2 * t, reduce_acc5(x));
    } else {
      Acc3 x = {(uint32_t)w[0], (uint32_t)w[1], (uint32_t)w[2]};
      fe_store(outv + 2 * t, reduce_acc3(x));
    }
  } else if (mode == 1) {
    const uint64_t *blk = in + 257 * t;
    if constexpr (BITS == 64) {
      MacAcc64 A;
      macc_zero(A);
      for (int i = 0; i < 128; i++) mac64(A, blk[1 + i], blk[129 + i]);
      Acc5 x = macc_normalize(A);
      acc5_add_u64(x, blk[0]);
      fe_store(outv + 2 * t, reduce_acc5(x));
    } else {
      Acc3 A = {0, 0, 0};
      for (int i = 0; i < 128; i++) mac32(A, (uint32_t)blk[1 + i], (uint32_t)blk[129 + i]);
      acc3_add_u64(A, blk[0]);
      fe_store(outv + 2 * t, reduce_acc3(A));
    }
  } else if (mode == 3) {
    const uint64_t *w = in + 3 * t;
    if constexpr (BITS == 64) {
      Acc5 x = {(uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32), (uint32_t)w[2]};
      outv[2 * t] = reduce_lo_acc5(x);
    } else {
      Acc3 x = {(uint32_t)w[0], (uint32_t)w[1], (uint32_t)w[2]};
      outv[2 * t] = reduce_lo_acc3(x);
    }
    outv[2 * t + 1] = 0;
  } else {
    outv[2 * t] = BITS == 64 ? mix64(in[t]) : mix32((uint32_t)in[t]);
    outv[2 * t + 1] = 0;
  }
}

}  // namespace pmp
