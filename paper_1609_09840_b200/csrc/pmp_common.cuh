// pmp_common.cuh -- width traits, exact-sum helpers, digest output, TMA / mbarrier / shared-memory helpers
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include <stdint.h>
#include <type_traits>
#include "pmp_arith.cuh"

namespace pmp {

constexpr uint32_t kShortMax = 127;      // bytes; k_short handles B <= kShortMax
constexpr uint32_t kBigBytes = 1u << 16; // work-list class "big" (processed first)
// k_short block shape (round-2 measurements, profiles/r02/s_block_shape_w31.txt):
// ONE block per SM of 31 consumer warps + the producer (1024 threads, 63
// registers) with a 160 KB byte ring and 992-string tiles: configs[1]
// 0.2650 -> 0.2555 ms against two blocks of 15 + 1 warps with 72 KB rings
// (29 / 27 consumer warps: 0.2716 / 0.2585; a 128 KB ring 0.2655)
#ifndef PMP_SHORT_WARPS
#define PMP_SHORT_WARPS 31
#endif
#ifndef PMP_SHORT_RING_KB
#define PMP_SHORT_RING_KB 160
#endif
constexpr int kShortWarps = PMP_SHORT_WARPS;  // consumer warps per k_short block (+1 producer)
constexpr int kWWarps = 4;               // warps per k_wstring / k_node block
constexpr uint32_t FULL = 0xffffffffu;
// k_short word-loop granularity (words between warp-uniform exit tests)
#ifndef PMP_SHORT_G64
#define PMP_SHORT_G64 2
#endif
#ifndef PMP_SHORT_G32
#define PMP_SHORT_G32 4
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
  // throughput path: strings of >= huge_min bytes go to the huge list (at most
  // huge_cap of them; pmp_huge.cuh); huge_min = ~0: none
  uint64_t huge_min;
  uint32_t huge_cap;
};

// ------------------------------------------------------------- key-generation contract
// (reading Q12; the paper is silent): xoshiro256** seeded with 4 successive
// splitmix64 outputs of the seed; per level j = 1..8: b_j = x (x >> 32 for
// 32-bit), then a_{j,1..128} by rejection to [1, p - kappa - 1] (P:543-544,
// P:619).  Host keygen (pmp_api.cu) and the device Monte Carlo of the quality
// suite (pmp_misc.cuh) draw from this one implementation.
struct KeyStream {
  uint64_t s[4];
  uint64_t amax;
  int bits;
  PMP_HDI static uint64_t splitmix(uint64_t &x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  PMP_HDI static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  PMP_HDI void init(uint64_t seed, int out_bits) {
    bits = out_bits;
    amax = out_bits == 64 ? 0xFFFFFFFFFFFFFFF4ULL /* 2^64 - 12 */ : 0xFFFFFFF2ULL /* 2^32 - 14 */;
    uint64_t x = seed;
    for (int i = 0; i < 4; i++) s[i] = splitmix(x);
  }
  PMP_HDI uint64_t next() {  // xoshiro256**
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  PMP_HDI uint64_t draw_b() {
    const uint64_t x = next();
    return bits == 64 ? x : (x >> 32);
  }
  PMP_HDI uint64_t draw_a() {
    uint64_t x;
    do {
      x = next();
      if (bits == 32) x >>= 32;
    } while (x == 0 || x > amax);
    return x;
  }
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
// BKT = false: digests only, the bucket code compiled out (the hot k_short
// instantiations: a 64-bit modulo by a runtime M in the kernel costs the
// configs[1] kernel 0.7% even when it never runs)
template <int BITS, bool BKT = true> PMP_DI void emit(const OutSpec &os, uint64_t i, uint64_t lo) {
  if constexpr (!BKT) {
    store_digest<BITS>(os.out, i, lo);
    return;
  }
  if (os.M == 0) {
    store_digest<BITS>(os.out, i, lo);
    return;
  }
  const uint64_t d = BITS == 64 ? mix64(lo) : (uint64_t)mix32((uint32_t)lo);
  const uint32_t b = (uint32_t)(d % os.M);
  reinterpret_cast<uint32_t *>(os.out)[i] = b;
  if (os.counts) atomicAdd(&os.counts[b], 1u);
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

}  // namespace pmp
