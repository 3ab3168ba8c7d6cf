// pmp_short.cuh -- strings of <= 127 bytes: one thread per string, warp-specialised TMA pipeline (k_short)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_common.cuh"
#include "pmp_huge_list.cuh"

namespace pmp {

#ifndef PMP_SHORT_ORDER
#define PMP_SHORT_ORDER 0
#endif
#ifndef PMP_SHORT_G0
// the fused two-width loop runs its first G0 words without an exit test, then
// tests every word (0: a test every PMP_SHORT_GD words).  configs[1] (warp
// maximum 7 or 8 full words): G0 = 6 0.2462 ms, 7 0.2489, 5 0.2503, 4 0.2547,
// 3 0.2582, 1 0.2665, against 0.2508 for a test every 8 words
// (profiles/r02/s_loop_g0.txt)
#define PMP_SHORT_G0 6
#endif
#ifndef PMP_SHORT_G0_64
// single-width loops (bucket mode, --separate-widths, the two-level variant's
// single schedule, k_small): the first G0 words untested, then a test per word
// (0: a test every kShortG64 / kShortG32 words).  configs[1] separate widths:
// 0.3859 -> 0.3822 ms with 6 / 13 (5 / 12: 0.3816-0.3822, 7 / 14: 0.3851;
// profiles/r02/s_loop_g0.txt)
#define PMP_SHORT_G0_64 6
#endif
#ifndef PMP_SHORT_G0_32
#define PMP_SHORT_G0_32 13
#endif
#ifndef PMP_SHORT_STATIC_FIRST
#define PMP_SHORT_STATIC_FIRST 0
#endif
#ifndef PMP_SHORT_ANDMASK
#define PMP_SHORT_ANDMASK 0
#endif
#ifndef PMP_SHORT_NESTED
#define PMP_SHORT_NESTED 0
#endif
#ifndef PMP_SHORT_FIN32_FIRST
#define PMP_SHORT_FIN32_FIRST 0
#endif
#ifndef PMP_SHORT_PF
#define PMP_SHORT_PF 0
#endif
#ifndef PMP_SHORT_MARKER_EARLY
#define PMP_SHORT_MARKER_EARLY 0
#endif
#ifndef PMP_SHORT_G1
#define PMP_SHORT_G1 1   // after the first G0 words, an exit test every G1 words
#endif
#ifndef PMP_SHORT_BRANCHLESS
#define PMP_SHORT_BRANCHLESS 1   // marker-word branches as selects: configs[1] 0.2691 -> 0.2652 ms
#endif

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
    auto step = [&](int t, uint32_t y1, uint32_t y2) {
      uint32_t lo = funnel(y0, y1, sh), hi = funnel(y1, y2, sh);
      y0 = y2;
      if ((uint32_t)t >= (uint32_t)tlast) lo = hi = 0;         // past this lane's full words
      mac64(A, (uint32_t)K.a[t], (uint32_t)(K.a[t] >> 32), lo, hi);  // Eq. (1), lazy
    };
#if PMP_SHORT_G0_64
    // the first PMP_SHORT_G0_64 words without exit tests, then a test per word
    if (V2 || tfull_max > 0) {
#pragma unroll
      for (int t = 0; t < 15; t++) {
        if (t >= PMP_SHORT_G0_64 && t >= tfull_max) break;    // warp-uniform
        step(t, fetch(2 * t + 1), fetch(2 * t + 2));
      }
    }
#else
#pragma unroll
    for (int tb = 0; tb < 16; tb += kShortG64) {
      if (tb >= tfull_max) break;                              // warp-uniform, once per kShortG64 words
#pragma unroll
      for (int j = 0; j < kShortG64; j++) {
        const int t = tb + j;
        if (t >= 15) break;                                    // compile-time
        step(t, fetch(2 * t + 1), fetch(2 * t + 2));
      }
    }
#endif
    const uint32_t z0 = fetch(2 * tlast), z1 = fetch(2 * tlast + 1), z2 = fetch(2 * tlast + 2);
    const uint32_t zl = funnel(z0, z1, sh), zh = funnel(z1, z2, sh);
    // bytes || 0x01 || 0: mask the half holding byte r, keep / drop the other
    const uint32_t mb = 1u << (8 * (r & 3)), wh = (((r & 4) ? zh : zl) & (mb - 1)) | mb;
    const uint64_t w = (r & 4) ? ((uint64_t)wh << 32) | zl : (uint64_t)wh;
#if PMP_SHORT_BRANCHLESS
    if constexpr (!V2) {
      mac64(A, skeys[tlast], w);
      Acc5 x = macc_normalize(A);
      acc5_add_u64(x, K.b);
      const uint64_t r = reduce_lo_acc5(x);
      return tlast == 0 ? w : r;                               // |sigma| = 1: no f_j (reading Q2)
    }
#endif
    if (!V2 && tlast == 0) return w;                           // |sigma| = 1: no f_j (reading Q2)
    mac64(A, skeys[tlast], w);
    Acc5 x = macc_normalize(A);
    acc5_add_u64(x, K.b);
    if constexpr (V2) {
      const Fe64 v0 = reduce_fe_acc5(x);
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
    auto step = [&](int t, uint32_t y1) {
      uint32_t w = funnel(y0, y1, sh);
      y0 = y1;
      if ((uint32_t)t >= (uint32_t)tlast) w = 0;
      mac32(A, (uint32_t)K.a[t], w);
    };
#if PMP_SHORT_G0_32
    // the first PMP_SHORT_G0_32 words without exit tests, then a test per word
    if (V2 || tfull_max > 0) {
#pragma unroll
      for (int t = 0; t < 31; t++) {
        if (t >= PMP_SHORT_G0_32 && t >= tfull_max) break;    // warp-uniform
        step(t, fetch(t + 1));
      }
    }
#else
#pragma unroll
    for (int tb = 0; tb < 32; tb += kShortG32) {
      if (tb >= tfull_max) break;                              // warp-uniform, once per kShortG32 words
#pragma unroll
      for (int j = 0; j < kShortG32; j++) {
        const int t = tb + j;
        if (t >= 31) break;
        step(t, fetch(t + 1));
      }
    }
#endif
    const uint32_t z0 = fetch(tlast), z1 = fetch(tlast + 1);
    uint32_t w = funnel(z0, z1, sh);
    w = (w & ((1u << (8 * r)) - 1)) | (1u << (8 * r));
#if PMP_SHORT_BRANCHLESS
    if constexpr (!V2) {
      mac32(A, (uint32_t)skeys[tlast], w);
      acc3_add_u64(A, K.b);
      const uint32_t r = reduce_lo_acc3(A);
      return tlast == 0 ? w : r;
    }
#endif
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
#if PMP_SHORT_MARKER_EARLY   // (tuning: the marker words' loads issued before the loop)
  const uint32_t z0 = fetch(2 * tl64), z1 = fetch(2 * tl64 + 1), z2 = fetch(2 * tl64 + 2);
#endif
  uint32_t y0 = fetch(0);
  // exit test granularity (PMP_SHORT_GD, when PMP_SHORT_G0 is 0): the warp
  // maximum is 7 or 8 full words for configs[1]; every 8 words measured 0.4%
  // faster than every 4 on the round-2 code (stable to 0.1% with the bench's
  // head start), 5% faster than every 2 (profiles/r02/s_knobs_final.txt)
#if PMP_SHORT_DIAG >= 3 && PMP_SHORT_DIAG <= 5   // (diagnostic builds 3-5: the loop capped, see below)
  [[maybe_unused]] constexpr int G = 4;
#else
#ifndef PMP_SHORT_GD
#define PMP_SHORT_GD 8   // exit test every 8 words (final round-2 code: 0.2649 vs 0.2660 ms for 4, 0.2787 for 2)
#endif
  [[maybe_unused]] constexpr int G = V2 ? kShortG64 : PMP_SHORT_GD;   // (the PMP_SHORT_G0 == 0 loop)
#endif
  auto step2 = [&](int t, uint32_t y1, uint32_t y2) {       // full 64-bit word t (both widths)
    const uint32_t lo = funnel(y0, y1, sh), hi = funnel(y1, y2, sh);
    y0 = y2;
    // both halves of a full 64-bit word are full PM+32 words; the one PM+32
    // word beyond them (the low half at t = tl64 when B mod 8 >= 4) is added
    // with the markers below
    const bool f64 = t < tl64;
#if PMP_SHORT_ANDMASK   // (tuning: the masks as AND with an all-ones / zero word)
    const uint32_t msk = 0u - (uint32_t)f64;
    const uint32_t lm = lo & msk, hm = hi & msk;
#else
    const uint32_t lm = f64 ? lo : 0u, hm = f64 ? hi : 0u;
#endif
    if (t < 15) {
#if PMP_SHORT_ORDER   // (tuning build: the PM+32 multiply-adds first)
      mac32(C, K.a32[2 * t], lm);
      mac32(C, K.a32[2 * t + 1], hm);
      mac64(A, (uint32_t)K.a[t], (uint32_t)(K.a[t] >> 32), lm, hm);
#else
#if PMP_SHORT_DIAG != 7   // (diagnostic builds 6 / 7: one width's loop multiply-adds left out)
      mac64(A, (uint32_t)K.a[t], (uint32_t)(K.a[t] >> 32), lm, hm);  // Eq. (1)
#endif
#if PMP_SHORT_DIAG != 6
      mac32(C, K.a32[2 * t], lm);
      mac32(C, K.a32[2 * t + 1], hm);
#endif
#endif
    }
  };
  auto step = [&](int t) { step2(t, fetch(2 * t + 1), fetch(2 * t + 2)); };
#if PMP_SHORT_G0 && !(PMP_SHORT_DIAG >= 3 && PMP_SHORT_DIAG <= 5)
  // the first PMP_SHORT_G0 words without exit tests, then a test per word
  if (V2 || tfull_max > 0) {
#if PMP_SHORT_PF   // (tuning: the tested words' loads issued one word ahead, before each test)
#pragma unroll
    for (int t = 0; t < PMP_SHORT_G0; t++) step(t);
    uint32_t n1 = fetch(2 * PMP_SHORT_G0 + 1), n2 = fetch(2 * PMP_SHORT_G0 + 2);
#pragma unroll
    for (int t = PMP_SHORT_G0; t < 15; t++) {
      if (t >= tfull_max) break;                             // warp-uniform
      const uint32_t y1 = n1, y2 = n2;
      if (t + 1 < 15) {
        n1 = fetch(2 * t + 3);
        n2 = fetch(2 * t + 4);
      }
      step2(t, y1, y2);
    }
#elif PMP_SHORT_NESTED   // (tuning: the tested words as nested ifs, t = G0, G0 + 1 only, then the loop)
#pragma unroll
    for (int t = 0; t < PMP_SHORT_G0; t++) step(t);
    if (tfull_max > PMP_SHORT_G0) {
      step(PMP_SHORT_G0);
      if (tfull_max > PMP_SHORT_G0 + 1) {
        step(PMP_SHORT_G0 + 1);
#pragma unroll
        for (int t = PMP_SHORT_G0 + 2; t < 15; t++) {
          if (t >= tfull_max) break;
          step(t);
        }
      }
    }
#else
#pragma unroll
    for (int t = 0; t < 15; t++) {
      if (t >= PMP_SHORT_G0 && (t - PMP_SHORT_G0) % PMP_SHORT_G1 == 0 && t >= tfull_max) break;  // warp-uniform
      step(t);
    }
#endif
  }
#else
#pragma unroll
  for (int tb = 0; tb < 16; tb += G) {
    if (tb >= tfull_max) break;                              // warp-uniform
#pragma unroll
    for (int j = 0; j < G; j++) {
      const int t = tb + j;
      if (t >= 16) break;                                    // compile-time
      step(t);
    }
  }
#endif
  // marker words: the 8 bytes at 8 tl64, and its half holding byte 4 tl32
#if !PMP_SHORT_MARKER_EARLY
  const uint32_t z0 = fetch(2 * tl64), z1 = fetch(2 * tl64 + 1), z2 = fetch(2 * tl64 + 2);
#endif
  const uint32_t zl = funnel(z0, z1, sh), zh = funnel(z1, z2, sh);
  // the partial 32-bit word is the PM+32 marker word, and a half of the PM+64 one
  const bool up = (B & 4) != 0;                              // B mod 8 >= 4
  const uint32_t mb = 1u << (8 * (B & 3));
  const uint32_t w32 = ((up ? zh : zl) & (mb - 1)) | mb;
  const uint64_t w = up ? ((uint64_t)w32 << 32) | zl : (uint64_t)w32;
#if PMP_SHORT_BRANCHLESS   // the marker-word branches as selects (tree pass)
  if constexpr (!V2) {
#if PMP_SHORT_FIN32_FIRST   // (tuning: the PM+32 finish first)
    mac32(C, up ? skeys32[2 * tl64] : 0u, zl);
    mac32(C, skeys32[tl32], w32);
    acc3_add_u64(C, K.b32);
    const uint32_t r32 = reduce_lo_acc3(C);
    lo32 = tl32 == 0 ? w32 : r32;
    mac64(A, skeys[tl64], w);
    Acc5 x = macc_normalize(A);
    acc5_add_u64(x, K.b);
    const uint64_t r64 = reduce_lo_acc5(x);
    lo64 = tl64 == 0 ? w : r64;
    return;
#else
    mac32(C, up ? skeys32[2 * tl64] : 0u, zl);               // the full PM+32 word 2 tl64 (key 0 if none)
    mac64(A, skeys[tl64], w);
    Acc5 x = macc_normalize(A);
    acc5_add_u64(x, K.b);
    const uint64_t r64 = reduce_lo_acc5(x);
    lo64 = tl64 == 0 ? w : r64;                              // |sigma| = 1 (reading Q2)
    mac32(C, skeys32[tl32], w32);
    acc3_add_u64(C, K.b32);
    const uint32_t r32 = reduce_lo_acc3(C);
    lo32 = tl32 == 0 ? w32 : r32;
    return;
#endif
  }
#endif
  if (up) mac32(C, skeys32[2 * tl64], zl);                   // the full PM+32 word 2 tl64 (a select here: +0.3% slower)
  if (!V2 && tl64 == 0) {
    lo64 = w;                                                // |sigma| = 1 (reading Q2)
  } else {
    mac64(A, skeys[tl64], w);
    Acc5 x = macc_normalize(A);
    acc5_add_u64(x, K.b);
    if constexpr (V2) {
      const Fe64 v0 = reduce_fe_acc5(x);
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

#ifndef PMP_SHORT_APPEND_NOINLINE
#define PMP_SHORT_APPEND_NOINLINE 0
#endif
// Long strings of a warp's 32 to the work lists (k_wstring's mid / big lists,
// k_huge's list); out of line in tuning builds (PMP_SHORT_APPEND_NOINLINE)
template <int BITS, bool DUAL>
#if PMP_SHORT_APPEND_NOINLINE
__device__ __noinline__
#else
PMP_DI
#endif
void append_long(const ParamKeys &K, uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount, uint64_t n,
                 uint64_t i, uint64_t Bl, bool is_long, int lane) {
  const unsigned lt = (1u << lane) - 1;
  // huge strings (>= K.huge_min bytes) to the huge list (k_huge) while it
  // has room (pmp_huge.cuh); the others: warp-aggregated append, big
  // strings from the back, others from the front
  const bool huge = is_long && Bl >= K.huge_min;
  const unsigned hugemask = __ballot_sync(FULL, huge);
  bool listed = is_long;
  if (hugemask) {
    uint32_t hbase = 0;
    if (lane == 0) hbase = atomicAdd(&wcount[8], (uint32_t)__popc(hugemask));
    hbase = __shfl_sync(FULL, hbase, 0);
    const uint32_t slot = hbase + __popc(hugemask & lt);
    if (huge && slot < K.huge_cap) {
      uint32_t np = (uint32_t)huge_parts_of<BITS>(Bl);
      if constexpr (DUAL) np = max(np, (uint32_t)huge_parts_of<32>(Bl));
      huge_append(wlist, n, K.huge_cap, slot, (uint32_t)i, np);
      listed = false;
    }
  }
  const bool big = listed && Bl >= kBigBytes;
  const unsigned bigmask = __ballot_sync(FULL, big), midmask = __ballot_sync(FULL, listed) & ~bigmask;
  uint32_t mbase = 0, bbase = 0;
  if (lane == 0) {
    if (midmask) mbase = atomicAdd(&wcount[0], (uint32_t)__popc(midmask));
    if (bigmask) bbase = atomicAdd(&wcount[1], (uint32_t)__popc(bigmask));
  }
  mbase = __shfl_sync(FULL, mbase, 0);
  bbase = __shfl_sync(FULL, bbase, 0);
  if (listed && !big) wlist[mbase + __popc(midmask & lt)] = (uint32_t)i;
  if (big) wlist[n - 1 - (bbase + __popc(bigmask & lt))] = (uint32_t)i;
}

// k_short: warp-specialised TMA pipeline.  A block = 1 producer warp + kShortWarps
// consumer warps, working on tiles of kTile = 32 * kShortWarps consecutive
// strings (claimed dynamically, see below).  Shared memory holds
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
constexpr int kTile = 32 * kShortWarps;                        // 992 strings per tile (31 consumer warps)
#ifndef PMP_SHORT_SLOTS
#define PMP_SHORT_SLOTS 4   // round 2 (15-warp blocks): 4 slots, offsets 2 tiles ahead, -0.8% vs 8
#endif
#ifndef PMP_SHORT_OFF_AHEAD
#define PMP_SHORT_OFF_AHEAD (PMP_SHORT_SLOTS / 2)
#endif
constexpr int kRing = PMP_SHORT_SLOTS, kOffAhead = PMP_SHORT_OFF_AHEAD;  // tile slots (power of 2), offsets prefetch
constexpr uint32_t kByteRing = PMP_SHORT_RING_KB * 1024;
// (Length sorting / partitioning of the tiles, to cut the zero-padding
// multiply-adds, was measured five ways in round 1 and with a dedicated sorter
// warp in round 2 -- 2x slower: profiles/r01f, profiles/r02/README.md.)
#ifndef PMP_SHORT_SPAN_KB
#define PMP_SHORT_SPAN_KB 64   // staged tiles up to 64 KB (992 strings of 8..64 B: ~36 KB)
#endif
constexpr uint32_t kSpanMaxTile = kByteRing / 2 < PMP_SHORT_SPAN_KB * 1024 ? kByteRing / 2 : PMP_SHORT_SPAN_KB * 1024;  // larger spans go direct
constexpr int kOffBytes = ((kTile + 1) * 8 + 15) & ~15;        // 7952
constexpr int kSlack = 144;                                    // fetch() reads <= 136 B past a start
constexpr uint32_t kModeEnd = 2;
#ifndef PMP_SHORT_DIAG
#define PMP_SHORT_DIAG 0
#endif
struct TileHdr {
  uint64_t alo;    // global address of staged byte 0
  uint32_t pos;    // ring position of staged byte 0
  uint32_t mode;   // bits 0-1: 0 staged, 1 direct; bits 2-31: tile index; kModeEnd: no more tiles
};
constexpr int kShortThreads = (kShortWarps + 1) * 32;     // consumer warps + the producer warp
constexpr size_t kShortSmem = 384 /* keys */ + kByteRing + kSlack + 16 + (size_t)kRing * kOffBytes +
                              (size_t)kRing * sizeof(TileHdr) +
                              (size_t)(3 * kRing) * 8 + 128;

#ifndef PMP_SHORT_TRACE
#define PMP_SHORT_TRACE 0
#endif
#if PMP_SHORT_TRACE  // diagnostic build: clock64 timeline of blocks 0 and 1 (pmp_trace_read)
constexpr int kTrTiles = 256;
__device__ unsigned long long g_trace[2][kShortWarps + 1][kTrTiles][4];
__device__ unsigned long long g_trace_blk[1024][3];   // per block: smid, tiles consumed, end clock
#define PMP_TR(w, k, e)                                                                   \
  do {                                                                                    \
    if (blockIdx.x < 2 && lane == 0 && (k) < (uint32_t)kTrTiles)                          \
      g_trace[blockIdx.x][(w)][(k)][(e)] = clock64();                                     \
  } while (0)
#else
#define PMP_TR(w, k, e) \
  do {                  \
  } while (0)
#endif

// DUAL: BITS = 64 and a second, 32-bit schedule in K.a32 / K.b32 whose digests go to os2
// (PMP_SHORT_MINB = min resident blocks for ptxas: 1 for the product's
// 1024-thread block (<= 64 registers either way); the earlier 512-thread
// shape used 2.  PMP_SHORT_MAXNREG: register cap, tuning only)
#ifndef PMP_SHORT_MINB
#define PMP_SHORT_MINB 1
#endif
template <int BITS, bool V2 = false, bool DUAL = false, bool BKT = false>
#if defined(PMP_SHORT_MAXNREG)
__global__ void __maxnreg__(PMP_SHORT_MAXNREG)
#elif defined(PMP_SHORT_MINB)
__global__ void __launch_bounds__(kShortThreads, PMP_SHORT_MINB)
#else
__global__ void __launch_bounds__(kShortThreads)
#endif
k_short(const ParamKeys K, const uint8_t *__restrict__ bytes, const uint64_t *__restrict__ offsets,
        uint64_t n, const OutSpec os, uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount,
        const OutSpec os2) {
  extern __shared__ __align__(128) uint8_t smem[];
  // let the dependent k_wstring grid (programmatic dependent launch) be
  // scheduled now: its blocks take SM slots as this grid's blocks retire and
  // wait in griddepcontrol.wait for this grid's completion, so the launch
  // latency of the long-string pass overlaps this grid's tail
  asm volatile("griddepcontrol.launch_dependents;");
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
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) wcount[7] = K.huge_cap;   // for k_huge (pmp_huge_list.cuh)
    for (int q = 0; q < kRing; q++) {
      mbar_init(&bar_off[q], 1);
      mbar_init(&bar_done[q], kShortWarps);
      mbar_init(&bar_full[q], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const uint32_t ntiles = (uint32_t)((n + kTile - 1) / kTile);
  // Tiles are claimed dynamically (one global counter, wcount[6]) by the
  // producer when it fetches their offsets, so blocks that run faster take more
  // tiles: a static grid-stride split left 18% of the warp slots idle at the
  // end (ncu achieved occupancy 27.8 of 34 warps).  Slot k of the ring holds
  // the block's k-th claimed tile; a failed claim ends the block (kModeEnd).
  uint32_t *const tile_ctr = wcount + 6;
  __shared__ uint32_t tids[kRing];                     // claimed tile of each slot (producer)
  auto off_slot = [&](uint32_t k) { return offs + (size_t)(k & (kRing - 1)) * (kOffBytes / 8); };

  if (wib == kShortWarps) {
    // ------------------------------------------------------------ producer warp
    auto wait_done = [&](uint32_t k) {  // tile k fully consumed
      mbar_wait(&bar_done[k & (kRing - 1)], (k / kRing) & 1);
    };
    uint32_t k_end = 0xffffffffu;            // first slot whose claim failed (warp-uniform)
    // Single-width kernels claim one call ahead: the atomic fired by one
    // issue_offs call is read by the next, so its round trip overlaps the
    // producer's other work (every fired claim is read: a call follows until a
    // claim fails); separate widths 0.420 -> 0.407 ms.  The fused dual-width
    // kernel measured 0.7% slower that way and claims when it needs the tile.
#ifdef PMP_CLAIM_AHEAD
    constexpr bool kClaimAhead = PMP_CLAIM_AHEAD;
#else
    constexpr bool kClaimAhead = !DUAL;
#endif
    // (PMP_SHORT_STATIC_FIRST: block b's first tile is tile b, claimed
    // without an atomic; later claims draw from the counter + gridDim.x)
    const uint32_t cbase = PMP_SHORT_STATIC_FIRST ? gridDim.x : 0u;
    uint32_t claim = 0;
    if (kClaimAhead && lane == 0) claim = PMP_SHORT_STATIC_FIRST ? blockIdx.x : atomicAdd(tile_ctr, 1u);
    auto issue_offs = [&](uint32_t k) {
      if (k >= kRing) wait_done(k - kRing);  // slot reuse
      if (!kClaimAhead && lane == 0)
        claim = (PMP_SHORT_STATIC_FIRST && k == 0) ? blockIdx.x : cbase + atomicAdd(tile_ctr, 1u);
      const uint32_t t = __shfl_sync(FULL, claim, 0);
      if (t >= ntiles) {
        k_end = k;
        return;
      }
      if (lane == 0) {
        if (kClaimAhead) claim = cbase + atomicAdd(tile_ctr, 1u);  // for the next call
        const int q = (int)(k & (kRing - 1));
        tids[q] = t;
        const uint64_t base = (uint64_t)t * kTile;
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
    for (uint32_t k = 0; k < (uint32_t)kOffAhead && k_end == 0xffffffffu; k++) issue_offs(k);
    for (uint32_t k = 0;; k++) {
      const int q = (int)(k & (kRing - 1));
      if (k == k_end) {                      // no more tiles: tell the consumers
        __syncwarp();
        if (lane == 0) {
          hdr[q].mode = kModeEnd;
          mbar_arrive_tx(&bar_full[q], 0);
        }
        break;
      }
      PMP_TR(kShortWarps, k, 3);
      mbar_wait(&bar_off[q], (k / kRing) & 1);
      __syncwarp();
      PMP_TR(kShortWarps, k, 0);
      const uint32_t tid = tids[q];
      const uint64_t base = (uint64_t)tid * kTile;
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
      PMP_TR(kShortWarps, k, 1);
      if (lane == 0) {
        tend[q] = head;
        hdr[q].alo = (uint64_t)alo;
        hdr[q].pos = pos;
        hdr[q].mode = mode | (tid << 2);     // the consumers' tile index
#if PMP_SHORT_DIAG == 2 || PMP_SHORT_DIAG == 4  // diagnostic build: hashing only (the byte copies skipped, ring bytes stale)
        mbar_arrive_tx(&bar_full[q], 0);
#else
        mbar_arrive_tx(&bar_full[q], nb);   // release: hdr and offsets visible to consumers
        if (nb) bulk_g2s(ring + pos, reinterpret_cast<const void *>(alo), nb, &bar_full[q]);
#endif
      }
      __syncwarp();
      PMP_TR(kShortWarps, k, 2);
      // claim + offsets of tile k + kOffAhead after tile k's bytes are on their
      // way (the claim is a global atomic round trip)
      if (k_end == 0xffffffffu) issue_offs(k + kOffAhead);
    }
    return;
  }
  // -------------------------------------------------------------- consumer warps
  // shared-window addresses computed once (the loop uses explicit ld.shared)
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t offs_s = smem_u32(offs) + 8u * (32u * wib + lane);
  const uint32_t hdr_s = smem_u32(hdr), full_s = smem_u32(bar_full), done_s = smem_u32(bar_done);
  const uint32_t ct = 32u * wib + lane;                 // consumer thread = string slot in the tile
  for (uint32_t k = 0;; k++) {
    const uint32_t q = k & (kRing - 1);
    PMP_TR(wib, k, 0);
    mbar_wait_s(full_s + 8 * q, (k / kRing) & 1);
    PMP_TR(wib, k, 1);
    uint64_t ralo;
    uint32_t rpos, mode;
    lds_hdr(hdr_s + 16 * q, ralo, rpos, mode);
    if (mode == kModeEnd) {
#if PMP_SHORT_TRACE
      if (wib == 0 && lane == 0 && blockIdx.x < 1024) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_trace_blk[blockIdx.x][0] = smid;
        g_trace_blk[blockIdx.x][1] = k;
        g_trace_blk[blockIdx.x][2] = clock64();
      }
#endif
      break;
    }
    const uint64_t ibase = (uint64_t)(mode >> 2) * kTile;
    mode &= 3;
    uint64_t i = ibase + ct;
    bool valid = i < n;
    uint64_t o0, o1;
    lds_u64x2(offs_s + q * kOffBytes, o0, o1);      // offsets[i], offsets[i+1] (slot-local)
    const uint64_t Bl = valid ? o1 - o0 : 0;
    bool is_short = Bl <= kShortMax;                 // invalid lanes: an empty string, not stored
    const bool is_long = !is_short;
    uint32_t B = (uint32_t)Bl;
    const unsigned longmask = __ballot_sync(FULL, is_long);
    if (longmask) append_long<BITS, DUAL>(K, wlist, wcount, n, i, Bl, is_long, lane);
    // warp max of the number of full words (the marker word is handled apart)
#if PMP_SHORT_DIAG >= 3 && PMP_SHORT_DIAG <= 5  // diagnostic builds: the word loop capped at 4 words (what padding costs); 5: no loop
    const int tfm = min(PMP_SHORT_DIAG == 5 ? 0 : 4, (int)__reduce_max_sync(FULL, is_short ? B / (BITS / 8) : 0u));
#else
    const int tfm = (int)__reduce_max_sync(FULL, is_short ? B / (BITS / 8) : 0u);
#endif
    if (is_short) {
      uint64_t lo;
      uint32_t lo32 = 0;
      if (mode == 0) {
        // (lanes past n read the tile's first bytes: in bounds, result not stored)
        const uint32_t sofs = rpos + (valid ? (uint32_t)((uintptr_t)(bytes + o0) - (uintptr_t)ralo) : 0u);
        const uint32_t pa = ring_s + (sofs & ~3u);
        auto fetch = [&](int kk) { return lds_u32(pa + 4 * kk); };
#if PMP_SHORT_DIAG == 1  // diagnostic build: the data pipeline alone (one shared load per string, no hashing)
        lo = fetch(0) ^ B;
        lo32 = (uint32_t)lo;
        if (0)
#endif
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
        emit<BITS, BKT>(os, i, lo);
        if constexpr (DUAL) emit<32, BKT>(os2, i, lo32);
      }
    }
    __syncwarp();
    PMP_TR(wib, k, 2);
    if (lane == 0) mbar_arrive_s(done_s + 8 * q);
  }
}

}  // namespace pmp
