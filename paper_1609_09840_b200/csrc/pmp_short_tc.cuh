// pmp_short_tc.cuh -- strings of <= 64 bytes with the level-1 sum on the int8 tensor cores (k_short_tc)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
//
// The level-1 sum of a short string, S = sum_t a_t s_t (Eq. (1), the
// marker word included), is a dot product of the string's words with a
// key vector that every string of the batch shares: over a tile of strings it
// is a matrix-vector product.  Written in bytes, with s_t = sum_j s_{t,j} 2^{8j}
// and a_t = sum_k a_{t,k} 2^{8k},
//     S = sum_d 2^{8d} D_d,   D_d = sum_t sum_{j+k=d} s_{t,j} a_{t,k},
// so D = X * Bk with X the (strings x bytes) matrix of the strings' bytes and Bk
// a (bytes x diagonals) matrix of key bytes -- an exact u8 x u8 -> s32 product
// (every D_d < 2^23), which tcgen05.mma kind::i8 computes on the tensor cores
// with the result in TMEM.  One MMA of M = 128 strings, K = 64 bytes, N = 32
// columns: D_0..D_14 of the 64-bit schedule (PM+64 words: j, k < 8) in columns
// 0-14 and D'_0..D'_6 of the 32-bit schedule (PM+32 words: j, k < 4) in
// columns 16-22 (dual-width pass), or one schedule in columns 0-14 / 0-6.
// What remains per string on the SM: lay its bytes out as a row (bytes, 0x01,
// zeros: the marker word is then part of the product), and afterwards sum the
// 15 + 7 diagonals into the exact S (shifts and adds) and reduce it as before.
// This moves the ~50 IMAD.WIDE per string of the word loop (k_short, the
// kernel's bound: profiles/r02/README.md) onto the tensor cores -- but the row
// pass costs about as much as they did (measured on configs[1]: 0.266 ms
// against k_short's 0.265 at the same two-block shape, and k_short's one-block
// shape reaches 0.2555), so this kernel is an option
// (pmp_set_short_tc), bit-exact and tested, not the default.
//
// Strings of 65..127 bytes in these tiles take k_short's word loop (the same
// code, in the same kernel); longer ones go to the work list as in k_short.
#pragma once
#include "pmp_short.cuh"

namespace pmp {

#ifndef PMP_TC_QUADS
#define PMP_TC_QUADS 4   // consumer warp quads per block (one M = 128 MMA per quad and tile)
#endif
#ifndef PMP_TC_RING_KB
#define PMP_TC_RING_KB 56
#endif
#ifndef PMP_TC_SLOTS
#define PMP_TC_SLOTS 4
#endif
#ifndef PMP_TC_MINB
#define PMP_TC_MINB 2
#endif
#ifndef PMP_TC_DIAG
#define PMP_TC_DIAG 0   // diagnostic builds: 1 no row pass, 2 no epilogue arithmetic, 3 neither (digests wrong)
#endif

constexpr int kTcQuads = PMP_TC_QUADS;
constexpr int kTcWarps = 4 * kTcQuads;                  // consumer warps
constexpr int kTcTile = 32 * kTcWarps;                  // strings per tile
constexpr uint32_t kTcMax = 64;                         // bytes: strings hashed on the tensor cores
constexpr int kTcSlots = PMP_TC_SLOTS, kTcOffAhead = PMP_TC_SLOTS / 2;
constexpr uint32_t kTcByteRing = PMP_TC_RING_KB * 1024;
constexpr uint32_t kTcSpanMax = kTcByteRing / 2 < 32 * 1024 ? kTcByteRing / 2 : 32 * 1024;
constexpr int kTcOffBytes = ((kTcTile + 1) * 8 + 15) & ~15;
constexpr int kTcThreads = (kTcWarps + 1) * 32;
constexpr uint32_t kTcRow = 64;                         // bytes per string row (K of the MMA)
constexpr uint32_t kTcATile = 128 * kTcRow;             // 8 KB: one quad's 128 rows
constexpr uint32_t kTcBMat = 32 * kTcRow;               // 2 KB: 32 columns of key bytes
constexpr uint32_t kTcTmemCols = kTcQuads * 64 <= 64 ? 64 : kTcQuads * 64 <= 128 ? 128 : kTcQuads * 64 <= 256 ? 256 : 512;  // 2 buffers of <= 32 columns per quad
// dynamic shared memory: [align 128] A tiles | B matrix | keys | byte ring + slack | offsets ring | headers | barriers
constexpr size_t kTcSmem = 128 + (size_t)kTcQuads * kTcATile + kTcBMat + 384 + kTcByteRing + kSlack + 16 +
                           (size_t)kTcSlots * kTcOffBytes + (size_t)kTcSlots * sizeof(TileHdr) +
                           (size_t)(3 * kTcSlots + 2 * kTcQuads) * 8 + 64;

// ---- tcgen05 helpers (PTX ISA: tcgen05 family; descriptors as the sm_100 UMMA layout)
// shared-memory matrix descriptor, K-major, no swizzle: 8-row x 16-byte core
// matrices; lbo = byte step between core matrices along K, sbo = along M/N
PMP_DI uint64_t tc_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);   // version 1 (sm_100), layout 0
}
// instruction descriptor, kind::i8: D s32, A and B unsigned 8-bit, both K-major, M = 128
template <int N> constexpr uint32_t tc_idesc_u8() {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
}
PMP_DI void tc_mma_u8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
PMP_DI void tc_commit(uint32_t mbar_s) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_s)
               : "memory");
}
PMP_DI void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
PMP_DI void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
PMP_DI void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
PMP_DI void tc_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
PMP_DI void tc_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}
PMP_DI void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
PMP_DI void sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// byte (row n, column b) of the key matrix: row n < 15 (PM+64 diagonal d = n):
// byte d - (b mod 8) of a_{b/8}; rows 16..22 of the dual pass (PM+32 diagonal
// d = n - 16): byte d - (b mod 4) of the 32-bit a_{b/4}; else 0
template <int BITS, bool DUAL>
PMP_DI uint32_t tc_key_byte(const ParamKeys &K, int n, int b) {
  if (BITS == 64 && n < 15) {
    const int k = n - (b & 7);
    return (k >= 0 && k < 8) ? (uint32_t)(K.a[b >> 3] >> (8 * k)) & 255u : 0u;
  }
  const int d = DUAL ? n - 16 : n;
  if ((DUAL || BITS == 32) && d >= 0 && d < 7) {
    const int k = d - (b & 3);
    const uint32_t a = DUAL ? K.a32[b >> 2] : (uint32_t)K.a[b >> 2];
    return (k >= 0 && k < 4) ? (a >> (8 * k)) & 255u : 0u;
  }
  return 0u;
}

// Exact S = sum_d D_d 2^{8d} from the diagonals (every D_d < 2^23), on the
// integer ALU (no multiplies): the pairs P_e = D_{2e} + D_{2e+1} 2^8 < 2^32
// need no carry, the even pairs are the limbs of E = sum P_{2f} 2^{32f}, the
// odd ones those of O = sum P_{2f+1} 2^{32f}, and S = E + O 2^16.
PMP_DI uint32_t tc_pair(uint32_t lo, uint32_t hi) {  // lo + hi * 2^8 (< 2^32 for lo, hi < 2^23)
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\tshl.b32 t, %2, 8;\n\tadd.u32 %0, %1, t;\n\t}" : "=r"(r) : "r"(lo), "r"(hi));
  return r;
}
PMP_DI Acc5 tc_sum15(const uint32_t (&d)[16]) {   // diagonals 0..14 -> S < 2^135
  const uint32_t e0 = tc_pair(d[0], d[1]), e1 = tc_pair(d[4], d[5]), e2 = tc_pair(d[8], d[9]),
                 e3 = tc_pair(d[12], d[13]);
  const uint32_t o0 = tc_pair(d[2], d[3]), o1 = tc_pair(d[6], d[7]), o2 = tc_pair(d[10], d[11]), o3 = d[14];
  Acc5 r;
  asm("{\n\t.reg .u32 s0, s1, s2, s3, s4;\n\t"
      "shl.b32 s0, %9, 16;\n\t"                 // O 2^16 as five limbs
      "shf.l.clamp.b32 s1, %9, %10, 16;\n\t"
      "shf.l.clamp.b32 s2, %10, %11, 16;\n\t"
      "shf.l.clamp.b32 s3, %11, %12, 16;\n\t"
      "shr.b32 s4, %12, 16;\n\t"
      "add.cc.u32  %0, %5, s0;\n\t"             // E + O 2^16
      "addc.cc.u32 %1, %6, s1;\n\t"
      "addc.cc.u32 %2, %7, s2;\n\t"
      "addc.cc.u32 %3, %8, s3;\n\t"
      "addc.u32    %4, s4, 0;\n\t}"
      : "=r"(r.c0), "=r"(r.c1), "=r"(r.c2), "=r"(r.c3), "=r"(r.c4)
      : "r"(e0), "r"(e1), "r"(e2), "r"(e3), "r"(o0), "r"(o1), "r"(o2), "r"(o3));
  return r;
}
PMP_DI Acc3 tc_sum7(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t x4, uint32_t x5,
                    uint32_t x6) {               // diagonals 0..6 -> S < 2^71
  const uint32_t e0 = tc_pair(x0, x1), e1 = tc_pair(x4, x5), o0 = tc_pair(x2, x3), o1 = x6;
  Acc3 r;
  asm("{\n\t.reg .u32 s0, s1, s2;\n\t"
      "shl.b32 s0, %5, 16;\n\t"
      "shf.l.clamp.b32 s1, %5, %6, 16;\n\t"
      "shr.b32 s2, %6, 16;\n\t"
      "add.cc.u32  %0, %3, s0;\n\t"
      "addc.cc.u32 %1, %4, s1;\n\t"
      "addc.u32    %2, s2, 0;\n\t}"
      : "=r"(r.c0), "=r"(r.c1), "=r"(r.c2)
      : "r"(e0), "r"(e1), "r"(o0), "r"(o1));
  return r;
}

// The row of one string of B <= 64 bytes (bytes, 0x01, zeros: P:456) at
// shared address row_s (row r of a quad's A tile: 4 chunks of 16 bytes, 128
// bytes apart).  fetch(k) = the k-th aligned 32-bit word of the region that
// starts at the word holding the first byte, sh = that byte's bit offset.
// w0, w1 = the row's first two words (the marker word when B < 8: |sigma| = 1).
// All loads are issued first (their latency overlaps), then the shifts, masks
// and stores.
template <class Fetch>
PMP_DI void tc_row(Fetch fetch, uint32_t sh, uint32_t B, uint32_t row_s, uint32_t &w0, uint32_t &w1) {
  const uint32_t cw = B >> 2;                    // the marker word's index
  uint32_t y[17];
#pragma unroll
  for (int j = 0; j < 17; j++) y[j] = fetch((uint32_t)j);
  const uint32_t m0 = fetch(cw), m1 = fetch(cw + 1);
#pragma unroll
  for (int c4 = 0; c4 < 4; c4++) {
    uint32_t v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const uint32_t c = 4 * c4 + k;
      v[k] = c < cw ? funnel(y[c], y[c + 1], sh) : 0u;   // full words; the marker word and beyond: 0 here
    }
    if (c4 == 0) {
      w0 = v[0];
      w1 = v[1];
    }
    sts_v4(row_s + 128 * c4, v[0], v[1], v[2], v[3]);
  }
  if (cw < 16) {                                 // the marker word: the last B mod 4 bytes, 0x01, zeros
    const uint32_t mb = 1u << (8 * (B & 3));
    const uint32_t mw = (funnel(m0, m1, sh) & (mb - 1)) | mb;
    sts_u32(row_s + 128 * (cw >> 2) + 4 * (cw & 3), mw);
    if (cw == 0) w0 = mw;
    if (cw == 1) w1 = mw;
  }
}

// per-string state carried from a tile's row pass to its epilogue (one tile later)
struct TcPend {
  uint32_t i;        // string index (n < 2^32)
  uint32_t B;        // bytes
  uint32_t w0, w1;   // first row words
  uint32_t flags;    // 1: tensor-core string, 2: word-loop string (digests in lo / lo32)
  uint32_t lo32;
  uint64_t lo;
};

template <int BITS, bool DUAL>
#if defined(PMP_TC_MINB)
__global__ void __launch_bounds__(kTcThreads, PMP_TC_MINB)
#else
__global__ void __launch_bounds__(kTcThreads)
#endif
k_short_tc(const ParamKeys K, const uint8_t *__restrict__ bytes, const uint64_t *__restrict__ offsets, uint64_t n,
           const OutSpec os, uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount, const OutSpec os2) {
  static_assert(BITS == 64 || !DUAL, "dual = 64-bit + 32-bit schedules");
  constexpr int kN = DUAL ? 32 : 16;             // MMA N (columns of D)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t base_s = (smem_u32(smem_raw) + 127u) & ~127u;
  uint8_t *smem = smem_raw + (base_s - smem_u32(smem_raw));
  const uint32_t a_s = base_s;                                           // kTcQuads x kTcATile
  const uint32_t bm_s = a_s + kTcQuads * kTcATile;                       // kTcBMat
  uint8_t *keys_p = smem + (bm_s - base_s) + kTcBMat;
  uint64_t *skeys = reinterpret_cast<uint64_t *>(keys_p);                // a_{1,0..31}
  uint32_t *skeys32 = reinterpret_cast<uint32_t *>(keys_p + 256);        // dual: 32-bit a_{1,0..31}
  uint8_t *ring = keys_p + 384;
  uint64_t *offs = reinterpret_cast<uint64_t *>(ring + kTcByteRing + kSlack + 16);
  TileHdr *hdr = reinterpret_cast<TileHdr *>(reinterpret_cast<uint8_t *>(offs) + (size_t)kTcSlots * kTcOffBytes);
  uint64_t *bar_off = reinterpret_cast<uint64_t *>(hdr + kTcSlots);
  uint64_t *bar_done = bar_off + kTcSlots;
  uint64_t *bar_full = bar_done + kTcSlots;
  uint64_t *bar_mma = bar_full + kTcSlots;                               // kTcQuads: MMA done
  uint64_t *bar_rows = bar_mma + kTcQuads;                               // kTcQuads: the quad's rows written
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar_rows + kTcQuads);
  if (threadIdx.x < 32) skeys[threadIdx.x] = K.a[threadIdx.x];
  if (DUAL && threadIdx.x < 32) skeys32[threadIdx.x] = K.a32[threadIdx.x];
  // the key matrix (K-major core-matrix layout: row n, byte b at
  // (n/8)*512 + (b/16)*128 + (n%8)*16 + b%16), one 32-bit word per thread step
  for (int idx = threadIdx.x; idx < (int)(kTcBMat / 4); idx += kTcThreads) {
    const int nrow = idx >> 4, b0 = (idx & 15) * 4;
    uint32_t w = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) w |= tc_key_byte<BITS, DUAL>(K, nrow, b0 + q) << (8 * q);
    sts_u32(bm_s + (nrow >> 3) * 512 + (b0 >> 4) * 128 + (nrow & 7) * 16 + (b0 & 15), w);
  }
  fence_async_smem();
  if (threadIdx.x == 0) {
    for (int q = 0; q < kTcSlots; q++) {
      mbar_init(&bar_off[q], 1);
      mbar_init(&bar_done[q], kTcWarps);
      mbar_init(&bar_full[q], 1);
    }
    for (int q = 0; q < kTcQuads; q++) {
      mbar_init(&bar_mma[q], 1);
      mbar_init(&bar_rows[q], 4);
    }
    mbar_fence_init();
  }
  if (wib == 0) {   // TMEM for the quads' accumulators (32 columns each)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTcTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t ntiles = (uint32_t)((n + kTcTile - 1) / kTcTile);
  uint32_t *const tile_ctr = wcount + 6;
  __shared__ uint32_t tids[kTcSlots];
  auto off_slot = [&](uint32_t k) { return offs + (size_t)(k & (kTcSlots - 1)) * (kTcOffBytes / 8); };

  if (wib == kTcWarps) {
    // ------------------------------------------------------------ producer warp (as k_short's)
    auto wait_done = [&](uint32_t k) { mbar_wait(&bar_done[k & (kTcSlots - 1)], (k / kTcSlots) & 1); };
    uint32_t k_end = 0xffffffffu;
    uint32_t claim = 0;
    auto issue_offs = [&](uint32_t k) {
      if (k >= kTcSlots) wait_done(k - kTcSlots);
      if (lane == 0) claim = atomicAdd(tile_ctr, 1u);
      const uint32_t t = __shfl_sync(FULL, claim, 0);
      if (t >= ntiles) {
        k_end = k;
        return;
      }
      if (lane == 0) {
        const int q = (int)(k & (kTcSlots - 1));
        tids[q] = t;
        const uint64_t base = (uint64_t)t * kTcTile;
        const uint64_t cnt = min((uint64_t)kTcTile + 1, n + 1 - base);
        const uint32_t nb = (uint32_t)((cnt * 8 + 15) & ~15ULL);
        mbar_arrive_tx(&bar_off[q], nb);
        bulk_g2s(off_slot(k), offsets + base, nb, &bar_off[q]);
      }
    };
    uint32_t head = 0, tail = 0, oldest = 0;
    __shared__ uint32_t tend[kTcSlots];
    for (uint32_t k = 0; k < (uint32_t)kTcOffAhead && k_end == 0xffffffffu; k++) issue_offs(k);
    for (uint32_t k = 0;; k++) {
      const int q = (int)(k & (kTcSlots - 1));
      if (k == k_end) {
        __syncwarp();
        if (lane == 0) {
          hdr[q].mode = kModeEnd;
          mbar_arrive_tx(&bar_full[q], 0);
        }
        break;
      }
      mbar_wait(&bar_off[q], (k / kTcSlots) & 1);
      __syncwarp();
      const uint32_t tid = tids[q];
      const uint64_t base = (uint64_t)tid * kTcTile;
      const uint32_t nv = (uint32_t)min((uint64_t)kTcTile, n - base);
      const uint64_t *o = off_slot(k);
      uint32_t mode = 1, nb = 0, pos = 0;
      uintptr_t alo = 0;
      {
        const uint64_t first = o[0], endo = o[nv];
        alo = (uintptr_t)(bytes + first) & ~(uintptr_t)15;
        const uintptr_t ahi = ((uintptr_t)(bytes + endo) + 15) & ~(uintptr_t)15;
        const uint64_t span = first < endo ? (uint64_t)(ahi - alo) : 0;
        if (span <= kTcSpanMax) {
          mode = 0;
          nb = (uint32_t)span;
          uint32_t start = head;
          if ((start % kTcByteRing) + nb > kTcByteRing) start += kTcByteRing - (start % kTcByteRing);
          while (start + nb - tail > kTcByteRing) {
            wait_done(oldest);
            tail = tend[oldest & (kTcSlots - 1)];
            oldest++;
          }
          pos = start % kTcByteRing;
          head = start + nb;
        }
      }
      while (k - oldest >= (uint32_t)kTcSlots - 1) {
        wait_done(oldest);
        tail = tend[oldest & (kTcSlots - 1)];
        oldest++;
      }
      __syncwarp();
      if (lane == 0) {
        tend[q] = head;
        hdr[q].alo = (uint64_t)alo;
        hdr[q].pos = pos;
        hdr[q].mode = mode | (tid << 2);
        mbar_arrive_tx(&bar_full[q], nb);
        if (nb) bulk_g2s(ring + pos, reinterpret_cast<const void *>(alo), nb, &bar_full[q]);
      }
      __syncwarp();
      if (k_end == 0xffffffffu) issue_offs(k + kTcOffAhead);
    }
    return;
  }
  // -------------------------------------------------------------- consumer warps
  // One tile deep pipeline per quad: in iteration k the quad waits for MMA k-1
  // (its rows may then be overwritten), writes the rows of tile k, issues MMA k
  // into the other TMEM buffer and only then reads MMA k-1's result (epilogue
  // of tile k-1), so the MMA latency overlaps an epilogue and a tile wait.
  const int quad = wib >> 2, sub = wib & 3;
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t offs_s = smem_u32(offs) + 8u * (32u * wib + lane);
  const uint32_t hdr_s = smem_u32(hdr), full_s = smem_u32(bar_full), done_s = smem_u32(bar_done);
  const uint32_t mma_s = smem_u32(&bar_mma[quad]), rows_s = smem_u32(&bar_rows[quad]);
  const uint32_t r = 32u * sub + lane;                       // this thread's row of the quad's MMA
  const uint32_t aq_s = a_s + quad * kTcATile;
  const uint32_t row_s = aq_s + (r >> 3) * 512 + (r & 7) * 16;
  const uint32_t t_d = tmem_base + ((32u * sub) << 16) + 2u * kN * quad;   // lanes 32 sub.., the quad's 2 buffers
  const uint32_t ct = 32u * wib + lane;
  TcPend pend = {0, 0, 0, 0, 0, 0, 0};
  auto epilogue = [&](uint32_t kp) {             // tile kp's digests (MMA kp complete)
    const uint32_t td = t_d + (kp & 1) * kN;
    const bool tc = pend.flags & 1;
    const uint32_t B = pend.B;
    uint64_t lo = pend.lo;
    uint32_t lo32 = pend.lo32;
    if constexpr (BITS == 64) {
      uint32_t d[16];
      tc_ld16(td, d);
      uint32_t e[8];
      if constexpr (DUAL) tc_ld8(td + 16, e);
      tc_wait_ld();
#if PMP_TC_DIAG & 2
      if (tc) {
        lo = d[0] ^ pend.w0;
        if constexpr (DUAL) lo32 = e[0];
      }
      if (0) {
#else
      if (tc) {
#endif
        Acc5 x = tc_sum15(d);
        acc5_add_u64(x, K.b);
        acc5_add_u64(x, B == kTcMax ? K.a[8] : 0ull);          // B = 64: the marker word is a_8's
        const uint64_t r64 = reduce_lo_acc5(x);
        lo = B < 8 ? ((uint64_t)pend.w1 << 32) | pend.w0 : r64;   // |sigma| = 1 (reading Q2)
        if constexpr (DUAL) {
          Acc3 y = tc_sum7(e[0], e[1], e[2], e[3], e[4], e[5], e[6]);
          acc3_add_u64(y, K.b32);
          acc3_add_u64(y, B == kTcMax ? (uint64_t)K.a32[16] : 0ull);
          const uint32_t r32 = reduce_lo_acc3(y);
          lo32 = B < 4 ? pend.w0 : r32;
        }
      }
    } else {
      uint32_t e[8];
      tc_ld8(td, e);
      tc_wait_ld();
      if (tc) {
        Acc3 y = tc_sum7(e[0], e[1], e[2], e[3], e[4], e[5], e[6]);
        acc3_add_u64(y, K.b);
        acc3_add_u64(y, B == kTcMax ? K.a[16] : 0ull);
        const uint32_t r32 = reduce_lo_acc3(y);
        lo = B < 4 ? pend.w0 : r32;
      }
    }
    if (pend.flags) {
      emit<BITS, false>(os, pend.i, lo);
      if constexpr (DUAL) emit<32, false>(os2, pend.i, lo32);
    }
  };
  uint32_t k = 0;
  for (;; k++) {
    const uint32_t q = k & (kTcSlots - 1);
    mbar_wait_s(full_s + 8 * q, (k / kTcSlots) & 1);
    uint64_t ralo;
    uint32_t rpos, mode;
    lds_hdr(hdr_s + 16 * q, ralo, rpos, mode);
    if (mode == kModeEnd) break;
    const uint64_t ibase = (uint64_t)(mode >> 2) * kTcTile;
    mode &= 3;
    const uint64_t i = ibase + ct;
    const bool valid = i < n;
    uint64_t o0, o1;
    lds_u64x2(offs_s + q * kTcOffBytes, o0, o1);
    const uint64_t Bl = valid ? o1 - o0 : 0;
    const bool is_long = Bl > kShortMax;
    const unsigned longmask = __ballot_sync(FULL, is_long);
    if (longmask) {
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
    const uint32_t B = (uint32_t)Bl;
    const bool tc = valid && Bl <= kTcMax;
    const bool leg = valid && Bl > kTcMax && !is_long;     // 65..127 bytes: the word loop
    // MMA k-1 has read this quad's rows: they may be overwritten
    if (k > 0) mbar_wait_s(mma_s, (k - 1) & 1);
    uint32_t w0 = 0, w1 = 0;
    uint64_t lo = 0;
    uint32_t lo32 = 0;
    if (mode == 0) {
      const uint32_t sofs = rpos + (valid ? (uint32_t)((uintptr_t)(bytes + o0) - (uintptr_t)ralo) : 0u);
      const uint32_t pa = ring_s + (sofs & ~3u), sh = 8 * (sofs & 3);
      auto fetch = [&](uint32_t kk) { return lds_u32(pa + 4 * kk); };
#if PMP_TC_DIAG & 1
      if (tc) w0 = fetch(0);
#else
      if (tc) tc_row(fetch, sh, B, row_s, w0, w1);
#endif
      if (__any_sync(FULL, leg)) {
        const int tfm = (int)__reduce_max_sync(FULL, leg ? B / (BITS / 8) : 0u);
        if (leg) {
          auto fetchi = [&](int kk) { return lds_u32(pa + 4 * kk); };
          if constexpr (DUAL) short_tree_dual<false>(K, skeys, skeys32, B, sh, tfm, fetchi, lo, lo32);
          else lo = short_tree_lo<BITS, false>(K, skeys, B, sh, tfm, fetchi);
        }
      }
    } else {
      const uintptr_t sa = (uintptr_t)(bytes + o0), se = sa + B;
      const uintptr_t pa = sa & ~(uintptr_t)3;
      const uint32_t sh = 8 * (uint32_t)(sa & 3);
      auto fetch = [&](uint32_t kk) {
        const uintptr_t a = pa + 4 * (uintptr_t)kk;
        return (B > 0 && a < se) ? ld_u32(reinterpret_cast<const void *>(a)) : 0u;
      };
      if (tc) tc_row(fetch, sh, B, row_s, w0, w1);
      if (__any_sync(FULL, leg)) {
        const int tfm = (int)__reduce_max_sync(FULL, leg ? B / (BITS / 8) : 0u);
        if (leg) {
          auto fetchi = [&](int kk) { return fetch((uint32_t)kk); };
          if constexpr (DUAL) short_tree_dual<false>(K, skeys, skeys32, B, sh, tfm, fetchi, lo, lo32);
          else lo = short_tree_lo<BITS, false>(K, skeys, B, sh, tfm, fetchi);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_s(done_s + 8 * q);             // the ring slot is consumed
    // the warp's 32 rows are written (visible to the tensor core's async proxy);
    // when all 4 warps of the quad have arrived, one thread issues MMA k (K = 64
    // in two k32 steps) into TMEM buffer k & 1; its completion arrives on bar_mma
    fence_async_smem();
    tc_before_sync();
    __syncwarp();
    if (lane == 0) mbar_arrive_s(rows_s);
    if (sub == 0 && lane == 0) {
      mbar_wait_s(rows_s, k & 1);
      tc_after_sync();
      constexpr uint32_t idesc = tc_idesc_u8<kN>();
      const uint32_t dcol = tmem_base + 2u * kN * quad + (k & 1) * kN;
#pragma unroll
      for (uint32_t j = 0; j < 2; j++)
        tc_mma_u8(dcol, tc_sdesc(aq_s + 256 * j, 128, 512), tc_sdesc(bm_s + 256 * j, 128, 512), idesc, j);
      tc_commit(mma_s);
    }
    __syncwarp();
    if (k > 0) {
      tc_after_sync();
      epilogue(k - 1);
    }
    pend.i = (uint32_t)i;
    pend.B = B;
    pend.w0 = w0;
    pend.w1 = w1;
    pend.flags = (tc ? 1u : 0u) | (leg ? 2u : 0u);
    pend.lo = lo;
    pend.lo32 = lo32;
  }
  if (k > 0) {                                    // the last tile's epilogue
    mbar_wait_s(mma_s, (k - 1) & 1);
    tc_after_sync();
    epilogue(k - 1);
  }
  // all consumers done with TMEM: warp 0 frees it
  tc_before_sync();
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kTcWarps) : "memory");   // consumer warps only
  if (wib == 0) {
    tc_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTcTmemCols)
                 : "memory");
  }
}

}  // namespace pmp
