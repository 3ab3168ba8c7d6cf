// pmp_wstring.cuh -- strings of > 127 bytes in a batch: warp per big string, 8-lane group per mid string (k_wstring)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_engine.cuh"

namespace pmp {

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
#ifndef PMP_W_BLOCK_WARPS
#define PMP_W_BLOCK_WARPS 4
#endif
constexpr int kWBlockWarps = PMP_W_BLOCK_WARPS;
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
#ifndef PMP_M_STAGES
#define PMP_M_STAGES 2
#endif
constexpr size_t kWSmemPerWarpMid =   // mid_phase's layout (kept in step with kMSmemPerWarp)
    ((size_t)PMP_M_STAGES * (4 * (1024 + 32) + 4 * 32 + 8) + 15) & ~(size_t)15;
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
#ifndef PMP_M_DIAG
#define PMP_M_DIAG 0
#endif
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
                                       const uint32_t *__restrict__ wlist, uint32_t *__restrict__ claims,
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
    if (lane == 0) base = atomicAdd(&claims[1], 32u);
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
      // fix-up and multiply-add of the half's 4 units.  The two-level variant
      // inlines it into both load paths, so the units stay in the registers
      // they were loaded into (its shared tail cost 16 register moves per half:
      // two-level fixed4k +3.4%); the tree variant measured 1% faster with
      // one shared tail.
#ifdef PMP_M_DUPTAIL
      constexpr bool kDupTail = PMP_M_DUPTAIL;
#else
      constexpr bool kDupTail = POLY;
#endif
      uint4 U[4];
      auto mac_half = [&](uint4 (&U)[4]) {
#if PMP_M_DIAG  // diagnostic build: the mid-phase pipeline alone (units folded by XOR, no multiply-adds)
        if constexpr (BITS == 64) {
#pragma unroll
          for (int j = 0; j < 4; j++) A64.L ^= ((uint64_t)U[j].y << 32 | U[j].x) ^ ((uint64_t)U[j].w << 32 | U[j].z);
        } else {
          Acc3 A = {U[0].x ^ U[1].y ^ U[2].z ^ U[3].w, 0, 0};
          part[hp < CPG ? hp : 0] = A;
        }
        return;
#endif
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
      };
      if (aligned) {
#pragma unroll
        for (int j = 0; j < 4; j++)
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(U[j].x), "=r"(U[j].y), "=r"(U[j].z), "=r"(U[j].w) : "r"(ub + 128 * (4 * hp + j)));
        if constexpr (kDupTail) mac_half(U);
      } else {
        const uint32_t a0 = ub + (delta & ~3u), sh = 8 * (delta & 3);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const uint32_t a = a0 + 128 * (4 * hp + j);
          const uint32_t y0 = lds_u32(a), y1 = lds_u32(a + 4), y2 = lds_u32(a + 8), y3 = lds_u32(a + 12),
                         y4 = lds_u32(a + 16);
          U[j] = make_uint4(funnel(y0, y1, sh), funnel(y1, y2, sh), funnel(y2, y3, sh), funnel(y3, y4, sh));
        }
        if constexpr (kDupTail) mac_half(U);
      }
      if constexpr (!kDupTail) mac_half(U);
      if constexpr (BITS == 64) {
        if (hp == 1) part[0] = macc_normalize(A64);
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
// The kernel body over blocks bid = 0 .. nblocks-1 of its launch; work counts
// in wcount[0..1] (mid, big), claim counters in claims[0..1] (next big string,
// next mid batch) -- one pair per key schedule when two share a launch.
template <int BITS, bool POLY>
__device__ __forceinline__ void wstring_body(const uint64_t *__restrict__ keys, const uint8_t *__restrict__ bytes,
                                             const uint64_t *__restrict__ offsets, uint64_t n, const OutSpec &os,
                                             const uint32_t *__restrict__ wlist, const uint32_t *__restrict__ wcount,
                                             uint32_t *__restrict__ claims, uint32_t bid, uint32_t nblocks) {
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
  // launched with programmatic dependent launch after k_short (pmp_api.cu): the
  // work list is k_short's output, so wait for that grid (and its memory) first
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // k_huge (programmatic dependent launch after this grid) may be scheduled
  // now: its blocks take what this persistent grid leaves free and wait there
  asm volatile("griddepcontrol.launch_dependents;");
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
  const uint32_t gw = bid * kWBlockWarps + wib, nw = nblocks * kWBlockWarps;
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
    if (lane == 0) cl_item = atomicAdd(&claims[0], 1u);
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
  mid_phase<BITS, POLY>(keys, bytes, offsets, os, wlist, claims, nmid, s_a2, s_mklo, s_mkhi, s_a1, b1, b2,
                        v1mk, wbase);
#endif
}

template <int BITS, bool POLY = false>
__global__ void __launch_bounds__(kWBlockWarps * 32, PMP_W_MINB)
k_wstring(const uint64_t *__restrict__ keys, const uint8_t *__restrict__ bytes,
          const uint64_t *__restrict__ offsets, uint64_t n, const OutSpec os,
          const uint32_t *__restrict__ wlist, uint32_t *__restrict__ wcount) {
  wstring_body<BITS, POLY>(keys, bytes, offsets, n, os, wlist, wcount, wcount + 2, blockIdx.x, gridDim.x);
}

// Both schedules of a fused two-width pass in one launch over the shared work
// list: the first half of the blocks hashes it under the 64-bit schedule, the
// second half under the 32-bit one (own claim counters wcount[2..3], [4..5]).
// One launch instead of two (an empty k_wstring launch costs ~6 us, as much as
// 2% of the configs[1] step).
template <bool POLY = false>
__global__ void __launch_bounds__(kWBlockWarps * 32, PMP_W_MINB)
k_wstring_dual(const uint64_t *__restrict__ keys64, const uint64_t *__restrict__ keys32,
               const uint8_t *__restrict__ bytes, const uint64_t *__restrict__ offsets, uint64_t n,
               const OutSpec os64, const OutSpec os32, const uint32_t *__restrict__ wlist,
               uint32_t *__restrict__ wcount) {
  const uint32_t half = gridDim.x / 2;
  if (blockIdx.x < half)
    wstring_body<64, POLY>(keys64, bytes, offsets, n, os64, wlist, wcount, wcount + 2, blockIdx.x, half);
  else
    wstring_body<32, POLY>(keys32, bytes, offsets, n, os32, wlist, wcount, wcount + 4, blockIdx.x - half,
                           gridDim.x - half);
}

}  // namespace pmp
