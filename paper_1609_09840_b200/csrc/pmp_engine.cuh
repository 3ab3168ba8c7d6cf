// pmp_engine.cuh -- the warp chunk engine (level-1 blocks and level-2 sums of one string range)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_common.cuh"

namespace pmp {

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

}  // namespace pmp
