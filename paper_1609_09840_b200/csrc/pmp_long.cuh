// pmp_long.cuh -- one long string, block-parallel over level-2 nodes, split across callers (k_node, k_level, k_combine)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_engine.cuh"

namespace pmp {

// ============================================================= long string
// Partial tree of one long string split across callers (ranks): every level-1
// chunk value v_1 includes b_1; every level >= 2 sums a_{j,r} * child over the
// children the caller owns, without b_j.  The key-only constant C (all v_1 = 0)
// is added once in k_combine, so V = C + sum over callers ("Long
// strings: affine split").
template <int BITS>
#ifdef PMP_NODE_MINB   // (tuning build; an explicit minBlocks of 1 changes ptxas's choice: 123 -> 134 registers)
__global__ void __launch_bounds__(kWWarps * 32, PMP_NODE_MINB)
#else
__global__ void __launch_bounds__(kWWarps * 32)
#endif
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

}  // namespace pmp
