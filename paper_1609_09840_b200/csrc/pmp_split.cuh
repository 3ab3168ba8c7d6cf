// pmp_split.cuh -- one string's tree split over several warps on the device (the affine split of
// DESIGN.md section 7 with the key-only constant computed on the device)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_engine.cuh"

namespace pmp {

// Every level of Algorithm 1 is affine over F_p, so the tree value
// of a string of T words is
//     V = C(T) + sum_q W(q) v2'(q)  (mod p),
// where v2'(q) = sum_{c in node q} a_{2, c mod 128} v_1(c) is level-2 node q's
// sum without b_2 (Eq. (1), the b_j of the levels >= 2 omitted),
// W(q) = prod_{j=3..L_eff} a_{j, digit_{j-3}(q)} its path weight (digit k of q
// in base 128 is its ancestor's position at level k + 3), and C(T) the tree
// value with every v_1 = 0 (keys only).  The host computes the same C(T) for
// pmp_hash_long_combine (pmp_api.cu, long_constant).

// W(q) v2'(q) for level-2 node q of a string of T1 level-1 blocks and L_eff
// levels (warp-collective; every lane returns it).
template <int BITS>
PMP_DI typename Tr<BITS>::Fe node_term(const uint64_t *__restrict__ keys, const StrView &s, uint64_t T1, int leff,
                                       uint64_t q, const LaneKeys<BITS> &lk, int lane) {
  using Fe = typename Tr<BITS>::Fe;
  const uint64_t *bk = keys, *ak = keys + kL;
  const uint64_t ce = min(128 * q + 128, T1);
  const ChunkOut<BITS> co = warp_chunks<BITS, false, true>(s, 128 * q, ce, lk, bk[0], ak + kM, lane);
  Fe v = acc_reduce(co.acc2);
  uint64_t d = q;
  for (int j = 3; j <= leff; j++) {
    v = fe_mul(fe_from_word(ak[(uint64_t)(j - 1) * kM + (d & 127)], (Fe *)nullptr), v);
    d >>= 7;
  }
  return v;
}

// sum_{r < m} a_{j,r} mod p over the warp (exact, then reduced; every lane returns it)
template <int BITS>
PMP_DI typename Tr<BITS>::Fe key_prefix_sum(const uint64_t *__restrict__ aj, uint32_t m, int lane) {
  using Acc = typename Tr<BITS>::Acc;
  Acc x;
  acc_zero(x);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const uint32_t r = (uint32_t)lane + 32u * k;
    if (r < m) acc_add_word(x, aj[r]);
  }
#pragma unroll
  for (int sh = 1; sh < 32; sh <<= 1) {
    Acc y = acc_shfl_xor(x, sh);
    acc_add(x, y);
  }
  return acc_reduce(x);
}

// C(T): the root of the tree whose level-1 values are all 0.  At level j >= 2
// every node but the last of its level has 128 non-last children, so two
// values per level suffice: cf (a full node) and cl (the last node):
//   cf_j = b_j + cf_{j-1} sum_{r<128} a_{j,r},
//   cl_j = b_j + cf_{j-1} sum_{r<m-1} a_{j,r} + a_{j,m-1} cl_{j-1}   (m children).
// Warp-collective; every lane returns it.
template <int BITS>
PMP_DI typename Tr<BITS>::Fe key_only_constant(const uint64_t *__restrict__ keys, const Geom &gm, int lane) {
  using Acc = typename Tr<BITS>::Acc;
  using Fe = typename Tr<BITS>::Fe;
  const uint64_t *bk = keys, *ak = keys + kL;
  Fe cf = fe_from_word(0, (Fe *)nullptr), cl = cf;
  for (int j = 2; j <= gm.leff; j++) {
    const uint64_t *aj = ak + (uint64_t)(j - 1) * kM;
    const uint32_t m = (uint32_t)(gm.T[j - 1] - 128 * (gm.T[j] - 1));   // children of the last node
    const Fe sa = key_prefix_sum<BITS>(aj, 128, lane), sl = key_prefix_sum<BITS>(aj, m - 1, lane);
    Acc f, l;
    acc_zero(f);
    acc_zero(l);
    acc_add_word(f, bk[j - 1]);
    acc_add_word(l, bk[j - 1]);
    acc_mac_fe_full(f, sa, cf);
    acc_mac_fe_full(l, sl, cf);
    acc_mac_fe(l, aj[m - 1], cl);
    cf = acc_reduce(f);
    cl = acc_reduce(l);
  }
  return cl;
}

// sum_{q = first, first + step, ...} W(q) v2'(q) over the level-2 nodes of one
// string (warp-collective; every lane returns it): one warp's share of V - C(T).
template <int BITS>
PMP_DI typename Tr<BITS>::Fe strided_partial(const uint64_t *__restrict__ keys, const StrView &s, const Geom &gm,
                                             uint64_t first, uint64_t step, int lane) {
  using Acc = typename Tr<BITS>::Acc;
  LaneKeys<BITS> lk;
  lk.load(keys + kL, lane & 7);
  Acc x;
  acc_zero(x);
  for (uint64_t q = first; q < gm.T[2]; q += step) acc_add_fe(x, node_term<BITS>(keys, s, gm.T[1], gm.leff, q, lk, lane));
  return acc_reduce(x);
}

PMP_DI StrView whole_string(const uint8_t *sa, uint64_t B) {
  StrView s;
  s.base = sa;
  s.g0 = 0;
  s.avail_end = B;
  s.B = B;
  s.delta = (uint32_t)((uintptr_t)sa & 15);
  return s;
}

}  // namespace pmp
