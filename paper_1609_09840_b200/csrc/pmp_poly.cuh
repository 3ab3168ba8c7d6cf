// pmp_poly.cuh -- the two-level variant (reading Q19):
// level 1 is PM+-Multilinear f_1 on 128-word chunks exactly as in the tree,
// level 2 is a polynomial in r over the C chunk values,
//   V = (b_2 + sum_{c<C} v_c r^(C-c)) mod p,   r = a_{2,1},
// digest = mix(V mod 2^n), for every string (T == 1 included).
//
// GPU layout of the sum.  Prefix d = (-C) mod 128 virtual zero chunks so that
// C + d = 128 Q'; chunk c sits at c' = c + d, in node q' = c' / 128 at
// position i = c' mod 128, and
//   r^(C-c) = r^(128-i) * R^(Q'-1-q'),   R = r^128.
// So a node is the tree's level-2 node with the key table a_{2,i} replaced by
// W[i] = r^(128-i) (field elements, up to 2^n + k - 1: the multiply-add takes
// the extra bit) and the node sum is weighted by R^(Q'-1-q') from a
// square ladder RP[k] = R^(2^k).  Both tables are computed on the device
// from r when the key schedule is uploaded (k_poly_setup).  The sum is linear
// in the chunk values, so any chunk-aligned split across callers adds up
// (partial + combine), exactly as the tree's affine split.
#pragma once
#include "pmp_kernels.cuh"

namespace pmp {

// (kPolyW, kPolyRP, kBlobWords and poly_pow_R live in pmp_wstring.cuh, shared
// with the batch pipeline k_wstring<BITS, true>.)

// W[i] = r^(128-i), RP[k] = R^(2^k) with R = r^128 = W[0].  One thread.
template <int BITS>
__global__ void k_poly_setup(uint64_t *blob) {
  using Fe = typename Tr<BITS>::Fe;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const Fe r = fe_from_word(blob[kL + kM], (Fe *)nullptr);  // a_{2,1}
  Fe pw = r;
  fe_store(blob + kPolyW + 2 * 127, pw);
  for (int i = 126; i >= 0; i--) {
    pw = fe_mul(pw, r);
    fe_store(blob + kPolyW + 2 * i, pw);
  }
  Fe x = pw;  // r^128
  for (uint32_t k = 0; k < kPolyLadder; k++) {
    fe_store(blob + kPolyRP + 2 * k, x);
    x = fe_mul(x, x);
  }
}

// Warp: sum over virtual nodes q' in [qf, ql] of R^(Q'-1-q') * (node sum over
// the chunks [cb, ce) it owns).  Every lane returns the same exact sum.
template <int BITS>
PMP_DI typename Tr<BITS>::Acc poly_nodes(const uint64_t *__restrict__ keys, const StrView &s, uint64_t cb,
                                         uint64_t ce, uint64_t C, uint64_t q_begin, uint64_t q_end,
                                         uint64_t q_step, const LaneKeys<BITS> &lk, int lane) {
  using Acc = typename Tr<BITS>::Acc;
  using Fe = typename Tr<BITS>::Fe;
  const uint32_t d = (uint32_t)((128 - C % 128) % 128);
  const uint64_t Qp = (C + d) / 128;
  Acc sum;
  acc_zero(sum);
  if (q_begin >= q_end) return sum;
  // The warp visits its nodes last to first, so the weight R^(Q'-1-q) grows by
  // the constant factor R^q_step per node: one multiply per node instead of a
  // ladder product of up to 17 (same value in every lane).
  const uint64_t nt = (q_end - 1 - q_begin) / q_step + 1, q_last = q_begin + (nt - 1) * q_step;
  Fe Rp = poly_pow_R<BITS>(keys, Qp - 1 - q_last);
  const Fe Rstep = nt > 1 ? poly_pow_R<BITS>(keys, q_step) : Rp;
  for (uint64_t t = nt; t-- > 0;) {
    const uint64_t q = q_begin + t * q_step;
    const uint64_t first = q * 128 >= d ? q * 128 - d : 0;
    const uint64_t lo = max(first, cb), hi = min(q * 128 + 128 - d, ce);
    if (lo < hi) {
      ChunkOut<BITS> co = warp_chunks<BITS, true, true>(s, lo, hi, lk, keys[0], keys + kPolyW, lane, d);
      Fe nv = acc_reduce(co.acc2);
      if (q + 1 < Qp) nv = fe_mul(nv, Rp);
      acc_add_fe(sum, nv);
    }
    if (t) Rp = fe_mul(Rp, Rstep);
  }
  return sum;
}

// Block-wide sum of one Acc per warp -> out[blockIdx.x] (field element pair).
template <int BITS>
PMP_DI void block_sum_store(typename Tr<BITS>::Acc x, uint64_t *__restrict__ out) {
  using Acc = typename Tr<BITS>::Acc;
  __shared__ uint32_t s_acc[32][5];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) store_acc(s_acc[wid], x);
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t;
    acc_zero(t);
    for (int w = 0; w < nw; w++) {
      Acc y;
      load_acc(s_acc[w], y);
      acc_add(t, y);
    }
    fe_store(out + 2 * blockIdx.x, acc_reduce(t));
  }
}

// Long string, chunks [cb, ce) of a string of C chunks (the caller's block-
// aligned share, bytes readable through s): warps take virtual nodes
// grid-strided; one partial per block.
template <int BITS>
__global__ void __launch_bounds__(kWWarps * 32, 4)
k_poly_node(const uint64_t *__restrict__ keys, StrView s, uint64_t cb, uint64_t ce, uint64_t C,
            uint64_t *__restrict__ block_part) {
  const int lane = threadIdx.x & 31;
  const uint32_t d = (uint32_t)((128 - C % 128) % 128);
  const uint64_t qf = (cb + d) / 128, ql = (ce - 1 + d) / 128;
  const uint64_t warp = (uint64_t)blockIdx.x * kWWarps + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kWWarps;
  typename Tr<BITS>::Acc x;
  acc_zero(x);
  if (qf + warp <= ql) {
    LaneKeys<BITS> lk;
    lk.load(keys + kL, lane & 7);
    x = poly_nodes<BITS>(keys, s, cb, ce, C, qf + warp, ql + 1, nw, lk, lane);
  }
  block_sum_store<BITS>(x, block_part);
}

// Sum of np field-element partials (+ b_2 when `final`); writes the field
// element (final == 0) or the digest mix(V mod 2^n) (final == 1).
template <int BITS>
__global__ void __launch_bounds__(256)
k_poly_sum(const uint64_t *__restrict__ keys, const uint64_t *__restrict__ parts, uint64_t np, int final,
           void *__restrict__ out) {
  using Acc = typename Tr<BITS>::Acc;
  using Fe = typename Tr<BITS>::Fe;
  __shared__ uint32_t s_acc[8][5];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Acc x;
  acc_zero(x);
  for (uint64_t i = threadIdx.x; i < np; i += blockDim.x) {
    Fe v;
    fe_load(parts + 2 * i, v);
    acc_add_fe(x, v);
  }
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {
    Acc y = acc_shfl_xor(x, m);
    acc_add(x, y);
  }
  if (lane == 0) store_acc(s_acc[wid], x);
  __syncthreads();
  if (threadIdx.x != 0) return;
  Acc t;
  acc_zero(t);
  for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
    Acc y;
    load_acc(s_acc[w], y);
    acc_add(t, y);
  }
  if (final) {
    acc_add_word(t, keys[1]);  // b_2
    store_digest<BITS>(out, 0, fe_lo(acc_reduce(t)));
  } else {
    fe_store((uint64_t *)out, acc_reduce(t));
  }
}

}  // namespace pmp
