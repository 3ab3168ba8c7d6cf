// pmp_small.cuh -- latency path for small batches (k_small): one launch, no scratch
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_engine.cuh"
#include "pmp_short.cuh"
#include "pmp_split.cuh"

namespace pmp {

// ============================================================= k_small
// A batch of n <= kSmallMax strings in ONE launch with no scratch memory and
// no host-side work besides the launch: the throughput path (k_short's TMA
// pipeline, a zeroed work list, k_wstring) costs ~20 us of fixed latency that
// dominates a call of a few thousand strings (BASELINE configs[0]: 1,000).
//   - a block takes kSmallPer consecutive strings, one lane of its warp 0 each;
//     a string of <= kShortMax bytes is hashed straight from global memory by
//     the same word loop as k_short (short_tree_lo / short_tree_dual, the
//     `direct` fetch: aligned 32-bit loads of the words overlapping the
//     string, never past its end);
//   - longer strings are listed in shared memory and hashed afterwards by the
//     block's warps, one warp per string: level-2 nodes by the warp chunk
//     engine (warp_chunks), levels >= 3 streamed bottom-up.
//     (Round 2 had 256 strings per block, so a small batch of long strings got
//     one warp per 32 of them: 4,096 x 64 KiB took 568 us, 1,024 x 256 KiB
//     2,044 us; tools/small_batches.py, profiles/r02/small_batches.txt.)
constexpr int kSmallThreads = 256;
constexpr uint64_t kSmallMax = 4096;   // strings per call routed here (pmp_api.cu)
// strings per block (at most): so that every long string of a small batch gets
// a warp of its own (a block's 8 warps), not one warp per 32 of them.  Fewer
// when the batch is small (pmp_api.cu: about two blocks per SM), so that the
// spare warps of a block split its long strings (pmp_split.cuh)
#ifndef PMP_SMALL_PER
#define PMP_SMALL_PER 8
#endif
constexpr int kSmallPer = PMP_SMALL_PER;
static_assert(kSmallPer >= 1 && kSmallPer <= 32, "warp 0 lists the block's strings");

// V mod 2^n of one string of B > kShortMax bytes hashed by one warp (every
// lane returns the value).  Keys from the device blob (b[8], a[8][128]).
template <int BITS>
__device__ __noinline__ uint64_t warp_hash_string(const uint64_t *__restrict__ blob, const uint8_t *sa, uint64_t B,
                                                  int lane) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  const uint64_t *bk = blob, *ak = blob + kL;
  const Geom gm = make_geom(B / Tr<BITS>::W + 1);
  StrView s;
  s.base = sa;
  s.g0 = 0;
  s.avail_end = B;
  s.B = B;
  s.delta = (uint32_t)((uintptr_t)sa & 15);
  LaneKeys<BITS> lk;
  lk.load(ak, lane & 7);
  if (gm.leff <= 1) {          // one level-1 block: its value is the tree value
    const ChunkOut<BITS> co = warp_chunks<BITS>(s, 0, 1, lk, bk[0], ak + kM, lane);
    return fe_lo(co.v1_first);
  }
  // levels 3..leff: the open node's exact running sum and child count per level
  Acc up[kL + 1];
  uint64_t cnt[kL + 1];
#pragma unroll
  for (int j = 0; j <= (int)kL; j++) {
    acc_zero(up[j]);
    cnt[j] = 0;
  }
  Fe root = Fe();
  for (uint64_t q = 0; q < gm.T[2]; q++) {
    const uint64_t ce = min(128 * q + 128, gm.T[1]);
    ChunkOut<BITS> co = warp_chunks<BITS, false, true>(s, 128 * q, ce, lk, bk[0], ak + kM, lane);
    acc_add_word(co.acc2, bk[1]);                       // b_2 + sum_r a_{2,r} v_1 (Eq. (1))
    Fe v = acc_reduce(co.acc2);
    // push v up: level j receives child cnt[j] of its open node
    for (int j = 3; j <= gm.leff; j++) {
      acc_mac_fe(up[j], ak[(uint64_t)(j - 1) * kM + (cnt[j] & 127)], v);
      cnt[j]++;
      if ((cnt[j] & 127) != 0 && cnt[j] != gm.T[j - 1]) break;   // node still open
      acc_add_word(up[j], bk[j - 1]);
      v = acc_reduce(up[j]);
      acc_zero(up[j]);
    }
    if (gm.leff == 2 || (q + 1 == gm.T[2])) root = v;  // the last close reaches the root
  }
  return fe_lo(root);
}

template <int BITS, bool DUAL>
__global__ void __launch_bounds__(kSmallThreads)
k_small(const ParamKeys K, const uint64_t *__restrict__ blob, const uint64_t *__restrict__ blob32,
        const uint8_t *__restrict__ bytes, const uint64_t *__restrict__ offsets, uint64_t n, const OutSpec os,
        const OutSpec os2, uint32_t per) {
  __shared__ uint64_t skeys[32];
  __shared__ uint32_t skeys32[32];
  __shared__ uint32_t longs[kSmallPer];
  __shared__ uint32_t nlong;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (wib == 0) {
    // warp 0: the block's `per` (<= kSmallPer) strings, one lane each; the
    // short ones are hashed here, the long ones listed for the block's warps
    skeys[lane] = K.a[lane];
    if (DUAL) skeys32[lane] = K.a32[lane];
    __syncwarp();
    const uint64_t i = (uint64_t)blockIdx.x * per + lane;
    const bool valid = lane < (int)per && i < n;
    const uint64_t o0 = valid ? offsets[i] : 0, B64 = valid ? offsets[i + 1] - o0 : 0;
    const bool is_short = valid && B64 <= kShortMax;
    const unsigned lm = __ballot_sync(FULL, valid && !is_short);
    if (lane == 0) nlong = (uint32_t)__popc(lm);
    if (valid && !is_short) longs[__popc(lm & ((1u << lane) - 1))] = (uint32_t)i;
    const uint32_t B = is_short ? (uint32_t)B64 : 0u;
    const int tfm = (int)__reduce_max_sync(FULL, B / (BITS / 8));
    if (is_short) {
      const uintptr_t sa = (uintptr_t)(bytes + o0), se = sa + B;
      const uintptr_t pa = sa & ~(uintptr_t)3;
      auto fetch = [&](int kk) {
        const uintptr_t a = pa + 4 * (uintptr_t)kk;
        return (B > 0 && a < se) ? ld_u32(reinterpret_cast<const void *>(a)) : 0u;
      };
      const uint32_t sh = 8 * (uint32_t)(sa & 3);
      if constexpr (DUAL) {
        uint64_t lo;
        uint32_t lo32;
        short_tree_dual<false>(K, skeys, skeys32, B, sh, tfm, fetch, lo, lo32);
        emit<64>(os, i, lo);
        emit<32>(os2, i, lo32);
      } else {
        emit<BITS>(os, i, short_tree_lo<BITS, false>(K, skeys, B, sh, tfm, fetch));
      }
    }
  }
  __syncthreads();
  const uint32_t nl = nlong;
  if (nl == 0) return;
  constexpr int nw = kSmallThreads / 32;
  if (nl >= (uint32_t)nw) {
    // the block's long strings, one warp each
    for (uint32_t j = (uint32_t)wib; j < nl; j += nw) {
      const uint32_t si = longs[j];
      const uint64_t a0 = offsets[si], len = offsets[si + 1] - a0;
      if constexpr (DUAL) {
        const uint64_t lo = warp_hash_string<64>(blob, bytes + a0, len, lane);
        const uint64_t lo32 = warp_hash_string<32>(blob32, bytes + a0, len, lane);
        if (lane == 0) {
          emit<64>(os, si, lo);
          emit<32>(os2, si, lo32);
        }
      } else {
        const uint64_t lo = warp_hash_string<BITS>(blob, bytes + a0, len, lane);
        if (lane == 0) emit<BITS>(os, si, lo);
      }
    }
    return;
  }
  // fewer long strings than warps: string js = w mod nl gets the nsub warps
  // w = js, js + nl, ...; a string of several level-2 nodes is split over them
  // by the affine identity (pmp_split.cuh: each warp sums W(q) v2'(q) over
  // every nsub-th node, the first warp adds the partials and C(T)), the others
  // are hashed by their first warp alone
  __shared__ uint64_t spart[nw][2][2];   // per warp and schedule: partial (lo, hi)
  const uint32_t js = (uint32_t)wib % nl, sub = (uint32_t)wib / nl, nsub = (nw - 1 - js) / nl + 1;
  const uint32_t si = longs[js];
  const uint64_t a0 = offsets[si], len = offsets[si + 1] - a0;
  const StrView sv = whole_string(bytes + a0, len);
  auto split_of = [&](int bits, Geom &gm) {
    gm = make_geom(len / (uint64_t)(bits / 8) + 1);
    return nsub > 1 && gm.leff >= 2 && gm.T[2] > 1;
  };
  auto part = [&](auto tag, const uint64_t *kb, int sch) {   // this warp's partial, or the whole digest
    constexpr int B2 = decltype(tag)::value;
    using Fe = typename Tr<B2>::Fe;
    Geom gm;
    if (split_of(B2, gm)) {
      const Fe v = strided_partial<B2>(kb, sv, gm, sub, nsub, lane);
      uint64_t w2[2];
      fe_store(w2, v);
      if (lane == 0) {
        spart[wib][sch][0] = w2[0];
        spart[wib][sch][1] = w2[1];
      }
    } else if (sub == 0) {
      const uint64_t lo = warp_hash_string<B2>(kb, bytes + a0, len, lane);
      if (lane == 0) emit<B2>(sch ? os2 : os, si, lo);
    }
  };
  auto combine = [&](auto tag, const uint64_t *kb, int sch) {  // first warp of a split string: V = C(T) + sum
    constexpr int B2 = decltype(tag)::value;
    using Acc = typename Tr<B2>::Acc;
    using Fe = typename Tr<B2>::Fe;
    Geom gm;
    if (sub != 0 || !split_of(B2, gm)) return;
    Acc x;
    acc_zero(x);
    acc_add_fe(x, key_only_constant<B2>(kb, gm, lane));
    for (uint32_t k = 0; k < nsub; k++) {
      Fe v;
      fe_load(&spart[js + k * nl][sch][0], v);
      acc_add_fe(x, v);
    }
    if (lane == 0) emit<B2>(sch ? os2 : os, si, fe_lo(acc_reduce(x)));
  };
  if constexpr (DUAL) {
    part(std::integral_constant<int, 64>(), blob, 0);
    part(std::integral_constant<int, 32>(), blob32, 1);
  } else {
    part(std::integral_constant<int, BITS>(), blob, 0);
  }
  __syncthreads();
  if constexpr (DUAL) {
    combine(std::integral_constant<int, 64>(), blob, 0);
    combine(std::integral_constant<int, 32>(), blob32, 1);
  } else {
    combine(std::integral_constant<int, BITS>(), blob, 0);
  }
}

}  // namespace pmp

namespace pmp {

// ============================================================= quality suite: collision Monte Carlo
// SURVEY 8(f2) / SPEC quality_suite collision_monte_carlo (Table 3's almost
// Delta-universality; "h mod M" stays almost universal):
// thread i draws the key schedule of seed0 + i on the device (the keygen
// contract, KeyStream: b_1 then a_{1,0..31}, the only keys a string of <= 127
// bytes touches) and hashes the fixed pair (s1, s2) with the same short-string
// path as the batch kernels; counts schedules whose digests are equal in all n
// bits, and in their low 16 / 12 / 8 bits (the bucket of a table of 2^k).
template <int BITS>
__global__ void __launch_bounds__(256)
k_collide_mc(uint64_t seed0, uint64_t nsched, const uint8_t *__restrict__ s1, uint32_t len1,
             const uint8_t *__restrict__ s2, uint32_t len2, uint64_t *__restrict__ dig1,
             uint64_t *__restrict__ dig2, unsigned long long *__restrict__ counts) {
  __shared__ unsigned long long bc[4];
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsched) {
    KeyStream g;
    g.init(seed0 + i, BITS);
    ParamKeys K;
    K.b = g.draw_b();
#pragma unroll
    for (int t = 0; t < 32; t++) K.a[t] = g.draw_a();
    auto one = [&](const uint8_t *sp, uint32_t B) -> uint64_t {
      const uintptr_t sa = (uintptr_t)sp, se = sa + B, pa = sa & ~(uintptr_t)3;
      auto fetch = [&](int kk) {
        const uintptr_t a = pa + 4 * (uintptr_t)kk;
        return (B > 0 && a < se) ? ld_u32(reinterpret_cast<const void *>(a)) : 0u;
      };
      const uint64_t lo = short_tree_lo<BITS, false>(K, K.a, B, 8 * (uint32_t)(sa & 3), (int)(B / (BITS / 8)), fetch);
      return BITS == 64 ? mix64(lo) : (uint64_t)mix32((uint32_t)lo);
    };
    const uint64_t d1 = one(s1, len1), d2 = one(s2, len2);
    if (dig1) dig1[i] = d1;
    if (dig2) dig2[i] = d2;
    const uint64_t x = d1 ^ d2;
    if (x == 0) atomicAdd(&bc[0], 1ull);
    if ((x & 0xFFFF) == 0) atomicAdd(&bc[1], 1ull);
    if ((x & 0xFFF) == 0) atomicAdd(&bc[2], 1ull);
    if ((x & 0xFF) == 0) atomicAdd(&bc[3], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < 4 && bc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], bc[threadIdx.x]);
}

}  // namespace pmp
