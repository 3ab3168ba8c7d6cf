// pmp_huge.cuh -- huge strings of a batch, node-parallel over the whole grid (k_huge)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_split.cuh"
#include "pmp_huge_list.cuh"

namespace pmp {

// ============================================================= k_huge
// k_wstring hashes a big string with one warp (~2-5 GB/s), so a batch holding
// a few strings of many MiB is bound by those warps (8 x 4 MiB: ~1 ms).  The
// throughput path's k_short therefore lists strings of >= ParamKeys::huge_min
// bytes apart (up to huge_cap of them; beyond that they stay on the big list),
// and k_huge hashes them by parts of kHugePart bytes -- whole level-2 nodes of
// both widths -- claimed by any warp of a persistent grid:
//   part p of string h adds sum_{q in p} W(q) v2'(q) (pmp_split.cuh) to the
//   string's exact running sum (two 64-bit words, atomics with the carry
//   counted); the warp finishing the last part adds C(T), reduces
//   and stores the digest.
// Claims: each listed string owns a range of part indices (prefix sums over
// the slots, huge_ranges); a warp draws the next index from one cursor per
// schedule and finds its string by binary search over the range starts.

PMP_DI void acc_add_fe_shl64(Acc5 &x, uint64_t hi) {   // x += hi 2^64
  asm("add.cc.u32  %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32    %2, %2, 0;"
      : "+r"(x.c2), "+r"(x.c3), "+r"(x.c4)
      : "r"((uint32_t)hi), "r"((uint32_t)(hi >> 32)));
}
PMP_DI void acc_add_fe_shl64(Acc3 &x, uint64_t hi) { x.c2 += (uint32_t)hi; }   // (hi < 2^24: PM+32 parts < 2^33)

// this warp's part p of string s under one schedule, added to (st[0], st[1])
template <int BITS>
PMP_DI void huge_part(const uint64_t *__restrict__ keys, const StrView &s, uint64_t p, uint64_t *st, int lane) {
  using Acc = typename Tr<BITS>::Acc;
  const uint64_t T = s.B / Tr<BITS>::W + 1, T1 = (T + 127) / 128, T2 = (T1 + 127) / 128;
  const int leff = levels_of(T);
  const uint64_t per = kHugePart / (128 * (uint64_t)Tr<BITS>::CHUNK);
  const uint64_t q0 = p * per, q1 = min(q0 + per, T2);
  if (q0 >= q1) return;
  LaneKeys<BITS> lk;
  lk.load(keys + kL, lane & 7);
  Acc x;
  acc_zero(x);
  for (uint64_t q = q0; q < q1; q++) acc_add_fe(x, node_term<BITS>(keys, s, T1, leff, q, lk, lane));
  uint64_t w2[2];
  fe_store(w2, acc_reduce(x));
  if (lane == 0) {
    const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long *>(st), (unsigned long long)w2[0]);
    const uint64_t carry = old + w2[0] < old ? 1 : 0;
    if (w2[1] + carry) atomicAdd(reinterpret_cast<unsigned long long *>(st + 1), (unsigned long long)(w2[1] + carry));
  }
}

// the string's digest under one schedule: V = C(T) + (st[0] + st[1] 2^64) mod p
template <int BITS>
__device__ __noinline__ void huge_finish(const uint64_t *__restrict__ keys, uint64_t B, uint64_t *st, const OutSpec &os, uint32_t i,
                        int lane) {
  using Acc = typename Tr<BITS>::Acc;
  const Geom gm = make_geom(B / Tr<BITS>::W + 1);
  const uint64_t lo = atomicAdd(reinterpret_cast<unsigned long long *>(st), 0ull);
  const uint64_t hi = atomicAdd(reinterpret_cast<unsigned long long *>(st + 1), 0ull);
  Acc x;
  acc_zero(x);
  acc_add_word(x, lo);
  acc_add_fe_shl64(x, hi);
  acc_add_fe(x, key_only_constant<BITS>(keys, gm, lane));
  if (lane == 0) emit<BITS>(os, i, fe_lo(acc_reduce(x)));
}

// The huge strings' parts under one key schedule (sched 0 / 1: the first /
// second of a fused two-width pass).  Part p of string h adds
// sum_{q in p} W(q) v2'(q) to the string's exact sum; the warp finishing its
// last part adds C(T) and stores the digest.
template <int BITS>
PMP_DI void huge_pool(const uint64_t *__restrict__ keys, const uint8_t *__restrict__ bytes,
                      const uint64_t *__restrict__ offsets, uint64_t n, const OutSpec os, uint32_t *wlist,
                      uint32_t *wcount, uint32_t nh, uint64_t total, int sched) {
  const int lane = threadIdx.x & 31;
  const uint32_t *hl = huge_list(wlist, n);
  uint64_t *hst = huge_state(wlist, n, wcount[7]);
  unsigned long long *cursor = reinterpret_cast<unsigned long long *>(wcount + 10 + 2 * sched);
  for (;;) {
    unsigned long long x = 0;
    if (lane == 0) x = atomicAdd(cursor, 1ull);
    x = __shfl_sync(FULL, x, 0);
    if (x >= total) break;
    // the last slot whose first part <= x: a 32-way search (one load per lane
    // and round, ~log32(nh) dependent rounds instead of log2(nh)); invariant
    // first[lo] <= x < first[hi] (hi == nh: no bound)
    uint32_t lo = 0, hi = nh;
    while (hi - lo > 1) {
      const uint32_t step = (hi - lo + 31) / 32;
      const uint32_t h = lo + (uint32_t)lane * step;
      const bool le = h < hi && __ldcg(hst + (size_t)kHugeState * h + 5) <= x;
      const int k = 31 - __clz(__ballot_sync(FULL, le));   // lane 0 always (h = lo)
      lo += (uint32_t)k * step;
      hi = min(hi, lo + step);
    }
    uint64_t *st = hst + (size_t)kHugeState * lo;
    const uint64_t p = x - __ldcg(st + 5), np = st[4] >> 32;
    const uint32_t si = hl[lo];
    const uint64_t a0 = offsets[si], B = offsets[si + 1] - a0;
    huge_part<BITS>(keys, whole_string(bytes + a0, B), p, st + 2 * sched, lane);
    __threadfence();
    uint32_t d = 0;
    if (lane == 0) d = atomicAdd(reinterpret_cast<unsigned int *>(st + 6) + sched, 1u);
    d = __shfl_sync(FULL, d, 0);
    if (d + 1 == np) {                               // the last part: the digest
      __threadfence();
      huge_finish<BITS>(keys, B, st + 2 * sched, os, si, lane);
    }
  }
}

// Part ranges: slot h owns parts [first_h, first_h + np_h), first = the
// exclusive prefix sum of np over the slots (block 0 of k_huge; the other
// blocks wait for its flag -- the grid is one resident wave).  Returns the total.
PMP_DI uint64_t huge_ranges(uint32_t *wlist, uint64_t n, uint32_t *wcount, uint32_t nh) {
  uint64_t *hst = huge_state(wlist, n, wcount[7]);
  volatile uint32_t *flag = wcount + 9;
  unsigned long long *tot = reinterpret_cast<unsigned long long *>(wcount + 14);
  if (blockIdx.x == 0) {
    __shared__ uint64_t carry, wsum[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nh; b0 += blockDim.x) {
      const uint32_t h = b0 + threadIdx.x;
      const uint64_t np = h < nh ? hst[(size_t)kHugeState * h + 4] >> 32 : 0;
      uint64_t incl = np;
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t t = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += t;
      }
      if (lane == 31) wsum[w] = incl;
      __syncthreads();
      uint64_t before = carry;
      for (int k = 0; k < w; k++) before += wsum[k];
      if (h < nh) hst[(size_t)kHugeState * h + 5] = before + incl - np;
      __syncthreads();
      if (threadIdx.x == 0) for (int k = 0; k < nw; k++) carry += wsum[k];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *tot = carry;
      __threadfence();
      *flag = 1;
    }
    __syncthreads();
    return carry;
  }
  if (threadIdx.x == 0)
    while (*flag == 0) __nanosleep(256);
  __syncthreads();
  __threadfence();
  return *(volatile unsigned long long *)tot;
}

// k_huge: launched after k_wstring (programmatic dependent launch); returns
// at once when k_short listed no huge string.  (Calling huge_pool from
// k_wstring's warps instead saves this launch, ~1.5 us per configs[1] step,
// but its register demand made ptxas spill in k_wstring's hot loops: fixed4k
// 0.90 -> 0.85 of HBM, profiles/r02/small_batches.txt.)
constexpr int kHugeThreads = 128;                // 4 warps per block, as k_node
#ifndef PMP_HUGE_MINB
#define PMP_HUGE_MINB 4                          // 4 blocks per SM (128 registers)
#endif
template <int BITS, bool DUAL>
__global__ void __launch_bounds__(kHugeThreads, PMP_HUGE_MINB)
k_huge(const uint64_t *__restrict__ blob, const uint64_t *__restrict__ blob32, const uint8_t *__restrict__ bytes,
       const uint64_t *__restrict__ offsets, uint64_t n, const OutSpec os, const OutSpec os2, uint32_t *wlist,
       uint32_t *wcount) {
  asm volatile("griddepcontrol.wait;" ::: "memory");   // k_short (and k_wstring) complete
  const uint32_t nh = min(wcount[8], wcount[7]);
  if (nh == 0) return;
  const uint64_t total = huge_ranges(wlist, n, wcount, nh);
  huge_pool<BITS>(blob, bytes, offsets, n, os, wlist, wcount, nh, total, 0);
  if constexpr (DUAL) huge_pool<32>(blob32, bytes, offsets, n, os2, wlist, wcount, nh, total, 1);
}

}  // namespace pmp
