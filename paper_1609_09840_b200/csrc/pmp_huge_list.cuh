// pmp_huge_list.cuh -- the huge-string list of the throughput path's scratch (written by
// k_short, read by k_huge; pmp_huge.cuh)
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_common.cuh"

namespace pmp {

// scratch of the throughput path (pmp_api.cu): header of kWHeader u32 counters,
// the work list (n u32), the huge list (cap u32), the huge states (cap x
// kHugeState u64).  Header: [0] mid, [1] big, [2..5] claims, [6] k_short tile
// claims, [7] huge capacity (written by k_short), [8] huge slots taken, [9]
// k_huge's "part ranges ready" flag, [10..13] part cursor per key schedule,
// [14..15] total parts.
constexpr int kWHeader = 16;
constexpr uint64_t kHugePart = 128 * 1024;      // bytes per part: 1 level-2 node (PM+64), 2 (PM+32)
constexpr int kHugeState = 8;                    // per string: (lo, hi) x 2 schedules, parts << 32, first part, parts done x 2
PMP_HDI uint32_t *huge_list(uint32_t *wlist, uint64_t n) { return wlist + n; }
PMP_HDI uint64_t *huge_state(uint32_t *wlist, uint64_t n, uint32_t cap) {
  return reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(wlist + n + cap) + 15) & ~(uintptr_t)15);
}

// parts of a string of B bytes under one width: its level-2 nodes (Algorithm 1's
// level sizes) in groups of kHugePart bytes
template <int BITS>
PMP_HDI uint64_t huge_parts_of(uint64_t B) {
  constexpr uint64_t W = BITS / 8, chunk = 128 * W;
  const uint64_t T1 = (B / W + 1 + 127) / 128, nodes = (T1 + 127) / 128;
  const uint64_t per = kHugePart / (128 * chunk);   // nodes per part
  return (nodes + per - 1) / per;
}

// k_short: string i (>= huge_min bytes, np parts) takes huge slot `slot`
PMP_DI void huge_append(uint32_t *wlist, uint64_t n, uint32_t cap, uint32_t slot, uint32_t i, uint32_t np) {
  huge_list(wlist, n)[slot] = i;
  uint64_t *st = huge_state(wlist, n, cap) + (size_t)kHugeState * slot;
#pragma unroll
  for (int k = 0; k < 4; k++) st[k] = 0;
  st[4] = (uint64_t)np << 32;
  st[6] = 0;                    // parts done per schedule (two u32); st[5] (first part) is set by k_huge
}

}  // namespace pmp
