// pmp_kernels.cuh -- PM+ hot-path kernels for sm_100a.
//
// Layout of the work, one header per part:
//   pmp_common.cuh   width traits, exact-sum helpers, digest output, TMA /
//                    mbarrier / shared-memory helpers
//   pmp_short.cuh    k_short: strings <= kShortMax bytes, one thread per string,
//                    a producer warp staging 512-string tiles by TMA; one or two
//                    key schedules per pass; longer strings go to a work list
//   pmp_engine.cuh   the warp chunk engine: level-1 blocks of a string range,
//                    lane shares of the level-2 sums
//   pmp_wstring.cuh  k_wstring: the work list -- warp per big string (>= 64 KiB,
//                    TMA tile ring, streamed upper levels), then 8-lane
//                    groups per mid string; tree and two-level variant
//   pmp_long.cuh     k_node / k_level / k_combine: one long string, block-
//                    parallel over level-2 nodes, split across callers
//   pmp_stream.cuh   incremental hashing with device-resident level state
//   pmp_misc.cuh     self-test hooks, the hash-table histogram pass
//   pmp_split.cuh    one string's tree split over warps (affine split, C(T) on the device)
//   pmp_huge.cuh     k_huge: strings of many MiB in a batch, parts claimed grid-wide
//   pmp_small.cuh    k_small: the latency path for small batches (one launch)
//   pmp_short_tc.cuh k_short_tc: strings <= 64 bytes, the level-1 sum as an
//                    exact u8 x u8 -> s32 product on the tensor cores (tcgen05)
//   pmp_poly.cuh     (included by pmp_api.cu) long strings, two-level variant
//
// Citations: P:n = PAPER.md line n.  Eq. (1); Algorithm 1 P:427-443;
// byte packing P:456; reduction P:659-709; finaliser P:722-734.
#pragma once
#include "pmp_common.cuh"
#include "pmp_short.cuh"
#include "pmp_engine.cuh"
#include "pmp_wstring.cuh"
#include "pmp_long.cuh"
#include "pmp_stream.cuh"
#include "pmp_misc.cuh"
#include "pmp_split.cuh"
#include "pmp_small.cuh"
#include "pmp_huge.cuh"
#include "pmp_short_tc.cuh"
