// pmp_misc.cuh -- self-test hooks and the hash-table histogram pass
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_common.cuh"

namespace pmp {

// ============================================================= self-test hooks
// mode 0: reduce the exact value (w0 + w1 2^n + w2 2^2n) mod p through the
//         3->2 reduction + Algorithm 2; in = 3 words, out = (lo, hi).
// mode 1: one block f(s) = (b + sum a_i s_i) mod p with the hot-loop MAC;
//         in = [b, a_0..a_127, s_0..s_127], out = (lo, hi).
// mode 2: out = mix(in[0]).
// mode 3: as mode 0 but only (value mod p) mod 2^n (the digest input).
// Histogram of bucket ids (the hash-table consumer's counts):
// a separate pass over the n bucket ids, privatised per block in shared memory
// when M fits (one global atomic per non-empty bucket and block), so the
// hashing kernels never contend on a few hundred global counters.
constexpr uint32_t kHistSmemMax = 12288;     // counters per block (48 KB)
__global__ void __launch_bounds__(512)
k_histogram(const uint32_t *__restrict__ buckets, uint64_t n, uint32_t M, uint32_t *__restrict__ counts) {
  extern __shared__ uint32_t h[];
  const bool priv = M <= kHistSmemMax;
  if (priv) {
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) h[i] = 0;
    __syncthreads();
  }
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t b = __ldcs(buckets + i);
    if (priv) atomicAdd(&h[b], 1u);
    else atomicAdd(&counts[b], 1u);
  }
  if (priv) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x)
      if (h[i]) atomicAdd(&counts[i], h[i]);
  }
}

template <int BITS>
__global__ void k_selftest(int mode, const uint64_t *__restrict__ in, uint64_t n, uint64_t *__restrict__ outv) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  if (mode == 0) {
    const uint64_t *w = in + 3 * t;
    if constexpr (BITS == 64) {
      Acc5 x = {(uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32), (uint32_t)w[2]};
      fe_store(outv + 2 * t, reduce_acc5(x));
    } else {
      Acc3 x = {(uint32_t)w[0], (uint32_t)w[1], (uint32_t)w[2]};
      fe_store(outv + 2 * t, reduce_acc3(x));
    }
  } else if (mode == 1) {
    const uint64_t *blk = in + 257 * t;
    if constexpr (BITS == 64) {
      MacAcc64 A;
      macc_zero(A);
      for (int i = 0; i < 128; i++) mac64(A, blk[1 + i], blk[129 + i]);
      Acc5 x = macc_normalize(A);
      acc5_add_u64(x, blk[0]);
      fe_store(outv + 2 * t, reduce_acc5(x));
    } else {
      Acc3 A = {0, 0, 0};
      for (int i = 0; i < 128; i++) mac32(A, (uint32_t)blk[1 + i], (uint32_t)blk[129 + i]);
      acc3_add_u64(A, blk[0]);
      fe_store(outv + 2 * t, reduce_acc3(A));
    }
  } else if (mode == 4) {
    const uint64_t *w = in + 3 * t;
    if constexpr (BITS == 64) {
      Acc5 x = {(uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32), (uint32_t)w[2]};
      fe_store(outv + 2 * t, reduce_fe_acc5(x));
    } else {
      Acc3 x = {(uint32_t)w[0], (uint32_t)w[1], (uint32_t)w[2]};
      fe_store(outv + 2 * t, reduce_acc3(x));
    }
  } else if (mode == 3) {
    const uint64_t *w = in + 3 * t;
    if constexpr (BITS == 64) {
      Acc5 x = {(uint32_t)w[0], (uint32_t)(w[0] >> 32), (uint32_t)w[1], (uint32_t)(w[1] >> 32), (uint32_t)w[2]};
      outv[2 * t] = reduce_lo_acc5(x);
    } else {
      Acc3 x = {(uint32_t)w[0], (uint32_t)w[1], (uint32_t)w[2]};
      outv[2 * t] = reduce_lo_acc3(x);
    }
    outv[2 * t + 1] = 0;
  } else {
    outv[2 * t] = BITS == 64 ? mix64(in[t]) : mix32((uint32_t)in[t]);
    outv[2 * t + 1] = 0;
  }
}

}  // namespace pmp

namespace pmp {

// ============================================================= bucket partition
// The step after the histogram in a GPU hash join / group-by (P:87-95,
// P:188-192): string indices grouped by bucket.  k_part_scan turns the counts
// into bucket starts (exclusive prefix sums, one block); k_part_scatter places
// every index: per chunk of kPartChunk strings a block ranks its strings inside
// their buckets with shared-memory atomics, reserves one range per non-empty
// bucket with a single global atomic on the bucket's cursor, and writes the
// indices there (order inside a bucket is unspecified).  M > kHistSmemMax uses
// one global atomic per string.
#ifndef PMP_PART_PER
#define PMP_PART_PER 8
#endif
constexpr int kPartThreads = 512, kPartPer = PMP_PART_PER;
constexpr uint32_t kPartChunk = (uint32_t)kPartThreads * kPartPer;
#ifndef PMP_PART_STAGE
#define PMP_PART_STAGE 1
#endif
// buckets for the staged scatter (shared: 8 M + 6 chunk bytes); with fewer
// buckets the direct writes already form long runs (measured faster, s43)
constexpr uint32_t kPartStageMin = 128, kPartStageMax = 2048;

__global__ void __launch_bounds__(1024)
k_part_scan(uint32_t *__restrict__ counts, uint32_t M, uint64_t n, uint64_t *__restrict__ starts) {
  __shared__ uint64_t s_w[32];
  const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t seg = (M + blockDim.x - 1) / blockDim.x, b0 = min(M, t * seg), b1 = min(M, b0 + seg);
  uint64_t local = 0;
  for (uint32_t b = b0; b < b1; b++) local += counts[b];
  uint64_t incl = local;                                  // block-wide inclusive scan of the segment sums
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(FULL, incl, d);
    if ((int)lane >= d) incl += y;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint64_t x = lane < (blockDim.x >> 5) ? s_w[lane] : 0, xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, xi, d);
      if ((int)lane >= d) xi += y;
    }
    s_w[lane] = xi - x;                                   // exclusive warp offsets
  }
  __syncthreads();
  uint64_t run = s_w[w] + incl - local;
  for (uint32_t b = b0; b < b1; b++) {
    const uint32_t c = counts[b];
    starts[b] = run;
    counts[b] = (uint32_t)run;                            // becomes the bucket's cursor
    run += c;
  }
  if (t == 0) starts[M] = n;
}

__global__ void __launch_bounds__(kPartThreads)
k_part_scatter(const uint32_t *__restrict__ buckets, uint64_t n, uint32_t M, uint32_t *__restrict__ cursor,
               uint32_t *__restrict__ perm) {
  extern __shared__ uint32_t h[];
  if (M > kHistSmemMax) {                                 // many buckets: one global atomic per string
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      perm[atomicAdd(&cursor[__ldcs(buckets + i)], 1u)] = (uint32_t)i;
    return;
  }
#if PMP_PART_STAGE
  if (M >= kPartStageMin && M <= kPartStageMax) {
    // staged: the chunk's indices are first placed in shared memory in bucket
    // order (local prefix sums of the chunk's bucket sizes), then written out
    // slot by slot, so consecutive threads write consecutive positions of a
    // bucket's range instead of one scattered word each
    uint32_t *g = h + M;                                  // global base per bucket (this chunk)
    uint32_t *stage = g + M;                              // kPartChunk indices in bucket order
    uint16_t *stage_b = reinterpret_cast<uint16_t *>(stage + kPartChunk);
    __shared__ uint32_t s_wsum[kPartThreads / 32];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr uint32_t kPer = (kPartStageMax + kPartThreads - 1) / kPartThreads;
    for (uint64_t c0 = (uint64_t)blockIdx.x * kPartChunk; c0 < n; c0 += (uint64_t)gridDim.x * kPartChunk) {
      for (uint32_t b = threadIdx.x; b < M; b += blockDim.x) h[b] = 0;
      __syncthreads();
      uint32_t bk[kPartPer], rk[kPartPer];
#pragma unroll
      for (int j = 0; j < kPartPer; j++) {
        const uint64_t i = c0 + (uint64_t)j * blockDim.x + threadIdx.x;
        bk[j] = i < n ? __ldcs(buckets + i) : 0u;
        rk[j] = i < n ? atomicAdd(&h[bk[j]], 1u) : 0u;
      }
      __syncthreads();
      for (uint32_t b = threadIdx.x; b < M; b += blockDim.x)  // global ranges, in bucket order
        g[b] = h[b] ? atomicAdd(&cursor[b], h[b]) : 0u;
      // exclusive scan of h (thread t owns buckets [t kPer, (t+1) kPer)) -> local starts
      const uint32_t b0 = threadIdx.x * kPer;
      uint32_t loc = 0;
#pragma unroll
      for (uint32_t e = 0; e < kPer; e++) loc += b0 + e < M ? h[b0 + e] : 0u;
      uint32_t incl = loc;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, d);
        if ((int)lane >= d) incl += y;
      }
      if (lane == 31) s_wsum[wid] = incl;
      __syncthreads();
      uint32_t woff = 0;
      for (uint32_t w = 0; w < wid; w++) woff += s_wsum[w];
      uint32_t run = woff + incl - loc;
#pragma unroll
      for (uint32_t e = 0; e < kPer; e++)
        if (b0 + e < M) {
          const uint32_t c = h[b0 + e];
          h[b0 + e] = run;                                // local start of the bucket
          run += c;
        }
      __syncthreads();
      const uint32_t nv = (uint32_t)min((uint64_t)kPartChunk, n - c0);
#pragma unroll
      for (int j = 0; j < kPartPer; j++) {
        const uint64_t i = c0 + (uint64_t)j * blockDim.x + threadIdx.x;
        if (i < n) {
          const uint32_t sl = h[bk[j]] + rk[j];
          stage[sl] = (uint32_t)i;
          stage_b[sl] = (uint16_t)bk[j];
        }
      }
      __syncthreads();
      for (uint32_t sl = threadIdx.x; sl < nv; sl += blockDim.x) {
        const uint32_t b = stage_b[sl];
        perm[g[b] + (sl - h[b])] = stage[sl];
      }
      __syncthreads();
    }
    return;
  }
#endif
  for (uint64_t c0 = (uint64_t)blockIdx.x * kPartChunk; c0 < n; c0 += (uint64_t)gridDim.x * kPartChunk) {
    for (uint32_t b = threadIdx.x; b < M; b += blockDim.x) h[b] = 0;
    __syncthreads();
    uint32_t bk[kPartPer], rk[kPartPer];
#pragma unroll
    for (int j = 0; j < kPartPer; j++) {                  // rank inside the bucket, this chunk
      const uint64_t i = c0 + (uint64_t)j * blockDim.x + threadIdx.x;
      bk[j] = i < n ? __ldcs(buckets + i) : 0u;
      rk[j] = i < n ? atomicAdd(&h[bk[j]], 1u) : 0u;
    }
    __syncthreads();
    // one range per non-empty bucket; the reservations walk the buckets in
    // order, so a warp's atomics hit consecutive counters (measured 2.5x
    // faster than reserving from each bucket's first string, s40/s41)
    for (uint32_t b = threadIdx.x; b < M; b += blockDim.x)
      if (h[b]) h[b] = atomicAdd(&cursor[b], h[b]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPartPer; j++) {
      const uint64_t i = c0 + (uint64_t)j * blockDim.x + threadIdx.x;
      if (i < n) perm[h[bk[j]] + rk[j]] = (uint32_t)i;
    }
    __syncthreads();
  }
}

}  // namespace pmp
