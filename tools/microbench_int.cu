// microbench_int.cu -- sm_100a integer pipe throughput for the PM+ hot loop.
//
// Measures warp-instructions per cycle per SM for the SASS opcodes the PM+
// multiply-accumulate compiles to ("measure the IMAD.WIDE issue
// rate first"): IMAD.WIDE.U32 with carry-out (mad.lo.cc/madc.hi.cc pair),
// IMAD.WIDE.U32 without carry, IADD3/IADD3.X, SHF.R.W (funnel shift), LDS.
// Each thread runs 8 independent chains so latency is hidden; the grid fills
// every SM.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// microbench_int.cu -o mb && ./mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_mad_wide_cc(uint32_t *out, uint32_t a, uint32_t b) {
  uint32_t lo[8], hi[8], c[8];
  for (int j = 0; j < 8; j++) { lo[j] = threadIdx.x + j; hi[j] = j; c[j] = 0; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
                   : "+r"(lo[j]), "+r"(hi[j]), "+r"(c[j]) : "r"(a + j), "r"(b));
    }
  }
  uint32_t s = 0;
  for (int j = 0; j < 8; j++) s += lo[j] ^ hi[j] ^ c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mad_wide(uint64_t *out, uint32_t a, uint32_t b) {
  uint64_t acc[8];
  for (int j = 0; j < 8; j++) acc[j] = threadIdx.x + j;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(a + j), "r"(b + (uint32_t)it));
  }
  uint64_t s = 0;
  for (int j = 0; j < 8; j++) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_iadd3(uint32_t *out, uint32_t a, uint32_t b) {
  uint32_t x[8];
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[j]) : "r"(a ^ j));
  }
  uint32_t s = 0;
  for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_shf(uint32_t *out, uint32_t a, uint32_t b) {
  uint32_t x[8];
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) x[j] = __funnelshift_r(x[j], a + j, b);
  }
  uint32_t s = 0;
  for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double *out, uint32_t a, uint32_t b) {
  double x[8];
  const double m = 1.0 + 1e-9 * a, c = 1e-7 * b;
  for (int j = 0; j < 8; j++) x[j] = threadIdx.x + j;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[j]) : "d"(m), "d"(c));
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// one IMAD.WIDE.U32 and one DFMA per chain step: do the fma-heavy and the
// fp64 pipes overlap (sum of the two rates) or share a limit?
__global__ void k_wide_plus_dfma(double *out, uint32_t a, uint32_t b) {
  uint64_t acc[8];
  double x[8];
  const double m = 1.0 + 1e-9 * a, c = 1e-7 * b;
  for (int j = 0; j < 8; j++) { acc[j] = threadIdx.x + j; x[j] = j; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc[j]) : "r"(a + j), "r"(b + (uint32_t)it));
      asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[j]) : "d"(m), "d"(c));
    }
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += x[j] + (double)acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// u32 -> f64 via the magic-exponent trick: (2^52 | s) as bits, minus 2^52 (exact)
__global__ void k_u2d_magic(double *out, uint32_t a, uint32_t b) {
  double x[8];
  for (int j = 0; j < 8; j++) x[j] = j;
  uint32_t v = threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const double d = __hiloint2double(0x43300000, (int)(v + j * b)) - 4503599627370496.0;
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(x[j]) : "d"(d), "d"((double)a));
    }
    v += a;
  }
  double s = 0;
  for (int j = 0; j < 8; j++) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K, class T>
double run(K kern, T *buf, int blocks, int threads, int sass_per_op) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(buf, 3u, 0x9e3779b9u);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(buf, 3u, 0x9e3779b9u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  double warp_ops = (double)blocks * threads / 32 * ITERS * 8 * sass_per_op;
  double cycles = ms * 1e-3 * clk * 1e3;
  return warp_ops / cycles / sms;  // warp-instructions per cycle per SM (at max clock)
}

int main() {
  int blocks = 148 * 8, threads = 256;
  void *buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  printf("{\"unit\": \"warp-instr/cycle/SM at clocks.max\",\n");
  printf(" \"IMAD.WIDE.U32 with carry-out, + IADD3.X per 2 (mad.lo.cc/madc.hi.cc/addc)\": %.3f,\n",
         run(k_mad_wide_cc, (uint32_t *)buf, blocks, threads, 1));
  printf(" \"IMAD.WIDE.U32 (64-bit accumulate, no carry)\": %.3f,\n", run(k_mad_wide, (uint64_t *)buf, blocks, threads, 1));
  printf(" \"IADD3\": %.3f,\n", run(k_iadd3, (uint32_t *)buf, blocks, threads, 1));
  printf(" \"SHF.R.W (funnel shift)\": %.3f,\n", run(k_shf, (uint32_t *)buf, blocks, threads, 1));
  printf(" \"DFMA\": %.3f,\n", run(k_dfma, (double *)buf, blocks, threads, 1));
  printf(" \"IMAD.WIDE + DFMA pairs (pairs per cycle)\": %.3f,\n", run(k_wide_plus_dfma, (double *)buf, blocks, threads, 1));
  printf(" \"u32->f64 magic (MOV/DADD) + DFMA (per value)\": %.3f}\n", run(k_u2d_magic, (double *)buf, blocks, threads, 1));
  return 0;
}
