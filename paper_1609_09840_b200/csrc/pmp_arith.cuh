// pmp_arith.cuh -- exact PM+ arithmetic on the sm_100a 32-bit integer pipes.
//
// Independent of oracle/ (shares no code); checked against it end to end.
// Citations: P:n = PAPER.md line n (arXiv:1609.09840 LaTeX), S:n = SPEC.md.
//
//  * Exact chunk sums: S = b + sum_{i<128} a_i s_i is never reduced
//    inside a chunk ("one modulo per m products").  PM+64: S < 2^135, held
//    in five 32-bit limbs; PM+32: S < 2^71, three limbs.
//  * The hot-loop accumulator is a redundant carry-save form (MacAcc64): the four
//    32x32->64 partial products of a 64x64 product go to three 64-bit
//    accumulators at weights 2^0, 2^32, 2^64, each with its own carry counter, so
//    every product is one IMAD.WIDE.U32 (carry out) + one IADD3.X, with no carry
//    chain across limbs.  Normalised to exact limbs once per lane per chunk.
//  * 3-word -> 2-word reduction: S == (w0 + k^2 w2 + k u1) + (2^n + k - u0)
//    with k w1 = u1 2^n + u0; then Algorithm 2 with the v1 = 2 branch
//    read as 2^n + v0 - k (prose P:690-691; reading Q6 -- the printed "v0 - k" is
//    a misprint).
//  * Field elements at levels >= 2 are (lo, hi) with hi in {0,1}; the
//    products a * v fit in 2n bits because a <= p - kappa - 1 (reading Q7).
//  * Finaliser: V mod 2^n = lo, then the mixer of P:722-734.
#pragma once
#include <stdint.h>

#define PMP_DI __device__ __forceinline__
#define PMP_HDI __host__ __device__ __forceinline__

namespace pmp {

constexpr uint32_t kM = 128;    // block width m (Table 2)
constexpr uint32_t kL = 8;      // levels L
constexpr uint64_t kK64 = 13;   // p = 2^64 + 13
constexpr uint64_t kK32 = 15;   // p = 2^32 + 15

// ----------------------------------------------------------------- finaliser
PMP_HDI uint64_t mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}
PMP_HDI uint32_t mix32(uint32_t z) {
  z ^= z >> 13;
  z *= 0xab3be54fU;
  z ^= z >> 16;
  return z;
}

// ----------------------------------------------------------------- PM+64
struct Fe64 {        // value lo + hi * 2^64 in [0, p), hi in {0,1}
  uint64_t lo;
  uint32_t hi;
};

struct Acc5 {        // exact value c0 + c1 2^32 + ... + c4 2^128
  uint32_t c0, c1, c2, c3, c4;
};

struct MacAcc64 {    // carry-save: L + cL 2^64 + (M + cM 2^64 + N + cN 2^64) 2^32 + (H + cH 2^64) 2^64
  uint64_t L, M, N, H;  // 64-bit so each product lands in an aligned register pair (one IMAD.WIDE.U32)
  uint32_t cL, cM, cN, cH;
};

PMP_DI void macc_zero(MacAcc64 &A) {
  A.L = A.M = A.N = A.H = 0;
  A.cL = A.cM = A.cN = A.cH = 0;
}

// A += a * s  (a, s < 2^64).  One IMAD.WIDE.U32 (carry out) per 32x32 partial
// product plus carry-counter updates (IADD3.X / IMAD.X); the four partial
// products go to four independent accumulators (no serial dependence inside a word).
#ifndef PMP_MAC_ORDER
// 1: the two products of s0, then the two of s1 (the shared operand stays in
// the operand reuse cache): configs[1] k_short 0.2555 -> 0.2548 ms, configs[2]
// k_wstring 0.7356 -> 0.7285, long string neutral, two-level configs[1] +1%
// (profiles/r02/s_mac_order.txt)
#define PMP_MAC_ORDER 1
#endif
PMP_DI void mac64(MacAcc64 &A, uint32_t a0, uint32_t a1, uint32_t s0, uint32_t s1) {
#if PMP_MAC_ORDER
  asm("{\n\t.reg .u32 l0, l1, m0, m1, n0, n1, h0, h1;\n\t"
      "mov.b64 {l0, l1}, %0;\n\t"
      "mov.b64 {m0, m1}, %1;\n\t"
      "mov.b64 {n0, n1}, %2;\n\t"
      "mov.b64 {h0, h1}, %3;\n\t"
      "mad.lo.cc.u32  l0, %8, %10, l0;\n\t"
      "madc.hi.cc.u32 l1, %8, %10, l1;\n\t"
      "addc.u32       %4, %4, 0;\n\t"
      "mad.lo.cc.u32  n0, %9, %10, n0;\n\t"
      "madc.hi.cc.u32 n1, %9, %10, n1;\n\t"
      "addc.u32       %6, %6, 0;\n\t"
      "mad.lo.cc.u32  m0, %8, %11, m0;\n\t"
      "madc.hi.cc.u32 m1, %8, %11, m1;\n\t"
      "addc.u32       %5, %5, 0;\n\t"
      "mad.lo.cc.u32  h0, %9, %11, h0;\n\t"
      "madc.hi.cc.u32 h1, %9, %11, h1;\n\t"
      "addc.u32       %7, %7, 0;\n\t"
      "mov.b64 %0, {l0, l1};\n\t"
      "mov.b64 %1, {m0, m1};\n\t"
      "mov.b64 %2, {n0, n1};\n\t"
      "mov.b64 %3, {h0, h1};\n\t}"
      : "+l"(A.L), "+l"(A.M), "+l"(A.N), "+l"(A.H), "+r"(A.cL), "+r"(A.cM), "+r"(A.cN), "+r"(A.cH)
      : "r"(a0), "r"(a1), "r"(s0), "r"(s1));
  return;
#endif
  asm("{\n\t.reg .u32 l0, l1, m0, m1, n0, n1, h0, h1;\n\t"
      "mov.b64 {l0, l1}, %0;\n\t"
      "mov.b64 {m0, m1}, %1;\n\t"
      "mov.b64 {n0, n1}, %2;\n\t"
      "mov.b64 {h0, h1}, %3;\n\t"
      "mad.lo.cc.u32  l0, %8, %10, l0;\n\t"
      "madc.hi.cc.u32 l1, %8, %10, l1;\n\t"
      "addc.u32       %4, %4, 0;\n\t"
      "mad.lo.cc.u32  m0, %8, %11, m0;\n\t"
      "madc.hi.cc.u32 m1, %8, %11, m1;\n\t"
      "addc.u32       %5, %5, 0;\n\t"
      "mad.lo.cc.u32  n0, %9, %10, n0;\n\t"
      "madc.hi.cc.u32 n1, %9, %10, n1;\n\t"
      "addc.u32       %6, %6, 0;\n\t"
      "mad.lo.cc.u32  h0, %9, %11, h0;\n\t"
      "madc.hi.cc.u32 h1, %9, %11, h1;\n\t"
      "addc.u32       %7, %7, 0;\n\t"
      "mov.b64 %0, {l0, l1};\n\t"
      "mov.b64 %1, {m0, m1};\n\t"
      "mov.b64 %2, {n0, n1};\n\t"
      "mov.b64 %3, {h0, h1};\n\t}"
      : "+l"(A.L), "+l"(A.M), "+l"(A.N), "+l"(A.H), "+r"(A.cL), "+r"(A.cM), "+r"(A.cN), "+r"(A.cH)
      : "r"(a0), "r"(a1), "r"(s0), "r"(s1));
}
PMP_DI void mac64(MacAcc64 &A, uint64_t a, uint64_t s) {
  mac64(A, (uint32_t)a, (uint32_t)(a >> 32), (uint32_t)s, (uint32_t)(s >> 32));
}

// carry-save -> exact limbs (value unchanged):
//   S = L + (M + N) 2^32 + H 2^64 + cL 2^64 + (cM + cN) 2^96 + cH 2^128
PMP_DI Acc5 macc_normalize(const MacAcc64 &A) {
  Acc5 r;
  r.c0 = (uint32_t)A.L;
  asm("add.cc.u32  %0, %5, %6;\n\t"     // c1 = L1 + M0
      "addc.cc.u32 %1, %7, %8;\n\t"     // c2 = M1 + H0 + cy
      "addc.cc.u32 %2, %9, %10;\n\t"    // c3 = H1 + cM + cy
      "addc.u32    %3, %11, 0;\n\t"     // c4 = cH + cy
      "add.cc.u32  %1, %1, %4;\n\t"     // c2 += cL
      "addc.cc.u32 %2, %2, 0;\n\t"
      "addc.u32    %3, %3, 0;\n\t"
      "add.cc.u32  %0, %0, %12;\n\t"    // c1 += N0
      "addc.cc.u32 %1, %1, %13;\n\t"    // c2 += N1 + cy
      "addc.cc.u32 %2, %2, %14;\n\t"    // c3 += cN + cy
      "addc.u32    %3, %3, 0;"
      : "=r"(r.c1), "=r"(r.c2), "=r"(r.c3), "=r"(r.c4)
      : "r"(A.cL), "r"((uint32_t)(A.L >> 32)), "r"((uint32_t)A.M), "r"((uint32_t)(A.M >> 32)),
        "r"((uint32_t)A.H), "r"((uint32_t)(A.H >> 32)), "r"(A.cM), "r"(A.cH),
        "r"((uint32_t)A.N), "r"((uint32_t)(A.N >> 32)), "r"(A.cN));
  return r;
}

PMP_DI void acc5_add(Acc5 &x, const Acc5 &y) {
  asm("add.cc.u32  %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, %6;\n\t"
      "addc.cc.u32 %2, %2, %7;\n\t"
      "addc.cc.u32 %3, %3, %8;\n\t"
      "addc.u32    %4, %4, %9;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2), "+r"(x.c3), "+r"(x.c4)
      : "r"(y.c0), "r"(y.c1), "r"(y.c2), "r"(y.c3), "r"(y.c4));
}

PMP_DI void acc5_add_u64(Acc5 &x, uint64_t v) {  // x += v (v < 2^64)
  asm("add.cc.u32  %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, %6;\n\t"
      "addc.cc.u32 %2, %2, 0;\n\t"
      "addc.cc.u32 %3, %3, 0;\n\t"
      "addc.u32    %4, %4, 0;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2), "+r"(x.c3), "+r"(x.c4)
      : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)));
}

// x += a * v for a field element v (mul_field): a*lo + (hi ? a 2^64 : 0)
PMP_DI void acc5_mac_fe(Acc5 &x, uint64_t a, const Fe64 &v) {
  uint64_t plo = a * v.lo;
  uint64_t phi = __umul64hi(a, v.lo);
  uint64_t ahi = v.hi ? a : 0ULL;
  asm("add.cc.u32  %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, %6;\n\t"
      "addc.cc.u32 %2, %2, %7;\n\t"
      "addc.cc.u32 %3, %3, %8;\n\t"
      "addc.u32    %4, %4, 0;\n\t"
      "add.cc.u32  %2, %2, %9;\n\t"
      "addc.cc.u32 %3, %3, %10;\n\t"
      "addc.u32    %4, %4, 0;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2), "+r"(x.c3), "+r"(x.c4)
      : "r"((uint32_t)plo), "r"((uint32_t)(plo >> 32)), "r"((uint32_t)phi),
        "r"((uint32_t)(phi >> 32)), "r"((uint32_t)ahi), "r"((uint32_t)(ahi >> 32)));
}

// x += a * (v0 + v1 2^64) for a 3->2-reduced value (v1 <= 2): any
// representative of v_1 mod p gives the same next-level value, so Algorithm 2
// is skipped for values that are only multiplied into the next level.
PMP_DI void acc5_mac_v01(Acc5 &x, uint64_t a, uint64_t v0, uint32_t v1) {
  const uint64_t plo = a * v0, phi = __umul64hi(a, v0);
  const uint64_t q = a * v1;                           // a v1 mod 2^64
  const uint32_t qh = v1 == 2 ? (uint32_t)(a >> 63) : 0u;
  asm("add.cc.u32  %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, %6;\n\t"
      "addc.cc.u32 %2, %2, %7;\n\t"
      "addc.cc.u32 %3, %3, %8;\n\t"
      "addc.u32    %4, %4, %11;\n\t"
      "add.cc.u32  %2, %2, %9;\n\t"
      "addc.cc.u32 %3, %3, %10;\n\t"
      "addc.u32    %4, %4, 0;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2), "+r"(x.c3), "+r"(x.c4)
      : "r"((uint32_t)plo), "r"((uint32_t)(plo >> 32)), "r"((uint32_t)phi), "r"((uint32_t)(phi >> 32)),
        "r"((uint32_t)q), "r"((uint32_t)(q >> 32)), "r"(qh));
}

PMP_DI Acc5 acc5_shfl_xor(const Acc5 &x, int m) {
  Acc5 r;
  r.c0 = __shfl_xor_sync(0xffffffffu, x.c0, m);
  r.c1 = __shfl_xor_sync(0xffffffffu, x.c1, m);
  r.c2 = __shfl_xor_sync(0xffffffffu, x.c2, m);
  r.c3 = __shfl_xor_sync(0xffffffffu, x.c3, m);
  r.c4 = __shfl_xor_sync(0xffffffffu, x.c4, m);
  return r;
}

// Section 6.2: S = w0 + w1 2^64 + w2 2^128 -> (v0, v1), v1 <= 2
PMP_HDI void reduce3to2_64(uint64_t w0, uint64_t w1, uint64_t w2, uint64_t &v0, uint32_t &v1) {
#ifdef __CUDA_ARCH__
  uint64_t u1 = __umul64hi(w1, kK64);
#else
  uint64_t u1 = (uint64_t)(((unsigned __int128)w1 * kK64) >> 64);
#endif
  uint64_t u0 = w1 * kK64;                              // k w1 = u1 2^64 + u0
  uint64_t t = kK64 * kK64 * w2 + kK64 * u1;            // k^2 w2 + k u1 (< 2^40)
  uint64_t x0 = w0 + t;                                 // X = w0 + k^2 w2 + k u1
  uint32_t x1 = x0 < t;
  uint64_t y0 = kK64 - u0;                              // Y = 2^64 + k - u0
  uint32_t y1 = u0 <= kK64;
  v0 = x0 + y0;
  v1 = x1 + y1 + (uint32_t)(v0 < x0);
}

// Algorithm 2, v1 = 2 branch corrected (reading Q6).
PMP_HDI Fe64 alg2_64(uint64_t v0, uint32_t v1) {
  Fe64 z;
  if (kK64 * v1 <= v0) {                 // line 2-3: v0 - k v1
    z.lo = v0 - kK64 * v1;
    z.hi = 0;
  } else if (v1 == 1) {                  // line 4-5: v0 + 2^n (v0 < k)
    z.lo = v0;
    z.hi = 1;
  } else {                               // v1 == 2: 2^n + v0 - k (v0 < 2k)
    z.lo = v0 - kK64;
    z.hi = v0 >= kK64;
  }
  return z;
}

// V mod 2^64 only (the digest input) of S = w0 + w1 2^64 + w2 2^128
// (w2 < 2^24), by the same congruences as Section 6.2 (2^64 = -k, 2^128 = k^2
// mod p), folded so that no 64x64 product is formed:
//   -k w1 = k ~w1 + k - k 2^64 = k ~w1 + k + k^2  (mod p),  ~w1 = 2^64 - 1 - w1,
//   so S = Y := w0 + k ~w1 + k^2 w2 + k^2 + k, with Y = y0 + y1 2^64, y1 <= 14;
//   S = y0 - k y1 (mod p), and y0 - k y1 is in [-(k^2 + k), 2^64): if it is
//   negative, V = y0 - k y1 + p and V mod 2^64 = y0 - k y1 + k (mod 2^64).
// Equal to the 3->2 reduction followed by Algorithm 2 (corrected, reading Q6)
// and taking the low word: checked on the device against the oracle
// (test_reduction_fuzz_and_algorithm2_branches, mode 3).
PMP_HDI uint64_t reduce_lo_words64(uint64_t w0, uint64_t w1, uint64_t w2) {
  const uint32_t K = (uint32_t)w2 * (uint32_t)(kK64 * kK64) + (uint32_t)(kK64 * kK64 + kK64);
  const uint64_t A = (uint64_t)(~(uint32_t)w1) * kK64 + K;            // k ~w1_lo + k^2 w2 + k^2 + k
  const uint64_t Bm = (uint64_t)(~(uint32_t)(w1 >> 32)) * kK64;       // k ~w1_hi (weight 2^32)
  uint64_t y0 = w0 + A;
  uint32_t y1 = y0 < A;
  const uint64_t bs = Bm << 32;
  y0 += bs;
  y1 += (uint32_t)(y0 < bs) + (uint32_t)(Bm >> 32);
  const uint64_t kv = kK64 * y1;
  return y0 - kv + (y0 < kv ? kK64 : 0);
}
// The same folding, returning the canonical residue V = S mod p (lo, hi):
// V = y0 - k y1 when y0 >= k y1; otherwise V = y0 - k y1 + k + 2^64, which is
// >= 2^64 (hi = 1) exactly when y0 + k >= k y1.  Used where the full value
// feeds another multiply (the two-level variant's short strings).
PMP_HDI Fe64 reduce_fe_words64(uint64_t w0, uint64_t w1, uint64_t w2) {
  const uint32_t K = (uint32_t)w2 * (uint32_t)(kK64 * kK64) + (uint32_t)(kK64 * kK64 + kK64);
  const uint64_t A = (uint64_t)(~(uint32_t)w1) * kK64 + K;
  const uint64_t Bm = (uint64_t)(~(uint32_t)(w1 >> 32)) * kK64;
  uint64_t y0 = w0 + A;
  uint32_t y1 = y0 < A;
  const uint64_t bs = Bm << 32;
  y0 += bs;
  y1 += (uint32_t)(y0 < bs) + (uint32_t)(Bm >> 32);
  const uint64_t kv = kK64 * y1;
  const bool neg = y0 < kv;
  Fe64 v;
  v.lo = y0 - kv + (neg ? kK64 : 0);
  v.hi = neg && (y0 + kK64 >= kv);
  return v;
}
PMP_HDI Fe64 reduce_fe_acc5(const Acc5 &x) {
  return reduce_fe_words64(((uint64_t)x.c1 << 32) | x.c0, ((uint64_t)x.c3 << 32) | x.c2, x.c4);
}
PMP_HDI uint64_t reduce_lo_acc5(const Acc5 &x) {
  return reduce_lo_words64(((uint64_t)x.c1 << 32) | x.c0, ((uint64_t)x.c3 << 32) | x.c2, x.c4);
}

PMP_HDI Fe64 reduce_acc5(const Acc5 &x) {
  uint64_t w0 = ((uint64_t)x.c1 << 32) | x.c0;
  uint64_t w1 = ((uint64_t)x.c3 << 32) | x.c2;
  uint64_t v0;
  uint32_t v1;
  reduce3to2_64(w0, w1, x.c4, v0, v1);
  return alg2_64(v0, v1);
}

// ----------------------------------------------------------------- PM+32
struct Acc3 {        // exact value c0 + c1 2^32 + c2 2^64
  uint32_t c0, c1, c2;
};

PMP_DI void mac32(Acc3 &A, uint32_t a, uint32_t s) {  // one IMAD.WIDE.U32 + one IADD3.X
  asm("mad.lo.cc.u32  %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
      "addc.u32       %2, %2, 0;"
      : "+r"(A.c0), "+r"(A.c1), "+r"(A.c2)
      : "r"(a), "r"(s));
}

PMP_DI void acc3_add(Acc3 &x, const Acc3 &y) {
  asm("add.cc.u32  %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32    %2, %2, %5;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2)
      : "r"(y.c0), "r"(y.c1), "r"(y.c2));
}

PMP_DI void acc3_add_u64(Acc3 &x, uint64_t v) {
  asm("add.cc.u32  %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32    %2, %2, 0;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2)
      : "r"((uint32_t)v), "r"((uint32_t)(v >> 32)));
}

// x += a * v, v < p = 2^32 + 15 held in a u64 (lo 32 bits + hi bit)
PMP_DI void acc3_mac_fe(Acc3 &x, uint32_t a, uint64_t v) {
  uint64_t prod = (uint64_t)a * (uint32_t)v;
  uint32_t ahi = (v >> 32) ? a : 0u;
  asm("add.cc.u32  %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32    %2, %2, 0;\n\t"
      "add.cc.u32  %1, %1, %5;\n\t"
      "addc.u32    %2, %2, 0;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2)
      : "r"((uint32_t)prod), "r"((uint32_t)(prod >> 32)), "r"(ahi));
}

// x += a * (v0 + v1 2^32), v1 <= 2 (see acc5_mac_v01)
PMP_DI void acc3_mac_v01(Acc3 &x, uint32_t a, uint32_t v0, uint32_t v1) {
  const uint64_t prod = (uint64_t)a * v0;
  const uint64_t q = (uint64_t)a * v1;                 // < 2^34, weight 2^32
  asm("add.cc.u32  %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32    %2, %2, 0;\n\t"
      "add.cc.u32  %1, %1, %5;\n\t"
      "addc.u32    %2, %2, %6;"
      : "+r"(x.c0), "+r"(x.c1), "+r"(x.c2)
      : "r"((uint32_t)prod), "r"((uint32_t)(prod >> 32)), "r"((uint32_t)q), "r"((uint32_t)(q >> 32)));
}

PMP_DI Acc3 acc3_shfl_xor(const Acc3 &x, int m) {
  Acc3 r;
  r.c0 = __shfl_xor_sync(0xffffffffu, x.c0, m);
  r.c1 = __shfl_xor_sync(0xffffffffu, x.c1, m);
  r.c2 = __shfl_xor_sync(0xffffffffu, x.c2, m);
  return r;
}

// Section 6.2 for n = 32, k = 15: (v0, v1) with v1 <= 2 for w2 < 2^24
PMP_HDI void reduce3to2_32(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t &v0, uint32_t &v1) {
  uint64_t u = (uint64_t)w1 * kK32;                     // u1 2^32 + u0
  uint64_t u0 = (uint32_t)u, u1 = u >> 32;
  uint64_t x = (uint64_t)w0 + kK32 * kK32 * w2 + kK32 * u1;
  uint64_t y = (1ULL << 32) + kK32 - u0;
  uint64_t v = x + y;
  v0 = (uint32_t)v;
  v1 = (uint32_t)(v >> 32);
}

PMP_HDI uint64_t alg2_32(uint32_t v0, uint32_t v1) {  // Algorithm 2 (corrected), value < p
  if (kK32 * v1 <= v0) return (uint64_t)v0 - kK32 * v1;
  if (v1 == 1) return (1ULL << 32) + v0;
  return (1ULL << 32) + v0 - kK32;
}

// V mod 2^32 only, the same folding for n = 32 in 64-bit arithmetic:
//   v = w0 + k^2 w2 + k u1 + 2^32 + k - u0 (< 3 * 2^32), v0 = v mod 2^32, v1 = v >> 32,
//   lo = v0 - k v1 + k [v0 < k v1]  (mod 2^32).
PMP_HDI uint32_t reduce_lo_acc3(const Acc3 &x) {
  const uint64_t u = (uint64_t)x.c1 * kK32;
  const uint64_t v = (uint64_t)x.c0 + kK32 * kK32 * x.c2 + kK32 * (u >> 32) + (1ULL << 32) + kK32 - (uint32_t)u;
  const uint32_t v0 = (uint32_t)v, kv = (uint32_t)(kK32 * (v >> 32));
  return v0 - kv + (v0 < kv ? (uint32_t)kK32 : 0u);
}

PMP_HDI uint64_t reduce_acc3(const Acc3 &x) {
  uint32_t v0, v1;
  reduce3to2_32(x.c0, x.c1, x.c2, v0, v1);
  return alg2_32(v0, v1);
}

}  // namespace pmp
