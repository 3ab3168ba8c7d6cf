/*
 * pmp_oracle.h -- plain, slow, obviously-correct CPU oracle for PM+ hashing.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1609_09840_b200/, libpmp.so) never includes, links
 * or calls anything here, and this file shares no code with it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source of
 * arXiv:1609.09840), "S:n" = SPEC.md line n.  Readings of ambiguous passages
 * are the Q-numbered readings listed in DESIGN.md ("Readings of the paper").
 *
 * Arithmetic: unsigned __int128 with a `% p` after every product, exactly as
 * Eq. (1) is written; no lazy reduction, no 3-word accumulator, no
 * Algorithm 2 -- those are the GPU path's business and are checked against
 * this file, not shared with it.
 *
 * Values that may reach p (> 2^64) cross the ABI as (lo, hi) uint64 pairs.
 */
#ifndef PMP_ORACLE_H
#define PMP_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMPO_M 128 /* Table 2: m = 128 */
#define PMPO_L 8   /* Table 2: L = 8 levels */

/* Table 2 constants for a word size (bits = 32 or 64).  Returns 0, or -1 on a
 * bad width.  p = 2^n + k, a_max = p - kappa - 1 (the
 * PM+32 interval printed as (0, 2^64-13) is read as (0, 2^32-13), reading Q8). */
int pmpo_params(int bits, uint64_t *p_lo, uint64_t *p_hi, uint64_t *k,
                uint64_t *kappa, uint64_t *a_max);

/* Project key-generation contract (reading Q12; the paper is silent):
 * state = 4 successive splitmix64 outputs from `seed`, generator xoshiro256**.
 * For j = 1..8: b_j = x (64-bit) or x>>32 (32-bit); then a_{j,1..128} by
 * rejection: accept 1 <= x <= a_max (x>>32 for 32-bit).
 * b: 8 words, a: 8*128 words (level-major).  Returns 0, -1 on bad width. */
int pmpo_keygen(uint64_t seed, int bits, uint64_t *b, uint64_t *a);

/* The generator streams of that contract, for pinning against published
 * reference outputs: n successive splitmix64 outputs from `state`, and n
 * successive xoshiro256** outputs from the state s[4] (s is not modified). */
void pmpo_splitmix64_stream(uint64_t state, uint64_t n, uint64_t *out);
void pmpo_xoshiro256ss_stream(const uint64_t s[4], uint64_t n, uint64_t *out);

/* Mixing finalizer, P:722-734 (64-bit: 33 / 0xc4ceb9fe1a85ec53 / 33;
 * 32-bit: 13 / 0xab3be54f / 16) and its inverse ("invertible"). */
uint64_t pmpo_mix(int bits, uint64_t z);
uint64_t pmpo_unmix(int bits, uint64_t z);

/* sigma word t of a byte string (reading Q3/Q4): little-endian n-bit
 * word of bytes [t*w, t*w+w) where byte `len` reads 0x01 and later bytes 0. */
uint64_t pmpo_sigma_word(int bits, const uint8_t *bytes, uint64_t len, uint64_t t);

/* Number of sigma words T = floor(len / w) + 1. */
uint64_t pmpo_num_words(int bits, uint64_t len);

/* One PM+-Multilinear block, Eq. (1), over an arbitrary modulus
 * p = (p_lo, p_hi) < 2^66 and block width m:
 *   out = (b + sum_{i<m} a_i * x_i) mod p,  x_i = (x_lo[i], x_hi[i]) < p.
 * Keys are uint64 (a_i < p - kappa <= 2^n).  out = (out[0], out[1]). */
void pmpo_block(uint64_t p_lo, uint64_t p_hi, int m, uint64_t b,
                const uint64_t *a, const uint64_t *x_lo, const uint64_t *x_hi,
                uint64_t *out);

/* Algorithm 1, literal, over a given character string sigma
 * (already including the appended 1), with modulus p and block width m,
 * starting at level index j0 (0-based: the first level applied uses
 * b[j0], a[j0*m .. j0*m+m)).  b has L entries, a has L*m entries.
 * Loop: while |sigma| > 1 { zero-pad to a multiple of m; map blocks with f_j;
 * j++ }.  Returns the number of levels applied (0 when T == 1), or -1 if more
 * than L - j0 levels would be needed.  out = (lo, hi) of the sole value. */
int pmpo_tree_generic(uint64_t p_lo, uint64_t p_hi, int m, int L, int j0,
                      const uint64_t *b, const uint64_t *a,
                      const uint64_t *x_lo, const uint64_t *x_hi, uint64_t T,
                      uint64_t *out);

/* PM+ tree value V = Tree(sigma) in [0,p) for a byte string:
 * level 1 is evaluated block by block straight from the bytes (each block of
 * 128 sigma words materialised), higher levels by Algorithm 1.
 * `nthreads` > 1 evaluates the independent level-1 blocks on that many
 * threads (a parallel map; the arithmetic of each block is unchanged).
 * Returns levels applied or -1. */
int pmpo_tree_value(int bits, const uint64_t *b, const uint64_t *a,
                    const uint8_t *bytes, uint64_t len, int nthreads,
                    uint64_t *out);

/* digest = mix_n(V mod 2^n). */
uint64_t pmpo_hash(int bits, const uint64_t *b, const uint64_t *a,
                   const uint8_t *bytes, uint64_t len);

/* Many strings: string i = bytes[offsets[i], offsets[i+1]) (reading Q13);
 * strings are split over `nthreads` pthreads (0 = 1).  out[i] = digest. */
void pmpo_hash_batch(int bits, const uint64_t *b, const uint64_t *a,
                     const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                     uint64_t *out, int nthreads);

/* One long string with a multithreaded level-1 map; digest. */
uint64_t pmpo_hash_long(int bits, const uint64_t *b, const uint64_t *a,
                        const uint8_t *bytes, uint64_t len, int nthreads);

/* Two-level variant (reading Q19): level 1 = f_1 on each
 * 128-word chunk (as the tree), level 2 = Horner polynomial in r = a_{2,1}
 * over the C chunk values, V = (b_2 + sum_c v_c r^(C-c)) mod p, for every
 * string (T == 1 included).  `nthreads` parallelises the level-1 map only. */
int pmpo_hash2_value(int bits, const uint64_t *b, const uint64_t *a,
                     const uint8_t *bytes, uint64_t len, int nthreads, uint64_t *out);
uint64_t pmpo_hash2(int bits, const uint64_t *b, const uint64_t *a,
                    const uint8_t *bytes, uint64_t len, int nthreads);

void pmpo_hash2_batch(int bits, const uint64_t *b, const uint64_t *a,
                      const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                      uint64_t *out, int nthreads);

/* x * y mod p (x, y < p < 2^66) by shift-and-add; out = (lo, hi). */
void pmpo_mulmod(uint64_t p_lo, uint64_t p_hi, uint64_t x_lo, uint64_t x_hi,
                 uint64_t y_lo, uint64_t y_hi, uint64_t *out);

#ifdef __cplusplus
}
#endif
#endif
