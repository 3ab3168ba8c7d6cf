/*
 * pmp.h -- C ABI of libpmp.so: PM+ hashing (Ivanchykhin, Ignatchenko, Lemire,
 * "Regular and almost universal hashing: an efficient implementation",
 * arXiv:1609.09840) on NVIDIA B200 (sm_100a).
 *
 * Citations: "P:n" is line n of the paper's LaTeX source; "S:n" is
 * line n of SPEC.md.  Ambiguous passages follow the readings Q1..Q16 listed in
 * DESIGN.md ("Readings of the paper").
 *
 * What is computed: for a byte string s,
 *   sigma  = s || 0x01 || 0x00...  up to a multiple of w = n/8 bytes, read as
 *            little-endian n-bit words (readings Q3, Q4);
 *   V      = Tree(sigma): Algorithm 1 with the PM+-Multilinear
 *            family f_j(x_1..x_128) = (b_j + sum_i a_{j,i} x_i) mod p, Eq. (1)
 *            P:543, f_1 at the leaves (reading Q1); when sigma has one word the
 *            loop never runs and V = sigma_0 (reading Q2);
 *   digest = mix_n(V mod 2^n) with the finaliser of P:722-734.
 * PM+64: n = 64, p = 2^64+13; PM+32: n = 32, p = 2^32+15 (Table 2).
 *
 * Conventions for every call:
 *   - Return 0 on success or a negative PMP_E* code (pmp_strerror()).
 *   - Pointers marked (device) are device memory of the key handle's device,
 *     owned by the caller; the library writes only the `out` / `partial`
 *     buffers and allocates its scratch stream-ordered (cudaMallocAsync).
 *   - Hash calls are asynchronous and ordered on `stream` (a cudaStream_t; NULL
 *     is the legacy default stream).  Results are valid after the stream is
 *     synchronised; execution faults surface there, launch errors are returned
 *     as PMP_ECUDA.
 *   - No CPU fallback exists: without a CUDA device every hash call returns
 *     PMP_ENODEV.
 */
#ifndef PMP_H
#define PMP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st; /* = cudaStream_t */

#define PMP_OK 0
#define PMP_EINVAL (-1)   /* bad argument (NULL with n > 0, bad width, key out of range, misaligned split) */
#define PMP_ETOOLONG (-2) /* more than 2^56 - 1 words (Table 3: L = 8 levels of m = 128) */
#define PMP_ECUDA (-3)    /* CUDA runtime error at launch / allocation */
#define PMP_ENOMEM (-4)   /* host or device allocation failure */
#define PMP_ENODEV (-5)   /* no CUDA device, or the key handle has no device copy */
#define PMP_EBADFILE (-6) /* KeyFile: wrong magic or wrong length (SPEC "BadMagic") */
#define PMP_EVERSION (-7) /* KeyFile: unsupported version, word size or level count */
#define PMP_EKEYRANGE (-8) /* KeyFile: a key outside its range (SPEC "KeyOutOfRange") */

/* Opaque key schedule: b_j and a_{j,1..128} for j = 1..8 (Alg. 1 REQUIRE,
 * P:431; Eq. (1)).  Immutable after creation; may be shared by any
 * number of threads and streams on its device. */
typedef struct pmp_keys pmp_keys;

/* Expand `seed` into a key schedule for out_bits = 32 or 64 and upload it to
 * the current CUDA device.  Key-generation contract (reading Q12; the paper is
 * silent): xoshiro256** seeded with 4 splitmix64 outputs of `seed`; per level
 * j = 1..8, b_j = x (x>>32 for 32-bit) then a_{j,i} by rejection sampling to
 * [1, p - kappa - 1] (kappa = 24 / 28).  Every process calling
 * with the same seed gets identical keys.  Returns NULL on a bad width or
 * allocation failure.  Without a CUDA device the handle is created host-only
 * (export works, hash calls return PMP_ENODEV). */
pmp_keys *pmp_keygen(uint64_t seed, int out_bits);

/* Build a schedule from explicit words (host arrays: b[8], a[8*128],
 * level-major).  Validates b_j < 2^n and 1 <= a_{j,i} <= p - kappa - 1
 * (SPEC "KeyOutOfRange"); returns NULL when a key is out of range. */
pmp_keys *pmp_keys_from_words(int out_bits, const uint64_t *b, const uint64_t *a);

/* Copy the schedule to host arrays b[8], a[8*128]; returns 0 or PMP_EINVAL. */
int pmp_keys_export(const pmp_keys *keys, uint64_t *b, uint64_t *a);

/* 32 or 64, or PMP_EINVAL for NULL. */
int pmp_keys_bits(const pmp_keys *keys);

/* KeyFile (layout SPEC S:289-295, "invented artifact plumbing"):
 *   bytes 0-3 "PMPH", 4 version = 0x01, 5 word size in bits (0x20 | 0x40),
 *   6 levels = 0x08, 7 reserved = 0x00, then for j = 1..8: b_j followed by
 *   a_{j,1..128}, each a little-endian word of n/8 bytes.
 * pmp_keyfile_size: 8 + 8 * 129 * n/8 = 8264 (64-bit) / 4136 (32-bit) bytes,
 *   0 for a bad width.
 * pmp_keys_save: serialise `keys` into the host buffer out[cap]; returns 0, or
 *   PMP_EINVAL for NULL or cap < pmp_keyfile_size.
 * pmp_keys_load: parse a host buffer buf[len] and upload the schedule as
 *   pmp_keys_from_words does.  Validates the magic and exact length
 *   (PMP_EBADFILE), version / word size / level count / reserved byte
 *   (PMP_EVERSION), and every key range, b_j < 2^n and 1 <= a <= p - kappa - 1
 *   (PMP_EKEYRANGE).  Returns the handle, or NULL with *err (if err != NULL)
 *   set to the code; *err = 0 on success.  load(save(k)) exports the same
 *   words as k. */
uint64_t pmp_keyfile_size(int out_bits);
int pmp_keys_save(const pmp_keys *keys, uint8_t *out, uint64_t cap);
pmp_keys *pmp_keys_load(const uint8_t *buf, uint64_t len, int *err);

void pmp_keys_free(pmp_keys *keys);

/* Hash n byte strings.  String i is bytes[offsets[i], offsets[i+1]) (CSR,
 * reading Q13); strings may start at any byte alignment and may be empty.
 *   bytes   (device) payload; only bytes inside [offsets[0], offsets[n]) are
 *           used -- the kernels read whole aligned 16-byte units that contain
 *           at least one such byte, never a unit outside that range;
 *   offsets (device) n+1 uint64, non-decreasing (precondition, not checked);
 *   out     (device) n digests: uint64 for 64-bit keys, uint32 for 32-bit keys,
 *           in string order.
 * n == 0 is a no-op; n must be < 2^32.  Strings of <= 127 bytes take the
 * thread-per-string path, longer ones a warp per string. */
int pmp_hash_batch(const pmp_keys *keys, const uint8_t *bytes, const uint64_t *offsets,
                   uint64_t n, void *out, struct CUstream_st *stream);

/* Hash-table consumer: the same batch hash, fused with the
 * bucket mapping b_i = digest_i mod M (M >= 1).  By the paper's lemmas the
 * bucket map keeps almost Delta-universality up to a factor ceil((2|Y|-1)/M)
 * and is 2-regular, regular when M divides 2^n.
 *   buckets (device) n uint32;
 *   counts  (device) M uint32 incremented atomically per string (the caller
 *           zeroes it; histograms of several calls accumulate), or NULL.
 * Same conventions and errors as pmp_hash_batch; PMP_EINVAL for M == 0. */
int pmp_hash_batch_buckets(const pmp_keys *keys, const uint8_t *bytes, const uint64_t *offsets,
                           uint64_t n, uint32_t M, uint32_t *buckets, uint32_t *counts,
                           struct CUstream_st *stream);

/* Bucket partition, the step after the histogram in a GPU hash join /
 * group-by (the paper's motivating use):
 * the string indices 0..n-1 grouped by bucket id.
 *   buckets (device) n uint32, each < M (e.g. from pmp_hash_batch_buckets; an
 *           id >= M is a precondition violation, not checked);
 *   hist    (device) M uint32, the bucket sizes of exactly these n ids (e.g. the
 *           counts of one pmp_hash_batch_buckets call into zeroed counters), or
 *           NULL: the library counts them (one more pass over the ids);
 *   starts  (device, out) M+1 uint64: bucket b occupies perm[starts[b],
 *           starts[b+1]) (exclusive prefix sums of the bucket sizes); starts[M] = n;
 *   perm    (device, out) n uint32: the indices, bucket by bucket; the order
 *           inside a bucket is unspecified (it depends on scheduling).
 * 1 <= M <= 2^24 and n < 2^32, else PMP_EINVAL (also for NULL with n > 0);
 * n = 0 writes starts (all zero).  Runs on the current device, stream-ordered;
 * scratch (M counters) is stream-allocated.  PMP_ENODEV without a device. */
int pmp_bucket_partition(const uint32_t *buckets, uint64_t n, uint32_t M, const uint32_t *hist,
                         uint64_t *starts, uint32_t *perm, struct CUstream_st *stream);

#define PMP_HOST_MAX_KEYS 4
/* Several key schedules over one device batch (1 <= nkeys <= PMP_HOST_MAX_KEYS;
 * outs[k]: device, n digests for keys[k]).  Equal to nkeys pmp_hash_batch
 * calls; a 64-bit and a 32-bit schedule are paired into one fused pass over
 * the short strings (each string read once for both digests, configs[1]'s
 * "both 32-bit and 64-bit outputs"), long strings are hashed per schedule.
 * Errors as pmp_hash_batch. */
int pmp_hash_batch_multi(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                         uint64_t n, void *const *outs, struct CUstream_st *stream);

/* Host-resident batch (the e2e path): the same digests as pmp_hash_batch for
 * bytes / offsets / outs in HOST memory, under nkeys key schedules at once
 * (1 <= nkeys <= PMP_HOST_MAX_KEYS; e.g. a 64-bit and a 32-bit schedule, all on
 * one device).  The library cuts the batch into string-aligned pieces of about
 * piece_bytes payload bytes (0: 64 MiB; a longer string is a piece alone) and
 * streams them through the device on internal streams: the host->device copy
 * of one piece, the hashing of the previous one and the device->host copy of
 * the one before overlap.  Host buffers should be page-locked
 * (cudaHostAlloc / cudaHostRegister) for the copies to run asynchronously.
 *   bytes   (host) payload, string i = bytes[offsets[i], offsets[i+1]);
 *   offsets (host) n+1 uint64, non-decreasing;
 *   outs[k] (host) n digests for keys[k] (uint64 / uint32 by its width).
 * Stream-ordered like every call: the pieces start after prior work on
 * `stream`, and the digests are in host memory once `stream` has reached this
 * point (synchronise it before reading outs); the host buffers must stay
 * valid until then.  Device scratch is stream-ordered and released by then.
 * Errors as pmp_hash_batch, and PMP_EINVAL for keys on different devices. */
int pmp_hash_batch_host(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                        uint64_t n, void *const *outs, uint64_t piece_bytes, struct CUstream_st *stream);

/* Host-resident long string (the e2e path of configs[3]): the same digest as
 * pmp_hash_long for `len` bytes at `bytes` in HOST memory.  The string is cut
 * into pieces of piece_bytes (0: 256 MiB; rounded down to whole level-1
 * blocks) that are copied host->device on internal streams into three device
 * slots and fed to a device-resident incremental state (the pmp_stream_*
 * machinery) on `stream`, so the copy of one piece overlaps the
 * hashing of the previous one.  The digest (uint64 / uint32 by the keys'
 * width) is written to `out_host` (HOST memory).  Stream-ordered: starts after
 * prior work on `stream`; `out_host` holds the digest once `stream` has
 * reached this point; `bytes` must stay valid until then.  `bytes` should be
 * page-locked for the copies to run asynchronously.  Errors as pmp_hash_long. */
int pmp_hash_long_host(const pmp_keys *keys, const uint8_t *bytes, uint64_t len, void *out_host,
                       uint64_t piece_bytes, struct CUstream_st *stream);

/* Hash one string of `len` bytes at `bytes` (device, any alignment); writes
 * one digest (uint64 / uint32) to `out` (device).  Block-parallel over the
 * level-2 nodes of the tree (128 level-1 blocks each), then one launch per
 * upper level.  PMP_ETOOLONG beyond 2^56 - 1 words. */
int pmp_hash_long(const pmp_keys *keys, const uint8_t *bytes, uint64_t len, void *out,
                  struct CUstream_st *stream);

/* Multi-GPU split of one long string (the tree is affine in its level-1 block
 * values):
 * The caller holds bytes [global_offset, global_offset + local_len) of a string
 * of total_len bytes at `local` (device).  global_offset must be a multiple of
 * the level-1 block size (1024 bytes for PM+64, 512 for PM+32) and so must
 * local_len unless global_offset + local_len == total_len.  The tail block (the
 * one holding the marker word) belongs to the one range that holds the
 * last byte total_len - 1; an empty range never owns it, so any number of empty
 * ranges may appear anywhere in the split.  Writes to `partial` (device, 2
 * uint64: lo, hi) the field element P = sum over the caller's blocks c of
 * K_c * v_1(c) mod p, where K_c is the product of the level keys on c's path
 * to the root (an empty range writes 0).  Ranges of all callers must tile
 * [0, total_len).  For the empty message (total_len == 0) every partial is 0
 * and the combine supplies the value sigma_0 = 1 (reading Q2). */
int pmp_hash_long_partial(const pmp_keys *keys, const uint8_t *local, uint64_t local_len,
                          uint64_t global_offset, uint64_t total_len, uint64_t *partial,
                          struct CUstream_st *stream);

/* Combine G partials (device, 2*G uint64, e.g. the result of an all-gather):
 * V = C(total_len) + sum_g P_g mod p, C being the key-only tree value with
 * all v_1 = 0; writes the digest to `out` (device). */
int pmp_hash_long_combine(const pmp_keys *keys, const uint64_t *partials, int G,
                          uint64_t total_len, void *out, struct CUstream_st *stream);

/* Incremental hashing (the bounded-memory evaluation of
 * Algorithm 1).  The digest of all bytes fed through
 * pmp_stream_update equals pmp_hash_long of their concatenation, for every way
 * of cutting it into updates (split invariance).  Device state: one
 * open-node running sum per level (O(L)) plus < one level-1 block of pending
 * bytes; each update hashes its whole blocks with the block-parallel node
 * kernel.  A stream is single-owner; calls are ordered on `stream`.
 *   pmp_stream_new:    state on the keys' device (NULL on failure);
 *   pmp_stream_update: `bytes` (device, any alignment, any length); the
 *                      caller may reuse the buffer once the stream reaches it;
 *   pmp_stream_final:  writes the digest (uint64/uint32) to `out` (device);
 *                      further updates return PMP_EINVAL until a reset;
 *   pmp_stream_reset:  start a new message with the same keys. */
typedef struct pmp_stream pmp_stream;
pmp_stream *pmp_stream_new(const pmp_keys *keys);
int pmp_stream_update(pmp_stream *s, const uint8_t *bytes, uint64_t len, struct CUstream_st *stream);
int pmp_stream_final(pmp_stream *s, void *out, struct CUstream_st *stream);
int pmp_stream_reset(pmp_stream *s, struct CUstream_st *stream);
void pmp_stream_free(pmp_stream *s);

/* ---- Two-level variant ("a two-level approach where
 * only the first level uses Multilinear, while the second level uses a
 * polynomial hash family"; the formula is reading Q19 in DESIGN.md):
 *   v_c = f_1(chunk c) = (b_1 + sum_i a_{1,i} sigma_{128c+i}) mod p, c < C = ceil(T/128)
 *   V   = (b_2 + sum_{c<C} v_c r^(C-c)) mod p,   r = a_{2,1}
 *   digest = mix(V mod 2^n)   -- for every string, T == 1 included.
 * It uses the same key schedule (keygen / KeyFile) and produces different
 * digests from the tree.  Conventions, arguments and errors are those of the
 * tree calls of the same shape:
 *   pmp_hash2_batch        ~ pmp_hash_batch
 *   pmp_hash2_batch_multi  ~ pmp_hash_batch_multi (a 64- and a 32-bit schedule fused likewise)
 *   pmp_hash2_long         ~ pmp_hash_long
 *   pmp_hash2_long_partial ~ pmp_hash_long_partial: the caller's chunks
 *       contribute sum v_c r^(C-c) (a field element, 2 words) -- no key-only
 *       constant is needed, the sum is linear in the v_c.  The tail chunk
 *       belongs to the range holding byte total_len - 1 (never to an empty
 *       range); the empty message (total_len == 0, one marker-only chunk)
 *       must be hashed as a single range;
 *   pmp_hash2_long_combine: digest of b_2 + sum_g P_g (G partials, device). */
int pmp_hash2_batch(const pmp_keys *keys, const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                    void *out, struct CUstream_st *stream);
int pmp_hash2_batch_multi(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                          uint64_t n, void *const *outs, struct CUstream_st *stream);
int pmp_hash2_long(const pmp_keys *keys, const uint8_t *bytes, uint64_t len, void *out,
                   struct CUstream_st *stream);
int pmp_hash2_long_partial(const pmp_keys *keys, const uint8_t *local, uint64_t local_len,
                           uint64_t global_offset, uint64_t total_len, uint64_t *partial,
                           struct CUstream_st *stream);
int pmp_hash2_long_combine(const pmp_keys *keys, const uint64_t *partials, int G, void *out,
                           struct CUstream_st *stream);

/* Host-only helper: split [0, total_len) into G contiguous ranges aligned to
 * level-1 blocks with equal block counts (+- 1); begins[0..G] (host),
 * begins[G] = total_len.  Returns 0 or PMP_EINVAL. */
int pmp_long_split(int out_bits, uint64_t total_len, int G, uint64_t *begins);

/* Host-only helper (test hook): the key-only constant C(total_len) as (lo, hi). */
int pmp_long_constant(const pmp_keys *keys, uint64_t total_len, uint64_t *c2);

/* Quality suite (SPEC quality_suite collision_monte_carlo):
 * Monte Carlo over nsched random key schedules, schedule i being
 * pmp_keygen(seed0 + i, out_bits) (drawn on the device by the same contract),
 * of a FIXED pair of strings s1, s2 (device, <= 127 bytes each: one level-1
 * block, so only b_1 and a_{1,0..31} are drawn).  Adds to counts[0..3]
 * (device, 4 uint64, caller-zeroed) the number of schedules whose digests are
 * equal in all n bits, in their low 16, 12 and 8 bits.  dig1 / dig2 (device,
 * nsched uint64 each, or NULL) receive the digests.  Table 3 bounds the
 * full-digest collision probability of distinct equal-length strings by
 * eps ~ 2^-60 (PM+64) / 2^-28 (PM+32); s1 == s2 collides always.
 * PMP_EINVAL for a longer string or a bad width. */
int pmp_quality_collisions(int out_bits, uint64_t seed0, uint64_t nsched, const uint8_t *s1, uint32_t len1,
                           const uint8_t *s2, uint32_t len2, uint64_t *dig1, uint64_t *dig2, uint64_t *counts,
                           struct CUstream_st *stream);

/* Device self-test hooks running the hot path's own device functions:
 * mode 0: in = n triples (w0, w1, w2) -> (w0 + w1 2^n + w2 2^2n) mod p via the
 *         Section 6.2 reduction and Algorithm 2; w2 <= 2^16;
 * mode 1: in = n records [b, a_0..a_127, s_0..s_127] -> Eq. (1) via the
 *         hot-loop multiply-accumulate;
 * mode 2: in = n words -> mix_n(word);
 * mode 3: as mode 0 but returns only (value mod p) mod 2^n, the folded
 *         form the digest path uses;
 * mode 4: as mode 0 by the folded reduction returning the full residue
 *         (PM+64; PM+32 as mode 0), used by the two-level short strings.
 * in/out (device); out gets 2 uint64 per record (lo, hi). */
int pmp_selftest(int out_bits, int mode, const uint64_t *in, uint64_t n, uint64_t *out,
                 struct CUstream_st *stream);

/* Instrumentation.  pmp_launch_count(): kernels launched by this library so
 * far in this process.  With pmp_prof_enable(1), every launch is bracketed
 * by CUDA events on its own stream; pmp_prof_read() synchronises those events
 * and returns the summed milliseconds and launch count of kernels whose name
 * starts with `prefix` ("k_short", "k_wstring", "k_node", ...). */
uint64_t pmp_launch_count(void);

/* Batch routing (tuning / test hook).  A batch call with n <= this threshold
 * takes the latency path (k_small: one launch, no scratch, one thread per
 * short string, one warp per longer string); larger batches take the
 * throughput path (k_short's TMA pipeline + k_wstring).  Both give identical
 * digests.  Default 4096; 0 sends every batch to the throughput path.  Sets
 * the process-wide value and returns the previous one.  The two-level
 * variant always takes the throughput path. */
uint64_t pmp_set_small_batch_max(uint64_t n);

/* Huge strings in a batch (tuning / test hook).  The throughput path hashes a
 * string of >= `bytes` bytes node-parallel (k_huge: parts of 128 KiB
 * claimed by every warp of a persistent grid, combined by the affine identity
 * of DESIGN.md section 7 with the key-only constant computed on the device)
 * instead of with one warp; at most `cap` such strings per call (the rest
 * keep the one-warp path).  Identical digests either way.  Defaults: 4 MiB,
 * 65,536.  pmp_set_huge_min(0) only queries; values below 64 KiB act as
 * 64 KiB.  pmp_set_huge_cap(0) turns the huge path off.  Both set the
 * process-wide value and return the previous one.  The two-level variant and
 * the tensor-core short-string option keep the one-warp path. */
uint64_t pmp_set_huge_min(uint64_t bytes);
uint32_t pmp_set_huge_cap(uint32_t cap);

/* Short-string kernel of the throughput path (tuning / test hook).  1: the
 * level-1 sums of strings of <= 64 bytes run as an exact u8 x u8 -> s32
 * matrix product on the tensor cores (k_short_tc, tcgen05.mma kind::i8);
 * 0: every short string takes k_short's per-thread word loop.  Both give
 * identical digests.  Applies to the tree variant without buckets (the
 * two-level variant and bucket mode always take k_short).  on < 0 only
 * queries.  Default 0: the tensor-core kernel is bit-exact but not faster
 * on configs[1]; the environment PMP_SHORT_TC=1 selects
 * 1.  Returns the previous setting. */
int pmp_set_short_tc(int on);
void pmp_prof_enable(int on);
void pmp_prof_reset(void);
int pmp_prof_read(const char *prefix, double *ms, uint64_t *count);

const char *pmp_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif
