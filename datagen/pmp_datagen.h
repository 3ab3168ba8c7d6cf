/*
 * pmp_datagen.h -- seeded synthetic inputs shared by tests, smoke() and bench.
 *
 * This module holds NO PM+ arithmetic: only the input generators, so that the
 * oracle (host) and the CUDA path (device) can regenerate the same bytes
 * without either importing the other.
 *
 * Stream contract ("seeded xoshiro256**", BASELINE.json configs):
 *   stream(seed, id): xoshiro256** whose state is 4 successive splitmix64
 *   outputs from seed ^ (id * 0x9E3779B97F4A7C15).
 *   - lengths: stream id 1, one draw per string in order;
 *   - payload: the contiguous payload buffer is cut in 4 KiB pages; page q is
 *     filled by stream id 2 + q, output r -> bytes [4096 q + 8 r, +8) little-
 *     endian.  Payload bytes depend only on (seed, absolute buffer position),
 *     so any string (or any sample of a 16 GiB buffer) can be regenerated.
 */
#ifndef PMP_DATAGEN_H
#define PMP_DATAGEN_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMPD_PAGE 4096u

enum pmpd_len_kind {
  PMPD_LEN_FIXED = 0,      /* every length = lo */
  PMPD_LEN_UNIFORM = 1,    /* lo + ((x>>32) * (hi-lo+1)) >> 32 */
  PMPD_LEN_LOGUNIFORM = 2  /* floor(2^(u*log2(hi))) clamped to [lo,hi], u = (x>>11)*2^-53 */
};

/* n string lengths drawn from stream (seed, 1). */
void pmpd_lengths(int kind, uint64_t seed, uint64_t n, uint64_t lo, uint64_t hi,
                  uint64_t *lengths);

/* The generators behind the contract (for pinning to published outputs):
 * n splitmix64 outputs from `state`; n xoshiro256** outputs from s[4];
 * n outputs of stream(seed, id). */
void pmpd_splitmix64_stream(uint64_t state, uint64_t n, uint64_t *out);
void pmpd_xoshiro256ss_stream(const uint64_t *s, uint64_t n, uint64_t *out);
void pmpd_stream(uint64_t seed, uint64_t id, uint64_t n, uint64_t *out);

/* CSR offsets: offsets[0] = 0, offsets[i+1] = offsets[i] + lengths[i].
 * Returns offsets[n]. */
uint64_t pmpd_offsets(const uint64_t *lengths, uint64_t n, uint64_t *offsets);

/* Host: payload bytes [start, start + nbytes) of the buffer for `seed`. */
void pmpd_fill_host(uint64_t seed, uint64_t start, uint64_t nbytes, uint8_t *out);

/* Device: fill dev[0, nbytes) with payload bytes [0, nbytes) on `stream`
 * (a cudaStream_t passed as void*).  Returns 0 or a cudaError_t value. */
int pmpd_fill_device(uint64_t seed, uint8_t *dev, uint64_t nbytes, void *stream);

/* Device: fill dev[0, nbytes) with payload bytes [4096*page0, 4096*page0 + nbytes). */
int pmpd_fill_device_at(uint64_t seed, uint8_t *dev, uint64_t nbytes, uint64_t page0, void *stream);

#ifdef __cplusplus
}
#endif
#endif
