/* pmp_c_client.c -- a plain C program using only include/pmp.h and the CUDA
 * runtime (no Python, no torch): the boundary as a C caller sees it.
 * tests/test_c_client.py builds it against the in-tree libpmp.so and compares
 * its digests with the oracle.
 *
 * Input (stdin, text): bits n, then n lengths, then the payload is generated as
 * byte i = (i * 131 + 7) & 255 over the concatenation.  Output (stdout): one
 * line per string for pmp_hash_batch, the same via pmp_hash_batch_host, then
 * pmp_hash_long of the whole concatenation, pmp_stream_* of it in 3 pieces,
 * pmp_hash_long_host of it from host memory, and the batch again through the
 * throughput path (pmp_set_small_batch_max(0)).
 */
#include <cuda_runtime.h>
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>

#include "pmp.h"

#define CK(x)                                                          \
  do {                                                                 \
    int rc_ = (x);                                                     \
    if (rc_) {                                                         \
      fprintf(stderr, "%s: %d %s\n", #x, rc_, pmp_strerror(rc_));      \
      return 1;                                                        \
    }                                                                  \
  } while (0)
#define CU(x)                                                          \
  do {                                                                 \
    cudaError_t e_ = (x);                                              \
    if (e_ != cudaSuccess) {                                           \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));         \
      return 1;                                                        \
    }                                                                  \
  } while (0)

static uint64_t digest_at(const void *out, int bits, uint64_t i) {
  return bits == 64 ? ((const uint64_t *)out)[i] : ((const uint32_t *)out)[i];
}

int main(void) {
  int bits;
  uint64_t n;
  if (scanf("%d %" SCNu64, &bits, &n) != 2) return 2;
  uint64_t *off = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
  off[0] = 0;
  for (uint64_t i = 0; i < n; i++) {
    uint64_t len;
    if (scanf("%" SCNu64, &len) != 1) return 2;
    off[i + 1] = off[i] + len;
  }
  const uint64_t total = off[n];
  uint8_t *bytes;
  CU(cudaMallocHost((void **)&bytes, total + 1));
  for (uint64_t i = 0; i < total; i++) bytes[i] = (uint8_t)((i * 131 + 7) & 255);
  const size_t w = bits / 8;

  pmp_keys *k = pmp_keygen(2, bits);
  if (!k) {
    fprintf(stderr, "pmp_keygen failed\n");
    return 1;
  }
  cudaStream_t st;
  CU(cudaStreamCreate(&st));
  uint8_t *d_bytes;
  uint64_t *d_off;
  void *d_out;
  CU(cudaMalloc((void **)&d_bytes, total + 16));
  CU(cudaMalloc((void **)&d_off, (n + 1) * sizeof(uint64_t)));
  CU(cudaMalloc(&d_out, (n ? n : 1) * w));
  CU(cudaMemcpy(d_bytes, bytes, total, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_off, off, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice));

  /* device batch */
  void *out = malloc((n ? n : 1) * w);
  CK(pmp_hash_batch(k, d_bytes, d_off, n, d_out, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaMemcpy(out, d_out, n * w, cudaMemcpyDeviceToHost));
  for (uint64_t i = 0; i < n; i++) printf("batch %" PRIu64 " %016" PRIx64 "\n", i, digest_at(out, bits, i));

  /* host-resident batch (small pieces: several pieces, copy/compute overlap) */
  void *hout;
  CU(cudaMallocHost(&hout, (n ? n : 1) * w));
  const pmp_keys *ks[1] = {k};
  void *outs[1] = {hout};
  CK(pmp_hash_batch_host(ks, 1, bytes, off, n, outs, 4096, st));
  CU(cudaStreamSynchronize(st));
  for (uint64_t i = 0; i < n; i++) printf("host %" PRIu64 " %016" PRIx64 "\n", i, digest_at(hout, bits, i));

  /* the concatenation as one long string, and streamed in three pieces */
  CK(pmp_hash_long(k, d_bytes, total, d_out, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaMemcpy(out, d_out, w, cudaMemcpyDeviceToHost));
  printf("long %016" PRIx64 "\n", digest_at(out, bits, 0));
  pmp_stream *s = pmp_stream_new(k);
  if (!s) return 1;
  const uint64_t c1 = total / 3, c2 = 2 * total / 3 + 1 < total ? 2 * total / 3 + 1 : total;
  CK(pmp_stream_update(s, d_bytes, c1, st));
  CK(pmp_stream_update(s, d_bytes + c1, c2 - c1, st));
  CK(pmp_stream_update(s, d_bytes + c2, total - c2, st));
  CK(pmp_stream_final(s, d_out, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaMemcpy(out, d_out, w, cudaMemcpyDeviceToHost));
  printf("stream %016" PRIx64 "\n", digest_at(out, bits, 0));
  pmp_stream_free(s);

  /* the concatenation from pinned HOST memory, streamed in 2 KiB pieces */
  uint64_t hdig = 0;
  CK(pmp_hash_long_host(k, bytes, total, &hdig, 2048, st));
  CU(cudaStreamSynchronize(st));
  printf("longhost %016" PRIx64 "\n", bits == 64 ? hdig : (uint64_t)(uint32_t)hdig);

  /* the latency path (k_small) and the throughput path give the same digests */
  const uint64_t prev = pmp_set_small_batch_max(0);
  CK(pmp_hash_batch(k, d_bytes, d_off, n, d_out, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaMemcpy(out, d_out, n * w, cudaMemcpyDeviceToHost));
  pmp_set_small_batch_max(prev);
  for (uint64_t i = 0; i < n; i++) printf("tput %" PRIu64 " %016" PRIx64 "\n", i, digest_at(out, bits, i));

  /* errors are reported, not crashed on */
  printf("einval %d\n", pmp_hash_batch(k, NULL, d_off, n ? n : 1, d_out, st));
  pmp_keys_free(k);
  cudaFree(d_bytes);
  cudaFree(d_off);
  cudaFree(d_out);
  cudaFreeHost(bytes);
  cudaFreeHost(hout);
  free(out);
  free(off);
  return 0;
}
