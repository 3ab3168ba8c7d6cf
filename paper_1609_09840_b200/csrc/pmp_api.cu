#include <cstdio>
#include <cstdlib>
// pmp_api.cu -- libpmp.so: the C ABI declared in include/pmp.h.
//
// Host side of the PM+ path: key generation (project contract, reading Q12),
// argument checks, tree geometry, the key-only constant of the affine split,
// stream-ordered scratch, kernel launches and launch instrumentation.  Every
// step of the hash itself runs in the kernels of pmp_kernels.cuh; there is no
// CPU fallback.
#include "../../include/pmp.h"
#include "pmp_kernels.cuh"
#include "pmp_poly.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace pmp;

struct pmp_keys {
  int bits;
  uint64_t b[kL];
  uint64_t a[kL * kM];
  int device;       // -1: host-only handle
  uint64_t *d_blob; // device: b[8] then a[8*128], then the two-level variant's power tables
  // the power tables are built on first use of the two-level variant (ensure_poly)
  mutable std::atomic<int> poly_ready{0};
  mutable std::mutex poly_mu;
};

namespace {

typedef unsigned __int128 u128;

uint64_t amax_of(int bits) {  // p - kappa - 1
  return bits == 64 ? 0xFFFFFFFFFFFFFFF4ULL /* 2^64 - 12 */ : 0xFFFFFFF2ULL /* 2^32 - 14 */;
}
u128 prime_of(int bits) { return bits == 64 ? (((u128)1 << 64) + 13) : (((u128)1 << 32) + 15); }

// A private non-blocking stream per device for key uploads and one-time table
// setup, so that creating a handle never synchronises the whole device.
cudaStream_t util_stream(int dev);

int upload(pmp_keys *k) {
  k->device = -1;
  k->d_blob = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return 0;  // host-only handle
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PMP_ECUDA;
  std::vector<uint64_t> blob(kL + kL * kM);  // b, a (the variant's tables follow, built lazily)
  memcpy(blob.data(), k->b, sizeof(k->b));
  memcpy(blob.data() + kL, k->a, sizeof(k->a));
  if (cudaMalloc(&k->d_blob, (size_t)kBlobWords * 8) != cudaSuccess) return PMP_ENOMEM;
  cudaStream_t us = util_stream(dev);
  if (!us || cudaMemcpyAsync(k->d_blob, blob.data(), blob.size() * 8, cudaMemcpyHostToDevice, us) != cudaSuccess ||
      cudaStreamSynchronize(us) != cudaSuccess) {
    cudaFree(k->d_blob);
    k->d_blob = nullptr;
    return PMP_ECUDA;
  }
  k->poly_ready.store(0);
  k->device = dev;
  return 0;
}

// The two-level variant's power tables W[i] = r^(128-i) and the ladder R^(2^k)
// (pmp_poly.cuh), built once per handle before its first two-level call.
int ensure_poly(const pmp_keys *k) {
  if (k->poly_ready.load(std::memory_order_acquire)) return 0;
  std::lock_guard<std::mutex> lk(k->poly_mu);
  if (k->poly_ready.load(std::memory_order_relaxed)) return 0;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != k->device) cudaSetDevice(k->device);
  cudaStream_t us = util_stream(k->device);
  int rc = 0;
  if (!us) {
    rc = PMP_ECUDA;
  } else {
    if (k->bits == 64) k_poly_setup<64><<<1, 32, 0, us>>>(k->d_blob);
    else k_poly_setup<32><<<1, 32, 0, us>>>(k->d_blob);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(us) != cudaSuccess) rc = PMP_ECUDA;
  }
  if (cur != k->device) cudaSetDevice(cur);
  if (!rc) k->poly_ready.store(1, std::memory_order_release);
  return rc;
}

// ----------------------------------------------------------------- device info
struct DevInfo {
  int sms = 0;
  bool init = false;
};
std::mutex g_mu;
DevInfo g_dev[64];

cudaStream_t util_stream(int dev) {
  static cudaStream_t us[64] = {};
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!us[dev]) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != dev) cudaSetDevice(dev);
    if (cudaStreamCreateWithFlags(&us[dev], cudaStreamNonBlocking) != cudaSuccess) us[dev] = nullptr;
    if (cur != dev) cudaSetDevice(cur);
  }
  return us[dev];
}

int sm_count(int dev) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (dev < 0 || dev >= 64) return 148;
  if (!g_dev[dev].init) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_dev[dev].sms = v > 0 ? v : 148;
    // keep stream-ordered scratch cached in the device's default pool instead
    // of returning it to the OS at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_dev[dev].init = true;
  }
  return g_dev[dev].sms;
}

// ----------------------------------------------------------------- instrumentation
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_small_max{kSmallMax};  // batches of <= this many strings take k_small
// throughput path: strings of >= g_huge_min bytes (at most g_huge_cap per call)
// are hashed node-parallel by k_huge instead of one warp each (pmp_huge.cuh)
#ifndef PMP_HUGE_MIN_DEFAULT
#define PMP_HUGE_MIN_DEFAULT (4ull << 20)
#endif
std::atomic<uint64_t> g_huge_min{PMP_HUGE_MIN_DEFAULT};
std::atomic<uint32_t> g_huge_cap{65536};
// short strings: 1 = k_short_tc (the level-1 sum on the tensor cores) for the
// tree variant without buckets, 0 = k_short's word loop; -1 = not chosen yet
// (environment PMP_SHORT_TC, default 0 while the tensor-core kernel is not faster)
std::atomic<int> g_short_tc{-1};
static bool use_short_tc() {
  int v = g_short_tc.load(std::memory_order_relaxed);
  if (v < 0) {
    const char *e = getenv("PMP_SHORT_TC");
    v = (e && e[0] == '1') ? 1 : 0;
    int expect = -1;
    g_short_tc.compare_exchange_strong(expect, v);
    v = g_short_tc.load(std::memory_order_relaxed);
  }
  return v != 0;
}
std::atomic<int> g_prof{0};
struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::vector<ProfRec> g_pending;
std::vector<std::pair<std::string, std::pair<double, uint64_t>>> g_done;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t get_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <class F>
int launch(const char *name, cudaStream_t st, F &&f) {
  const bool prof = g_prof.load(std::memory_order_relaxed) != 0;
  cudaEvent_t a = nullptr, b = nullptr;
  if (prof) {
    std::lock_guard<std::mutex> lk(g_mu);
    a = get_event();
    b = get_event();
  }
  if (prof) cudaEventRecord(a, st);
  f();
  cudaError_t e = cudaGetLastError();
  if (prof) {
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> lk(g_mu);
    g_pending.push_back({name, a, b});
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return e == cudaSuccess ? 0 : PMP_ECUDA;
}

int check_keys(const pmp_keys *k) {
  if (!k) return PMP_EINVAL;
  if (!k->d_blob) return PMP_ENODEV;
  return 0;
}

ParamKeys param_keys(const pmp_keys *k) {
  ParamKeys pk;
  for (int i = 0; i < 32; i++) pk.a[i] = k->a[i];
  pk.b = k->b[0];
  pk.r = k->a[kM];  // a_{2,1}
  pk.b2 = k->b[1];
  pk.huge_min = ~0ull;   // (the throughput path sets its own, hash_batch_impl)
  pk.huge_cap = 0;
  return pk;
}

// ----------------------------------------------------------------- geometry
int chunk_bytes(int bits) { return bits == 64 ? 1024 : 512; }
uint64_t words_of(int bits, uint64_t len) { return len / (uint64_t)(bits / 8) + 1; }

// C = root value of the tree whose level-1 values are all 0.  At
// level j >= 2 every node except the last of its level has 128 children that
// are themselves non-last nodes, so two values per level suffice.
u128 long_constant(const pmp_keys *k, uint64_t len) {
  const Geom gm = make_geom(words_of(k->bits, len));
  if (gm.leff <= 1) return 0;
  const u128 p = prime_of(k->bits);
  u128 cf = 0, cl = 0;  // level 1: all zero
  for (int j = 2; j <= gm.leff; j++) {
    const uint64_t *aj = k->a + (uint64_t)(j - 1) * kM;
    const uint64_t nprev = gm.T[j - 1], ncur = gm.T[j];
    const uint64_t last_children = nprev - 128 * (ncur - 1);
    u128 nf = k->b[j - 1] % p, nl = k->b[j - 1] % p;
    for (uint64_t r = 0; r < 128; r++) nf = (nf + ((u128)aj[r] * cf) % p) % p;
    for (uint64_t r = 0; r + 1 < last_children; r++) nl = (nl + ((u128)aj[r] * cf) % p) % p;
    nl = (nl + ((u128)aj[last_children - 1] * cl) % p) % p;
    cf = nf;
    cl = nl;
  }
  return cl;
}

const char *kErr[] = {"ok", "invalid argument", "string too long (> 2^56-1 words)", "CUDA error",
                      "out of memory", "no CUDA device for this key handle",
                      "bad key file (magic or length)", "unsupported key file version, word size or levels",
                      "key out of range"};

struct Scratch {
  void *p = nullptr;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  int alloc(size_t n) { return cudaMallocAsync(&p, n, st) == cudaSuccess ? 0 : PMP_ENOMEM; }
  ~Scratch() {
    if (p) cudaFreeAsync(p, st);
  }
};

template <int BITS>
int long_partial_impl(const pmp_keys *k, const uint8_t *local, uint64_t local_len, uint64_t g0,
                      uint64_t total, uint64_t *partial, cudaStream_t st) {
  const uint64_t CB = (uint64_t)chunk_bytes(BITS);
  const Geom gm = make_geom(words_of(BITS, total));
  StrView s;
  s.base = local;
  s.g0 = g0;
  s.avail_end = g0 + local_len;
  s.B = total;
  s.delta = (uint32_t)((uintptr_t)local & 15);
  // The tail block (the one holding the marker word) belongs to the one
  // range that holds the last byte, total - 1, so an empty range never owns it
  // (several empty ranges may end at `total`).  For total == 0 no range owns
  // it: the whole value is sigma_0 = 1 (reading Q2), added by the combine.
  const bool owns_tail = local_len > 0 && g0 + local_len == total;
  const uint64_t cb = g0 / CB;
  const uint64_t ce = owns_tail ? gm.T[1] : (g0 + local_len) / CB;
  const int sms = sm_count(k->device);
  if (gm.leff <= 1) {  // one level-1 block (or none): only the caller holding byte 0 contributes
    if (cb == 0 && ce >= 1) {
      return launch("k_node", st, [&] { k_node<BITS><<<1, kWWarps * 32, 0, st>>>(k->d_blob, s, 0, 1, 0, 1, 1, partial); });
    }
    return cudaMemsetAsync(partial, 0, 16, st) == cudaSuccess ? 0 : PMP_ECUDA;
  }
  if (ce <= cb) return cudaMemsetAsync(partial, 0, 16, st) == cudaSuccess ? 0 : PMP_ECUDA;
  // level-2 nodes [qb, qe) and the index ranges of every upper level
  uint64_t lo[kL + 1], hi[kL + 1];
  lo[2] = cb / 128;
  hi[2] = (ce + 127) / 128;
  size_t total_vals = 0;
  for (int j = 2; j <= gm.leff; j++) {
    if (j > 2) {
      lo[j] = lo[j - 1] / 128;
      hi[j] = (hi[j - 1] + 127) / 128;
    }
    if (j < gm.leff) total_vals += hi[j] - lo[j];
  }
  Scratch sc(st);
  if (total_vals && sc.alloc(total_vals * 16)) return PMP_ENOMEM;
  uint64_t *buf = (uint64_t *)sc.p;
  uint64_t *lvl[kL + 1];
  size_t off = 0;
  for (int j = 2; j <= gm.leff; j++) {
    if (j == gm.leff) {
      lvl[j] = partial;  // top level: exactly one node (index 0)
    } else {
      lvl[j] = buf + 2 * off;
      off += hi[j] - lo[j];
    }
  }
  {
    const uint64_t nodes = hi[2] - lo[2];
    const uint64_t maxgrid = (uint64_t)sms * 16;
    uint64_t grid = (nodes + kWWarps - 1) / kWWarps;
    if (grid > maxgrid) grid = maxgrid;
    int rc = launch("k_node", st, [&] {
      k_node<BITS><<<(unsigned)grid, kWWarps * 32, 0, st>>>(k->d_blob, s, cb, ce, lo[2], hi[2], 0, lvl[2]);
    });
    if (rc) return rc;
  }
  for (int j = 3; j <= gm.leff; j++) {
    const uint64_t nodes = hi[j] - lo[j];
    uint64_t grid = (nodes + kWWarps - 1) / kWWarps;
    if (grid > (uint64_t)sms * 16) grid = (uint64_t)sms * 16;
    int rc = launch("k_level", st, [&] {
      k_level<BITS><<<(unsigned)grid, kWWarps * 32, 0, st>>>(k->d_blob, j, lvl[j - 1], lo[j - 1],
                                                             hi[j - 1] - lo[j - 1], lvl[j], lo[j], nodes);
    });
    if (rc) return rc;
  }
  return 0;
}

// Two-level variant (8(f4)): sum over the caller's chunks [cb, ce) of
// v_c r^(C-c) (pmp_poly.cuh), into `dst` as a field element (final == 0) or,
// with b_2 added, as the digest (final == 1).
template <int BITS>
int poly_long_impl(const pmp_keys *k, const uint8_t *local, uint64_t local_len, uint64_t g0, uint64_t total,
                   int final, void *dst, cudaStream_t st) {
  const uint64_t CB = (uint64_t)chunk_bytes(BITS);
  const uint64_t C = (words_of(BITS, total) + 127) / 128;
  StrView s;
  s.base = local;
  s.g0 = g0;
  s.avail_end = g0 + local_len;
  s.B = total;
  s.delta = (uint32_t)((uintptr_t)local & 15);
  // tail chunk: owned by the range holding byte total - 1; the empty message
  // (total == 0) has no such range, so there the caller passing g0 == 0 owns
  // it -- a split of the empty message must be a single range (pmp.h)
  const bool owns_tail = g0 + local_len == total && (local_len > 0 || total == 0);
  const uint64_t cb = g0 / CB;
  const uint64_t ce = owns_tail ? C : (g0 + local_len) / CB;
  const int sms = sm_count(k->device);
  uint64_t grid = 1;
  if (ce > cb) {
    const uint64_t d = (128 - C % 128) % 128;
    const uint64_t nodes = (ce - 1 + d) / 128 - (cb + d) / 128 + 1;
    grid = (nodes + kWWarps - 1) / kWWarps;
    if (grid > (uint64_t)sms * 16) grid = (uint64_t)sms * 16;
  }
  Scratch sc(st);
  if (sc.alloc(grid * 16)) return PMP_ENOMEM;
  uint64_t *parts = (uint64_t *)sc.p;
  int rc;
  if (ce > cb) {
    rc = launch("k_poly_node", st, [&] {
      k_poly_node<BITS><<<(unsigned)grid, kWWarps * 32, 0, st>>>(k->d_blob, s, cb, ce, C, parts);
    });
  } else {
    rc = cudaMemsetAsync(parts, 0, 16, st) == cudaSuccess ? 0 : PMP_ECUDA;
  }
  if (rc) return rc;
  return launch("k_poly_sum", st, [&] { k_poly_sum<BITS><<<1, 256, 0, st>>>(k->d_blob, parts, grid, final, dst); });
}

int poly_args(const pmp_keys *k, const uint8_t *local, uint64_t local_len, uint64_t g0, uint64_t total) {
  if (!k || (!local && local_len > 0)) return PMP_EINVAL;
  if (words_of(k->bits, total) > (1ULL << 56)) return PMP_ETOOLONG;
  const uint64_t CB = (uint64_t)chunk_bytes(k->bits);
  if (g0 % CB != 0 || g0 + local_len > total || g0 + local_len < g0) return PMP_EINVAL;
  if (g0 + local_len != total && local_len % CB != 0) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  return ensure_poly(k);
}

}  // namespace

struct pmp_stream {
  const pmp_keys *k;
  StreamState *d_state;
  uint8_t *d_tail;      // < one level-1 block of pending bytes (+16 B read slack)
  uint64_t *d_s2;       // scratch for node partial sums
  size_t s2_cap;        // entries (pairs)
  uint64_t tail_len, c_done;
  bool finalized;
};

namespace {
template <int BITS>
int stream_range(pmp_stream *s, const uint8_t *base, uint64_t c0, uint64_t N, cudaStream_t st) {
  const uint64_t CB = (uint64_t)chunk_bytes(BITS);
  const uint64_t qb = c0 / 128, qe = (c0 + N + 127) / 128, nq = qe - qb;
  const int sms = sm_count(s->k->device);
  int P = 1;  // pieces per node: keep >= 32 warps per SM busy on short updates
  while (P < 32 && nq * (uint64_t)P < (uint64_t)sms * 32) P *= 2;
  const uint64_t need = nq * (uint64_t)P;
  if (need > s->s2_cap) {  // s2 (nq * P partials), two merge value arrays, per-node piece counters
    uint64_t *p = nullptr;
    if (cudaMallocAsync(&p, 3 * need * 16 + need * 4, st) != cudaSuccess) return PMP_ENOMEM;
    if (cudaMemsetAsync(p + 6 * need, 0, need * 4, st) != cudaSuccess) return PMP_ECUDA;
    if (s->d_s2) cudaFreeAsync(s->d_s2, st);
    s->d_s2 = p;
    s->s2_cap = need;
  }
  StrView v;
  v.base = base;
  v.g0 = c0 * CB;
  v.avail_end = v.g0 + N * CB;
  v.B = ~0ULL;  // no marker inside an update: every block is full
  v.delta = (uint32_t)((uintptr_t)base & 15);
  uint64_t grid = (need + kWWarps - 1) / kWWarps;
  if (grid > (uint64_t)sms * 16) grid = (uint64_t)sms * 16;
  return launch("k_stream_node", st, [&] {
    k_stream_node<BITS><<<(unsigned)grid, kWWarps * 32, 0, st>>>(s->k->d_blob, v, c0, N, qb, qe, P, s->d_s2,
                                                                   (uint32_t *)(s->d_s2 + 6 * s->s2_cap),
                                                                   s->d_state, s->d_s2 + 2 * s->s2_cap,
                                                                   s->d_s2 + 4 * s->s2_cap);
  });
}

template <int BITS>
int stream_update(pmp_stream *s, const uint8_t *data, uint64_t len, cudaStream_t st) {
  const uint64_t CB = (uint64_t)chunk_bytes(BITS);
  if (s->tail_len > 0 || len < CB) {
    const uint64_t fill = min(len, CB - s->tail_len);
    if (fill && cudaMemcpyAsync(s->d_tail + s->tail_len, data, fill, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return PMP_ECUDA;
    s->tail_len += fill;
    data += fill;
    len -= fill;
    if (s->tail_len < CB) return 0;
    if (int rc = stream_range<BITS>(s, s->d_tail, s->c_done, 1, st)) return rc;
    s->c_done += 1;
    s->tail_len = 0;
  }
  const uint64_t N = len / CB;
  if (N) {
    if (int rc = stream_range<BITS>(s, data, s->c_done, N, st)) return rc;
    s->c_done += N;
    data += N * CB;
    len -= N * CB;
  }
  if (len) {
    if (cudaMemcpyAsync(s->d_tail, data, len, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return PMP_ECUDA;
    s->tail_len = len;
  }
  return 0;
}

template <int BITS>
int stream_final(pmp_stream *s, void *out, cudaStream_t st) {
  const uint64_t CB = (uint64_t)chunk_bytes(BITS);
  const uint64_t Btot = s->c_done * CB + s->tail_len;
  const int leff = levels_of(words_of(BITS, Btot));
  if (s->s2_cap < 1) {
    if (cudaMallocAsync(&s->d_s2, 3 * 16 + 4, st) != cudaSuccess) return PMP_ENOMEM;
    if (cudaMemsetAsync(s->d_s2 + 6, 0, 4, st) != cudaSuccess) return PMP_ECUDA;
    s->s2_cap = 1;
  }
  StrView v;
  v.base = s->d_tail;
  v.g0 = s->c_done * CB;
  v.avail_end = v.g0 + s->tail_len;
  v.B = Btot;
  v.delta = 0;
  int rc;
  if (s->c_done == 0) {  // the whole string is in the tail: one block or less
    v.g0 = 0;
    rc = launch("k_node", st, [&] { k_node<BITS><<<1, kWWarps * 32, 0, st>>>(s->k->d_blob, v, 0, 1, 0, 1, 1, s->d_s2); });
  } else {               // the last block (tail bytes + marker) of node c_done / 128
    const uint64_t c = s->c_done;
    rc = launch("k_node", st, [&] {
      k_node<BITS><<<1, kWWarps * 32, 0, st>>>(s->k->d_blob, v, c, c + 1, c / 128, c / 128 + 1, 0, s->d_s2);
    });
  }
  if (rc) return rc;
  return launch("k_stream_final", st, [&] {
    k_stream_final<BITS><<<1, 32, 0, st>>>(s->k->d_blob, s->d_state, s->d_s2, leff, out);
  });
}
}  // namespace

// =================================================================== C ABI
extern "C" {

pmp_stream *pmp_stream_new(const pmp_keys *k) {
  if (!k || !k->d_blob) return nullptr;
  pmp_stream *s = new (std::nothrow) pmp_stream;
  if (!s) return nullptr;
  s->k = k;
  s->d_state = nullptr;
  s->d_tail = nullptr;
  s->d_s2 = nullptr;
  s->s2_cap = 0;
  s->tail_len = s->c_done = 0;
  s->finalized = false;
  if (cudaMalloc(&s->d_state, sizeof(StreamState)) != cudaSuccess ||
      cudaMalloc(&s->d_tail, (size_t)chunk_bytes(k->bits) + 32) != cudaSuccess ||
      cudaMemset(s->d_state, 0, sizeof(StreamState)) != cudaSuccess) {
    if (s->d_state) cudaFree(s->d_state);
    if (s->d_tail) cudaFree(s->d_tail);
    delete s;
    return nullptr;
  }
  return s;
}

int pmp_stream_update(pmp_stream *s, const uint8_t *bytes, uint64_t len, cudaStream_t st) {
  if (!s || (!bytes && len) || s->finalized) return PMP_EINVAL;
  if (len == 0) return 0;
  const uint64_t CB = (uint64_t)chunk_bytes(s->k->bits);
  if (words_of(s->k->bits, s->c_done * CB + s->tail_len + len) > (1ULL << 56)) return PMP_ETOOLONG;
  return s->k->bits == 64 ? stream_update<64>(s, bytes, len, st) : stream_update<32>(s, bytes, len, st);
}

int pmp_stream_final(pmp_stream *s, void *out, cudaStream_t st) {
  if (!s || !out || s->finalized) return PMP_EINVAL;
  s->finalized = true;
  return s->k->bits == 64 ? stream_final<64>(s, out, st) : stream_final<32>(s, out, st);
}

int pmp_stream_reset(pmp_stream *s, cudaStream_t st) {
  if (!s) return PMP_EINVAL;
  s->tail_len = s->c_done = 0;
  s->finalized = false;
  return cudaMemsetAsync(s->d_state, 0, sizeof(StreamState), st) == cudaSuccess ? 0 : PMP_ECUDA;
}

void pmp_stream_free(pmp_stream *s) {
  if (!s) return;
  cudaDeviceSynchronize();
  cudaFree(s->d_state);
  cudaFree(s->d_tail);
  if (s->d_s2) cudaFree(s->d_s2);
  delete s;
}


const char *pmp_strerror(int code) {
  if (code > 0 || code < -8) return "unknown error";
  return kErr[-code];
}

pmp_keys *pmp_keygen(uint64_t seed, int out_bits) {
  if (out_bits != 32 && out_bits != 64) return nullptr;
  pmp_keys *k = new (std::nothrow) pmp_keys;
  if (!k) return nullptr;
  k->bits = out_bits;
  KeyStream g;  // the key-generation contract, reading Q12 (pmp_common.cuh)
  g.init(seed, out_bits);
  for (uint32_t j = 0; j < kL; j++) {
    k->b[j] = g.draw_b();
    for (uint32_t i = 0; i < kM; i++) k->a[j * kM + i] = g.draw_a();
  }
  if (upload(k) != 0) {
    delete k;
    return nullptr;
  }
  return k;
}

pmp_keys *pmp_keys_from_words(int out_bits, const uint64_t *b, const uint64_t *a) {
  if ((out_bits != 32 && out_bits != 64) || !b || !a) return nullptr;
  const uint64_t amax = amax_of(out_bits);
  for (uint32_t j = 0; j < kL; j++) {
    if (out_bits == 32 && b[j] >> 32) return nullptr;
    for (uint32_t i = 0; i < kM; i++)
      if (a[j * kM + i] == 0 || a[j * kM + i] > amax) return nullptr;
  }
  pmp_keys *k = new (std::nothrow) pmp_keys;
  if (!k) return nullptr;
  k->bits = out_bits;
  memcpy(k->b, b, sizeof(k->b));
  memcpy(k->a, a, sizeof(k->a));
  if (upload(k) != 0) {
    delete k;
    return nullptr;
  }
  return k;
}

int pmp_keys_export(const pmp_keys *k, uint64_t *b, uint64_t *a) {
  if (!k || !b || !a) return PMP_EINVAL;
  memcpy(b, k->b, sizeof(k->b));
  memcpy(a, k->a, sizeof(k->a));
  return 0;
}

int pmp_keys_bits(const pmp_keys *k) { return k ? k->bits : PMP_EINVAL; }

uint64_t pmp_keyfile_size(int out_bits) {
  if (out_bits != 32 && out_bits != 64) return 0;
  return 8 + (uint64_t)kL * (1 + kM) * (out_bits / 8);
}

int pmp_keys_save(const pmp_keys *k, uint8_t *out, uint64_t cap) {
  if (!k || !out || cap < pmp_keyfile_size(k->bits)) return PMP_EINVAL;
  const int w = k->bits / 8;
  memcpy(out, "PMPH", 4);
  out[4] = 0x01;
  out[5] = (uint8_t)k->bits;
  out[6] = (uint8_t)kL;
  out[7] = 0x00;
  uint8_t *p = out + 8;
  auto put = [&](uint64_t x) {
    for (int i = 0; i < w; i++) *p++ = (uint8_t)(x >> (8 * i));
  };
  for (uint32_t j = 0; j < kL; j++) {
    put(k->b[j]);
    for (uint32_t i = 0; i < kM; i++) put(k->a[j * kM + i]);
  }
  return 0;
}

pmp_keys *pmp_keys_load(const uint8_t *buf, uint64_t len, int *err) {
  int e = 0;
  if (!err) err = &e;
  *err = PMP_EINVAL;
  if (!buf) return nullptr;
  *err = PMP_EBADFILE;
  if (len < 8 || memcmp(buf, "PMPH", 4) != 0) return nullptr;
  const int bits = buf[5];
  *err = PMP_EVERSION;
  if (buf[4] != 0x01 || (bits != 32 && bits != 64) || buf[6] != kL || buf[7] != 0x00) return nullptr;
  *err = PMP_EBADFILE;
  if (len != pmp_keyfile_size(bits)) return nullptr;
  const int w = bits / 8;
  const uint8_t *p = buf + 8;
  auto get = [&]() {
    uint64_t x = 0;
    for (int i = 0; i < w; i++) x |= (uint64_t)*p++ << (8 * i);
    return x;
  };
  pmp_keys *k = new (std::nothrow) pmp_keys;
  *err = PMP_ENOMEM;
  if (!k) return nullptr;
  k->bits = bits;
  k->device = -1;
  k->d_blob = nullptr;
  const uint64_t amax = amax_of(bits);
  for (uint32_t j = 0; j < kL; j++) {
    k->b[j] = get();  // a w-byte word is < 2^n by construction
    for (uint32_t i = 0; i < kM; i++) {
      const uint64_t a = get();
      if (a == 0 || a > amax) {
        delete k;
        *err = PMP_EKEYRANGE;
        return nullptr;
      }
      k->a[j * kM + i] = a;
    }
  }
  if (upload(k) != 0) {
    delete k;
    *err = PMP_ENOMEM;
    return nullptr;
  }
  *err = 0;
  return k;
}

void pmp_keys_free(pmp_keys *k) {
  if (!k) return;
  if (k->d_blob) cudaFree(k->d_blob);
  delete k;
}

// A launch with programmatic dependent launch (PDL): the grid may be scheduled
// before the previous kernel on the stream completes; it must start with
// griddepcontrol.wait before touching that kernel's results (k_wstring).
static void launch_pdl(const void *f, unsigned grid, unsigned threads, void **args, size_t smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelExC(&cfg, f, args);
}

// Resident blocks per SM of k_short_tc from its resources (registers, shared
// memory, threads, TMEM columns).
static int tc_resident_blocks(const void *f, int threads, size_t smem, int device) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return 1;
  int smem_sm = 0, regs_sm = 0, thr_sm = 0;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, device);
  cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, device);
  const int warps = (threads + 31) / 32;
  const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
  int b = (int)(smem_sm / (smem + fa.sharedSizeBytes + 1024));
  b = std::min(b, regs_sm / std::max(1, regs_warp * warps));
  b = std::min(b, thr_sm / threads);
  b = std::min(b, (int)(512 / kTcTmemCols));
  if (getenv("PMP_VERBOSE")) fprintf(stderr, "pmp: k_short_tc %d blocks/SM from its resources\n", b);
  return std::max(b, 1);
}

// Resident blocks per SM of a kernel (registers, shared memory), cached per
// kernel: the persistent grids are exactly one wave.  tc_device >= 0: the
// tensor-core kernel, counted from its resources -- the occupancy calculator
// reports 1 block/SM for it (it uses TMEM); registers, shared memory and TMEM
// columns (512 per SM, kTcTmemCols per block) admit 2, and 2 co-reside
// (measured: 0.336 -> 0.266 ms on configs[1]).
static int resident_blocks(const void *f, int threads, size_t smem, const char *name, int tc_device = -1) {
  static std::mutex mu;
  static std::vector<std::pair<const void *, int>> cache;
  std::lock_guard<std::mutex> lk(mu);
  for (auto &e : cache)
    if (e.first == f) return e.second;
  int b = 0;
  if (tc_device >= 0) b = tc_resident_blocks(f, threads, smem, tc_device);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, f, threads, smem);
  if (b < 1) b = 1;
  if (getenv("PMP_VERBOSE")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, f);
    fprintf(stderr, "pmp: %s smem %zu B, %d blocks/SM (regs %d, static smem %zu, max dyn smem %d, carveout %d)\n",
            name, smem, b, fa.numRegs, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes,
            fa.preferredShmemCarveout);
  }
  cache.push_back({f, b});
  return b;
}

// One batch under schedule k (digests to os) and, for the dual-width fused
// short-string pass, a second schedule k2 (k 64-bit, k2 32-bit, tree only;
// digests to *os2): short strings are read once for both, long strings (the
// work list, shared) are hashed per schedule by k_wstring.
static int hash_batch_impl(const pmp_keys *k, const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                           const OutSpec &os, cudaStream_t st, bool v2 = false, const pmp_keys *k2 = nullptr,
                           const OutSpec *os2 = nullptr) {
  if (!k) return PMP_EINVAL;
  if (n == 0) return 0;
  if (!bytes || !offsets || !os.out || n >= (1ULL << 32)) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  const bool dual = k2 != nullptr;
  if (dual && (!os2 || !os2->out || k->bits != 64 || k2->bits != 32 || k2->device != k->device))
    return PMP_EINVAL;
  if (v2) {
    if (int rc = ensure_poly(k)) return rc;
    if (dual)
      if (int rc = ensure_poly(k2)) return rc;
  }
  const int sms = sm_count(k->device);
  ParamKeys pk = param_keys(k);
  if (dual) {
    for (int i = 0; i < 32; i++) pk.a32[i] = (uint32_t)k2->a[i];
    pk.b32 = k2->b[0];
    pk.r32 = k2->a[kM];   // a_{2,1}
    pk.b2_32 = k2->b[1];
  }
  if (!v2 && n <= g_small_max.load(std::memory_order_relaxed)) {
    // latency path: one launch, no scratch, no work list (pmp_small.cuh)
    // strings per block: kSmallPer, or fewer for batches that do not fill ~2
    // blocks per SM, so the spare warps split long strings (pmp_split.cuh)
    const uint64_t per = std::min<uint64_t>(kSmallPer, std::max<uint64_t>(1, (n + 2 * sms - 1) / (2 * sms)));
    const unsigned grid = (unsigned)((n + per - 1) / per);
    const uint32_t per32 = (uint32_t)per;
    const uint64_t *b1 = k->d_blob, *b2 = dual ? k2->d_blob : k->d_blob;
    const OutSpec o2 = dual ? *os2 : os;
    return launch("k_small", st, [&] {
      if (dual) k_small<64, true><<<grid, kSmallThreads, 0, st>>>(pk, b1, b2, bytes, offsets, n, os, o2, per32);
      else if (k->bits == 64) k_small<64, false><<<grid, kSmallThreads, 0, st>>>(pk, b1, b2, bytes, offsets, n, os, o2, per32);
      else k_small<32, false><<<grid, kSmallThreads, 0, st>>>(pk, b1, b2, bytes, offsets, n, os, o2, per32);
    });
  }
  Scratch sc(st), sc_off(st);
  // counters [mid, big, then per schedule: next big, next mid batch; k_short
  // tile claims; huge capacity, slots and parts; part cursors] + work list (n u32) + huge list
  // and states (pmp_huge_list.cuh; the two-level variant has none)
  const uint64_t huge_min = v2 ? ~0ull : std::max<uint64_t>(g_huge_min.load(), kBigBytes);
  const uint32_t huge_cap = v2 ? 0u : (uint32_t)std::min<uint64_t>(n, g_huge_cap.load());
  pk.huge_min = huge_cap ? huge_min : ~0ull;
  pk.huge_cap = huge_cap;
  if (sc.alloc((size_t)(kWHeader + n + huge_cap) * 4 + 16 + (size_t)huge_cap * kHugeState * 8)) return PMP_ENOMEM;
  uint32_t *wcount = (uint32_t *)sc.p;
  uint32_t *wlist = wcount + kWHeader;
  if (cudaMemsetAsync(wcount, 0, kWHeader * 4, st) != cudaSuccess) return PMP_ECUDA;
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    const void *fs[8] = {(const void *)k_short<64>, (const void *)k_short<32>, (const void *)k_short<64, true>,
                         (const void *)k_short<32, true>, (const void *)k_short<64, false, true>,
                         (const void *)k_short<64, true, true>, (const void *)k_short<64, false, false, true>,
                         (const void *)k_short<32, false, false, true>};
    for (const void *f : fs) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kShortSmem);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    }
    const void *ws[6] = {(const void *)k_wstring<64>, (const void *)k_wstring<32>, (const void *)k_wstring<64, true>,
                         (const void *)k_wstring<32, true>, (const void *)k_wstring_dual<false>,
                         (const void *)k_wstring_dual<true>};
    for (const void *f : ws) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWSmem);
    const void *ts[3] = {(const void *)k_short_tc<64, true>, (const void *)k_short_tc<64, false>,
                         (const void *)k_short_tc<32, false>};
    for (const void *f : ts) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    }
  });
  // the offsets ring is fed by TMA bulk copies, which need 16-byte aligned sources
  if ((uintptr_t)offsets & 15) {
    void *al = nullptr;
    if (cudaMallocAsync(&al, (size_t)(n + 1) * 8, st) != cudaSuccess) return PMP_ENOMEM;
    if (cudaMemcpyAsync(al, offsets, (size_t)(n + 1) * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return PMP_ECUDA;
    sc_off.p = al;
    offsets = (const uint64_t *)al;
  }
  // ---- short strings (and the work list of long ones)
  // (buckets, os.M != 0: the instantiations with the bucket code; the hot ones store digests only)
  const bool bkt = os.M != 0;
  if (bkt && (dual || v2)) return PMP_EINVAL;
  const void *kshort = bkt ? (k->bits == 64 ? (const void *)k_short<64, false, false, true>
                                            : (const void *)k_short<32, false, false, true>)
                     : dual ? (v2 ? (const void *)k_short<64, true, true> : (const void *)k_short<64, false, true>)
                            : v2 ? (k->bits == 64 ? (const void *)k_short<64, true> : (const void *)k_short<32, true>)
                                 : (k->bits == 64 ? (const void *)k_short<64> : (const void *)k_short<32>);
  // (tree variant, digests: the tensor-core kernel, k_short_tc)
  const bool tcp = !bkt && !v2 && use_short_tc();
  const void *kshort_tc = dual ? (const void *)k_short_tc<64, true>
                               : (k->bits == 64 ? (const void *)k_short_tc<64, false> : (const void *)k_short_tc<32, false>);
  const void *ks = tcp ? kshort_tc : kshort;
  const int threads = tcp ? kTcThreads : kShortThreads;  // consumers + producer warps
  const size_t smem = tcp ? kTcSmem : kShortSmem;
  const uint64_t tile = tcp ? (uint64_t)kTcTile : (uint64_t)kTile;
  uint64_t grid = (n + tile - 1) / tile;
  int rb = resident_blocks(ks, threads, smem, tcp ? "k_short_tc" : "k_short", tcp ? k->device : -1);
  if (tcp)
    if (const char *e = getenv("PMP_TC_BLOCKS")) rb = atoi(e) > 0 ? atoi(e) : rb;   // (tuning)
  const uint64_t maxgrid = (uint64_t)sms * rb;  // persistent grid
  if (grid > maxgrid) grid = maxgrid;
  const OutSpec o2 = dual ? *os2 : os;
  int rc = launch(tcp ? "k_short_tc" : "k_short", st, [&] {
    void *args[] = {(void *)&pk, (void *)&bytes, (void *)&offsets, (void *)&n, (void *)&os, (void *)&wlist,
                    (void *)&wcount, (void *)&o2};
    cudaLaunchKernel(ks, dim3((unsigned)grid), dim3(threads), args, smem, st);
  });
  if (rc) return rc;
  // ---- long strings: warp per big string, 8-lane group per mid string (persistent
  // grid of exactly the resident blocks)
  auto launch_w = [&](const pmp_keys *kk, const OutSpec &o) -> int {
    const void *kw = v2 ? (kk->bits == 64 ? (const void *)k_wstring<64, true> : (const void *)k_wstring<32, true>)
                        : (kk->bits == 64 ? (const void *)k_wstring<64> : (const void *)k_wstring<32>);
    const unsigned wgrid = (unsigned)(sms * resident_blocks(kw, kWBlockWarps * 32, kWSmem, "k_wstring"));
    const uint64_t *blob = kk->d_blob;
    return launch("k_wstring", st, [&] {
      void *args[] = {(void *)&blob, (void *)&bytes, (void *)&offsets, (void *)&n, (void *)&o, (void *)&wlist,
                      (void *)&wcount};
      launch_pdl(kw, wgrid, kWBlockWarps * 32, args, kWSmem, st);
    });
  };
  // ---- huge strings (k_short's huge list), node-parallel; returns at once when empty
  auto launch_h = [&]() -> int {
    if (!huge_cap || tcp) return 0;   // (k_short_tc keeps every long string on the work list)
    const void *kh = dual ? (const void *)k_huge<64, true>
                          : (k->bits == 64 ? (const void *)k_huge<64, false> : (const void *)k_huge<32, false>);
    const unsigned hgrid = (unsigned)(sms * resident_blocks(kh, kHugeThreads, 0, "k_huge"));
    const uint64_t *hb1 = k->d_blob, *hb2 = dual ? k2->d_blob : k->d_blob;
    const OutSpec ho2 = dual ? *os2 : os;
    return launch("k_huge", st, [&] {
      void *args[] = {(void *)&hb1, (void *)&hb2, (void *)&bytes, (void *)&offsets, (void *)&n, (void *)&os,
                      (void *)&ho2, (void *)&wlist, (void *)&wcount};
      launch_pdl(kh, hgrid, kHugeThreads, args, 0, st);
    });
  };
  if (!dual) {
    if (int rc2 = launch_w(k, os)) return rc2;
    return launch_h();
  }
  // both schedules over the shared work list in one launch (half the blocks each)
  const void *kw = v2 ? (const void *)k_wstring_dual<true> : (const void *)k_wstring_dual<false>;
  const unsigned wgrid = (unsigned)(2 * ((sms * resident_blocks(kw, kWBlockWarps * 32, kWSmem, "k_wstring") + 1) / 2));
  const uint64_t *b64 = k->d_blob, *b32 = k2->d_blob;
  const OutSpec o32 = *os2;
  rc = launch("k_wstring", st, [&] {
    void *args[] = {(void *)&b64, (void *)&b32, (void *)&bytes, (void *)&offsets, (void *)&n, (void *)&os,
                    (void *)&o32, (void *)&wlist, (void *)&wcount};
    launch_pdl(kw, wgrid, kWBlockWarps * 32, args, kWSmem, st);
  });
  if (rc) return rc;
  return launch_h();
}

int pmp_hash_batch(const pmp_keys *k, const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                   void *out, cudaStream_t st) {
  OutSpec os;
  os.out = out;
  os.M = 0;
  os.counts = nullptr;
  return hash_batch_impl(k, bytes, offsets, n, os, st);
}

int pmp_hash_batch_buckets(const pmp_keys *k, const uint8_t *bytes, const uint64_t *offsets, uint64_t n,
                           uint32_t M, uint32_t *buckets, uint32_t *counts, cudaStream_t st) {
  if (M == 0) return PMP_EINVAL;
  OutSpec os;
  os.out = buckets;
  os.M = M;
  os.counts = nullptr;   // counted by k_histogram below, not by atomics in the hash kernels
  if (int rc = hash_batch_impl(k, bytes, offsets, n, os, st)) return rc;
  if (!counts || n == 0) return 0;
  const int sms = sm_count(k->device);
  const size_t smem = M <= kHistSmemMax ? (size_t)M * 4 : 0;
  uint64_t grid = (n + 511) / 512;
  if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
  return launch("k_histogram", st,
                [&] { k_histogram<<<(unsigned)grid, 512, smem, st>>>(buckets, n, M, counts); });
}

int pmp_bucket_partition(const uint32_t *buckets, uint64_t n, uint32_t M, const uint32_t *hist, uint64_t *starts,
                         uint32_t *perm, cudaStream_t st) {
  if (M == 0 || M > (1u << 24) || !starts || n >= (1ULL << 32) || (n && (!buckets || !perm))) return PMP_EINVAL;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return PMP_ENODEV;
  const int sms = sm_count(dev);
  Scratch sc(st);
  if (sc.alloc((size_t)M * 4)) return PMP_ENOMEM;
  uint32_t *counts = (uint32_t *)sc.p;
  const size_t smem = M <= kHistSmemMax ? (size_t)M * 4 : 0;
  if (hist) {                                            // the caller's histogram of these buckets
    if (cudaMemcpyAsync(counts, hist, (size_t)M * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return PMP_ECUDA;
  } else if (cudaMemsetAsync(counts, 0, (size_t)M * 4, st) != cudaSuccess) {
    return PMP_ECUDA;
  }
  if (n && !hist) {
    uint64_t grid = (n + 511) / 512;
    if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
    if (int rc = launch("k_histogram", st,
                        [&] { k_histogram<<<(unsigned)grid, 512, smem, st>>>(buckets, n, M, counts); }))
      return rc;
  }
  if (int rc = launch("k_part_scan", st, [&] { k_part_scan<<<1, 1024, 0, st>>>(counts, M, n, starts); })) return rc;
  if (n == 0) return 0;
  uint64_t grid = M <= kHistSmemMax ? (n + kPartChunk - 1) / kPartChunk : (n + kPartThreads - 1) / kPartThreads;
  if (grid > (uint64_t)sms * 4) grid = (uint64_t)sms * 4;
  const size_t psmem =
      PMP_PART_STAGE && M >= kPartStageMin && M <= kPartStageMax ? (size_t)M * 8 + (size_t)kPartChunk * 6 : smem;
  static std::once_flag part_attr;                       // 48 KB of counters + the static scan scratch
  std::call_once(part_attr, [] {
    cudaFuncSetAttribute(k_part_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  });
  return launch("k_part_scatter", st, [&] {
    k_part_scatter<<<(unsigned)grid, kPartThreads, psmem, st>>>(buckets, n, M, counts, perm);
  });
}

static int batch_multi_impl(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                            uint64_t n, void *const *outs, cudaStream_t st, bool v2) {
  if (!keys || !outs || nkeys < 1 || nkeys > PMP_HOST_MAX_KEYS) return PMP_EINVAL;
  for (int k = 0; k < nkeys; k++)
    if (!keys[k]) return PMP_EINVAL;
  if (n == 0) return 0;
  for (int k = 0; k < nkeys; k++)
    if (!outs[k]) return PMP_EINVAL;
  bool done[PMP_HOST_MAX_KEYS] = {false, false, false, false};
  // pair a 64-bit with a 32-bit schedule: one fused pass over the short strings
  for (int k = 0; k < nkeys; k++) {
    if (done[k] || keys[k]->bits != 64) continue;
    for (int j = 0; j < nkeys; j++) {
      if (done[j] || keys[j]->bits != 32 || keys[j]->device != keys[k]->device) continue;
      OutSpec a{outs[k], 0, nullptr}, b{outs[j], 0, nullptr};
      if (int rc = hash_batch_impl(keys[k], bytes, offsets, n, a, st, v2, keys[j], &b)) return rc;
      done[k] = done[j] = true;
      break;
    }
  }
  for (int k = 0; k < nkeys; k++) {
    if (done[k]) continue;
    OutSpec a{outs[k], 0, nullptr};
    if (int rc = hash_batch_impl(keys[k], bytes, offsets, n, a, st, v2)) return rc;
  }
  return 0;
}

int pmp_hash_batch_multi(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                         uint64_t n, void *const *outs, cudaStream_t st) {
  return batch_multi_impl(keys, nkeys, bytes, offsets, n, outs, st, false);
}

int pmp_hash2_batch_multi(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                          uint64_t n, void *const *outs, cudaStream_t st) {
  return batch_multi_impl(keys, nkeys, bytes, offsets, n, outs, st, true);
}

// Host-resident batches: string-aligned pieces streamed through the device on
// kHostSlots internal streams, so that the host->device copy of one piece, the
// hashing of another and the device->host copy of a third overlap (the copy
// engines of both directions and the SMs work at once).
namespace {
constexpr int kHostSlots = 3;
struct HostStreams {
  bool init = false;
  cudaStream_t st[kHostSlots];
};
HostStreams g_host_st[64];
}  // namespace

int pmp_hash_batch_host(const pmp_keys *const *keys, int nkeys, const uint8_t *bytes, const uint64_t *offsets,
                        uint64_t n, void *const *outs, uint64_t piece_bytes, cudaStream_t stream) {
  if (!keys || !outs || nkeys < 1 || nkeys > PMP_HOST_MAX_KEYS) return PMP_EINVAL;
  if (n == 0) return 0;
  if (!bytes || !offsets || n >= (1ULL << 32)) return PMP_EINVAL;
  for (int k = 0; k < nkeys; k++) {
    if (!keys[k] || !outs[k]) return PMP_EINVAL;
    if (int rc = check_keys(keys[k])) return rc;
    if (keys[k]->device != keys[0]->device) return PMP_EINVAL;
  }
  const int dev = keys[0]->device;
  if (dev < 0 || dev >= 64) return PMP_EINVAL;
  if (piece_bytes == 0) piece_bytes = 64ull << 20;
  // string-aligned pieces of <= piece_bytes payload (a longer string is a piece alone)
  std::vector<uint64_t> cut{0};
  uint64_t max_span = 0, max_cnt = 0;
  while (cut.back() < n) {
    const uint64_t s0 = cut.back();
    const uint64_t *e = std::upper_bound(offsets + s0 + 1, offsets + n + 1, offsets[s0] + piece_bytes);
    uint64_t s1 = (uint64_t)(e - offsets) - 1;
    if (s1 <= s0) s1 = s0 + 1;
    cut.push_back(s1);
    max_span = std::max(max_span, offsets[s1] - offsets[s0]);
    max_cnt = std::max(max_cnt, s1 - s0);
  }
  // everything below runs on the keys' device (its streams, its memory pool,
  // its kernels); the caller's current device is restored on return
  int cur_dev = 0;
  if (cudaGetDevice(&cur_dev) != cudaSuccess) return PMP_ECUDA;
  struct DevGuard {
    int prev, now;
    ~DevGuard() {
      if (prev != now) cudaSetDevice(prev);
    }
  } guard{cur_dev, dev};
  if (cur_dev != dev && cudaSetDevice(dev) != cudaSuccess) return PMP_ECUDA;
  if (cut.size() == 2) {
    // one piece (a small batch): nothing to overlap, so no internal streams or
    // events -- H2D, hash, D2H in order on the caller's stream, one scratch slab
    const uint64_t b0 = offsets[0], nb = offsets[n] - b0, sh = b0 & 15;
    const size_t cap_b = ((size_t)nb + 48 + 255) & ~(size_t)255, cap_o = ((size_t)(n + 1) * 8 + 255) & ~(size_t)255;
    const size_t cap_d = ((size_t)n * 8 + 255) & ~(size_t)255;
    uint8_t *slab = nullptr;
    if (cudaMallocAsync((void **)&slab, cap_b + cap_o + (size_t)nkeys * cap_d, stream) != cudaSuccess) return PMP_ENOMEM;
    uint64_t *d_o = (uint64_t *)(slab + cap_b);
    void *d_outs[PMP_HOST_MAX_KEYS];
    for (int k = 0; k < nkeys; k++) d_outs[k] = slab + cap_b + cap_o + (size_t)k * cap_d;
    int rc = 0;
    if (nb && cudaMemcpyAsync(slab + sh, bytes + b0, nb, cudaMemcpyHostToDevice, stream) != cudaSuccess) rc = PMP_ECUDA;
    if (!rc && cudaMemcpyAsync(d_o, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, stream) != cudaSuccess) rc = PMP_ECUDA;
    if (!rc) rc = pmp_hash_batch_multi(keys, nkeys, slab + sh - b0, d_o, n, d_outs, stream);
    for (int k = 0; k < nkeys && !rc; k++)
      if (cudaMemcpyAsync(outs[k], d_outs[k], n * (keys[k]->bits / 8), cudaMemcpyDeviceToHost, stream) != cudaSuccess)
        rc = PMP_ECUDA;
    cudaFreeAsync(slab, stream);
    return rc;
  }
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_host_st[dev].init) {
      for (int q = 0; q < kHostSlots; q++) cudaStreamCreateWithFlags(&g_host_st[dev].st[q], cudaStreamNonBlocking);
      g_host_st[dev].init = true;
    }
  }
  cudaStream_t *st = g_host_st[dev].st;
  // stream order: the pieces start after prior work on `stream`, and later work on
  // `stream` starts after every piece's digests are in host memory
  cudaEvent_t ev_in = nullptr, ev_out[kHostSlots] = {nullptr, nullptr, nullptr};
  if (cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming) != cudaSuccess) return PMP_ECUDA;
  cudaEventRecord(ev_in, stream);
  for (int q = 0; q < kHostSlots; q++) cudaStreamWaitEvent(st[q], ev_in, 0);
  cudaEventDestroy(ev_in);
  // per slot: payload (+16 B alignment shift, +32 B tail for whole 16-byte units), offsets, digests per key
  const size_t cap_b = (size_t)max_span + 48, cap_o = (size_t)(max_cnt + 1) * 8, cap_d = (size_t)max_cnt * 8;
  const size_t slot_bytes = ((cap_b + 255) & ~(size_t)255) + ((cap_o + 255) & ~(size_t)255) + (size_t)nkeys * ((cap_d + 255) & ~(size_t)255);
  uint8_t *slot[kHostSlots] = {nullptr, nullptr, nullptr};
  int rc = 0;
  for (int q = 0; q < kHostSlots && !rc; q++)
    if (cudaMallocAsync((void **)&slot[q], slot_bytes, st[q]) != cudaSuccess) rc = PMP_ENOMEM;
  for (size_t p = 0; p + 1 < cut.size() && !rc; p++) {
    const int q = (int)(p % kHostSlots);
    const uint64_t s0 = cut[p], s1 = cut[p + 1], cnt = s1 - s0;
    uint8_t *d_b = slot[q];
    uint64_t *d_o = (uint64_t *)(slot[q] + ((cap_b + 255) & ~(size_t)255));
    uint8_t *d_d = (uint8_t *)d_o + ((cap_o + 255) & ~(size_t)255);
    const uint64_t b0 = offsets[s0], nb = offsets[s1] - b0, sh = b0 & 15;
    // the kernels address string i at bytes + offsets[i]: keep the global offsets and
    // shift the base (same 16-byte phase as the host copy, so units stay aligned)
    const uint8_t *d_base = d_b + sh - b0;
    if (nb && cudaMemcpyAsync(d_b + sh, bytes + b0, nb, cudaMemcpyHostToDevice, st[q]) != cudaSuccess) rc = PMP_ECUDA;
    if (!rc && cudaMemcpyAsync(d_o, offsets + s0, (cnt + 1) * 8, cudaMemcpyHostToDevice, st[q]) != cudaSuccess)
      rc = PMP_ECUDA;
    void *d_outs[PMP_HOST_MAX_KEYS];
    for (int k = 0; k < nkeys; k++) d_outs[k] = d_d + (size_t)k * ((cap_d + 255) & ~(size_t)255);
    if (!rc) rc = pmp_hash_batch_multi(keys, nkeys, d_base, d_o, cnt, d_outs, st[q]);
    for (int k = 0; k < nkeys && !rc; k++) {
      const size_t w = keys[k]->bits / 8;
      if (cudaMemcpyAsync((uint8_t *)outs[k] + s0 * w, d_outs[k], cnt * w, cudaMemcpyDeviceToHost, st[q]) !=
          cudaSuccess)
        rc = PMP_ECUDA;
    }
  }
  for (int q = 0; q < kHostSlots; q++) {
    if (slot[q]) cudaFreeAsync(slot[q], st[q]);
    if (cudaEventCreateWithFlags(&ev_out[q], cudaEventDisableTiming) != cudaSuccess) {
      if (!rc) rc = PMP_ECUDA;
      continue;
    }
    cudaEventRecord(ev_out[q], st[q]);
    cudaStreamWaitEvent(stream, ev_out[q], 0);
    cudaEventDestroy(ev_out[q]);
  }
  if (!rc && cudaGetLastError() != cudaSuccess) rc = PMP_ECUDA;
  return rc;
}

int pmp_hash_long_host(const pmp_keys *k, const uint8_t *bytes, uint64_t len, void *out_host, uint64_t piece_bytes,
                       cudaStream_t stream) {
  if (!k || !out_host || (!bytes && len > 0)) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  if (words_of(k->bits, len) > (1ULL << 56)) return PMP_ETOOLONG;
  const int dev = k->device;
  if (dev < 0 || dev >= 64) return PMP_EINVAL;
  const uint64_t CB = (uint64_t)chunk_bytes(k->bits);
  if (piece_bytes == 0) piece_bytes = 256ull << 20;
  piece_bytes = piece_bytes < CB ? CB : piece_bytes - piece_bytes % CB;
  int cur_dev = 0;
  if (cudaGetDevice(&cur_dev) != cudaSuccess) return PMP_ECUDA;
  struct DevGuard {
    int prev, now;
    ~DevGuard() {
      if (prev != now) cudaSetDevice(prev);
    }
  } guard{cur_dev, dev};
  if (cur_dev != dev && cudaSetDevice(dev) != cudaSuccess) return PMP_ECUDA;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_host_st[dev].init) {
      for (int q = 0; q < kHostSlots; q++) cudaStreamCreateWithFlags(&g_host_st[dev].st[q], cudaStreamNonBlocking);
      g_host_st[dev].init = true;
    }
  }
  cudaStream_t *cst = g_host_st[dev].st;
  // incremental state, stream-ordered on `stream` (allocated and released there)
  pmp_stream s;
  s.k = k;
  s.d_state = nullptr;
  s.d_tail = nullptr;
  s.d_s2 = nullptr;
  s.s2_cap = 0;
  s.tail_len = s.c_done = 0;
  s.finalized = false;
  const size_t nslot = len > piece_bytes ? kHostSlots : 1;
  const size_t slot_bytes = (size_t)(len < piece_bytes ? len : piece_bytes) + 16;
  uint8_t *slab = nullptr;   // state | tail | digest | slots
  const size_t st_bytes = (sizeof(StreamState) + 255) & ~(size_t)255;
  const size_t hdr = st_bytes + (((size_t)CB + 32 + 255) & ~(size_t)255) + 256;
  if (cudaMallocAsync((void **)&slab, hdr + nslot * ((slot_bytes + 255) & ~(size_t)255), stream) != cudaSuccess)
    return PMP_ENOMEM;
  s.d_state = (StreamState *)slab;
  s.d_tail = slab + st_bytes;
  uint64_t *d_dig = (uint64_t *)(slab + hdr - 256);
  uint8_t *slot[kHostSlots];
  for (size_t q = 0; q < nslot; q++) slot[q] = slab + hdr + q * ((slot_bytes + 255) & ~(size_t)255);
  int rc = 0;
  if (cudaMemsetAsync(s.d_state, 0, sizeof(StreamState), stream) != cudaSuccess) rc = PMP_ECUDA;
  cudaEvent_t ev_start = nullptr, copied[kHostSlots] = {}, consumed[kHostSlots] = {};
  if (!rc && cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) != cudaSuccess) rc = PMP_ECUDA;
  for (int q = 0; q < kHostSlots && !rc; q++)
    if (cudaEventCreateWithFlags(&copied[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&consumed[q], cudaEventDisableTiming) != cudaSuccess)
      rc = PMP_ECUDA;
  if (!rc) {
    cudaEventRecord(ev_start, stream);  // the copies start after prior work on `stream` (and the allocation)
    for (int q = 0; q < kHostSlots; q++) cudaStreamWaitEvent(cst[q], ev_start, 0);
  }
  for (uint64_t off = 0, p = 0; off < len && !rc; off += piece_bytes, p++) {
    const int q = (int)(p % nslot);
    const uint64_t sz = len - off < piece_bytes ? len - off : piece_bytes;
    if (p >= nslot) cudaStreamWaitEvent(cst[q], consumed[q], 0);   // the slot's previous piece is hashed
    if (cudaMemcpyAsync(slot[q], bytes + off, sz, cudaMemcpyHostToDevice, cst[q]) != cudaSuccess) rc = PMP_ECUDA;
    cudaEventRecord(copied[q], cst[q]);
    cudaStreamWaitEvent(stream, copied[q], 0);
    if (!rc) rc = k->bits == 64 ? stream_update<64>(&s, slot[q], sz, stream) : stream_update<32>(&s, slot[q], sz, stream);
    cudaEventRecord(consumed[q], stream);
  }
  if (!rc) rc = k->bits == 64 ? stream_final<64>(&s, d_dig, stream) : stream_final<32>(&s, d_dig, stream);
  if (!rc && cudaMemcpyAsync(out_host, d_dig, (size_t)k->bits / 8, cudaMemcpyDeviceToHost, stream) != cudaSuccess)
    rc = PMP_ECUDA;
  if (s.d_s2) cudaFreeAsync(s.d_s2, stream);
  cudaFreeAsync(slab, stream);
  if (ev_start) cudaEventDestroy(ev_start);
  for (int q = 0; q < kHostSlots; q++) {
    if (copied[q]) cudaEventDestroy(copied[q]);
    if (consumed[q]) cudaEventDestroy(consumed[q]);
  }
  if (!rc && cudaGetLastError() != cudaSuccess) rc = PMP_ECUDA;
  return rc;
}

int pmp_hash_long_partial(const pmp_keys *k, const uint8_t *local, uint64_t local_len, uint64_t g0,
                          uint64_t total, uint64_t *partial, cudaStream_t st) {
  if (!k || !partial || (!local && local_len > 0)) return PMP_EINVAL;
  if (words_of(k->bits, total) > (1ULL << 56)) return PMP_ETOOLONG;
  const uint64_t CB = (uint64_t)chunk_bytes(k->bits);
  if (g0 % CB != 0 || g0 + local_len > total || g0 + local_len < g0) return PMP_EINVAL;
  if (g0 + local_len != total && local_len % CB != 0) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  return k->bits == 64 ? long_partial_impl<64>(k, local, local_len, g0, total, partial, st)
                       : long_partial_impl<32>(k, local, local_len, g0, total, partial, st);
}

int pmp_hash_long_combine(const pmp_keys *k, const uint64_t *partials, int G, uint64_t total,
                          void *out, cudaStream_t st) {
  if (!k || !partials || !out || G < 1) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  // key-only part of V; for the empty message the whole value, sigma_0 = 1
  // (no range owns a tail there, see long_partial_impl)
  const u128 c = total == 0 ? (u128)1 : long_constant(k, total);
  const uint64_t clo = (uint64_t)c, chi = (uint64_t)(c >> 64);
  if (k->bits == 64)
    return launch("k_combine", st, [&] { k_combine<64><<<1, 32, 0, st>>>(partials, G, clo, chi, out); });
  return launch("k_combine", st, [&] { k_combine<32><<<1, 32, 0, st>>>(partials, G, clo, chi, out); });
}

int pmp_hash_long(const pmp_keys *k, const uint8_t *bytes, uint64_t len, void *out, cudaStream_t st) {
  if (!k || !out || (!bytes && len > 0)) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  Scratch sc(st);
  if (sc.alloc(16)) return PMP_ENOMEM;
  uint64_t *partial = (uint64_t *)sc.p;
  int rc = pmp_hash_long_partial(k, bytes, len, 0, len, partial, st);
  if (rc) return rc;
  return pmp_hash_long_combine(k, partial, 1, len, out, st);
}

int pmp_hash2_batch(const pmp_keys *k, const uint8_t *bytes, const uint64_t *offsets, uint64_t n, void *out,
                    cudaStream_t st) {
  OutSpec os;
  os.out = out;
  os.M = 0;
  os.counts = nullptr;
  return hash_batch_impl(k, bytes, offsets, n, os, st, true);
}

int pmp_hash2_long(const pmp_keys *k, const uint8_t *bytes, uint64_t len, void *out, cudaStream_t st) {
  if (!out) return PMP_EINVAL;
  if (int rc = poly_args(k, bytes, len, 0, len)) return rc;
  return k->bits == 64 ? poly_long_impl<64>(k, bytes, len, 0, len, 1, out, st)
                       : poly_long_impl<32>(k, bytes, len, 0, len, 1, out, st);
}

int pmp_hash2_long_partial(const pmp_keys *k, const uint8_t *local, uint64_t local_len, uint64_t g0,
                           uint64_t total, uint64_t *partial, cudaStream_t st) {
  if (!partial) return PMP_EINVAL;
  if (int rc = poly_args(k, local, local_len, g0, total)) return rc;
  return k->bits == 64 ? poly_long_impl<64>(k, local, local_len, g0, total, 0, partial, st)
                       : poly_long_impl<32>(k, local, local_len, g0, total, 0, partial, st);
}

int pmp_hash2_long_combine(const pmp_keys *k, const uint64_t *partials, int G, void *out, cudaStream_t st) {
  if (!k || !partials || !out || G < 1) return PMP_EINVAL;
  if (int rc = check_keys(k)) return rc;
  if (int rc = ensure_poly(k)) return rc;
  if (k->bits == 64)
    return launch("k_poly_sum", st, [&] { k_poly_sum<64><<<1, 256, 0, st>>>(k->d_blob, partials, (uint64_t)G, 1, out); });
  return launch("k_poly_sum", st, [&] { k_poly_sum<32><<<1, 256, 0, st>>>(k->d_blob, partials, (uint64_t)G, 1, out); });
}

int pmp_long_split(int out_bits, uint64_t total, int G, uint64_t *begins) {
  if ((out_bits != 32 && out_bits != 64) || G < 1 || !begins) return PMP_EINVAL;
  const uint64_t CB = (uint64_t)chunk_bytes(out_bits);
  const uint64_t full = total / CB;  // whole level-1 blocks present in the bytes
  for (int g = 0; g < G; g++) begins[g] = (uint64_t)(((u128)full * (uint64_t)g) / (uint64_t)G) * CB;
  begins[G] = total;
  return 0;
}

int pmp_long_constant(const pmp_keys *k, uint64_t total, uint64_t *c2) {
  if (!k || !c2) return PMP_EINVAL;
  const u128 c = long_constant(k, total);
  c2[0] = (uint64_t)c;
  c2[1] = (uint64_t)(c >> 64);
  return 0;
}

int pmp_selftest(int out_bits, int mode, const uint64_t *in, uint64_t n, uint64_t *out, cudaStream_t st) {
  if ((out_bits != 32 && out_bits != 64) || mode < 0 || mode > 4 || (n && (!in || !out))) return PMP_EINVAL;
  if (n == 0) return 0;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return PMP_ENODEV;
  const unsigned grid = (unsigned)((n + 127) / 128);
  if (out_bits == 64)
    return launch("k_selftest", st, [&] { k_selftest<64><<<grid, 128, 0, st>>>(mode, in, n, out); });
  return launch("k_selftest", st, [&] { k_selftest<32><<<grid, 128, 0, st>>>(mode, in, n, out); });
}

uint64_t pmp_launch_count(void) { return g_launches.load(); }

uint64_t pmp_set_small_batch_max(uint64_t n) { return g_small_max.exchange(n); }
uint64_t pmp_set_huge_min(uint64_t bytes) { return bytes ? g_huge_min.exchange(bytes) : g_huge_min.load(); }
uint32_t pmp_set_huge_cap(uint32_t cap) { return g_huge_cap.exchange(cap); }
int pmp_set_short_tc(int on) {
  const int prev = use_short_tc() ? 1 : 0;
  if (on >= 0) g_short_tc.store(on ? 1 : 0);
  return prev;
}

#if PMP_SHORT_TRACE
// diagnostic builds only: the k_short clock64 timeline (pmp_short.cuh)
int pmp_trace_read(uint64_t *out, uint64_t n) {
  const uint64_t cap = sizeof(g_trace) / 8;
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(out, g_trace, n * 8) == cudaSuccess ? (int)n : PMP_ECUDA;
}
int pmp_trace_blocks(uint64_t *out, uint64_t n) {
  const uint64_t cap = sizeof(g_trace_blk) / 8;
  if (n > cap) n = cap;
  return cudaMemcpyFromSymbol(out, g_trace_blk, n * 8) == cudaSuccess ? (int)n : PMP_ECUDA;
}
#endif

int pmp_quality_collisions(int out_bits, uint64_t seed0, uint64_t nsched, const uint8_t *s1, uint32_t len1,
                           const uint8_t *s2, uint32_t len2, uint64_t *dig1, uint64_t *dig2, uint64_t *counts,
                           cudaStream_t st) {
  if ((out_bits != 32 && out_bits != 64) || !counts || len1 > kShortMax || len2 > kShortMax ||
      (len1 && !s1) || (len2 && !s2))
    return PMP_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return PMP_ENODEV;
  if (nsched == 0) return 0;
  const uint64_t grid = (nsched + 255) / 256;
  if (grid >= (1ull << 31)) return PMP_EINVAL;
  unsigned long long *c = reinterpret_cast<unsigned long long *>(counts);
  if (out_bits == 64)
    return launch("k_collide_mc", st, [&] {
      k_collide_mc<64><<<(unsigned)grid, 256, 0, st>>>(seed0, nsched, s1, len1, s2, len2, dig1, dig2, c);
    });
  return launch("k_collide_mc", st, [&] {
    k_collide_mc<32><<<(unsigned)grid, 256, 0, st>>>(seed0, nsched, s1, len1, s2, len2, dig1, dig2, c);
  });
}

void pmp_prof_enable(int on) { g_prof.store(on ? 1 : 0); }

static void prof_drain() {
  std::vector<ProfRec> pend;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    pend.swap(g_pending);
  }
  for (auto &r : pend) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    std::lock_guard<std::mutex> lk(g_mu);
    bool found = false;
    for (auto &d : g_done)
      if (d.first == r.name) {
        d.second.first += ms;
        d.second.second += 1;
        found = true;
      }
    if (!found) g_done.push_back({r.name, {ms, 1}});
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
}

void pmp_prof_reset(void) {
  prof_drain();
  std::lock_guard<std::mutex> lk(g_mu);
  g_done.clear();
}

int pmp_prof_read(const char *prefix, double *ms, uint64_t *count) {
  if (!prefix || !ms || !count) return PMP_EINVAL;
  prof_drain();
  std::lock_guard<std::mutex> lk(g_mu);
  *ms = 0;
  *count = 0;
  const size_t pl = strlen(prefix);
  for (auto &d : g_done)
    if (d.first.compare(0, pl, prefix) == 0) {
      *ms += d.second.first;
      *count += d.second.second;
    }
  return 0;
}

}  // extern "C"
