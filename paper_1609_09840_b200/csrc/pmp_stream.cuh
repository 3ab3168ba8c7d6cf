// pmp_stream.cuh -- incremental hashing with device-resident level state
// (part of the kernels included by pmp_kernels.cuh; citations as there)
#pragma once
#include "pmp_long.cuh"

namespace pmp {

// ============================================================= streaming
// Device state of an incremental hash (the tree evaluated bottom-up
// with bounded memory).  Instead of buffering up to m values per level, every
// level keeps the exact running sum of its open node (sum_r a_{j,r} x_r, b_j
// added when the node closes) -- O(L) state, same arithmetic.
struct StreamState {
  uint32_t acc[kL + 1][5];   // open node sums of levels 2..8 (Acc5, or Acc3 in the first words)
  uint32_t cnt[kL + 1];      // children already in the open node of level j
  uint64_t last[kL + 1][2];  // last value emitted at level j (field element)
  uint64_t emitted[kL + 1];  // values emitted so far at level j (cnt[j+1] == emitted[j] mod 128)
  uint32_t blocks_done;      // k_stream_node: blocks finished in the current launch
};

template <int BITS> struct StreamOps {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  const uint64_t *bk, *ak;
  StreamState *st;
  PMP_DI void close(int j) {  // node of level j complete: emit it and push into level j+1
    for (;;) {
      Acc a;
      load_acc(st->acc[j], a);
      acc_add_word(a, bk[j - 1]);
      const Fe v = acc_reduce(a);
      fe_store(st->last[j], v);
      acc_zero(a);
      store_acc(st->acc[j], a);
      st->cnt[j] = 0;
      if (j + 1 > (int)kL) return;  // only reachable past the string's own top level
      if (!push(j + 1, v)) return;
      j++;
    }
  }
  // adds child v to level j's open node; true if that node is now full (the caller closes it)
  PMP_DI bool push(int j, const Fe &v) {
    Acc a;
    load_acc(st->acc[j], a);
    acc_mac_fe(a, ak[(uint64_t)(j - 1) * kM + st->cnt[j]], v);
    store_acc(st->acc[j], a);
    return ++st->cnt[j] == kM;
  }
};

// Sum of the P piece partials of one level-2 node, by one warp (lanes over
// pieces), result in every lane.
template <int BITS>
PMP_DI typename Tr<BITS>::Acc node_pieces_sum(const uint64_t *s2, uint64_t qi, int P, int lane) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  Acc x;
  acc_zero(x);
  if (lane < P) {
    Fe v;
    fe_load_cg(s2 + 2 * (qi * P + lane), v);
    acc_add_fe(x, v);
  }
#pragma unroll
  for (int mm = 1; mm < 32; mm <<= 1) {
    Acc y = acc_shfl_xor(x, mm);
    acc_add(x, y);
  }
  return x;
}

// Folds one update (level-1 blocks [c0, c0+N) = level-2 nodes qb .. qb+nq-1,
// P pieces each) into the stream state, on the one block that finished last.
// The grid has already written va[qi] = v_2 of every node the update completes
// except node qb when it was open before (its earlier children live in the
// state).  Here: that node, the open node at the end of the update, and levels
// >= 3 -- level by level, one warp per level-j node over its <= 128 new
// children (as k_level); complete nodes emit in parallel and only the open
// node of each level (first/last of the batch) meets the persistent state.
// The new open sum is staged in shared memory and committed after a barrier,
// so the warp reading the old one never races the warp replacing it.
// va/vb: values of two adjacent levels (>= nq each).
template <int BITS>
__device__ void stream_merge_block(const uint64_t *__restrict__ keys, StreamState *st,
                                   const uint64_t *__restrict__ s2, uint64_t qb, uint64_t nq, uint64_t c0,
                                   uint64_t N, int P, bool open0, uint64_t *__restrict__ va,
                                   uint64_t *__restrict__ vb) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  const uint64_t *bk = keys, *ak = keys + kL;
  __shared__ uint64_t s_m, s_e;
  __shared__ uint32_t s_open[5];
  __shared__ int s_has_open;
  // ---------------- level 2: the boundary nodes
  const uint64_t end = c0 + N;
  const uint64_t m2 = end / 128 - qb;               // nodes this update completes
  if (wid == 0 && open0 && m2 > 0) {                // node qb: earlier children + this update's
    Acc x = node_pieces_sum<BITS>(s2, 0, P, lane);
    if (lane == 0) {
      Acc o;
      load_acc(st->acc[2], o);
      acc_add(x, o);
      acc_add_word(x, bk[1]);
      fe_store(va, acc_reduce(x));
    }
  }
  if (wid == nwarps - 1 && lane == 0) s_has_open = 0;
  if (wid == nwarps - 1 && m2 < nq) {               // the update ends inside node qb + nq - 1
    Acc x = node_pieces_sum<BITS>(s2, nq - 1, P, lane);
    if (lane == 0) {
      if (m2 == 0) {                                // still node qb: keep its earlier children
        Acc o;
        load_acc(st->acc[2], o);
        acc_add(x, o);
      }
      store_acc(s_open, x);
      s_has_open = 1;
    }
  }
  __syncthreads();
  if (tid == 0) {
    Acc o;
    if (s_has_open) load_acc(s_open, o);
    else acc_zero(o);
    store_acc(st->acc[2], o);
    st->cnt[2] = (uint32_t)(end % 128);
    s_e = st->emitted[2];
    st->emitted[2] += m2;
    if (m2) {
      Fe v;
      fe_load_cg(va + 2 * (m2 - 1), v);
      fe_store(&st->last[2][0], v);
    }
    s_m = m2;
    s_has_open = 0;
  }
  __syncthreads();
  // ---------------- levels 3..8: the new values of level j-1 join level-j nodes
  uint64_t *in = va, *outv = vb;
  for (int j = 3; j <= (int)kL; j++) {
    const uint64_t m_in = s_m, e_in = s_e;          // new values have level-(j-1) indices [e_in, e_in + m_in)
    if (m_in == 0) break;
    const uint64_t kf = e_in / 128, kl = (e_in + m_in - 1) / 128;
    const uint64_t m_out = (e_in + m_in) / 128 - kf; // level-j nodes completed by this batch
    const uint64_t *aj = ak + (uint64_t)(j - 1) * kM;
    const bool openj = st->cnt[j] != 0;
    for (uint64_t k = kf + wid; k <= kl; k += nwarps) {
      Acc x;
      acc_zero(x);
#pragma unroll
      for (int r0 = 0; r0 < 128; r0 += 32) {
        const uint64_t g = k * 128 + r0 + lane;
        if (g >= e_in && g < e_in + m_in) {
          Fe v;
          fe_load_cg(in + 2 * (g - e_in), v);
          acc_mac_fe(x, aj[r0 + lane], v);
        }
      }
#pragma unroll
      for (int mm = 1; mm < 32; mm <<= 1) {
        Acc y = acc_shfl_xor(x, mm);
        acc_add(x, y);
      }
      if (lane == 0) {
        if (k == kf && openj) {
          Acc o;
          load_acc(st->acc[j], o);
          acc_add(x, o);
        }
        if (k - kf < m_out) {                       // complete node: emit its value
          acc_add_word(x, bk[j - 1]);
          fe_store(outv + 2 * (k - kf), acc_reduce(x));
        } else {                                    // the batch ends inside it: it stays open
          store_acc(s_open, x);
          s_has_open = 1;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      Acc o;
      if (s_has_open) load_acc(s_open, o);
      else acc_zero(o);
      store_acc(st->acc[j], o);
      st->cnt[j] = (uint32_t)((e_in + m_in) % 128);
      s_e = st->emitted[j];
      st->emitted[j] += m_out;
      if (m_out) {
        Fe v;
        fe_load_cg(outv + 2 * (m_out - 1), v);
        fe_store(&st->last[j][0], v);
      }
      s_m = m_out;
      s_has_open = 0;
    }
    __syncthreads();
    uint64_t *t = in;
    in = outv;
    outv = t;
  }
}

// One update of a stream in one launch.  Warps compute the partial level-2
// sums of (node, piece) items, P pieces of 128/P level-1 blocks per node (as
// k_node); the warp that finishes a node's last piece (per-node counter,
// self-resetting) emits v_2 of every complete node the state has no share in;
// the block that finishes last runs stream_merge_block.
template <int BITS>
__global__ void __launch_bounds__(kWWarps * 32)
k_stream_node(const uint64_t *__restrict__ keys, StrView s, uint64_t c0, uint64_t N, uint64_t qb, uint64_t qe,
              int P, uint64_t *__restrict__ s2, uint32_t *__restrict__ node_cnt, StreamState *st,
              uint64_t *__restrict__ va, uint64_t *__restrict__ vb) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  const int lane = threadIdx.x & 31;
  const uint64_t *bk = keys, *ak = keys + kL;
  const uint64_t warp = (uint64_t)blockIdx.x * kWWarps + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kWWarps;
  const uint64_t nu = (qe - qb) * (uint64_t)P, span = 128 / P;
  const uint64_t m2 = (c0 + N) / 128 - qb;          // nodes the update completes
  const bool open0 = st->cnt[2] != 0;
  if (warp < nu) {
    LaneKeys<BITS> lk;
    lk.load(ak, lane & 7);
    for (uint64_t u = warp; u < nu; u += nw) {
      const uint64_t qi = u / P;
      const uint64_t c = (qb + qi) * 128 + (u % P) * span;
      const uint64_t lo = max(c, c0), hi = min(c + span, c0 + N);
      Acc x;
      if (lo < hi) {
        ChunkOut<BITS> co = warp_chunks<BITS, false, true>(s, lo, hi, lk, bk[0], ak + kM, lane);
        x = co.acc2;
      } else {
        acc_zero(x);
      }
      if (qi >= m2 || (qi == 0 && open0)) {         // boundary node: the merge sums its pieces
        if (lane == 0) fe_store(s2 + 2 * u, acc_reduce(x));
        continue;
      }
      bool last_piece = true;
      if (P > 1) {
        int done = 0;
        if (lane == 0) {
          fe_store(s2 + 2 * u, acc_reduce(x));
          __threadfence();
          done = atomicAdd(&node_cnt[qi], 1u) == (unsigned)P - 1;
        }
        last_piece = __shfl_sync(0xffffffffu, done, 0);
        if (!last_piece) continue;
        __threadfence();
        x = node_pieces_sum<BITS>(s2, qi, P, lane);
      }
      if (lane == 0) {
        if (P > 1) node_cnt[qi] = 0;
        acc_add_word(x, bk[1]);
        fe_store(va + 2 * qi, acc_reduce(x));
      }
    }
  }
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&st->blocks_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  stream_merge_block<BITS>(keys, st, s2, qb, qe - qb, c0, N, P, open0, va, vb);
  if (threadIdx.x == 0) st->blocks_done = 0;
}

// Final: fold the last level-1 block (partial sum in s2last), close every open
// node bottom-up through the top level leff, whose single value is the root
// (Algorithm 1's "while |sigma| > 1"); leff <= 1: s2last is the root.
template <int BITS>
__global__ void k_stream_final(const uint64_t *__restrict__ keys, StreamState *st, const uint64_t *__restrict__ s2last,
                               int leff, void *__restrict__ out) {
  using Fe = typename Tr<BITS>::Fe;
  using Acc = typename Tr<BITS>::Acc;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Fe root;
  if (leff <= 1) {
    fe_load(s2last, root);
  } else {
    StreamOps<BITS> ops{keys, keys + kL, st};
    Fe v;
    fe_load(s2last, v);
    Acc a;
    load_acc(st->acc[2], a);
    acc_add_fe(a, v);
    store_acc(st->acc[2], a);
    if (++st->cnt[2] == kM) ops.close(2);
    for (int j = 2; j <= leff; j++) {
      if (st->cnt[j] == 0) continue;
      // close level j (zero padding) and push into j+1 unless j is the top
      Acc x;
      load_acc(st->acc[j], x);
      acc_add_word(x, keys[j - 1]);
      const Fe w = acc_reduce(x);
      fe_store(st->last[j], w);
      acc_zero(x);
      store_acc(st->acc[j], x);
      st->cnt[j] = 0;
      if (j < leff && ops.push(j + 1, w)) ops.close(j + 1);
    }
    fe_load(st->last[leff], root);
  }
  store_digest<BITS>(out, 0, fe_lo(root));
}

// V = C + sum_g P_g mod p; digest = mix(V mod 2^n)
template <int BITS>
__global__ void k_combine(const uint64_t *__restrict__ partials, int G, uint64_t c_lo, uint64_t c_hi,
                          void *__restrict__ out) {
  using T = Tr<BITS>;
  using Acc = typename T::Acc;
  using Fe = typename T::Fe;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Acc x;
  acc_zero(x);
  uint64_t cw[2] = {c_lo, c_hi};
  Fe c;
  fe_load(cw, c);
  acc_add_fe(x, c);
  for (int g = 0; g < G; g++) {
    Fe v;
    fe_load(partials + 2 * g, v);
    acc_add_fe(x, v);
  }
  store_digest<BITS>(out, 0, fe_lo(acc_reduce(x)));
}

}  // namespace pmp
