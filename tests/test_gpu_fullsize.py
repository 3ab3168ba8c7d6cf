"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Inputs are generated on the device (datagen, the shared input generator); the
oracle regenerates the bytes it needs on the host from the same seeded streams
(never from the CUDA path's buffers).  EVERY digest is compared: configs[1]
(2^24 strings, both widths), configs[2] (2^20 x 4 KiB), configs[3] (one 16 GiB
string, plus partition invariance and streaming) and configs[4] (all 2^22
strings, ~295 GiB, hashed as bench.py's 8 byte-balanced shards one after
another on this GPU).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import datagen
import paper_1609_09840_b200 as pmp
from paper_1609_09840_b200 import parallel

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
NT = os.cpu_count() or 4


@pytest.fixture(scope="module")
def dev():
    import torch

    import __graft_entry__

    __graft_entry__.build()
    torch.cuda.set_device(0)
    yield torch.device("cuda:0")
    torch.cuda.empty_cache()


def host_payload_parallel(seed, start, nbytes, chunk=256 << 20):
    out = np.empty(nbytes, dtype=np.uint8)

    def job(o):
        n = min(chunk, nbytes - o)
        out[o:o + n] = datagen.payload_host(seed, start + o, n)

    with ThreadPoolExecutor(NT) as ex:
        list(ex.map(job, range(0, nbytes, chunk)))
    return out


def _device_batch(dev, seed, offs, start_byte=0):
    import torch

    total = int(offs[-1]) - int(offs[0])
    page0 = start_byte - start_byte % datagen.PAGE
    lead = start_byte - page0
    buf = torch.empty(total + lead + 16, dtype=torch.uint8, device=dev)
    datagen.fill_device(seed, buf.data_ptr(), total + lead, torch.cuda.current_stream().cuda_stream, start=page0)
    d_off = torch.from_numpy((offs - offs[0]).view(np.int64)).to(dev)
    return buf[lead:], d_off


def _check_sample(oracle_lib, keys_o, seed, offs, got, idx, base_byte=0):
    bad = []
    for i in idx:
        o0, o1 = int(offs[i]), int(offs[i + 1])
        data = datagen.payload_host(seed, base_byte + o0, o1 - o0)
        if int(got[i]) != oracle_lib.hash_bytes(keys_o, data):
            bad.append(int(i))
    assert not bad, bad[:10]


def _oracle_all(oracle_lib, keys_o, seed, offs, base_byte=0, piece=2 << 30):
    """Every digest of the batch with CSR ``offs`` (relative to payload byte
    ``base_byte`` of the seeded stream) by the multithreaded oracle, the payload
    regenerated on the host piece by piece (string-aligned pieces of ~2 GiB)."""
    n = offs.size - 1
    out = np.empty(n, dtype=np.uint64)
    i = 0
    while i < n:
        j = int(np.searchsorted(offs, np.uint64(int(offs[i]) + piece), side="right")) - 1
        j = min(max(j, i + 1), n)
        o0 = int(offs[i])
        pay = host_payload_parallel(seed, base_byte + o0, int(offs[j]) - o0)
        out[i:j] = oracle_lib.hash_batch(keys_o, pay, offs[i:j + 1] - np.uint64(o0), nthreads=NT)
        i = j
    return out


def _assert_all_equal(got, want, bits):
    want = want.astype(np.uint64) if bits == 64 else want.astype(np.uint32)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad.size, bad[:10])


def test_hashtable_full_size_every_hash(dev, oracle_lib):
    """configs[1] in bench.py's launch configuration: 2^24 strings U[8,64] B,
    seed 2, both widths in one fused pass (pmp_hash_batch_multi).  EVERY digest
    of both widths equals the oracle's, and so do the per-width launches
    (pmp_hash_batch, the k_short single-width kernels) -- with the word loop
    (k_short) and with the level-1 sums on the tensor cores (k_short_tc)."""
    import torch

    wl = datagen.WORKLOADS["hashtable"]
    offs = datagen.offsets_from_lengths(wl.lengths())
    pay, d_off = _device_batch(dev, wl.seed, offs)
    k64, k32 = pmp.Keys.generate(wl.seed, 64), pmp.Keys.generate(wl.seed, 32)
    got = {}
    prev = pmp.pmp_set_short_tc(0)
    try:
        for tc in (0, 1):   # the word loop (k_short, default) and the tensor-core kernel (k_short_tc)
            pmp.pmp_set_short_tc(tc)
            o64, o32 = pmp.hash_batch_multi([k64, k32], pay, d_off)
            s64 = pmp.hash_batch(k64, pay, d_off)
            s32 = pmp.hash_batch(k32, pay, d_off)
            torch.cuda.synchronize()
            got[tc] = [pmp.as_u64(x) for x in (o64, s64, o32, s32)]
    finally:
        pmp.pmp_set_short_tc(prev)
    del pay
    torch.cuda.empty_cache()
    w64 = _oracle_all(oracle_lib, oracle_lib.keygen(wl.seed, 64), wl.seed, offs)
    w32 = _oracle_all(oracle_lib, oracle_lib.keygen(wl.seed, 32), wl.seed, offs)
    for tc in (0, 1):
        g64, s64, g32, s32 = got[tc]
        _assert_all_equal(g64, w64, 64)
        _assert_all_equal(s64, w64, 64)
        _assert_all_equal(g32, w32, 32)
        _assert_all_equal(s32, w32, 32)


def test_fixed4k_full_size_every_hash(dev, oracle_lib):
    """configs[2]: 2^20 x 4096 B (4 GiB), PM+64, seed 3 -- every digest."""
    import torch

    wl = datagen.WORKLOADS["fixed4k"]
    offs = datagen.offsets_from_lengths(wl.lengths())
    pay, d_off = _device_batch(dev, wl.seed, offs)
    keys = pmp.Keys.generate(wl.seed, 64)
    got = pmp.as_u64(pmp.hash_batch(keys, pay, d_off))
    torch.cuda.synchronize()
    del pay
    torch.cuda.empty_cache()
    _assert_all_equal(got, _oracle_all(oracle_lib, oracle_lib.keygen(wl.seed, 64), wl.seed, offs), 64)


def test_long16g_full(dev, oracle_lib):
    """configs[3]: one 16 GiB string, PM+64, seed 4 (reading Q16).  The digest of
    pmp_hash_long equals the oracle's literal Algorithm 1 over all 16 GiB, and
    the G = 2, 4, 8 block-aligned splits (partial + combine) give the same; the
    two-level variant's digest of the same string equals the oracle's."""
    import torch

    wl = datagen.WORKLOADS["long16g"]
    total = wl.lo
    buf = torch.empty(total + 16, dtype=torch.uint8, device=dev)
    datagen.fill_device(wl.seed, buf.data_ptr(), total, torch.cuda.current_stream().cuda_stream)
    keys = pmp.Keys.generate(wl.seed, 64)
    got = int(pmp.as_u64(pmp.hash_long(keys, buf, total))[0])
    for G in (2, 4, 8):
        parts = torch.zeros(2 * G, dtype=torch.int64, device=dev)
        for g, (b, e) in enumerate(parallel.long_ranges(64, total, G)):
            pmp.hash_long_partial(keys, buf[b:], e - b, b, total, partial=parts[2 * g:2 * g + 2])
        assert int(pmp.as_u64(pmp.hash_long_combine(keys, parts, total))[0]) == got, G
    # streaming (8(f1)): one 16 GiB update (1 piece per node) and ~1 GiB misaligned
    # pieces (8 pieces per node, level-3/4 nodes closing across updates)
    for cuts in ([total], [(1 << 30) + 4099] * 15 + [total - 15 * ((1 << 30) + 4099)]):
        st = pmp.Stream(keys)
        pos = 0
        for c in cuts:
            st.update(buf[pos:], c)
            pos += c
        assert int(pmp.as_u64(st.final())[0]) == got, len(cuts)
        st.close()
    # the two-level variant (8(f4)) over the same 16 GiB: 131,072 virtual nodes,
    # more than the resident warps, so warps walk several nodes (weights
    # R^(Q'-1-q) stepped by R^q_step)
    got2 = int(pmp.as_u64(pmp.hash2_long(keys, buf, total))[0])
    del buf
    torch.cuda.empty_cache()
    host = host_payload_parallel(wl.seed, 0, total)
    okeys = oracle_lib.keygen(wl.seed, 64)
    want = oracle_lib.hash_long(okeys, host, nthreads=NT)
    assert got == want
    assert got2 == oracle_lib.hash2(okeys, host, nthreads=NT)


def test_mixed_corpus_every_hash(dev, oracle_lib):
    """configs[4]: 2^22 strings, log-uniform [1, 2^20] B, PM+32, seed 5 (~295 GiB
    in total, reading Q15).  The 8 byte-balanced shards of bench.py's 8-GPU
    split are hashed one after another on this GPU (pmp_hash_batch, rebased
    offsets, as each rank does) and EVERY digest of the corpus equals the
    oracle's (payload regenerated on the host piece by piece)."""
    import torch

    wl = datagen.WORKLOADS["mixed"]
    offs_all = datagen.offsets_from_lengths(wl.lengths())
    keys = pmp.Keys.generate(wl.seed, 32)
    okeys = oracle_lib.keygen(wl.seed, 32)
    shards = parallel.shard_batch(offs_all, 8)
    assert shards[0][0] == 0 and shards[-1][1] == wl.n
    for lo, hi in shards:
        sub, b0, b1 = parallel.rebase_offsets(offs_all, lo, hi)
        pay, d_off = _device_batch(dev, wl.seed, offs_all[lo:hi + 1], start_byte=b0)
        got = pmp.as_u64(pmp.hash_batch(keys, pay, d_off))
        torch.cuda.synchronize()
        del pay, d_off
        torch.cuda.empty_cache()
        _assert_all_equal(got, _oracle_all(oracle_lib, okeys, wl.seed, sub, base_byte=b0), 32)
