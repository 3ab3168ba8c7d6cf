"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Inputs are generated on the device (datagen, the shared input generator); the
oracle regenerates the bytes it needs on the host from the same seeded streams
(never from the CUDA path's buffers) and recomputes sampled digests one by one.
configs[3] (one 16 GiB string) is checked in full against the oracle and for
partition invariance; configs[4] (2^22 strings, ~295 GiB, sized for 8 GPUs) is
checked on rank 0's byte-balanced shard of 8.
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


@pytest.mark.parametrize("bits", [64, 32])
def test_hashtable_full_size_sampled(dev, oracle_lib, bits):
    """configs[1]: 2^24 strings U[8,64] B, seed 2 -- all hashed on the GPU,
    20,000 random + first/last 500 digests recomputed by the oracle."""
    import torch

    wl = datagen.WORKLOADS["hashtable"]
    offs = datagen.offsets_from_lengths(wl.lengths())
    pay, d_off = _device_batch(dev, wl.seed, offs)
    keys = pmp.Keys.generate(wl.seed, bits)
    got = pmp.as_u64(pmp.hash_batch(keys, pay, d_off))
    torch.cuda.synchronize()
    n = wl.n
    rng = np.random.default_rng(bits)
    idx = np.unique(np.concatenate([rng.integers(0, n, 20000), np.arange(500), np.arange(n - 500, n)]))
    _check_sample(oracle_lib, oracle_lib.keygen(wl.seed, bits), wl.seed, offs, got, idx)


def test_hashtable_full_size_fused_both_widths(dev, oracle_lib):
    """configs[1] in bench.py's launch configuration: both widths in one fused
    pass (pmp_hash_batch_multi); 20,000 random + first/last 500 digests of
    each width recomputed by the oracle, and both equal the per-width launches
    on a further 100,000 indices."""
    import torch

    wl = datagen.WORKLOADS["hashtable"]
    offs = datagen.offsets_from_lengths(wl.lengths())
    pay, d_off = _device_batch(dev, wl.seed, offs)
    k64, k32 = pmp.Keys.generate(wl.seed, 64), pmp.Keys.generate(wl.seed, 32)
    o64, o32 = pmp.hash_batch_multi([k64, k32], pay, d_off)
    s64 = pmp.hash_batch(k64, pay, d_off)
    s32 = pmp.hash_batch(k32, pay, d_off)
    torch.cuda.synchronize()
    g64, g32 = pmp.as_u64(o64), pmp.as_u64(o32)
    n = wl.n
    rng = np.random.default_rng(64 + 32)
    idx = np.unique(np.concatenate([rng.integers(0, n, 20000), np.arange(500), np.arange(n - 500, n)]))
    _check_sample(oracle_lib, oracle_lib.keygen(wl.seed, 64), wl.seed, offs, g64, idx)
    _check_sample(oracle_lib, oracle_lib.keygen(wl.seed, 32), wl.seed, offs, g32, idx)
    j = rng.integers(0, n, 100000)
    assert np.array_equal(g64[j], pmp.as_u64(s64)[j]) and np.array_equal(g32[j], pmp.as_u64(s32)[j])


def test_fixed4k_full_size_sampled(dev, oracle_lib):
    """configs[2]: 2^20 x 4096 B (4 GiB), PM+64, seed 3; 3,000 sampled digests."""
    import torch

    wl = datagen.WORKLOADS["fixed4k"]
    offs = datagen.offsets_from_lengths(wl.lengths())
    pay, d_off = _device_batch(dev, wl.seed, offs)
    keys = pmp.Keys.generate(wl.seed, 64)
    got = pmp.as_u64(pmp.hash_batch(keys, pay, d_off))
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    idx = np.unique(np.concatenate([rng.integers(0, wl.n, 3000), [0, wl.n - 1]]))
    _check_sample(oracle_lib, oracle_lib.keygen(wl.seed, 64), wl.seed, offs, got, idx)
    del pay
    torch.cuda.empty_cache()


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


def test_mixed_shard_sampled(dev, oracle_lib):
    """configs[4]: 2^22 strings, log-uniform [1, 2^20] B, PM+32, seed 5 (~295 GiB
    in total, reading Q15).  Rank 0's byte-balanced shard of 8 (~37 GiB) is hashed
    on the GPU; 3,000 random strings and the 40 longest are checked."""
    import torch

    wl = datagen.WORKLOADS["mixed"]
    offs_all = datagen.offsets_from_lengths(wl.lengths())
    lo, hi = parallel.shard_batch(offs_all, 8)[0]
    sub, b0, b1 = parallel.rebase_offsets(offs_all, lo, hi)
    pay, d_off = _device_batch(dev, wl.seed, offs_all[lo:hi + 1], start_byte=b0)
    keys = pmp.Keys.generate(wl.seed, 32)
    got = pmp.as_u64(pmp.hash_batch(keys, pay, d_off))
    torch.cuda.synchronize()
    n = hi - lo
    lens = np.diff(sub.astype(np.int64))
    rng = np.random.default_rng(5)
    idx = np.unique(np.concatenate([rng.integers(0, n, 3000), np.argsort(lens)[-40:], [0, n - 1]]))
    _check_sample(oracle_lib, oracle_lib.keygen(wl.seed, 32), wl.seed, sub, got, idx, base_byte=b0)
    del pay
    torch.cuda.empty_cache()
