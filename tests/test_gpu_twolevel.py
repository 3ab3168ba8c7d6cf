"""GPU parity of the two-level variant (reading Q19) through the
C ABI against the oracle's pmpo_hash2*, bit-exact: short strings (k_short<V2>),
the warp-per-string path, long strings (k_poly_node), block-aligned splits
(partial + combine), and keys whose powers r^j exceed 2^n (the extra-bit
multiply-add that random keys essentially never reach)."""
import os

import numpy as np
import pytest

import datagen
import paper_1609_09840_b200 as pmp

pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 4


@pytest.fixture(scope="module")
def dev():
    import torch

    import __graft_entry__

    __graft_entry__.build()
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


def _batch(dev, keys, payload, offsets):
    import torch

    d_pay = torch.from_numpy(np.ascontiguousarray(payload) if payload.size else np.zeros(16, np.uint8)).to(dev)
    d_off = torch.from_numpy(np.ascontiguousarray(offsets).view(np.int64)).to(dev)
    out = pmp.hash2_batch(keys, d_pay, d_off)
    torch.cuda.synchronize()
    return pmp.as_u64(out)


def _want(oracle_lib, okeys, payload, offsets):
    d = oracle_lib.hash2_batch(okeys, payload, offsets, nthreads=NT)
    return d if okeys.bits == 64 else d.astype(np.uint32).astype(np.uint64)


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("shift", [0, 5])
def test_hash2_batch_length_sweep(dev, oracle_lib, bits, shift):
    """Every length 0..2600 (T == 1 strings, the short kernel, 1..6 chunks on the
    warp path, marker-only chunks), shuffled, payload shifted by `shift`."""
    lens = np.arange(0, 2601, dtype=np.uint64)
    np.random.default_rng(shift + bits).shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + shift
    pay = datagen.payload_host(51 + shift, 0, int(off[-1]))
    got = _batch(dev, pmp.Keys.generate(50, bits), pay, off)
    want = _want(oracle_lib, oracle_lib.keygen(50, bits), pay, off)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:5], np.diff(off)[bad[:5]])


@pytest.mark.parametrize("bits", [32, 64])
def test_hash2_mid_strings_group_path(dev, oracle_lib, bits):
    """Mid strings through the 8-lane group phase (one virtual node, weights
    W[c + 128 - C]): lengths around every multiple of 1 KiB up to the 64 KiB
    big-string boundary plus a log-uniform crowd, misaligned."""
    rng = np.random.default_rng(bits + 7)
    edge = [k * 1024 + d for k in range(1, 64) for d in (-1, 0, 1)] + [65535, 65536, 128, 129, 512, 513]
    crowd = np.floor(2.0 ** rng.uniform(7, 16, size=1501)).astype(np.uint64)
    lens = np.concatenate([np.array(edge, dtype=np.uint64), crowd, rng.integers(0, 128, size=200, dtype=np.uint64)])
    rng.shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + 3
    pay = datagen.payload_host(61, 0, int(off[-1]))
    got = _batch(dev, pmp.Keys.generate(61, bits), pay, off)
    want = _want(oracle_lib, oracle_lib.keygen(61, bits), pay, off)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(int(i), int(lens[i])) for i in bad[:10]]


@pytest.mark.parametrize("bits", [32, 64])
def test_hash2_batch_tiny_config_and_long_members(dev, oracle_lib, bits):
    """configs[0] shapes plus members of 70 KiB - 1 MiB (several virtual nodes,
    R^e weights) in one batch."""
    wl = datagen.WORKLOADS["tiny"]
    lens = wl.lengths().astype(np.uint64)
    lens = np.concatenate([lens, np.array([70_000, 131_072, 131_073, 262_144 + 7, 1 << 20], dtype=np.uint64)])
    off = datagen.offsets_from_lengths(lens) + 3
    pay = datagen.payload_host(wl.seed, 0, int(off[-1]))
    got = _batch(dev, pmp.Keys.generate(wl.seed, bits), pay, off)
    want = _want(oracle_lib, oracle_lib.keygen(wl.seed, bits), pay, off)
    assert np.array_equal(got, want)


LONG = [0, 1, 7, 1023, 1024, 1025, 128 * 1024 - 1, 128 * 1024, 128 * 1024 + 1, 129 * 128 * 1024 + 5,
        (3 << 20) + 17, 128 * 128 * 1024 + 999]


@pytest.mark.parametrize("bits", [32, 64])
def test_hash2_long_lengths(dev, oracle_lib, bits):
    import torch

    keys = pmp.Keys.generate(52, bits)
    okeys = oracle_lib.keygen(52, bits)
    for n in LONG:
        data = datagen.payload_host(53, 0, n)
        d = torch.from_numpy(np.concatenate([np.zeros(1, np.uint8), data])).to(dev)[1:]  # misaligned base
        got = int(pmp.as_u64(pmp.hash2_long(keys, d, n))[0])
        assert got == oracle_lib.hash2(okeys, data, nthreads=NT), n


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("G", [2, 3, 5])
def test_hash2_partition_invariance(dev, oracle_lib, bits, G):
    import torch

    n = 300 * 128 * 128 * (bits // 8) + 4321  # 300 level-2 nodes' worth of chunks plus a ragged tail
    keys = pmp.Keys.generate(54, bits)
    data = datagen.payload_host(55, 0, n)
    d = torch.from_numpy(data).to(dev)
    whole = int(pmp.as_u64(pmp.hash2_long(keys, d, n))[0])
    parts = torch.zeros(2 * G, dtype=torch.int64, device=dev)
    b = pmp.pmp_long_split(bits, n, G)
    for g in range(G):
        pmp.hash2_long_partial(keys, d[b[g]:], b[g + 1] - b[g], b[g], n, partial=parts[2 * g:2 * g + 2])
    assert int(pmp.as_u64(pmp.hash2_long_combine(keys, parts))[0]) == whole
    assert whole == oracle_lib.hash2(oracle_lib.keygen(54, bits), data, nthreads=NT)


def _sqrt_mod(t, p):
    """Tonelli-Shanks: some x with x^2 = t (mod p), or None."""
    if pow(t, (p - 1) // 2, p) != 1:
        return None
    q, s = p - 1, 0
    while q % 2 == 0:
        q //= 2
        s += 1
    z = 2
    while pow(z, (p - 1) // 2, p) != p - 1:
        z += 1
    m, c, x, r = s, pow(z, q, p), pow(t, (q + 1) // 2, p), pow(t, q, p)
    while r != 1:
        i, rr = 0, r
        while rr != 1:
            rr = rr * rr % p
            i += 1
        bb = pow(c, 1 << (m - i - 1), p)
        m, c, x, r = i, bb * bb % p, x * bb % p, r * bb * bb % p
    return x


@pytest.mark.parametrize("bits", [32, 64])
def test_hash2_power_above_2n(dev, oracle_lib, bits):
    """a_{2,1} = r chosen with r^2 mod p in [2^n, p): the first chunk of every
    2-chunk string is weighted by r^2, which takes the extra-bit path."""
    p = 2**bits + (13 if bits == 64 else 15)
    amax = p - (25 if bits == 64 else 29)
    base = oracle_lib.keygen(56, bits)
    r = None
    for t in range(2**bits, p):
        x = _sqrt_mod(t, p)
        if x is not None:
            for cand in (x, p - x):
                if 1 <= cand <= amax:
                    r = cand
                    break
        if r is not None:
            break
    assert r is not None and pow(r, 2, p) >= 2**bits
    a = base.a.copy()
    a[1][0] = r
    keys = pmp.Keys.from_words(bits, base.b, a)
    okeys = oracle_lib.Keys(bits, base.b, a)
    cb = 128 * bits // 8
    lens = np.array([cb, cb + 1, 2 * cb - 1, cb + 77, 5, 0, 2 * cb, 3 * cb + 1], dtype=np.uint64)
    off = datagen.offsets_from_lengths(lens)
    pay = datagen.payload_host(57, 0, int(off[-1]))
    assert np.array_equal(_batch(dev, keys, pay, off), _want(oracle_lib, okeys, pay, off))


@pytest.mark.parametrize("order", [(64, 32), (32, 64)])
def test_hash2_multi_fused(dev, oracle_lib, order):
    """pmp_hash2_batch_multi: the two-level variant under a 64- and a 32-bit
    schedule in one fused pass over the short strings (every length 0..300,
    T = 1 strings included, all alignments) plus long members."""
    import torch

    rng = np.random.default_rng(7)
    lens = np.concatenate([np.repeat(np.arange(0, 301), 3), [5000, 70_000, 1024, 0]]).astype(np.uint64)
    rng.shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + 5
    pay = datagen.payload_host(71, 0, int(off[-1]))
    seeds = [71, 72]
    keys = [pmp.Keys.generate(s, b) for s, b in zip(seeds, order)]
    d_pay = torch.from_numpy(pay).to(dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(dev)
    n = lens.size
    outs = [torch.empty(n, dtype=torch.int64 if b == 64 else torch.int32, device=dev) for b in order]
    rc = pmp.pmp_hash2_batch_multi([k.handle for k in keys], d_pay.data_ptr(), d_off.data_ptr(), n,
                                   [o.data_ptr() for o in outs], 0)
    assert rc == 0
    torch.cuda.synchronize()
    for s, b, o in zip(seeds, order, outs):
        got = pmp.as_u64(o).astype(np.uint64)
        want = _want(oracle_lib, oracle_lib.keygen(s, b), pay, off)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (b, [(int(i), int(lens[i])) for i in bad[:8]])
