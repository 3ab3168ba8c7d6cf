"""GPU parity: the CUDA path (through the C ABI) against the oracle, bit-exact.

Integer hashing has exactly one correct digest per input, so every
comparison is element-by-element equality.  Sizes span several 4 KiB warp
tiles, level-2 nodes (128 blocks) and ragged tails; alignment offsets 0..15 are
swept for the realignment path.
"""
import os
import random

import numpy as np
import pytest

import datagen
import paper_1609_09840_b200 as pmp

pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 4


@pytest.fixture(scope="module")
def torch_dev():
    import torch

    import __graft_entry__

    __graft_entry__.build()
    torch.cuda.set_device(0)
    return torch.device("cuda:0")


@pytest.fixture(params=["tensor", "wordloop", "latency", "huge"])
def batch_path(request, torch_dev):
    """Run a batch test through the throughput path with short strings on the
    tensor cores (k_short_tc + k_wstring), with short strings in the word loop
    (k_short + k_wstring), through the latency path (k_small, batches of
    <= 4096 strings), and through the word-loop throughput path with the huge
    threshold lowered to 64 KiB (every string of >= 64 KiB node-parallel in
    k_huge)."""
    prev = pmp.pmp_set_small_batch_max(4096 if request.param == "latency" else 0)
    prev_tc = pmp.pmp_set_short_tc(1 if request.param == "tensor" else 0)
    prev_huge = pmp.pmp_set_huge_min(64 << 10 if request.param == "huge" else 4 << 20)
    yield request.param
    pmp.pmp_set_small_batch_max(prev)
    pmp.pmp_set_short_tc(prev_tc)
    pmp.pmp_set_huge_min(prev_huge)


def _u(bits):
    return np.uint64 if bits == 64 else np.uint32


def run_batch(torch_dev, keys, payload: np.ndarray, offsets: np.ndarray):
    import torch

    d_pay = torch.from_numpy(np.ascontiguousarray(payload) if payload.size else np.zeros(16, np.uint8)).to(torch_dev)
    d_off = torch.from_numpy(np.ascontiguousarray(offsets).view(np.int64)).to(torch_dev)
    out = pmp.hash_batch(keys, d_pay, d_off)
    torch.cuda.synchronize()
    return pmp.as_u64(out)


def oracle_batch(oracle_lib, seed, bits, payload, offsets):
    ok = oracle_lib.keygen(seed, bits)
    return oracle_lib.hash_batch(ok, payload, offsets, nthreads=NT).astype(_u(bits))


# ------------------------------------------------------------ device arithmetic
@pytest.mark.parametrize("bits", [32, 64])
def test_reduction_fuzz_and_algorithm2_branches(torch_dev, oracle_lib, bits):
    """Section 6.2 + Algorithm 2 on the device vs the exact residue mod p.
    Random 3-word values with w2 <= 128 plus constructed witnesses that
    reach every Algorithm 2 branch, including v1 = 2 (reading Q6), which random
    inputs never reach."""
    import torch

    n_bits = bits
    p = oracle_lib.params(bits)["p"]
    k = p - 2**bits
    mask = 2**n_bits - 1
    rng = random.Random(bits)
    cases = []
    for _ in range(200_000):
        cases.append((rng.getrandbits(n_bits), rng.getrandbits(n_bits), rng.randrange(0, 129)))
    # witnesses: v1 = 2 branch (w0 = 2^n - j), v1 = 1 branch (0,1,0), boundary battery
    for j in range(1, 2 * k + 3):
        cases.append(((2**n_bits - j) & mask, 0, 0))
    cases += [(0, 1, 0), (0, 0, 0), (k - 1, 0, 0), (2 * k - 1, 2, 0), (mask, mask, 128),
              (30, 2, 0), (k, 0, 0), (p & mask, p >> n_bits, 0), ((p - 1) & mask, (p - 1) >> n_bits, 0)]
    arr = np.array(cases, dtype=np.uint64)
    d_in = torch.from_numpy(arr.view(np.int64)).to(torch_dev)
    outs = {}
    for mode in (0, 3, 4):  # full residue (Alg. 2); folded V mod 2^n (digests); folded full residue
        d_out = torch.zeros(2 * len(cases), dtype=torch.int64, device=torch_dev)
        rc = pmp.pmp_selftest(bits, mode, d_in.data_ptr(), len(cases), d_out.data_ptr(),
                              torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        outs[mode] = d_out.cpu().numpy().view(np.uint64).reshape(-1, 2)
    for (w0, w1, w2), (lo, hi), (lo3, _), (lo4, hi4) in zip(cases, outs[0], outs[3], outs[4]):
        val = int(w0) + (int(w1) << n_bits) + (int(w2) << (2 * n_bits))
        got = int(lo) + (int(hi) << 64) if bits == 64 else int(lo)
        assert got == val % p, (w0, w1, w2)
        assert int(lo3) == (val % p) & mask, (w0, w1, w2)
        got4 = int(lo4) + (int(hi4) << 64) if bits == 64 else int(lo4)
        assert got4 == val % p, (w0, w1, w2)


@pytest.mark.parametrize("bits", [32, 64])
def test_block_mac_matches_oracle(torch_dev, oracle_lib, bits):
    """The hot-loop multiply-accumulate + reduction on full 128-word blocks,
    including maximal keys and words, vs the oracle's Eq. (1)."""
    import torch

    pr = oracle_lib.params(bits)
    rng = np.random.default_rng(bits)
    n = 3000
    recs = np.zeros((n, 257), dtype=np.uint64)
    hi = 2**bits - 1
    recs[:, 0] = rng.integers(0, hi, size=n, dtype=np.uint64, endpoint=True)
    recs[:, 1:129] = rng.integers(1, pr["a_max"], size=(n, 128), dtype=np.uint64, endpoint=True)
    recs[:, 129:] = rng.integers(0, hi, size=(n, 128), dtype=np.uint64, endpoint=True)
    recs[0, 0], recs[0, 1:129], recs[0, 129:] = hi, pr["a_max"], hi  # S:73 maximal case
    recs[1, 129:] = 0
    d_in = torch.from_numpy(recs.reshape(-1).view(np.int64)).to(torch_dev)
    d_out = torch.zeros(2 * n, dtype=torch.int64, device=torch_dev)
    assert pmp.pmp_selftest(bits, 1, d_in.data_ptr(), n, d_out.data_ptr(),
                            torch.cuda.current_stream().cuda_stream) == 0
    out = d_out.cpu().numpy().view(np.uint64).reshape(-1, 2)
    for t in range(n):
        want = oracle_lib.block(pr["p"], 128, int(recs[t, 0]), recs[t, 1:129], recs[t, 129:])
        assert int(out[t, 0]) + (int(out[t, 1]) << 64) == want, t


@pytest.mark.parametrize("bits", [32, 64])
def test_mixer_matches_oracle(torch_dev, oracle_lib, bits):
    import torch

    rng = np.random.default_rng(5)
    x = rng.integers(0, 2**bits - 1, size=10000, dtype=np.uint64, endpoint=True)
    x[:3] = [0, 1, 2**bits - 1]
    d_in = torch.from_numpy(x.view(np.int64)).to(torch_dev)
    d_out = torch.zeros(2 * x.size, dtype=torch.int64, device=torch_dev)
    assert pmp.pmp_selftest(bits, 2, d_in.data_ptr(), x.size, d_out.data_ptr(),
                            torch.cuda.current_stream().cuda_stream) == 0
    out = d_out.cpu().numpy().view(np.uint64).reshape(-1, 2)[:, 0]
    assert all(int(o) == oracle_lib.mix(bits, int(v)) for o, v in zip(out, x))


# ------------------------------------------------------------ batch path
@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.usefixtures("batch_path")
def test_tiny_config_every_hash(torch_dev, oracle_lib, bits):
    """configs[0] (1,000 strings, U[1,64] B, seed 1), every digest; at 32 bits too."""
    wl = datagen.WORKLOADS["tiny"]
    lens = wl.lengths()
    off = datagen.offsets_from_lengths(lens)
    pay = datagen.payload_host(wl.seed, 0, int(off[-1]))
    keys = pmp.Keys.generate(wl.seed, bits)
    got = run_batch(torch_dev, keys, pay, off)
    want = oracle_batch(oracle_lib, wl.seed, bits, pay, off)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("bits", [32, 64])
def test_keyfile_schedule_hashes_like_generated(torch_dev, oracle_lib, bits):
    """A schedule round-tripped through the KeyFile (8(f3)) is uploaded and used
    by the kernels exactly like the generated one: configs[0] against the oracle."""
    wl = datagen.WORKLOADS["tiny"]
    off = datagen.offsets_from_lengths(wl.lengths())
    pay = datagen.payload_host(wl.seed, 0, int(off[-1]))
    keys = pmp.Keys.load(pmp.Keys.generate(wl.seed, bits).save())
    assert np.array_equal(run_batch(torch_dev, keys, pay, off), oracle_batch(oracle_lib, wl.seed, bits, pay, off))


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("shift", [0, 1, 3, 8, 13])
@pytest.mark.usefixtures("batch_path")
def test_length_sweep_all_paths(torch_dev, oracle_lib, bits, shift):
    """Every length 0..2100 (short path <= 127 B, warp path beyond, 1..3 level-1
    blocks, ragged tails, marker-only blocks), payload shifted by `shift` bytes."""
    lens = np.arange(0, 2101, dtype=np.uint64)
    rng = np.random.default_rng(shift)
    rng.shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + shift
    pay = datagen.payload_host(11 + shift, 0, int(off[-1]))
    keys = pmp.Keys.generate(11, bits)
    got = run_batch(torch_dev, keys, pay, off)
    want = oracle_batch(oracle_lib, 11, bits, pay, off)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(int(i), int(lens[i])) for i in bad[:10]]


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.usefixtures("batch_path")
def test_all_short_batch_alignments(torch_dev, oracle_lib, bits):
    """The staged all-short warp path with every start alignment and empty strings."""
    rng = np.random.default_rng(bits + 100)
    lens = rng.integers(0, 128, size=20000, dtype=np.uint64)
    lens[::17] = 0
    off = datagen.offsets_from_lengths(lens) + 5
    pay = datagen.payload_host(3, 0, int(off[-1]))
    keys = pmp.Keys.generate(3, bits)
    assert np.array_equal(run_batch(torch_dev, keys, pay, off), oracle_batch(oracle_lib, 3, bits, pay, off))


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("shift", [0, 5])
@pytest.mark.usefixtures("batch_path")
def test_mid_strings_group_path(torch_dev, oracle_lib, bits, shift):
    """Mid strings (128 B <= B < 64 KiB: one 8-lane group per string, four per
    warp, warp batches of 32 handed out as groups finish): lengths at and around
    every multiple of 1 KiB (marker-only trailing blocks folded), the 64 KiB
    big-string boundary, and a log-uniform crowd so that batches rotate while
    groups are at different points of their strings; string count not a
    multiple of 32, short strings interleaved."""
    rng = np.random.default_rng(bits * 10 + shift)
    edge = [k * 1024 + d for k in range(1, 64) for d in (-1, 0, 1)] + [65535, 65536, 65537, 128, 129, 511, 512, 513]
    crowd = np.floor(2.0 ** rng.uniform(7, 16, size=3001)).astype(np.uint64)
    shorts = rng.integers(0, 128, size=500, dtype=np.uint64)
    lens = np.concatenate([np.array(edge, dtype=np.uint64), crowd, shorts])
    rng.shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + shift
    pay = datagen.payload_host(31 + shift, 0, int(off[-1]))
    keys = pmp.Keys.generate(31, bits)
    got = run_batch(torch_dev, keys, pay, off)
    want = oracle_batch(oracle_lib, 31, bits, pay, off)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, [(int(i), int(lens[i])) for i in bad[:10]]


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.usefixtures("batch_path")
def test_long_strings_in_batch(torch_dev, oracle_lib, bits):
    """Warp-per-string path across level-2 (128 blocks) and level-3 (128^2 blocks)
    boundaries, misaligned starts, mixed with short strings and big ones first."""
    cb = 128 * bits // 8
    lens = [cb * 128 - 1, cb * 128, cb * 128 + 1, cb * 128 * 2 + 5, 300_000, 70_000, 5, 0, 127, 128,
            cb * 128 * 128 + cb + 3, 3 * cb, 3 * cb + 1]
    lens = np.array(lens, dtype=np.uint64)
    off = datagen.offsets_from_lengths(lens) + 7
    pay = datagen.payload_host(21, 0, int(off[-1]))
    keys = pmp.Keys.generate(21, bits)
    got = run_batch(torch_dev, keys, pay, off)
    want = oracle_batch(oracle_lib, 21, bits, pay, off)
    assert np.array_equal(got, want), np.nonzero(got != want)[0]


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.usefixtures("batch_path")
def test_algorithm2_rare_branches_end_to_end(torch_dev, oracle_lib, bits):
    """Key schedules built so a block sum equals 2^n - j (v1 = 2 branch of
    Algorithm 2) or 2^n (v1 = 1 branch): b = 2^n - 2 - j, a = 1, one data word 1
    and the marker word 1 -> S = b + 1 + 1."""
    import torch

    w = bits // 8
    for j in [0, 1, 5, 12, 13, 14, 15, 16, 29, 30, 31]:
        bval = (2**bits - 2 - j) % 2**bits
        b = np.full(8, bval, dtype=np.uint64)
        a = np.ones((8, 128), dtype=np.uint64)
        keys = pmp.Keys.from_words(bits, b, a)
        data = (1).to_bytes(w, "little")
        pay = np.frombuffer(data * 3 + b"\x00" * 13, dtype=np.uint8).copy()
        off = np.array([0, w, 2 * w, 3 * w], dtype=np.uint64)
        got = run_batch(torch_dev, keys, pay, off)
        ok = oracle_lib.Keys(bits, b, a)
        want = oracle_lib.hash_batch(ok, pay, off).astype(_u(bits))
        assert np.array_equal(got, want), j
        d = torch.from_numpy(pay[:w].copy()).to(torch_dev)
        assert int(pmp.as_u64(pmp.hash_long(keys, d, w))[0]) == int(want[0])


# ------------------------------------------------------------ long path
LONG_LENS = [0, 1, 7, 8, 9, 1000, 1023, 1024, 1025, 4096, 128 * 1024 - 8, 128 * 1024, 128 * 1024 + 1,
             128 * 512, 128 * 512 + 3, 1 << 20, (1 << 20) + 13, 128 * 128 * 1024 + 1024 + 9,
             128 * 128 * 1024, 128 * 128 * 512 - 4]


@pytest.mark.parametrize("bits", [32, 64])
def test_hash_long_lengths(torch_dev, oracle_lib, bits):
    import torch

    ok = oracle_lib.keygen(4, bits)
    keys = pmp.Keys.generate(4, bits)
    big = datagen.payload_host(4, 0, max(LONG_LENS) + 64)
    d_big = torch.from_numpy(big).to(torch_dev)
    for L in LONG_LENS:
        for shift in (0, 5):
            got = int(pmp.as_u64(pmp.hash_long(keys, d_big[shift:], L))[0])
            want = oracle_lib.hash_long(ok, big[shift:shift + L], nthreads=NT)
            assert got == want, (L, shift)


@pytest.mark.parametrize("bits", [32, 64])
def test_long_partition_invariance(torch_dev, oracle_lib, bits):
    """Partial + combine over G block-aligned ranges gives the same digest as
    one call, for G = 1..8 and random splits (SURVEY 8(c.3) partition invariance)."""
    import torch

    cb = 128 * bits // 8
    total = 3 * 128 * 128 * cb // 2 + 777  # three level-3 subtrees' worth, ragged
    keys = pmp.Keys.generate(8, bits)
    data = datagen.payload_host(8, 0, total)
    d = torch.from_numpy(data).to(torch_dev)
    ref = int(pmp.as_u64(pmp.hash_long(keys, d, total))[0])
    want = oracle_lib.hash_long(oracle_lib.keygen(8, bits), data, nthreads=NT)
    assert ref == want
    rng = random.Random(bits)
    splits = [pmp.pmp_long_split(bits, total, G) for G in (1, 2, 3, 4, 8)]
    for _ in range(4):
        cuts = sorted(rng.sample(range(1, total // cb), 5))
        splits.append([0] + [c * cb for c in cuts] + [total])
    for b in splits:
        G = len(b) - 1
        parts = torch.zeros(2 * G, dtype=torch.int64, device=torch_dev)
        for g in range(G):
            pmp.hash_long_partial(keys, d[b[g]:], b[g + 1] - b[g], b[g], total, partial=parts[2 * g:2 * g + 2])
        got = int(pmp.as_u64(pmp.hash_long_combine(keys, parts, total))[0])
        assert got == ref, b


@pytest.mark.parametrize("bits", [32, 64])
def test_long_partition_degenerate_ranges(torch_dev, oracle_lib, bits):
    """Splits with empty ranges: the tail block belongs to the range
    holding the last byte only, so pmp_long_split(total, G) for tiny totals,
    trailing / leading / repeated empty ranges, and the empty message give the
    one-call digest (= the oracle's) for every G."""
    import torch

    cb = 128 * bits // 8
    keys = pmp.Keys.generate(9, bits)
    okeys = oracle_lib.keygen(9, bits)
    for total in (0, 1, 3, 5, cb - 1, cb, 2 * cb, 3 * cb + 7, 128 * cb, 128 * cb + 1):
        data = datagen.payload_host(9, 0, max(total, 1))[:total]
        d = torch.from_numpy(np.concatenate([data, np.zeros(16, np.uint8)])).to(torch_dev)
        want = oracle_lib.hash_long(okeys, data, nthreads=NT)
        assert int(pmp.as_u64(pmp.hash_long(keys, d, total))[0]) == want, total
        splits = [pmp.pmp_long_split(bits, total, G) for G in (1, 2, 3, 8)]
        nb = total // cb
        splits += [[0, 0, total], [0, 0, 0, total]]
        if total % cb == 0:                   # a range may start at `total` only if block-aligned
            splits += [[0, total, total], [0, 0, total, total, total]]
            if nb >= 2:
                splits += [[0, cb, total, total]]
        if nb >= 2:
            splits += [[0, cb, cb, total]]
        for b in splits:
            G = len(b) - 1
            parts = torch.zeros(2 * G, dtype=torch.int64, device=torch_dev)
            for g in range(G):
                pmp.hash_long_partial(keys, d[b[g]:], b[g + 1] - b[g], b[g], total,
                                      partial=parts[2 * g:2 * g + 2])
            got = int(pmp.as_u64(pmp.hash_long_combine(keys, parts, total))[0])
            assert got == want, (total, b)


# ------------------------------------------------------------ hash-table consumer
@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("M", [1, 7, 1024, 50_000, 2**32 - 1])   # 50,000: histogram without the smem copy
@pytest.mark.usefixtures("batch_path")
def test_buckets_and_histogram(torch_dev, oracle_lib, bits, M):
    """pmp_hash_batch_buckets == oracle digest mod M, and its fused histogram ==
    bincount, for a batch mixing short, long, empty and misaligned strings."""
    import torch

    rng = np.random.default_rng(M % 1000 + bits)
    lens = rng.integers(0, 300, size=5000).astype(np.uint64)
    lens[::97] = rng.integers(1000, 70000, size=lens[::97].size).astype(np.uint64)
    off = datagen.offsets_from_lengths(lens) + 3
    pay = datagen.payload_host(31, 0, int(off[-1]))
    keys = pmp.Keys.generate(31, bits)
    d_pay = torch.from_numpy(pay).to(torch_dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
    Mc = min(M, 1 << 16)
    counts = torch.zeros(Mc, dtype=torch.int32, device=torch_dev) if M == Mc else None
    b = pmp.hash_batch_buckets(keys, d_pay, d_off, M, counts=counts)
    torch.cuda.synchronize()
    got = b.cpu().numpy().view(np.uint32).astype(np.uint64)
    want = oracle_batch(oracle_lib, 31, bits, pay, off).astype(np.uint64) % np.uint64(M)
    assert np.array_equal(got, want)
    if counts is not None:
        assert np.array_equal(counts.cpu().numpy().astype(np.int64), np.bincount(want.astype(np.int64), minlength=M))


@pytest.mark.parametrize("M,n", [(1, 3000), (7, 5000), (1024, 5000), (1024, 1 << 20), (12288, 200000),
                                 (50000, 200000), (1 << 24, 70000)])
def test_bucket_partition(torch_dev, oracle_lib, M, n):
    """pmp_bucket_partition after pmp_hash_batch_buckets: starts
    == exclusive prefix sums of the oracle buckets' bincount; perm is a
    permutation of 0..n-1 whose oracle buckets are grouped in bucket order and
    match starts (the order inside a bucket is free).  Covers the shared-memory
    ranked path (M <= 12288) and the global-atomic path."""
    import torch

    rng = np.random.default_rng(M + n)
    lens = rng.integers(0, 100, size=n).astype(np.uint64)
    off = datagen.offsets_from_lengths(lens)
    pay = datagen.payload_host(41, 0, int(off[-1]))
    keys = pmp.Keys.generate(41, 64)
    d_pay = torch.from_numpy(pay).to(torch_dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
    hist = torch.zeros(M, dtype=torch.int32, device=torch_dev) if M <= 65536 else None
    b = pmp.hash_batch_buckets(keys, d_pay, d_off, M, counts=hist)
    starts, perm = pmp.bucket_partition(b, M)
    if hist is not None:                                   # the caller's histogram instead of a recount
        starts2, perm2 = pmp.bucket_partition(b, M, hist=hist)
        assert torch.equal(starts2, starts)
        p2 = perm2.cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(np.sort(p2), np.arange(n))
    torch.cuda.synchronize()
    ob = (oracle_batch(oracle_lib, 41, 64, pay, off).astype(np.uint64) % np.uint64(M)).astype(np.int64)
    want_starts = np.concatenate([[0], np.cumsum(np.bincount(ob, minlength=M))])
    assert np.array_equal(starts.cpu().numpy(), want_starts)
    p = perm.cpu().numpy().view(np.uint32).astype(np.int64)
    assert np.array_equal(np.sort(p), np.arange(n))
    grouped = ob[p]
    assert np.all(np.diff(grouped) >= 0)
    assert np.array_equal(np.searchsorted(grouped, np.arange(M + 1), side="left"), want_starts)


# ------------------------------------------------------------ quality suite
@pytest.mark.parametrize("bits,length", [(64, 8), (64, 16), (32, 4), (32, 12)])
def test_avalanche_bias_small(torch_dev, oracle_lib, bits, length):
    """SPEC S:437 threshold (worst bias < 0.03); 3e4 trials keep the binomial
    noise (sd 0.003) far below it.  The digest path is cross-checked against
    the oracle on one trial's batch."""
    from paper_1609_09840_b200 import quality

    keys = pmp.Keys.generate(77, bits)
    worst, freq, (pay, off, dig) = quality.avalanche(keys, length, 30000, seed=5, first_batch=True)
    assert freq.shape == (8 * length, bits)
    assert worst < 0.03, worst
    # the digests the statistics came from: the first chunk's batch (4096 inputs
    # and all their single-bit flips) recomputed by the oracle, digest by digest
    want = oracle_batch(oracle_lib, 77, bits, pay, off)
    assert np.array_equal(dig, want)


@pytest.mark.parametrize("bits", [32, 64])
def test_collision_monte_carlo(torch_dev, oracle_lib, bits):
    """SPEC quality_suite collision_monte_carlo (Table 3 P:644-646,
    h mod M P:188-192): for fixed pairs, 10^6 device-drawn key schedules.
    The first 1,000 schedules' digests of both strings equal the oracle's with
    keygen(seed0 + i); distinct pairs never collide in all n bits (rate <= 1e-4,
    expected 0); low-8 / low-16-bit collisions (buckets of 2^8 / 2^16-entry
    tables) occur at rate 2^-k within 6 sigma; the (s, s) control collides
    always; sub-word strings (|sigma| = 1, reading Q2) are key-independent."""
    from paper_1609_09840_b200 import quality

    rng = np.random.default_rng(bits)
    a = bytes(rng.integers(0, 256, 37, dtype=np.uint8))
    b = bytearray(a)
    b[5] ^= 0x10                                   # one bit apart
    pairs = [(a, bytes(b)), (a[:12], a[1:13]), (a[:1], a[:2] if bits == 64 else a[:3]), (b"", b"\x00"),
             (a + a[:90], a[::-1] + a[:90])]
    N = 1_000_000
    seed0 = 1 << 33
    for s1, s2 in pairs:
        r = quality.collision_monte_carlo(bits, s1, s2, 1000, seed0=seed0, return_digests=True)
        g1, g2 = r["digests"]
        ok1 = [oracle_lib.hash_bytes(oracle_lib.keygen(seed0 + i, bits), s1) for i in range(0, 1000, 7)]
        ok2 = [oracle_lib.hash_bytes(oracle_lib.keygen(seed0 + i, bits), s2) for i in range(0, 1000, 7)]
        assert [int(x) for x in g1[::7]] == ok1 and [int(x) for x in g2[::7]] == ok2, (s1, s2)
        r = quality.collision_monte_carlo(bits, s1, s2, N, seed0=seed0)
        assert r["full"] == 0 and r["rate_full"] <= 1e-4, (s1, s2, r)
        if len(s1) >= bits // 8 or len(s2) >= bits // 8:
            for k, key in ((8, "rate_low8"), (16, "rate_low16")):
                pk = 2.0 ** -k
                assert abs(r[key] - pk) <= 6 * (pk * (1 - pk) / N) ** 0.5 + 1e-9, (k, r)
        else:                                      # both |sigma| = 1: digests do not depend on the keys
            assert r["low8"] in (0, N) and r["low16"] in (0, N)
    r = quality.collision_monte_carlo(bits, a, a, N, seed0=seed0)
    assert r["full"] == r["low16"] == r["low8"] == N


@pytest.mark.parametrize("bits", [32, 64])
def test_single_word_sweep_regularity(torch_dev, oracle_lib, bits):
    """Component-wise regularity at production scale: <= p - 2^n collisions over
    a 2^24-value sweep (a random function would give ~2^47/2^n)."""
    from paper_1609_09840_b200 import quality

    keys = pmp.Keys.generate(78, bits)
    coll = quality.word_sweep(keys, 1 << 24, seed=6)
    assert 0 <= coll <= quality.bound(bits)


# ------------------------------------------------------------ streaming
@pytest.mark.parametrize("bits", [32, 64])
def test_stream_split_invariance(torch_dev, oracle_lib, bits):
    """pmp_stream_update over random cuts (tiny, block-straddling, multi-node,
    misaligned) gives the digest of pmp_hash_long / the oracle on the whole."""
    import torch

    cb = 128 * bits // 8
    rng = random.Random(bits)
    keys = pmp.Keys.generate(90, bits)
    ok = oracle_lib.keygen(90, bits)
    for total in [0, 1, 7, cb - 1, cb, cb + 1, 3 * cb + 5, 128 * cb, 128 * cb + 1, 300 * cb + 77,
                  128 * 128 * cb + 3 * cb + 9]:
        data = datagen.payload_host(91 + total % 7, 0, total)
        d = torch.from_numpy(data if total else np.zeros(1, np.uint8)).to(torch_dev)
        want = oracle_lib.hash_long(ok, data, nthreads=NT)
        for trial in range(3):
            st = pmp.Stream(keys)
            pos = 0
            while pos < total:
                kind = rng.random()
                step = rng.randrange(1, 17) if kind < 0.4 else (rng.randrange(1, 3 * cb) if kind < 0.8
                                                               else rng.randrange(1, 300 * cb))
                step = min(step, total - pos)
                st.update(d[pos:], step)
                pos += step
            got = int(pmp.as_u64(st.final())[0])
            assert got == want, (total, trial)
            st.close()


@pytest.mark.parametrize("bits", [32, 64])
def test_stream_large_pieces(torch_dev, oracle_lib, bits):
    """Pieces of 2-40 MiB (hundreds of level-2 nodes per update, so fewer
    pieces per node in k_node and many nodes completing inside one merge),
    with level-3 nodes closing mid-update, against the oracle."""
    import torch

    cb = 128 * bits // 8
    total = 3 * 128 * 128 * cb + 5 * cb + 3
    data = datagen.payload_host(95 + bits, 0, total)
    d = torch.from_numpy(data).to(torch_dev)
    keys = pmp.Keys.generate(94, bits)
    want = oracle_lib.hash_long(oracle_lib.keygen(94, bits), data, nthreads=NT)
    for cuts in ([total], [total // 3 + 17, total // 2 + 1000], [2 * 128 * 128 * cb - 1, 1, 5 << 20]):
        st = pmp.Stream(keys)
        pos = 0
        for c in cuts + [total - sum(cuts)]:
            if c:
                st.update(d[pos:], c)
            pos += c
        assert int(pmp.as_u64(st.final())[0]) == want, cuts
        st.close()


def test_stream_reset_and_reuse(torch_dev, oracle_lib):
    import torch

    keys = pmp.Keys.generate(92, 64)
    st = pmp.Stream(keys)
    for total in (5000, 17, 0):
        data = datagen.payload_host(93, 0, total)
        d = torch.from_numpy(data if total else np.zeros(1, np.uint8)).to(torch_dev)
        if total:
            st.update(d, total)
        got = int(pmp.as_u64(st.final())[0])
        assert got == oracle_lib.hash_long(oracle_lib.keygen(92, 64), data)
        with pytest.raises(pmp.PmpError):
            st.update(d, 1)
        st.reset()


@pytest.mark.parametrize("piece", [0, 4096, 100_000])
@pytest.mark.usefixtures("batch_path")
def test_host_batch_streaming(torch_dev, oracle_lib, piece):
    """pmp_hash_batch_host (host-resident bytes/offsets/digests, two key
    schedules at once) equals the device path and the oracle: pieces smaller
    than one string (a string alone in its piece), pieces ending anywhere,
    a batch that starts at an odd offset of its buffer."""
    rng = np.random.default_rng(piece + 1)
    lens = np.concatenate([rng.integers(0, 200, size=3000), [70_000, 5000, 0, 1, 127, 128, 9000]]).astype(np.uint64)
    rng.shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + 11
    pay = datagen.payload_host(41, 0, int(off[-1]))
    k64, k32 = pmp.Keys.generate(41, 64), pmp.Keys.generate(42, 32)
    got64, got32 = pmp.hash_batch_host([k64, k32], pay, off, piece_bytes=piece)
    assert np.array_equal(got64, oracle_batch(oracle_lib, 41, 64, pay, off))
    assert np.array_equal(got32, oracle_batch(oracle_lib, 42, 32, pay, off))
    assert np.array_equal(got64, run_batch(torch_dev, k64, pay, off))


@pytest.mark.parametrize("bits", [32, 64])
def test_long_host_streaming(torch_dev, oracle_lib, bits):
    """pmp_hash_long_host (host-resident string -> pieces copied into three device
    slots on internal streams -> incremental device state): equal to
    pmp_hash_long and the oracle for lengths around block / node boundaries and
    piece sizes smaller than, equal to and larger than the string."""
    import torch

    cb = 128 * bits // 8
    keys = pmp.Keys.generate(61, bits)
    ok = oracle_lib.keygen(61, bits)
    for total in (0, 1, 7, cb - 1, cb, cb + 1, 128 * cb + 5, 3 * 128 * cb + 777):
        data = datagen.payload_host(61, 0, max(total, 1))[:total]
        want = oracle_lib.hash_long(ok, data, nthreads=NT)
        pinned = torch.from_numpy(data.copy()).pin_memory() if total else torch.zeros(0, dtype=torch.uint8)
        for piece in (0, cb, 3 * cb, 1 << 20):
            assert pmp.hash_long_host(keys, pinned, piece_bytes=piece) == want, (total, piece)
        assert pmp.hash_long_host(keys, data, piece_bytes=5 * cb) == want, total   # pageable host memory


@pytest.mark.parametrize("nlong", [1, 2, 3, 5, 7, 8])
def test_small_batch_long_strings_split(torch_dev, oracle_lib, nlong):
    """Latency path (k_small, 8 strings per block): a block with fewer long
    strings than warps splits each multi-node string over its spare warps by
    the affine identity (V = C(T) + sum_q W(q) v2'(q), C(T) on the device,
    pmp_split.cuh); 8 long strings take one warp each.  Sizes around level-2
    node edges, strings with a level-3 and level-4 tree, misaligned starts;
    both widths and the fused two-schedule call, equal to the oracle."""
    import torch

    rng = np.random.default_rng(nlong)
    prev = pmp.pmp_set_small_batch_max(4096)
    try:
        cands = [128 * 1024 * 2 + 5, 128 * 1024 * 3 - 1, 128 * 1024 + 1, 128 * 512 * 5 + 17, 1_000_003,
                 128 * 1024 * 128 + 1024 + 3, 128 * 512 * 129 + 7, 128 * 1024 - 1, 400_000]
        for rep in range(2):
            longs = list(rng.choice(cands, size=nlong, replace=False)) if rep == 0 else list(cands[:nlong])
            lens = np.array(longs + list(rng.integers(0, 128, size=8 - nlong)) + [3, 200_000, 9], dtype=np.uint64)
            perm = rng.permutation(8)
            lens[:8] = lens[:8][perm]
            off = datagen.offsets_from_lengths(lens) + int(rng.integers(0, 16))
            pay = datagen.payload_host(60 + nlong, 0, int(off[-1]))
            d_pay = torch.from_numpy(pay).to(torch_dev)
            d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
            k64, k32 = pmp.Keys.generate(61, 64), pmp.Keys.generate(62, 32)
            w64 = oracle_batch(oracle_lib, 61, 64, pay, off)
            w32 = oracle_batch(oracle_lib, 62, 32, pay, off)
            s64, s32 = pmp.hash_batch(k64, d_pay, d_off), pmp.hash_batch(k32, d_pay, d_off)
            m64, m32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
            torch.cuda.synchronize()
            for name, o, w in (("64", s64, w64), ("32", s32, w32), ("dual64", m64, w64), ("dual32", m32, w32)):
                got = pmp.as_u64(o)
                bad = np.nonzero(got != w)[0]
                assert bad.size == 0, (name, rep, [(int(i), int(lens[i])) for i in bad[:8]])
    finally:
        pmp.pmp_set_small_batch_max(prev)


@pytest.mark.parametrize("cap", [65536, 2])
def test_huge_strings_throughput_path(torch_dev, oracle_lib, cap):
    """Throughput path with the huge threshold lowered to 64 KiB: long strings
    go to k_huge (parts of 128 KiB claimed grid-wide, exact sums by atomics,
    C(T) added by the warp finishing the last part; pmp_huge.cuh), at most
    `cap` of them per call (the rest stay on k_wstring's big list).  Sizes at
    level-2 node edges of both widths, level-3 and level-4 trees, misaligned
    starts, mixed with short and mid strings; single schedules, the fused
    two-schedule call and bucket mode, equal to the oracle."""
    import torch

    rng = np.random.default_rng(cap)
    prev = (pmp.pmp_set_small_batch_max(0), pmp.pmp_set_huge_min(64 << 10), pmp.pmp_set_huge_cap(cap))
    try:
        big = [64 << 10, (128 << 10) - 1, 128 << 10, (128 << 10) + 1, (512 << 10) + 3, 1_000_003,
               (128 << 20) // 8 + 1024 + 3, (64 << 10) * 129 + 7, 300_000]
        lens = np.concatenate([rng.integers(0, 128, size=3000), rng.integers(128, 60000, size=200), big])
        lens = lens.astype(np.uint64)
        rng.shuffle(lens)
        off = datagen.offsets_from_lengths(lens) + 5
        pay = datagen.payload_host(70, 0, int(off[-1]))
        d_pay = torch.from_numpy(pay).to(torch_dev)
        d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
        k64, k32 = pmp.Keys.generate(71, 64), pmp.Keys.generate(72, 32)
        w64 = oracle_batch(oracle_lib, 71, 64, pay, off)
        w32 = oracle_batch(oracle_lib, 72, 32, pay, off)
        s64, s32 = pmp.hash_batch(k64, d_pay, d_off), pmp.hash_batch(k32, d_pay, d_off)
        m64, m32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
        M = 1000
        bk = torch.empty(len(lens), dtype=torch.int32, device=torch_dev)
        rc = pmp.pmp_hash_batch_buckets(k64.handle, d_pay.data_ptr(), d_off.data_ptr(), len(lens), M, bk.data_ptr(),
                                        None, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        for name, o, w in (("64", s64, w64), ("32", s32, w32), ("dual64", m64, w64), ("dual32", m32, w32)):
            got = pmp.as_u64(o)
            bad = np.nonzero(got != w)[0]
            assert bad.size == 0, (name, [(int(i), int(lens[i])) for i in bad[:8]])
        assert np.array_equal(bk.cpu().numpy().view(np.uint32), (w64 % M).astype(np.uint32))
    finally:
        pmp.pmp_set_small_batch_max(prev[0])
        pmp.pmp_set_huge_min(prev[1])
        pmp.pmp_set_huge_cap(prev[2])


@pytest.mark.parametrize("order", [(64, 32), (32, 64), (64, 64, 32), (32,)])
@pytest.mark.usefixtures("batch_path")
def test_multi_schedule_fused_pass(torch_dev, oracle_lib, order):
    """pmp_hash_batch_multi: a 64-bit and a 32-bit schedule are fused into one
    pass over the short strings (the 32-bit words are the halves of the 64-bit
    ones; markers and masks per width), long strings per schedule over the
    shared work list.  Every length 0..300 (both markers in every position,
    both |sigma| = 1 cases), all alignments, plus long members; equal to the
    oracle under each schedule."""
    import torch

    rng = np.random.default_rng(len(order))
    lens = np.concatenate([np.repeat(np.arange(0, 301), 3), [5000, 70_000, 1024, 4096, 0]]).astype(np.uint64)
    rng.shuffle(lens)
    off = datagen.offsets_from_lengths(lens) + 9
    pay = datagen.payload_host(51, 0, int(off[-1]))
    seeds = [51 + i for i in range(len(order))]
    keys = [pmp.Keys.generate(s, b) for s, b in zip(seeds, order)]
    d_pay = torch.from_numpy(pay).to(torch_dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
    outs = pmp.hash_batch_multi(keys, d_pay, d_off)
    torch.cuda.synchronize()
    for s, b, o in zip(seeds, order, outs):
        got = pmp.as_u64(o)
        want = oracle_batch(oracle_lib, s, b, pay, off)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (b, [(int(i), int(lens[i])) for i in bad[:8]])


@pytest.mark.parametrize("trial", range(32))
@pytest.mark.usefixtures("batch_path")
def test_random_batches_soak(torch_dev, oracle_lib, trial):
    """Randomised batches through every batch entry point (pmp_hash_batch,
    the fused two-schedule pmp_hash_batch_multi, the host-resident path):
    random count, length law (short / mid / big / mixed), payload shift, key
    seeds; bit-exact against the oracle."""
    import torch

    rng = np.random.default_rng(1000 + trial)
    n = int(rng.integers(1, 4000))
    law = trial % 4
    if law == 0:
        lens = rng.integers(0, 128, size=n)
    elif law == 1:
        lens = np.floor(2.0 ** rng.uniform(7, 16, size=n))
    elif law == 2:
        n = int(rng.integers(1, 40))
        lens = np.floor(2.0 ** rng.uniform(16, 19, size=n))
    else:
        lens = np.floor(2.0 ** rng.uniform(0, 18, size=n))
    lens = lens.astype(np.uint64)
    off = datagen.offsets_from_lengths(lens) + int(rng.integers(0, 16))
    pay = datagen.payload_host(int(rng.integers(1, 1 << 30)), 0, int(off[-1]))
    s64, s32 = int(rng.integers(1, 1 << 40)), int(rng.integers(1, 1 << 40))
    k64, k32 = pmp.Keys.generate(s64, 64), pmp.Keys.generate(s32, 32)
    want64 = oracle_batch(oracle_lib, s64, 64, pay, off)
    want32 = oracle_batch(oracle_lib, s32, 32, pay, off)
    d_pay = torch.from_numpy(pay if pay.size else np.zeros(16, np.uint8)).to(torch_dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
    o64, o32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
    torch.cuda.synchronize()
    assert np.array_equal(pmp.as_u64(o64), want64)
    assert np.array_equal(pmp.as_u64(o32), want32)
    assert np.array_equal(run_batch(torch_dev, k64, pay, off), want64)
    h64, h32 = pmp.hash_batch_host([k64, k32], pay, off, piece_bytes=int(rng.integers(1, 1 << 20)))
    assert np.array_equal(h64, want64) and np.array_equal(h32, want32)


@pytest.mark.usefixtures("batch_path")
def test_entry_points_edge_cases(torch_dev, oracle_lib):
    """n = 0 is a no-op and n = 1 works through every batch entry point; an
    offsets array that is not 16-byte aligned (the kernels' TMA source) is
    accepted; NULL arguments are PMP_EINVAL, not a fault."""
    import torch

    k64, k32 = pmp.Keys.generate(5, 64), pmp.Keys.generate(6, 32)
    pay = datagen.payload_host(9, 0, 5000)
    d_pay = torch.from_numpy(pay).to(torch_dev)
    for lens in ([], [0], [1], [127], [128], [4999]):
        off = datagen.offsets_from_lengths(np.array(lens, dtype=np.uint64)) + 1
        d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
        o64, o32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
        h64, h32 = pmp.hash_batch_host([k64, k32], pay, off)
        torch.cuda.synchronize()
        if lens:
            assert np.array_equal(pmp.as_u64(o64), oracle_batch(oracle_lib, 5, 64, pay, off))
            assert np.array_equal(pmp.as_u64(o32), oracle_batch(oracle_lib, 6, 32, pay, off))
            assert np.array_equal(h64, pmp.as_u64(o64)) and np.array_equal(h32, pmp.as_u64(o32))
    # offsets starting 8 bytes into an allocation (not 16-byte aligned)
    lens = np.arange(0, 300, dtype=np.uint64)
    off = datagen.offsets_from_lengths(lens)
    buf = torch.from_numpy(np.concatenate([[0], off.view(np.int64)])).to(torch_dev)
    d_off = buf[1:]
    assert d_off.data_ptr() % 16 == 8
    big = torch.from_numpy(datagen.payload_host(9, 0, int(off[-1]))).to(torch_dev)
    got = pmp.as_u64(pmp.hash_batch(k64, big, d_off))
    assert np.array_equal(got, oracle_batch(oracle_lib, 5, 64, big.cpu().numpy(), off))
    assert pmp.pmp_hash_batch(k64.handle, 0, d_off.data_ptr(), 3, d_off.data_ptr(), 0) == pmp.PMP_EINVAL
    assert pmp.pmp_hash_batch_multi([k64.handle], big.data_ptr(), d_off.data_ptr(), 3, [0], 0) == pmp.PMP_EINVAL


@pytest.mark.parametrize("n", [479, 480, 481, 960, 961, 4097, 296 * 480 - 1, 296 * 480 + 1, 3 * 296 * 480 + 77,
                               296 * 512 + 1])
@pytest.mark.usefixtures("batch_path")
def test_short_tile_claims_at_tile_boundaries(torch_dev, oracle_lib, n):
    """k_short claims its 480-string tiles dynamically (one global counter; a
    failed claim ends the block; single-width kernels claim one call ahead):
    string counts around tile multiples and beyond one tile per resident block
    hash every string exactly once -- fused two-width pass and both single
    widths, bit-exact against the oracle."""
    import torch

    rng = np.random.default_rng(n)
    lens = rng.integers(0, 128, size=n).astype(np.uint64)
    lens[rng.integers(0, n, size=max(1, n // 5000))] = 3000  # a few work-list strings
    off = datagen.offsets_from_lengths(lens) + int(rng.integers(0, 16))
    pay = datagen.payload_host(n, 0, int(off[-1]))
    k64, k32 = pmp.Keys.generate(21, 64), pmp.Keys.generate(22, 32)
    want64 = oracle_batch(oracle_lib, 21, 64, pay, off)
    want32 = oracle_batch(oracle_lib, 22, 32, pay, off)
    d_pay = torch.from_numpy(pay).to(torch_dev)
    d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
    o64, o32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
    torch.cuda.synchronize()
    assert np.array_equal(pmp.as_u64(o64), want64)
    assert np.array_equal(pmp.as_u64(o32), want32)
    assert np.array_equal(run_batch(torch_dev, k64, pay, off), want64)
    assert np.array_equal(run_batch(torch_dev, k32, pay, off), want32)


def test_concurrent_calls_share_key_handles(torch_dev, oracle_lib):
    """Key handles are shareable across threads and streams (S:174, S:269,
    S:326): four host threads hash different batches (throughput path, latency
    path, host-resident path, long string) with the SAME handles on their own
    streams at once; every result equals the oracle's."""
    import threading

    import torch

    k64, k32 = pmp.Keys.generate(71, 64), pmp.Keys.generate(72, 32)
    rng = np.random.default_rng(71)
    jobs = []
    for j in range(4):
        lens = rng.integers(0, 300, size=6000 if j % 2 == 0 else 1500).astype(np.uint64)
        off = datagen.offsets_from_lengths(lens) + j
        pay = datagen.payload_host(80 + j, 0, int(off[-1]))
        jobs.append((off, pay))
    long_data = datagen.payload_host(90, 0, 3 * 1024 * 128 + 11)
    results, errors = {}, []

    def work(j):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                off, pay = jobs[j]
                if j == 2:
                    results[j] = pmp.hash_batch_host([k64, k32], pay, off)
                else:
                    d_pay = torch.from_numpy(pay).to(torch_dev, non_blocking=False)
                    d_off = torch.from_numpy(off.view(np.int64)).to(torch_dev)
                    o64, o32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
                    st.synchronize()
                    results[j] = (pmp.as_u64(o64), pmp.as_u64(o32))
                if j == 3:
                    d = torch.from_numpy(long_data).to(torch_dev)
                    out = pmp.hash_long(k64, d, long_data.size)
                    st.synchronize()
                    results["long"] = int(pmp.as_u64(out)[0])
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ths = [threading.Thread(target=work, args=(j,)) for j in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    for j in range(4):
        off, pay = jobs[j]
        assert np.array_equal(results[j][0], oracle_batch(oracle_lib, 71, 64, pay, off)), j
        assert np.array_equal(results[j][1], oracle_batch(oracle_lib, 72, 32, pay, off)), j
    assert results["long"] == oracle_lib.hash_long(oracle_lib.keygen(71, 64), long_data, nthreads=NT)
