"""CPU checks of the C-ABI library: it loads, exports every symbol include/pmp.h
declares, validates arguments, and its host logic (key generation, long-string
split, key-only constant) matches the oracle.  No compute call needs a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1609_09840_b200 as pmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__

    __graft_entry__.build()
    return pmp.lib()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pmp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(L, s), s
    # and nothing in the product library links the oracle
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", pmp.LIB_PATH], capture_output=True, text=True).stdout
    assert "pmpo_" not in out


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4, 5, 2**64 - 1])
def test_keygen_matches_oracle_contract(L, oracle_lib, bits, seed):
    """Both sides implement the Q12 key contract independently; the schedules
    must be word-for-word identical."""
    h = pmp.pmp_keygen(seed, bits)
    assert h
    k = pmp.Keys(h, bits)
    b, a = k.export()
    ok = oracle_lib.keygen(seed, bits)
    assert np.array_equal(b, ok.b) and np.array_equal(a, ok.a)


def test_bad_arguments(L):
    assert pmp.pmp_keygen(1, 48) == 0
    b = np.zeros(8, dtype=np.uint64)
    a = np.ones(1024, dtype=np.uint64)
    assert pmp.pmp_keys_from_words(64, b.ctypes.data, a.ctypes.data) != 0
    a[5] = 0  # a key must be non-zero
    assert pmp.pmp_keys_from_words(64, b.ctypes.data, a.ctypes.data) == 0
    a[5] = 2**64 - 11  # above p - kappa - 1 = 2^64 - 12
    assert pmp.pmp_keys_from_words(64, b.ctypes.data, a.ctypes.data) == 0
    a[5] = 2**64 - 12
    h = pmp.pmp_keys_from_words(64, b.ctypes.data, a.ctypes.data)
    assert h
    a[5] = 2**32 - 13  # PM+32: max is 2^32 - 14
    assert pmp.pmp_keys_from_words(32, b.ctypes.data, a.ctypes.data) == 0
    a[5] = 7
    b[3] = 2**32  # b must be < 2^n
    assert pmp.pmp_keys_from_words(32, b.ctypes.data, a.ctypes.data) == 0
    k = pmp.Keys(h, 64)
    assert pmp.pmp_hash_batch(0, 0, 0, 1, 0, 0) == pmp.PMP_EINVAL
    assert pmp.pmp_hash_batch(k.handle, 0, 0, 0, 0, 0) == 0  # n == 0 is a no-op
    assert pmp.pmp_hash_batch(k.handle, 0, 0, 5, 0, 0) == pmp.PMP_EINVAL
    assert pmp.pmp_hash_long_partial(k.handle, 1, 1000, 512, 5000, 1, 0) == pmp.PMP_EINVAL  # misaligned
    assert pmp.strerror(pmp.PMP_ETOOLONG).startswith("string too long")
    assert pmp.lib().pmp_keys_bits(k.handle) == 64


def test_no_cpu_fallback_without_gpu(L):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    k = pmp.Keys.generate(1, 64)
    assert pmp.pmp_hash_batch(k.handle, 8, 8, 1, 8, 0) == pmp.PMP_ENODEV
    assert pmp.pmp_hash_long(k.handle, 8, 10, 8, 0) == pmp.PMP_ENODEV
    with pytest.raises(pmp.PmpError):
        pmp._check(pmp.pmp_hash_long(k.handle, 8, 10, 8, 0), "hash_long")


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("total,G", [(16 << 30, 8), (16 << 30, 3), (1 << 20, 4), (1000, 4), (0, 2), (123457, 5)])
def test_long_split_is_block_aligned_tiling(L, bits, total, G):
    cb = 1024 if bits == 64 else 512
    b = pmp.pmp_long_split(bits, total, G)
    assert b[0] == 0 and b[-1] == total and len(b) == G + 1
    assert all(b[i] <= b[i + 1] for i in range(G))
    assert all(x % cb == 0 for x in b[:-1])
    full = total // cb
    sizes = [(b[i + 1] - b[i]) // cb for i in range(G - 1)]
    assert all(abs(s - full / G) <= 1 for s in sizes)


@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("length", [0, 5, 100, 1024, 1025, 200_000, 128 * 128 * 1024 + 77, 16 << 30])
def test_long_constant_matches_oracle_tree_of_zero_blocks(L, oracle_lib, bits, length):
    """C(T) = Algorithm 1 run from level 2 on T_1 zero level-1 values
    (DESIGN.md 'affine split'); the oracle evaluates that tree literally."""
    keys = pmp.Keys.generate(40 + length % 97, bits)
    c2 = np.zeros(2, dtype=np.uint64)
    assert pmp.lib().pmp_long_constant(keys.handle, length, c2.ctypes.data) == 0
    got = int(c2[0]) | (int(c2[1]) << 64)
    ok = oracle_lib.keygen(40 + length % 97, bits)
    w = bits // 8
    T = length // w + 1
    T1 = -(-T // 128)
    if T1 <= 1:
        want = 0
    else:
        p = oracle_lib.params(bits)["p"]
        z = np.zeros(T1, dtype=np.uint64)
        want, _ = oracle_lib.tree_generic_np(p, 128, 8, ok.b, ok.a, z, z, j0=1)
    assert got == want


def test_bucket_call_rejects_zero_modulus(L):
    k = pmp.Keys.generate(1, 64)
    assert pmp.pmp_hash_batch_buckets(k.handle, 8, 8, 1, 0, 8, 0, 0) == pmp.PMP_EINVAL


def test_bucket_partition_argument_checks(L):
    """pmp_bucket_partition: M == 0, M > 2^24, NULL starts, NULL buckets/perm
    with n > 0 and n >= 2^32 are PMP_EINVAL before any device work."""
    E = pmp.PMP_EINVAL
    assert pmp.pmp_bucket_partition(8, 10, 0, 0, 8, 8) == E
    assert pmp.pmp_bucket_partition(8, 10, (1 << 24) + 1, 0, 8, 8) == E
    assert pmp.pmp_bucket_partition(8, 10, 16, 0, 0, 8) == E
    assert pmp.pmp_bucket_partition(0, 10, 16, 0, 8, 8) == E
    assert pmp.pmp_bucket_partition(8, 10, 16, 0, 8, 0) == E
    assert pmp.pmp_bucket_partition(8, 1 << 32, 16, 0, 8, 8) == E


@pytest.mark.parametrize("bits,size", [(64, 8264), (32, 4136)])
def test_keyfile_roundtrip_and_layout(L, bits, size):
    """KeyFile: exact size, header bytes, and the
    payload parsed here independently (b_j then a_{j,1..128}, LE n/8-byte
    words) equals the schedule; load(save(k)) exports the same words."""
    assert pmp.pmp_keyfile_size(bits) == size and pmp.pmp_keyfile_size(48) == 0
    k = pmp.Keys.generate(77, bits)
    raw = k.save()
    assert len(raw) == size
    assert raw[:4] == b"PMPH" and raw[4] == 1 and raw[5] == bits and raw[6] == 8 and raw[7] == 0
    words = np.frombuffer(raw[8:], dtype="<u8" if bits == 64 else "<u4").astype(np.uint64).reshape(8, 129)
    b, a = k.export()
    assert np.array_equal(words[:, 0], b) and np.array_equal(words[:, 1:], a)
    k2 = pmp.Keys.load(raw)
    assert k2.bits == bits
    b2, a2 = k2.export()
    assert np.array_equal(b2, b) and np.array_equal(a2, a)
    assert k2.save() == raw


@pytest.mark.parametrize("bits", [32, 64])
def test_keyfile_rejects_corrupt_files(L, bits):
    raw = bytearray(pmp.Keys.generate(78, bits).save())
    w = bits // 8
    amax = 2**64 - 12 if bits == 64 else 2**32 - 14

    def err(buf):
        with pytest.raises(pmp.PmpError) as e:
            pmp.Keys.load(bytes(buf))
        return e.value.code

    bad = bytearray(raw); bad[0:4] = b"PMPX"
    assert err(bad) == pmp.PMP_EBADFILE
    assert err(raw[:-1]) == pmp.PMP_EBADFILE            # truncated
    assert err(raw + b"\0") == pmp.PMP_EBADFILE         # trailing bytes
    assert err(raw[:3]) == pmp.PMP_EBADFILE
    for pos, val in ((4, 2), (5, 0x30), (5, 96 - bits), (6, 7), (7, 1)):
        bad = bytearray(raw); bad[pos] = val
        assert err(bad) == (pmp.PMP_EVERSION if not (pos == 5 and val == 96 - bits) else pmp.PMP_EBADFILE)
    for level, idx, val in ((0, 1, 0), (7, 128, 0), (3, 5, amax + 1), (5, 77, 2**bits - 1)):
        bad = bytearray(raw)
        o = 8 + (level * 129 + idx) * w
        bad[o:o + w] = val.to_bytes(w, "little")
        assert err(bad) == pmp.PMP_EKEYRANGE, (level, idx, val)
    ok = bytearray(raw)                                  # boundary values are legal
    for level, idx, val in ((2, 1, 1), (2, 2, amax), (4, 0, 2**bits - 1)):
        o = 8 + (level * 129 + idx) * w
        ok[o:o + w] = val.to_bytes(w, "little")
    pmp.Keys.load(bytes(ok))
    assert pmp.strerror(pmp.PMP_EKEYRANGE) == "key out of range"


def test_two_level_variant_arguments(L):
    """pmp_hash2_* validate like their tree counterparts and never fall back."""
    k = pmp.Keys.generate(3, 64)
    assert pmp.pmp_hash2_batch(0, 0, 0, 1, 0, 0) == pmp.PMP_EINVAL
    assert pmp.pmp_hash2_batch(k.handle, 0, 0, 0, 0, 0) == 0
    assert pmp.pmp_hash2_long(k.handle, 8, 10, 0, 0) == pmp.PMP_EINVAL              # out NULL
    assert pmp.pmp_hash2_long_partial(k.handle, 1, 1000, 512, 5000, 1, 0) == pmp.PMP_EINVAL  # misaligned
    assert pmp.pmp_hash2_long_partial(k.handle, 1, 1000, 1024, 5000, 1, 0) == pmp.PMP_EINVAL  # not whole blocks
    assert pmp.pmp_hash2_long_combine(k.handle, 8, 0, 8, 0) == pmp.PMP_EINVAL
    import torch

    if not torch.cuda.is_available():
        assert pmp.pmp_hash2_long(k.handle, 8, 10, 8, 0) == pmp.PMP_ENODEV
        assert pmp.pmp_hash2_batch(k.handle, 8, 8, 1, 8, 0) == pmp.PMP_ENODEV


def test_routing_hooks_set_and_query(L):
    """Batch-routing hooks are host state: each returns the previous value;
    pmp_set_huge_min(0) only queries (include/pmp.h)."""
    prev_min = pmp.pmp_set_huge_min(0)
    assert prev_min == 4 << 20                       # the documented default
    assert pmp.pmp_set_huge_min(1 << 20) == prev_min
    assert pmp.pmp_set_huge_min(0) == 1 << 20
    assert pmp.pmp_set_huge_min(prev_min) == 1 << 20
    prev_cap = pmp.pmp_set_huge_cap(7)
    assert prev_cap == 65536
    assert pmp.pmp_set_huge_cap(prev_cap) == 7
    prev_small = pmp.pmp_set_small_batch_max(100)
    assert prev_small == 4096
    assert pmp.pmp_set_small_batch_max(prev_small) == 100
