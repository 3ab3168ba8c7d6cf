"""Pins for the oracle's two-level variant (reading Q19 in
DESIGN.md): V = (b_2 + sum_c v_c r^(C-c)) mod p, v_c = f_1(chunk c) (Eq. (1),
P:543), r = a_{2,1}, digest = mix(V mod 2^n).  The oracle evaluates it by
Horner with a shift-and-add mulmod; these pins use other routes:

  overflow / truncation in mulmod          -> test_mulmod_*  (Python big ints)
  wrong exponent (off by one), ascending powers, dropped b_2, wrong r key
                                           -> test_hash2_closed_form (pow(r, C-c, p),
                                              sigma and f_1 rebuilt here from the bytes)
  not a polynomial of degree C in r        -> test_hash2_degree_in_r (finite differences)
  level 1 or final mod 2^n wrong           -> test_hash2_single_word_sweep_pm32 (regularity)
"""
import os
import random
from math import comb, factorial

import numpy as np
import pytest

NT = os.cpu_count() or 1


def _p(bits):
    return 2**bits + (13 if bits == 64 else 15)


def _sigma(bits, data):
    """bytes || 0x01 || zeros to a word boundary, little-endian words."""
    w = bits // 8
    raw = bytes(data) + b"\x01"
    raw += b"\0" * (-len(raw) % w)
    return [int.from_bytes(raw[i:i + w], "little") for i in range(0, len(raw), w)]


def _closed_form(keys, data):
    bits = keys.bits
    p = _p(bits)
    s = _sigma(bits, data)
    C = -(-len(s) // 128)
    s += [0] * (128 * C - len(s))
    a1 = [int(x) for x in keys.a[0]]
    b1 = int(keys.b[0])
    r, beta = int(keys.a[1][0]), int(keys.b[1])
    V = beta
    for c in range(C):
        v = (b1 + sum(a1[i] * s[128 * c + i] for i in range(128))) % p
        V += v * pow(r, C - c, p)
    return V % p, C


@pytest.mark.parametrize("bits", [32, 64])
def test_mulmod_edges_and_random(oracle_lib, bits):
    p = _p(bits)
    edge = [0, 1, 2, p - 1, p - 2, 2**bits - 1, 2**bits, 2**bits + 1, 2**(bits - 1), 12345]
    for x in edge:
        for y in edge:
            assert oracle_lib.mulmod(p, x, y) == x * y % p, (x, y)
    rng = random.Random(bits)
    for _ in range(2000):
        x, y = rng.randrange(p), rng.randrange(p)
        assert oracle_lib.mulmod(p, x, y) == x * y % p


LENGTHS = {64: [0, 1, 7, 8, 9, 1015, 1016, 1023, 1024, 1025, 3 * 1024 + 5, 130 * 1024 + 1],
           32: [0, 1, 3, 4, 5, 507, 508, 511, 512, 513, 5 * 512 + 2, 129 * 512]}


@pytest.mark.parametrize("bits", [32, 64])
def test_hash2_closed_form(oracle_lib, bits):
    """Horner in the oracle == b_2 + sum_c v_c r^(C-c) evaluated with pow() from
    a sigma and f_1 rebuilt here; chunk counts 1..131 incl. marker-only chunks."""
    keys = oracle_lib.keygen(600 + bits, bits)
    rng = np.random.default_rng(bits)
    for n in LENGTHS[bits]:
        data = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        want, C = _closed_form(keys, data)
        assert oracle_lib.hash2_value(keys, data) == want, n
        assert oracle_lib.hash2(keys, data) == oracle_lib.mix(bits, want & (2**bits - 1))
        assert oracle_lib.hash2_value(keys, data, nthreads=5) == want


@pytest.mark.parametrize("bits,n", [(64, 5), (64, 1500), (64, 2500), (32, 700)])
def test_hash2_degree_in_r(oracle_lib, bits, n):
    """V(r) - b_2 is a polynomial of degree C in r with leading coefficient v_0:
    its (C+1)-th finite difference vanishes and its C-th equals C! v_0 (mod p).
    r is varied by rewriting a_{2,1} in an explicit schedule."""
    base = oracle_lib.keygen(700 + n, bits)
    p = _p(bits)
    data = np.random.default_rng(n).integers(0, 256, size=n, dtype=np.uint8).tobytes()
    s = _sigma(bits, data)
    C = -(-len(s) // 128)
    s0 = s[:128] + [0] * max(0, 128 - len(s))
    v0 = (int(base.b[0]) + sum(int(base.a[0][i]) * s0[i] for i in range(128))) % p
    vals = []
    for k in range(C + 2):
        a = base.a.copy()
        a[1][0] = 1000 + k
        vals.append(oracle_lib.hash2_value(oracle_lib.Keys(bits, base.b, a), data))
    d_c1 = sum((-1) ** (C + 1 - k) * comb(C + 1, k) * vals[k] for k in range(C + 2)) % p
    d_c = sum((-1) ** (C - k) * comb(C, k) * vals[k] for k in range(C + 1)) % p
    assert d_c1 == 0
    assert d_c == factorial(C) * v0 % p


def test_hash2_single_word_sweep_pm32(oracle_lib):
    """Component-wise regularity of the variant ("good regularity in both
    levels"): for 8-byte strings V = b_2 + r (b_1 + a_{1,1} s_0 + a_{1,2} s_1 +
    a_{1,3}), injective in s_1, so sweeping s_1 over 2^20 values gives at most
    p - 2^32 = 15 digest collisions (a random function: ~128)."""
    keys = oracle_lib.keygen(23, 32)
    N = 1 << 20
    payload = np.zeros((N, 8), dtype=np.uint8)
    payload[:, :4] = np.random.default_rng(4).integers(0, 256, size=4, dtype=np.uint8)
    payload[:, 4:] = np.arange(N, dtype=np.uint32).view(np.uint8).reshape(N, 4)
    offsets = np.arange(N + 1, dtype=np.uint64) * 8
    d = oracle_lib.hash2_batch(keys, payload.reshape(-1), offsets, nthreads=NT)
    assert N - np.unique(d).size <= 15
    # batch == per-string
    for i in (0, 1, N - 1):
        assert d[i] == oracle_lib.hash2(keys, payload[i].tobytes())
