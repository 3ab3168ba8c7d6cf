"""Pins for the CPU oracle (oracle/pmp_oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.

Citations: P:n = PAPER.md line n, S:n = SPEC.md line n; goldens live in
tests/golden/ with their citations.  All tests here are CPU-only.

What each pin catches (a plausible oracle mistake -> the failing test):
  wrong prime / kappa / key range          -> test_table2_*, test_keygen_ranges
  wrong mixer constant or shift            -> test_mix_goldens (inputs with high bits set
                                              catch a wrong first shift)
  wrong generator / draw order in keygen   -> test_oracle_pins_bigint.py::test_*prng*, ::test_keygen_draw_order
  wrong absolute tree value (b_j terms)    -> test_oracle_pins_bigint.py::test_absolute_tree_value_*
  wrong byte order / marker / word count   -> test_sigma_words_*, test_short_strings_*
  dropped b, wrong key index in Eq. (1)    -> test_block_spec_examples, test_block_textbook_sum,
                                              test_affinity_*
  wrong level order (f_L at leaves), wrong padding, wrong termination
                                           -> test_fig1_shapes, test_affinity_*, test_levels_applied
  wrong final `mod 2^n`                    -> test_regularity_single_word_sweep_pm32
"""
import os
import random

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MASK64 = 2**64 - 1


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line


def _is_prime(n):
    if n < 2:
        return False
    for q in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41):
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


# ---------------------------------------------------------------- constants
@pytest.mark.parametrize("bits", [32, 64])
def test_table2_prime_is_smallest_above_power_of_two(oracle_lib, bits):
    """Table 1: p is the smallest prime larger than 2^n."""
    p = oracle_lib.params(bits)["p"]
    assert _is_prime(p)
    assert all(not _is_prime(2**bits + j) for j in range(1, p - 2**bits))


@pytest.mark.parametrize("bits", [32, 64])
def test_table2_kappa_is_minimal_for_two_word_products(oracle_lib, bits):
    """P:618-619 + Table 2: every product a*s with a <= p-kappa-1, s <= p-1 fits
    in 2n bits, and kappa is the least value with that property (reading Q7)."""
    pr = oracle_lib.params(bits)
    p, kappa = pr["p"], pr["kappa"]
    assert (p - kappa - 1) * (p - 1) < 2 ** (2 * bits)
    assert (p - (kappa - 1) - 1) * (p - 1) >= 2 ** (2 * bits)
    assert pr["a_max"] == p - kappa - 1
    assert pr["a_max"] < 2**bits  # a_i is a machine word


# ---------------------------------------------------------------- mixer
def test_mix_goldens(oracle_lib):
    n = 0
    for line in _lines("mix.txt"):
        bits, z, want = line.split()
        assert oracle_lib.mix(int(bits), int(z, 16)) == int(want, 16), line
        n += 1
    assert n == 11


@pytest.mark.parametrize("bits", [32, 64])
def test_mix_is_invertible(oracle_lib, bits):
    """the finalizer is a bijection on n-bit words."""
    rng = random.Random(7)
    mask = 2**bits - 1
    for _ in range(20000):
        z = rng.getrandbits(bits)
        assert oracle_lib.unmix(bits, oracle_lib.mix(bits, z)) == z
        assert oracle_lib.mix(bits, oracle_lib.unmix(bits, z)) == z
        assert oracle_lib.mix(bits, z) <= mask


# ---------------------------------------------------------------- Eq. (1)
def test_block_spec_examples(oracle_lib):
    n = 0
    for line in _lines("spec_arith.txt"):
        parts = line.split()
        if parts[0] == "block":
            p, m, b = int(parts[1]), int(parts[2]), int(parts[3])
            a = [int(x) for x in parts[4].split(",")]
            s = [int(x) for x in parts[5].split(",")]
            assert oracle_lib.block(p, m, b, a, s) == int(parts[6]), line
            n += 1
        elif parts[0] == "modp":
            bits, value, want = int(parts[1]), int(parts[2]), int(parts[3])
            p = oracle_lib.params(bits)["p"]
            assert oracle_lib.block(p, 1, 0, [1], [value]) == want, line
            n += 1
    assert n == 5


@pytest.mark.parametrize("bits", [32, 64])
def test_block_zero_input_gives_offset_and_identity_coefficient(oracle_lib, bits):
    """S:149 all s_i = 0 -> b; S:160 a single s_i = p-1 with a_i = 1, b = 0 -> p-1."""
    p = oracle_lib.params(bits)["p"]
    rng = random.Random(bits)
    a = [rng.randrange(1, 2**bits - 20) for _ in range(128)]
    b = rng.getrandbits(bits)
    assert oracle_lib.block(p, 128, b, a, [0] * 128) == b
    a2 = list(a)
    a2[37] = 1
    x = [0] * 128
    x[37] = p - 1
    assert oracle_lib.block(p, 128, 0, a2, x) == p - 1


@pytest.mark.parametrize("bits", [32, 64])
def test_block_textbook_sum(oracle_lib, bits):
    """With all keys 1 and b = 0, Eq. (1) is the plain sum of the inputs mod p
    (a special case that reduces to integer addition)."""
    p = oracle_lib.params(bits)["p"]
    x = [2**bits - 1 - i for i in range(128)]
    assert oracle_lib.block(p, 128, 0, [1] * 128, x) == sum(x) % p
    # maximal operands (S:73 setting): 128 maximal products plus b
    amax = oracle_lib.params(bits)["a_max"]
    got = oracle_lib.block(p, 128, 2**bits - 1, [amax] * 128, [p - 1] * 128)
    # (b + 128 * amax * (p-1)) mod p == (b - 128*amax) mod p since p-1 == -1
    assert got == (2**bits - 1 - 128 * amax) % p


# ---------------------------------------------------------------- packing
def test_sigma_words_marker_and_order(oracle_lib):
    """P:456 'pad with a 1-byte and zeros to the nearest machine word boundary';
    little-endian words (reading Q3); a whole word 1 when len % w == 0 (Q4)."""
    sw = oracle_lib.sigma_word
    assert oracle_lib.num_words(64, 0) == 1 and sw(64, b"", 0) == 1
    assert sw(64, b"a", 0) == 0x0161
    assert sw(64, b"abcdefgh", 0) == int.from_bytes(b"abcdefgh", "little")
    assert oracle_lib.num_words(64, 8) == 2 and sw(64, b"abcdefgh", 1) == 1
    assert sw(64, b"abcdefghi", 1) == 0x0169
    assert oracle_lib.num_words(32, 7) == 2 and sw(32, b"abcdefg", 1) == 0x01676665
    assert sw(32, b"abcd", 1) == 1 and oracle_lib.num_words(32, 4) == 2
    assert oracle_lib.num_words(32, 3) == 1 and sw(32, b"abc", 0) == 0x01636261


def test_sigma_distinguishes_trailing_zero_bytes(oracle_lib):
    """S:257 prefix distinction: s, s||0x00, s||0x00 0x00 give different sigma."""
    for bits in (32, 64):
        seen = set()
        for extra in range(0, 17):
            s = b"\x07" + b"\x00" * extra
            T = oracle_lib.num_words(bits, len(s))
            seen.add(tuple(oracle_lib.sigma_word(bits, s, t) for t in range(T)))
        assert len(seen) == 17


@pytest.mark.parametrize("bits", [32, 64])
def test_short_strings_are_key_independent(oracle_lib, bits):
    """|sigma| == 1 (len < w): Algorithm 1's loop never runs, so the digest
    is mix(sigma_0) for every key schedule (reading Q2; S:236 for the empty input)."""
    k1, k2 = oracle_lib.keygen(11, bits), oracle_lib.keygen(12, bits)
    w = bits // 8
    for length in range(w):
        s = bytes(range(0x41, 0x41 + length))
        want = oracle_lib.mix(bits, int.from_bytes(s + b"\x01", "little"))
        assert oracle_lib.hash_bytes(k1, s) == want
        assert oracle_lib.hash_bytes(k2, s) == want
    golden = {64: 0xC4CEB9FE78E2B0AC, 32: 0xAB3B4E74}[bits]
    assert oracle_lib.hash_bytes(k1, b"") == golden


# ---------------------------------------------------------------- Algorithm 1
def test_fig1_shapes(oracle_lib):
    """Figure 1 with m = 4 over the toy field p = 257 (Table 1):
    'ab' -> f1(a,b,1,0) and 'abcde' -> f2(f1(a,b,c,d), f1(e,1,0,0), 0, 0).
    The tree is the oracle's literal Algorithm 1; the shapes are composed
    here from single blocks (Eq. (1), pinned above)."""
    p, m, Lv = 257, 4, 3
    rng = random.Random(1)
    b = [rng.randrange(0, 256) for _ in range(Lv)]
    a = [rng.randrange(1, 255) for _ in range(Lv * m)]

    def f(j, xs):  # f_j, 1-based level
        return oracle_lib.block(p, m, b[j - 1], a[(j - 1) * m:j * m], xs)

    shapes = dict((ln.split()[0], ln.split()[1]) for ln in _lines("fig1.txt"))
    chars = {c: rng.randrange(0, 256) for c in "abcde"}
    s_ab = [chars[c] for c in shapes["ab"]] + [1]
    got, lv = oracle_lib.tree_generic(p, m, Lv, b, a, s_ab)
    assert lv == 1 and got == f(1, [chars["a"], chars["b"], 1, 0])
    s5 = [chars[c] for c in shapes["abcde"]] + [1]
    got, lv = oracle_lib.tree_generic(p, m, Lv, b, a, s5)
    want = f(2, [f(1, [chars[c] for c in "abcd"]), f(1, [chars["e"], 1, 0, 0]), 0, 0])
    assert lv == 2 and got == want


def test_levels_applied_and_length_limit(oracle_lib):
    """Alg. 1 input bound N <= m^L - 1, i.e. |sigma| <= m^L."""
    p, m, Lv = 17, 2, 3
    b, a = [1, 2, 3], [1, 2, 3, 4, 5, 6]
    for T, levels in [(1, 0), (2, 1), (3, 2), (4, 2), (5, 3), (8, 3)]:
        _, lv = oracle_lib.tree_generic(p, m, Lv, b, a, [1] * T)
        assert lv == levels, T
    _, lv = oracle_lib.tree_generic(p, m, Lv, b, a, [1] * 9)
    assert lv == -1


def _path_key(keys, t, levels):
    """K(t) = prod_{j=1..levels} a_{j, digit_{j}(t)}, digit_j(t) = floor(t/128^(j-1)) mod 128:
    the coefficient of sigma_t obtained by unrolling the affine levels of
    Algorithm 1.  Not a formula the oracle contains."""
    p = keys_p(keys)
    k = 1
    for j in range(levels):
        k = k * int(keys.a[j, (t // 128**j) % 128]) % p
    return k


def keys_p(keys):
    return 2**keys.bits + (13 if keys.bits == 64 else 15)


@pytest.mark.parametrize("bits,length", [(64, 9), (64, 1016), (64, 1023), (64, 1024), (64, 3000),
                                         (32, 13), (32, 511), (32, 512), (32, 1500)])
def test_affinity_in_each_word(oracle_lib, bits, length):
    """BASELINE north_star invariant: changing word t by d shifts the pre-finalizer
    value by K(t)*d mod p, with K(t) the product of the path keys."""
    keys = oracle_lib.keygen(99 + length, bits)
    rng = random.Random(length * bits)
    w = bits // 8
    data = bytearray(rng.getrandbits(8) for _ in range(length))
    T = oracle_lib.num_words(bits, length)
    levels = 0
    n = T
    while n > 1:
        n = (n + 127) // 128
        levels += 1
    V, lv = oracle_lib.tree_value(keys, bytes(data))
    assert lv == levels
    p = keys_p(keys)
    full_words = length // w
    for t in sorted({0, 1, full_words // 2, full_words - 1} & set(range(full_words))):
        old = int.from_bytes(data[t * w:(t + 1) * w], "little")
        new = rng.getrandbits(bits)
        mod = bytearray(data)
        mod[t * w:(t + 1) * w] = new.to_bytes(w, "little")
        V2, _ = oracle_lib.tree_value(keys, bytes(mod))
        assert (V2 - V) % p == _path_key(keys, t, levels) * (new - old) % p, t


@pytest.mark.parametrize("bits,T", [(64, 2), (64, 129), (64, 16386), (32, 257)])
def test_closed_form_against_literal_tree(oracle_lib, bits, T):
    """V(s) - V(0^len) = sum_t K(t) (sigma_t(s) - sigma_t(0^len)) mod p for every
    s of a given length (the unrolled tree)."""
    keys = oracle_lib.keygen(5 * T + bits, bits)
    w = bits // 8
    length = (T - 1) * w + (3 if T % 2 else 0)
    rng = np.random.default_rng(T)
    data = rng.integers(0, 256, size=length, dtype=np.uint8).tobytes()
    V, lv = oracle_lib.tree_value(keys, data)
    V0, _ = oracle_lib.tree_value(keys, bytes(length))
    p = keys_p(keys)
    acc = 0
    for t in range(T):
        d = oracle_lib.sigma_word(bits, data, t) - oracle_lib.sigma_word(bits, bytes(length), t)
        if d:
            acc += _path_key(keys, t, lv) * d
    assert (V - V0) % p == acc % p
    assert 0 <= V < p


def test_tree_value_multithreaded_is_same(oracle_lib):
    keys = oracle_lib.keygen(3, 64)
    data = np.random.default_rng(0).integers(0, 256, size=300_000, dtype=np.uint8).tobytes()
    assert oracle_lib.tree_value(keys, data, 1) == oracle_lib.tree_value(keys, data, 7)


# ---------------------------------------------------------------- properties
def test_component_wise_regularity_toy_exhaustive(oracle_lib):
    """Lemma P:574 'component-wise regular': over p = 257, m = 4, sweeping
    one component over [0,p) is a permutation; after mod 256 every output has
    1 or 2 preimages (lemma regularismarvellous)."""
    p, m = 257, 4
    rng = random.Random(5)
    for trial in range(20):
        b = rng.randrange(0, 256)
        a = [rng.randrange(1, 255) for _ in range(m)]
        i = rng.randrange(m)
        fixed = [rng.randrange(0, p) for _ in range(m)]
        outs = []
        for v in range(p):
            x = list(fixed)
            x[i] = v
            outs.append(oracle_lib.block(p, m, b, a, x))
        assert sorted(outs) == list(range(p))
        counts = np.bincount(np.array(outs) % 256, minlength=256)
        assert counts.min() >= 1 and counts.max() <= 2 and counts.sum() == 257


def test_delta_universality_toy_exhaustive(oracle_lib):
    """P[f(s) - f(s') = c mod p] <= 1/(p-1-kappa) over random keys
    (p = 17, kappa = 2, m = 2, all (a1, a2, b) enumerated)."""
    p, kappa, m = 17, 2, 2
    rng = random.Random(9)
    for _ in range(6):
        s = [rng.randrange(p) for _ in range(m)]
        s2 = list(s)
        while s2 == s:
            s2 = [rng.randrange(p) for _ in range(m)]
        c = rng.randrange(p)
        hits = total = 0
        for a1 in range(1, p - kappa):
            for a2 in range(1, p - kappa):
                for b in range(16):
                    d = oracle_lib.block(p, m, b, [a1, a2], s) - oracle_lib.block(p, m, b, [a1, a2], s2)
                    hits += (d % p) == c
                    total += 1
        assert hits * (p - 1 - kappa) <= total


def test_regularity_single_word_sweep_pm32(oracle_lib):
    """Component-wise regularity at production scale: fixing all words but one and
    sweeping it over N values, V is injective, so digest collisions are bounded
    by the values V in [0, p - 2^n) that alias mod 2^32: at most k = 15
    (SURVEY.md 8(c.3)).  A random function would give ~N^2/2^33 = 128."""
    keys = oracle_lib.keygen(21, 32)
    N = 1 << 20
    rng = np.random.default_rng(3)
    prefix = rng.integers(0, 256, size=4, dtype=np.uint8)
    payload = np.zeros((N, 8), dtype=np.uint8)
    payload[:, :4] = prefix
    payload[:, 4:] = np.arange(N, dtype=np.uint32).view(np.uint8).reshape(N, 4)
    offsets = np.arange(N + 1, dtype=np.uint64) * 8
    d = oracle_lib.hash_batch(keys, payload.reshape(-1), offsets, nthreads=os.cpu_count() or 1)
    collisions = N - np.unique(d).size
    assert collisions <= 15


@pytest.mark.parametrize("bits", [32, 64])
def test_keygen_ranges_and_determinism(oracle_lib, bits):
    """Key ranges of Eq. (1): b in [0, 2^n), a in [1, p-kappa-1];
    same seed -> same schedule."""
    k = oracle_lib.keygen(123, bits)
    k2 = oracle_lib.keygen(123, bits)
    k3 = oracle_lib.keygen(124, bits)
    amax = oracle_lib.params(bits)["a_max"]
    assert np.array_equal(k.a, k2.a) and np.array_equal(k.b, k2.b)
    assert not np.array_equal(k.a, k3.a)
    a = k.a.astype(object)
    assert (a >= 1).all() and (a <= amax).all()
    assert all(int(x) < 2**bits for x in k.b)
    # uniformity sanity: mean of 1024 keys within 5 sigma of the midpoint
    mean = float(np.mean(k.a.astype(np.float64)))
    sd = amax / np.sqrt(12) / np.sqrt(k.a.size)
    assert abs(mean - amax / 2) < 5 * sd
