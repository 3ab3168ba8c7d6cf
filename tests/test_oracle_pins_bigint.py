"""Pins for the oracle's absolute values and its random inputs.

1. Absolute tree values.  An independent Python big-integer evaluation of the
   paper's definitions -- the literal Algorithm 1 (Section 4) and,
   separately, its unrolled closed form -- is compared
   with the oracle's V = Tree(sigma) *absolutely* (not as differences, so every
   b_j term counts), at T in {1, 2, 127-130, 255-257, 128^2-1 .. 128^2+2} and
   both widths, with schedule keys and with extreme keys.
   Neither Python evaluation shares code with oracle/pmp_oracle.c: byte packing
   (P:456), the level loop, the zero padding and the key indexing are written
   here from the paper.

2. The generators behind the key schedule (reading Q12) and the input streams
   (datagen/pmp_datagen.h) against their published reference outputs
   (tests/golden/prng.txt), and the keygen draw order composed from those
   pinned generators.

CPU only.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import os
import random

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
M = 128
MASK64 = 2**64 - 1


# ------------------------------------------------------------ independent big-int side
def _p(bits):
    """Table 2: p = 2^64 + 13, 2^32 + 15 (smallest primes above 2^n, Table 1)."""
    return 2**bits + (13 if bits == 64 else 15)


def _sigma(data: bytes, bits: int):
    """append a 1-byte, pad with zeros to the word boundary; little-endian
    n-bit words (readings Q3/Q4)."""
    w = bits // 8
    s = bytes(data) + b"\x01"
    s += b"\x00" * (-len(s) % w)
    return [int.from_bytes(s[i:i + w], "little") for i in range(0, len(s), w)]


def _alg1_literal(sigma, b, a, p, m=M):
    """Algorithm 1 with Python integers: while |sigma| > 1, append
    zeros to a multiple of m and replace sigma by the values f_j of its blocks,
    f_j(x) = (b_j + sum_r a_{j,r} x_r) mod p (Eq. (1)); j from 1 upward
    (f_1 at the leaves, reading Q1).  Returns (V, levels)."""
    x = list(sigma)
    j = 0
    while len(x) > 1:
        x = x + [0] * (-len(x) % m)
        x = [(b[j] + sum(a[j][r] * x[q * m + r] for r in range(m))) % p for q in range(len(x) // m)]
        j += 1
    return x[0], j


def _closed_form(sigma, b, a, p, m=M):
    """The unrolled tree: with level sizes T_0 = T,
    T_j = ceil(T_{j-1} / m) down to 1 (L levels), and the weight of node q of
    level j
        W_j(q) = prod_{i=1}^{L-j} a_{j+i, digit_{i-1}(q)},  digit_i(q) = floor(q / m^i) mod m,
    the tree value is
        V = sum_t W_0(t) sigma_t + sum_{j=1}^{L} b_j sum_{q < T_j} W_j(q)  (mod p).
    A formula that never forms a block value; every b_j enters absolutely."""
    sizes = [len(sigma)]
    while sizes[-1] > 1:
        sizes.append(-(-sizes[-1] // m))
    L = len(sizes) - 1

    def W(j, q):
        w = 1
        for i in range(1, L - j + 1):
            w = w * a[j + i - 1][(q // m ** (i - 1)) % m] % p
        return w

    V = sum(W(0, t) * s for t, s in enumerate(sigma))
    for j in range(1, L + 1):
        V += b[j - 1] * sum(W(j, q) for q in range(sizes[j]))
    return V % p, L


class _K:
    """A key schedule in the oracle binding's layout (b[8], a[8][128])."""

    def __init__(self, bits, b, a):
        self.bits = bits
        self.b = np.array(b, dtype=np.uint64)
        self.a = np.array(a, dtype=np.uint64).reshape(8, M)


def _schedules(oracle_lib, bits, seed):
    k = oracle_lib.keygen(seed, bits)
    yield "keygen", k
    amax = oracle_lib.params(bits)["a_max"]
    # extreme keys: every a at its maximum, b = 2^n - 1 (maximal operands)
    yield "max", _K(bits, [2**bits - 1] * 8, [[amax] * M] * 8)
    # small keys: a in {1, 2}, b in {0, 1} (near-identity coefficients)
    rng = random.Random(seed)
    yield "small", _K(bits, [rng.randrange(2) for _ in range(8)], [[rng.randrange(1, 3) for _ in range(M)] for _ in range(8)])


_TS = [1, 2, 127, 128, 129, 130, 255, 256, 257, 128 * 128 - 1, 128 * 128, 128 * 128 + 1, 128 * 128 + 2]


@pytest.mark.parametrize("bits", [64, 32])
@pytest.mark.parametrize("T", _TS)
def test_absolute_tree_value_against_bigint_alg1_and_closed_form(oracle_lib, bits, T):
    w = bits // 8
    rng = np.random.default_rng(T * 131 + bits)
    r = int(rng.integers(0, w))                       # bytes in the last (marker) word
    length = (T - 1) * w + r                          # T = floor(len / w) + 1
    data = rng.integers(0, 256, size=length, dtype=np.uint8).tobytes()
    sigma = _sigma(data, bits)
    assert len(sigma) == T
    p = _p(bits)
    for name, keys in _schedules(oracle_lib, bits, T + bits):
        b = [int(x) for x in keys.b]
        a = [[int(x) for x in row] for row in keys.a]
        want, lv = _alg1_literal(sigma, b, a, p)
        V, olv = oracle_lib.tree_value(keys, data)
        assert V == want, (name, T)
        assert olv == lv, (name, T)
        if T <= 257 or name == "keygen":                # closed form: O(T L), every T once
            cf, L = _closed_form(sigma, b, a, p)
            assert cf == want and L == lv, (name, T)
        # the digest is the mixer of V mod 2^n (mixer pinned in tests/golden/mix.txt)
        assert oracle_lib.hash_bytes(keys, data) == oracle_lib.mix(bits, V & (2**bits - 1))


def test_closed_form_reduces_to_textbook_cases():
    """Sanity of the test-side closed form itself on cases with a known answer:
    one block with all keys 1 is b_1 + plain sum (Eq. (1)); T = 1 is sigma_0."""
    p = _p(64)
    b = [5, 7, 0, 0, 0, 0, 0, 0]
    a = [[1] * M for _ in range(8)]
    sig = list(range(1, 11))
    assert _closed_form(sig, b, a, p)[0] == (5 + sum(sig)) % p == _alg1_literal(sig, b, a, p)[0]
    assert _closed_form([42], b, a, p) == (42, 0) == _alg1_literal([42], b, a, p)
    # two levels, all keys 1: b_2 + (b_1 * nblocks) + sum
    sig = list(range(300))
    assert _closed_form(sig, b, a, p)[0] == (7 + 5 * 3 + sum(sig)) % p


# ------------------------------------------------------------ generators
def _prng_golden():
    g = {"splitmix64": [], "xoshiro256ss": []}
    with open(os.path.join(GOLDEN, "prng.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                name, idx, val = line.split()
                assert int(idx) == len(g[name])
                g[name].append(int(val))
    return g


def test_oracle_prng_matches_published_outputs(oracle_lib):
    g = _prng_golden()
    assert oracle_lib.splitmix64_stream(0, 4) == g["splitmix64"]
    assert oracle_lib.xoshiro256ss_stream([1, 2, 3, 4], 10) == g["xoshiro256ss"]


def test_datagen_prng_matches_published_outputs():
    import datagen

    g = _prng_golden()
    assert datagen.splitmix64_stream(0, 4) == g["splitmix64"]
    assert datagen.xoshiro256ss_stream([1, 2, 3, 4], 10) == g["xoshiro256ss"]


@pytest.mark.parametrize("bits", [64, 32])
@pytest.mark.parametrize("seed", [0, 2, 0xDEADBEEF])
def test_keygen_draw_order(oracle_lib, bits, seed):
    """Reading Q12: xoshiro256** seeded with 4 successive splitmix64 outputs of
    the seed; for j = 1..8: b_j = x (x >> 32 for 32-bit), then a_{j,1..128} by
    rejection to [1, p - kappa - 1].  Composed here from the two generators
    (pinned above), so a wrong draw order or rejection bound fails."""
    state = oracle_lib.splitmix64_stream(seed, 4)
    draws = iter(oracle_lib.xoshiro256ss_stream(state, 8 * 200))
    amax = oracle_lib.params(bits)["a_max"]
    shift = 0 if bits == 64 else 32
    b, a = [], []
    for _ in range(8):
        b.append(next(draws) >> shift)
        row = []
        while len(row) < M:
            x = next(draws) >> shift
            if 1 <= x <= amax:
                row.append(x)
        a.append(row)
    k = oracle_lib.keygen(seed, bits)
    assert [int(x) for x in k.b] == b
    assert [[int(x) for x in r] for r in k.a] == a


def test_datagen_stream_contract(oracle_lib):
    """pmp_datagen.h: stream(seed, id) = xoshiro256** seeded with 4 splitmix64
    outputs of seed ^ (id * 0x9E3779B97F4A7C15); payload page q = LE bytes of
    stream(seed, 2 + q); lengths U[lo, hi] = lo + ((x >> 32) (hi - lo + 1)) >> 32
    from stream(seed, 1).  Composed from the pinned generators."""
    import datagen

    for seed, sid in [(2, 1), (5, 2), (3, 1000)]:
        st = datagen.splitmix64_stream(seed ^ ((sid * 0x9E3779B97F4A7C15) & MASK64), 4)
        assert datagen.stream(seed, sid, 6) == datagen.xoshiro256ss_stream(st, 6)
    page = datagen.payload_host(7, 3 * 4096 + 8, 24)
    want = b"".join(x.to_bytes(8, "little") for x in datagen.stream(7, 2 + 3, 4))[8:32]
    assert page.tobytes() == want
    lens = datagen.lengths(datagen.LEN_UNIFORM, 2, 5, 8, 64)
    xs = datagen.stream(2, 1, 5)
    assert [int(v) for v in lens] == [8 + (((x >> 32) * 57) >> 32) for x in xs]


@pytest.mark.parametrize("bits", [64, 32])
def test_batch_and_long_entry_points_against_bigint(oracle_lib, bits):
    """pmpo_hash_batch (reading Q13 CSR layout, threaded over strings) and
    pmpo_hash_long (threaded level-1 map) against the big-int Algorithm 1
    followed by the golden-pinned mixer."""
    rng = np.random.default_rng(bits)
    lens = [0, 1, 3, 4, 7, 8, 9, 63, 64, 127, 128, 1023, 1024, 1025, 2047, 4100] + \
        [int(x) for x in rng.integers(0, 300, size=40)]
    offs = np.zeros(len(lens) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum(lens)
    payload = rng.integers(0, 256, size=int(offs[-1]), dtype=np.uint8)
    keys = oracle_lib.keygen(77, bits)
    b = [int(x) for x in keys.b]
    a = [[int(x) for x in row] for row in keys.a]
    p, mask = _p(bits), 2**bits - 1
    got = oracle_lib.hash_batch(keys, payload, offs, nthreads=3)
    for i, ln in enumerate(lens):
        s = payload[int(offs[i]):int(offs[i + 1])].tobytes()
        V, _ = _alg1_literal(_sigma(s, bits), b, a, p)
        assert int(got[i]) == oracle_lib.mix(bits, V & mask), (i, ln)
    w = bits // 8
    data = rng.integers(0, 256, size=(128 * 128 + 1) * w + 3, dtype=np.uint8).tobytes()
    V, _ = _alg1_literal(_sigma(data, bits), b, a, p)
    assert oracle_lib.hash_long(keys, data, nthreads=5) == oracle_lib.mix(bits, V & mask)
