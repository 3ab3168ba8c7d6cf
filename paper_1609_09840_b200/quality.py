"""GPU quality suite for PM+ (SURVEY 8(f2)), built on the batch kernel.

* ``avalanche``: "changing a single bit of the input should flip
  roughly half the bits of the output" (the mixer of P:722-734 is there for
  this).  For `trials` random inputs of `length` bytes and each of their
  8*length single-bit flips, the flip frequency of every output bit is measured;
  SPEC S:437 sets the pass threshold worst |freq - 1/2| < 0.03 at 1e5 trials.
* ``word_sweep``: component-wise regularity (lemma P:573-574) at
  production scale: fix every word of an 8-byte (PM+32) / 16-byte (PM+64)
  string but one and sweep that word over N values.  V is then injective, and
  only values V in [2^n, p) can alias after mod 2^n (the mixer is a bijection),
  so the digests have at most p - 2^n collisions (15 / 13); a random function
  would give about N^2 / 2^(n+1).

* ``collision_monte_carlo``: Table 3 bounds the probability, over
  the random key schedule, that two distinct strings collide; h mod M stays
  almost universal.  For a fixed pair, nsched schedules
  (pmp_keygen(seed0 + i), drawn on the device) count full-digest collisions
  (expected 0 at production scale, SPEC S:451-459 asserts rate <= 1e-4) and
  low-k-bit collisions (the bucket of a 2^k table, rate ~ 2^-k); the pair
  (s, s) is the control (rate 1).

Hashing runs in libpmp's kernels; the statistics are plain torch reductions on
the device (report code, not part of the hash path).
"""
from __future__ import annotations

import numpy as np

from . import Keys, _check, hash_batch, lib


def avalanche(keys: Keys, length: int, trials: int, seed: int = 1, chunk: int = 4096, first_batch: bool = False):
    """Returns (worst_bias, freq[8*length, n]) for single-bit input flips; with
    first_batch, also (payload, offsets, digests) of the first chunk's batch
    (host numpy arrays) so a test can recompute those digests with the oracle."""
    import torch

    import datagen

    dev = torch.device("cuda")
    nbits_in, nbits_out = 8 * length, keys.bits
    counts = torch.zeros(nbits_in, nbits_out, dtype=torch.int64, device=dev)
    flips = torch.zeros(nbits_in, length, dtype=torch.uint8, device=dev)
    ar = torch.arange(nbits_in, device=dev)
    flips[ar, ar // 8] = (1 << (ar % 8)).to(torch.uint8)
    shifts = torch.arange(nbits_out, device=dev, dtype=torch.int64)
    done = 0
    while done < trials:
        t = min(chunk, trials - done)
        base = torch.from_numpy(datagen.payload_host(seed, done * length, t * length)).to(dev).view(t, length)
        batch = torch.cat([base.unsqueeze(1), base.unsqueeze(1) ^ flips.unsqueeze(0)], dim=1)  # t x (1+nb) x L
        payload = batch.reshape(-1).contiguous()
        m = t * (nbits_in + 1)
        offsets = torch.arange(m + 1, device=dev, dtype=torch.int64) * length
        d = hash_batch(keys, payload, offsets).view(t, nbits_in + 1)
        if first_batch and done == 0:
            fb = (payload.cpu().numpy(), offsets.cpu().numpy().view(np.uint64),
                  d.reshape(-1).cpu().numpy().view(np.uint64 if keys.bits == 64 else np.uint32))
        d = d.to(torch.int64) if keys.bits == 64 else d.to(torch.int64) & 0xFFFFFFFF
        x = d[:, 1:] ^ d[:, :1]                                           # t x nb
        counts += ((x.unsqueeze(-1) >> shifts) & 1).sum(dim=0)            # nb x nbits_out
        done += t
    freq = counts.double() / trials
    if first_batch:
        return float((freq - 0.5).abs().max()), freq.cpu().numpy(), fb
    return float((freq - 0.5).abs().max()), freq.cpu().numpy()


def word_sweep(keys: Keys, N: int, seed: int = 3, word: int = 1, start: int = 0):
    """Digest collisions when word `word` of a 2-word string sweeps N values
    (the other word fixed to seeded random bytes)."""
    import torch

    import datagen

    dev = torch.device("cuda")
    w = keys.bits // 8
    fixed = torch.from_numpy(datagen.payload_host(seed, 0, 2 * w)).to(dev)
    vals = torch.arange(start, start + N, device=dev, dtype=torch.int64)
    payload = fixed.repeat(N, 1)
    for b in range(w):
        payload[:, word * w + b] = ((vals >> (8 * b)) & 0xFF).to(torch.uint8)
    offsets = torch.arange(N + 1, device=dev, dtype=torch.int64) * (2 * w)
    d = hash_batch(keys, payload.reshape(-1).contiguous(), offsets)
    uniq = torch.unique(d).numel()
    return N - uniq


def bound(bits: int) -> int:
    """p - 2^n: the most digests a single-word sweep can collide on."""
    return 15 if bits == 32 else 13


def collision_monte_carlo(bits: int, s1: bytes, s2: bytes, nsched: int, seed0: int = 1 << 32,
                          return_digests: bool = False, chunk: int = 1 << 24):
    """Collision counts of the fixed pair (s1, s2) over nsched key schedules
    (pmp_quality_collisions).  Returns {"full", "low16", "low12", "low8"} counts
    and rates (+ the digests of both strings if return_digests)."""
    import torch

    dev = torch.device("cuda")
    d1 = torch.tensor(list(s1) + [0] * 16, dtype=torch.uint8, device=dev)
    d2 = torch.tensor(list(s2) + [0] * 16, dtype=torch.uint8, device=dev)
    counts = torch.zeros(4, dtype=torch.int64, device=dev)
    g1 = torch.empty(nsched if return_digests else 0, dtype=torch.int64, device=dev)
    g2 = torch.empty_like(g1)
    st = int(torch.cuda.current_stream().cuda_stream)
    for c0 in range(0, nsched, chunk):
        m = min(chunk, nsched - c0)
        p1 = g1[c0:].data_ptr() if return_digests else 0
        p2 = g2[c0:].data_ptr() if return_digests else 0
        _check(lib().pmp_quality_collisions(bits, seed0 + c0, m, d1.data_ptr(), len(s1), d2.data_ptr(), len(s2),
                                            p1, p2, counts.data_ptr(), st), "pmp_quality_collisions")
    c = [int(x) for x in counts.cpu().tolist()]
    out = {"nsched": nsched, "full": c[0], "low16": c[1], "low12": c[2], "low8": c[3],
           "rate_full": c[0] / nsched, "rate_low16": c[1] / nsched, "rate_low12": c[2] / nsched,
           "rate_low8": c[3] / nsched}
    if return_digests:
        out["digests"] = (g1.cpu().numpy().view(np.uint64), g2.cpu().numpy().view(np.uint64))
    return out
