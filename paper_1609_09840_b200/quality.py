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

Hashing runs in libpmp's kernels; the statistics are plain torch reductions on
the device (report code, not part of the hash path).
"""
from __future__ import annotations

import numpy as np

from . import Keys, hash_batch


def avalanche(keys: Keys, length: int, trials: int, seed: int = 1, chunk: int = 4096):
    """Returns (worst_bias, freq[8*length, n]) for single-bit input flips."""
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
        d = d.to(torch.int64) if keys.bits == 64 else d.to(torch.int64) & 0xFFFFFFFF
        x = d[:, 1:] ^ d[:, :1]                                           # t x nb
        counts += ((x.unsqueeze(-1) >> shifts) & 1).sum(dim=0)            # nb x nbits_out
        done += t
    freq = counts.double() / trials
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
