#!/usr/bin/env python
"""Full-size GPU quality report: avalanche at 1e5 trials for
SPEC's lengths {4, 8, 16, 32, 64} bytes, the complete 2^32-value
single-word sweep for PM+32 (component-wise regularity at production scale),
and the collision Monte Carlo over 10^7 key schedules (Table 3).
Writes one JSON object to stdout."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1609_09840_b200 as pmp
    from paper_1609_09840_b200 import quality

    torch.cuda.set_device(0)
    out = {"avalanche": [], "sweep": []}
    trials = int(os.environ.get("PMP_AVAL_TRIALS", "100000"))
    for bits in (32, 64):
        keys = pmp.Keys.generate(2024, bits)
        for length in (4, 8, 16, 32, 64):
            t0 = time.time()
            worst, _ = quality.avalanche(keys, length, trials, seed=9)
            out["avalanche"].append({"bits": bits, "length": length, "trials": trials, "worst_bias": worst,
                                     "pass_lt_0.03": worst < 0.03, "seconds": time.time() - t0})
    # full sweep of one 32-bit word: 2^32 digests (uint32), counted distinct on the device
    keys = pmp.Keys.generate(2025, 32)
    N = 1 << 32
    step = 1 << 28
    digests = torch.empty(N, dtype=torch.int32, device="cuda")
    t0 = time.time()
    import datagen

    w = 4
    fixed = torch.from_numpy(datagen.payload_host(11, 0, 2 * w)).cuda()
    for s in range(0, N, step):
        vals = torch.arange(s, s + step, device="cuda", dtype=torch.int64)
        payload = fixed.repeat(step, 1)
        for b in range(w):
            payload[:, w + b] = ((vals >> (8 * b)) & 0xFF).to(torch.uint8)
        offsets = torch.arange(step + 1, device="cuda", dtype=torch.int64) * (2 * w)
        pmp.hash_batch(keys, payload.reshape(-1).contiguous(), offsets, out=digests[s:s + step])
        del payload, vals, offsets
    torch.cuda.synchronize()
    hashed = time.time() - t0
    # count equal digests per top-4-bit slice (torch sorts at most INT_MAX elements)
    collisions = 0
    top = (digests.to(torch.int64) & 0xFFFFFFFF) >> 28
    for k in range(16):
        part = digests[top == k]
        srt, _ = torch.sort(part)
        collisions += int((srt[1:] == srt[:-1]).sum().item())
        del part, srt
    out["sweep"].append({"bits": 32, "N": N, "collisions": collisions, "bound_p_minus_2n": 15,
                         "random_function_expectation": N * (N - 1) / 2 / 2**32,
                         "hash_seconds": hashed, "seconds": time.time() - t0})
    # collision Monte Carlo (Table 3): fixed pairs, 10^7 device-drawn schedules
    out["collision_monte_carlo"] = []
    nsched = int(os.environ.get("PMP_MC_SCHEDULES", "10000000"))
    import numpy as np

    rng = np.random.default_rng(7)
    a = bytes(rng.integers(0, 256, 64, dtype=np.uint8))
    b = bytearray(a)
    b[0] ^= 1
    pairs = {"one bit apart (64 B)": (a, bytes(b)), "shifted (16 B)": (a[:16], a[1:17]),
             "different lengths (63 / 64 B)": (a[:63], a), "control (s, s)": (a, a)}
    for bits in (32, 64):
        for name, (s1, s2) in pairs.items():
            t0 = time.time()
            r = quality.collision_monte_carlo(bits, s1, s2, nsched)
            r.update({"bits": bits, "pair": name, "seconds": time.time() - t0,
                      "table3_eps": (12 / (2**63 - 6)) if bits == 64 else (12 / (2**31 - 7))})
            out["collision_monte_carlo"].append(r)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
