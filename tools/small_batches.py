"""Batches across length classes: small ones (n <= 4096 strings) through the
latency route (k_small) and the throughput route (k_short + k_wstring + k_huge,
forced with pmp_set_small_batch_max(0)); larger ones with a few huge strings
through the throughput route with and without k_huge (pmp_set_huge_cap(0):
every long string one warp) and with a lower huge threshold.  Every digest is
checked against the oracle.

python tools/small_batches.py   -- prints one line per (n, length) case:
device time per call (CUDA events over back-to-back calls) on each route.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1609_09840_b200 as pmp  # noqa: E402

CASES = [(1000, "U[1,64]"), (4096, "U[8,64]"), (4096, "4096"), (4096, "65536"), (1024, "262144"),
         (64, "1048576"), (8, "4194304"), (100_000, "U[8,64]+8x4M"), (100_000, "U[8,64]+2x64M"),
         (20_000, "U[1,1M]log")]


def lengths(n, spec, rng):
    if spec.endswith("log"):   # log-uniform like configs[4]
        return np.clip(np.floor(2.0 ** (20 * rng.random(n))), 1, 1 << 20).astype(np.uint64)
    if "+" in spec:            # short strings with a few huge ones at random places
        base, extra = spec.split("+")
        cnt, size = extra.split("x")
        lens = lengths(n, base, rng)
        lens[rng.choice(n, int(cnt), replace=False)] = int(size[:-1]) << 20
        return lens
    if spec.startswith("U["):
        lo, hi = (int(x) for x in spec[2:-1].split(","))
        return rng.integers(lo, hi + 1, size=n).astype(np.uint64)
    return np.full(n, int(spec), dtype=np.uint64)


def main():
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(3)
    key = pmp.Keys.generate(3, 64)
    okey = oracle.keygen(3, 64)
    default_max = pmp.pmp_set_small_batch_max(-1) if False else 4096
    for n, spec in CASES:
        lens = lengths(n, spec, rng)
        offs = datagen.offsets_from_lengths(lens)
        pay = datagen.payload_host(7, 0, int(offs[-1]))
        d_pay = torch.from_numpy(np.concatenate([pay, np.zeros(16, np.uint8)])).to(dev)
        d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
        want = oracle.hash_batch(okey, pay, offs, nthreads=os.cpu_count() or 4)
        row = []
        routes = [("small", default_max, 65536, 4 << 20), ("throughput", 0, 65536, 4 << 20)]
        if n > default_max:
            routes = [("throughput", 0, 65536, 4 << 20), ("no-huge", 0, 0, 4 << 20),
                      ("huge>=256K", 0, 65536, 256 << 10)]
        for route, smax, cap, hmin in routes:
            prev_cap = pmp.pmp_set_huge_cap(cap)
            prev_min = pmp.pmp_set_huge_min(hmin)
            pmp.pmp_set_small_batch_max(smax)
            out = torch.empty(n, dtype=torch.int64, device=dev)
            for _ in range(3):
                pmp.hash_batch(key, d_pay, d_off, out=out)
            torch.cuda.synchronize()
            got = pmp.as_u64(out)
            bad = int(np.count_nonzero(got != want.astype(got.dtype)))
            steps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                pmp.hash_batch(key, d_pay, d_off, out=out)
            e1.record()
            torch.cuda.synchronize()
            row.append(f"{route} {e0.elapsed_time(e1) / steps * 1e3:9.1f} us ({bad} mismatches)")
            pmp.pmp_set_huge_cap(prev_cap)
            pmp.pmp_set_huge_min(prev_min)
        print(f"n={n:6d} len {spec:>13s} ({int(offs[-1]) / 2**20:8.1f} MiB): " + "  ".join(row), flush=True)
    pmp.pmp_set_small_batch_max(default_max)


if __name__ == "__main__":
    main()
