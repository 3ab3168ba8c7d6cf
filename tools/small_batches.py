"""Small batches (n <= 4096 strings, the k_small latency route) across length
classes, against the throughput route (k_short + k_wstring, forced with
pmp_set_small_batch_max(0)); also checks every digest against the oracle.

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
         (64, "1048576"), (8, "4194304")]


def lengths(n, spec, rng):
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
        for route, smax in (("small", default_max), ("throughput", 0)):
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
        print(f"n={n:5d} len {spec:>8s} ({int(offs[-1]) / 2**20:8.1f} MiB): " + "  ".join(row), flush=True)
    pmp.pmp_set_small_batch_max(default_max)


if __name__ == "__main__":
    main()
