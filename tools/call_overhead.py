"""Per-call cost of pmp_hash_batch_multi against its k_short time, for shrinking
batches of configs[1]'s shape (what one rank of an N-GPU strong-scaling run
hashes): python tools/call_overhead.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1609_09840_b200 as pmp  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    wl = datagen.WORKLOADS["hashtable"]
    lens = wl.lengths()
    k64, k32 = pmp.Keys.generate(2, 64), pmp.Keys.generate(2, 32)
    for shift in (0, 1, 2, 3, 4, 6):
        n = len(lens) >> shift
        offs = datagen.offsets_from_lengths(lens[:n])
        buf = torch.empty(int(offs[-1]) + 16, dtype=torch.uint8, device=dev)
        datagen.fill_device(wl.seed, buf.data_ptr(), int(offs[-1]), torch.cuda.current_stream().cuda_stream)
        d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
        o64 = torch.empty(n, dtype=torch.int64, device=dev)
        o32 = torch.empty(n, dtype=torch.int32, device=dev)
        for _ in range(5):
            pmp.hash_batch_multi([k64, k32], buf, d_off, outs=[o64, o32])
        torch.cuda.synchronize()
        steps = 50
        pmp.pmp_prof_reset()
        pmp.pmp_prof_enable(True)
        for _ in range(5):
            pmp.hash_batch_multi([k64, k32], buf, d_off, outs=[o64, o32])
        torch.cuda.synchronize()
        ks_ms, ks_n = pmp.pmp_prof_read("k_short")
        kw_ms, kw_n = pmp.pmp_prof_read("k_wstring")
        pmp.pmp_prof_enable(False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            pmp.hash_batch_multi([k64, k32], buf, d_off, outs=[o64, o32])
        e1.record()
        torch.cuda.synchronize()
        step = e0.elapsed_time(e1) / steps
        print(f"n={n:9d} step {step * 1e3:8.1f} us  k_short {ks_ms / max(ks_n, 1) * 1e3:8.1f} us  "
              f"k_wstring {kw_ms / max(kw_n, 1) * 1e3:6.1f} us  other {step * 1e3 - ks_ms / max(ks_n, 1) * 1e3:6.1f} us",
              flush=True)
        del buf, d_off, o64, o32
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
