"""Quick GPU check of k_short_tc against the oracle and k_short (bring-up tool).

python tools/tc_check.py [n]  -- n strings of U[0, 130] bytes (every length class
of the short path: |sigma| = 1, tensor-core rows, the 65..127-byte word loop,
work-list strings), both widths fused and each width alone; then configs[1]
(2^24 strings of 8..64 B, both widths) compared with the word-loop kernel.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1609_09840_b200 as pmp  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
    dev = torch.device("cuda:0")
    pmp.pmp_set_small_batch_max(0)
    rng = np.random.default_rng(7)
    lens = rng.integers(0, 131, size=n).astype(np.uint64)
    offs = datagen.offsets_from_lengths(lens)
    pay = datagen.payload_host(11, 0, int(offs[-1]))
    d_pay = torch.from_numpy(np.concatenate([pay, np.zeros(16, np.uint8)])).to(dev)
    d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
    k64, k32 = pmp.Keys.generate(5, 64), pmp.Keys.generate(6, 32)
    o64, o32 = oracle.keygen(5, 64), oracle.keygen(6, 32)
    w64 = oracle.hash_batch(o64, pay, offs, nthreads=os.cpu_count() or 4)
    w32 = oracle.hash_batch(o32, pay, offs, nthreads=os.cpu_count() or 4)
    ok = True
    for tc in (1, 0):
        pmp.pmp_set_short_tc(tc)
        g64, g32 = pmp.hash_batch_multi([k64, k32], d_pay, d_off)
        s64 = pmp.hash_batch(k64, d_pay, d_off)
        s32 = pmp.hash_batch(k32, d_pay, d_off)
        torch.cuda.synchronize()
        for name, got, want in (("dual64", g64, w64), ("dual32", g32, w32), ("single64", s64, w64),
                                ("single32", s32, w32)):
            g = pmp.as_u64(got)
            w = want.astype(g.dtype)
            bad = np.nonzero(g != w)[0]
            print(f"tc={tc} {name}: {bad.size} mismatches", "" if bad.size == 0 else
                  f"first {bad[:8].tolist()} lens {lens[bad[:8]].tolist()}", flush=True)
            ok &= bad.size == 0
    print("OK" if ok else "FAIL")


if __name__ == "__main__":
    main()
