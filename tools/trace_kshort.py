#!/usr/bin/env python
"""Timeline of k_short (diagnostic build PMP_SHORT_TRACE=1): run one configs[1]
step, read the clock64 stamps of blocks 0 and 1 and summarise where each
consumer warp's time goes (waiting for a tile vs hashing) and the producer's
per-tile stages.  Usage (on the GPU box):
    PMP_LIB_VARIANT=$PWD/paper_1609_09840_b200/libpmp_trace.so python tools/trace_kshort.py"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import datagen
    import paper_1609_09840_b200 as pmp

    wl = datagen.WORKLOADS["hashtable"]
    offs = datagen.offsets_from_lengths(wl.lengths())
    dev = torch.device("cuda:0")
    total = int(offs[-1])
    pay = torch.empty(total + 16, dtype=torch.uint8, device=dev)
    datagen.fill_device(wl.seed, pay.data_ptr(), total, torch.cuda.current_stream().cuda_stream)
    d_off = torch.from_numpy(offs.view(np.int64)).to(dev)
    keys = [pmp.Keys.generate(wl.seed, 64), pmp.Keys.generate(wl.seed, 32)]
    for _ in range(3):
        pmp.hash_batch_multi(keys, pay, d_off)
    torch.cuda.synchronize()
    W = 17
    n = 2 * W * 256 * 4
    buf = np.zeros(n, dtype=np.uint64)
    lib = pmp.lib()
    lib.pmp_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    lib.pmp_trace_read.restype = ctypes.c_int
    got = lib.pmp_trace_read(buf.ctypes.data, n)
    tr = buf.reshape(2, W, 256, 4).astype(np.int64)
    out = {}
    for b in range(2):
        cons = tr[b, :16]
        prod = tr[b, 16]
        ntile = int((cons[0, :, 2] > 0).sum())
        t0 = int(cons[:, 0, 0].min())
        waits = (cons[:, :ntile, 1] - cons[:, :ntile, 0])
        hashes = (cons[:, :ntile, 2] - cons[:, :ntile, 1])
        span = int(cons[:, ntile - 1, 2].max() - t0)
        # per tile: producer issue (stage 2) vs first / last consumer wait end
        rows = []
        for k in range(min(ntile, 12)):
            rows.append({"k": k, "prod_off_wait_end": int(prod[k, 0] - t0), "prod_ring_ok": int(prod[k, 1] - t0),
                         "prod_issued": int(prod[k, 2] - t0), "cons_first_ready": int(cons[:, k, 1].min() - t0),
                         "cons_last_ready": int(cons[:, k, 1].max() - t0), "cons_first_done": int(cons[:, k, 2].min() - t0),
                         "cons_last_done": int(cons[:, k, 2].max() - t0)})
        out[f"block{b}"] = {"tiles": ntile, "span_cycles": span,
                            "wait_cycles_per_tile_mean": float(waits.mean()), "hash_cycles_per_tile_mean": float(hashes.mean()),
                            "wait_fraction": float(waits.sum() / (waits.sum() + hashes.sum())),
                            "hash_cycles_per_warp_min_max": [float(hashes.mean(axis=1).min()), float(hashes.mean(axis=1).max())],
                            "first_tiles": rows}
    lib.pmp_trace_blocks.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    lib.pmp_trace_blocks.restype = ctypes.c_int
    bb = np.zeros(1024 * 3, dtype=np.uint64)
    lib.pmp_trace_blocks(bb.ctypes.data, bb.size)
    bb = bb.reshape(1024, 3).astype(np.int64)
    used = bb[:, 1] > 0
    per_sm = {}
    for smid, tiles in bb[used, :2]:
        per_sm.setdefault(int(smid), []).append(int(tiles))
    pairs = sorted(per_sm.values())
    tiles_sm = np.array([sum(v) for v in per_sm.values()])
    blk = bb[used, 1]
    out["blocks"] = {"n": int(used.sum()), "tiles_per_block_min_mean_max": [int(blk.min()), float(blk.mean()), int(blk.max())],
                     "sms": len(per_sm), "tiles_per_sm_min_mean_max": [int(tiles_sm.min()), float(tiles_sm.mean()), int(tiles_sm.max())],
                     "per_sm_block_tiles_sample": pairs[:5] + pairs[-5:]}
    print(json.dumps({"read": got, **out}, indent=1))


if __name__ == "__main__":
    main()
