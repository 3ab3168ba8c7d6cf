"""Multi-process (world_size 2, gloo, CPU) checks of the partitioning logic.

The GPU kernels cannot run here, so each rank computes its long-string partial
with an independent test-side evaluation of the affine split (Python big
integers over oracle-computed level-1 block values), all-gathers it through
torch.distributed, and combines with the library's key-only constant
C(total_len); the result must equal the oracle's literal Algorithm 1.  The
batch-sharding ranges are checked to tile the batch with balanced bytes.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _path_weight(a, c, leff):
    """K_c = prod_{j=2..leff} a_{j, digit_{j-2}(c)} with digits of the block index in base 128."""
    k = 1
    for j in range(2, leff + 1):
        k *= int(a[j - 1, (c // 128 ** (j - 2)) % 128])
    return k


def _worker(rank, world, port, bits, total, seed, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle
        import paper_1609_09840_b200 as pmp
        from paper_1609_09840_b200 import parallel

        keys = pmp.Keys.generate(seed, bits)
        ok = oracle.keygen(seed, bits)
        p = oracle.params(bits)["p"]
        w = bits // 8
        T = total // w + 1
        T1 = -(-T // 128)
        leff, n = 0, T
        while n > 1:
            n = -(-n // 128)
            leff += 1
        data = datagen.payload_host(seed, 0, total)
        b, e = parallel.long_ranges(bits, total, world)[rank]
        cb = b // (128 * w)
        ce = T1 if e == total else e // (128 * w)
        # this rank's partial: sum over its level-1 blocks of K_c * v_1(c) mod p
        part = 0
        for c in range(cb, ce):
            sig = [oracle.sigma_word(bits, data, 128 * c + r) if 128 * c + r < T else 0 for r in range(128)]
            v1 = oracle.block(p, 128, int(ok.b[0]), ok.a[0], sig)
            part = (part + _path_weight(ok.a, c, leff) * v1) % p
        # exchange the field element as four 32-bit limbs held in int64
        words = torch.tensor([(part >> s) & 0xFFFFFFFF for s in (0, 32, 64, 96)], dtype=torch.int64)
        gathered = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, words)
        total_part = sum(sum(int(x) << (32 * i) for i, x in enumerate(gw.tolist())) for gw in gathered)
        c2 = np.zeros(2, dtype=np.uint64)
        assert pmp.lib().pmp_long_constant(keys.handle, total, c2.ctypes.data) == 0
        C = int(c2[0]) | (int(c2[1]) << 64)
        V = (C + total_part) % p
        digest = oracle.mix(bits, V & (2**bits - 1))
        want = oracle.hash_long(ok, data, nthreads=2)
        q.put((rank, digest == want, (b, e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bits,total", [(64, 128 * 1024 * 2 + 5000), (32, 128 * 512 * 3 + 77), (64, 3000)])
def test_long_split_affine_combine_gloo(bits, total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bits, total, 17, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    ranges = sorted(r for _, _, r in res)
    assert ranges[0][0] == 0 and ranges[-1][1] == total and ranges[0][1] == ranges[1][0]


def test_shard_batch_tiles_and_balances():
    import sys

    sys.path.insert(0, ROOT)
    import datagen
    from paper_1609_09840_b200 import parallel

    lens = datagen.lengths(datagen.LEN_LOGUNIFORM, 5, 100_000, 1, 1 << 20)
    off = datagen.offsets_from_lengths(lens)
    for world in (1, 2, 4, 8):
        rs = parallel.shard_batch(off, world)
        assert rs[0][0] == 0 and rs[-1][1] == lens.size
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        sizes = [int(off[h]) - int(off[l]) for l, h in rs]
        assert sum(sizes) == int(off[-1])
        assert max(sizes) - min(sizes) <= 2 * (1 << 20)  # within two of the largest strings
        for l, h in rs:
            sub, b0, b1 = parallel.rebase_offsets(off, l, h)
            assert sub[0] == 0 and int(sub[-1]) == b1 - b0
