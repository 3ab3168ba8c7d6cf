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


def _gpu_worker(rank, world, port, bits, total, seed, q):
    """One rank on cuda:0: its byte range of the long string through the real
    pmp_hash_long_partial (parallel.hash_long_distributed: partial kernel ->
    host-staged gloo all-gather -> combine kernel), and its byte-balanced shard
    of a batch through pmp_hash_batch (parallel.shard_batch), digests gathered."""
    import sys

    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import paper_1609_09840_b200 as pmp
        from paper_1609_09840_b200 import parallel

        torch.cuda.set_device(0)
        keys = pmp.Keys.generate(seed, bits)
        b, e = parallel.long_ranges(bits, total, world)[rank]
        local = torch.from_numpy(datagen.payload_host(seed, b, e - b)).cuda()
        side = torch.cuda.Stream()
        dig = parallel.hash_long_distributed(keys, local, e - b, b, total, stream=side)
        side.synchronize()
        long_digest = int(pmp.as_u64(dig)[0])
        # batch shard (strong scaling: one global batch, byte-balanced ranges)
        lens = datagen.lengths(datagen.LEN_LOGUNIFORM, seed, 6000, 1, 1 << 16)
        off = datagen.offsets_from_lengths(lens)
        lo, hi = parallel.shard_batch(off, world)[rank]
        sub, b0, b1 = parallel.rebase_offsets(off, lo, hi)
        pay = torch.from_numpy(datagen.payload_host(seed, b0, b1 - b0)).cuda()
        out = pmp.hash_batch(keys, pay, torch.from_numpy(sub.view(np.int64)).cuda())
        mine = torch.from_numpy(pmp.as_u64(out).astype(np.uint64).view(np.int64))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([mine.numel()], dtype=torch.int64))
        mx = int(max(s.item() for s in sizes))
        padded = torch.zeros(mx, dtype=torch.int64)
        padded[:mine.numel()] = mine
        lst = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(lst, padded)
        batch = np.concatenate([l[:int(s.item())].numpy() for l, s in zip(lst, sizes)]).view(np.uint64)
        q.put((rank, long_digest, batch if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("bits,total", [(64, 128 * 128 * 1024 + 3 * 1024 + 77), (32, 128 * 512 * 5 + 13)])
def test_distributed_long_and_batch_on_gpu(bits, total):
    """World size 2 (gloo, both ranks on cuda:0 -- the collective is host-staged,
    so no kernel waits on another rank): the multi-rank long-string split and the
    strong-scaling batch shard run the real kernels and equal the one-GPU call
    and the oracle."""
    import sys

    sys.path.insert(0, ROOT)
    import datagen
    import oracle
    import paper_1609_09840_b200 as pmp

    world, seed = 2, 23
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, bits, total, seed, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
    ok = oracle.keygen(seed, bits)
    data = datagen.payload_host(seed, 0, total)
    want_long = oracle.hash_long(ok, data, nthreads=os.cpu_count() or 4)
    assert res[0][1] == want_long and res[1][1] == want_long
    torch.cuda.set_device(0)
    keys = pmp.Keys.generate(seed, bits)
    one = int(pmp.as_u64(pmp.hash_long(keys, torch.from_numpy(data).cuda(), total))[0])
    assert one == want_long
    lens = datagen.lengths(datagen.LEN_LOGUNIFORM, seed, 6000, 1, 1 << 16)
    off = datagen.offsets_from_lengths(lens)
    pay = datagen.payload_host(seed, 0, int(off[-1]))
    want_batch = oracle.hash_batch(ok, pay, off, nthreads=os.cpu_count() or 4)
    assert np.array_equal(res[0][2], want_batch.astype(np.uint64) if bits == 64 else want_batch.astype(np.uint32).astype(np.uint64))
