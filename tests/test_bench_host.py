"""CPU checks of bench.py's host logic (no GPU): the strong-scaling shards of the
one global batch tile it exactly and regenerate the same bytes, the weak mode
gives every rank its own recipe batch, and configs[4] is always split in 8."""
import numpy as np

import bench
import datagen


def _bytes_of(seed, offs, b0, i):
    o0, o1 = int(offs[i]), int(offs[i + 1])
    return datagen.payload_host(seed, b0 + o0, o1 - o0).tobytes()


def test_strong_shards_tile_the_global_batch():
    wl = datagen.WORKLOADS["tiny"]
    seed, lens, offs, b0 = bench.make_batch(wl, 0)
    assert b0 == 0 and lens.size == wl.n
    for world in (2, 3, 8):
        got_lens, got_bytes = [], []
        for r in range(world):
            s, l, o, bb = bench.make_batch(wl, r, world)
            assert s == wl.seed and o[0] == 0 and int(o[-1]) == int(l.sum())
            got_lens.append(l)
            got_bytes += [_bytes_of(s, o, bb, i) for i in range(l.size)]
        assert np.array_equal(np.concatenate(got_lens), lens)
        assert got_bytes == [_bytes_of(seed, offs, 0, i) for i in range(wl.n)]


def test_weak_mode_and_mixed_split():
    wl = datagen.WORKLOADS["tiny"]
    s0, l0, _, _ = bench.make_batch(wl, 0, 2, weak=True)
    s1, l1, _, _ = bench.make_batch(wl, 1, 2, weak=True)
    assert (s0, s1) == (wl.seed, wl.seed + 256) and l0.size == l1.size == wl.n
    assert bench.scaling_of(wl, weak=True) == "weak" and bench.scaling_of(wl, weak=False) == "strong"
    mixed = datagen.WORKLOADS["mixed"]
    assert bench.scaling_of(mixed, weak=False) == "weak"
    assert bench.scaling_of(datagen.WORKLOADS["long16g"], weak=True) == "strong"


def test_config_lines_name_the_baseline_config():
    for name, idx in (("tiny", 0), ("hashtable", 1), ("fixed4k", 2), ("long16g", 3), ("mixed", 4)):
        c = bench.workload_config(datagen.WORKLOADS[name], 1, False)
        assert c["workload"] == name and c["baseline_config"] == idx
    assert bench.ORDER[-1] == "hashtable"      # the headline line is printed last
