"""Multi-GPU partitioning of the PM+ path (one process per GPU, torch.distributed).

Two ways to split work:

* Batches of strings shard trivially: each rank hashes a contiguous range of
  strings with no collective.  ``shard_batch`` picks ranges with nearly equal
  payload bytes (binary search on the CSR offsets).

* One long string is split into contiguous ranges of whole level-1 blocks
  (``long_ranges`` -> ``pmp_long_split``).  Every rank computes its partial
  P_g = sum over its blocks c of K_c * v_1(c) mod p with
  ``pmp_hash_long_partial`` (K_c = product of the level keys on c's path to the
  root), the 16-byte partials are all-gathered (one NCCL collective), and every
  rank finishes with ``pmp_hash_long_combine`` (V = C + sum_g P_g mod p).
  This is exact because each level of Algorithm 1 is an
  affine map of the level below over F_p.

Argument marshalling only; the arithmetic runs in libpmp.so.
"""
from __future__ import annotations

import numpy as np

from . import Keys, _check, pmp_hash_long_combine, pmp_hash_long_partial, pmp_long_split, _stream_ptr


def shard_batch(offsets: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous string ranges [lo, hi) per rank with ~equal payload bytes.

    ``offsets`` is the host CSR array (n+1 entries).  Ranges tile [0, n)."""
    offsets = np.asarray(offsets, dtype=np.uint64)
    n = offsets.size - 1
    total = int(offsets[-1]) - int(offsets[0])
    bounds = [0]
    for g in range(1, world):
        target = int(offsets[0]) + (total * g) // world
        # first string whose start reaches the target byte count
        idx = int(np.searchsorted(offsets[:n], np.uint64(target), side="left"))
        bounds.append(max(bounds[-1], min(idx, n)))
    bounds.append(n)
    return [(bounds[g], bounds[g + 1]) for g in range(world)]


def rebase_offsets(offsets: np.ndarray, lo: int, hi: int) -> tuple[np.ndarray, int, int]:
    """Offsets of strings [lo, hi) relative to their first byte, plus the byte
    range [b0, b1) of the payload they need."""
    sub = np.asarray(offsets[lo:hi + 1], dtype=np.uint64)
    b0, b1 = int(sub[0]), int(sub[-1])
    return sub - np.uint64(b0), b0, b1


def long_ranges(bits: int, total_len: int, world: int) -> list[tuple[int, int]]:
    """Block-aligned byte ranges [b, e) of one long string, one per rank."""
    b = pmp_long_split(bits, total_len, world)
    return [(b[g], b[g + 1]) for g in range(world)]


def gather_partials(mine, world: int, group=None):
    """All-gather the 16-byte partials of every rank into one (2*world,) int64
    tensor on ``mine``'s device, on the current stream.  NCCL: one
    all_gather_into_tensor of device buffers.  Other backends (gloo, the CPU
    test path): the partial is staged through host memory."""
    import torch
    import torch.distributed as dist

    parts = torch.zeros(2 * world, dtype=torch.int64, device=mine.device)
    if world == 1:
        parts.copy_(mine)
        return parts
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(parts, mine, group=group)
        return parts
    host = mine.cpu()
    lst = [torch.zeros_like(host) for _ in range(world)]
    dist.all_gather(lst, host, group=group)
    parts.copy_(torch.cat(lst))
    return parts


def hash_long_distributed(keys: Keys, local, local_len: int, global_offset: int, total_len: int,
                          group=None, stream=None):
    """Partial on this rank's GPU -> all_gather of the 16-byte partials (NCCL,
    or host-staged for gloo) -> combine.  ``local`` is a uint8 CUDA tensor
    holding this rank's bytes [global_offset, global_offset + local_len).
    Every step (the partial kernel, the collective, the combine) is ordered on
    ``stream`` (default: the current stream).  Returns the digest tensor
    (1 element) on every rank."""
    import contextlib

    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    with torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext():
        sp = _stream_ptr(None)
        mine = torch.zeros(2, dtype=torch.int64, device=local.device)
        _check(pmp_hash_long_partial(keys.handle, local.data_ptr(), local_len, global_offset, total_len,
                                     mine.data_ptr(), sp), "pmp_hash_long_partial")
        parts = gather_partials(mine, world, group)
        out = torch.empty(1, dtype=torch.int64 if keys.bits == 64 else torch.int32, device=local.device)
        _check(pmp_hash_long_combine(keys.handle, parts.data_ptr(), world, total_len, out.data_ptr(), sp),
               "pmp_hash_long_combine")
    return out
