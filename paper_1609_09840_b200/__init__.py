"""PM+ hashing on B200 -- thin Python binding over libpmp.so (include/pmp.h).

Argument marshalling only: every step of the hash runs in the CUDA kernels of
``csrc/``.  The functions keep the C names (``pmp_keygen``, ``pmp_hash_batch``,
``pmp_hash_long``, ...) and take raw integers for device pointers and streams;
the ``hash_batch`` / ``hash_long`` conveniences accept torch CUDA tensors and
use torch only for device memory and the current stream.

There is no CPU fallback: importing works without a GPU (for the ABI checks),
but every hash call fails loudly when no CUDA device is present.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

# PMP_LIB_VARIANT: path of an in-tree tuning build (_build.build_variant), used by
# the measurement tools to compare kernel parameters; defaults to libpmp.so.
LIB_PATH = os.environ.get("PMP_LIB_VARIANT") or _build.LIB

PMP_OK, PMP_EINVAL, PMP_ETOOLONG, PMP_ECUDA, PMP_ENOMEM, PMP_ENODEV = 0, -1, -2, -3, -4, -5
PMP_EBADFILE, PMP_EVERSION, PMP_EKEYRANGE = -6, -7, -8

_u64, _vp, _int = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
_lib = None


class PmpError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {strerror(code)} ({code})")
        self.code = code


def lib() -> ctypes.CDLL:
    """Load the in-tree libpmp.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        h = ctypes.CDLL(LIB_PATH)
        sig = {
            "pmp_keygen": ([_u64, _int], _vp),
            "pmp_keys_from_words": ([_int, _vp, _vp], _vp),
            "pmp_keys_export": ([_vp, _vp, _vp], _int),
            "pmp_keys_bits": ([_vp], _int),
            "pmp_keyfile_size": ([_int], _u64),
            "pmp_keys_save": ([_vp, _vp, _u64], _int),
            "pmp_keys_load": ([_vp, _u64, ctypes.POINTER(_int)], _vp),
            "pmp_keys_free": ([_vp], None),
            "pmp_hash_batch": ([_vp, _vp, _vp, _u64, _vp, _vp], _int),
            "pmp_hash_batch_buckets": ([_vp, _vp, _vp, _u64, ctypes.c_uint32, _vp, _vp, _vp], _int),
            "pmp_bucket_partition": ([_vp, _u64, ctypes.c_uint32, _vp, _vp, _vp, _vp], _int),
            "pmp_hash_batch_host": ([_vp, _int, _vp, _vp, _u64, _vp, _u64, _vp], _int),
            "pmp_hash_batch_multi": ([_vp, _int, _vp, _vp, _u64, _vp, _vp], _int),
            "pmp_hash2_batch_multi": ([_vp, _int, _vp, _vp, _u64, _vp, _vp], _int),
            "pmp_hash_long": ([_vp, _vp, _u64, _vp, _vp], _int),
            "pmp_hash_long_host": ([_vp, _vp, _u64, _vp, _u64, _vp], _int),
            "pmp_hash_long_partial": ([_vp, _vp, _u64, _u64, _u64, _vp, _vp], _int),
            "pmp_hash_long_combine": ([_vp, _vp, _int, _u64, _vp, _vp], _int),
            "pmp_long_split": ([_int, _u64, _int, _vp], _int),
            "pmp_hash2_batch": ([_vp, _vp, _vp, _u64, _vp, _vp], _int),
            "pmp_hash2_long": ([_vp, _vp, _u64, _vp, _vp], _int),
            "pmp_hash2_long_partial": ([_vp, _vp, _u64, _u64, _u64, _vp, _vp], _int),
            "pmp_hash2_long_combine": ([_vp, _vp, _int, _vp, _vp], _int),
            "pmp_stream_new": ([_vp], _vp),
            "pmp_stream_update": ([_vp, _vp, _u64, _vp], _int),
            "pmp_stream_final": ([_vp, _vp, _vp], _int),
            "pmp_stream_reset": ([_vp, _vp], _int),
            "pmp_stream_free": ([_vp], None),
            "pmp_long_constant": ([_vp, _u64, _vp], _int),
            "pmp_selftest": ([_int, _int, _vp, _u64, _vp, _vp], _int),
            "pmp_launch_count": ([], _u64),
            "pmp_set_small_batch_max": ([_u64], _u64),
            "pmp_set_short_tc": ([ctypes.c_int], ctypes.c_int),
            "pmp_set_huge_min": ([ctypes.c_uint64], ctypes.c_uint64),
            "pmp_set_huge_cap": ([ctypes.c_uint32], ctypes.c_uint32),
            "pmp_quality_collisions": ([_int, _u64, _u64, _vp, ctypes.c_uint32, _vp, ctypes.c_uint32, _vp, _vp, _vp,
                                        _vp], _int),
            "pmp_prof_enable": ([_int], None),
            "pmp_prof_reset": ([], None),
            "pmp_prof_read": ([ctypes.c_char_p, _vp, _vp], _int),
            "pmp_strerror": ([_int], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = res
        _lib = h
    return _lib


def strerror(code: int) -> str:
    return lib().pmp_strerror(code).decode()


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise PmpError(rc, what)


# --------------------------------------------------------------- C-named calls
def pmp_keygen(seed: int, out_bits: int) -> int:
    return lib().pmp_keygen(seed & (2**64 - 1), out_bits) or 0


def pmp_keys_from_words(out_bits: int, b_ptr: int, a_ptr: int) -> int:
    return lib().pmp_keys_from_words(out_bits, b_ptr, a_ptr) or 0


def pmp_keys_export(keys: int, b_ptr: int, a_ptr: int) -> int:
    return lib().pmp_keys_export(keys, b_ptr, a_ptr)


def pmp_keyfile_size(out_bits: int) -> int:
    return int(lib().pmp_keyfile_size(out_bits))


def pmp_keys_save(keys: int, out_ptr: int, cap: int) -> int:
    return lib().pmp_keys_save(keys, out_ptr, cap)


def pmp_keys_load(buf_ptr: int, length: int) -> tuple[int, int]:
    """Returns (handle or 0, error code)."""
    err = _int(0)
    h = lib().pmp_keys_load(buf_ptr, length, ctypes.byref(err)) or 0
    return h, err.value


def pmp_keys_free(keys: int) -> None:
    lib().pmp_keys_free(keys)


def pmp_hash_batch(keys: int, bytes_ptr: int, offsets_ptr: int, n: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_hash_batch(keys, bytes_ptr, offsets_ptr, n, out_ptr, stream)


def pmp_hash_batch_multi(keys: list, bytes_ptr: int, offsets_ptr: int, n: int, out_ptrs: list, stream: int) -> int:
    """keys: list of pmp_keys* handles; out_ptrs: one device digest buffer per key."""
    ka = (_vp * len(keys))(*keys)
    oa = (_vp * len(out_ptrs))(*out_ptrs)
    return lib().pmp_hash_batch_multi(ka, len(keys), bytes_ptr, offsets_ptr, n, oa, stream)


def pmp_hash2_batch_multi(keys: list, bytes_ptr: int, offsets_ptr: int, n: int, out_ptrs: list, stream: int) -> int:
    """pmp_hash_batch_multi for the two-level variant."""
    ka = (_vp * len(keys))(*keys)
    oa = (_vp * len(out_ptrs))(*out_ptrs)
    return lib().pmp_hash2_batch_multi(ka, len(keys), bytes_ptr, offsets_ptr, n, oa, stream)


def pmp_hash_batch_host(keys: list, bytes_ptr: int, offsets_ptr: int, n: int, out_ptrs: list,
                        piece_bytes: int, stream: int) -> int:
    """keys: list of pmp_keys* handles; out_ptrs: one host digest buffer per key."""
    ka = (_vp * len(keys))(*keys)
    oa = (_vp * len(out_ptrs))(*out_ptrs)
    return lib().pmp_hash_batch_host(ka, len(keys), bytes_ptr, offsets_ptr, n, oa, piece_bytes, stream)


def pmp_hash_batch_buckets(keys: int, bytes_ptr: int, offsets_ptr: int, n: int, M: int, buckets_ptr: int,
                           counts_ptr: int, stream: int) -> int:
    return lib().pmp_hash_batch_buckets(keys, bytes_ptr, offsets_ptr, n, M, buckets_ptr, counts_ptr, stream)


def pmp_bucket_partition(buckets_ptr: int, n: int, M: int, hist_ptr: int, starts_ptr: int, perm_ptr: int,
                         stream: int = 0) -> int:
    return lib().pmp_bucket_partition(buckets_ptr, n, M, hist_ptr, starts_ptr, perm_ptr, stream)


def pmp_hash_long(keys: int, bytes_ptr: int, length: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_hash_long(keys, bytes_ptr, length, out_ptr, stream)


def pmp_hash_long_partial(keys: int, local_ptr: int, local_len: int, global_offset: int,
                          total_len: int, partial_ptr: int, stream: int) -> int:
    return lib().pmp_hash_long_partial(keys, local_ptr, local_len, global_offset, total_len,
                                       partial_ptr, stream)


def pmp_hash_long_combine(keys: int, partials_ptr: int, G: int, total_len: int, out_ptr: int,
                          stream: int) -> int:
    return lib().pmp_hash_long_combine(keys, partials_ptr, G, total_len, out_ptr, stream)


def pmp_hash2_batch(keys: int, bytes_ptr: int, offsets_ptr: int, n: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_hash2_batch(keys, bytes_ptr, offsets_ptr, n, out_ptr, stream)


def pmp_hash2_long(keys: int, bytes_ptr: int, length: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_hash2_long(keys, bytes_ptr, length, out_ptr, stream)


def pmp_hash2_long_partial(keys: int, local_ptr: int, local_len: int, global_offset: int,
                           total_len: int, partial_ptr: int, stream: int) -> int:
    return lib().pmp_hash2_long_partial(keys, local_ptr, local_len, global_offset, total_len,
                                        partial_ptr, stream)


def pmp_hash2_long_combine(keys: int, partials_ptr: int, G: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_hash2_long_combine(keys, partials_ptr, G, out_ptr, stream)


def pmp_stream_new(keys: int) -> int:
    return lib().pmp_stream_new(keys) or 0


def pmp_stream_update(s: int, bytes_ptr: int, length: int, stream: int) -> int:
    return lib().pmp_stream_update(s, bytes_ptr, length, stream)


def pmp_stream_final(s: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_stream_final(s, out_ptr, stream)


def pmp_stream_reset(s: int, stream: int) -> int:
    return lib().pmp_stream_reset(s, stream)


def pmp_stream_free(s: int) -> None:
    lib().pmp_stream_free(s)


def pmp_selftest(out_bits: int, mode: int, in_ptr: int, n: int, out_ptr: int, stream: int) -> int:
    return lib().pmp_selftest(out_bits, mode, in_ptr, n, out_ptr, stream)


def pmp_launch_count() -> int:
    return int(lib().pmp_launch_count())


def pmp_set_small_batch_max(n: int) -> int:
    return int(lib().pmp_set_small_batch_max(n))


def pmp_set_huge_min(nbytes: int) -> int:
    """Throughput path: strings of >= nbytes go node-parallel (k_huge); 0 queries."""
    return int(lib().pmp_set_huge_min(int(nbytes)))


def pmp_set_huge_cap(cap: int) -> int:
    """At most cap huge strings per call take k_huge (0: off).  Returns the previous cap."""
    return int(lib().pmp_set_huge_cap(int(cap)))


def pmp_set_short_tc(on: int) -> int:
    """1: short strings' level-1 sums on the tensor cores (k_short_tc), 0: the
    word loop (k_short), -1: query.  Returns the previous setting."""
    return int(lib().pmp_set_short_tc(int(on)))


def pmp_prof_enable(on: bool) -> None:
    lib().pmp_prof_enable(1 if on else 0)


def pmp_prof_reset() -> None:
    lib().pmp_prof_reset()


def pmp_prof_read(prefix: str) -> tuple[float, int]:
    ms = ctypes.c_double()
    cnt = ctypes.c_uint64()
    _check(lib().pmp_prof_read(prefix.encode(), ctypes.byref(ms), ctypes.byref(cnt)), "pmp_prof_read")
    return ms.value, cnt.value


def pmp_long_split(out_bits: int, total_len: int, G: int) -> list[int]:
    arr = (ctypes.c_uint64 * (G + 1))()
    _check(lib().pmp_long_split(out_bits, total_len, G, arr), "pmp_long_split")
    return [int(x) for x in arr]


# --------------------------------------------------------------- conveniences
class Keys:
    """Owning wrapper of a ``pmp_keys*`` handle (device copy on the current device)."""

    def __init__(self, handle: int, bits: int):
        if not handle:
            raise PmpError(PMP_EINVAL, "pmp_keygen / pmp_keys_from_words returned NULL")
        self.handle = handle
        self.bits = bits

    @classmethod
    def generate(cls, seed: int, bits: int) -> "Keys":
        return cls(pmp_keygen(seed, bits), bits)

    @classmethod
    def from_words(cls, bits: int, b, a) -> "Keys":
        import numpy as np

        b = np.ascontiguousarray(b, dtype=np.uint64)
        a = np.ascontiguousarray(a, dtype=np.uint64).reshape(-1)
        assert b.size == 8 and a.size == 8 * 128
        return cls(pmp_keys_from_words(bits, b.ctypes.data, a.ctypes.data), bits)

    def save(self) -> bytes:
        """The KeyFile bytes."""
        n = pmp_keyfile_size(self.bits)
        buf = ctypes.create_string_buffer(n)
        _check(pmp_keys_save(self.handle, ctypes.addressof(buf), n), "pmp_keys_save")
        return buf.raw

    @classmethod
    def load(cls, data: bytes) -> "Keys":
        buf = ctypes.create_string_buffer(bytes(data), len(data))
        h, err = pmp_keys_load(ctypes.addressof(buf), len(data))
        if not h:
            raise PmpError(err, "pmp_keys_load")
        return cls(h, lib().pmp_keys_bits(h))

    def export(self):
        import numpy as np

        b = np.zeros(8, dtype=np.uint64)
        a = np.zeros(8 * 128, dtype=np.uint64)
        _check(pmp_keys_export(self.handle, b.ctypes.data, a.ctypes.data), "pmp_keys_export")
        return b, a.reshape(8, 128)

    def close(self) -> None:
        if self.handle:
            pmp_keys_free(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def hash_batch(keys: Keys, payload, offsets, out=None, stream=None):
    """Hash the CSR batch (``payload`` uint8 CUDA tensor, ``offsets`` int64/uint64
    CUDA tensor of n+1 entries).  Returns ``out`` (uint64 or uint32 view in an
    int64/int32 tensor) -- asynchronous on the current torch stream."""
    import torch

    n = offsets.numel() - 1
    if out is None:
        out = torch.empty(max(n, 0), dtype=torch.int64 if keys.bits == 64 else torch.int32,
                          device=offsets.device)
    _check(pmp_hash_batch(keys.handle, payload.data_ptr(), offsets.data_ptr(), max(n, 0),
                          out.data_ptr(), _stream_ptr(stream)), "pmp_hash_batch")
    return out


def hash_batch_multi(keys: list, payload, offsets, outs=None, stream=None):
    """Several key schedules over one device batch (a 64-bit + 32-bit pair is
    fused into one pass over the short strings); returns one digest tensor per key."""
    import torch

    n = offsets.numel() - 1
    if outs is None:
        outs = [torch.empty(max(n, 0), dtype=torch.int64 if k.bits == 64 else torch.int32, device=offsets.device)
                for k in keys]
    _check(pmp_hash_batch_multi([k.handle for k in keys], payload.data_ptr(), offsets.data_ptr(), max(n, 0),
                                [o.data_ptr() for o in outs], _stream_ptr(stream)), "pmp_hash_batch_multi")
    return outs


def hash_batch_host(keys: list, payload, offsets, outs=None, piece_bytes: int = 0):
    """Host-resident batch (numpy uint8 payload, uint64 offsets, or pinned torch
    CPU tensors) under one or more key schedules; returns one host digest array
    per key.  Pieces stream through the device with copy/compute overlap
    (pmp_hash_batch_host); this wrapper waits for the digests."""
    import numpy as np

    def ptr(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    n = (offsets.numel() if hasattr(offsets, "numel") else offsets.size) - 1
    if outs is None:
        outs = [np.empty(max(n, 0), dtype=np.uint64 if k.bits == 64 else np.uint32) for k in keys]
    import torch

    st = torch.cuda.current_stream()
    _check(pmp_hash_batch_host([k.handle for k in keys], ptr(payload), ptr(offsets), max(n, 0),
                               [ptr(o) for o in outs], piece_bytes, int(st.cuda_stream)), "pmp_hash_batch_host")
    st.synchronize()
    return outs


def hash_long_host(keys: Keys, data, piece_bytes: int = 0) -> int:
    """One host-resident string (numpy uint8 array, bytes, or a pinned torch CPU
    tensor) streamed through the device (pmp_hash_long_host); returns the
    digest as a Python int."""
    import numpy as np
    import torch

    if isinstance(data, (bytes, bytearray)):
        data = np.frombuffer(bytes(data), dtype=np.uint8)
    n = data.numel() if hasattr(data, "numel") else data.size
    p = data.data_ptr() if hasattr(data, "data_ptr") else (data.ctypes.data if n else 0)
    out = np.zeros(1, dtype=np.uint64 if keys.bits == 64 else np.uint32)
    st = torch.cuda.current_stream()
    _check(lib().pmp_hash_long_host(keys.handle, p, n, out.ctypes.data, piece_bytes, int(st.cuda_stream)),
           "pmp_hash_long_host")
    st.synchronize()
    return int(out[0])


def hash_batch_buckets(keys: Keys, payload, offsets, M: int, counts=None, out=None, stream=None):
    """Bucket ids digest mod M (int32 tensor holding uint32) and, if ``counts``
    (int32 CUDA tensor of M zeros) is given, the per-bucket histogram."""
    import torch

    n = offsets.numel() - 1
    if out is None:
        out = torch.empty(max(n, 0), dtype=torch.int32, device=offsets.device)
    _check(pmp_hash_batch_buckets(keys.handle, payload.data_ptr(), offsets.data_ptr(), max(n, 0), M,
                                  out.data_ptr(), counts.data_ptr() if counts is not None else 0,
                                  _stream_ptr(stream)), "pmp_hash_batch_buckets")
    return out


def bucket_partition(buckets, M: int, hist=None, stream=None):
    """String indices grouped by bucket id (pmp_bucket_partition): returns
    (starts, perm) -- int64 tensor of M+1 bucket starts and int32 tensor (holding
    uint32) of the n indices, bucket by bucket (order inside a bucket
    unspecified).  ``hist``: optional int32 tensor of the M bucket sizes."""
    import torch

    n = buckets.numel()
    starts = torch.empty(M + 1, dtype=torch.int64, device=buckets.device)
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=buckets.device)
    _check(pmp_bucket_partition(buckets.data_ptr(), n, M, hist.data_ptr() if hist is not None else 0,
                                starts.data_ptr(), perm.data_ptr(), _stream_ptr(stream)), "pmp_bucket_partition")
    return starts, perm[:n]


def hash_long(keys: Keys, data, length: int | None = None, out=None, stream=None):
    import torch

    length = data.numel() if length is None else length
    if out is None:
        out = torch.empty(1, dtype=torch.int64 if keys.bits == 64 else torch.int32, device=data.device)
    _check(pmp_hash_long(keys.handle, data.data_ptr(), length, out.data_ptr(), _stream_ptr(stream)),
           "pmp_hash_long")
    return out


def hash_long_partial(keys: Keys, local, local_len: int, global_offset: int, total_len: int,
                      partial=None, stream=None):
    import torch

    if partial is None:
        partial = torch.zeros(2, dtype=torch.int64, device=local.device)
    _check(pmp_hash_long_partial(keys.handle, local.data_ptr(), local_len, global_offset, total_len,
                                 partial.data_ptr(), _stream_ptr(stream)), "pmp_hash_long_partial")
    return partial


def hash_long_combine(keys: Keys, partials, total_len: int, out=None, stream=None):
    import torch

    G = partials.numel() // 2
    if out is None:
        out = torch.empty(1, dtype=torch.int64 if keys.bits == 64 else torch.int32, device=partials.device)
    _check(pmp_hash_long_combine(keys.handle, partials.data_ptr(), G, total_len, out.data_ptr(),
                                 _stream_ptr(stream)), "pmp_hash_long_combine")
    return out


def hash2_batch(keys: Keys, payload, offsets, out=None, stream=None):
    """Two-level variant (8(f4)) of hash_batch."""
    import torch

    n = offsets.numel() - 1
    if out is None:
        out = torch.empty(max(n, 0), dtype=torch.int64 if keys.bits == 64 else torch.int32,
                          device=offsets.device)
    _check(pmp_hash2_batch(keys.handle, payload.data_ptr(), offsets.data_ptr(), max(n, 0),
                           out.data_ptr(), _stream_ptr(stream)), "pmp_hash2_batch")
    return out


def hash2_long(keys: Keys, data, length: int | None = None, out=None, stream=None):
    import torch

    length = data.numel() if length is None else length
    if out is None:
        out = torch.empty(1, dtype=torch.int64 if keys.bits == 64 else torch.int32, device=data.device)
    _check(pmp_hash2_long(keys.handle, data.data_ptr(), length, out.data_ptr(), _stream_ptr(stream)),
           "pmp_hash2_long")
    return out


def hash2_long_partial(keys: Keys, local, local_len: int, global_offset: int, total_len: int,
                       partial=None, stream=None):
    import torch

    if partial is None:
        partial = torch.zeros(2, dtype=torch.int64, device=local.device)
    _check(pmp_hash2_long_partial(keys.handle, local.data_ptr(), local_len, global_offset, total_len,
                                  partial.data_ptr(), _stream_ptr(stream)), "pmp_hash2_long_partial")
    return partial


def hash2_long_combine(keys: Keys, partials, out=None, stream=None):
    import torch

    G = partials.numel() // 2
    if out is None:
        out = torch.empty(1, dtype=torch.int64 if keys.bits == 64 else torch.int32, device=partials.device)
    _check(pmp_hash2_long_combine(keys.handle, partials.data_ptr(), G, out.data_ptr(), _stream_ptr(stream)),
           "pmp_hash2_long_combine")
    return out


class Stream:
    """Incremental hash (pmp_stream_*): ``update`` with uint8 CUDA tensors, then
    ``final`` -> digest tensor.  Keep fed tensors alive until the torch stream
    has consumed them."""

    def __init__(self, keys: Keys):
        self.keys = keys
        self.handle = pmp_stream_new(keys.handle)
        if not self.handle:
            raise PmpError(PMP_ENOMEM, "pmp_stream_new")

    def update(self, data, length: int | None = None, stream=None):
        length = data.numel() if length is None else length
        _check(pmp_stream_update(self.handle, data.data_ptr(), length, _stream_ptr(stream)), "pmp_stream_update")
        return self

    def final(self, out=None, stream=None):
        import torch

        if out is None:
            out = torch.empty(1, dtype=torch.int64 if self.keys.bits == 64 else torch.int32, device="cuda")
        _check(pmp_stream_final(self.handle, out.data_ptr(), _stream_ptr(stream)), "pmp_stream_final")
        return out

    def reset(self, stream=None):
        _check(pmp_stream_reset(self.handle, _stream_ptr(stream)), "pmp_stream_reset")

    def close(self):
        if self.handle:
            pmp_stream_free(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def as_u64(t) -> "object":
    """Digest tensor (int64/int32) -> numpy uint64/uint32 on host."""
    import numpy as np

    a = t.detach().cpu().numpy()
    return a.view(np.uint64) if a.dtype == np.int64 else a.view(np.uint32)
