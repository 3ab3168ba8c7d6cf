"""ctypes wrapper around the PM+ oracle (``oracle/libpmp_oracle.so``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1609_09840_b200``) never imports it.

Every function is a thin marshalling layer over ``pmp_oracle.c``; see that file
and ``pmp_oracle.h`` for the paper passages each one transcribes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpmp_oracle.so")
SRC_PATH = os.path.join(_HERE, "pmp_oracle.c")

M = 128
L = 8

_u64 = ctypes.c_uint64
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no CUDA, no shared code)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
        os.path.getmtime(SRC_PATH), os.path.getmtime(os.path.join(_HERE, "pmp_oracle.h"))
    ):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", SRC_PATH, "-o", tmp]
        )
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        h = ctypes.CDLL(LIB_PATH)
        h.pmpo_params.argtypes = [ctypes.c_int, _p, _p, _p, _p, _p]
        h.pmpo_params.restype = ctypes.c_int
        h.pmpo_keygen.argtypes = [_u64, ctypes.c_int, _p, _p]
        h.pmpo_keygen.restype = ctypes.c_int
        h.pmpo_mix.argtypes = [ctypes.c_int, _u64]
        h.pmpo_mix.restype = _u64
        h.pmpo_unmix.argtypes = [ctypes.c_int, _u64]
        h.pmpo_unmix.restype = _u64
        h.pmpo_sigma_word.argtypes = [ctypes.c_int, _p, _u64, _u64]
        h.pmpo_sigma_word.restype = _u64
        h.pmpo_num_words.argtypes = [ctypes.c_int, _u64]
        h.pmpo_num_words.restype = _u64
        h.pmpo_block.argtypes = [_u64, _u64, ctypes.c_int, _u64, _p, _p, _p, _p]
        h.pmpo_block.restype = None
        h.pmpo_tree_generic.argtypes = [_u64, _u64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        _p, _p, _p, _p, _u64, _p]
        h.pmpo_tree_generic.restype = ctypes.c_int
        h.pmpo_tree_value.argtypes = [ctypes.c_int, _p, _p, _p, _u64, ctypes.c_int, _p]
        h.pmpo_tree_value.restype = ctypes.c_int
        h.pmpo_hash.argtypes = [ctypes.c_int, _p, _p, _p, _u64]
        h.pmpo_hash.restype = _u64
        h.pmpo_hash_batch.argtypes = [ctypes.c_int, _p, _p, _p, _p, _u64, _p, ctypes.c_int]
        h.pmpo_hash_batch.restype = None
        h.pmpo_hash_long.argtypes = [ctypes.c_int, _p, _p, _p, _u64, ctypes.c_int]
        h.pmpo_hash_long.restype = _u64
        h.pmpo_hash2_value.argtypes = [ctypes.c_int, _p, _p, _p, _u64, ctypes.c_int, _p]
        h.pmpo_hash2_value.restype = ctypes.c_int
        h.pmpo_hash2.argtypes = [ctypes.c_int, _p, _p, _p, _u64, ctypes.c_int]
        h.pmpo_hash2.restype = _u64
        h.pmpo_hash2_batch.argtypes = [ctypes.c_int, _p, _p, _p, _p, _u64, _p, ctypes.c_int]
        h.pmpo_hash2_batch.restype = None
        h.pmpo_splitmix64_stream.argtypes = [_u64, _u64, _p]
        h.pmpo_splitmix64_stream.restype = None
        h.pmpo_xoshiro256ss_stream.argtypes = [_p, _u64, _p]
        h.pmpo_xoshiro256ss_stream.restype = None
        h.pmpo_mulmod.argtypes = [_u64, _u64, _u64, _u64, _u64, _u64, _p]
        h.pmpo_mulmod.restype = None
        _lib = h
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _bytes_arr(data) -> np.ndarray:
    if isinstance(data, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(bytes(data), dtype=np.uint8)
    else:
        arr = np.ascontiguousarray(data, dtype=np.uint8)
    if arr.size == 0:
        arr = np.zeros(1, dtype=np.uint8)[:0]
    return arr


def params(bits: int) -> dict:
    v = [ctypes.c_uint64() for _ in range(5)]
    rc = lib().pmpo_params(bits, *[ctypes.byref(x) for x in v])
    if rc != 0:
        raise ValueError(bits)
    p = v[0].value | (v[1].value << 64)
    return {"p": p, "k": v[2].value, "kappa": v[3].value, "a_max": v[4].value,
            "n": bits, "w": bits // 8}


class Keys:
    """Key schedule: b[8], a[8][128] (Alg. 1 REQUIRE; Eq. (1))."""

    def __init__(self, bits: int, b: np.ndarray, a: np.ndarray):
        self.bits = bits
        self.b = np.ascontiguousarray(b, dtype=np.uint64)
        self.a = np.ascontiguousarray(a, dtype=np.uint64).reshape(L, M)

    def b_list(self):
        return [int(x) for x in self.b]

    def a_list(self):
        return [[int(x) for x in row] for row in self.a]


def keygen(seed: int, bits: int) -> Keys:
    b = np.zeros(L, dtype=np.uint64)
    a = np.zeros(L * M, dtype=np.uint64)
    rc = lib().pmpo_keygen(seed & (2**64 - 1), bits, _ptr(b), _ptr(a))
    if rc != 0:
        raise ValueError(bits)
    return Keys(bits, b, a)


def splitmix64_stream(state: int, n: int) -> list:
    """n successive splitmix64 outputs from ``state`` (the keygen contract's seeding)."""
    out = np.zeros(n, dtype=np.uint64)
    lib().pmpo_splitmix64_stream(state & (2**64 - 1), n, _ptr(out))
    return [int(x) for x in out]


def xoshiro256ss_stream(state, n: int) -> list:
    """n successive xoshiro256** outputs from the 4-word state ``state``."""
    st = np.ascontiguousarray([int(x) & (2**64 - 1) for x in state], dtype=np.uint64)
    out = np.zeros(n, dtype=np.uint64)
    lib().pmpo_xoshiro256ss_stream(_ptr(st), n, _ptr(out))
    return [int(x) for x in out]


def mix(bits: int, z: int) -> int:
    return int(lib().pmpo_mix(bits, z & (2**64 - 1)))


def unmix(bits: int, z: int) -> int:
    return int(lib().pmpo_unmix(bits, z & (2**64 - 1)))


def num_words(bits: int, length: int) -> int:
    return int(lib().pmpo_num_words(bits, length))


def sigma_word(bits: int, data, t: int) -> int:
    arr = _bytes_arr(data)
    return int(lib().pmpo_sigma_word(bits, _ptr(arr), arr.size, t))


def block(p: int, m: int, b: int, a, x) -> int:
    a = np.ascontiguousarray([int(v) for v in a], dtype=np.uint64)
    xl = np.ascontiguousarray([int(v) & (2**64 - 1) for v in x], dtype=np.uint64)
    xh = np.ascontiguousarray([int(v) >> 64 for v in x], dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lib().pmpo_block(p & (2**64 - 1), p >> 64, m, b, _ptr(a), _ptr(xl), _ptr(xh), _ptr(out))
    return int(out[0]) | (int(out[1]) << 64)


def tree_generic(p: int, m: int, Lv: int, b, a, sigma, j0: int = 0):
    """Literal Algorithm 1 over a character string ``sigma`` (marker already
    appended).  ``a`` is a flat list of Lv*m keys.  Returns (value, levels)."""
    b = np.ascontiguousarray([int(v) for v in b], dtype=np.uint64)
    a = np.ascontiguousarray([int(v) for v in a], dtype=np.uint64)
    xl = np.ascontiguousarray([int(v) & (2**64 - 1) for v in sigma], dtype=np.uint64)
    xh = np.ascontiguousarray([int(v) >> 64 for v in sigma], dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lv = lib().pmpo_tree_generic(p & (2**64 - 1), p >> 64, m, Lv, j0, _ptr(b), _ptr(a),
                                 _ptr(xl), _ptr(xh), len(sigma), _ptr(out))
    return int(out[0]) | (int(out[1]) << 64), lv


def tree_generic_np(p: int, m: int, Lv: int, b, a, x_lo: np.ndarray, x_hi: np.ndarray, j0: int = 0):
    """Same as :func:`tree_generic` with numpy lo/hi arrays (large inputs)."""
    b = np.ascontiguousarray([int(v) for v in b], dtype=np.uint64)
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1))
    x_lo = np.ascontiguousarray(x_lo, dtype=np.uint64)
    x_hi = np.ascontiguousarray(x_hi, dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lv = lib().pmpo_tree_generic(p & (2**64 - 1), p >> 64, m, Lv, j0, _ptr(b), _ptr(a),
                                 _ptr(x_lo), _ptr(x_hi), x_lo.size, _ptr(out))
    return int(out[0]) | (int(out[1]) << 64), lv


def tree_value(keys: Keys, data, nthreads: int = 1):
    arr = _bytes_arr(data)
    out = np.zeros(2, dtype=np.uint64)
    lv = lib().pmpo_tree_value(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(arr), arr.size,
                               nthreads, _ptr(out))
    return int(out[0]) | (int(out[1]) << 64), lv


def hash_bytes(keys: Keys, data) -> int:
    arr = _bytes_arr(data)
    return int(lib().pmpo_hash(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(arr), arr.size))


def hash_long(keys: Keys, data, nthreads: int = 1) -> int:
    arr = _bytes_arr(data)
    return int(lib().pmpo_hash_long(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(arr),
                                    arr.size, nthreads))


def hash_batch(keys: Keys, payload: np.ndarray, offsets: np.ndarray, nthreads: int = 1) -> np.ndarray:
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = offsets.size - 1
    out = np.zeros(max(n, 0), dtype=np.uint64)
    if n > 0:
        lib().pmpo_hash_batch(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(payload),
                              _ptr(offsets), n, _ptr(out), nthreads)
    return out


# ---- two-level variant (reading Q19)
def mulmod(p: int, x: int, y: int) -> int:
    out = np.zeros(2, dtype=np.uint64)
    M = 2**64 - 1
    lib().pmpo_mulmod(p & M, p >> 64, x & M, x >> 64, y & M, y >> 64, _ptr(out))
    return int(out[0]) | (int(out[1]) << 64)


def hash2_value(keys: Keys, data, nthreads: int = 1) -> int:
    arr = _bytes_arr(data)
    out = np.zeros(2, dtype=np.uint64)
    rc = lib().pmpo_hash2_value(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(arr), arr.size, nthreads, _ptr(out))
    assert rc == 0
    return int(out[0]) | (int(out[1]) << 64)


def hash2(keys: Keys, data, nthreads: int = 1) -> int:
    arr = _bytes_arr(data)
    return int(lib().pmpo_hash2(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(arr), arr.size, nthreads))


def hash2_batch(keys: Keys, payload: np.ndarray, offsets: np.ndarray, nthreads: int = 1) -> np.ndarray:
    payload = np.ascontiguousarray(payload, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = offsets.size - 1
    out = np.zeros(max(n, 0), dtype=np.uint64)
    if n > 0:
        lib().pmpo_hash2_batch(keys.bits, _ptr(keys.b), _ptr(keys.a), _ptr(payload), _ptr(offsets), n,
                               _ptr(out), nthreads)
    return out
