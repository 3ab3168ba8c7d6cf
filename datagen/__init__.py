"""Seeded synthetic inputs (payload bytes, string lengths, CSR offsets).

Holds none of PM+'s arithmetic; it is the one module both the oracle side
(tests, cpu baseline) and the CUDA side (bench, GPU tests) draw inputs from.
The stream contract is documented in ``pmp_datagen.h``.

Workload recipes mirror BASELINE.json ``configs``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpmpdata.so")
SRC = os.path.join(_HERE, "datagen.cu")

LEN_FIXED, LEN_UNIFORM, LEN_LOGUNIFORM = 0, 1, 2
PAGE = 4096


def build(force: bool = False, nvcc: str = "nvcc") -> str:
    srcs = [SRC, os.path.join(_HERE, "pmp_datagen.h")]
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(map(os.path.getmtime, srcs)):
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call([nvcc, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-Xcompiler", "-fPIC", "-shared", SRC, "-o", tmp])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        h = ctypes.CDLL(LIB_PATH)
        u64, vp = ctypes.c_uint64, ctypes.c_void_p
        h.pmpd_lengths.argtypes = [ctypes.c_int, u64, u64, u64, u64, vp]
        h.pmpd_lengths.restype = None
        h.pmpd_offsets.argtypes = [vp, u64, vp]
        h.pmpd_offsets.restype = u64
        h.pmpd_fill_host.argtypes = [u64, u64, u64, vp]
        h.pmpd_fill_host.restype = None
        h.pmpd_fill_device.argtypes = [u64, vp, u64, vp]
        h.pmpd_fill_device.restype = ctypes.c_int
        h.pmpd_fill_device_at.argtypes = [u64, vp, u64, u64, vp]
        h.pmpd_fill_device_at.restype = ctypes.c_int
        h.pmpd_splitmix64_stream.argtypes = [u64, u64, vp]
        h.pmpd_splitmix64_stream.restype = None
        h.pmpd_xoshiro256ss_stream.argtypes = [vp, u64, vp]
        h.pmpd_xoshiro256ss_stream.restype = None
        h.pmpd_stream.argtypes = [u64, u64, u64, vp]
        h.pmpd_stream.restype = None
        _lib = h
    return _lib


def splitmix64_stream(state: int, n: int) -> list:
    out = np.zeros(n, dtype=np.uint64)
    lib().pmpd_splitmix64_stream(state & (2**64 - 1), n, out.ctypes.data)
    return [int(x) for x in out]


def xoshiro256ss_stream(state, n: int) -> list:
    st = np.ascontiguousarray([int(x) & (2**64 - 1) for x in state], dtype=np.uint64)
    out = np.zeros(n, dtype=np.uint64)
    lib().pmpd_xoshiro256ss_stream(st.ctypes.data, n, out.ctypes.data)
    return [int(x) for x in out]


def stream(seed: int, sid: int, n: int) -> list:
    """n outputs of stream(seed, id) (pmp_datagen.h contract)."""
    out = np.zeros(n, dtype=np.uint64)
    lib().pmpd_stream(seed & (2**64 - 1), sid & (2**64 - 1), n, out.ctypes.data)
    return [int(x) for x in out]


def lengths(kind: int, seed: int, n: int, lo: int, hi: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    if n:
        lib().pmpd_lengths(kind, seed, n, lo, hi, out.ctypes.data)
    return out


def offsets_from_lengths(lens: np.ndarray) -> np.ndarray:
    lens = np.ascontiguousarray(lens, dtype=np.uint64)
    off = np.zeros(lens.size + 1, dtype=np.uint64)
    lib().pmpd_offsets(lens.ctypes.data, lens.size, off.ctypes.data)
    return off


def payload_host(seed: int, start: int, nbytes: int) -> np.ndarray:
    out = np.zeros(nbytes, dtype=np.uint8)
    if nbytes:
        lib().pmpd_fill_host(seed, start, nbytes, out.ctypes.data)
    return out


def fill_device(seed: int, dev_ptr: int, nbytes: int, stream_ptr: int, start: int = 0) -> None:
    """Payload bytes [start, start + nbytes) on device; start must be page aligned."""
    assert start % PAGE == 0
    rc = lib().pmpd_fill_device_at(seed, dev_ptr, nbytes, start // PAGE, stream_ptr)
    if rc != 0:
        raise RuntimeError(f"pmpd_fill_device: cudaError {rc}")


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config."""
    name: str
    bits: tuple          # output widths hashed per step
    seed: int            # key seed == data seed
    n: int               # number of strings (1 for the long-string config)
    kind: int
    lo: int
    hi: int
    long: bool = False   # one string hashed with pmp_hash_long

    def lengths(self, n: int | None = None) -> np.ndarray:
        return lengths(self.kind, self.seed, self.n if n is None else n, self.lo, self.hi)


WORKLOADS = {
    # configs[0]: 1,000 strings, U[1,64] B, PM+64, seed 1
    "tiny": Workload("tiny", (64,), 1, 1000, LEN_UNIFORM, 1, 64),
    # configs[1]: 2^24 strings, U[8,64] B, packed + u64 offsets, PM+32 and PM+64, seed 2
    "hashtable": Workload("hashtable", (64, 32), 2, 1 << 24, LEN_UNIFORM, 8, 64),
    # configs[2]: 2^20 x 4096 B, PM+64, seed 3
    "fixed4k": Workload("fixed4k", (64,), 3, 1 << 20, LEN_FIXED, 4096, 4096),
    # configs[3]: one 16 GiB string, PM+64, seed 4 (reading Q16: the config names no seed)
    "long16g": Workload("long16g", (64,), 4, 1, LEN_FIXED, 16 << 30, 16 << 30, long=True),
    # configs[4]: 2^22 strings, log-uniform [1, 2^20] B, PM+32, seed 5 (reading Q15)
    "mixed": Workload("mixed", (32,), 5, 1 << 22, LEN_LOGUNIFORM, 1, 1 << 20),
}
