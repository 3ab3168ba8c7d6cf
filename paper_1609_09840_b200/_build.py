"""Compile libpmp.so in-tree for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libpmp.so")
SOURCES = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh"))] + [
    os.path.join(ROOT, "include", "pmp.h")
]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES)


def build(force: bool = False, verbose: bool = False, nvcc: str = "nvcc") -> str:
    if force or needs_build():
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc, *NVCC_FLAGS]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        cmd += [os.path.join(CSRC, "pmp_api.cu"), "-o", tmp]
        subprocess.check_call(cmd)
        os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines: dict, nvcc: str = "nvcc") -> str:
    """Tuning build: libpmp_<name>.so with -D overrides of the kernel
    parameters (e.g. {"PMP_SHORT_RING_KB": 80}); selected at run time with
    PMP_LIB_VARIANT.  The product build is always libpmp.so."""
    out = os.path.join(PKG, f"libpmp_{name}.so")
    cmd = [nvcc, *NVCC_FLAGS] + [f"-D{k}={v}" for k, v in defines.items()]
    cmd += [os.path.join(CSRC, "pmp_api.cu"), "-o", out]
    subprocess.check_call(cmd)
    return out
