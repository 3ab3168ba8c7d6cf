"""The C ABI from a plain C program (tests/c_client/pmp_c_client.c): it
includes only include/pmp.h and the CUDA runtime, links the in-tree libpmp.so,
and must produce the oracle's digests.  Compiling and linking it needs no GPU
(a CPU test); running it does."""
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1609_09840_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    import __graft_entry__

    __graft_entry__.build()
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = os.path.join(str(tmp_path), "pmp_c_client")
    subprocess.check_call([cc, "-std=c99", "-O2", "-Wall", "-Werror",
                           os.path.join(ROOT, "tests", "c_client", "pmp_c_client.c"),
                           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
                           "-L", PKG, "-lpmp", f"-Wl,-rpath,{PKG}",
                           "-L", os.path.join(CUDA, "lib64"), "-lcudart", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}",
                           "-o", exe])
    return exe


def test_c_client_compiles_and_links(tmp_path):
    """include/pmp.h is valid C99 and every entry point the client uses links."""
    assert os.path.exists(_build(tmp_path))


LENS = [0, 1, 3, 4, 7, 8, 9, 31, 64, 127, 128, 129, 1000, 1024, 4099, 70000, 5, 0, 200]


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [64, 32])
def test_c_client_matches_oracle(tmp_path, oracle_lib, bits):
    exe = _build(tmp_path)
    inp = f"{bits} {len(LENS)} " + " ".join(str(x) for x in LENS)
    res = subprocess.run([exe], input=inp, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    lines = [ln.split() for ln in res.stdout.splitlines()]
    off = np.concatenate([[0], np.cumsum(LENS)]).astype(np.uint64)
    total = int(off[-1])
    pay = ((np.arange(total, dtype=np.uint64) * 131 + 7) & 255).astype(np.uint8)
    ok = oracle_lib.keygen(2, bits)
    want = oracle_lib.hash_batch(ok, pay, off, nthreads=4).astype(np.uint64)
    if bits == 32:
        want = want.astype(np.uint32).astype(np.uint64)
    got_batch = [int(x[2], 16) for x in lines if x[0] == "batch"]
    got_host = [int(x[2], 16) for x in lines if x[0] == "host"]
    assert got_batch == [int(v) for v in want]
    assert got_host == got_batch
    long_d = [int(x[1], 16) for x in lines if x[0] == "long"][0]
    stream_d = [int(x[1], 16) for x in lines if x[0] == "stream"][0]
    want_long = int(oracle_lib.hash_long(ok, pay, nthreads=4))
    assert long_d == want_long and stream_d == want_long
    assert [int(x[1], 16) for x in lines if x[0] == "longhost"] == [want_long]
    assert [int(x[2], 16) for x in lines if x[0] == "tput"] == got_batch
    assert [int(x[1]) for x in lines if x[0] == "einval"] == [-1]
