"""Pin: the oracle's Philox4x32-10 (reading R3) equals the CUDA toolkit's
curand_Philox4x32_10 evaluated on its host code path
(/usr/local/cuda/include/curand_philox4x32_x.h, NV_IF_ELSE_TARGET host
branch), on 10^6 random (counter, key) pairs."""
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest

import oracle
from tests._ref import philox_np

CUDA_INC = "/usr/local/cuda/include"

_SRC = r"""
#include <vector_types.h>
#include <stdio.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main() {
  unsigned in[6];
  while (fread(in, 4, 6, stdin) == 6) {
    uint4 c = {in[0], in[1], in[2], in[3]};
    uint2 k = {in[4], in[5]};
    uint4 r = curand_Philox4x32_10(c, k);
    unsigned o[4] = {r.x, r.y, r.z, r.w};
    fwrite(o, 4, 4, stdout);
  }
  return 0;
}
"""


@pytest.fixture(scope="module")
def curand_host():
    if not os.path.exists(os.path.join(CUDA_INC, "curand_philox4x32_x.h")):
        pytest.skip("CUDA toolkit headers not present")
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no host C++ compiler")
    d = tempfile.mkdtemp()
    src = os.path.join(d, "ph.cpp")
    exe = os.path.join(d, "ph")
    open(src, "w").write(_SRC)
    subprocess.check_call([cxx, "-O2", "-I", CUDA_INC, src, "-o", exe])

    def run(inp):
        out = subprocess.run([exe], input=inp.astype(np.uint32).tobytes(),
                             capture_output=True, check=True).stdout
        return np.frombuffer(out, dtype=np.uint32).reshape(-1, 4)

    yield run
    shutil.rmtree(d, ignore_errors=True)


def test_oracle_philox_matches_curand(curand_host):
    rng = np.random.default_rng(12345)
    n = 20000
    inp = rng.integers(0, 2**32, size=(n, 6), dtype=np.uint64).astype(np.uint32)
    ref = curand_host(inp)
    got = np.stack([oracle.philox4x32_10(r[:4], r[4:]) for r in inp])
    np.testing.assert_array_equal(got, ref)


def test_numpy_philox_matches_curand_1e6(curand_host):
    """10^6 pairs: the independent numpy Philox used by the brute-force
    tests is also pinned to curand."""
    rng = np.random.default_rng(777)
    n = 1_000_000
    inp = rng.integers(0, 2**32, size=(n, 6), dtype=np.uint64).astype(np.uint32)
    ref = curand_host(inp)
    got = np.stack(philox_np(*(inp[:, i] for i in range(6))), axis=1)
    np.testing.assert_array_equal(got, ref)


def test_simulation_counters_and_edges(curand_host):
    """the (t, vid, 0, 0) counter layout used by the brake draw, incl. large
    t, vid and a 64-bit seed"""
    cases = np.array([[0, 0, 0, 0, 1, 0], [3599, 20889599, 0, 0, 1, 0],
                      [2**31, 2**32 - 1, 0, 0, 0xDEADBEEF, 0x12345678],
                      [2**32 - 1, 2**32 - 1, 2**32 - 1, 2**32 - 1, 2**32 - 1, 2**32 - 1]],
                     dtype=np.uint64).astype(np.uint32)
    ref = curand_host(cases)
    for r, e in zip(cases, ref):
        np.testing.assert_array_equal(oracle.philox4x32_10(r[:4], r[4:]), e)


def test_brake_frequency():
    """P(u < floor(0.2 * 2^32)) = 0.2 (statistical, 10^6 draws)"""
    t = np.zeros(10**6, np.uint32)
    vid = np.arange(10**6, dtype=np.uint32)
    u = philox_np(t, vid, 0, 0, 1, 0)[0]
    frac = np.mean(u.astype(np.uint64) < np.uint64(858993459))
    assert abs(frac - 0.2) < 2e-3
