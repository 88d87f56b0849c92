"""Bounds and race detection without a sanitizer (compute-sanitizer is not
available on the GPU pool): GPU parity and full-size invariant tests run
again against the -DTS_CHECKED build of the same sources, whose row kernel
counts every violation of its state invariants (one vehicle per cell,
PAPER.md:324; v <= vmax; vid lists consistent with the
occupancy planes and ranked onto occupied cells; nothing past a row end)
and whose node and general-tile kernels count theirs (a crosser lands
before the first occupied cell of its target lane; tile vehicles carry an
id and v <= vmax).
After every test the counters must be zero (tests/conftest.py), and the
results must still equal the oracle's."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [
    "tests/test_gpu_parity.py::test_bench_flags_full_state",
    "tests/test_gpu_parity.py::test_unstaged_groups",
    "tests/test_gpu_parity.py::test_graph_replay_grid",
    "tests/test_gpu_parity.py::test_grid_segmented_links",
    "tests/test_gpu_parity.py::test_handmade_intersections",
    "tests/test_gpu_parity.py::test_portland_small",
    "tests/test_gpu_parity.py::test_signalized_grid",
    "tests/test_gpu_domains.py::test_dense_grid_lane_changes",
    "tests/test_gpu_parity.py::test_config1_full",  # incl. every tile on the general kernels
    "tests/test_gpu_domains.py::test_config1_orb",  # split links: general tiles + strips
    "tests/test_gpu_configs.py::test_config4a_bench_routes_driver_window",
    "tests/test_gpu_configs.py::test_config4b_prefix",
    "tests/test_gpu_validation.py::test_full_size_grid_invariants_long_run",
]


def test_checked_build_invariants():
    from paper_cs_0105004_b200 import build as b
    so = b.build_checked()
    env = dict(os.environ, TSIM_LIB=so, TSIM_EXPECT_CHECKED="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        "-m", "gpu"] + CASES, cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail


def test_checked_build_selftest():
    """negative control: with the self-test armed, the checked row kernel
    reports a violation for every group of a step, so the counters do reach
    the host; disarmed, the same run is clean again"""
    from paper_cs_0105004_b200 import build as b
    so = b.build_checked()
    code = r'''
import scenarios
import paper_cs_0105004_b200 as tsim
s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=8, name="selftest")
g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
g.step(3)
assert tsim.debug_checks(reset=True)[0:2] == (1, 0)
tsim.debug_checks(arm_selftest=True)
g.step(2)
chk, bits, first, count = tsim.debug_checks(reset=True)
assert chk == 1 and bits == 128 and first == 0 and count > 0, (chk, bits, first, count)
g.step(2)
assert tsim.debug_checks(reset=True) == (1, 0, 0xFFFFFFFF, 0)
print("selftest ok", count)
'''
    env = dict(os.environ, TSIM_LIB=so)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "selftest ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
