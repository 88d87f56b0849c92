"""Flow-validation suite on the GPU path:
the fundamental-diagram properties the paper's validation rests on,
measured at GPU scale with the CUDA kernels (the same properties pin the
CPU oracle in test_oracle_nasch / test_oracle_lanechange)."""
import numpy as np
import pytest

import scenarios

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")


def ring_flow(n_cells, lanes, density, p, vmax=5, warm=1500, meas=1000, seed=3):
    s = scenarios.ring(n_cells=n_cells, lanes=lanes, density=density, seed=seed, vmax=vmax)
    s.p_slow = p
    g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    g.step(warm)
    t0 = g.t + 1
    g.step(meas)
    q = g.flow(t0, meas).astype(np.float64) / (n_cells * lanes)
    return float(q.mean())


@pytest.mark.parametrize("rho", [0.05, 0.1, 1 / 6, 0.25, 0.5, 0.8])
def test_deterministic_fundamental_diagram(rho):
    """p = 0, one lane: q = min(rho * V, 1 - rho) exactly in the steady state
    (north_star; capacity V/(V+1) at rho = 1/(V+1))"""
    L = 1000
    q = ring_flow(L, 1, rho, 0.0, warm=3000, meas=1000)
    n = round(rho * L)
    assert abs(q - min(n * 5, L - n) / L) < 1e-12


@pytest.mark.parametrize("p,rho", [(0.2, 0.1), (0.2, 0.3), (0.5, 0.5), (0.2, 0.7)])
def test_vmax1_exact_stationary_flow(p, rho):
    """V = 1 parallel NaSch: q = (1 - sqrt(1 - 4 (1-p) rho (1-rho))) / 2"""
    q = ring_flow(100_000, 1, rho, p, vmax=1, warm=2000, meas=2000)
    exact = 0.5 * (1 - np.sqrt(1 - 4 * (1 - p) * rho * (1 - rho)))
    assert abs(q - exact) < 2e-3, (q, exact)


def test_three_lanes_vs_one():
    """lane changing on a 3-lane ring: total flow >= 2.5 x one lane and the
    lanes carry equal flow within 10 %"""
    q1 = ring_flow(50_000, 1, 0.15, 0.2)
    s = scenarios.ring(n_cells=50_000, lanes=3, density=0.15, seed=4)
    g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    g.step(1500)
    t0 = g.t + 1
    g.step(1000)
    q3 = float(g.flow(t0, 1000).mean()) / 50_000  # per lane-length
    assert q3 >= 2.5 * q1, (q3, q1)
    veh = g.vehicles()
    act = veh["status"] == tsim.ACTIVE
    per_lane = np.array([np.sum(veh["v"][act & (veh["lane"] == k)]) for k in range(3)], float)
    assert per_lane.max() / per_lane.mean() < 1.10, per_lane
