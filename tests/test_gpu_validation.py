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


def discharge_network(m, green0, green1, p, queue=400, seed=11):
    """m independent approaches: a 3 km link (400 cells) filled with a
    standing queue, a signal at its downstream node (offsets spread over the
    cycle), a 750 m exit link; returns the scenario"""
    import scenarios
    from tests._ref import make_network
    nodes, links, veh = [], [], []
    for i in range(m):
        y = 2000.0 * i
        nodes += [(0.0, y), (3000.0, y), (3750.0, y)]
        links += [(3 * i, 3 * i + 1, 3000, 1, 1), (3 * i + 1, 3 * i + 2, 750, 1, 1)]
        veh += [dict(route=[2 * i, 2 * i + 1], place=(0, c, 0)) for c in range(queue)]
    s = make_network(nodes, links, veh, p_slow=p, seed=seed)
    cyc = green0 + green1
    off = (np.arange(m) * 7) % max(1, cyc)
    return scenarios.with_signals(s, nodes=np.arange(m) * 3 + 1, green0=green0, green1=green1,
                                  offset=off)


def passed_per_step(s, window):
    g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    g.step(window)
    v = g.vehicles()
    link = v["link"]
    through = (v["status"] == tsim.ARRIVED) | ((v["status"] == tsim.ACTIVE) & (link % 2 == 1))
    queued = (v["status"] == tsim.ACTIVE) & (link % 2 == 0)
    m = s.n_links // 2
    per = np.bincount(np.asarray(link)[queued] // 2, minlength=m)
    assert per.min() > 0  # every queue outlasts the window
    return through.sum() / (m * window)


@pytest.mark.parametrize("p", [0.0, 0.2])
def test_signal_half_green_half_saturation(p):
    """Fig. 4d (SPEC acceptance #4): a 30 s / 30 s
    fixed-time signal passes 0.5 x the saturation flow of the same approach
    always green, within the +-10 % of SPEC acceptance #4; averaged over 256
    approaches with spread offsets (measured at p = 0.2: 0.478, the start-up
    of the queue at every green costing time each cycle)."""
    sat = passed_per_step(discharge_network(256, 60, 0, p), 480)
    half = passed_per_step(discharge_network(256, 30, 30, p), 960)
    assert sat > 0.25
    assert 0.45 <= half / sat <= 0.55, (half, sat)


def _check_invariants(g, n_veh, vmax=5):
    """conservation; active vehicles on distinct (link, lane, cell); 0 <= v
    <= vmax; cursors inside their routes"""
    v = g.vehicles()
    st = v["status"]
    act = st == tsim.ACTIVE
    assert np.sum(act) + np.sum(st == tsim.PENDING) + np.sum(st == tsim.ARRIVED) == n_veh
    key = (v["link"][act].astype(np.int64) * 8 + v["lane"][act]) * 4_000_000 + v["cell"][act]
    assert np.unique(key).size == key.size, "two vehicles in one cell"
    assert v["v"][act].min(initial=0) >= 0 and v["v"][act].max(initial=0) <= vmax
    assert np.all(v["cursor"][act] >= 0)
    return v


def test_full_size_grid_invariants_long_run():
    """config 4a at full size (20.9 M vehicles, short routes): 600 steps in
    the bench's launch configuration, then the invariants hold and the
    counters agree with the state"""
    import scenarios as sc
    s = sc.big_grid(seed=2, dest_radius=6, name="config4a_full_inv")
    g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    g.step(600)
    v = _check_invariants(g, s.n_vehicles)
    tot = g.totals()
    assert tot["active"] == int(np.sum(v["status"] == tsim.ACTIVE))
    assert tot["arrived"] == int(np.sum(v["status"] == tsim.ARRIVED))
    assert tot["arrived"] > 0


def test_full_size_ring_invariants_long_run():
    """config 2 at full size for its 1,000 steps: no vehicle lost or
    duplicated on the 3 x 1,000,000-cell ring"""
    import scenarios as sc
    s = sc.config("2")
    g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED | tsim.FLAG_GRAPH)
    g.step(1000)
    _check_invariants(g, s.n_vehicles)
    assert g.totals()["active"] == s.n_vehicles


def _minor_throughput(s, veh):
    """minor-street vehicles that passed the stop line (now on the major exit
    or arrived), per junction, per flow level"""
    out = []
    for mb in s.minor_base:
        per = []
        for b in mb:
            cur = veh["cursor"][b:b + s.n_minor]
            st = veh["status"][b:b + s.n_minor]
            per.append(int(np.sum((st == tsim.ARRIVED) | ((st == tsim.ACTIVE) & (cur >= 1)))))
        out.append(np.asarray(per, np.float64))
    return out


def test_stop_sign_merge_capacity():
    """Fig. 4c ("merge flows through a stop sign"; SPEC.md
    merge_capacity): 64 T-junctions per major-flow level, each with a
    saturated stop-controlled minor queue merging right onto a 2-lane major
    road (gap acceptance R9).  Minor throughput over 1,800 s: > 0 with no
    major traffic; non-increasing in the major flow (means over the 64
    junctions, within 3 % of the free-road value for noise); exactly 0 when
    the major road is bumper-to-bumper.  The same run split into 2 and 4
    domains (split links, strip exchanges) is identical, and the CUDA path
    equals the oracle."""
    import oracle
    from paper_cs_0105004_b200 import domains
    s = scenarios.stop_sign_merges()
    steps = 1800
    g = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    g.step(steps)
    veh = g.vehicles()
    thr = [x.mean() for x in _minor_throughput(s, veh)]
    levels = s.headways
    assert levels[0] == 0 and levels[-1] == -1
    assert thr[0] > 100, thr  # free major road: the queue discharges
    for i in range(len(thr) - 1):
        assert thr[i + 1] <= thr[i] + 0.03 * thr[0], (levels, thr)
    assert thr[-1] == 0.0, thr
    assert thr[-2] < 0.7 * thr[0], thr  # a 2 s headway takes most of the gaps
    o = oracle.Oracle.from_scenario(s)
    o.step(steps)
    vo = o.vehicles()
    for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
        assert np.array_equal(vo[key], veh[key]), key
    for k in (2, 4):
        d = domains.LocalDomains(s, k, flags=tsim.FLAG_FUSED)
        d.step(steps)
        vd = d.vehicles()
        for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
            assert np.array_equal(vd[key], veh[key]), (k, key)
