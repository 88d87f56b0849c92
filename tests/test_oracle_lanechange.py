"""Pins for the oracle's lane-change sub-step (readings
R4-R7).  The lane-change constants themselves are only internally pinned
(parity unpinned against an external trajectory: Fig. 4b is unreadable,
SPEC.md:559) -- see DESIGN.md §4."""
import numpy as np
import pytest

import oracle
from tests._ref import brake_np, make_network, make_ring, ring_multilane_ref


@pytest.mark.parametrize("case", range(16))
def test_multilane_ring_brute_force(case):
    """independent grid/numpy implementation of the same rules on small
    2-4 lane rings, p = 0.3, 60 steps"""
    rng = np.random.default_rng(50 + case)
    lanes = int(rng.integers(2, 5))
    L = int(rng.integers(10, 25))
    N = int(rng.integers(1, lanes * L // 2))
    flat = np.sort(rng.choice(lanes * L, size=N, replace=False))
    lane, cell = flat // L, flat % L
    v = rng.integers(0, 6, size=N)
    seed = int(rng.integers(1, 2**31))
    p = 0.3
    s = make_ring(L, lane, cell, v, lanes=lanes, p_slow=p, seed=seed)
    o = oracle.Oracle.from_scenario(s)
    ref = ring_multilane_ref(L, lanes, lane, cell, v, 5, 60,
                             lambda t, ids: brake_np(t, ids, seed, p))
    for t in range(60):
        o.step(1)
        st = o.vehicles()
        rl, rc, rv = ref[t]
        np.testing.assert_array_equal(st["lane"], rl, err_msg=f"t={t}")
        np.testing.assert_array_equal(st["cell"], rc, err_msg=f"t={t}")
        np.testing.assert_array_equal(st["v"], rv, err_msg=f"t={t}")


@pytest.mark.parametrize("lanes", [2, 3, 4])
def test_lane_reflection_symmetry(lanes):
    """p = 0: reflecting lanes (l -> L-1-l) and swapping the step parity
    (start at t0 = 1) gives exactly the reflected trajectory; catches any
    left/right asymmetry in the rules (rules are symmetric)."""
    L = 300
    rng = np.random.default_rng(lanes)
    N = int(0.2 * L * lanes)
    flat = np.sort(rng.choice(lanes * L, size=N, replace=False))
    lane, cell = flat // L, flat % L
    v = rng.integers(0, 6, size=N)
    a = oracle.Oracle.from_scenario(make_ring(L, lane, cell, v, lanes=lanes), t0=0)
    b = oracle.Oracle.from_scenario(make_ring(L, lanes - 1 - lane, cell, v, lanes=lanes), t0=1)
    changes = 0
    for t in range(200):
        a.step(1)
        b.step(1)
        sa, sb = a.vehicles(), b.vehicles()
        np.testing.assert_array_equal(sa["lane"], lanes - 1 - sb["lane"])
        np.testing.assert_array_equal(sa["cell"], sb["cell"])
        np.testing.assert_array_equal(sa["v"], sb["v"])
        changes += a.counters()["lane_changes"]
    assert changes > 0


def _lane_flows(L, lanes, rho, steps=1500, warm=500, seed=2):
    rng = np.random.default_rng(seed)
    N = int(round(rho * L * lanes))
    flat = np.sort(rng.choice(lanes * L, size=N, replace=False))
    s = make_ring(L, flat // L, flat % L, rng.integers(0, 6, N), lanes=lanes, p_slow=0.2, seed=seed)
    o = oracle.Oracle.from_scenario(s)
    o.step(warm)
    q = np.zeros(lanes)
    lc = 0
    for _ in range(steps):
        o.step(1)
        st = o.vehicles()
        np.add.at(q, st["lane"], st["v"])
        lc += o.counters()["lane_changes"]
        assert o.counters()["collisions"] == 0
    return q / (steps * L), lc / (steps * N)


def test_lane_usage_symmetric_and_capacity():
    """per-lane flows equal within 10 %; 3-lane total flow
    >= 2.5 x 1-lane flow at the same density"""
    q3, lc_rate = _lane_flows(1000, 3, 0.15)
    assert q3.max() / q3.min() < 1.10
    q1, _ = _lane_flows(1000, 1, 0.15)
    assert q3.sum() >= 2.5 * q1.sum()
    assert 0 < lc_rate < 0.02


def _turn_net(place_lane, place_cell, v, second_link):
    # plus-shaped intersection: centre C(0,0); arms 1 km (133 cells)
    nodes = [(0, 0), (1000, 0), (-1000, 0), (0, 1000), (0, -1000)]
    links = [(2, 0, 1000, 2, 1),  # 0: W->C eastbound (major)
             (0, 1, 1000, 2, 1),  # 1: C->E
             (1, 0, 1000, 2, 1),  # 2: E->C westbound (major)
             (0, 2, 1000, 2, 1),  # 3: C->W
             (4, 0, 1000, 2, 0),  # 4: S->C northbound (minor)
             (0, 3, 1000, 2, 0),  # 5: C->N
             (3, 0, 1000, 2, 0),  # 6: N->C
             (0, 4, 1000, 2, 0)]  # 7: C->S
    veh = [dict(route=[0, second_link], place=(place_lane, place_cell, v))]
    return make_network(nodes, links, veh)


def test_turn_types():
    o = oracle.Oracle.from_scenario(_turn_net(0, 10, 0, 1))
    assert o.turn_type(0, 1) == 0  # straight
    assert o.turn_type(0, 5) == 1  # east then north: left
    assert o.turn_type(0, 7) == 2  # east then south: right
    assert o.turn_type(0, 3) == 1  # U-turn counts as left (R7)
    assert o.turn_type(4, 1) == 2  # north then east: right


def test_spec_lane_change_examples():
    """SPEC.md:122-124"""
    # single vehicle on a 1-lane link: unchanged lane
    o = oracle.Oracle.from_scenario(make_ring(50, [0], [5], [0], lanes=1))
    o.step(1)
    assert o.vehicles()["lane"][0] == 0
    # needs a left turn, in the right lane, target neighbourhood empty:
    # moves left one lane on a step with dir = +1 (t even), same cell
    o = oracle.Oracle.from_scenario(_turn_net(0, 20, 0, 5))
    o.step(1)
    st = o.vehicles()
    assert st["lane"][0] == 1 and st["cell"][0] == 21  # then moved 1 (v 0 -> 1)
    # needs a right turn, in the left lane: moves right on a step with dir = -1
    o = oracle.Oracle.from_scenario(_turn_net(1, 20, 0, 7))
    o.step(1)
    assert o.vehicles()["lane"][0] == 1  # t = 0: dir +1 points away
    o.step(1)
    assert o.vehicles()["lane"][0] == 0
    # blocked ahead (gap 0), adjacent lane gap >= v+1 ahead, >= vmax behind
    s = make_ring(60, [0, 0], [10, 11], [2, 0], lanes=2)
    o = oracle.Oracle.from_scenario(s)
    o.step(1)
    assert o.vehicles()["lane"][0] == 1
    # same, but a vehicle 3 cells behind in the target lane: no change
    s = make_ring(60, [0, 0, 1], [10, 11, 7], [2, 0, 0], lanes=2)
    o = oracle.Oracle.from_scenario(s)
    o.step(1)
    assert o.vehicles()["lane"][0] == 0


def test_desperation_schedule():
    """reading R6: the accepted gap shrinks linearly over the last D = 10
    cells; at d = 0 a wrong-lane vehicle changes into any free cell"""
    n = 133
    # left-turner at the stop line in lane 0, a vehicle directly behind in
    # lane 1 (backward gap 0): at d = 0 the required gaps are (0, 0)
    nodes = [(0, 0), (1000, 0), (-1000, 0), (0, 1000), (0, -1000)]
    links = [(2, 0, 1000, 2, 1), (0, 1, 1000, 2, 1), (1, 0, 1000, 2, 1), (0, 2, 1000, 2, 1),
             (4, 0, 1000, 2, 0), (0, 3, 1000, 2, 0), (3, 0, 1000, 2, 0), (0, 4, 1000, 2, 0)]
    veh = [dict(route=[0, 5], place=(0, n - 1, 0)), dict(route=[0, 1], place=(1, n - 2, 0))]
    o = oracle.Oracle.from_scenario(make_network(nodes, links, veh))
    o.step(1)
    assert o.vehicles()["lane"][0] == 1
    # at d = 20 the full gap is required: a vehicle 2 behind blocks the change
    veh = [dict(route=[0, 5], place=(0, n - 21, 0)), dict(route=[0, 1], place=(1, n - 23, 0))]
    o = oracle.Oracle.from_scenario(make_network(nodes, links, veh))
    o.step(1)
    assert o.vehicles()["lane"][0] == 0
