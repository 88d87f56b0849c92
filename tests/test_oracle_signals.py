"""Oracle pins for signalized intersections (PAPER.md:351-353,
"putting a virtual vehicle of maximum velocity zero at the end of the lane
when the traffic light is red"; reading R23 in DESIGN.md §3):

* SPEC.md:138-140 hand examples (red: the gap ends at the blocker; green:
  the vehicle leaves);
* an always-green signal on a single approach is exactly the unsignalized
  node (the blocker is never placed);
* green time 0 passes nothing;
* 30 s / 30 s throughput = 0.5 x the saturation flow of the same approach
  always green, within 10 % (Fig. 4d, acceptance #4);
* conservation, no collisions and domain-count invariance with signals on
  a grid."""
import numpy as np
import pytest

import oracle
import scenarios
from tests._ref import make_network

CHAIN_NODES = [(0, 0), (750, 0), (1500, 0)]
CHAIN_LINKS = [(0, 1, 750, 1, 1), (1, 2, 750, 1, 1)]  # 100 cells each, one lane


def chain(vehicles, sig=None, p=0.0):
    s = make_network(CHAIN_NODES, CHAIN_LINKS, vehicles, p_slow=p, seed=7)
    if sig is not None:
        g0, g1, off = sig
        s = scenarios.with_signals(s, nodes=[1], green0=g0, green1=g1, offset=off)
    return s


def test_red_blocker_limits_gap():
    """red, vehicle 3 cells from the link end with v = 3 ->
    gap 2 (blocker beyond the last cell), v becomes 2"""
    s = chain([dict(route=[0, 1], place=(0, 97, 3))], sig=(30, 30, 30))  # t=0: red
    o = oracle.Oracle.from_scenario(s)
    o.step(1)
    v = o.vehicles()
    assert v["link"][0] == 0 and v["cell"][0] == 99 and v["v"][0] == 2


def test_green_lets_the_vehicle_leave():
    """green, same state -> the vehicle crosses the node"""
    s = chain([dict(route=[0, 1], place=(0, 97, 3))], sig=(30, 30, 0))  # t=0: green
    o = oracle.Oracle.from_scenario(s)
    o.step(1)
    v = o.vehicles()
    # gap = min(5, d + E) = 5, v = min(3 + 1, 5) = 4: 2 cells to the end, 2 on
    assert v["link"][0] == 1 and v["cell"][0] == 1 and v["v"][0] == 4


def passed(o):
    """vehicles past the signal: arrived, or on the downstream link"""
    v = o.vehicles()
    return int(np.sum((v["status"] == oracle.ARRIVED) |
                      ((v["status"] == oracle.ACTIVE) & (v["link"] == 1))))


def queue_discharge(sig, window, p=0.2):
    """vehicles through the signal in `window` steps from a standing queue:
    the upstream link (400 cells) completely filled with stopped vehicles at
    t = 0, no further arrivals; the queue outlasts the window"""
    nodes = [(0, 0), (3000, 0), (3750, 0)]
    links = [(0, 1, 3000, 1, 1), (1, 2, 750, 1, 1)]
    veh = [dict(route=[0, 1], place=(0, c, 0)) for c in range(400)]
    s = make_network(nodes, links, veh, p_slow=p, seed=7)
    if sig is not None:
        s = scenarios.with_signals(s, nodes=[1], green0=sig[0], green1=sig[1], offset=sig[2])
    o = oracle.Oracle.from_scenario(s)
    o.step(window)
    v = o.vehicles()
    assert np.sum((v["status"] == oracle.ACTIVE) & (v["link"] == 0)) > 0  # still queued
    return passed(o)


def test_always_green_equals_unsignalized():
    """the blocker is never placed -> identical trajectories"""
    veh = [dict(route=[0, 1], depart=int(i // 3), entry=int(i % 7)) for i in range(300)]
    a = oracle.Oracle.from_scenario(chain(veh, p=0.2))
    b = oracle.Oracle.from_scenario(chain(veh, sig=(60, 0, 0), p=0.2))
    assert a.run_hashes(400) == b.run_hashes(400)


def test_zero_green_passes_nothing():
    assert queue_discharge((0, 60, 0), 600) == 0


@pytest.mark.parametrize("p", [0.0, 0.2])
def test_half_green_half_saturation_flow(p):
    """Fig. 4d / SPEC acceptance #4: 30 s / 30 s -> 0.5 x the saturation flow
    (discharge rate of a standing queue, always green) +- 10 %"""
    sat = queue_discharge((60, 0, 0), 480, p=p) / 480
    half = queue_discharge((30, 30, 0), 960, p=p) / 960
    assert sat > 0.25
    assert 0.45 <= half / sat <= 0.55, (half, sat)


def test_signalized_grid_conservation_and_domains():
    """signals at every node of config 1: no collisions, conservation, and
    the k-domain emulation equals the undivided run"""
    s = scenarios.with_signals(scenarios.config("1"), seed=3)
    o1 = oracle.Oracle.from_scenario(s)
    h1 = o1.run_hashes(250)
    c = o1.counters()
    assert c["collisions"] == 0
    assert c["active"] + c["pending"] + c["arrived"] == s.n_vehicles
    for k in (2, 4):
        ok = oracle.Oracle.from_scenario(s)
        ok.set_partition_k(k, np.arange(s.n_nodes, dtype=np.int32) % k)
        assert ok.run_hashes(250) == h1


def test_signal_input_errors():
    s = chain([dict(route=[0, 1], place=(0, 5, 0))])
    bad = scenarios.with_signals(s, nodes=[1], green0=0, green1=0, offset=0)
    with pytest.raises(Exception):
        oracle.Oracle.from_scenario(bad)
    bad = scenarios.with_signals(s, nodes=[7], green0=30, green1=30, offset=0)
    with pytest.raises(Exception):
        oracle.Oracle.from_scenario(bad)
