"""Pins for the oracle's network parts: discretisation (R1, R11),
intersections with priority and gap acceptance (R8-R10),
parking entry / exit (R12, R13), whole-step invariants
(SPEC.md:162-168)."""
import numpy as np
import pytest

import oracle
import scenarios
from tests._ref import make_network

PLUS_NODES = [(0, 0), (1000, 0), (-1000, 0), (0, 1000), (0, -1000)]
PLUS_LINKS = [(2, 0, 1000, 2, 1),  # 0: W->C eastbound (major)
              (0, 1, 1000, 2, 1),  # 1: C->E
              (1, 0, 1000, 2, 1),  # 2: E->C westbound (major)
              (0, 2, 1000, 2, 1),  # 3: C->W
              (4, 0, 1000, 2, 0),  # 4: S->C northbound (minor)
              (0, 3, 1000, 2, 0),  # 5: C->N
              (3, 0, 1000, 2, 0),  # 6: N->C
              (0, 4, 1000, 2, 0)]  # 7: C->S
N = 133  # 1000 m / 7.5 m rounded


def plus(veh, p=0.0):
    return oracle.Oracle.from_scenario(make_network(PLUS_NODES, PLUS_LINKS, veh, p_slow=p))


def chain_net(lengths_m):
    nodes = [(1000.0 * i, 0.0) for i in range(len(lengths_m) + 1)]
    links = [(i, i + 1, L, 1, 0) for i, L in enumerate(lengths_m)]
    return nodes, links


@pytest.mark.parametrize("length_m,cells", [(75.0, 10), (500.0, 67), (750.0, 100),
                                            (78.74, 10), (78.75, 11), (3000.0, 400)])
def test_cell_count(length_m, cells):
    """R1: n = round-half-up(length / 7.5 m) (SPEC.md:52 example 75 m -> 10;
    config 1: 500 m -> 67)"""
    nodes, links = chain_net([length_m])
    o = oracle.Oracle.from_scenario(make_network(nodes, links, []))
    assert o.n_cells(0) == cells


def test_invalid_networks():
    nodes, links = chain_net([7.5])
    with pytest.raises(oracle.OracleError, match="R11"):
        oracle.Oracle.from_scenario(make_network(nodes, links, []))
    with pytest.raises(oracle.OracleError, match="dangling"):
        oracle.Oracle.from_scenario(make_network([(0, 0)], [(0, 5, 100, 1, 0)], []))
    with pytest.raises(oracle.OracleError, match="non-positive"):
        oracle.Oracle.from_scenario(make_network([(0, 0), (1, 0)], [(0, 1, 0, 1, 0)], []))


def test_gap_acceptance_spec_examples():
    """SPEC.md:149-151 with G = 5: a minor-street vehicle at the stop line
    enters iff the last 5 cells of every major approach are empty"""
    minor = dict(route=[4, 5], place=(0, N - 1, 0))
    # empty priority street -> accepted
    o = plus([minor])
    o.step(1)
    st = o.vehicles()
    assert (st["link"][0], st["lane"][0], st["cell"][0], st["v"][0]) == (5, 0, 0, 1)
    # major vehicle 2 cells upstream of the stop line -> rejected
    o = plus([minor, dict(route=[0, 1], place=(0, N - 3, 0))])
    o.step(1)
    assert (o.vehicles()["link"][0], o.vehicles()["cell"][0]) == (4, N - 1)
    # major vehicle 6 cells upstream -> accepted
    o = plus([minor, dict(route=[0, 1], place=(0, N - 7, 0))])
    o.step(1)
    assert o.vehicles()["link"][0] == 5


def test_priority_one_winner_per_target_lane():
    """two majors (eastbound and westbound) both turning into C->N lane:
    one winner per target lane by (class, link id, lane) (R9)"""
    a = dict(route=[0, 5], place=(1, N - 1, 0))  # eastbound left turn -> lane 1
    b = dict(route=[2, 5], place=(0, N - 1, 0))  # westbound right turn -> lane 0
    c = dict(route=[2, 5], place=(1, N - 1, 0))  # westbound, lane 1, R -> lane 0
    o = plus([a, b, c])
    o.step(1)
    st = o.vehicles()
    assert st["link"][0] == 5 and st["lane"][0] == 1  # link 0 wins lane 1
    assert st["link"][1] == 5 and st["lane"][1] == 0  # (2, lane 0) wins lane 0
    assert st["link"][2] == 2  # (2, lane 1) loses lane 0 to (2, lane 0)


def test_entry_space_limits_crossing():
    """E = consecutive empty cells at the start of the target lane: the
    entrant lands at an index < E (R10)"""
    veh = [dict(route=[0, 1], place=(0, N - 1, 4)), dict(route=[1], place=(0, 2, 0))]
    o = plus(veh)
    o.step(1)
    st = o.vehicles()
    assert st["link"][0] == 1 and st["cell"][0] <= 1
    # blocked entirely: first cell of the target lane occupied
    veh = [dict(route=[0, 1], place=(0, N - 1, 4)), dict(route=[1], place=(0, 0, 0))]
    o = plus(veh)
    o.step(1)
    assert o.vehicles()["link"][0] == 0


def test_crossing_keeps_velocity():
    """R14: a crossing vehicle keeps v3; the next step clamps by min(v+1, V)"""
    veh = [dict(route=[0, 1], place=(0, N - 3, 4))]
    o = plus(veh)
    o.step(1)
    st = o.vehicles()
    assert (st["link"][0], st["cell"][0], st["v"][0], st["cursor"][0]) == (1, 2, 5, 1)


def test_injection_spec_examples():
    """SPEC.md:158-160"""
    nodes, links = chain_net([300.0, 300.0])
    n0 = 40
    veh = [dict(route=[0, 1], depart=10, entry=7),
           dict(route=[0, 1], depart=10, entry=7),
           dict(route=[1], place=(0, n0 - 3, 5))]
    o = oracle.Oracle.from_scenario(make_network(nodes, links, veh))
    o.step(9)
    assert o.vehicles()["status"][0] == oracle.PENDING
    o.step(1)  # S(10): vehicle 0 present at its entry cell, v = 0
    st = o.vehicles()
    assert (st["status"][0], st["cell"][0], st["v"][0]) == (oracle.ACTIVE, 7, 0)
    assert st["status"][1] == oracle.PENDING  # same cell taken: retry
    # final-link vehicle reached the end: removed
    assert st["status"][2] == oracle.ARRIVED
    o.step(1)  # vehicle 0 moved on (v 0 -> 1), vehicle 1 enters at t = 11
    st = o.vehicles()
    assert st["status"][1] == oracle.ACTIVE and st["cell"][1] == 7
    assert st["cell"][0] == 8
    c = o.counters()
    assert (c["active"], c["arrived"], c["pending"]) == (2, 1, 0)


def test_minor_blocked_while_major_jammed():
    """minor throughput is 0 while the priority street is
    bumper-to-bumper (here: the major approach is jammed because its exit
    link C->E is packed), and positive once it clears"""
    exitjam = [dict(route=[1, 2], place=(ln, x, 0)) for ln in (0, 1) for x in range(N)]
    major = [dict(route=[0, 1], place=(ln, N - 1 - i, 0)) for ln in (0, 1) for i in range(30)]
    minor = [dict(route=[4, 5], place=(0, N - 1, 0))]
    o = plus(minor + major + exitjam, p=0.2)
    first = None
    for t in range(600):
        o.step(1)
        if o.vehicles()["link"][0] == 5 and first is None:
            first = t
    assert first is not None and first > 100


@pytest.fixture(scope="module")
def cfg1():
    return scenarios.config("1")


def test_config1_invariants(cfg1):
    """conservation active + pending + arrived = total, no collision,
    velocity bounds, every step of 600"""
    o = oracle.Oracle.from_scenario(cfg1)
    nv = cfg1.n_vehicles
    for t in range(600):
        o.step(1)
        c = o.counters()
        assert c["active"] + c["pending"] + c["arrived"] == nv
        assert c["collisions"] == 0
        st = o.vehicles()
        act = st["status"] == oracle.ACTIVE
        assert ((st["v"][act] >= 0) & (st["v"][act] <= 5)).all()
        keys = st["link"][act].astype(np.int64) * 10**6 + st["lane"][act] * 10**4 + st["cell"][act]
        assert np.unique(keys).size == act.sum()
    assert c["arrived"] == nv  # the 4x4 grid drains


def test_determinism(cfg1):
    a = oracle.Oracle.from_scenario(cfg1)
    b = oracle.Oracle.from_scenario(cfg1)
    assert a.run_hashes(200) == b.run_hashes(200)
    c = oracle.Oracle.from_scenario(cfg1, seed=2)
    d = oracle.Oracle.from_scenario(cfg1)
    assert c.run_hashes(50) != d.run_hashes(50)
