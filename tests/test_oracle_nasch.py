"""Pins for the oracle's car-following / move step (
readings R2, R3, R12, R15): closed forms, exact results and brute force."""
import numpy as np
import pytest

import oracle
from tests._ref import brake_np, make_ring, nasch_ring_particles, nasch_v1_exact_flow


def ring_flow(L, N, vmax, p, warm, meas, seed=3, lanes=1):
    rng = np.random.default_rng(seed)
    cells = np.sort(rng.choice(L, size=N, replace=False))
    v = rng.integers(0, vmax + 1, size=N)
    s = make_ring(L, np.zeros(N), cells, v, lanes=lanes, vmax=vmax, p_slow=p, seed=seed)
    o = oracle.Oracle.from_scenario(s)
    o.step(warm)
    tot = 0
    for _ in range(meas):
        o.step(1)
        tot += o.counters()["sum_v"]
    return tot / (meas * L)


@pytest.mark.parametrize("rho", [0.05, 0.10, 0.15, 1 / 6, 0.2, 0.3, 0.5, 0.8])
def test_deterministic_fundamental_diagram(rho):
    """p = 0 single-lane ring: steady-state flow q = min(rho*V, 1-rho)
    (north_star; capacity V/(V+1) at rho = 1/(V+1))."""
    L, V = 1200, 5
    N = int(round(rho * L))
    q = ring_flow(L, N, V, 0.0, warm=3000, meas=200)
    expect = min(N / L * V, 1 - N / L)
    assert q == pytest.approx(expect, abs=1e-12)


@pytest.mark.parametrize("p", [0.2, 0.5])
@pytest.mark.parametrize("rho", [0.1, 0.3, 0.5, 0.7])
def test_vmax1_exact_flow(p, rho):
    """vmax = 1, p > 0: q = (1 - sqrt(1 - 4(1-p) rho (1-rho))) / 2, the
    exact stationary flow of the parallel-update NaSch model with vmax = 1."""
    L = 4000
    N = int(round(rho * L))
    q = ring_flow(L, N, 1, p, warm=1000, meas=1500)
    assert abs(q - nasch_v1_exact_flow(N / L, p)) < 4e-3


def test_flow_endpoints():
    """q(0) = 0 and q(1) = 0 exactly"""
    L = 50
    s = make_ring(L, np.zeros(L), np.arange(L), np.zeros(L), p_slow=0.2)
    o = oracle.Oracle.from_scenario(s)
    o.step(20)
    assert o.counters()["sum_v"] == 0
    s = make_ring(L, [], [], [], p_slow=0.2)
    o = oracle.Oracle.from_scenario(s)
    o.step(5)
    assert o.counters()["active"] == 0


@pytest.mark.parametrize("case", range(40))
def test_brute_force_small_rings(case):
    """SPEC acceptance #2: rings <= 30 cells, <= 5 vehicles, 100 steps,
    against an independent particle-list NaSch with the same Philox stream
    (half the cases p = 0, half p = 0.35)."""
    rng = np.random.default_rng(1000 + case)
    L = int(rng.integers(10, 31))
    N = int(rng.integers(1, 6))
    vmax = int(rng.integers(1, 6))
    p = 0.0 if case % 2 == 0 else 0.35
    seed = int(rng.integers(1, 2**40))
    cells = np.sort(rng.choice(L, size=N, replace=False))
    v = rng.integers(0, vmax + 1, size=N)
    s = make_ring(L, np.zeros(N), cells, v, vmax=vmax, p_slow=p, seed=seed)
    o = oracle.Oracle.from_scenario(s)
    ref = nasch_ring_particles(L, cells, v, vmax, 100,
                               lambda t, ids: brake_np(t, ids, seed, p))
    for t in range(100):
        o.step(1)
        st = o.vehicles()
        ids, x, vv = ref[t]
        np.testing.assert_array_equal(st["cell"][ids], x, err_msg=f"t={t}")
        np.testing.assert_array_equal(st["v"][ids], vv, err_msg=f"t={t}")


def test_all_brake_masks():
    """every subset of braking vehicles (2^N masks) for one step matches the
    particle model driven by the same mask"""
    rng = np.random.default_rng(5)
    for trial in range(6):
        L, N = 14, 5
        cells = np.sort(rng.choice(L, size=N, replace=False))
        v = rng.integers(0, 6, size=N)
        for mask in range(2 ** N):
            bits = np.array([(mask >> i) & 1 for i in range(N)], dtype=np.uint8)
            s = make_ring(L, np.zeros(N), cells, v, p_slow=0.5)
            o = oracle.Oracle.from_scenario(s)
            o.set_brake_override(bits)
            o.step(1)
            st = o.vehicles()
            ids, x, vv = nasch_ring_particles(L, cells, v, 5, 1,
                                              lambda t, ids: bits[ids].astype(bool))[0]
            np.testing.assert_array_equal(st["cell"][ids], x)
            np.testing.assert_array_equal(st["v"][ids], vv)


def test_spec_move_examples():
    """SPEC.md:131-133"""
    # v = 0 on an empty road, vmax 5, p = 0 -> v = 1, position + 1
    o = oracle.Oracle.from_scenario(make_ring(100, [0], [10], [0]))
    o.step(1)
    assert (o.vehicles()["v"][0], o.vehicles()["cell"][0]) == (1, 11)
    # v = 4, gap 2, p = 0 -> v = 2, advances 2
    o = oracle.Oracle.from_scenario(make_ring(100, [0, 0], [10, 13], [4, 0]))
    o.step(1)
    assert (o.vehicles()["v"][0], o.vehicles()["cell"][0]) == (2, 12)
    # lone vehicle at v = 5 on an empty ring cruises at 5 cells/step
    o = oracle.Oracle.from_scenario(make_ring(100, [0], [98], [5]))
    for t in range(30):
        o.step(1)
        assert o.vehicles()["v"][0] == 5
    assert o.vehicles()["cell"][0] == (98 + 150) % 100


def test_invariants_long_run():
    """conservation, no collision, cyclic order preservation, 0 <= v <= vmax
     on a 1-lane ring with p = 0.2"""
    L, N = 500, 120
    rng = np.random.default_rng(9)
    cells = np.sort(rng.choice(L, size=N, replace=False))
    o = oracle.Oracle.from_scenario(make_ring(L, np.zeros(N), cells, rng.integers(0, 6, N), p_slow=0.2))
    prev = None
    for t in range(300):
        o.step(1)
        st = o.vehicles()
        assert (st["status"] == oracle.ACTIVE).all()
        assert ((st["v"] >= 0) & (st["v"] <= 5)).all()
        assert np.unique(st["cell"]).size == N
        order = np.argsort(st["cell"])
        k = int(np.nonzero(order == 0)[0][0])
        cyc = np.roll(order, -k)
        if prev is not None:
            np.testing.assert_array_equal(cyc, prev)
        prev = cyc
    assert o.counters()["collisions"] == 0


def test_locality():
    """a vehicle's one-step update depends only on cells within 5 of it
    (PAPER.md:390-395): adding a vehicle changes nobody further away."""
    L = 200
    rng = np.random.default_rng(11)
    cells = np.sort(rng.choice(np.arange(0, 150), size=40, replace=False))
    v = rng.integers(0, 6, size=40)
    a = oracle.Oracle.from_scenario(make_ring(L, np.zeros(40), cells, v, p_slow=0.3))
    b = oracle.Oracle.from_scenario(make_ring(L, np.zeros(41), np.append(cells, 175),
                                              np.append(v, 2), p_slow=0.3))
    a.step(1)
    b.step(1)
    sa, sb = a.vehicles(), b.vehicles()
    far = (cells < 170 - 5) & (cells > (175 + 5) % L)
    np.testing.assert_array_equal(sa["cell"][:40][far], sb["cell"][:40][far])
    np.testing.assert_array_equal(sa["v"][:40][far], sb["v"][:40][far])
    near = ~far
    assert near.sum() >= 0
