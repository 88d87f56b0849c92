"""Pin: partition invariance of the oracle's k-domain emulation
(PAPER.md:369-411 domain decomposition with split links, update sequence
PAPER.md:412-427; "cell-by-cell simulation state at every
time step is identical for all p >= 1").  The emulated domains see only
their own cells plus the 5-cell strips received in the two exchanges;
every other cell is poisoned and a read of it is counted."""
import numpy as np
import pytest

import oracle
import scenarios


def stripes(x, k):
    """vertical stripes of equal node count (a simple geometric partition)"""
    order = np.argsort(x, kind="stable")
    d = np.empty(x.size, np.int32)
    d[order] = (np.arange(x.size) * k) // x.size
    return d


@pytest.fixture(scope="module")
def grid6():
    return scenarios.grid_trips(rows=6, cols=6, n_veh=800, depart_max=200, steps=400,
                                name="grid6")


def _compare(scn, partition_fn, steps, k, full_every=25):
    a = oracle.Oracle.from_scenario(scn)
    b = oracle.Oracle.from_scenario(scn)
    b.set_partition_k(k, partition_fn())
    for t in range(steps):
        a.step(1)
        b.step(1)
        assert a.state_hash() == b.state_hash(), f"t={t + 1}"
        if t % full_every == 0:
            va, vb = a.vehicles(), b.vehicles()
            for key in va:
                np.testing.assert_array_equal(va[key], vb[key], err_msg=key)
    ds = b.domain_stats()
    assert ds[0, 3] == 0, "a domain read a cell it cannot see"
    assert b.counters()["collisions"] == 0
    return a, b


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_grid_random_partition(grid6, k):
    rng = np.random.default_rng(k)
    dom = rng.integers(0, k, size=grid6.n_nodes)
    dom[:k] = np.arange(k)
    _compare(grid6, lambda: dom, 400, k)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_grid_stripes(grid6, k):
    _compare(grid6, lambda: stripes(grid6.node_x, k), 400, k)


@pytest.mark.parametrize("k", [2, 4, 8])
def test_ring_cuts(k):
    r = scenarios.ring(n_cells=400, lanes=3, density=0.2, seed=3, steps=200)
    _compare(r, lambda: np.zeros(1, np.int32), 300, k)


def test_repartition_mid_run(grid6):
    """re-partitioning during the run (SURVEY G1 rebalancing) never changes
    the trajectory"""
    a = oracle.Oracle.from_scenario(grid6)
    b = oracle.Oracle.from_scenario(grid6)
    b.set_partition_k(2, stripes(grid6.node_x, 2))
    rng = np.random.default_rng(0)
    for t in range(300):
        if t % 60 == 59:
            k = int(rng.integers(1, 6))
            d = rng.integers(0, k, size=grid6.n_nodes)
            d[:k] = np.arange(k)
            b.set_partition_k(k, d)
        a.step(1)
        b.step(1)
        assert a.state_hash() == b.state_hash()


def test_message_count(grid6):
    """one message per ordered neighbour pair per exchange, two exchanges
    per step"""
    k = 4
    d = stripes(grid6.node_x, k)
    b = oracle.Oracle.from_scenario(grid6)
    b.set_partition_k(k, d)
    b.step(1)
    pairs = set()
    for f, t in zip(grid6.link_from, grid6.link_to):
        if d[f] != d[t]:
            pairs.add((d[f], d[t]))
            pairs.add((d[t], d[f]))
    assert b.domain_stats()[:, 1].sum() == 2 * len(pairs)


def test_spec_acceptance_1_prefix():
    """SPEC.md:638 (acceptance 1) on a 600 s prefix: 10x10 grid, 2,000
    vehicles, p in {2, 4, 8} identical to p = 1"""
    scn = scenarios.grid_trips(rows=10, cols=10, n_veh=2000, depart_max=300, steps=600,
                               name="grid10")
    for k in (2, 4, 8):
        _compare(scn, lambda: stripes(scn.node_x + scn.node_y // 7, k), 600, k, full_every=200)
