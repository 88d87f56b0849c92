"""Partitioners: ORB (the paper's method for its runs)
and the multilevel graph partitioner (the METIS-style
alternative the paper compares with).  Host code: CPU tests."""
import numpy as np
import pytest

import scenarios
import paper_cs_0105004_b200 as tsim
from paper_cs_0105004_b200 import domains


@pytest.fixture(scope="module")
def portland():
    return scenarios.portland(n_nodes=2000, n_edges=2500, n_veh=100, side_km=20.0, n_zones=16,
                              seed=2)


def loads(scn, dom, k):
    w = domains.node_weights(scn)
    out = np.zeros(k)
    np.add.at(out, dom, w)
    return out


@pytest.mark.parametrize("k", [2, 3, 4, 8, 16])
def test_multilevel_valid_balanced(portland, k):
    dom = domains.partition(portland, k, method="multilevel")
    assert dom.shape == (portland.n_nodes,)
    assert set(np.unique(dom)) == set(range(k))
    ld = loads(portland, dom, k)
    assert ld.max() / ld.mean() <= 1.05 + 1e-9, ld


@pytest.mark.parametrize("k", [2, 4, 8])
def test_multilevel_cuts_fewer_links_than_orb(portland, k):
    """the paper's observation: the graph partitioner yields far fewer split
    links than ORB"""
    n_orb, _ = domains.split_stats(portland, domains.partition(portland, k))
    n_ml, _ = domains.split_stats(portland, domains.partition(portland, k, method="multilevel"))
    assert n_ml < n_orb, (n_ml, n_orb)


def test_multilevel_deterministic_and_seeded(portland):
    a = tsim.multilevel_partition(portland, 4, seed=3)
    b = tsim.multilevel_partition(portland, 4, seed=3)
    assert np.array_equal(a, b)


def test_orb_on_grid_is_blocks():
    """ORB of a regular lattice with uniform weights: contiguous blocks"""
    s = scenarios.config("1")
    dom = domains.partition(s, 4)
    g = dom.reshape(4, 4)
    assert len(np.unique(g[:2, :2])) == 1 and len(np.unique(g[2:, 2:])) == 1
    n_spl, pairs = domains.split_stats(s, dom)
    assert n_spl == 16 and len(pairs) == 8


def test_partition_input_errors():
    s = scenarios.config("1")
    with pytest.raises(tsim.TsError):
        tsim.multilevel_partition(s, 0)
    with pytest.raises(tsim.TsError):
        tsim.multilevel_partition(s, s.n_nodes + 1)
    with pytest.raises(tsim.TsError):
        tsim.orb_partition(s.node_x, s.node_y, s.n_nodes + 1)


def test_rebalance_weights_follow_measured_time():
    """link times = each domain's measured time split by its links' work
    (PAPER.md:730-733); a domain twice as slow per unit of work gets twice
    the weight, so ORB moves its boundary towards it"""
    from paper_cs_0105004_b200 import domains
    scn = scenarios.config("1")
    n = scn.n_links
    dom = (np.asarray(scn.node_x) > np.median(scn.node_x)).astype(np.int32)
    own = dom[np.asarray(scn.link_from)]  # work attributed to the from-node's domain
    work = [np.where(own == d, 100, 0) for d in (0, 1)]
    lt = domains.link_times(work, [2.0, 1.0])
    assert lt.sum() == pytest.approx(3.0)
    assert lt[own == 0].sum() == pytest.approx(2.0) and lt[own == 1].sum() == pytest.approx(1.0)
    w = domains.rebalance_weights(scn, work, [2.0, 1.0])
    assert w[dom == 0].sum() > 1.5 * w[dom == 1].sum()
    new = domains.partition(scn, 2, w)
    # the domain holding the slow (left) side now has fewer than half the nodes
    slow = new[int(np.argmin(np.asarray(scn.node_x)))]
    assert np.bincount(new, minlength=2)[slow] < scn.n_nodes // 2


def test_load_times_apportions_domain_time():
    """ts_load_times: a domain's time is split over its
    links and nodes in proportion to their work; the parts sum to the
    domain's time; domains accumulate into one pair of arrays; an idle
    domain adds nothing; negative inputs are rejected"""
    lw = np.array([0, 10, 30, 0, 60], np.int64)
    nw = np.array([0, 50, 50], np.int64)
    lt, nt = tsim.load_times(4.0, lw, nw)
    assert lt.sum() + nt.sum() == pytest.approx(4.0)
    assert lt == pytest.approx(4.0 * lw / 200.0) and nt == pytest.approx(4.0 * nw / 200.0)
    tsim.load_times(2.0, np.array([1, 0, 0, 0, 1], np.int64), np.zeros(3, np.int64), lt, nt)
    assert lt[0] == pytest.approx(1.0) and lt[4] == pytest.approx(1.2 + 1.0)
    before = lt.copy()
    tsim.load_times(7.0, np.zeros(5, np.int64), np.zeros(3, np.int64), lt, nt)
    assert np.array_equal(before, lt)
    with pytest.raises(tsim.TsError):
        tsim.load_times(1.0, np.array([-1, 2], np.int64))
    with pytest.raises(tsim.TsError):
        tsim.load_times(-1.0, np.array([1, 2], np.int64))


def test_rebalance_weights_closed_form():
    """ts_rebalance: node weight = own time + half of every attached link's
    time (+ the floor 1e-3 x total x static share of links), then ORB --
    the same partition as ts_orb_partition of those weights; multilevel is a
    valid k-way partition; bad inputs are rejected"""
    scn = scenarios.config("1")
    rng = np.random.default_rng(3)
    lt = rng.uniform(0, 2, scn.n_links)
    lt[rng.random(scn.n_links) < 0.3] = 0.0
    nt = rng.uniform(0, 0.5, scn.n_nodes)
    dom, w = tsim.rebalance(scn, 4, lt, nt)
    cells = (np.asarray(scn.link_len_mm) + 3750) // 7500
    stat = cells * np.asarray(scn.link_lanes, np.float64)
    fl = 1e-3 * lt.sum() / stat.sum()
    ref = 1e-9 + nt.copy()
    for j in range(scn.n_links):
        ref[scn.link_from[j]] += 0.5 * (lt[j] + fl * stat[j])
        ref[scn.link_to[j]] += 0.5 * (lt[j] + fl * stat[j])
    assert w == pytest.approx(ref, rel=1e-12)
    assert np.array_equal(dom, tsim.orb_partition(scn.node_x, scn.node_y, 4, ref))
    dm, _ = tsim.rebalance(scn, 4, lt, nt, method="multilevel")
    assert set(dm.tolist()) == {0, 1, 2, 3}
    with pytest.raises(tsim.TsError):
        tsim.rebalance(scn, scn.n_nodes + 1, lt)
    with pytest.raises(tsim.TsError):
        tsim.rebalance(scn, 2, -lt - 1.0)
