"""GPU parity of the domain-decomposed step (§4; G1, H2, H7): k
domains of a node partition, each a libtsim handle on the same GPU,
exchanging their boundary strips twice per step, must reproduce the
undivided CPU oracle bit for bit (results do not depend on the
partition).  Also: restore at time t and mid-run repartitioning."""
import numpy as np
import pytest

import oracle
import scenarios

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")
from paper_cs_0105004_b200 import domains  # noqa: E402

FUSED = tsim.FLAG_FUSED | tsim.FLAG_HASH


def assert_same(vo, vg, msg):
    for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
        bad = np.nonzero(vo[key] != vg[key])[0]
        assert bad.size == 0, (f"{msg} {key}: {bad.size} mismatches, first vid {bad[:5]} "
                               f"oracle {vo[key][bad[:5]]} gpu {vg[key][bad[:5]]}")


def run_domains(scn, k, steps, chunk=10, dom=None, flags=FUSED, **kw):
    o = oracle.Oracle.from_scenario(scn)
    d = domains.LocalDomains(scn, k, dom, flags=flags, **kw)
    assert d.state_hash() == o.state_hash()
    assert_same(o.vehicles(), d.vehicles(), "init")
    done = 0
    while done < steps:
        n = min(chunk, steps - done)
        t_from = o.t + 1
        oh = o.run_hashes(n)
        d.step(n)
        done += n
        assert d.t == o.t
        gh = d.history(t_from, n)["hash"]
        bad = [t_from + i for i in range(n) if gh[i] != oh[i]]
        assert not bad, f"k={k}: per-step hash differs at t={bad[:5]}"
    assert_same(o.vehicles(), d.vehicles(), f"k={k} t={o.t}")
    return o, d


@pytest.mark.parametrize("k", [2, 3, 4, 8])
def test_config1_orb(k):
    """BASELINE.json configs[0]: ORB partitions, 300 steps"""
    run_domains(scenarios.config("1"), k, 300)


@pytest.mark.parametrize("seed", [1, 2])
def test_random_partition(seed):
    """random node -> domain maps: many split links, domains with several
    neighbours, non-contiguous domains"""
    s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=200, seed=7, name="grid6d")
    rng = np.random.default_rng(seed)
    dom = rng.integers(0, 5, s.n_nodes).astype(np.int32)
    dom[:5] = np.arange(5)
    run_domains(s, 5, 250, chunk=25, dom=dom)


def test_dense_grid_lane_changes():
    """config-4a recipe on a 20x20 lattice, 4 domains: heavy lane changing
    next to the cuts (lane change reads the mirrors of exchange #2)"""
    s = scenarios.big_grid(rows=20, cols=20, seed=4, name="grid20dense")
    run_domains(s, 4, 120, chunk=40)


def test_portland_mixed_tiles():
    """Portland-shaped network: long links (several tiles) and short links
    (row kernel) on both sides of cuts"""
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64, seed=2)
    s.depart = (s.depart // 12).astype(np.int32)
    run_domains(s, 4, 200, chunk=50, tile_cells=64)


@pytest.mark.parametrize("k", [3, 6])
def test_multilevel_partition(k):
    """the multilevel partitioner's domains (irregular, few split links)"""
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64, seed=5)
    s.depart = (s.depart // 12).astype(np.int32)
    run_domains(s, k, 200, chunk=40, dom=domains.partition(s, k, method="multilevel"))


def test_restore_is_exact():
    """read S(t), restore into a fresh handle, continue: identical to the
    uninterrupted run (checkpoint / migration primitive)"""
    s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=8, name="grid6r")
    o = oracle.Oracle.from_scenario(s)
    g = tsim.Sim.from_scenario(s, flags=FUSED)
    g.step(120)
    o.step(120)
    state = g.vehicles()
    g.close()
    r = tsim.Sim(p_slow=s.p_slow, seed=s.seed, flags=FUSED)
    r.load(s, place=False)
    domains.restore_into(r, state, 120)
    assert r.state_hash() == o.state_hash()
    o.step(150)
    r.step(150)
    assert r.state_hash() == o.state_hash()
    assert_same(o.vehicles(), r.vehicles(), "restored t=270")


def test_repartition_mid_run():
    """adaptive rebalancing: k=2 by geometry, then k=4
    with weights from the measured per-link work; the trajectory is
    unchanged"""
    s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=9, name="grid6m")
    o = oracle.Oracle.from_scenario(s)
    d = domains.LocalDomains(s, 2, flags=FUSED | tsim.FLAG_LINK_WORK)
    d.step(100)
    o.step(100)
    assert d.state_hash() == o.state_hash()
    w = domains.node_weights(s, d.link_work())
    d.repartition(domains.partition(s, 4, w), k=4)
    assert d.state_hash() == o.state_hash()
    o.step(150)
    d.step(150)
    assert d.state_hash() == o.state_hash()
    assert_same(o.vehicles(), d.vehicles(), "after repartition")


def test_bad_domain_inputs():
    s = scenarios.config("1")
    g = tsim.Sim(p_slow=s.p_slow, seed=s.seed)
    g.load(s)
    with pytest.raises(tsim.TsError):
        g.set_domain(0, np.zeros(s.n_nodes, np.int32), 0)
    with pytest.raises(tsim.TsError):
        g.set_domain(2, np.full(s.n_nodes, 5, np.int32), 0)
    with pytest.raises(tsim.TsError):
        g.set_domain(s.n_nodes + 1, np.zeros(s.n_nodes, np.int32), 0)
    r = scenarios.ring(n_cells=500, lanes=2, density=0.2, seed=1)
    g2 = tsim.Sim(p_slow=r.p_slow, seed=r.seed)
    g2.load(r)
    with pytest.raises(tsim.TsError):
        g2.set_domain(2, np.zeros(r.n_nodes, np.int32), 0)


@pytest.mark.parametrize("k", [2, 4])
def test_signalized_grid_domains(k):
    """signals at every node of config 1, k ORB domains: identical to the
    undivided oracle (signal state is a function of t and the node only)"""
    s = scenarios.with_signals(scenarios.config("1"), seed=5)
    run_domains(s, k, 200, chunk=50)


def test_adaptive_rebalance_from_measured_times():
    """PAPER.md:730-735 / BASELINE config 5: every 60 steps the partition is
    recomputed from the measured per-domain device time apportioned to the
    links by their work; trips concentrated in one half of the network make
    the first partition unbalanced.  The run stays bit-exact with the
    undivided oracle across the migrations, and the load (measured link
    time) of the heaviest domain drops after the first rebalance."""
    s = scenarios.grid_trips(rows=8, cols=8, n_veh=6000, depart_max=100, seed=12,
                             name="grid8rebal", od_cols=(0, 3))
    o = oracle.Oracle.from_scenario(s)
    d = domains.LocalDomains(s, 4, flags=FUSED | tsim.FLAG_LINK_WORK)
    e_before = e_after = None
    for r in range(3):
        t_from = o.t + 1
        oh = o.run_hashes(60)
        d.step(60)
        gh = d.history(t_from, 60)["hash"]
        assert list(gh) == list(oh), f"round {r}"
        lw = [x.link_work() for x in d.sims]
        dom_old = d.dom.copy()
        new, ms = d.rebalance()
        lt = domains.link_times(lw, ms)
        load_old = np.bincount(dom_old[np.asarray(s.link_from)], weights=lt, minlength=4)
        load_new = np.bincount(np.asarray(new)[np.asarray(s.link_from)], weights=lt, minlength=4)
        if r == 0:
            e_before = load_old.mean() / load_old.max()
            e_after = load_new.mean() / load_new.max()
    assert e_after > e_before
    assert_same(o.vehicles(), d.vehicles(), "after rebalancing")


def test_ts_partition_matches_orb():
    """ts_partition: ORB of the handle's own network with the paper's node
    weights, the same partition as domains.partition, and the handle runs
    as that domain"""
    s = scenarios.config("1")
    g = tsim.Sim(p_slow=s.p_slow, seed=s.seed, flags=FUSED)
    g.load(s)
    dom = g.partition(4, 2)
    assert np.array_equal(dom, domains.partition(s, 4))
    g.init(0)
    assert len(g.exchange_plan()) >= 1


def test_load_statistics_links_and_nodes():
    """ts_get_load ("the execution time of each link and
    each intersection"): per-link vehicle updates sum to the vehicle updates
    of the run; per-node work (lanes in range + crossings) covers every
    crossing, is zero at nodes without incoming traffic, and the warp node
    kernel and the thread-per-node kernel count identically; a k-domain
    partition's loads add up to the undivided run's"""
    s = scenarios.config("1")
    flags = FUSED | tsim.FLAG_LINK_WORK
    a = tsim.Sim.from_scenario(s, flags=flags)
    b = tsim.Sim.from_scenario(s, flags=flags | 32)  # TS_FLAG_NODE_GENERAL: k_node
    a.step(150)
    b.step(150)
    lw, nw = a.load_stats()
    lw2, nw2 = b.load_stats()
    assert np.array_equal(lw, lw2) and np.array_equal(nw, nw2)
    h = a.history(0, 150)
    assert lw.sum() == a.totals()["vehicle_updates"] == int(np.sum(h["active"]))
    assert nw.sum() >= int(np.sum(a.history(1, 150)["crossings"])) > 0
    indeg = np.bincount(np.asarray(s.link_to), minlength=s.n_nodes)
    assert np.all(nw[indeg == 0] == 0)
    d = domains.LocalDomains(s, 4, flags=flags)
    d.step(150)
    parts = [x.load_stats() for x in d.sims]
    assert np.array_equal(sum(p[0] for p in parts), lw)
    assert np.array_equal(sum(p[1] for p in parts), nw)


@pytest.mark.parametrize("graph,split", [(False, False), (True, False), (False, True), (True, True)])
def test_local_step_in_library(graph, split, monkeypatch):
    """ts_local_step: whole steps of all k domains enqueued by the library
    (both exchanges per step), and with FLAG_GRAPH replayed from one CUDA
    graph holding every domain's stream and the exchanges: per-step hash
    equal to the undivided oracle for 300 steps in chunks of 7, 15, 31, 45
    steps (graph blocks + remainders); the phase-by-phase driver gives the
    same state.  split: the direct strip delivery as one kernel per
    receiving domain (TSIM_DIRECT_SPLIT, the structure of the multi-device
    peer-pointer transport: one kernel per receiving device) instead of one
    per exchange"""
    if split:
        monkeypatch.setenv("TSIM_DIRECT_SPLIT", "1")
    else:
        monkeypatch.delenv("TSIM_DIRECT_SPLIT", raising=False)
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64, seed=2)
    s.depart = (s.depart // 12).astype(np.int32)
    s = scenarios.with_signals(s, green0=20, green1=25, seed=4)
    flags = FUSED | (tsim.FLAG_GRAPH if graph else 0)
    o = oracle.Oracle.from_scenario(s)
    d = domains.LocalDomains(s, 8, flags=flags)
    p = domains.LocalDomains(s, 8, flags=FUSED)
    for chunk in (7, 15, 31, 45, 7, 15, 31, 45, 104):
        t_from = o.t + 1
        oh = o.run_hashes(chunk)
        d.step(chunk)
        p.step_phases(chunk)
        gh = d.history(t_from, chunk)["hash"]
        bad = [t_from + i for i in range(chunk) if gh[i] != oh[i]]
        assert not bad, f"per-step hash differs at t={bad[:5]}"
        assert d.state_hash() == p.state_hash() == o.state_hash()
    assert_same(o.vehicles(), d.vehicles(), "after 300 steps")
