"""The paper's performance model (SURVEY
§8(f) N2): closed forms and limits the paper states, and the partition
statistics checked by hand on the 4x4 grid."""
import math

import numpy as np
import pytest

import scenarios
from paper_cs_0105004_b200 import domains, perfmodel as pm


def test_n_nb_model_limits():
    # n_nb(1) = 0, n_nb -> 6 for p -> infinity
    assert pm.n_nb_model(1) == 0.0
    assert pm.n_nb_model(4) == pytest.approx(2.5)      # 2 (6-1)(2-1) / 4
    assert pm.n_nb_model(16) == pytest.approx(4.125)   # 2 (12-1)(4-1) / 16
    assert pm.n_nb_model(1e12) == pytest.approx(6.0, rel=1e-5)
    assert all(pm.n_nb_model(p) < pm.n_nb_model(p + 1) for p in range(1, 200))


def test_n_spl_fit():
    # 140 p^0.59 - 140, zero split links on one CPU
    assert pm.n_spl_fit(1) == 0.0
    assert pm.n_spl_fit(16) == pytest.approx(140 * 16 ** 0.59 - 140)


def test_switched_latency_saturation():
    # switched network (b_net = inf): T(p) -> N_sub * 6 * T_lt = 9.6 ms, the
    # latency term dominates
    c = pm.paper_params()
    big = pm.predict(0.25, [10 ** 8], c)[0]
    assert big.T == pytest.approx(2 * 6 * 0.8e-3, rel=2e-2)
    assert big.T_lat / big.T > 0.97
    # T(1) has no communication and rtr = 1 s / T
    one = pm.predict(0.25, [1], c)[0]
    assert one.T == 0.25 and one.T_lat == one.T_bnd == one.T_net == 0.0
    assert one.rtr == pytest.approx(4.0)


def test_bus_topology_grows_like_sqrt_p():
    # shared network (finite b_net): the N_spl * S_bnd / b_net term takes
    # over, T(p) ~ N_spl(p) -- sqrt(p) in the paper's geometric argument
    # (:945-961), p^0.59 with its own N_spl fit (:1003-1004)
    c = pm.paper_params()
    c.b_net = 100e6 / 8
    a, b = pm.predict(0.25, [10 ** 6, 4 * 10 ** 6], c)
    assert b.T / a.T == pytest.approx(4 ** 0.59, rel=0.02)
    assert b.T_net / b.T > 0.95


def test_speedup_efficiency_identities():
    # S(p) = T(1)/T(p), E(p) = S(p)/p, rtr(p) = 1/T(p)
    c = pm.paper_params()
    rows = pm.predict(0.3, [1, 2, 4, 8, 16], c)
    for r in rows:
        assert r.S == pytest.approx(rows[0].T / r.T)
        assert r.E == pytest.approx(r.S / r.p)
        assert r.rtr * r.T == pytest.approx(1.0)
        assert r.T == pytest.approx(r.T_cmp + r.T_lat + r.T_bnd + r.T_net)
    assert rows[0].S == 1.0 and rows[0].E == 1.0


def test_f_dmn_from_e_dmn():
    # f_dmn = 1/e_dmn - 1: e_dmn = 0.5 doubles T_cmp
    c = pm.paper_params()
    a = pm.predict(1.0, [4], c)[0]
    b = pm.predict(1.0, [4], c, e_dmn={4: 0.5})[0]
    assert b.T_cmp == pytest.approx(2 * a.T_cmp)


def test_partition_stats_grid_by_hand():
    # 4x4 grid, two domains of two columns each: the cut crosses one
    # horizontal edge per row, both directions: 8 split links, each domain
    # has one neighbour, equal loads by symmetry
    scn = scenarios.config("1")
    x = np.asarray(scn.node_x)
    dom = (x > np.median(x)).astype(np.int32)
    st = pm.partition_stats(scn, dom)
    assert st["N_spl"] == 8
    assert st["n_nb"] == 1.0
    assert st["e_dmn"] == pytest.approx(1.0)
    # brute force on the same map
    f, t = np.asarray(scn.link_from), np.asarray(scn.link_to)
    assert st["N_spl"] == sum(int(dom[a] != dom[b]) for a, b in zip(f, t))


def test_partition_stats_orb_k4():
    scn = scenarios.config("1")
    dom = domains.partition(scn, 4)
    st = pm.partition_stats(scn, dom)
    assert st["p"] == 4
    assert 0.5 < st["e_dmn"] <= 1.0
    assert 1.0 <= st["n_nb"] <= 3.0
    assert st["N_spl"] == sum(int(dom[a] != dom[b]) for a, b in zip(scn.link_from, scn.link_to))
