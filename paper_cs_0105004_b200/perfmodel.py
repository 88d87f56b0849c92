"""The paper's performance model of the parallel micro-simulation
(§6, :803-1073; speed-up and efficiency :1191-1238), evaluated with
the partition statistics of our own networks.

    T(p)     = T_cmp(p) + T_cmm(p)                                 (:816)
    T_cmp(p) = T_1 / p * (1 + f_ovr(p) + f_dmn(p))                 (:821)
    T_cmm(p) = N_sub * ( n_nb(p) T_lt + N_spl(p)/p * S_bnd/b_nd
                         + N_spl(p) * S_bnd/b_net )                (:888-893)
    n_nb(p)  = 2 (3 sqrt(p) - 1)(sqrt(p) - 1) / p                  (:907-908)
    N_spl(p) = 140 p^0.59 - 140   (20,024-link Portland fit, :1003-1004)
    f_dmn    = 1 / e_dmn - 1,  e_dmn = (total load / p) / max domain load
                                                                   (:827, :645-651)
    rtr(p)   = 1 s / T(p);  S(p) = T(1) / T(p);  E(p) = S(p) / p   (:979-983, :1203, :1233)

Host-side arithmetic only (no simulation): the measured inputs (T_1 from
bench.py, the exchange latency, the actual N_spl / n_nb / e_dmn of a
partition) are passed in.  `partition_stats` computes the actual values for
a partition of one of our networks; `paper_params` holds the paper's
switched 100 Mbit Ethernet parameters (:985-1011).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def n_nb_model(p: float) -> float:
    """neighbour domains per CPU of the paper's geometric argument
    (PAPER.md:907-908): 0 at p = 1, -> 6 as p -> infinity"""
    s = math.sqrt(p)
    return 2.0 * (3.0 * s - 1.0) * (s - 1.0) / p


def n_spl_fit(p: float, a: float = 140.0, b: float = 0.59) -> float:
    """split links of the 20,024-link Portland network under METIS
    """
    return a * p ** b - a


@dataclass
class CommParams:
    """hardware / implementation parameters of T_cmm"""
    T_lt: float            # latency per message [s]
    b_nd: float            # node (point-to-point) bandwidth [B/s]
    S_bnd: float           # bytes per split link per exchange
    N_sub: int = 2         # exchanges per time step
    b_net: float = math.inf  # network bandwidth [B/s]; inf = switched
    name: str = ""


def paper_params() -> CommParams:
    """switched 100 Mbit Ethernet of the paper: T_lt = 0.8 ms, b_nd = 50
    Mbit/s, S_bnd = 200 B, N_sub = 2, b_net negligible"""
    return CommParams(T_lt=0.8e-3, b_nd=50e6 / 8, S_bnd=200.0, N_sub=2, name="paper: switched 100 Mbit Ethernet")


@dataclass
class Prediction:
    p: int
    T: float
    T_cmp: float
    T_lat: float
    T_bnd: float
    T_net: float
    rtr: float
    S: float = float("nan")
    E: float = float("nan")
    inputs: dict = field(default_factory=dict)


def t_cmm(p: int, c: CommParams, n_nb: float, n_spl: float) -> tuple[float, float, float]:
    """latency, node-bandwidth and network-bandwidth terms of T_cmm(p)"""
    if p <= 1:
        return 0.0, 0.0, 0.0
    lat = c.N_sub * n_nb * c.T_lt
    bnd = c.N_sub * (n_spl / p) * c.S_bnd / c.b_nd
    net = c.N_sub * n_spl * c.S_bnd / c.b_net if math.isfinite(c.b_net) else 0.0
    return lat, bnd, net


def predict(T1: float, ps, c: CommParams, n_nb=None, n_spl=None, e_dmn=None,
            f_ovr=None) -> list[Prediction]:
    """T(p), its terms, rtr, S and E for every p in ps.  n_nb / n_spl / e_dmn
    / f_ovr map p -> value (dicts or callables); missing ones take the
    paper's model functions (n_nb_model, n_spl_fit, e_dmn = 1, f_ovr = 0)."""
    def get(m, p, default):
        if m is None:
            return default(p)
        if callable(m):
            return m(p)
        return m[p] if p in m else default(p)

    out = []
    for p in ps:
        nb = get(n_nb, p, n_nb_model)
        ns = get(n_spl, p, n_spl_fit)
        ed = get(e_dmn, p, lambda q: 1.0)
        fo = get(f_ovr, p, lambda q: 0.0)
        tc = T1 / p * (1.0 + fo + (1.0 / ed - 1.0))
        lat, bnd, net = t_cmm(p, c, nb, ns)
        T = tc + lat + bnd + net
        out.append(Prediction(p, T, tc, lat, bnd, net, 1.0 / T,
                              inputs=dict(n_nb=nb, N_spl=ns, e_dmn=ed, f_ovr=fo)))
    T_one = next((x.T for x in out if x.p == 1), T1)
    for x in out:
        x.S = T_one / x.T
        x.E = x.S / x.p
    return out


def partition_stats(scn, dom, load=None) -> dict:
    """actual N_spl (links whose end nodes lie in different domains), mean
    neighbour domains per domain n_nb, and e_dmn = (total / p) / max domain
    load for a node -> domain map.  Load of a
    domain: its nodes' weights (default: half of cells x lanes of every
    attached link, the ORB weight)."""
    from . import domains
    d = np.asarray(dom)
    p = int(d.max()) + 1
    n_spl, pairs = domains.split_stats(scn, d)
    nbrs = [set() for _ in range(p)]
    for a, b in pairs:
        nbrs[a].add(b)
        nbrs[b].add(a)
    w = domains.node_weights(scn) if load is None else np.asarray(load, np.float64)
    per = np.bincount(d, weights=w, minlength=p)
    return dict(p=p, N_spl=n_spl, n_nb=float(np.mean([len(s) for s in nbrs])),
                n_nb_max=max(len(s) for s in nbrs), e_dmn=float(per.sum() / p / per.max()),
                domain_load=per.tolist())
