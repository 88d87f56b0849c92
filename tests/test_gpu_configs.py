"""GPU parity at the BASELINE.json configs' stated sizes (north_star:
"bit-exact agreement with the CPU oracle on every config").

Every test runs the CPU oracle and two CUDA handles in lockstep on the same
seeded inputs:

* ``gh``: FLAG_FUSED | FLAG_HASH -- its per-step state hash S(t) is compared
  with the oracle's at EVERY step;
* ``gb``: FLAG_FUSED only -- exactly bench.py's launch flags (k_rows<5>,
  no hash instrument); its order-independent state hash is compared after
  every call and its full vehicle state (status, link, lane, cell, v,
  cursor, arrival time) at the listed times.

The update sequence (§4) must give cell-identical states
for any decomposition (acceptance #1), so the
k-domain runs of config 5 are compared with the UNDIVIDED oracle.
"""
import os

import numpy as np
import pytest

import oracle
import scenarios

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")
from paper_cs_0105004_b200 import domains  # noqa: E402

HASHED = tsim.FLAG_FUSED | tsim.FLAG_HASH
BENCH = tsim.FLAG_FUSED


def host_gb():
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                return int(ln.split()[1]) / 2**20
    except OSError:
        pass
    return 0.0


def same_state(o, g, msg):
    vo, vg = o.vehicles(), g.vehicles()
    for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
        bad = np.nonzero(vo[key] != vg[key])[0]
        assert bad.size == 0, (f"{msg} {key}: {bad.size} mismatches, first vid {bad[:5]} "
                               f"oracle {vo[key][bad[:5]]} gpu {vg[key][bad[:5]]}")


def lockstep(scn, steps, chunk, full_at=(), full_every=0):
    """oracle + hashed handle + bench-flags handle, `chunk` steps per call"""
    o = oracle.Oracle.from_scenario(scn)
    gh = tsim.Sim.from_scenario(scn, flags=HASHED)
    gb = tsim.Sim.from_scenario(scn, flags=BENCH)
    assert gh.state_hash() == o.state_hash() == gb.state_hash()
    same_state(o, gb, "init")
    done = 0
    while done < steps:
        n = min(chunk, steps - done)
        t_from = o.t + 1
        oh = o.run_hashes(n)
        gh.step(n)
        gb.step(n)
        done += n
        assert o.t == gh.t == gb.t
        hh = gh.history(t_from, n)["hash"]
        bad = [t_from + i for i in range(n) if hh[i] != oh[i]]
        assert not bad, f"{scn.name}: per-step hash differs at t={bad[:5]}"
        assert gb.state_hash() == oh[-1], f"{scn.name}: bench-flags hash differs at t={o.t}"
        if o.t in full_at or (full_every and done % full_every == 0) or done == steps:
            same_state(o, gb, f"{scn.name} t={o.t}")
    c = o.counters()
    assert gb.totals()["active"] == c["active"] and gb.totals()["arrived"] == c["arrived"]
    return o, gh, gb


def test_config2_full_length():
    """configs[1]: the 3-lane x 1,000,000-cell ring, 450,000 vehicles, all
    1,000 steps"""
    s = scenarios.config("2")
    lockstep(s, 1000, 50, full_every=250)


def test_config3_full_length():
    """configs[2]: the Portland-shaped network (~8,500 nodes, ~20,000 links,
    150,000 trips released over 1 h) for all 3,600 steps; full state every
    100 steps"""
    s = scenarios.config("3")
    o, gh, gb = lockstep(s, 3600, 100, full_every=100)
    assert o.counters()["arrived"] > 0


@pytest.mark.skipif(host_gb() < 48, reason="needs ~40 GB of host memory (14 GB of routes, twice)")
def test_config4a_bench_routes_driver_window():
    """configs[3] read as 4a, exactly the bench workload (scenarios.config
    ('4a'): 256 x 256 nodes, 104,448,000 lane-cells, 20,889,600 vehicles,
    full x-then-y Manhattan routes) through t = 25, which covers the driver's
    timed window (--warmup 5 --steps 20 -> steps 6..25): every per-step hash,
    the full state at t = 5, 15 and 25"""
    s = scenarios.config("4a")
    assert s.n_vehicles == 20_889_600
    lockstep(s, 25, 5, full_at=(5, 15, 25))


def test_config4b_prefix():
    """configs[3] read as 4b (1,000,000 vehicles on the 4a grid): 100 steps,
    full state every 20"""
    s = scenarios.config("4b")
    lockstep(s, 100, 10, full_every=20)


def test_config5_domains_rebalanced_vs_undivided_oracle():
    """configs[4]: the tiled Portland-shaped network in 8 domains on one GPU
    (ORB, split links, two strip exchanges per step), adaptively
    repartitioned every 300 steps from the measured per-domain device times
    and per-link work (§7) -- compared with the undivided
    CPU oracle: per-step hash every step, full state every 100 steps and
    after each repartition; the undivided GPU run with the bench flags in
    lockstep"""
    s = scenarios.config("5")
    o = oracle.Oracle.from_scenario(s)
    d = domains.LocalDomains(s, 8, flags=HASHED | tsim.FLAG_LINK_WORK)
    gb = tsim.Sim.from_scenario(s, flags=BENCH)
    assert d.state_hash() == o.state_hash() == gb.state_hash()
    doms = [d.dom.copy()]
    for block in range(2):
        for _ in range(3):
            t_from = o.t + 1
            oh = o.run_hashes(100)
            d.step(100)
            gb.step(100)
            hh = d.history(t_from, 100)["hash"]
            bad = [t_from + i for i in range(100) if hh[i] != oh[i]]
            assert not bad, f"8 domains: per-step hash differs at t={bad[:5]}"
            assert gb.state_hash() == oh[-1]
            same_state(o, d, f"8 domains t={o.t}")
            same_state(o, gb, f"undivided t={o.t}")
        dom, ms = d.rebalance()
        doms.append(np.asarray(dom).copy())
        assert len(ms) == 8 and min(ms) > 0
        same_state(o, d, f"after repartition at t={o.t}")
        assert d.state_hash() == o.state_hash()
    # the partition moved with the measured load
    assert any(not np.array_equal(doms[0], x) for x in doms[1:])
    assert o.counters()["active"] > 0
