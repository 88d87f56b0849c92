"""BASELINE config 5 on one GPU: the tiled Portland-shaped network in 8
domains (LocalDomains, in-process exchanges), adaptive repartitioning every
PERIOD steps from the measured per-domain device time (
Fig. 10 analog: per-domain times before / after each rebalance), and the
final state checked against the undivided run (partition invariance).
  python tools/config5_rebalance.py [steps] [period] > profiles/r1_config5_rebalance.json"""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402
from paper_cs_0105004_b200 import domains  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1800
period = int(sys.argv[2]) if len(sys.argv) > 2 else 300
k = 8
scn = scenarios.config("5")
t0 = time.perf_counter()
d = domains.LocalDomains(scn, k, flags=tsim.FLAG_FUSED | tsim.FLAG_LINK_WORK)
rounds = []
done = 0
while done < steps:
    n = min(period, steps - done)
    d.step(n)
    done += n
    lw = [s.link_work() for s in d.sims]
    base = getattr(d, "_lw_base", None)
    win = [w - b for w, b in zip(lw, base)] if base is not None else lw
    dom_old = d.dom.copy()
    n_spl_old = domains.split_stats(scn, dom_old)[0]
    new, ms = d.rebalance() if done < steps else (dom_old, [s.busy_time() for s in d.sims])
    lt = domains.link_times(win, ms)
    fr = np.asarray(scn.link_from)
    load_old = np.bincount(dom_old[fr], weights=lt, minlength=k)
    load_new = np.bincount(np.asarray(new)[fr], weights=lt, minlength=k)
    rounds.append(dict(t=int(d.t), domain_ms=[round(x, 3) for x in ms],
                       e_dmn_measured=float(load_old.mean() / load_old.max()),
                       e_dmn_next_partition=float(load_new.mean() / load_new.max()),
                       split_links=int(n_spl_old),
                       active=int(sum(s.totals()["active"] for s in d.sims))))
    print(json.dumps(rounds[-1]), file=sys.stderr, flush=True)
h_dom = d.state_hash()
wall = time.perf_counter() - t0
ref = tsim.Sim.from_scenario(scn, flags=tsim.FLAG_FUSED)
ref.step(steps)
print(json.dumps(dict(config="5 (config5_portland_x8)", domains=k, steps=steps, period=period,
                      rounds=rounds, final_hash_domains=hex(h_dom),
                      final_hash_undivided=hex(ref.state_hash()),
                      identical=bool(h_dom == ref.state_hash()), wall_s=round(wall, 1),
                      note="one GPU: the 8 domains run one after another with in-process "
                           "exchanges; the times are each domain's own device time")))
