import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, scenarios, paper_cs_0105004_b200 as tsim

KEYS = ("status", "link", "lane", "cell", "v", "cursor")

def cmp(scn, steps, flags, **kw):
    o = oracle.Oracle.from_scenario(scn)
    g = tsim.Sim.from_scenario(scn, flags=flags, **kw)
    for t in range(steps):
        vo = o.vehicles()
        o.step(1); g.step(1)
        wo, wg = o.vehicles(), g.vehicles()
        bad = np.zeros(scn.n_vehicles, bool)
        for k in KEYS: bad |= wo[k] != wg[k]
        if bad.any():
            print("flags", flags, "t", t, "nbad", bad.sum())
            for f in np.nonzero(bad)[0][:6]:
                r = scn.route[scn.route_off[f]:scn.route_off[f+1]]
                print(" vid", f, "route", r[:6], "before", [int(vo[k][f]) for k in KEYS],
                      "oracle", [int(wo[k][f]) for k in KEYS], "gpu", [int(wg[k][f]) for k in KEYS])
                k = int(vo["link"][f])
                if k >= 0:
                    print("   link", k, "lanes", scn.link_lanes[k], "cells", o.n_cells(k), "from", scn.link_from[k], "to", scn.link_to[k])
            return
    print("flags", flags, "ok", steps)

if __name__ == "__main__":
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64, seed=2)
    s.depart = (s.depart // 12).astype(np.int32)
    H = tsim.FLAG_HASH
    for fl in (H | tsim.FLAG_FUSED, H | tsim.FLAG_FUSED | 32, H | tsim.FLAG_GENERAL, H):
        try:
            cmp(s, 120, fl)
        except Exception as e:
            print("flags", fl, "EXC", e)
    # no injection: all vehicles depart at 0
    s2 = scenarios.portland(n_nodes=600, n_edges=800, n_veh=3000, side_km=8.0, n_zones=64, seed=2)
    s2.depart[:] = 0
    for fl in (H | tsim.FLAG_FUSED, H | tsim.FLAG_GENERAL):
        try:
            cmp(s2, 120, fl)
        except Exception as e:
            print("dep0 flags", fl, "EXC", e)
