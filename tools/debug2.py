import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, scenarios, paper_cs_0105004_b200 as tsim
s2 = scenarios.portland(n_nodes=600, n_edges=800, n_veh=3000, side_km=8.0, n_zones=64, seed=2)
s2.depart[:] = 0
o = oracle.Oracle.from_scenario(s2)
g = tsim.Sim.from_scenario(s2, flags=tsim.FLAG_HASH | tsim.FLAG_GENERAL)
def check(tag):
    bad = []
    for k in range(s2.n_links):
        code, vid = g.raw(k)
        for l in range(code.shape[0]):
            occ = code[l] < 0x80
            n = int(occ.sum())
            if (vid[l, :n] < 0).any() or (vid[l, :n] >= s2.n_vehicles).any():
                bad.append(k)
                if len(bad) < 4:
                    print(tag, "link", k, "lane", l, "w", o.n_cells(k), "L", code.shape[0], "n", n)
                    print("  code", code[l].tolist())
                    print("  vid ", vid[l].tolist())
                    print("  oracle", o.cells(k)[l].tolist())
    print(tag, "bad links", len(bad))
check("init")
for t in range(60):
    o.step(1); g.step(1)
    try:
        g.vehicles()
    except Exception as e:
        print("t", t+1, e)
        check(f"t{t+1}")
        break
print("done")
