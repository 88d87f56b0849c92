import sys, numpy as np
sys.path.insert(0, '.')
import oracle, scenarios, paper_cs_0105004_b200 as tsim
from tests._ref import make_ring

def cmp(scn, steps, flags, **kw):
    o = oracle.Oracle.from_scenario(scn)
    g = tsim.Sim.from_scenario(scn, flags=flags, **kw)
    print("init hash", o.state_hash() == g.state_hash())
    for t in range(steps):
        vo, vg = o.vehicles(), g.vehicles()
        o.step(1); g.step(1)
        wo, wg = o.vehicles(), g.vehicles()
        bad = np.zeros(scn.n_vehicles, bool)
        for k in ("status","link","lane","cell","v","cursor"):
            bad |= wo[k] != wg[k]
        if bad.any():
            idx = np.nonzero(bad)[0][:8]
            print("t", t, "nbad", bad.sum())
            for f in idx:
                print(" vid", f, "before", [vo[k][f] for k in ("status","link","lane","cell","v","cursor")],
                      "oracle", [wo[k][f] for k in ("status","link","lane","cell","v","cursor")],
                      "gpu", [wg[k][f] for k in ("status","link","lane","cell","v","cursor")])
            return
    print("ok", steps)

if __name__ == "__main__":
    scn = scenarios.grid_trips(rows=4, cols=4, n_veh=600, depart_max=30, name="smoke")
    for fl in (tsim.FLAG_HASH, tsim.FLAG_FUSED|tsim.FLAG_HASH):
        cmp(scn, 40, fl)
    r = make_ring(50, [0,0,1,1,2], [3,10,4,20,30], [0,5,2,3,1], lanes=3, p_slow=0.2)
    cmp(r, 30, tsim.FLAG_HASH)
    cmp(scenarios.ring(n_cells=3000, lanes=3, density=0.2, seed=5), 30, tsim.FLAG_FUSED|tsim.FLAG_HASH, tile_cells=128)
