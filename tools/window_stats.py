"""Per-step event rates in the driver's bench window (config 4a, steps
1..30): lane changes, crossings and mean speed per active vehicle -- what
the row kernel sees in its transient."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

scn = scenarios.config(sys.argv[1] if len(sys.argv) > 1 else "4a")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED)
sim.load(scn)
sim.init(0)
sim.step(n)
h = sim.history(1, n)
f = sim.flow(1, n)
for i in range(n):
    a = max(1, int(h["active"][i]))
    print(f"t={i + 1:3d} lc/veh {h['lane_changes'][i] / a:.4f} cross/veh {h['crossings'][i] / a:.4f} "
          f"mean v {f[i] / a:.3f}")
