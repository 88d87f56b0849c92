"""Per-step event rates on a config (GPU box): lane changes, crossings,
injections per step, as fractions of the active vehicles -- how often the
row kernel takes its general vid-list path."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

scn = scenarios.config(sys.argv[1] if len(sys.argv) > 1 else "4a")
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED)
sim.load(scn)
sim.init(0)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
sim.step(n)
h = sim.history(0, n)
act = np.maximum(h["active"], 1)
for key in ("lane_changes", "crossings", "injections", "arrivals"):
    r = h[key] / act
    print(f"{key:13s} per active vehicle per step: first10 {r[:10].mean():.4f}  "
          f"last50 {r[-50:].mean():.4f}  mean {r.mean():.4f}")
print("active", int(h["active"][0]), int(h["active"][-1]))
