"""Wall-clock breakdown of the end-to-end path on config 4a (GPU box):
generate, Sim(), load (network + vehicles), init, steps, readback."""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

T = {}
t = time.perf_counter()
scn = scenarios.config(sys.argv[1] if len(sys.argv) > 1 else "4a")
T["generate"] = time.perf_counter() - t
tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED).close()  # CUDA context (as bench.py)
t = time.perf_counter()
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED)
T["create"] = time.perf_counter() - t
t = time.perf_counter()
sim.load(scn)
T["load"] = time.perf_counter() - t
t = time.perf_counter()
sim.init(0)
T["init"] = time.perf_counter() - t
t = time.perf_counter()
sim.step(100)
T["step100"] = time.perf_counter() - t
t = time.perf_counter()
v = sim.vehicles()
T["read_vehicles"] = time.perf_counter() - t
T["route_entries"] = int(scn.route.size)
print(json.dumps(T))
