"""Profiling driver: config 4a, N warm-up steps then 3 steps (the profiled
launches).  python tools/prof.py [warm_steps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

warm = int(sys.argv[1]) if len(sys.argv) > 1 else 0
scn = scenarios.config('4a')
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED)
sim.load(scn)
sim.init(0)
if warm:
    sim.step(warm)
sim.step(3)
print(sim.last_timing())
