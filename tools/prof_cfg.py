"""Profiling driver for any config: W warm-up steps then 3 steps.
python tools/prof_cfg.py CONFIG [warm]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

cfg = sys.argv[1]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 50
scn = scenarios.config(cfg)
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED)
sim.load(scn)
sim.init(0)
sim.step(warm)
sim.step(3)
print(sim.last_timing())
