import sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenarios, paper_cs_0105004_b200 as tsim
gc = int(sys.argv[1]) if len(sys.argv) > 1 else 0
scn = scenarios.config('4a')
sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED, group_cells=gc)
sim.load(scn); sim.init(0)
sim.step(6)
print(sim.last_timing())
