import sys, time, json
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scenarios, paper_cs_0105004_b200 as tsim
scn = scenarios.config('4a')
for gc in [int(a) for a in sys.argv[1:]]:
    sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED, group_cells=gc)
    sim.load(scn); sim.init(0)
    sim.step(10)
    sim.step(100)
    tm = sim.last_timing()
    h = sim.history(sim.t - 99, 100)
    print(json.dumps(dict(group_cells=gc, ms_step=tm['total_ms']/100, ms_move=tm['move_ms']/100,
                          lc=int(np.mean(h['lane_changes'])), cross=int(np.mean(h['crossings'])),
                          active=int(h['active'][-1]))), flush=True)
    sim.close()
