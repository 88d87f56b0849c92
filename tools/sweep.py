"""config 4a: ms per step for several staging capacities (group_cells)"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

scn = scenarios.config('4a')
for gc in [int(a) for a in sys.argv[1:]]:
    sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED, group_cells=gc)
    sim.load(scn)
    sim.init(0)
    sim.step(200)
    sim.step(100)
    tm = sim.last_timing()
    print(json.dumps(dict(cap=gc, ms_step=tm['total_ms'] / 100, ms_move=tm['move_ms'] / max(1, tm['move_launches']))),
          flush=True)
    sim.close()
