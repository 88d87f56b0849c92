"""ms per step of the small configurations (launch-bound regime): config 1
(4x4 grid), 2 (3-lane ring), 3 (Portland-shaped), 4b (1 M vehicles)."""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402

flags = tsim.FLAG_FUSED | (int(sys.argv[2]) if len(sys.argv) > 2 else 0)
tile_cells = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3"]):
    scn = scenarios.config(cfg)
    sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=flags, tile_cells=tile_cells)
    sim.load(scn)
    sim.init(0)
    sim.step(50)
    t = time.perf_counter()
    sim.step(1000)
    wall = time.perf_counter() - t
    tm = sim.last_timing()
    tot = sim.totals()
    print(json.dumps(dict(config=cfg, tile_cells=tile_cells, ms_step_gpu=tm["total_ms"] / 1000, ms_step_wall=wall,
                          active=tot.get("active"), tiles=tot.get("tiles"))), flush=True)
    sim.close()
