"""Per-domain step times of the multi-domain step on one GPU, next to the
undivided runs (verdict r1 item 6): configs 3 and 5,
k = 8 in-process domains stepped by the library (ts_local_step), without and
with CUDA-graph replay of all domains' streams; each domain's device time
of its phases (ts_busy_time, phases timed without graphs), and the wall
clock per step of the whole k-domain step.
  python tools/domain_step_times.py [steps] > profiles/r2_domain_step_times.json"""
import json
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402
from paper_cs_0105004_b200 import domains  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
out = {}
for cfg in ("3", "5"):
    scn = scenarios.config(cfg)
    g = tsim.Sim.from_scenario(scn, flags=tsim.FLAG_FUSED)
    g.step(600)  # into the departure profile
    g.step(steps)
    und = g.last_timing()["total_ms"] / steps
    t_und = g.t
    hash_und = g.state_hash()
    g.close()
    r = {"undivided_ms_per_step": und}
    for graph in (False, True):
        flags = tsim.FLAG_FUSED | (tsim.FLAG_GRAPH if graph else 0)
        d = domains.LocalDomains(scn, 8, flags=flags)
        d.step(600)
        for s in d.sims:
            s.busy_time()
        w0 = time.perf_counter()
        d.step(steps)
        wall = (time.perf_counter() - w0) / steps * 1e3
        per = [s.busy_time() / steps for s in d.sims]
        assert d.t == t_und and d.state_hash() == hash_und, "partition changed the result"
        r["graph" if graph else "launches"] = {
            "wall_ms_per_step": wall,
            "per_domain_busy_ms_per_step": per if not graph else None,
            "max_domain_busy_ms": max(per) if not graph else None}
        d.close()
    out[cfg] = r
    print(json.dumps({cfg: r}), file=sys.stderr, flush=True)
out["note"] = ("one GPU: the 8 domains' streams share it; wall = host wall clock per step of "
               "ts_local_step over all domains (device-bound when graph-replayed); busy = each "
               "domain's own phase device time (not recorded inside replayed graphs); the final "
               "state hash of the 8-domain runs equals the undivided run's")
print(json.dumps(out, indent=1))
