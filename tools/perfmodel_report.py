"""Evaluate the paper's performance model (paper_cs_0105004_b200/perfmodel.py,
PAPER.md:803-1073) on our networks: actual ORB partition statistics at
p = 1, 2, 4, 8 (N_spl, n_nb, e_dmn), T_1 from a bench line, and the B200
communication parameters; plus the paper's own switched-Ethernet curve.

  python tools/perfmodel_report.py [BENCH_JSON] > profiles/r1_perfmodel.md

T_lt on B200 is an assumption (this round's pool has one GPU per call, so
no inter-GPU message was timed): one NCCL send/recv pair over NVLink per
neighbour and exchange, 10 us; b_nd = 900 GB/s (NVLink 5, one direction)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenarios  # noqa: E402
from paper_cs_0105004_b200 import domains, perfmodel as pm, tsim  # noqa: E402


def main():
    bench = {}
    if len(sys.argv) > 1:
        with open(sys.argv[1]) as f:
            bench = json.loads(f.read().strip().splitlines()[-1])
    T1 = bench.get("ms_per_step", 0.244) / 1e3
    strip = tsim.strip_bytes() if hasattr(tsim, "strip_bytes") else 144
    out = {"T1_s": T1, "source": sys.argv[1] if len(sys.argv) > 1 else "default 0.244 ms"}
    print("# Performance model (PAPER.md:803-1073) on B200 -- round 1\n")
    print(f"T_1 = {T1*1e3:.3f} ms/step (config 4a, bench line {out['source']}).  "
          f"B200 parameters: T_lt = 10 us (assumed; not timed on this single-GPU pool), "
          f"b_nd = 900 GB/s, S_bnd = lanes x {strip} B per split link and exchange "
          f"(one Strip per lane), N_sub = 2, switched (b_net = inf).\n")
    rows_all = {}
    for cfg in ("4a", "3"):
        scn = scenarios.config(cfg)
        lanes = scn.link_lanes
        stats = {}
        for p in (1, 2, 4, 8):
            dom = domains.partition(scn, p) if p > 1 else [0] * scn.n_nodes
            st = pm.partition_stats(scn, dom)
            cut = [i for i in range(len(scn.link_from))
                   if dom[scn.link_from[i]] != dom[scn.link_to[i]]]
            st["mean_lanes_split"] = float(sum(int(lanes[i]) for i in cut) / max(1, len(cut)))
            stats[p] = st
        mean_lanes = max(1.0, stats[8]["mean_lanes_split"])
        c = pm.CommParams(T_lt=10e-6, b_nd=900e9, S_bnd=strip * mean_lanes, N_sub=2,
                          name="B200 NVLink 5 (T_lt assumed)")
        T1c = T1 if cfg == "4a" else float("nan")
        rows = pm.predict(T1c if cfg == "4a" else 1e-4, [1, 2, 4, 8], c,
                          n_nb={p: stats[p]["n_nb"] for p in stats},
                          n_spl={p: stats[p]["N_spl"] for p in stats},
                          e_dmn={p: stats[p]["e_dmn"] for p in stats})
        print(f"## config {cfg} ({scn.name}), ORB partitions\n")
        print("| p | N_spl | n_nb (mean) | e_dmn | T_cmp ms | T_lat ms | T_bnd ms | T(p) ms | rtr | S | E |")
        print("|---|---|---|---|---|---|---|---|---|---|---|")
        for r in rows:
            st = stats[r.p]
            print(f"| {r.p} | {st['N_spl']} | {st['n_nb']:.2f} | {st['e_dmn']:.3f} | "
                  f"{r.T_cmp*1e3:.4f} | {r.T_lat*1e3:.4f} | {r.T_bnd*1e3:.5f} | {r.T*1e3:.4f} | "
                  f"{r.rtr:.0f} | {r.S:.2f} | {r.E:.2f} |")
        if cfg != "4a":
            print("\n(config 3: T_1 = 0.1 ms placeholder -- its step is launch-bound, not measured here)")
        print()
        rows_all[cfg] = dict(stats={str(k): v for k, v in stats.items()},
                             predict=[r.__dict__ for r in rows])
    # the paper's own curve: T_1 implied by rtr(16) = 40
    c = pm.paper_params()
    t16 = 1 / 40.0
    lat, bnd, net = pm.t_cmm(16, c, pm.n_nb_model(16), pm.n_spl_fit(16))
    T1p = (t16 - lat - bnd - net) * 16
    rows = pm.predict(T1p, [1, 2, 4, 8, 16, 32, 64, 128], c)
    print("## The paper's parameters (switched 100 Mbit Ethernet, PAPER.md:985-1011)\n")
    print(f"T_1 = {T1p*1e3:.0f} ms implied by rtr(16) = 40 (PAPER.md:1040-1043).\n")
    print("| p | n_nb | N_spl | T(p) ms | latency share | rtr |")
    print("|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r.p} | {r.inputs['n_nb']:.2f} | {r.inputs['N_spl']:.0f} | {r.T*1e3:.2f} | "
              f"{r.T_lat/r.T:.2f} | {r.rtr:.1f} |")
    rows_all["paper"] = dict(T1_implied=T1p, predict=[r.__dict__ for r in rows])
    with open(os.path.join(ROOT, "profiles", "r1_perfmodel.json"), "w") as f:
        json.dump(rows_all, f, indent=1, default=float)


if __name__ == "__main__":
    main()
