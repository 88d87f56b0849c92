"""N2 calibration of the paper's performance model on one B200 (PAPER.md
§6, :803-1073; Fig. 12 analog :1056-1073 -- the run without vehicles gives
the latency floor).

For configs 3 and 4a:
  * T_1      : device time per step of the undivided run with vehicles;
  * T_0(k)   : per-domain device time per step of k = 1, 2, 4, 8 in-process
               domains (LocalDomains on one GPU) with NO vehicles -- kernel
               launches, strip packs / unpacks and the in-process exchange
               copies only;
  * T_lt     : fitted from T_0(k) = T_0(1) + N_sub * n_nb(k) * T_lt (least
               squares over both configs and k = 2, 4, 8), the paper's
               latency term;
  * predicted per-domain step time with vehicles
               T(k) = T_1 / k * (1 + f_dmn) + T_0(1) + N_sub * n_nb * T_lt
    against the measured per-domain device time (max over domains) of the
    same k-domain run with vehicles.
The domains of one GPU share its SMs, so the measured per-domain times of
a k-domain run are those of domains running side by side on one device.

  python tools/n2_calibrate.py [steps] > profiles/r2_perfmodel.md
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import scenarios  # noqa: E402
import paper_cs_0105004_b200 as tsim  # noqa: E402
from paper_cs_0105004_b200 import domains, perfmodel as pm  # noqa: E402

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 60
KS = (2, 4, 8)


def empty(scn):
    """the same network without vehicles"""
    import copy
    s = copy.copy(scn)
    z = np.zeros(0, np.int32)
    s.route_off = np.zeros(1, np.int64)
    s.route, s.depart, s.entry = z, z.copy(), z.copy()
    s.place_vid, s.place_lane, s.place_cell, s.place_v = z, z.copy(), z.copy(), z.copy()
    s.name = scn.name + "_empty"
    return s


def undivided_ms(scn, steps, warm=5):
    g = tsim.Sim.from_scenario(scn, flags=tsim.FLAG_FUSED)
    g.step(warm)
    g.step(steps)
    ms = g.last_timing()["total_ms"] / steps
    g.close()
    return ms


def domain_ms(scn, k, steps, warm=5):
    """k in-process domains stepped one domain at a time (each domain's
    phase runs alone on the GPU, as on a GPU of its own): per-domain device
    ms per step (ts_busy_time: the phases' kernels) and the host-measured ms
    of one exchange (ts_exchange_local + completion)"""
    d = domains.LocalDomains(scn, k, flags=tsim.FLAG_FUSED)
    d.step(warm)
    for s in d.sims:
        s.busy_time()
    xch = []

    def exchange():
        t = time.perf_counter()
        d._exchange()
        for s in d.sims:
            s.sync()
        xch.append(time.perf_counter() - t)

    for i in range(steps):
        for s in d.sims:
            s.phase(0)
            s.sync()
        exchange()
        for s in d.sims:
            s.phase(1, more=i < steps - 1)
            s.sync()
        exchange()
        for s in d.sims:
            s.phase(2)
            s.sync()
    per = [s.busy_time() / steps for s in d.sims]
    stats = pm.partition_stats(scn, d.dom)
    d.close()
    return per, float(np.median(xch)) * 1e3, stats


def main():
    out = {}
    for cfg in ("3", "4a"):
        scn = scenarios.config(cfg)
        ez = empty(scn)
        T1 = undivided_ms(scn, STEPS)
        T0 = {1: undivided_ms(ez, STEPS)}
        zero, full = {}, {}
        for k in KS:
            per, xms, st = domain_ms(ez, k, STEPS)
            zero[k] = dict(busy_ms=max(per), xchg_ms=xms, max_ms=max(per) + 2 * xms, **st)
            per, xms, st = domain_ms(scn, k, STEPS)
            full[k] = dict(busy_ms=max(per), xchg_ms=xms, max_ms=max(per) + 2 * xms,
                           per_domain_ms=per, **st)
        out[cfg] = dict(name=scn.name, T1_ms=T1, T0_1_ms=T0[1], zero=zero, full=full)
        print(json.dumps({cfg: dict(T1=T1, T0=T0[1], zero={k: zero[k]["max_ms"] for k in KS},
                                    full={k: full[k]["max_ms"] for k in KS})}), file=sys.stderr,
              flush=True)
    # fit T_lt: T_0(k) - T_0(1) = N_sub * n_nb(k) * T_lt (least squares through 0)
    xs, ys = [], []
    for cfg, r in out.items():
        for k in KS:
            xs.append(2 * r["zero"][k]["n_nb"])
            ys.append(r["zero"][k]["max_ms"] - r["T0_1_ms"])
    xs, ys = np.asarray(xs), np.asarray(ys)
    T_lt = float(np.sum(xs * ys) / np.sum(xs * xs))
    print("# Performance model (PAPER.md:803-1073) calibrated on one B200 -- round 2\n")
    print(f"Measured with `tools/n2_calibrate.py {STEPS}`.  k domains = k libtsim handles of "
          "one process on one GPU, stepped one domain at a time (each domain's phase alone on "
          "the device, as if it had a GPU of its own); per-domain step time = the device time of "
          "its phases (ts_busy_time, CUDA events on its stream) + 2 x the host-measured time of "
          "one in-process exchange (ts_exchange_local + completion).  FLAG_FUSED.\n")
    print("Zero-vehicle runs (Fig. 12 analog, PAPER.md:1056-1073): the per-domain step time "
          "without vehicles is the latency floor T_0(k) = T_0(1) + N_sub n_nb(k) T_lt "
          "(PAPER.md:888-895), N_sub = 2.  Least-squares fit over configs 3 and 4a, "
          f"k = 2, 4, 8: **T_lt = {T_lt * 1e3:.1f} us** per neighbour and exchange "
          "(the paper: 0.8 ms on switched 100 Mbit Ethernet, PAPER.md:985-1011).\n")
    for cfg, r in out.items():
        print(f"## config {cfg} ({r['name']})\n")
        print(f"T_1 = {r['T1_ms'] * 1e3:.1f} us/step (undivided, with vehicles); "
              f"T_0(1) = {r['T0_1_ms'] * 1e3:.1f} us/step (undivided, no vehicles).\n")
        print("| k | N_spl | n_nb | e_dmn | exchange us | T_0(k) measured us | T_0(k) model us | "
              "T(k) predicted us | T(k) measured us (max domain) | pred / meas |")
        print("|---|---|---|---|---|---|---|---|---|---|")
        for k in KS:
            z, f = r["zero"][k], r["full"][k]
            t0m = r["T0_1_ms"] + 2 * z["n_nb"] * T_lt
            pred = r["T1_ms"] / k / f["e_dmn"] + t0m
            print(f"| {k} | {f['N_spl']} | {f['n_nb']:.2f} | {f['e_dmn']:.3f} | {f['xchg_ms'] * 1e3:.1f} | "
                  f"{z['max_ms'] * 1e3:.1f} | {t0m * 1e3:.1f} | {pred * 1e3:.1f} | "
                  f"{f['max_ms'] * 1e3:.1f} | {pred / f['max_ms']:.2f} |")
            r["full"][k]["predicted_ms"] = pred
        print()
    out["T_lt_ms"] = T_lt
    with open(os.path.join(ROOT, "profiles", "r2_perfmodel.json"), "w") as fh:
        json.dump(out, fh, indent=1, default=float)


if __name__ == "__main__":
    main()
