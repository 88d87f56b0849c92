#!/usr/bin/env python3
"""Benchmark of the B200 TRANSIMS CA step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4a]
                    [--impl tsim|reference]

One step = one full pass of the hot path (lane change, intersections,
velocity update + move, injection) over every lane-cell
of the workload.  Default workload: BASELINE.json configs[3] read as 4a
(256x256 grid, 4 lanes, 100-cell links, 104,448,000 lane-cells, 20,889,600
vehicles): the one configuration larger than L2, where the HBM roofline is
meaningful.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import scenarios  # noqa: E402

NOMINAL_HBM_GBS = 8000.0  # north_star: "against the B200's ~8 TB/s"

FALLBACK_HBM_GBS = 6650.0


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + throttle reasons during the timed region: NVML every
    millisecond (the driver's 20-step window is ~5 ms long), else nvidia-smi.
    The wait for the sampler thread at exit is recorded (`exit_s`) so that
    wall-clock timings can leave the harness out."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.rows = []
        self.stop = threading.Event()
        self.th = None
        self.exit_s = 0.0
        self.source = "nvidia-smi"
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(gpu))
            self.source = "nvml"
        except Exception:
            self.nvml = None

    def _sample_nvml(self):
        nv, h = self.nvml
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        act = lambda bit: "Active" if r & bit else "Not Active"  # noqa: E731
        return [str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                str(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)), hex(r),
                act(nv.nvmlClocksEventReasonHwSlowdown), act(nv.nvmlClocksEventReasonHwThermalSlowdown),
                act(nv.nvmlClocksEventReasonSwThermalSlowdown), act(nv.nvmlClocksEventReasonSwPowerCap)]

    def _run(self):
        while not self.stop.is_set():
            try:
                if self.nvml:
                    self.rows.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.001 if self.nvml else 0.05)

    def __enter__(self):
        if self.nvml:  # one sample before the region starts
            try:
                self.rows.append(self._sample_nvml())
            except Exception:
                pass
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        t = time.perf_counter()
        self.stop.set()
        if self.th:
            self.th.join(timeout=10)
        self.exit_s = time.perf_counter() - t

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows), "source": self.source}


def ncu_traffic():
    """DRAM bytes per launch of k_rows from the committed ncu --set full
    capture (profiles/traffic_k_rows.json, written by tools/ncu_traffic.py)."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic_k_rows.json")
    try:
        with open(p) as f:
            t = json.load(f)
        return {"bytes": t["traffic_bytes_per_launch"],
                "inst": t.get("warp_instructions_per_launch"),
                "source": f"ncu --set full, {t['report']}: {t['note']}"}
    except (OSError, KeyError, ValueError):
        return {"bytes": None, "inst": None, "source": None}


def issue_roof(inst, kernel_ms, sm_mhz):
    """the kernel's secondary roof, instruction issue: the
    warp instructions of one launch (committed ncu capture) over the live
    CUDA-event duration, against 148 SMs x 4 schedulers x 1 warp
    instruction per cycle at the sampled SM clock"""
    if not inst or not kernel_ms:
        return None
    mhz = sm_mhz or 1965.0
    peak = 148 * 4 * mhz * 1e6
    achieved = inst / (kernel_ms / 1e3)
    return {"achieved": achieved, "peak": peak, "unit": "warp-instructions/s",
            "frac": achieved / peak, "warp_instructions_per_launch": inst,
            "note": "instruction count from the ncu capture (traffic_source), time and clock live"}


def workload(name):
    scn = scenarios.config(name)
    return scn


def sample_workload(name):
    """bounded sample of the same workload for the CPU oracle: same recipe on
    a smaller network"""
    if name in ("4a", "4b"):
        kw = dict(rows=32, cols=32, seed=1, name=f"config{name}_sample32")
        if name == "4b":
            kw["n_veh"] = int(1_000_000 * (32 * 31) / (256 * 255))
        return scenarios.big_grid(**kw), "32x32-node sub-grid, same lanes/cells/density/route recipe"
    if name == "2":
        return scenarios.ring(n_cells=100_000, lanes=3, density=0.15, seed=1), "3 x 100,000-cell ring"
    if name == "3":
        s = scenarios.config("3")
        return s, "full network"
    return workload(name), "full workload"


def run_oracle(name, steps, warmup, budget_s=None):
    import oracle
    scn, desc = sample_workload(name)
    o = oracle.Oracle.from_scenario(scn)
    o.step(warmup)
    u0 = o.counters()["vehicle_updates"]
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        o.step(1)
        done += 1
        if budget_s and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    upd = o.counters()["vehicle_updates"] - u0
    return dict(value=upd / dt, steps=done, seconds=dt, desc=desc,
                lane_cells=int(o.lib.or_total_lane_cells(o.h)))


# names of the scenarios (scenarios.config(name).name) without generating them
WORKLOAD_NAMES = {"1": "config1_grid4x4", "2": "config2_ring", "3": "config3_portland",
                  "4a": "config4a_grid256", "4b": "config4b_grid256_1M",
                  "5": "config5_portland_x8"}


def bench_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    r = run_oracle(args.config, args.steps, args.warmup)
    out = {
        "impl": "reference", "metric": "vehicle-updates/s", "value": r["value"],
        "unit": "vehicle-updates/s", "n_gpus": args.gpus, "steps": r["steps"],
        "warmup": args.warmup, "ms_per_step": 1000 * r["seconds"] / max(1, r["steps"]),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_NAMES.get(args.config, f"config{args.config}"),
                   "sample": r["desc"], "l2": "sample runs on the host (CPU oracle)",
                   "parallelism": "1 host thread"},
        "cpu_baseline": {"value": r["value"], "unit": "vehicle-updates/s", "cores": 1,
                         "kind": "oracle", "sample": r["desc"]},
        "e2e": {"value": r["value"], "unit": "vehicle-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def bench_tsim(args):
    import paper_cs_0105004_b200 as tsim
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        return bench_multi(args)
    hbm_peak, peak_src = measured_peaks()
    traffic = ncu_traffic()
    t_gen = time.perf_counter()
    scn = workload(args.config)
    t_gen = time.perf_counter() - t_gen
    flags = tsim.FLAG_FUSED | (tsim.FLAG_HASH if args.hash else 0)
    # e2e: wall clock around the public API from host arrays to the final
    # state on the host (H2D of network + vehicles, W+K steps, D2H of state)
    h2d = scenario_bytes(scn)
    # process start-up happens before the timed region: the CUDA context,
    # the lazily loaded kernel modules and the driver's staging buffers,
    # warmed by a throwaway 8x8-node grid of the same recipe run through the
    # same calls (nothing of it is reused: it has its own handle and data)
    warm_up(tsim, scn, flags)
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))  # (set up outside the timed region)
    ph = {}  # wall-clock phases of the e2e region
    w0 = time.perf_counter()
    sim = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=flags)
    sim.load(scn)
    ph["load"] = time.perf_counter() - w0
    sim.init(0)
    ph["init"] = time.perf_counter() - w0 - ph["load"]
    sim.step(args.warmup)
    tot = sim.totals()
    with clk:
        t_from = sim.t
        sim.step(args.steps)
    timing = sim.last_timing()
    hist = sim.history(t_from, args.steps + 1)
    t_rd = time.perf_counter()
    vst = sim.vehicles()
    ph["readback"] = time.perf_counter() - t_rd
    e2e_wall = time.perf_counter() - w0 - clk.exit_s  # (the clock sampler is harness)
    ph["steps_and_stats"] = e2e_wall - ph["load"] - ph["init"] - ph["readback"]
    d2h = sum(a.nbytes for a in vst.values())
    ms_total = timing["total_ms"]
    updates = int(np.sum(hist["active"][:args.steps]))
    value = updates / (ms_total / 1e3)
    rtr = args.steps / (ms_total / 1e3)
    # roofline of the dominant kernel (k_rows): algorithmic bytes per launch
    # = 2 B x lane-cells (codes in + out) + 8 B x active vehicles (vid in +
    # out) + 12 B x node crossers
    lane_cells = tot["lane_cells"]
    alg = 2 * lane_cells * args.steps + 8 * updates + 12 * int(np.sum(hist["crossings"][1:]))
    alg_per_launch = alg / args.steps
    mv_ms = timing["move_ms"] / max(1, timing["move_launches"])
    achieved = alg_per_launch / (mv_ms / 1e3) / 1e9
    # the warm-up steps update the vehicles of S(0) .. S(W-1)
    upd_all = updates + int(np.sum(sim.history(0, args.warmup)["active"]))
    out = {
        "metric": "vehicle-updates/s", "value": value, "unit": "vehicle-updates/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded generator, DESIGN.md §5)",
        "config": {"workload": scn.name, "recipe": scn.recipe, "lane_cells": lane_cells,
                   "vehicles": scn.n_vehicles, "tiles": tot["tiles"],
                   "l2": l2_note(lane_cells),
                   "parallelism": "1 GPU, 1 domain", "flags": "fused" + ("+hash" if args.hash else "")},
        "real_time_ratio": rtr,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic["bytes"],
                     "traffic_source": traffic["source"], "kernel": "k_rows",
                     "alg_bytes_per_launch": alg_per_launch, "kernel_ms": mv_ms,
                     "kernel_share": mv_ms * args.steps / ms_total,
                     "kernel_launches_timed": timing["move_launches"], "peak_source": peak_src,
                     # also against north_star's nominal ~8 TB/s, and
                     # the whole step (node kernel included) against the measured peak
                     "nominal_peak": NOMINAL_HBM_GBS, "frac_nominal": achieved / NOMINAL_HBM_GBS,
                     "step_frac": alg_per_launch / (ms_total / args.steps * 1e-3) / 1e9 / hbm_peak},
        "e2e": {"value": upd_all / e2e_wall, "unit": "vehicle-updates/s",
                "h2d_bytes_per_step": h2d / (args.steps + args.warmup),
                "d2h_bytes_per_step": d2h / (args.steps + args.warmup),
                "wall_s": e2e_wall, "phases_s": {k: round(v, 4) for k, v in ph.items()},
                "scope": "load+init+W+K steps+state readback (CUDA context created before)"},
        "clocks": clk.summary(),
        "gpu_launches": 1 + 2 * args.steps,
        "gen_s": t_gen,
    }
    # (the captured launch is from the driver's window: its instruction count
    # holds for that run only -- the steady state executes ~30 % fewer)
    out["roofline"]["issue"] = (issue_roof(traffic.get("inst"), mv_ms, out["clocks"].get("sm_mhz"))
                                if (args.steps, args.warmup, args.config) == (20, 5, "4a") else None)
    sim.close()
    if args.cpu_baseline and rank == 0:
        import multiprocessing
        r = run_oracle(args.config, 400, 5, budget_s=20.0)
        out["cpu_baseline"] = {"value": r["value"], "unit": "vehicle-updates/s", "cores": 1,
                               "kind": "oracle", "host_cores": multiprocessing.cpu_count(),
                               "sample": f"{r['steps']} steps of {r['desc']} "
                                         f"({r['lane_cells']} lane-cells), {r['seconds']:.1f} s"}
    print(json.dumps(out), flush=True)


def warm_up(tsim, scn, flags, device=0):
    """process start-up outside the timed region: CUDA context, lazily
    loaded kernel modules, the driver's staging buffers -- a throwaway 8x8
    grid of the 4a recipe through load / init / step / read"""
    warm = scenarios.big_grid(rows=8, cols=8, seed=scn.seed + 1, name="warm-up")
    ws = tsim.Sim(p_slow=warm.p_slow, seed=warm.seed, flags=flags, device=device)
    ws.load(warm)
    ws.init(0)
    ws.step(3)
    ws.step(2)
    ws.vehicles()
    ws.close()


def l2_note(lane_cells):
    """between timed steps the state is re-read from HBM only if it is larger
    than the 126 MB L2 (no flush is done)"""
    if 2 * lane_cells > 126e6:
        return "inputs larger than L2 (state read+written per step > 126 MB)"
    return "state fits in L2 (no flush between steps: a small-config number, not a roofline one)"


def scenario_bytes(scn):
    """host bytes the public API copies to the device for one scenario"""
    return sum(a.nbytes for a in (scn.node_x, scn.node_y, scn.link_from, scn.link_to,
                                  scn.link_len_mm, scn.link_lanes, scn.link_vmax, scn.link_class,
                                  scn.route_off, scn.route, scn.depart, scn.entry, scn.place_vid,
                                  scn.place_lane, scn.place_cell, scn.place_v))


def bench_multi(args):
    """N > 1: one process per GPU, one domain of an ORB partition per rank
    (§4), two strip exchanges per step with the neighbour domains
    over NCCL (NVLink).  The workload is the same as at N = 1 (strong
    scaling); the step time is the max over ranks of the device-timed K
    steps."""
    import torch
    import torch.distributed as dist

    import paper_cs_0105004_b200 as tsim
    from paper_cs_0105004_b200 import domains
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TSIM_BENCH_BACKEND=gloo: a functional check of this multi-rank path with
    # fewer GPUs than ranks (ranks share devices, strips staged through host
    # memory); its timings are not scaling numbers
    backend = os.environ.get("TSIM_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        dist.init_process_group(backend)
    hbm_peak, peak_src = measured_peaks()
    scn = workload(args.config)
    dom = domains.partition(scn, world)
    n_spl, pairs = domains.split_stats(scn, dom)
    h2d = scenario_bytes(scn)  # every rank loads the whole network and plan set
    warm_up(tsim, scn, tsim.FLAG_FUSED, device=local)
    clk = ClockSampler(local)  # (NVML set up outside the timed region)
    w0 = time.perf_counter()
    # native exchanges (the library's own NCCL communicator, whole steps per
    # ts_step call); torch.distributed send/recv between the phases otherwise
    try:
        d = domains.DistDomain(scn, dom, device=local, flags=tsim.FLAG_FUSED,
                               native=backend == "nccl")
    except tsim.TsError:
        d = domains.DistDomain(scn, dom, device=local, flags=tsim.FLAG_FUSED)
    d.step(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        t_from = d.t
        e0.record(d.stream)
        d.step(args.steps)
        e1.record(d.stream)
        torch.cuda.synchronize()
    dist.barrier()
    red_dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # exchange time, reported separately: mean device time of one exchange
    # (timed on every 8th step by the library), max over ranks
    xms, xn = d.sim.last_exchange_timing() if d.native else (0.0, 0)
    xchg = torch.tensor([xms / max(1, xn)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(xchg, op=dist.ReduceOp.MAX)
    hist = d.sim.history(t_from, args.steps + 1)
    tot = d.sim.totals()
    vst = d.sim.vehicles()
    e2e_local = time.perf_counter() - w0 - clk.exit_s
    # the warm-up steps update the vehicles of S(0) .. S(W-1) (counted for e2e)
    upd_w = float(np.sum(d.sim.history(0, args.warmup)["active"]))
    loc = torch.tensor([float(np.sum(hist["active"][:args.steps])), float(tot["lane_cells"]),
                        float(np.sum(hist["crossings"][1:])), e2e_local, upd_w],
                       dtype=torch.float64, device=red_dev)
    s = loc.clone()
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    e2e = loc[3:4].clone()
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    ms_total = float(ms.item())
    # every rank reports the whole network's lane-cells (ts_get_totals): once
    updates, lane_cells, cross, upd_all = (float(s[0]), float(s[1]) / world, float(s[2]),
                                           float(s[0] + s[4]))
    if rank == 0:
        value = updates / (ms_total / 1e3)
        alg = (2 * lane_cells * args.steps + 8 * updates + 12 * cross) / world
        achieved = alg / (ms_total / 1e3) / 1e9
        out = {
            "metric": "vehicle-updates/s", "value": value, "unit": "vehicle-updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded generator, DESIGN.md §5)",
            "config": {"workload": scn.name, "recipe": scn.recipe, "lane_cells": int(lane_cells),
                       "vehicles": scn.n_vehicles,
                       "l2": l2_note(lane_cells),
                       "parallelism": f"{world} ranks, ORB domains, split links, 2 strip exchanges "
                                      f"per step ({'native NCCL' if d.native else 'torch.distributed ' + backend})",
                       "split_links": n_spl,
                       "domain_pairs": len(pairs)},
            "real_time_ratio": args.steps / (ms_total / 1e3),
            "exchange": {"ms_per_exchange": float(xchg.item()) if d.native else None,
                         "exchanges_per_step": 2,
                         "share_of_step": 2 * float(xchg.item()) / (ms_total / args.steps)
                         if d.native else None,
                         "transport": "native NCCL" if d.native else f"torch.distributed {backend}"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": None,
                         "kernel": "whole step per GPU (incl. exchanges)",
                         "alg_bytes_per_launch": alg / args.steps, "peak_source": peak_src},
            "e2e": {"value": upd_all / float(e2e.item()), "unit": "vehicle-updates/s",
                    "h2d_bytes_per_step": h2d / (args.steps + args.warmup), "d2h_bytes_per_step": sum(
                        a.nbytes for a in vst.values()) / (args.steps + args.warmup),
                    "wall_s": float(e2e.item()),
                    "scope": "per rank: load+init+W+K steps+state readback, max over ranks"},
            "clocks": clk.summary(),
            "gpu_launches": 1 + 4 * args.steps,
        }
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="4a")
    ap.add_argument("--impl", default="tsim", choices=["tsim", "reference"])
    ap.add_argument("--hash", action="store_true")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_tsim(args)


if __name__ == "__main__":
    main()
