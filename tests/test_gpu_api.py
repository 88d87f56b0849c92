"""Host-side contract of the C-ABI on the GPU: long runs
past the per-step statistics ring, per-handle asynchronous stepping."""
import numpy as np
import pytest

import scenarios

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")


def test_long_single_call_keeps_totals():
    """ts_step(n) with n > the 4,096-slot statistics ring: run in blocks and
    folded block by block, so the totals (vehicle updates, arrivals,
    injections, active) equal those of the same run in small calls and
    conserve the vehicles"""
    s = scenarios.grid_trips(rows=4, cols=4, n_veh=1500, depart_max=4000, seed=3, name="long")
    a = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    b = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    a.step(5000)
    for _ in range(50):
        b.step(100)
    ta, tb = a.totals(), b.totals()
    assert a.t == b.t == 5000
    for k in ("active", "pending", "arrived", "vehicle_updates"):
        assert ta[k] == tb[k], k
    assert ta["active"] + ta["pending"] + ta["arrived"] == s.n_vehicles
    assert ta["arrived"] > 0 and a.state_hash() == b.state_hash()
    tm = a.last_timing()
    assert tm["total_ms"] > 0 and tm["move_launches"] > 0
    # the most recent history is readable after the long call
    h = a.history(a.t - 100, 101)
    assert int(h["active"][-1]) == ta["active"]


def test_interleaved_async_handles():
    """ts_step_async / ts_sync keep their state per handle: A and B
    interleaved give each its own timing and totals; a sync without a
    pending async run just synchronises; a second async call before the
    sync is rejected"""
    s = scenarios.config("1")
    a = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    b = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    ref = tsim.Sim.from_scenario(s, flags=tsim.FLAG_FUSED)
    a.step_async(30)
    b.step_async(70)
    with pytest.raises(tsim.TsError):
        a.step_async(5)
    a.sync()
    b.sync()
    b.sync()
    ref.step(70)
    assert a.t == 30 and b.t == 70
    assert b.state_hash() == ref.state_hash()
    assert b.totals()["vehicle_updates"] == ref.totals()["vehicle_updates"]
    assert a.last_timing()["total_ms"] > 0 and b.last_timing()["total_ms"] > 0
    a.step_async(5000)  # longer than the ring: leading blocks finish first
    a.sync()
    assert a.t == 5030
    t = a.totals()
    assert t["active"] + t["pending"] + t["arrived"] == s.n_vehicles


@pytest.mark.parametrize("which", ["grid", "portland", "ring", "split"])
def test_device_init_equals_host_init(which, monkeypatch):
    """The row-tile placement built on the device (default) gives the same
    state as the host build (TSIM_HOST_INIT=1): identical vehicle state at
    t0 and after 30 steps, with general tiles (links > 128 cells), ring
    rows and a split domain (at t0) in the mix"""
    if which in ("grid", "split"):
        s = scenarios.grid_trips(rows=4, cols=4, n_veh=3000, depart_max=20, seed=5, name="g")
    elif which == "portland":
        s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=6000, side_km=8.0, n_zones=16, seed=4)
    else:
        s = scenarios.ring(n_cells=20_000, lanes=3, density=0.2, seed=2, steps=30)

    def run(host):
        if host:
            monkeypatch.setenv("TSIM_HOST_INIT", "1")
        else:
            monkeypatch.delenv("TSIM_HOST_INIT", raising=False)
        sim = tsim.Sim(p_slow=s.p_slow, seed=s.seed, flags=tsim.FLAG_FUSED | tsim.FLAG_HASH)
        sim.load(s)
        if which == "split":
            sim.partition(2, 0)
        sim.init(0)
        out = [sim.vehicles(), sim.totals()["active"]]
        if which != "split":  # (a lone domain with neighbours does not step)
            sim.step(30)
        out += [sim.vehicles(), sim.state_hash()]
        sim.close()
        return out

    a, b = run(False), run(True)
    for x, y in ((a[0], b[0]), (a[2], b[2])):
        for k in x:
            assert np.array_equal(x[k], y[k]), k
    assert a[1] == b[1] and a[3] == b[3]


@pytest.mark.parametrize("general", [False, True])
def test_entrant_record_time_wrap(general):
    """The node kernel's entrant record carries the crossing time in 21 bits
    ((t + 1) mod 2^21).  A target lane whose last entrant crossed at step T
    and that sees none afterwards must not get it again at T + 2^21 (nor a
    never-written record at t + 1 = 2^21): config 1 (every vehicle arrived
    after ~600 steps) is run past 2^21 + 800 steps with graph replay, row
    kernel or general tiles, and must stay empty with every vehicle arrived"""
    s = scenarios.config("1")
    flags = tsim.FLAG_FUSED | tsim.FLAG_GRAPH | (tsim.FLAG_GENERAL if general else 0)
    sim = tsim.Sim.from_scenario(s, flags=flags)
    sim.step(800)
    tot = sim.totals()
    assert tot["arrived"] == s.n_vehicles and tot["active"] == 0
    sim.step((1 << 21) + 800)
    tot = sim.totals()
    assert tot["active"] == 0 and tot["arrived"] == s.n_vehicles, tot
    st = sim.vehicles()
    assert (st["status"] == tsim.ARRIVED).all()
