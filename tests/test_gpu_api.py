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
