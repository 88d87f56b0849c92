"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle,
bit-exact in every vehicle's (status, link, lane, cell, v, cursor) and in the
per-step state hash (north_star: "bit-exact to the oracle in every vehicle's
cell, lane, velocity and link at every step")."""
import numpy as np
import pytest

import oracle
import scenarios
from tests._ref import make_network, make_ring

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")

FUSED = tsim.FLAG_FUSED | tsim.FLAG_HASH
UNFUSED = tsim.FLAG_HASH
GENERAL = tsim.FLAG_FUSED | tsim.FLAG_HASH | tsim.FLAG_GENERAL  # warp-per-tile kernels


def assert_same_state(o, g, msg=""):
    vo, vg = o.vehicles(), g.vehicles()
    for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
        bad = np.nonzero(vo[key] != vg[key])[0]
        assert bad.size == 0, (f"{msg} {key}: {bad.size} mismatches, first vid {bad[:5]} "
                               f"oracle {vo[key][bad[:5]]} gpu {vg[key][bad[:5]]}")


def run_parity(scn, steps, flags, full_every=1, t0=0, tile_cells=0, hash_every=1, group_cells=0):
    o = oracle.Oracle.from_scenario(scn, t0=t0)
    g = tsim.Sim.from_scenario(scn, t0=t0, flags=flags, tile_cells=tile_cells,
                               group_cells=group_cells)
    assert g.state_hash() == o.state_hash()
    assert_same_state(o, g, "init")
    done = 0
    while done < steps:
        n = min(hash_every, steps - done)
        t_from = o.t + 1
        ohash = o.run_hashes(n)  # oracle: one step at a time
        g.step(n)  # GPU: n steps in one call (fused lane change inside)
        done += n
        assert o.t == g.t
        if flags & tsim.FLAG_HASH:
            gh = g.history(t_from, n)["hash"]
            bad = [t_from + i for i in range(n) if gh[i] != ohash[i]]
            assert not bad, f"per-step hash differs at t={bad[:5]}"
        assert g.state_hash() == o.state_hash(), f"hash differs at t={o.t}"
        if full_every and (done % full_every == 0 or done == steps):
            assert_same_state(o, g, f"t={o.t}")
    return o, g


@pytest.mark.parametrize("case", range(24))
def test_small_rings(case):
    """single-tile periodic lanes (the tile's own strips as halos), 1-4
    lanes, every step in full"""
    rng = np.random.default_rng(900 + case)
    lanes = int(rng.integers(1, 5))
    L = int(rng.integers(10, 80))
    N = int(rng.integers(0, lanes * L))
    flat = np.sort(rng.choice(lanes * L, size=N, replace=False))
    vmax = int(rng.integers(1, 6))
    s = make_ring(L, flat // L, flat % L, rng.integers(0, vmax + 1, N), lanes=lanes,
                  vmax=vmax, p_slow=float(rng.choice([0.0, 0.2, 0.5])),
                  seed=int(rng.integers(1, 2**62)))
    run_parity(s, 60, FUSED if case % 2 else UNFUSED)


@pytest.mark.parametrize("tile_cells", [16, 37, 128, 512])
def test_ring_multi_tile(tile_cells):
    """segmented periodic link: halos and ghost moves across tile seams"""
    s = scenarios.ring(n_cells=3000, lanes=3, density=0.2, seed=5)
    run_parity(s, 150, FUSED, full_every=10, tile_cells=tile_cells)
    run_parity(s, 150, FUSED, full_every=0, tile_cells=tile_cells, hash_every=30)


@pytest.mark.parametrize("flags", [FUSED, UNFUSED, GENERAL])
def test_config1_full(flags):
    """BASELINE.json configs[0] for all 600 steps, one step per call"""
    s = scenarios.config("1")
    run_parity(s, 600, flags, full_every=20)


@pytest.mark.parametrize("flags", [FUSED, GENERAL])
@pytest.mark.parametrize("chunk", [7, 50])
def test_multistep_calls(flags, chunk):
    """several steps per ts_step call: the lane change of step t+1 runs
    inside the move kernel of step t; every per-step hash is checked"""
    s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=8, name="grid6c")
    run_parity(s, 400, flags, full_every=0, hash_every=chunk)
    s = scenarios.big_grid(rows=20, cols=20, seed=4, name="grid20dense")
    run_parity(s, 150, flags, full_every=0, hash_every=chunk)


@pytest.mark.parametrize("flags", [FUSED, UNFUSED, GENERAL])
def test_grid_with_departures(flags):
    """injection retries, conflicting entry cells, nodes at every step"""
    s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, steps=500, seed=7,
                             name="grid6b")
    run_parity(s, 500, flags, full_every=25)


def test_grid_segmented_links():
    """links longer than one tile: halo tiles on non-periodic links,
    injection and node records on segmented links"""
    s = scenarios.grid_trips(rows=4, cols=4, spacing_mm=1_500_000, lanes=3, n_veh=2500,
                             depart_max=200, seed=3, name="grid4long")
    run_parity(s, 400, UNFUSED, full_every=20, tile_cells=64)


@pytest.mark.parametrize("flags", [FUSED, GENERAL, "node_general"])
def test_portland_small(flags):
    """Portland-shaped network (row and general tiles, trips departing and
    arriving); "node_general": every node resolved by the thread-per-node
    kernel k_node (its grants by row slot, including the open end R12 of a
    front on its final link)"""
    if flags == "node_general":
        flags = NODE_GENERAL
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64,
                           seed=2)
    # departures compressed into the first 300 s
    s.depart = (s.depart // 12).astype(np.int32)
    run_parity(s, 400, flags, full_every=50)
    run_parity(s, 400, flags, full_every=0, hash_every=40)


# ------------------------------------- the benchmarked path, without the hash
BENCH = tsim.FLAG_FUSED  # exactly bench.py's flags (k_rows<5>, no hash instrument)


@pytest.mark.parametrize("chunk", [7, 25, 50])
@pytest.mark.parametrize("net", ["grid6", "grid24dense", "portland"])
def test_bench_flags_full_state(net, chunk):
    """bench.py's launch flags (FLAG_FUSED only: k_rows<5>, whose unchanged
    rows take the prefix-copy vid path): the full vehicle state (status,
    link, lane, cell, v, cursor, arrival) against the oracle after every
    call of `chunk` steps, so two vids swapped inside a row would fail"""
    if net == "grid6":
        s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=8, name="grid6nh")
        steps = 300
    elif net == "grid24dense":
        s = scenarios.big_grid(rows=24, cols=24, seed=3, name="grid24dense_nh")
        steps = 100
    else:
        s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64,
                               seed=2)
        s.depart = (s.depart // 12).astype(np.int32)
        steps = 300
    run_parity(s, steps, BENCH, full_every=chunk, hash_every=chunk)


@pytest.mark.parametrize("net,group_cells", [("grid6", 64), ("grid24dense", 64), ("grid24dense", 512),
                                             ("portland", 96)])
def test_unstaged_groups(net, group_cells):
    """the row kernel's paths for a 32-row group whose vehicles exceed its
    shared-memory staging (vid blocks read and written in HBM, draws and
    vid lists out of line): a small staging capacity (group_cells) sends
    most or some groups there; injections, lane changes and node traffic
    included; bench flags and hashed fused flags, full state checked"""
    if net == "grid6":
        s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=8, name="grid6u")
        steps = 200
    elif net == "grid24dense":
        s = scenarios.big_grid(rows=24, cols=24, seed=3, name="grid24dense_u")
        steps = 60
    else:
        s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64,
                               seed=2)
        s.depart = (s.depart // 12).astype(np.int32)
        steps = 200
    run_parity(s, steps, BENCH, full_every=20, hash_every=20, group_cells=group_cells)
    run_parity(s, steps // 2, FUSED, full_every=10, hash_every=10, group_cells=group_cells)


def test_big_grid_dense():
    """config-4a recipe (density 0.2, 4 lanes, 100-cell links, Manhattan
    routes) on a 24x24 lattice: heavy lane changing and node traffic"""
    s = scenarios.big_grid(rows=24, cols=24, seed=3, name="grid24dense")
    run_parity(s, 200, FUSED, full_every=20)


def test_t0_and_odd_start():
    s = scenarios.ring(n_cells=500, lanes=3, density=0.3, seed=9)
    run_parity(s, 50, FUSED, t0=7)


def test_handmade_intersections():
    nodes = [(0, 0), (1000, 0), (-1000, 0), (0, 1000), (0, -1000)]
    links = [(2, 0, 1000, 2, 1), (0, 1, 1000, 2, 1), (1, 0, 1000, 2, 1), (0, 2, 1000, 2, 1),
             (4, 0, 1000, 2, 0), (0, 3, 1000, 2, 0), (3, 0, 1000, 2, 0), (0, 4, 1000, 2, 0)]
    rng = np.random.default_rng(4)
    routes = [[0, 1], [0, 5], [0, 7], [0, 3], [2, 3], [2, 5], [2, 7], [4, 5], [4, 1], [4, 3],
              [6, 7], [6, 1], [6, 3], [1], [3], [5], [7]]
    veh = []
    for i in range(400):
        r = routes[int(rng.integers(len(routes)))]
        veh.append(dict(route=r, depart=int(rng.integers(0, 120)),
                        entry=int(rng.integers(0, 120))))
    s = make_network(nodes, links, veh, p_slow=0.25, seed=11)
    run_parity(s, 300, FUSED)


def test_config2_full_size_prefix():
    """BASELINE.json configs[1] at full size (3 x 1,000,000 cells, 450,000
    vehicles): hash every step for 40 steps, full state at the end"""
    s = scenarios.config("2")
    run_parity(s, 40, FUSED, full_every=40)


def test_history_stream():
    s = scenarios.config("1")
    o = oracle.Oracle.from_scenario(s)
    g = tsim.Sim.from_scenario(s, flags=FUSED)
    g.step(100)
    hist = g.history(1, 100)
    for t in range(100):
        o.step(1)
        assert hist["hash"][t] == o.state_hash(), t
        assert hist["active"][t] == o.counters()["active"]


# ---------------------------------------------------- signals
NODE_GENERAL = tsim.FLAG_FUSED | tsim.FLAG_HASH | 32  # TS_FLAG_NODE_GENERAL: thread-per-node kernel


@pytest.mark.parametrize("flags", [FUSED, UNFUSED, GENERAL, NODE_GENERAL])
def test_signalized_grid(flags):
    """config 1 with fixed-time 30 s / 30 s signals at every node (reading
    R23): red approaches see the virtual blocker, green
    ones cross without gap acceptance; bit-exact against the oracle"""
    s = scenarios.with_signals(scenarios.config("1"), seed=3)
    run_parity(s, 300, flags, full_every=25, hash_every=25)


@pytest.mark.parametrize("g0,g1", [(1, 1), (7, 23), (45, 5)])
def test_signalized_portland(g0, g1):
    """unequal phases and short cycles on the Portland-shaped network (mixed
    row and general tiles, nodes of in-degree up to the network's maximum)"""
    s = scenarios.portland(n_nodes=400, n_edges=560, n_veh=5000, side_km=6.0, n_zones=48, seed=5)
    s.depart = (s.depart // 20).astype(np.int32)
    s = scenarios.with_signals(s, green0=g0, green1=g1, seed=g0)
    run_parity(s, 250, FUSED, full_every=50, hash_every=50)


# ------------------------------------------- CUDA-graph replay (TS_FLAG_GRAPH)
GRAPH = FUSED | tsim.FLAG_GRAPH
GRAPH_GENERAL = GENERAL | tsim.FLAG_GRAPH


@pytest.mark.parametrize("chunk", [15, 47, 100])
def test_graph_replay_grid(chunk):
    """steps replayed from one captured graph of 15 steps (the step time read
    from the device clock) plus normally launched remainders: every
    per-step hash equals the oracle's"""
    s = scenarios.grid_trips(rows=6, cols=6, n_veh=3000, depart_max=300, seed=8, name="grid6g")
    run_parity(s, 400, GRAPH, full_every=0, hash_every=chunk)
    s = scenarios.big_grid(rows=20, cols=20, seed=4, name="grid20g")
    run_parity(s, 150, GRAPH, full_every=0, hash_every=chunk)


@pytest.mark.parametrize("flags", [GRAPH, GRAPH_GENERAL])
def test_graph_replay_mixed(flags):
    """row and general tiles, signals, long links, injection: graph replays
    across 400 steps, full state checked after every call"""
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64, seed=2)
    s.depart = (s.depart // 12).astype(np.int32)
    s = scenarios.with_signals(s, green0=20, green1=25, seed=4)
    run_parity(s, 400, flags, full_every=1, hash_every=45)


def test_graph_replay_ring():
    """the periodic ring (general tiles only, lane change not fusable)"""
    s = scenarios.ring(n_cells=3000, lanes=3, density=0.2, seed=5)
    run_parity(s, 150, GRAPH, full_every=1, hash_every=30)


def test_config4a_full_size_prefix():
    """BASELINE.json configs[3] at full size (256 x 256 nodes, 104,448,000
    lane-cells, 20,889,600 vehicles at density 0.2) in the bench's launch
    configuration: per-step hash and full state against the oracle for the
    first steps.  Routes are short (destination within 4 rows / columns) so
    the oracle's copy fits the host; cells, vehicles and kernels are the
    bench's."""
    s = scenarios.big_grid(seed=1, dest_radius=4, name="config4a_full_shortroutes")
    assert s.n_vehicles == 20_889_600
    run_parity(s, 3, tsim.FLAG_FUSED | tsim.FLAG_HASH, full_every=3, hash_every=3)


def test_spec_text_files_load():
    """network and plans in the SPEC text formats (ts_load_network_text /
    ts_load_plans_text) give the same run as the array loaders"""
    s = scenarios.config("1")
    ids = np.arange(s.n_links) * 10 + 3  # arbitrary file ids
    net = ["NODES"] + [f"{i + 100} {x / 1000} {y / 1000}" for i, (x, y) in
                       enumerate(zip(s.node_x, s.node_y))]
    net += ["LINKS"] + [f"{ids[k]} {a + 100} {b + 100} {ln / 1000} {la} {vm}" for k, (a, b, ln, la, vm)
                        in enumerate(zip(s.link_from, s.link_to, s.link_len_mm, s.link_lanes,
                                         s.link_vmax))]
    plans = [f"{f} {s.depart[f]} {s.entry[f]} " +
             " ".join(str(ids[k]) for k in s.route[s.route_off[f]:s.route_off[f + 1]])
             for f in range(s.n_vehicles)]
    # the text network's class is the lane count (R9): align the array run
    s.link_class = np.asarray(s.link_lanes, np.int32).copy()
    o = oracle.Oracle.from_scenario(s)
    g = tsim.Sim(p_slow=s.p_slow, seed=s.seed, flags=FUSED)
    g.load_text("\n".join(net) + "\n", "\n".join(plans) + "\n")
    g.init(0)
    assert g.state_hash() == o.state_hash()
    oh = o.run_hashes(200)
    g.step(200)
    assert list(g.history(1, 200)["hash"]) == list(oh)


# ------------------------------------------------------------- edge cases
@pytest.mark.parametrize("p", [0.0, 1.0])
def test_degenerate_slowdown_probabilities(p):
    """p = 0 (no draw ever brakes: the unique deterministic trajectory,
    R22) and p = 1 (every mover brakes, P32 = 2^32 compares as 64-bit)"""
    s = scenarios.big_grid(rows=8, cols=8, seed=6, name="grid8p")
    s.p_slow = p
    run_parity(s, 120, FUSED, full_every=40, hash_every=40)
    r = scenarios.ring(n_cells=2000, lanes=3, density=0.3, seed=4)
    r.p_slow = p
    run_parity(r, 120, FUSED, full_every=40, hash_every=40)


def test_empty_networks():
    """no vehicles at all: every step runs (and exchanges), the state stays
    empty, the hash is 0"""
    s = scenarios.grid_trips(rows=4, cols=4, n_veh=0, name="grid_empty")
    o, g = run_parity(s, 30, FUSED, full_every=10, hash_every=10)
    assert g.state_hash() == 0 and g.totals()["active"] == 0
    r = scenarios.ring(n_cells=500, lanes=2, n_veh=0, seed=1)
    o, g = run_parity(r, 30, FUSED, full_every=10, hash_every=10)
    assert g.state_hash() == 0


@pytest.mark.parametrize("cells", [128, 129])
def test_row_width_limit(cells):
    """links of exactly 128 cells (row tiles with all four 32-cell words
    full: the last cell is bit 31 of word 3) and of 129 (one cell too many
    for a row: general tiles), dense, 4 lanes, bench and hashed flags"""
    s = scenarios.big_grid(rows=8, cols=8, lanes=4, cells=cells, density=0.25, seed=11,
                           name=f"grid8w{cells}")
    run_parity(s, 120, BENCH, full_every=20, hash_every=20)
    run_parity(s, 60, FUSED, full_every=20, hash_every=20)


def test_eight_lane_links_and_minimum_ring():
    """the widest links (8 lanes, kMaxLanes) on a dense grid, and the
    smallest ring (10 cells, one segment that is its own neighbour)"""
    s = scenarios.big_grid(rows=6, cols=6, lanes=8, cells=40, density=0.25, seed=9,
                           name="grid6x8lanes")
    run_parity(s, 120, FUSED, full_every=30, hash_every=30)
    r = scenarios.ring(n_cells=10, lanes=3, n_veh=9, seed=2)
    run_parity(r, 200, FUSED, full_every=20, hash_every=20)
