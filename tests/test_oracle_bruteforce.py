"""Brute-force pins of the oracle's lane-change and intersection rules
(SURVEY.md §8(c) "What pins each part": "brute force over the last and first
5 cells on a tiny T-junction").

The oracle's one-step result on thousands of independent junction copies
(one network, one oracle run) is compared with ``tests/_ref_net.py``, an
independent vehicle-list implementation written from PAPER.md §3 and the
readings R4-R12 -- different data structure, no shared code.  A mistake in
the candidate condition, the gap acceptance, the tie order between approach
links, the entry lane or the entry space (R8-R10), or in the desperation
schedule R6 at any distance 0 < d < D, fails one of these.
"""
import itertools

import numpy as np
import pytest

import oracle
import scenarios
from tests import _ref_net as rn

M = 75_000  # 10 cells, mm


def build(nodes, links, vehicles, p_slow, seed):
    """scenario from (x, y) nodes in mm, links (from, to, cells, lanes, class)
    and vehicles (route, lane, cell, v) placed on route[0] at t0"""
    i32 = lambda a: np.asarray(a, np.int32)  # noqa: E731
    routes = [v[0] for v in vehicles]
    off = np.zeros(len(routes) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in routes])
    n = len(vehicles)
    s = scenarios.Scenario(
        name="bruteforce", node_x=np.asarray([p[0] for p in nodes], np.int64),
        node_y=np.asarray([p[1] for p in nodes], np.int64),
        link_from=i32([a[0] for a in links]), link_to=i32([a[1] for a in links]),
        link_len_mm=np.asarray([a[2] * 7500 for a in links], np.int64),
        link_lanes=i32([a[3] for a in links]), link_vmax=i32([5] * len(links)),
        link_class=i32([a[4] for a in links]), periodic_link=-1, route_off=off,
        route=i32([k for r in routes for k in r]), depart=i32([0] * n),
        entry=i32([v[2] for v in vehicles]), place_vid=i32(np.arange(n)),
        place_lane=i32([v[1] for v in vehicles]), place_cell=i32([v[2] for v in vehicles]),
        place_v=i32([v[3] for v in vehicles]), p_slow=p_slow, seed=seed)
    net = rn.Net(s.node_x, s.node_y, s.link_from, s.link_to, s.link_len_mm, s.link_lanes,
                 s.link_vmax, s.link_class, routes)
    state = {f: [v[0][0], v[1], v[2], v[3], 0] for f, v in enumerate(vehicles)}
    return s, net, state


def compare_one_step(s, net, state, t0, steps=1):
    """oracle vs reference, `steps` steps from S(t0); returns the reference
    state after the last step"""
    o = oracle.Oracle.from_scenario(s, t0=t0)
    arrived = set()
    for i in range(steps):
        t = t0 + i
        state, arr = rn.step(net, state, t, s.seed, s.p_slow)
        arrived |= set(arr)
        o.step(1)
        vo = o.vehicles()
        assert o.counters()["collisions"] == 0
        for f in range(s.n_vehicles):
            if f in arrived:
                assert vo["status"][f] == oracle.ARRIVED, (t, f)
                continue
            k, l, x, v, cur = state[f]
            got = (int(vo["link"][f]), int(vo["lane"][f]), int(vo["cell"][f]), int(vo["v"][f]),
                   int(vo["cursor"][f]))
            assert got == (k, l, x, v, cur), f"t={t + 1} vid {f}: oracle {got} reference {(k, l, x, v, cur)}"
    return state


# ------------------------------------------------------------ plus nodes
def plus_copies(n_copies, rng, two_lane_p=0.5):
    """independent 4-way junctions: W/E approaches major (class 1), N/S minor
    (class 0); lanes 1 or 2 per link; random occupancy and velocity of every
    cell of every approach (denser in the last 5) and exit"""
    nodes, links, veh = [], [], []
    arms = [(-M, 0), (M, 0), (0, M), (0, -M)]  # W, E, N, S
    for c in range(n_copies):
        cx, cy = (c % 60) * 4 * M, (c // 60) * 4 * M
        base = len(nodes)
        nodes.append((cx, cy))
        for ax, ay in arms:
            nodes.append((cx + ax, cy + ay))
        lb = len(links)
        for a in range(4):  # approaches a -> centre: links lb + a
            L = 2 if rng.random() < two_lane_p else 1
            links.append((base + 1 + a, base, 10, L, 1 if a < 2 else 0))
        for a in range(4):  # exits centre -> arm a: links lb + 4 + a
            L = 2 if rng.random() < two_lane_p else 1
            links.append((base, base + 1 + a, 10, L, 1 if a < 2 else 0))
        for a in range(4):
            k, L = lb + a, links[lb + a][3]
            for l in range(L):
                for x in range(10):
                    if rng.random() < (0.55 if x >= 5 else 0.3):
                        exits = [lb + 4 + b for b in range(4) if b != a]  # no U-turns
                        r = [k] if rng.random() < 0.1 else [k, int(rng.choice(exits))]
                        veh.append((r, l, x, int(rng.integers(0, 6))))
        for a in range(4):
            k, L = lb + 4 + a, links[lb + 4 + a][3]
            for l in range(L):
                for x in range(10):
                    if rng.random() < (0.4 if x < 5 else 0.2):
                        veh.append(([k], l, x, int(rng.integers(0, 6))))
    return nodes, links, veh


@pytest.mark.parametrize("t0", [0, 1])
@pytest.mark.parametrize("p", [0.0, 0.2])
def test_plus_nodes_one_step(t0, p):
    """3,000 random 4-way junctions, 1-2 lanes per link: the oracle's step
    (lane change incl. both turn lanes, candidates, gap acceptance, one
    winner per target lane by (class, link, lane), entry lane and entry
    space, move, exit) equals the reference for every vehicle"""
    rng = np.random.default_rng(100 + 10 * t0 + int(p * 10))
    nodes, links, veh = plus_copies(3000, rng)
    s, net, state = build(nodes, links, veh, p, seed=12345 + t0)
    compare_one_step(s, net, state, t0)


def test_plus_nodes_many_steps():
    """the same junctions for 12 steps (vehicles cross, queue, exit): the
    reference and the oracle stay identical"""
    rng = np.random.default_rng(7)
    nodes, links, veh = plus_copies(600, rng)
    s, net, state = build(nodes, links, veh, 0.2, seed=99)
    compare_one_step(s, net, state, 0, steps=12)


# ------------------------------------------------------- T-junction, exhaustive
def test_t_junction_exhaustive():
    """every combination of the front vehicle of the three approaches of a
    T-junction (majors W->C, E->C class 1; minor S->C class 0; one lane):
    absent, or at distance d = 0..4 from the stop line (v = 5, a candidate)
    turning to either of its two exits; times every occupancy of the first
    cell of the three exits: 11^3 x 2^3 = 10,648 junctions in one network"""
    nodes, links, veh = [], [], []
    arms = [(-M, 0), (M, 0), (0, -M)]  # W, E, S
    opts = [None] + [(d, e) for d in range(5) for e in range(2)]
    combos = list(itertools.product(opts, opts, opts, range(8)))
    for c, (o0, o1, o2, occ) in enumerate(combos):
        cx, cy = (c % 100) * 4 * M, (c // 100) * 4 * M
        base = len(nodes)
        nodes.append((cx, cy))
        for ax, ay in arms:
            nodes.append((cx + ax, cy + ay))
        lb = len(links)
        for a in range(3):
            links.append((base + 1 + a, base, 10, 1, 1 if a < 2 else 0))
        for a in range(3):
            links.append((base, base + 1 + a, 10, 1, 1 if a < 2 else 0))
        for a, opt in enumerate((o0, o1, o2)):
            if opt is None:
                continue
            d, e = opt
            exits = [lb + 3 + b for b in range(3) if b != a]
            veh.append(([lb + a, exits[e]], 0, 9 - d, 5))
        for b in range(3):
            if (occ >> b) & 1:
                veh.append(([lb + 3 + b], 0, 0, 0))
    s, net, state = build(nodes, links, veh, 0.0, seed=1)
    compare_one_step(s, net, state, 0)


# ------------------------------------------------------- desperation (R6)
def desperation_copies(turn_left, d_max=11):
    """a wrong-lane vehicle wanting its turn lane at every distance d =
    0..d_max from the stop line and speed v = 0..5, against every occupancy
    of the target lane in the 5 cells behind and ahead of it (and its own
    cell there); its exit is blocked at cell 0 so it stays on the link"""
    nodes, links, veh, cases = [], [], [], []
    sgn = 1 if turn_left else -1
    for c, (d, v, pat) in enumerate(itertools.product(range(d_max + 1), range(6), range(2048))):
        cx, cy = (c % 200) * 6 * M, (c // 200) * 6 * M
        base = len(nodes)
        nodes += [(cx, cy), (cx + 2 * M, cy), (cx + 2 * M, cy + sgn * M)]
        lb = len(links)
        links.append((base, base + 1, 20, 2, 1))   # approach, 20 cells, 2 lanes
        links.append((base + 1, base + 2, 10, 2, 1))  # the turn, blocked at cell 0
        x = 19 - d
        own, tgt = (0, 1) if turn_left else (1, 0)
        veh.append(([lb, lb + 1], own, x, v))
        cases.append((len(veh) - 1, d, v, pat, x, own, tgt))
        for j in range(11):  # target-lane cells x-5 .. x+5
            y = x - 5 + j
            if (pat >> j) & 1 and 0 <= y <= 19:
                veh.append(([lb], tgt, y, 0))
        veh.append(([lb + 1], 0, 0, 0))
        veh.append(([lb + 1], 1, 0, 0))
    return nodes, links, veh, cases


@pytest.mark.parametrize("turn_left", [True, False])
def test_desperation_schedule_enumerated(turn_left):
    """R6 ("accepted gap decreases with decreasing
    distance"): for d = 0..11, v = 0..5 and all 2^11 target-lane patterns,
    the oracle's lane-change decision equals the scalar rule: target cell
    empty, free cells ahead (to the link end, <= 5) >= floor(min(v+1,5)
    min(d,D)/D) ... written out below, and free cells behind (before the link
    start empty) >= floor(5 min(d,D)/D).  Left turns change lane 0 -> 1 on
    even t; right turns lane 1 -> 0 on odd t."""
    nodes, links, veh, cases = desperation_copies(turn_left)
    s, net, state = build(nodes, links, veh, 0.0, seed=1)
    t0 = 0 if turn_left else 1
    o = oracle.Oracle.from_scenario(s, t0=t0)
    o.step(1)
    lane = o.vehicles()["lane"]
    n_change = 0
    for f, d, v, pat, x, own, tgt in cases:
        occ = {x - 5 + j for j in range(11) if (pat >> j) & 1 and 0 <= x - 5 + j <= 19}
        free_ahead = 0
        while free_ahead < 5 and x + free_ahead + 1 <= 19 and (x + free_ahead + 1) not in occ:
            free_ahead += 1
        free_behind = 0
        while free_behind < 5 and (x - free_behind - 1) not in occ:
            free_behind += 1
        D = 10
        need_f = min(v + 1, 5) if d >= D else (min(v + 1, 5) * d) // D
        need_b = 5 if d >= D else (5 * d) // D
        expect = x not in occ and free_ahead >= need_f and free_behind >= need_b
        n_change += expect
        assert lane[f] == (tgt if expect else own), (
            f"d={d} v={v} pattern={pat:011b}: oracle lane {lane[f]}, expected "
            f"{'change' if expect else 'stay'} (ahead {free_ahead} >= {need_f}, "
            f"behind {free_behind} >= {need_b})")
    assert 0 < n_change < len(cases)


# --------------------------------------------------- small grid, many steps
def test_grid_many_steps_vs_reference():
    """a 4x4 two-lane grid (config-1 shape) with 700 placed vehicles on random
    no-U-turn routes: 60 steps, every vehicle after every step"""
    base = scenarios.grid_trips(rows=4, cols=4, n_veh=700, seed=21, name="bf_grid")
    rng = np.random.default_rng(5)
    n_cells = (np.asarray(base.link_len_mm) + 3750) // 7500
    taken = set()
    veh = []
    for f in range(base.n_vehicles):
        r = base.route[base.route_off[f]:base.route_off[f + 1]].tolist()
        k = r[0]
        for _ in range(20):
            l, x = int(rng.integers(0, base.link_lanes[k])), int(rng.integers(0, n_cells[k]))
            if (k, l, x) not in taken:
                taken.add((k, l, x))
                veh.append((r, l, x, int(rng.integers(0, 6))))
                break
    nodes = list(zip(base.node_x.tolist(), base.node_y.tolist()))
    links = [(int(a), int(b), int(n), int(L), int(c)) for a, b, n, L, c in
             zip(base.link_from, base.link_to, n_cells, base.link_lanes, base.link_class)]
    s, net, state = build(nodes, links, veh, 0.2, seed=3)
    compare_one_step(s, net, state, 0, steps=60)
