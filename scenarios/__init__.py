"""Seeded synthetic scenario generators (shared INPUT module).

This module produces plain arrays -- road network, routes, departures,
initial placements -- that both the CPU oracle (``oracle/``) and the CUDA
library (``paper_cs_0105004_b200``) consume.  It contains none of the
method's arithmetic: no cell discretisation (R1), no turn classification
(R7), no driving rule.  Link lengths are given in integer millimetres and the
simulators discretise them themselves.

The recipes follow BASELINE.json ``configs`` and SURVEY.md §8(d) (restated
in DESIGN.md §5).  The paper's own workloads (Portland EMME/2 20,024 links,
TIGER 200k links, Dallas) are not available; the
Portland-shaped generator stands in for them.
"""
from __future__ import annotations

import ctypes
import dataclasses
import heapq
import os
import subprocess

import numpy as np

CELL_MM = 7500  # only used to size link lengths as whole cells

_HERE = os.path.dirname(os.path.abspath(__file__))


@dataclasses.dataclass
class Scenario:
    name: str
    node_x: np.ndarray  # int64 mm
    node_y: np.ndarray  # int64 mm
    link_from: np.ndarray  # int32
    link_to: np.ndarray  # int32
    link_len_mm: np.ndarray  # int64
    link_lanes: np.ndarray  # int32
    link_vmax: np.ndarray  # int32
    link_class: np.ndarray  # int32
    periodic_link: int
    route_off: np.ndarray  # int64 [nv+1]
    route: np.ndarray  # int32
    depart: np.ndarray  # int32
    entry: np.ndarray  # int32
    place_vid: np.ndarray  # int32 (active at t0)
    place_lane: np.ndarray
    place_cell: np.ndarray
    place_v: np.ndarray
    steps: int = 100
    p_slow: float = 0.2
    seed: int = 1
    recipe: str = ""
    # fixed-time signals (reading R23): node ids, green of phase 0 / 1, offset
    sig_node: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))
    sig_g0: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))
    sig_g1: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))
    sig_off: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))

    @property
    def n_nodes(self) -> int:
        return int(self.node_x.shape[0])

    @property
    def n_links(self) -> int:
        return int(self.link_from.shape[0])

    @property
    def n_vehicles(self) -> int:
        return int(self.depart.shape[0])


def with_signals(scn, nodes=None, green0=30, green1=30, offset=None, seed=0):
    """the same scenario with fixed-time two-phase signals (reading R23) at
    `nodes` (default: every node with >= 2 incoming links); offsets seeded
    uniform in [0, cycle) unless given"""
    import copy
    s = copy.copy(scn)
    if nodes is None:
        indeg = np.bincount(np.asarray(scn.link_to), minlength=scn.n_nodes)
        nodes = np.nonzero(indeg >= 2)[0]
    nodes = _i32(nodes)
    n = nodes.size
    if offset is None:
        offset = np.random.default_rng(seed).integers(0, green0 + green1, n)
    s.sig_node = nodes
    s.sig_g0 = _i32(np.broadcast_to(green0, n))
    s.sig_g1 = _i32(np.broadcast_to(green1, n))
    s.sig_off = _i32(np.broadcast_to(offset, n))
    s.name = scn.name + "_signals"
    s.recipe = scn.recipe + f"; fixed-time signals {green0}/{green1} s at {n} nodes"
    return s


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _empty_place():
    e = np.zeros(0, dtype=np.int32)
    return e, e.copy(), e.copy(), e.copy()


# ------------------------------------------------------------------ networks
def grid_network(rows: int, cols: int, spacing_mm: int, lanes: int, vmax: int = 5):
    """rows x cols lattice, both directions on every edge.

    Link numbering (shared with gen_routes.c): east links, west links, north
    links, south links.  Horizontal links have priority class 1, vertical 0
    ("horizontal major").
    """
    assert rows >= 2 and cols >= 2
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    node_x = (c.ravel() * spacing_mm).astype(np.int64)
    node_y = (r.ravel() * spacing_mm).astype(np.int64)
    nid = lambda rr, cc: rr * cols + cc  # noqa: E731
    hr, hc = np.meshgrid(np.arange(rows), np.arange(cols - 1), indexing="ij")
    vr, vc = np.meshgrid(np.arange(rows - 1), np.arange(cols), indexing="ij")
    hr, hc, vr, vc = hr.ravel(), hc.ravel(), vr.ravel(), vc.ravel()
    east = (nid(hr, hc), nid(hr, hc + 1))
    west = (nid(hr, hc + 1), nid(hr, hc))
    north = (nid(vr, vc), nid(vr + 1, vc))
    south = (nid(vr + 1, vc), nid(vr, vc))
    frm = np.concatenate([east[0], west[0], north[0], south[0]])
    to = np.concatenate([east[1], west[1], north[1], south[1]])
    nh, nv = hr.size, vr.size
    cls = np.concatenate([np.ones(2 * nh), np.zeros(2 * nv)])
    nl = frm.size
    return dict(
        node_x=node_x,
        node_y=node_y,
        link_from=_i32(frm),
        link_to=_i32(to),
        link_len_mm=np.full(nl, spacing_mm, dtype=np.int64),
        link_lanes=np.full(nl, lanes, dtype=np.int32),
        link_vmax=np.full(nl, vmax, dtype=np.int32),
        link_class=_i32(cls),
    )


def successors(link_from, link_to, n_nodes):
    """Line graph of the network: k -> k2 when to(k) == from(k2), without
    U-turns unless the node is a dead end (SURVEY.md §8(d) "no-U-turn")."""
    out = [[] for _ in range(n_nodes)]
    for k2, a in enumerate(link_from.tolist()):
        out[a].append(k2)
    succ = []
    for k in range(link_from.size):
        h, tail = int(link_to[k]), int(link_from[k])
        s = [k2 for k2 in out[h] if int(link_to[k2]) != tail]
        if not s:
            s = list(out[h])
        succ.append(sorted(s))
    return succ


def dijkstra_route(succ, cost, o, q):
    """Shortest link path o -> q (cost = length of each entered link); ties
    resolve to the lower link id through the heap order."""
    dist = {o: 0}
    pred = {o: -1}
    heap = [(0, o)]
    done = set()
    while heap:
        d, k = heapq.heappop(heap)
        if k in done:
            continue
        done.add(k)
        if k == q:
            break
        for k2 in succ[k]:
            nd = d + int(cost[k2])
            if k2 not in dist or nd < dist[k2]:
                dist[k2] = nd
                pred[k2] = k
                heapq.heappush(heap, (nd, k2))
    if q not in done:
        return None
    path = [q]
    while path[-1] != o:
        path.append(pred[path[-1]])
    return path[::-1]


def _routes_csr(routes):
    off = np.zeros(len(routes) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(r) for r in routes])
    flat = np.fromiter((k for r in routes for k in r), dtype=np.int32, count=int(off[-1]))
    return off, flat


# ------------------------------------------------------------------- config 1
def grid_trips(rows=4, cols=4, spacing_mm=500_000, lanes=2, n_veh=1000, seed=1,
               steps=600, depart_max=0, name="config1_grid4x4", od_cols=None):
    """BASELINE.json configs[0]: 4x4 grid, 48 links of 500 m (67 cells),
    2 lanes, unsignalled priority intersections, 1,000 vehicles with seeded
    random shortest-path routes, all departing at t = 0 on lane 0.
    od_cols=(c0, c1) (tests): origins and destinations only on links between
    nodes of columns c0..c1 (a spatially concentrated load)."""
    net = grid_network(rows, cols, spacing_mm, lanes)
    rng = np.random.default_rng(seed)
    nl = net["link_from"].size
    succ = successors(net["link_from"], net["link_to"], rows * cols)
    pool = np.arange(nl)
    if od_cols is not None:
        cf, ct = net["link_from"] % cols, net["link_to"] % cols
        pool = np.nonzero((cf >= od_cols[0]) & (cf <= od_cols[1]) &
                          (ct >= od_cols[0]) & (ct <= od_cols[1]))[0]
    routes = []
    for _ in range(n_veh):
        while True:
            o, q = (int(pool[v]) for v in rng.integers(0, pool.size, size=2))
            if o == q:
                continue
            r = dijkstra_route(succ, net["link_len_mm"], o, q)
            if r is not None:
                break
        routes.append(r)
    off, flat = _routes_csr(routes)
    first = flat[off[:-1]]
    span = net["link_len_mm"][first] // CELL_MM  # entry cell in [0, len/7.5 m)
    entry = (rng.random(n_veh) * span).astype(np.int32)
    depart = rng.integers(0, depart_max + 1, size=n_veh).astype(np.int32)
    pv, pl, pc, pvv = _empty_place()
    return Scenario(name=name, periodic_link=-1, route_off=off, route=flat,
                    depart=depart, entry=entry, place_vid=pv, place_lane=pl,
                    place_cell=pc, place_v=pvv, steps=steps, seed=seed,
                    recipe=f"grid {rows}x{cols}, {spacing_mm/1000:.0f} m links, "
                           f"{lanes} lanes, {n_veh} vehicles, no-U-turn Dijkstra routes",
                    **net)


# ------------------------------------------------------------------- config 2
def ring(n_cells=1_000_000, lanes=3, density=0.15, n_veh=None, seed=1, steps=1000,
         vmax=5, v_init="uniform", name="config2_ring"):
    """BASELINE.json configs[1]: one periodic link, lanes x n_cells, vehicles
    at distinct lane-cells uniformly without replacement, velocities uniform
    in 0..vmax, vids in flat (lane, cell) order."""
    rng = np.random.default_rng(seed)
    total = n_cells * lanes
    if n_veh is None:
        n_veh = int(round(density * total))
    flat_cells = np.sort(rng.choice(total, size=n_veh, replace=False)).astype(np.int64)
    lane = (flat_cells // n_cells).astype(np.int32)
    cell = (flat_cells % n_cells).astype(np.int32)
    if v_init == "uniform":
        v = rng.integers(0, vmax + 1, size=n_veh).astype(np.int32)
    else:
        v = np.full(n_veh, int(v_init), dtype=np.int32)
    vid = np.arange(n_veh, dtype=np.int32)
    off = np.arange(n_veh + 1, dtype=np.int64)
    return Scenario(
        name=name, node_x=np.zeros(1, np.int64), node_y=np.zeros(1, np.int64),
        link_from=_i32([0]), link_to=_i32([0]),
        link_len_mm=_i64([n_cells * CELL_MM]), link_lanes=_i32([lanes]),
        link_vmax=_i32([vmax]), link_class=_i32([0]), periodic_link=0,
        route_off=off, route=np.zeros(n_veh, np.int32),
        depart=np.zeros(n_veh, np.int32), entry=cell.copy(),
        place_vid=vid, place_lane=lane, place_cell=cell, place_v=v,
        steps=steps, seed=seed,
        recipe=f"periodic ring {lanes} x {n_cells} cells, {n_veh} vehicles "
               f"(density {n_veh/total:.4f}), v uniform 0..{vmax}")


# ------------------------------------------------------------------- config 4
_libgen = None


def _gen_lib():
    global _libgen
    if _libgen is None:
        so = os.path.join(_HERE, "libgen_routes.so")
        src = os.path.join(_HERE, "gen_routes.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", so, src])
        lib = ctypes.CDLL(so)
        P = ctypes.c_void_p
        lib.manhattan_lengths.argtypes = [ctypes.c_int64, P, P, ctypes.c_int64, ctypes.c_int64, P]
        lib.manhattan_fill.argtypes = [ctypes.c_int64, P, P, ctypes.c_int64, ctypes.c_int64, P, P]
        _libgen = lib
    return _libgen


def big_grid(rows=256, cols=256, cells=100, lanes=4, density=0.2, n_veh=None,
             seed=1, steps=3600, name="config4a_grid256", dest_radius=None):
    """BASELINE.json configs[3]: rows x cols
    lattice of `cells`-cell links with `lanes` lanes; vehicles placed at t = 0
    uniformly without replacement at v = 0; destination node uniform; route
    = canonical x-then-y Manhattan path from the head node of the first link
    (U-turns allowed).  dest_radius (tests only): destination uniform within
    +-dest_radius rows / columns of the first link's head node instead, so
    the full-size network carries short routes (small host memory)."""
    net = grid_network(rows, cols, cells * CELL_MM, lanes)
    rng = np.random.default_rng(seed)
    nl = net["link_from"].size
    per_link = lanes * cells
    total = nl * per_link
    if n_veh is None:
        n_veh = int(round(density * total))
    flat = np.sort(rng.choice(total, size=n_veh, replace=False))
    first = (flat // per_link).astype(np.int32)
    rem = flat % per_link
    lane = (rem // cells).astype(np.int32)
    cell = (rem % cells).astype(np.int32)
    del flat, rem
    dest = rng.integers(0, rows * cols, size=n_veh).astype(np.int32)
    if dest_radius is not None:
        head = np.asarray(net["link_to"])[first].astype(np.int64)
        hr, hc = head // cols, head % cols
        dr = np.clip(hr + rng.integers(-dest_radius, dest_radius + 1, n_veh), 0, rows - 1)
        dc = np.clip(hc + rng.integers(-dest_radius, dest_radius + 1, n_veh), 0, cols - 1)
        dest = (dr * cols + dc).astype(np.int32)
    lib = _gen_lib()
    lens = np.empty(n_veh, dtype=np.int64)
    lib.manhattan_lengths(n_veh, first.ctypes.data, dest.ctypes.data, rows, cols, lens.ctypes.data)
    off = np.zeros(n_veh + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    route = np.empty(int(off[-1]), dtype=np.int32)
    lib.manhattan_fill(n_veh, first.ctypes.data, dest.ctypes.data, rows, cols,
                       off.ctypes.data, route.ctypes.data)
    vid = np.arange(n_veh, dtype=np.int32)
    return Scenario(name=name, periodic_link=-1, route_off=off, route=route,
                    depart=np.zeros(n_veh, np.int32), entry=cell.copy(),
                    place_vid=vid, place_lane=lane, place_cell=cell,
                    place_v=np.zeros(n_veh, np.int32), steps=steps, seed=seed,
                    recipe=f"grid {rows}x{cols}, {cells}-cell links, {lanes} lanes, "
                           f"{n_veh} vehicles placed uniformly (density {n_veh/total:.4f}), "
                           "x-then-y Manhattan routes to a uniform destination node",
                    **net)


# ------------------------------------------------------------------- config 3
def _planar_network(rng, n_nodes, n_edges, side_mm, x0=0, y0=0):
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import minimum_spanning_tree
    from scipy.spatial import Delaunay

    pts = rng.uniform(0, side_mm, size=(n_nodes, 2))
    tri = Delaunay(pts)
    e = np.concatenate([tri.simplices[:, [0, 1]], tri.simplices[:, [1, 2]],
                        tri.simplices[:, [0, 2]]])
    e = np.unique(np.sort(e, axis=1), axis=0)
    d = np.hypot(*(pts[e[:, 0]] - pts[e[:, 1]]).T)
    m = coo_matrix((d, (e[:, 0], e[:, 1])), shape=(n_nodes, n_nodes))
    mst = minimum_spanning_tree(m).tocoo()
    mst_set = set(zip(np.minimum(mst.row, mst.col).tolist(), np.maximum(mst.row, mst.col).tolist()))
    in_mst = np.array([(a, b) in mst_set for a, b in e.tolist()])
    order = np.argsort(d[~in_mst], kind="stable")
    extra = np.nonzero(~in_mst)[0][order][: max(0, n_edges - in_mst.sum())]
    keep = np.concatenate([np.nonzero(in_mst)[0], extra])
    e, d = e[keep], d[keep]
    x = (np.round(pts[:, 0]) + x0).astype(np.int64)
    y = (np.round(pts[:, 1]) + y0).astype(np.int64)
    return x, y, e, d


def _portland_links(rng, e, d):
    # lognormal lengths (median 300 m, sigma 0.8) clamped to [75, 3000] m,
    # assigned by rank of Euclidean length (reading R20)
    draws = np.exp(np.log(300.0) + 0.8 * rng.standard_normal(e.shape[0]))
    draws = np.clip(draws, 75.0, 3000.0)
    length = np.empty(e.shape[0])
    length[np.argsort(d, kind="stable")] = np.sort(draws)
    length_mm = np.round(length * 1000).astype(np.int64)
    lanes = rng.choice([1, 2, 3], size=e.shape[0], p=[0.6, 0.3, 0.1]).astype(np.int32)
    return length_mm, lanes


def _directed(e, length_mm, lanes, cls):
    frm = np.empty(2 * e.shape[0], np.int32)
    to = np.empty_like(frm)
    frm[0::2], to[0::2] = e[:, 0], e[:, 1]
    frm[1::2], to[1::2] = e[:, 1], e[:, 0]
    rep = lambda a: np.repeat(a, 2)  # noqa: E731
    return frm, to, rep(length_mm), rep(lanes).astype(np.int32), rep(cls).astype(np.int32)


def _zone_routes(rng, frm, to, length_mm, n_nodes, origins, zone_of_vehicle, zones):
    """Routes from origin links to destination (zone) links along free-flow
    shortest paths (reverse Dijkstra tree per zone; scipy)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra

    succ_lists = successors(frm, to, n_nodes)
    rows = np.fromiter((k for k, s in enumerate(succ_lists) for _ in s), dtype=np.int64)
    cols = np.fromiter((k2 for s in succ_lists for k2 in s), dtype=np.int64)
    nl = frm.size
    w = length_mm[cols].astype(np.float64)
    g_rev = csr_matrix((w, (cols, rows)), shape=(nl, nl))
    n_veh = origins.size
    routes = [None] * n_veh
    for zi, z in enumerate(zones.tolist()):
        sel = np.nonzero(zone_of_vehicle == zi)[0]
        if sel.size == 0:
            continue
        _, pred = dijkstra(g_rev, directed=True, indices=z, return_predecessors=True)
        for i in sel.tolist():
            o = int(origins[i])
            while o == z or (pred[o] < 0):
                o = int(rng.integers(0, nl))
            path = [o]
            while path[-1] != z:
                path.append(int(pred[path[-1]]))
            routes[i] = path
    return routes


def portland(n_nodes=8500, n_edges=10_000, n_veh=150_000, side_km=55.0, n_zones=512,
             seed=1, steps=3600, name="config3_portland"):
    """BASELINE.json configs[2]: synthetic Portland-shaped planar network
    (~8,500 nodes, ~20,000 directed links), lognormal link lengths (median
    300 m, max 3 km), lanes 1-3 (60/30/10 %), priority class = lanes;
    150,000 vehicles released over one hour by a triangular time-of-day
    profile (reading R20).  Destinations are drawn uniformly from `n_zones`
    zone links (activity locations) so that routing is one Dijkstra tree
    per zone."""
    rng = np.random.default_rng(seed)
    x, y, e, d = _planar_network(rng, n_nodes, n_edges, side_km * 1e6)
    length_mm, lanes = _portland_links(rng, e, d)
    frm, to, lm, ln, cl = _directed(e, length_mm, lanes, lanes)
    nl = frm.size
    dep = np.floor(rng.triangular(0, 1800, 3600, size=n_veh)).astype(np.int32)
    origins = rng.integers(0, nl, size=n_veh)
    zones = rng.choice(nl, size=min(n_zones, nl), replace=False)
    zone_of = rng.integers(0, zones.size, size=n_veh)
    routes = _zone_routes(rng, frm, to, lm, x.size, origins, zone_of, zones)
    off, flat = _routes_csr(routes)
    first = flat[off[:-1]]
    entry = (rng.random(n_veh) * (lm[first] // CELL_MM)).astype(np.int32)
    pv, pl, pc, pvv = _empty_place()
    return Scenario(name=name, node_x=x, node_y=y, link_from=frm, link_to=to,
                    link_len_mm=lm, link_lanes=ln, link_vmax=np.full(nl, 5, np.int32),
                    link_class=cl, periodic_link=-1, route_off=off, route=flat,
                    depart=dep, entry=entry, place_vid=pv, place_lane=pl, place_cell=pc,
                    place_v=pvv, steps=steps, seed=seed,
                    recipe=f"Portland-shaped: {x.size} nodes, {nl} links, {n_veh} vehicles, "
                           f"triangular(0,1800,3600) departures, {zones.size} zones")


def portland_tiled(tiles_x=4, tiles_y=2, n_nodes=8500, n_edges=10_000, n_veh=150_000,
                   side_km=55.0, stitches=20, n_zones=128, seed=1, steps=3600,
                   name="config5_portland_x8"):
    """BASELINE.json configs[4]: the Portland-shaped network tiled 4 x 2 with
    `stitches` two-way links across each shared tile border; tile-local trips;
    tile i's departure peak at 1800 + 300 (i - 3.5) s so load moves across
    the map during the hour."""
    rng = np.random.default_rng(seed)
    side = side_km * 1e6
    xs, ys, es, ds, tile_of_node = [], [], [], [], []
    base = 0
    for ty in range(tiles_y):
        for tx in range(tiles_x):
            x, y, e, d = _planar_network(rng, n_nodes, n_edges, side, tx * side, ty * side)
            xs.append(x)
            ys.append(y)
            es.append(e + base)
            ds.append(d)
            tile_of_node.append(np.full(x.size, ty * tiles_x + tx))
            base += x.size
    x, y = np.concatenate(xs), np.concatenate(ys)
    tile_of_node = np.concatenate(tile_of_node)
    e, d = np.concatenate(es), np.concatenate(ds)
    length_mm, lanes = _portland_links(rng, e, d)
    # stitches: per shared border, `stitches` bands; join the nodes closest
    # to the border on both sides
    se = []
    for ty in range(tiles_y):
        for tx in range(tiles_x):
            a = ty * tiles_x + tx
            for (bx, by) in ((tx + 1, ty), (tx, ty + 1)):
                if bx >= tiles_x or by >= tiles_y:
                    continue
                b = by * tiles_x + bx
                vertical = bx != tx
                border = (bx if vertical else by) * side
                ia, ib = np.nonzero(tile_of_node == a)[0], np.nonzero(tile_of_node == b)[0]
                along_a = (y if vertical else x)[ia]
                along_b = (y if vertical else x)[ib]
                lo = (ty if vertical else tx) * side
                for s in range(stitches):
                    b0, b1 = lo + s * side / stitches, lo + (s + 1) * side / stitches
                    ca = ia[(along_a >= b0) & (along_a < b1)]
                    cb = ib[(along_b >= b0) & (along_b < b1)]
                    if ca.size == 0 or cb.size == 0:
                        continue
                    pa = ca[np.argmin(np.abs((x if vertical else y)[ca] - border))]
                    pb = cb[np.argmin(np.abs((x if vertical else y)[cb] - border))]
                    se.append((pa, pb))
    se = np.array(se, dtype=np.int64)
    sd = np.hypot(x[se[:, 0]] - x[se[:, 1]], y[se[:, 0]] - y[se[:, 1]])
    s_len = np.round(np.maximum(sd, 75_000.0)).astype(np.int64)
    s_lanes = np.full(se.shape[0], 2, np.int32)
    e = np.concatenate([e, se])
    length_mm = np.concatenate([length_mm, s_len])
    lanes = np.concatenate([lanes, s_lanes])
    frm, to, lm, ln, cl = _directed(e, length_mm, lanes, lanes)
    nl = frm.size
    n_tiles = tiles_x * tiles_y
    routes, deps = [], []
    link_tile = tile_of_node[frm]
    intra = tile_of_node[frm] == tile_of_node[to]
    for i in range(n_tiles):
        peak = 1800 + 300 * (i - (n_tiles - 1) / 2)
        dep = np.floor(rng.triangular(peak - 1800, peak, peak + 1800, size=n_veh))
        deps.append(np.clip(dep, 0, 3599).astype(np.int32))
        tl = np.nonzero((link_tile == i) & intra)[0]
        origins = rng.choice(tl, size=n_veh)
        zones = rng.choice(tl, size=min(n_zones, tl.size), replace=False)
        zone_of = rng.integers(0, zones.size, size=n_veh)
        routes += _zone_routes(rng, frm, to, lm, x.size, origins, zone_of, zones)
    off, flat = _routes_csr(routes)
    first = flat[off[:-1]]
    nv = off.size - 1
    entry = (rng.random(nv) * (lm[first] // CELL_MM)).astype(np.int32)
    pv, pl, pc, pvv = _empty_place()
    return Scenario(name=name, node_x=x, node_y=y, link_from=frm, link_to=to,
                    link_len_mm=lm, link_lanes=ln, link_vmax=np.full(nl, 5, np.int32),
                    link_class=cl, periodic_link=-1, route_off=off, route=flat,
                    depart=np.concatenate(deps), entry=entry, place_vid=pv, place_lane=pl,
                    place_cell=pc, place_v=pvv, steps=steps, seed=seed,
                    recipe=f"Portland-shaped x{n_tiles} tiles: {x.size} nodes, {nl} links, "
                           f"{nv} vehicles, shifted departure peaks")


# --------------------------------------------------------------- named configs
def config(name: str, **kw) -> Scenario:
    """The BASELINE.json configs by short name (1, 2, 3, 4a, 4b, 5)."""
    if name == "1":
        return grid_trips(**kw)
    if name == "2":
        return ring(**kw)
    if name == "3":
        return portland(**kw)
    if name == "4a":
        return big_grid(**kw)
    if name == "4b":
        kw.setdefault("n_veh", 1_000_000)
        kw.setdefault("name", "config4b_grid256_1M")
        return big_grid(**kw)
    if name == "5":
        return portland_tiled(**kw)
    raise KeyError(name)


def stop_sign_merges(headways=(0, 12, 8, 6, 4, 3, 2, -1), copies=64, steps=2400, n_minor=1500,
                     seed=1, name="fig4c_stop_sign_merge"):
    """Fig. 4c ("merge flows through a stop sign"; SPEC.md
    merge_capacity): independent T-junctions, `copies` per priority-flow
    level.  Each: a 2-lane major road A -> J -> B (class 1, 40 cells each)
    and a 1-lane stop-controlled minor approach M -> J (class 0, 40 cells)
    whose right turn merges onto J -> B.  The minor approach holds a
    saturated queue (n_minor trips departing at t = 0 at its entry cell,
    retrying injection every step).  Major flow level h > 0: one major trip
    every h s (offset per copy) at the start of A -> J; h = 0: no major
    traffic; h = -1: the major road is bumper-to-bumper -- every cell of
    A -> J, J -> B and B -> C occupied at t = 0 by vehicles routed through
    node C, whose signal is never green (reading R23), so nothing on it ever
    moves.  Returns the scenario; the minor trips of copy c of level i are
    vids [minor_base[i][c], + n_minor)."""
    rng = np.random.default_rng(seed)
    cell = 7500
    nx, ny, frm, to, ln, la, cls = [], [], [], [], [], [], []
    routes, dep, ent = [], [], []
    pv, pl, pc, pvv = [], [], [], []
    sig_nodes = []
    minor_base = []
    meta = []
    for i, h in enumerate(headways):
        mb = []
        for c in range(copies):
            x0, y0 = c * 200 * cell, i * 200 * cell
            b = len(nx)
            # A, J, B, M, C, D
            for (x, y) in ((0, 0), (40, 0), (80, 0), (40, -40), (120, 0), (130, 0)):
                nx.append(x0 + x * cell)
                ny.append(y0 + y * cell)
            A, J, B, Mn, C, D = range(b, b + 6)
            k = len(frm)
            for (u, v, n, L, cl) in ((A, J, 40, 2, 1), (J, B, 40, 2, 1), (Mn, J, 40, 1, 0),
                                     (B, C, 40, 2, 1), (C, D, 10, 2, 1)):
                frm.append(u)
                to.append(v)
                ln.append(n * cell)
                la.append(L)
                cls.append(cl)
            kAJ, kJB, kMJ, kBC, kCD = range(k, k + 5)
            mb.append(len(routes))
            for _ in range(n_minor):  # the saturated stop-controlled queue
                routes.append([kMJ, kJB])
                dep.append(0)
                ent.append(0)
            if h > 0:
                off = int(rng.integers(0, h))
                for t in range(off, steps, h):
                    routes.append([kAJ, kJB])
                    dep.append(t)
                    ent.append(0)
            elif h < 0:  # jammed major road behind a never-green signal at C
                sig_nodes.append(C)
                for kk in (kAJ, kJB, kBC):
                    for lane in range(2):
                        for x in range(40):
                            pv.append(len(routes))
                            routes.append([kk, kCD] if kk == kBC else
                                          ([kJB, kBC, kCD] if kk == kJB else [kAJ, kJB, kBC, kCD]))
                            dep.append(0)
                            ent.append(x)
                            pl.append(lane)
                            pc.append(x)
                            pvv.append(0)
        minor_base.append(mb)
        meta.append(h)
    off = np.zeros(len(routes) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in routes])
    s = Scenario(name=name, node_x=_i64(nx), node_y=_i64(ny), link_from=_i32(frm), link_to=_i32(to),
                 link_len_mm=_i64(ln), link_lanes=_i32(la), link_vmax=_i32([5] * len(frm)),
                 link_class=_i32(cls), periodic_link=-1, route_off=off,
                 route=_i32([k for r in routes for k in r]), depart=_i32(dep), entry=_i32(ent),
                 place_vid=_i32(pv), place_lane=_i32(pl), place_cell=_i32(pc), place_v=_i32(pvv),
                 steps=steps, recipe=f"{copies} T-junctions per major headway {list(headways)}")
    if sig_nodes:
        n = len(sig_nodes)
        s.sig_node = _i32(sig_nodes)
        s.sig_g0 = _i32([0] * n)   # phase 0 (the maximal class: the only approach) never green
        s.sig_g1 = _i32([1] * n)
        s.sig_off = _i32([0] * n)
    s.minor_base = minor_base
    s.n_minor = n_minor
    s.headways = list(meta)
    return s
