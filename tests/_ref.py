"""Independent brute-force helpers for the oracle pins (tests only).

These are written from the paper / the textbook definitions in a different
representation (particle lists, numpy) from the oracle's lane-cell grid, so
that an indexing or sign mistake in the oracle shows up as a mismatch.
"""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox_np(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on numpy uint32 arrays (Salmon et al. 2011)."""
    c = [np.asarray(a, dtype=np.uint64) for a in (c0, c1, c2, c3)]
    k = [np.asarray(k0, dtype=np.uint64), np.asarray(k1, dtype=np.uint64)]
    for r in range(10):
        if r:
            k = [(k[0] + np.uint64(W0)) & MASK, (k[1] + np.uint64(W1)) & MASK]
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> np.uint64(32)) ^ c[1] ^ k[0]) & MASK, p1 & MASK,
             ((p0 >> np.uint64(32)) ^ c[3] ^ k[1]) & MASK, p0 & MASK]
    return [a.astype(np.uint32) for a in c]


def brake_np(t, vids, seed, p):
    u = philox_np(np.full(len(vids), t), np.asarray(vids), 0, 0,
                  seed & 0xFFFFFFFF, seed >> 32)[0]
    return u.astype(np.uint64) < np.uint64(int(p * 4294967296.0))


def nasch_ring_particles(L, x, v, vmax, steps, brake_fn):
    """Single-lane periodic NaSch on a particle list (positions sorted).
    brake_fn(t, idx_array) -> bool array.  Returns list of (x, v) per step."""
    x = np.array(x, dtype=np.int64)
    v = np.array(v, dtype=np.int64)
    order = np.argsort(x)
    x, v = x[order], v[order]
    ids = order.copy()
    out = []
    N = len(x)
    for t in range(steps):
        if N == 1:
            gap = np.array([L - 1])
        else:
            gap = (np.roll(x, -1) - x - 1) % L
        gap = np.minimum(gap, 5)
        v1 = np.minimum(v + 1, vmax)
        v2 = np.minimum(v1, gap)
        b = brake_fn(t, ids) & (v2 > 0)
        v3 = v2 - b.astype(np.int64)
        x = (x + v3) % L
        v = v3
        out.append((ids.copy(), x.copy(), v.copy()))
    return out


def nasch_v1_exact_flow(rho, p):
    """Exact steady-state flow of parallel-update NaSch with vmax = 1
    (Schadschneider & Schreckenberg 1993; Nagel & Schreckenberg 1992)."""
    q = 1 - p
    return 0.5 * (1 - np.sqrt(1 - 4 * q * rho * (1 - rho)))


def make_ring(L, lane, cell, v, lanes=1, vmax=5, p_slow=0.0, seed=1):
    """Scenario for a periodic ring with explicit placement (vid = index)."""
    import scenarios

    lane = np.asarray(lane, dtype=np.int32)
    cell = np.asarray(cell, dtype=np.int32)
    v = np.asarray(v, dtype=np.int32)
    n = cell.size
    s = scenarios.ring(n_cells=L, lanes=lanes, n_veh=0, seed=seed, vmax=vmax)
    s.place_vid = np.arange(n, dtype=np.int32)
    s.place_lane, s.place_cell, s.place_v = lane, cell, v
    s.route_off = np.arange(n + 1, dtype=np.int64)
    s.route = np.zeros(n, np.int32)
    s.depart = np.zeros(n, np.int32)
    s.entry = cell.copy()
    s.p_slow = p_slow
    s.seed = seed
    return s


def make_network(nodes_xy_m, links, vehicles, p_slow=0.0, seed=1):
    """Small hand-built network.  links: list of (from, to, length_m, lanes,
    class); vehicles: list of dicts(route=[...], depart=, entry=, place=(lane,
    cell, v) or None)."""
    import scenarios

    xy = np.asarray(nodes_xy_m, dtype=np.float64)
    frm = [l[0] for l in links]
    to = [l[1] for l in links]
    pv, pl, pc, pvv = [], [], [], []
    routes = []
    for i, veh in enumerate(vehicles):
        routes.append(list(veh["route"]))
        if veh.get("place") is not None:
            ln, c, vv = veh["place"]
            pv.append(i)
            pl.append(ln)
            pc.append(c)
            pvv.append(vv)
    off = np.zeros(len(routes) + 1, np.int64)
    off[1:] = np.cumsum([len(r) for r in routes])
    i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731
    return scenarios.Scenario(
        name="handmade", node_x=np.round(xy[:, 0] * 1000).astype(np.int64),
        node_y=np.round(xy[:, 1] * 1000).astype(np.int64),
        link_from=i32(frm), link_to=i32(to),
        link_len_mm=np.asarray([round(l[2] * 1000) for l in links], dtype=np.int64),
        link_lanes=i32([l[3] for l in links]), link_vmax=i32([5] * len(links)),
        link_class=i32([l[4] for l in links]), periodic_link=-1,
        route_off=off, route=i32([k for r in routes for k in r]),
        depart=i32([veh.get("depart", 0) for veh in vehicles]),
        entry=i32([veh.get("entry", 0) for veh in vehicles]),
        place_vid=i32(pv), place_lane=i32(pl), place_cell=i32(pc), place_v=i32(pvv),
        p_slow=p_slow, seed=seed)


def ring_multilane_ref(L, lanes, lane, cell, v, vmax, steps, brake_fn, t0=0):
    """Independent multi-lane periodic ring reference (grid of vids,
    numpy per lane): lane change by reading R4/R5 (direction by step parity,
    'other lane faster' + gap check), then per-lane NaSch.  Returns per step
    arrays (lane, cell, v) indexed by vid."""
    n = len(cell)
    lane = np.array(lane, dtype=np.int64)
    cell = np.array(cell, dtype=np.int64)
    v = np.array(v, dtype=np.int64)
    out = []

    def grid_of(lane, cell):
        g = -np.ones((lanes, L), dtype=np.int64)
        g[lane, cell] = np.arange(n)
        return g

    def ahead(g, l, x):
        c = 0
        for j in range(1, 6):
            if g[l, (x + j) % L] >= 0:
                break
            c += 1
        return c

    def behind(g, l, x):
        c = 0
        for j in range(1, 6):
            if g[l, (x - j) % L] >= 0:
                break
            c += 1
        return c

    for s in range(steps):
        t = t0 + s
        d = 1 if t % 2 == 0 else -1
        g = grid_of(lane, cell)
        new_lane = lane.copy()
        for i in range(n):
            l2 = lane[i] + d
            if l2 < 0 or l2 >= lanes or g[l2, cell[i]] >= 0:
                continue
            gc = ahead(g, lane[i], cell[i])
            if gc < v[i] + 1 and ahead(g, l2, cell[i]) > gc and behind(g, l2, cell[i]) >= vmax:
                new_lane[i] = l2
        lane = new_lane
        g = grid_of(lane, cell)
        v_new = v.copy()
        for l in range(lanes):
            ids = np.nonzero(lane == l)[0]
            if ids.size == 0:
                continue
            ids = ids[np.argsort(cell[ids])]
            x = cell[ids]
            gap = (np.roll(x, -1) - x - 1) % L if ids.size > 1 else np.array([L - 1])
            gap = np.minimum(gap, 5)
            v2 = np.minimum(np.minimum(v[ids] + 1, vmax), gap)
            b = brake_fn(t, ids) & (v2 > 0)
            v_new[ids] = v2 - b
        v = v_new
        cell = (cell + v) % L
        out.append((lane.copy(), cell.copy(), v.copy()))
    return out
