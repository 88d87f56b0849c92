"""Input validation of the C-ABI loaders (include/tsim.h ts_load_vehicles,
ts_place_vehicles_at, ts_init): the checks run in parallel on the host cores
and must report the first failing record in input order, leave the handle
usable after a rejected batch, and catch two placements on one cell."""
import dataclasses

import numpy as np
import pytest

import scenarios

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")


def _scn():
    return scenarios.config("1")


def _sim(scn, **kw):
    s = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, **kw)
    return s


def _load_routes(s, scn, route_off, route, entry):
    i32 = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
    nx = np.ascontiguousarray(scn.node_x, np.int64)
    ny = np.ascontiguousarray(scn.node_y, np.int64)
    arr = [i32(scn.link_from), i32(scn.link_to), np.ascontiguousarray(scn.link_len_mm, np.int64),
           i32(scn.link_lanes), i32(scn.link_vmax), i32(scn.link_class)]
    s._check(s.lib.ts_load_network(s.h, scn.n_nodes, nx.ctypes.data, ny.ctypes.data, scn.n_links,
                                   *(a.ctypes.data for a in arr), int(scn.periodic_link)))
    ro = np.ascontiguousarray(route_off, np.int64)
    r, d, e = i32(route), i32(scn.depart[: ro.size - 1]), i32(entry)
    s._check(s.lib.ts_load_vehicles(s.h, ro.size - 1, ro.ctypes.data, r.ctypes.data,
                                    d.ctypes.data, e.ctypes.data))
    s.n_veh = ro.size - 1


@pytest.mark.parametrize("kind,msg", [
    ("empty", "vehicle 7: empty route"),
    ("badlink", "vehicle 7: bad link"),
    ("gap", "vehicle 7: route links not consecutive"),
    ("entry", "vehicle 7: entry cell outside link"),
])
def test_load_vehicles_first_error(kind, msg):
    scn = _scn()
    ro = np.array(scn.route_off, np.int64)
    route = np.array(scn.route, np.int32)
    entry = np.array(scn.entry, np.int32)
    bad = [7, 500, 900]  # several failing vehicles: the first is reported
    for f in bad:
        a = int(ro[f])
        if kind == "badlink":
            route[a] = scn.n_links + 3
        elif kind == "gap":
            # a link that does not start at the end of the first one
            k0 = int(route[a])
            if int(ro[f + 1]) - a < 2:
                route = np.insert(route, a + 1, k0)
                ro[f + 1:] += 1
            route[a + 1] = next(k for k in range(scn.n_links)
                                if scn.link_from[k] != scn.link_to[k0])
        elif kind == "entry":
            entry[f] = 10 ** 6
    if kind == "empty":
        for f in bad:  # drop the route of f
            a, b = int(ro[f]), int(ro[f + 1])
            route = np.delete(route, np.arange(a, b))
            ro[f + 1:] -= b - a
    s = _sim(scn)
    with pytest.raises(tsim.TsError, match=msg):
        _load_routes(s, scn, ro, route, entry)


def test_place_first_error_and_retry():
    scn = _scn()
    s = _sim(scn)
    s.load(dataclasses.replace(scn, place_vid=np.zeros(0, np.int32)), place=False)
    n = 40
    vid = np.arange(n, dtype=np.int32)
    cur = np.zeros(n, np.int32)
    lane = np.zeros(n, np.int32)
    v = np.zeros(n, np.int32)
    # each vehicle on a distinct cell of its first link
    first = np.array(scn.route)[np.array(scn.route_off)[:n]]
    cell = np.zeros(n, np.int32)
    used = {}
    for i, k in enumerate(first):
        cell[i] = used.get(int(k), 0)
        used[int(k)] = cell[i] + 1
    cases = [
        ("dup", lambda a: a["vid"].__setitem__(31, 5), "placement 31: vehicle placed twice"),
        ("vid", lambda a: a["vid"].__setitem__(12, -4), "placement 12: bad vid"),
        ("cursor", lambda a: a["cur"].__setitem__(9, 10 ** 5), "placement 9: cursor outside the route"),
        ("lane", lambda a: a["lane"].__setitem__(20, 9), "placement 20: cell outside link"),
        ("v", lambda a: a["v"].__setitem__(33, 6), "placement 33: velocity"),
    ]
    for _, mut, msg in cases:
        a = dict(vid=vid.copy(), cur=cur.copy(), lane=lane.copy(), v=v.copy())
        mut(a)
        with pytest.raises(tsim.TsError, match=msg):
            s.place_at(a["vid"], a["cur"], a["lane"], cell, a["v"])
    # a rejected batch leaves nothing placed: the clean batch goes through
    s.place_at(vid, cur, lane, cell, v)
    with pytest.raises(tsim.TsError, match="placement 0: vehicle placed twice"):
        s.place_at(vid[3:4], cur[3:4], lane[3:4], cell[3:4], v[3:4])
    s.init(0)
    st = s.vehicles()
    assert (st["status"][:n] == tsim.ACTIVE).all()
    assert (st["cell"][:n] == cell).all() and (st["link"][:n] == first).all()


def test_init_cell_taken():
    scn = _scn()
    s = _sim(scn)
    s.load(dataclasses.replace(scn, place_vid=np.zeros(0, np.int32)), place=False)
    first = np.array(scn.route)[np.array(scn.route_off)[:-1]]
    k = int(first[0])
    same = np.flatnonzero(first == k)[:3].astype(np.int32)
    assert same.size == 3
    z = np.zeros(3, np.int32)
    s.place_at(same, z, z, np.array([4, 4, 6], np.int32), z)
    with pytest.raises(tsim.TsError, match="placement 1: cell taken"):
        s.init(0)
