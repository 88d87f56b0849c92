"""ctypes binding of libtsim (include/tsim.h) -- argument marshalling only.

Every step of the CA path runs in the CUDA kernels of csrc/.  There is no
CPU fallback: without the built library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TSIM_LIB selects another in-tree build of the same sources (tuning
# variants built by tools/variants.py); the default is the in-tree library
_SO = os.environ.get("TSIM_LIB") or os.path.join(_HERE, "libtsim.so")

FLAG_FUSED, FLAG_HASH, FLAG_LINK_WORK, FLAG_GRAPH, FLAG_GENERAL = 1, 2, 4, 8, 16
PENDING, ACTIVE, ARRIVED, ABSENT = 0, 1, 2, 3


class TsError(RuntimeError):
    pass


class Config(ctypes.Structure):
    _fields_ = [("p_slow", ctypes.c_double), ("seed", ctypes.c_uint64),
                ("gap_accept_G", ctypes.c_int32), ("desperation_D", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("device", ctypes.c_int32),
                ("tile_cells", ctypes.c_int32), ("group_cells", ctypes.c_int32)]


_lib = None


def load_library():
    """Load libtsim.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        raise TsError(f"{_SO} is missing: run __graft_entry__.build() (no CPU fallback)")
    lib = ctypes.CDLL(_SO)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sig = {
        "ts_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(P)]),
        "ts_destroy": (None, [P]),
        "ts_last_error": (ctypes.c_char_p, [P]),
        "ts_load_network": (ctypes.c_int, [P, I32, P, P, I32, P, P, P, P, P, P, I32]),
        "ts_load_vehicles": (ctypes.c_int, [P, I32, P, P, P, P]),
        "ts_place_vehicles": (ctypes.c_int, [P, I32, P, P, P, P]),
        "ts_init": (ctypes.c_int, [P, I32]),
        "ts_step": (ctypes.c_int, [P, I32]),
        "ts_step_async": (ctypes.c_int, [P, I32]),
        "ts_sync": (ctypes.c_int, [P]),
        "ts_time": (I32, [P]),
        "ts_read_vehicles": (ctypes.c_int, [P, P, P, P, P, P, P, P]),
        "ts_read_cells": (ctypes.c_int, [P, I32, P]),
        "ts_link_cells": (I32, [P, I32]),
        "ts_read_raw": (ctypes.c_int, [P, I32, P, P, P]),
        "ts_state_hash": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_uint64)]),
        "ts_debug_checks": (ctypes.c_int, [P, I32]),
        "ts_read_history": (ctypes.c_int, [P, I32, I32, P, P, P, P, P, P]),
        "ts_get_totals": (ctypes.c_int, [P, P]),
        "ts_read_flow": (ctypes.c_int, [P, I32, I32, P]),
        "ts_get_link_work": (ctypes.c_int, [P, P]),
        "ts_get_load": (ctypes.c_int, [P, P, P]),
        "ts_load_times": (ctypes.c_int, [ctypes.c_double, I32, P, I32, P, P, P]),
        "ts_rebalance": (ctypes.c_int, [I32, P, P, I32, P, P, P, P, P, P, I32, I32,
                                        ctypes.c_double, ctypes.c_uint64, P, P]),
        "ts_orb_partition": (ctypes.c_int, [I32, P, P, P, I32, P]),
        "ts_multilevel_partition": (ctypes.c_int, [I32, P, P, I32, P, P, P, P, I32,
                                                   ctypes.c_double, ctypes.c_uint64, P]),
        "ts_place_vehicles_at": (ctypes.c_int, [P, I32, P, P, P, P, P]),
        "ts_set_arrived": (ctypes.c_int, [P, I32, P, P]),
        "ts_set_domain": (ctypes.c_int, [P, I32, P, I32]),
        "ts_set_signals": (ctypes.c_int, [P, I32, P, P, P, P]),
        "ts_domain_plan": (ctypes.c_int, [I32, I32, P, P, P, P, I32, P, I32, I32, P, P, P]),
        "ts_strip_bytes": (I32, []),
        "ts_nccl_unique_id": (ctypes.c_int, [P]),
        "ts_parse_network_text": (ctypes.c_int, [P, ctypes.c_size_t, P, P, P, P, P, P, P, P, P, P,
                                                 P, P, P, P, P, P]),
        "ts_load_network_text": (ctypes.c_int, [P, P, ctypes.c_size_t]),
        "ts_parse_plans_text": (ctypes.c_int, [P, ctypes.c_size_t, I32, P, P, P, P, P, P, P, P, P]),
        "ts_load_plans_text": (ctypes.c_int, [P, P, ctypes.c_size_t]),
        "ts_partition": (ctypes.c_int, [P, I32, P, I32, P]),
        "ts_nccl_init": (ctypes.c_int, [P, P, I32, I32]),
        "ts_exchange": (ctypes.c_int, [P]),
        "ts_busy_time": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double)]),
        "ts_last_exchange_timing": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double),
                                                   ctypes.POINTER(ctypes.c_int64)]),
        "ts_resume": (ctypes.c_int, [P, I32]),
        "ts_step_phase": (ctypes.c_int, [P, I32, I32]),
        "ts_exchange_plan": (ctypes.c_int, [P, I32, P, P, P, P]),
        "ts_exchange_buffers": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(P)]),
        "ts_stream": (P, [P]),
        "ts_exchange_local": (ctypes.c_int, [ctypes.POINTER(P), I32]),
        "ts_local_step": (ctypes.c_int, [ctypes.POINTER(P), I32, I32]),
        "ts_last_timing": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_int64)]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(lib, name):  # an older in-tree variant (tools/variants.py)
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    """Names declared in include/tsim.h (for the ABI test)."""
    import re
    hdr = open(os.path.join(os.path.dirname(_HERE), "include", "tsim.h")).read()
    return sorted(set(re.findall(r"\b(ts_[a-z_]+)\s*\(", hdr)))


def _a(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def orb_partition(node_x, node_y, k, weight=None):
    """Orthogonal recursive bisection -> domain per node."""
    lib = load_library()
    x, y = _a(node_x, np.int64), _a(node_y, np.int64)
    w = None if weight is None else _a(weight, np.float64)
    out = np.zeros(x.size, np.int32)
    rc = lib.ts_orb_partition(x.size, x.ctypes.data, y.ctypes.data, _p(w), int(k), out.ctypes.data)
    if rc:
        raise TsError(f"ts_orb_partition failed ({rc})")
    return out


def multilevel_partition(scn, k, weight=None, imbalance=0.05, seed=1):
    """multilevel k-way partition (METIS-style) -> domain
    per node; edges weighted by lanes (strips per exchange)"""
    lib = load_library()
    x, y = _a(scn.node_x, np.int64), _a(scn.node_y, np.int64)
    fr, to, la = _a(scn.link_from, np.int32), _a(scn.link_to, np.int32), _a(scn.link_lanes, np.int32)
    w = None if weight is None else _a(weight, np.float64)
    out = np.zeros(x.size, np.int32)
    rc = lib.ts_multilevel_partition(x.size, x.ctypes.data, y.ctypes.data, fr.size, fr.ctypes.data,
                                     to.ctypes.data, la.ctypes.data, _p(w), int(k),
                                     float(imbalance), int(seed), out.ctypes.data)
    if rc:
        raise TsError(f"ts_multilevel_partition failed ({rc})")
    return out


def load_times(domain_ms, link_work, node_work=None, link_time=None, node_time=None):
    """one domain's measured time apportioned to its links and nodes by
    their work (ts_load_times); adds into (and returns)
    link_time / node_time"""
    lib = load_library()
    lw = _a(link_work, np.int64)
    nw = None if node_work is None else _a(node_work, np.int64)
    lt = np.zeros(lw.size, np.float64) if link_time is None else link_time
    nt = (np.zeros(0 if nw is None else nw.size, np.float64) if node_time is None else node_time)
    assert lt.dtype == np.float64 and lt.flags.c_contiguous and nt.dtype == np.float64
    rc = lib.ts_load_times(float(domain_ms), lw.size, _p(lw), 0 if nw is None else nw.size, _p(nw),
                           _p(lt), _p(nt) if nw is not None else None)
    if rc:
        raise TsError(f"ts_load_times failed ({rc})")
    return lt, nt


def rebalance(scn, k, link_time, node_time=None, method="orb", imbalance=0.05, seed=1):
    """the next partition from measured link / node times (ts_rebalance,
    PAPER.md:726-735) -> (domain_of_node, node weights)"""
    lib = load_library()
    i32 = lambda a: _a(a, np.int32)  # noqa: E731
    x, y = _a(scn.node_x, np.int64), _a(scn.node_y, np.int64)
    fr, to, la = i32(scn.link_from), i32(scn.link_to), i32(scn.link_lanes)
    ln = _a(scn.link_len_mm, np.int64)
    lt = _a(link_time, np.float64)
    nt = None if node_time is None or len(node_time) == 0 else _a(node_time, np.float64)
    w = np.zeros(x.size, np.float64)
    dom = np.zeros(x.size, np.int32)
    rc = lib.ts_rebalance(x.size, x.ctypes.data, y.ctypes.data, fr.size, fr.ctypes.data,
                          to.ctypes.data, la.ctypes.data, ln.ctypes.data, lt.ctypes.data, _p(nt),
                          int(k), {"orb": 0, "multilevel": 1}[method], float(imbalance), int(seed),
                          w.ctypes.data, dom.ctypes.data)
    if rc:
        raise TsError(f"ts_rebalance failed ({rc})")
    return dom, w


def strip_bytes():
    """bytes of one exchanged strip (5 cells of one lane next to a cut)"""
    return int(load_library().ts_strip_bytes())


def domain_plan(scn, k, domain_of_node, me):
    """Exchange partners of domain `me` and strips per message (pure host,
    no device; one buffer per neighbour)."""
    lib = load_library()
    i32 = lambda a: _a(a, np.int32)  # noqa: E731
    fr, to, ln = i32(scn.link_from), i32(scn.link_to), _a(scn.link_len_mm, np.int64)
    la, dom = i32(scn.link_lanes), i32(domain_of_node)
    cap = int(k)
    nb = np.zeros(cap, np.int32)
    ns = np.zeros(cap, np.int64)
    n = ctypes.c_int32()
    rc = lib.ts_domain_plan(scn.n_nodes, scn.n_links, fr.ctypes.data, to.ctypes.data, ln.ctypes.data,
                            la.ctypes.data, int(k), dom.ctypes.data, int(me), cap, nb.ctypes.data,
                            ns.ctypes.data, ctypes.byref(n))
    if rc:
        raise TsError(f"ts_domain_plan failed ({rc})")
    return nb[:n.value].tolist(), ns[:n.value].tolist()


def parse_network_text(text):
    """SPEC network file -> arrays (pure host; ts_parse_network_text)"""
    lib = load_library()
    b = text.encode() if isinstance(text, str) else bytes(text)
    nn, nl, ns = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    err = ctypes.create_string_buffer(256)
    z = [None] * 12
    if lib.ts_parse_network_text(b, len(b), ctypes.byref(nn), ctypes.byref(nl), ctypes.byref(ns),
                                 *z, err):
        raise TsError(err.value.decode())
    out = dict(node_x_mm=np.zeros(nn.value, np.int64), node_y_mm=np.zeros(nn.value, np.int64),
               link_from=np.zeros(nl.value, np.int32), link_to=np.zeros(nl.value, np.int32),
               link_len_mm=np.zeros(nl.value, np.int64), link_lanes=np.zeros(nl.value, np.int32),
               link_vmax=np.zeros(nl.value, np.int32), link_class=np.zeros(nl.value, np.int32),
               link_id=np.zeros(nl.value, np.int32), sig_node=np.zeros(ns.value, np.int32),
               sig_green=np.zeros(ns.value, np.int32), sig_red=np.zeros(ns.value, np.int32))
    lib.ts_parse_network_text(b, len(b), ctypes.byref(nn), ctypes.byref(nl), ctypes.byref(ns),
                              *(a.ctypes.data for a in out.values()), err)
    return out


def parse_plans_text(text, link_id):
    """SPEC plans file -> (route_off, route, depart, entry, vehicle_id) with
    route links as indices into link_id (pure host; ts_parse_plans_text)"""
    lib = load_library()
    b = text.encode() if isinstance(text, str) else bytes(text)
    ids = _a(link_id, np.int32)
    nv, ne = ctypes.c_int32(), ctypes.c_int64()
    err = ctypes.create_string_buffer(256)
    if lib.ts_parse_plans_text(b, len(b), ids.size, ids.ctypes.data, ctypes.byref(nv),
                               ctypes.byref(ne), *([None] * 5), err):
        raise TsError(err.value.decode())
    off = np.zeros(nv.value + 1, np.int64)
    route = np.zeros(max(1, ne.value), np.int32)
    dep, ent, vid = (np.zeros(nv.value, np.int32) for _ in range(3))
    lib.ts_parse_plans_text(b, len(b), ids.size, ids.ctypes.data, ctypes.byref(nv), ctypes.byref(ne),
                            off.ctypes.data, route.ctypes.data, dep.ctypes.data, ent.ctypes.data,
                            vid.ctypes.data, err)
    return off, route[:ne.value], dep, ent, vid


def debug_checks(reset=True, arm_selftest=False):
    """ts_debug_checks: (checked_build, violated_bits, first_group, count)."""
    lib = load_library()
    out = (ctypes.c_uint32 * 4)()
    mode = 2 if arm_selftest else (1 if reset else 0)
    if lib.ts_debug_checks(ctypes.cast(out, ctypes.c_void_p), mode) != 0:
        raise TsError("ts_debug_checks failed")
    return tuple(int(x) for x in out)


def nccl_unique_id():
    """128-byte NCCL communicator id for ts_nccl_init (one rank creates it)"""
    buf = ctypes.create_string_buffer(128)
    if load_library().ts_nccl_unique_id(buf):
        raise TsError("ts_nccl_unique_id failed (libnccl.so.2 not found?)")
    return buf.raw


def exchange_local(sims):
    """in-process exchange among the handles of one partition"""
    lib = load_library()
    arr = (ctypes.c_void_p * len(sims))(*[s.h for s in sims])
    rc = lib.ts_exchange_local(arr, len(sims))
    if rc:
        raise TsError(lib.ts_last_error(sims[0].h).decode())


def local_step(sims, n):
    """n whole steps of the in-process domains of one partition (ts_local_step)"""
    lib = load_library()
    arr = (ctypes.c_void_p * len(sims))(*[s.h for s in sims])
    rc = lib.ts_local_step(arr, len(sims), int(n))
    if rc:
        raise TsError(lib.ts_last_error(sims[0].h).decode())


class Sim:
    """One simulation handle (one domain, or the whole network) on one GPU."""

    def __init__(self, p_slow=0.2, seed=1, gap_G=5, desp_D=10, flags=FLAG_FUSED | FLAG_HASH,
                 device=0, tile_cells=0, group_cells=0):
        self.lib = load_library()
        cfg = Config(float(p_slow), int(seed), int(gap_G), int(desp_D), int(flags), int(device),
                     int(tile_cells), int(group_cells))
        h = ctypes.c_void_p()
        rc = self.lib.ts_create(ctypes.byref(cfg), ctypes.byref(h))
        if rc:
            raise TsError(self.lib.ts_last_error(None).decode())
        self.h = h
        self.flags = flags

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ts_destroy(self.h)
            self.h = None

    def close(self):
        self.__del__()

    def _check(self, rc):
        if rc:
            raise TsError(self.lib.ts_last_error(self.h).decode())

    @classmethod
    def from_scenario(cls, scn, t0=0, **kw):
        kw.setdefault("p_slow", scn.p_slow)
        kw.setdefault("seed", scn.seed)
        s = cls(**kw)
        s.load(scn)
        s.init(t0)
        return s

    def load(self, scn, place=True):
        i32 = lambda a: _a(a, np.int32)  # noqa: E731
        i64 = lambda a: _a(a, np.int64)  # noqa: E731
        nx, ny = i64(scn.node_x), i64(scn.node_y)
        arr = [i32(scn.link_from), i32(scn.link_to), i64(scn.link_len_mm), i32(scn.link_lanes),
               i32(scn.link_vmax), i32(scn.link_class)]
        self._check(self.lib.ts_load_network(self.h, scn.n_nodes, nx.ctypes.data, ny.ctypes.data,
                                             scn.n_links, *(a.ctypes.data for a in arr),
                                             int(scn.periodic_link)))
        veh = [i64(scn.route_off), i32(scn.route), i32(scn.depart), i32(scn.entry)]
        self._check(self.lib.ts_load_vehicles(self.h, scn.n_vehicles, *(_p(a) for a in veh)))
        self.n_veh = scn.n_vehicles
        self.n_links = scn.n_links
        self._n_nodes = scn.n_nodes
        self.lanes = np.asarray(scn.link_lanes, dtype=np.int32)
        sig = getattr(scn, "sig_node", None)
        if sig is not None and len(sig):
            a = [i32(scn.sig_node), i32(scn.sig_g0), i32(scn.sig_g1), i32(scn.sig_off)]
            self._check(self.lib.ts_set_signals(self.h, a[0].size, *(x.ctypes.data for x in a)))
        if place and scn.place_vid.size:
            pl = [i32(scn.place_vid), i32(scn.place_lane), i32(scn.place_cell), i32(scn.place_v)]
            self._check(self.lib.ts_place_vehicles(self.h, pl[0].size, *(a.ctypes.data for a in pl)))

    def load_text(self, network_text, plans_text):
        """load a SPEC network file and plans file (ts_load_network_text,
        ts_load_plans_text)"""
        for fn, t in (("ts_load_network_text", network_text), ("ts_load_plans_text", plans_text)):
            b = t.encode() if isinstance(t, str) else bytes(t)
            self._check(getattr(self.lib, fn)(self.h, b, len(b)))
        self.n_veh = sum(1 for ln in (plans_text if isinstance(plans_text, str)
                                      else plans_text.decode()).splitlines()
                         if ln.split("#")[0].strip())
        net = parse_network_text(network_text)
        self.n_links = net["link_from"].size
        self.lanes = net["link_lanes"]

    def place_at(self, vid, cursor, lane, cell, v):
        """place vehicles on link route[cursor] (restore / repartition)"""
        a = [_a(x, np.int32) for x in (vid, cursor, lane, cell, v)]
        self._check(self.lib.ts_place_vehicles_at(self.h, a[0].size, *(_p(x) for x in a)))

    def set_arrived(self, vid, t_arrive):
        a = [_a(x, np.int32) for x in (vid, t_arrive)]
        self._check(self.lib.ts_set_arrived(self.h, a[0].size, *(_p(x) for x in a)))

    def set_domain(self, k, domain_of_node, me):
        d = _a(domain_of_node, np.int32)
        self._check(self.lib.ts_set_domain(self.h, int(k), _p(d), int(me)))

    def resume(self, t):
        self._check(self.lib.ts_resume(self.h, int(t)))

    def phase(self, p, more=False):
        self._check(self.lib.ts_step_phase(self.h, int(p), int(bool(more))))

    def exchange_plan(self):
        """[(partner domain, strips per message, first strip of its segment)]"""
        cap = 4096
        nb, ns, off = np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)
        n = ctypes.c_int32()
        self._check(self.lib.ts_exchange_plan(self.h, cap, nb.ctypes.data, ns.ctypes.data,
                                              off.ctypes.data, ctypes.byref(n)))
        return [(int(nb[i]), int(ns[i]), int(off[i])) for i in range(n.value)]

    def partition(self, k, me, node_weight=None, n_nodes=None):
        """ORB of the loaded network + this handle as domain `me`
        (ts_partition); returns the partition"""
        n = int(n_nodes if n_nodes is not None else self._n_nodes)
        out = np.zeros(n, np.int32)
        w = None if node_weight is None else _a(node_weight, np.float64)
        self._check(self.lib.ts_partition(self.h, int(k), None if w is None else w.ctypes.data,
                                          int(me), out.ctypes.data))
        return out

    def nccl_init(self, unique_id, nranks, rank):
        """join the library's own NCCL communicator (native exchanges)"""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        self._check(self.lib.ts_nccl_init(self.h, buf, int(nranks), int(rank)))

    def exchange(self):
        """one native exchange of the packed strips (after ts_nccl_init)"""
        self._check(self.lib.ts_exchange(self.h))

    def exchange_buffers(self):
        """device pointers (send, recv) of the packed strip buffers"""
        s, r = ctypes.c_void_p(), ctypes.c_void_p()
        self._check(self.lib.ts_exchange_buffers(self.h, ctypes.byref(s), ctypes.byref(r)))
        return s.value, r.value

    def stream(self):
        return self.lib.ts_stream(self.h)

    def init(self, t0=0):
        self._check(self.lib.ts_init(self.h, int(t0)))

    def step(self, n=1):
        self._check(self.lib.ts_step(self.h, int(n)))

    def step_async(self, n=1):
        self._check(self.lib.ts_step_async(self.h, int(n)))

    def sync(self):
        self._check(self.lib.ts_sync(self.h))

    @property
    def t(self):
        return int(self.lib.ts_time(self.h))

    def n_cells(self, link):
        return int(self.lib.ts_link_cells(self.h, int(link)))

    def state_hash(self):
        out = ctypes.c_uint64()
        self._check(self.lib.ts_state_hash(self.h, ctypes.byref(out)))
        return int(out.value)

    def vehicles(self):
        n = self.n_veh
        st = np.zeros(n, np.int8)
        arrs = [np.zeros(n, np.int32) for _ in range(6)]
        self._check(self.lib.ts_read_vehicles(self.h, _p(st), *(_p(a) for a in arrs)))
        return dict(status=st, link=arrs[0], lane=arrs[1], cell=arrs[2], v=arrs[3],
                    cursor=arrs[4], t_arrive=arrs[5])

    def cells(self, link):
        n = self.n_cells(link)
        out = np.zeros(int(self.lanes[link]) * n, np.int32)
        self._check(self.lib.ts_read_cells(self.h, int(link), out.ctypes.data))
        return out.reshape(int(self.lanes[link]), n)

    def raw(self, link):
        """raw per-lane codes and vid regions of a single-tile link"""
        L = int(self.lanes[link])
        wp = (self.n_cells(link) + 3) & ~3
        code = np.zeros(L * wp, np.uint8)
        vid = np.zeros(L * wp, np.int32)
        pitch = ctypes.c_int32()
        self._check(self.lib.ts_read_raw(self.h, int(link), code.ctypes.data, vid.ctypes.data,
                                         ctypes.byref(pitch)))
        return code.reshape(L, wp), vid.reshape(L, wp)

    def history(self, t_from, n):
        h = np.zeros(n, np.uint64)
        cols = [np.zeros(n, np.int64) for _ in range(5)]
        self._check(self.lib.ts_read_history(self.h, int(t_from), int(n), _p(h),
                                             *(_p(c) for c in cols)))
        return dict(hash=[int(x) for x in h], active=cols[0], arrivals=cols[1],
                    injections=cols[2], lane_changes=cols[3], crossings=cols[4])

    def flow(self, t_from, n):
        """sum of velocities of S(t), t in [t_from, t_from + n)"""
        out = np.zeros(n, np.int64)
        self._check(self.lib.ts_read_flow(self.h, int(t_from), int(n), _p(out)))
        return out

    def totals(self):
        out = np.zeros(8, np.int64)
        self._check(self.lib.ts_get_totals(self.h, out.ctypes.data))
        keys = ["active", "pending", "arrived", "vehicle_updates", "lane_cells", "tiles",
                "device_bytes", "alg_bytes_per_step"]
        return dict(zip(keys, out.tolist()))

    def link_work(self):
        out = np.zeros(self.n_links, np.int64)
        self._check(self.lib.ts_get_link_work(self.h, out.ctypes.data))
        return out

    def load_stats(self):
        """accumulated load statistics (ts_get_load): (vehicle updates per
        link, node units per node)"""
        lw = np.zeros(self.n_links, np.int64)
        nw = np.zeros(self._n_nodes, np.int64)
        self._check(self.lib.ts_get_load(self.h, lw.ctypes.data, nw.ctypes.data))
        return lw, nw

    def last_exchange_timing(self):
        """(total ms, count) of the timed native exchanges of the last ts_step"""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(self.lib.ts_last_exchange_timing(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def busy_time(self):
        """device ms of all step work since the previous call (resets)"""
        ms = ctypes.c_double()
        self._check(self.lib.ts_busy_time(self.h, ctypes.byref(ms)))
        return ms.value

    def last_timing(self):
        tot, mv, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        self._check(self.lib.ts_last_timing(self.h, ctypes.byref(tot), ctypes.byref(mv),
                                            ctypes.byref(n)))
        return dict(total_ms=tot.value, move_ms=mv.value, move_launches=n.value)

    def run_hashes(self, n):
        hs = []
        for _ in range(n):
            self.step(1)
            hs.append(self.state_hash())
        return hs
