"""CPU oracle of the TRANSIMS CA step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the cpu_baseline /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product path (``paper_cs_0105004_b200``) never imports it.

Thin ctypes wrapper over ``tsim_oracle.c`` (plain single-threaded C, see
its header for the paper passages it follows).  Parity status of each
function is listed in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "tsim_oracle.c")
_lib = None

PENDING, ACTIVE, ARRIVED = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no CUDA involved)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "tsim_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-g", "-std=c99", "-Wall", "-shared", "-fPIC",
                               "-o", _SO, _SRC])
    return _SO


def _load():
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(build())
    P, I32, I64, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    lib.or_create.restype = P
    lib.or_create.argtypes = [ctypes.c_double, U64, I32, I32]
    lib.or_destroy.argtypes = [P]
    lib.or_last_error.restype = ctypes.c_char_p
    lib.or_last_error.argtypes = [P]
    lib.or_load_network.argtypes = [P, I32, P, P, I32, P, P, P, P, P, P, I32]
    lib.or_load_vehicles.argtypes = [P, I32, P, P, P, P]
    lib.or_place_vehicles.argtypes = [P, I32, P, P, P, P]
    lib.or_init.argtypes = [P, I32]
    lib.or_step.argtypes = [P, I32]
    lib.or_time.restype = I32
    lib.or_time.argtypes = [P]
    lib.or_n_cells.restype = I32
    lib.or_n_cells.argtypes = [P, I32]
    lib.or_total_lane_cells.restype = I64
    lib.or_total_lane_cells.argtypes = [P]
    lib.or_state_hash.restype = U64
    lib.or_state_hash.argtypes = [P]
    lib.or_counters.argtypes = [P, P]
    lib.or_read_vehicles.argtypes = [P, P, P, P, P, P, P, P]
    lib.or_read_cells.argtypes = [P, I32, P]
    lib.or_turn_type.restype = I32
    lib.or_turn_type.argtypes = [P, I32, I32]
    lib.or_philox4x32_10.argtypes = [P, P, P]
    lib.or_mix.restype = U64
    lib.or_mix.argtypes = [I32, I32, I32, I32, I32]
    lib.or_set_partition.argtypes = [P, I32, P]
    lib.or_domain_stats.argtypes = [P, P, I32]
    lib.or_set_brake_override.argtypes = [P, P]
    lib.or_set_signals.argtypes = [P, I32, P, P, P, P]
    _lib = lib
    return lib


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


def philox4x32_10(ctr, key):
    """Philox4x32-10 of the oracle; ctr uint32[4], key uint32[2] -> uint32[4]."""
    lib = _load()
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib.or_philox4x32_10(c.ctypes.data, k.ctypes.data, out.ctypes.data)
    return out


def mix(vid, link, lane, cell, v):
    return int(_load().or_mix(vid, link, lane, cell, v))


class OracleError(RuntimeError):
    pass


class Oracle:
    """One simulation on the CPU oracle."""

    def __init__(self, p_slow=0.2, seed=1, gap_G=5, desp_D=10):
        self.lib = _load()
        self.h = self.lib.or_create(float(p_slow), int(seed), int(gap_G), int(desp_D))
        self._keep = []

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.or_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self.lib.or_last_error(self.h).decode())

    @classmethod
    def from_scenario(cls, scn, t0=0, p_slow=None, seed=None, **kw):
        o = cls(p_slow=scn.p_slow if p_slow is None else p_slow,
                seed=scn.seed if seed is None else seed, **kw)
        o.load(scn)
        o.init(t0)
        return o

    def load(self, scn):
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
        net = [i64(scn.node_x), i64(scn.node_y), i32(scn.link_from), i32(scn.link_to),
               i64(scn.link_len_mm), i32(scn.link_lanes), i32(scn.link_vmax),
               i32(scn.link_class)]
        self._check(self.lib.or_load_network(
            self.h, scn.n_nodes, net[0].ctypes.data, net[1].ctypes.data, scn.n_links,
            *(a.ctypes.data for a in net[2:]), int(scn.periodic_link)))
        veh = [i64(scn.route_off), i32(scn.route), i32(scn.depart), i32(scn.entry)]
        self._check(self.lib.or_load_vehicles(self.h, scn.n_vehicles,
                                              *(_p(a) for a in veh)))
        self.n_veh = scn.n_vehicles
        self.n_links = scn.n_links
        self.lanes = np.asarray(scn.link_lanes, dtype=np.int32)
        if scn.place_vid.size:
            pl = [i32(scn.place_vid), i32(scn.place_lane), i32(scn.place_cell),
                  i32(scn.place_v)]
            self._check(self.lib.or_place_vehicles(self.h, pl[0].size, *(a.ctypes.data for a in pl)))
        sig = getattr(scn, "sig_node", None)
        if sig is not None and len(sig):
            a = [i32(scn.sig_node), i32(scn.sig_g0), i32(scn.sig_g1), i32(scn.sig_off)]
            self._check(self.lib.or_set_signals(self.h, a[0].size, *(x.ctypes.data for x in a)))

    def init(self, t0=0):
        self._check(self.lib.or_init(self.h, int(t0)))

    def step(self, n=1):
        self._check(self.lib.or_step(self.h, int(n)))

    @property
    def t(self):
        return int(self.lib.or_time(self.h))

    def n_cells(self, link):
        return int(self.lib.or_n_cells(self.h, int(link)))

    def state_hash(self):
        return int(self.lib.or_state_hash(self.h))

    def counters(self):
        out = np.zeros(10, dtype=np.int64)
        self.lib.or_counters(self.h, out.ctypes.data)
        keys = ["active", "pending", "arrived", "collisions", "lane_changes", "crossings",
                "injections", "arrivals", "vehicle_updates", "sum_v"]
        return dict(zip(keys, out.tolist()))

    def vehicles(self):
        n = self.n_veh
        st = np.zeros(n, np.int8)
        arrs = [np.zeros(n, np.int32) for _ in range(6)]
        self._check(self.lib.or_read_vehicles(self.h, st.ctypes.data, *(a.ctypes.data for a in arrs)))
        return dict(status=st, link=arrs[0], lane=arrs[1], cell=arrs[2], v=arrs[3],
                    cursor=arrs[4], t_arrive=arrs[5])

    def cells(self, link):
        n = self.n_cells(link)
        out = np.zeros(int(self.lanes[link]) * n, np.int32)
        self._check(self.lib.or_read_cells(self.h, int(link), out.ctypes.data))
        return out.reshape(int(self.lanes[link]), n)

    def turn_type(self, k, k2):
        return int(self.lib.or_turn_type(self.h, int(k), int(k2)))

    def set_partition(self, domain_of_node):
        d = np.ascontiguousarray(domain_of_node, dtype=np.int32)
        k = int(d.max()) + 1 if d.size else 1
        self._check(self.lib.or_set_partition(self.h, k, d.ctypes.data))
        self.k = k

    def set_partition_k(self, k, domain_of_node):
        d = np.ascontiguousarray(domain_of_node, dtype=np.int32)
        self._check(self.lib.or_set_partition(self.h, int(k), d.ctypes.data))
        self.k = int(k)

    def domain_stats(self):
        k = getattr(self, "k", 1)
        out = np.zeros(max(4, 4 * k), np.int64)
        self.lib.or_domain_stats(self.h, out.ctypes.data, out.size)
        return out.reshape(-1, 4)

    def set_brake_override(self, mask):
        if mask is None:
            self.lib.or_set_brake_override(self.h, None)
        else:
            m = np.ascontiguousarray(mask, dtype=np.uint8)
            self.lib.or_set_brake_override(self.h, m.ctypes.data)

    def run_hashes(self, n):
        """hash of S(t+1) after each of n steps"""
        hs = []
        for _ in range(n):
            self.step(1)
            hs.append(self.state_hash())
        return hs
