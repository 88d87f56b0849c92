"""Domain decomposition of the TRANSIMS CA step (§4, :366-452).

The network is cut into k domains by orthogonal recursive bisection of its
nodes; a link whose end nodes fall into different
domains is split at its middle (R16) and each side keeps a mirror of the
other side's 5-cell strip next to the cut (R17).  Every step exchanges the
strips twice -- after the lane change and after the move
-- with each neighbour domain, one buffer per neighbour.
The simulation result does not depend on k or on the partition
(SPEC.md:326), which is what the tests check against the CPU oracle.

Each domain is one libtsim handle; its kernels, the strip packing and
unpacking all run in the library (csrc/).  This module only moves the
packed buffers between handles:

* ``LocalDomains``: all k domains in this process (one or several GPUs);
  the exchange is an in-process device copy (``ts_exchange_local``).
* ``DistDomain``: one domain per rank of a torch.distributed group (one
  process per GPU); the exchange is point-to-point send/recv with every
  neighbour -- NCCL over NVLink on B200s, gloo in the CPU tests.

Adaptive rebalancing: per-link work counters and the
measured per-domain step times give node weights; a new ORB partition is
computed and the state migrates by a read / restore at the current time
(exact: the state S(t) is the whole simulation state).
"""
from __future__ import annotations

import numpy as np

from . import tsim as _t

ACTIVE, ARRIVED, PENDING, ABSENT = _t.ACTIVE, _t.ARRIVED, _t.PENDING, _t.ABSENT


# ------------------------------------------------------------- partition
def link_cells(scn):
    """cells per link, round-half-up of length / 7.5 m (R1)"""
    return np.maximum(1, (np.asarray(scn.link_len_mm, np.int64) + 3750) // 7500)


def node_weights(scn, link_work=None):
    """ORB node weights: half of the load of every attached link
    (SPEC.md:373-379).  Load = cells x lanes, or the
    measured per-link work when given."""
    if link_work is None:
        lw = link_cells(scn) * np.asarray(scn.link_lanes, np.int64)
    else:
        lw = np.asarray(link_work, np.float64)
    w = np.zeros(scn.n_nodes, np.float64)
    np.add.at(w, np.asarray(scn.link_from), 0.5 * lw)
    np.add.at(w, np.asarray(scn.link_to), 0.5 * lw)
    return w + 1e-9


def partition(scn, k, weights=None, method="orb"):
    """domain of every node: ORB on the node coordinates
    or the multilevel graph partitioner"""
    if weights is None:
        weights = node_weights(scn)
    if method == "multilevel":
        return _t.multilevel_partition(scn, k, weights)
    return _t.orb_partition(scn.node_x, scn.node_y, k, weights)


def link_times(link_work_per_domain, domain_ms):
    """execution time per link ("we collect the execution
    time of each link and intersection"): each domain's measured step time
    apportioned to its links by their share of the domain's work (vehicle
    updates; a split link's halves are counted by their owners) -- the
    library's ts_load_times"""
    lt = np.zeros(len(link_work_per_domain[0]), np.float64)
    for lw, ms in zip(link_work_per_domain, domain_ms):
        _t.load_times(ms, lw, link_time=lt)
    return lt


def load_times(windows, domain_ms, n_nodes):
    """link and node times of a window from every domain's (link work, node
    work) and measured time (ts_load_times, accumulated over the domains)"""
    lt = np.zeros(len(windows[0][0]), np.float64)
    nt = np.zeros(n_nodes, np.float64)
    for (lw, nw), ms in zip(windows, domain_ms):
        _t.load_times(ms, lw, nw, link_time=lt, node_time=nt)
    return lt, nt


def rebalance_weights(scn, link_work_per_domain, domain_ms):
    """node weights for the next partition from the measured link times
    (ts_rebalance: half of every attached link; links
    without work keep a floor of their static load share)"""
    lt = link_times(link_work_per_domain, domain_ms)
    return _t.rebalance(scn, 1, lt)[1]


def split_stats(scn, dom):
    """N_spl (split links) and the domain neighbour graph"""
    d = np.asarray(dom)
    a, b = d[np.asarray(scn.link_from)], d[np.asarray(scn.link_to)]
    cut = a != b
    pairs = set(zip(a[cut].tolist(), b[cut].tolist()))
    return int(cut.sum()), sorted(pairs)


# ----------------------------------------------------------------- merge
def merge_vehicles(parts):
    """merge per-domain vehicle reads: per vehicle, the domain reporting it
    ACTIVE, else ARRIVED, else PENDING (include/tsim.h)"""
    out = {k: np.array(v, copy=True) for k, v in parts[0].items()}
    rank = np.zeros(4, np.int8)
    rank[[ACTIVE, ARRIVED, PENDING, ABSENT]] = [3, 2, 1, 0]
    best = rank[out["status"]]
    for p in parts[1:]:
        r = rank[p["status"]]
        take = r > best
        for k in out:
            out[k][take] = p[k][take]
        best = np.maximum(best, r)
    if np.any(best == 0):
        raise _t.TsError(f"{int(np.sum(best == 0))} vehicles reported by no domain")
    return out


def merge_vehicles_dist(part, group=None):
    """merge_vehicles across the ranks of a torch.distributed group: every
    rank passes its own domain's read and gets the merged state (per
    vehicle the report of the rank with the highest status rank; two
    max-reductions, so any backend works: NCCL on GPUs, gloo on CPUs)"""
    import torch
    import torch.distributed as dist
    dev = (torch.device("cuda", torch.cuda.current_device())
           if dist.get_backend(group) == "nccl" else torch.device("cpu"))
    order = np.array([1, 3, 2, 0], np.int32)  # PENDING 0, ACTIVE 1, ARRIVED 2, ABSENT 3 -> rank
    key = torch.as_tensor(order[np.asarray(part["status"], np.int64)], device=dev)
    best = key.clone()
    dist.all_reduce(best, op=dist.ReduceOp.MAX, group=group)
    if bool((best == 0).any()):
        raise _t.TsError(f"{int((best == 0).sum())} vehicles reported by no domain")
    mine = key == best
    out = {}
    lo = torch.iinfo(torch.int32).min
    for k, v in part.items():
        x = torch.as_tensor(np.asarray(v, np.int32), device=dev)
        x = torch.where(mine, x, torch.full_like(x, lo))
        dist.all_reduce(x, op=dist.ReduceOp.MAX, group=group)
        out[k] = x.cpu().numpy().astype(np.asarray(v).dtype)
    return out


def restore_into(sim, state, t):
    """place a vehicle state (merged read at time t) into a fresh handle
    (loaded without initial placement) and resume at t"""
    st = state["status"]
    a = np.nonzero(st == ACTIVE)[0]
    if a.size:
        sim.place_at(a, state["cursor"][a], state["lane"][a], state["cell"][a], state["v"][a])
    r = np.nonzero(st == ARRIVED)[0]
    if r.size:
        sim.set_arrived(r, state["t_arrive"][r])
    sim.resume(t)


# ------------------------------------------------------ in-process domains
class LocalDomains:
    """k domains of one partition, all in this process."""

    def __init__(self, scn, k, domain_of_node=None, t0=0, devices=(0,),
                 flags=_t.FLAG_FUSED | _t.FLAG_HASH, state=None, **kw):
        self.scn, self.k, self.flags, self.kw = scn, int(k), flags, kw
        self.dom = np.asarray(partition(scn, k) if domain_of_node is None else domain_of_node,
                              np.int32)
        self.devices = list(devices)
        self.sims = []
        for me in range(self.k):
            s = _t.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=flags,
                       device=self.devices[me % len(self.devices)], **kw)
            s.load(scn, place=state is None)
            s.set_domain(self.k, self.dom, me)
            if state is None:
                s.init(t0)
            else:
                restore_into(s, state, t0)
            self.sims.append(s)
        self._exchange()
        for s in self.sims:
            s.phase(2)

    def _exchange(self):
        if self.k > 1:
            _t.exchange_local(self.sims)

    def step(self, n=1):
        """n whole steps of all domains inside the library (ts_local_step;
        CUDA-graph replays with FLAG_GRAPH)"""
        if n > 0:
            _t.local_step(self.sims, n)

    def step_phases(self, n=1):
        """the same steps driven phase by phase from here (ts_step_phase +
        ts_exchange_local)"""
        for i in range(n):
            for s in self.sims:
                s.phase(0)
            self._exchange()
            for s in self.sims:
                s.phase(1, more=i < n - 1)
            self._exchange()
            for s in self.sims:
                s.phase(2)

    @property
    def t(self):
        return self.sims[0].t

    def vehicles(self):
        return merge_vehicles([s.vehicles() for s in self.sims])

    def state_hash(self):
        return sum(s.state_hash() for s in self.sims) & (2**64 - 1)

    def history(self, t_from, n):
        hs = [s.history(t_from, n) for s in self.sims]
        out = {"hash": [sum(h["hash"][i] for h in hs) & (2**64 - 1) for i in range(n)]}
        for key in ("active", "arrivals", "injections", "lane_changes", "crossings"):
            out[key] = sum(h[key] for h in hs)
        return out

    def totals(self):
        ts = [s.totals() for s in self.sims]
        return {k: sum(t[k] for t in ts) for k in ts[0]}

    def link_work(self):
        return sum(s.link_work() for s in self.sims)

    def rebalance(self, method="orb"):
        """adaptive repartition (BASELINE: "rebalanced from
        measured per-domain step times"): per-domain device time and per-link
        / per-node work since the last rebalance (ts_busy_time, ts_get_load)
        -> link and node times (ts_load_times) -> node weights and a new
        partition (ts_rebalance); the state migrates exactly.  Needs
        FLAG_LINK_WORK.  Returns (new domain_of_node, per-domain ms of the
        window)."""
        ms = [s.busy_time() for s in self.sims]
        loads = [s.load_stats() for s in self.sims]
        base = getattr(self, "_load_base", None)
        win = ([(lw - bl, nw - bn) for (lw, nw), (bl, bn) in zip(loads, base)]
               if base is not None and len(base) == len(loads) else loads)
        lt, nt = load_times(win, ms, self.scn.n_nodes)
        dom, _ = _t.rebalance(self.scn, self.k, lt, nt, method=method)
        self.repartition(dom)
        self._load_base = [s.load_stats() for s in self.sims]
        for s in self.sims:  # the migration's own work is not step time
            s.busy_time()
        return dom, ms

    def repartition(self, domain_of_node, k=None):
        """migrate to a new partition at the current time (exact)"""
        t, state = self.t, self.vehicles()
        self.close()
        self.__init__(self.scn, self.k if k is None else k, domain_of_node, t0=t,
                      devices=self.devices, flags=self.flags, state=state, **self.kw)

    def close(self):
        for s in self.sims:
            s.close()
        self.sims = []


# ------------------------------------------------- one domain per rank
def exchange_p2p(sends, recvs, peers, group=None):
    """one message to and from every peer (batched isend / irecv); blocks
    until the receives are complete (NCCL: until the current stream is
    ordered after them)"""
    import torch.distributed as dist
    if not peers:
        return
    ops = []
    for s, r, p in zip(sends, recvs, peers):
        g = p if group is None else dist.get_global_rank(group, p)
        ops.append(dist.P2POp(dist.isend, s, g, group))
        ops.append(dist.P2POp(dist.irecv, r, g, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


class _CudaBuf:
    """zero-copy view of a library-owned device buffer for torch"""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


class DistDomain:
    """The domain of this rank.  Exchanges: native (the library's own NCCL
    communicator; ts_step runs whole steps) when `native` and the group is
    the whole world with ranks = domains, else torch.distributed
    batched isend / irecv between the phases."""

    def __init__(self, scn, domain_of_node, device=0, t0=0, flags=_t.FLAG_FUSED, group=None,
                 state=None, native=False, **kw):
        import torch
        import torch.distributed as dist
        self.group = group
        self.scn, self.flags, self.kw = scn, flags, kw
        self.rank = dist.get_rank(group)
        self.k = dist.get_world_size(group)
        self.dev = device
        self.sim = _t.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=flags, device=device, **kw)
        self.sim.load(scn, place=state is None)
        self.sim.set_domain(self.k, np.asarray(domain_of_node, np.int32), self.rank)
        if state is None:
            self.sim.init(t0)
        else:
            restore_into(self.sim, state, t0)
        self.plan = self.sim.exchange_plan()
        sb = _t.strip_bytes()
        sp, rp = self.sim.exchange_buffers()
        cuda = f"cuda:{device}"
        self.peers = [p for p, _, _ in self.plan]
        self.sends = [torch.as_tensor(_CudaBuf(sp + off * sb, n * sb), device=cuda)
                      for _, n, off in self.plan]
        self.recvs = [torch.as_tensor(_CudaBuf(rp + off * sb, n * sb), device=cuda)
                      for _, n, off in self.plan]
        self.stream = torch.cuda.ExternalStream(self.sim.stream(), device=cuda)
        # a backend without device tensors (gloo) exchanges host copies of
        # the packed strips
        self.host_staging = dist.get_backend(group) != "nccl"
        if self.host_staging:  # pageable: no host-allocator events on the library's stream
            self.hsends = [torch.empty(t.numel(), dtype=torch.uint8) for t in self.sends]
            self.hrecvs = [torch.empty(t.numel(), dtype=torch.uint8) for t in self.recvs]
        self.exchange_ms = 0.0
        self.native = False
        if native and group is None:
            # every rank must take the same transport: probe libnccl on all
            # ranks first (a rank missing it would leave the others waiting in
            # the communicator's collective init)
            try:
                _t.nccl_unique_id()
                ok = 1
            except _t.TsError:
                ok = 0
            dev = (torch.device(cuda) if dist.get_backend() == "nccl" else torch.device("cpu"))
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 1:
                uid = [_t.nccl_unique_id() if self.rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                self.sim.nccl_init(uid[0], self.k, self.rank)
                self.native = True
        self.exchange()
        self.sim.phase(2)

    def exchange(self):
        if self.native:
            self.sim.exchange()
            return
        import torch
        if self.host_staging:  # device -> host, exchange, host -> device
            with torch.cuda.stream(self.stream):
                for h, d in zip(self.hsends, self.sends):
                    h.copy_(d)
            exchange_p2p(self.hsends, self.hrecvs, self.peers, self.group)
            with torch.cuda.stream(self.stream):
                for d, h in zip(self.recvs, self.hrecvs):
                    d.copy_(h)
            self.stream.synchronize()
            return
        with torch.cuda.stream(self.stream):
            exchange_p2p(self.sends, self.recvs, self.peers, self.group)

    def step(self, n=1):
        if self.native:  # whole steps inside the library (both exchanges native)
            self.sim.step(n)
            return
        for i in range(n):
            self.sim.phase(0)
            self.exchange()
            self.sim.phase(1, more=i < n - 1)
            self.exchange()
            self.sim.phase(2)

    @property
    def t(self):
        return self.sim.t

    def close(self):
        """drop the torch views of the library's buffers and stream, then the
        handle (its stream and memory go away with it)"""
        import torch
        torch.cuda.synchronize(self.dev)
        self.sends = self.recvs = self.hsends = self.hrecvs = []
        self.stream = None
        self.sim.close()

    def vehicles(self):
        """the merged state of all ranks (every rank gets it)"""
        return merge_vehicles_dist(self.sim.vehicles(), self.group)

    def rebalance(self, method="orb"):
        """adaptive repartition across the ranks: this
        domain's device time since the last rebalance split over its links by
        their work, summed over the ranks into link times -> node weights ->
        the same new partition on every rank; the merged state S(t) is
        restored into a new handle.  Needs FLAG_LINK_WORK."""
        import torch
        import torch.distributed as dist
        ms = self.sim.busy_time()
        lw, nw = self.sim.load_stats()
        base = getattr(self, "_load_base", None)
        if base is not None:
            lw, nw = lw - base[0], nw - base[1]
        lt_me, nt_me = _t.load_times(ms, lw, nw)
        dev = (torch.device("cuda", self.dev) if dist.get_backend(self.group) == "nccl"
               else torch.device("cpu"))
        both = torch.as_tensor(np.concatenate([lt_me, nt_me]), dtype=torch.float64, device=dev)
        dist.all_reduce(both, op=dist.ReduceOp.SUM, group=self.group)
        both = both.cpu().numpy()
        lt, nt = both[:lw.size], both[lw.size:]
        dom, _ = _t.rebalance(self.scn, self.k, lt, nt, method=method)
        t, state = self.t, self.vehicles()
        self.close()
        self.__init__(self.scn, dom, device=self.dev, t0=t, flags=self.flags, group=self.group,
                      state=state, native=self.native, **self.kw)
        self._load_base = self.sim.load_stats()
        self.sim.busy_time()
        return dom
