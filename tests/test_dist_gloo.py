"""The N > 1 host path on CPU (world size 2 and 4, gloo): the exchange plan
every rank derives on its own must pair up (one buffer per neighbour, the
same size both ways), the point-to-point exchange
routine used by DistDomain must deliver every buffer to its partner, the
per-domain reads must merge to one state, and the max-over-ranks timing
reduction used by bench.py must take the slowest rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import scenarios


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_cs_0105004_b200 as tsim
    from paper_cs_0105004_b200 import domains
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scn = scenarios.config("1")
        dom = domains.partition(scn, world)
        peers, strips = tsim.domain_plan(scn, world, dom, rank)
        plans = [None] * world
        dist.all_gather_object(plans, (peers, strips))
        # symmetric: my message to p has the size of p's message to me
        for p, n in zip(peers, strips):
            pp, pn = plans[p]
            assert rank in pp and pn[pp.index(rank)] == n, (rank, p)
        # N_spl / neighbour graph agree with the plan
        n_spl, pairs = domains.split_stats(scn, dom)
        nb = sorted({b for a, b in pairs if a == rank} | {a for a, b in pairs if b == rank})
        assert nb == peers
        sb = tsim.strip_bytes()
        sends = [torch.full((n * sb,), (rank * 16 + p) % 251, dtype=torch.uint8)
                 for p, n in zip(peers, strips)]
        recvs = [torch.zeros(n * sb, dtype=torch.uint8) for n in strips]
        for _ in range(3):  # two exchanges per step, several steps
            domains.exchange_p2p(sends, recvs, peers)
            for p, r in zip(peers, recvs):
                assert torch.all(r == (p * 16 + rank) % 251), (rank, p)
        # slowest rank decides the step time (bench.py)
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == float(world)
        q.put((rank, "ok", n_spl, len(peers)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_exchange_plan(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, msg, n_spl, nnb in res:
        assert msg == "ok", (rank, msg)
        assert nnb >= 1


def test_merge_vehicles():
    from paper_cs_0105004_b200 import domains
    A, R, P, X = domains.ACTIVE, domains.ARRIVED, domains.PENDING, domains.ABSENT
    n = 5
    base = {k: np.full(n, -1, np.int32) for k in ("link", "lane", "cell", "v", "cursor",
                                                    "t_arrive")}
    p0 = dict(base, status=np.array([A, X, P, X, R], np.int8))
    p1 = dict(base, status=np.array([X, A, X, R, R], np.int8))
    p0["link"] = np.array([7, -1, -1, -1, -1], np.int32)
    p1["link"] = np.array([-1, 9, -1, -1, -1], np.int32)
    m = domains.merge_vehicles([p0, p1])
    assert m["status"].tolist() == [A, A, P, R, R]
    assert m["link"].tolist()[:2] == [7, 9]
    p2 = dict(base, status=np.array([X, X, X, X, X], np.int8))
    with pytest.raises(Exception):
        domains.merge_vehicles([p2, p2])


def test_orb_weights_balance():
    """ORB with the cells x lanes weights balances the load"""
    from paper_cs_0105004_b200 import domains
    scn = scenarios.portland(n_nodes=600, n_edges=800, n_veh=100, side_km=8.0, n_zones=16, seed=2)
    for k in (2, 4, 8):
        dom = domains.partition(scn, k)
        lw = domains.link_cells(scn) * np.asarray(scn.link_lanes)
        load = np.zeros(k)
        np.add.at(load, dom[scn.link_from], 0.5 * lw)
        np.add.at(load, dom[scn.link_to], 0.5 * lw)
        assert load.max() / load.mean() < 1.25, (k, load)


def _merge_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_cs_0105004_b200 import domains
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        parts = _synthetic_parts(world)
        got = domains.merge_vehicles_dist(parts[rank])
        want = domains.merge_vehicles(parts)
        q.put((rank, all(np.array_equal(got[k], want[k]) for k in want)))
    finally:
        dist.destroy_process_group()


def _synthetic_parts(world, n=5000, seed=3):
    """per-domain reads of one state: every vehicle reported ACTIVE /
    ARRIVED / PENDING by exactly one domain, ABSENT by the others"""
    from paper_cs_0105004_b200 import domains
    rng = np.random.default_rng(seed)
    owner = rng.integers(0, world, n)
    st = rng.choice([domains.ACTIVE, domains.ARRIVED, domains.PENDING], n)
    parts = []
    for d in range(world):
        mine = owner == d
        p = {"status": np.where(mine, st, domains.ABSENT).astype(np.int8)}
        for k in ("link", "lane", "cell", "v", "cursor", "t_arrive"):
            val = rng.integers(0, 1000, n).astype(np.int32)
            p[k] = np.where(mine, (np.arange(n) * 7 + len(k)) % 997, val).astype(np.int32)
        parts.append(p)
    return parts


@pytest.mark.parametrize("world", [2, 3])
def test_merge_vehicles_dist_matches_local(world):
    """the cross-rank merge used by DistDomain.vehicles / rebalance equals
    the in-process merge of the same per-domain reads"""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_merge_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
