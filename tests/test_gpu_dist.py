"""The multi-rank data plane on one GPU (G1, H2/H7; PAPER.md:404-427 and
:897-900): two PROCESSES, one domain each (DistDomain), exchanging the real
packed boundary strips twice per step through torch.distributed (gloo,
strips staged through host memory), bit-exact with the undivided CPU oracle
at every step; then one adaptive rebalance across the ranks (ts_get_load ->
ts_load_times -> all-reduce -> ts_rebalance) and more
steps, still bit-exact.  The ranks never wait on one another inside a
kernel (every wait is on the host), so sharing one GPU is safe."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scenario(name):
    import scenarios
    if name == "config1":
        return scenarios.config("1")
    s = scenarios.portland(n_nodes=600, n_edges=800, n_veh=8000, side_km=8.0, n_zones=64, seed=2)
    s.depart = (s.depart // 12).astype(np.int32)
    return s


def _worker(rank, world, port, name, steps, q):
    import torch
    import torch.distributed as dist

    import paper_cs_0105004_b200 as tsim
    from paper_cs_0105004_b200 import domains
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scn = _scenario(name)
        o = None
        if rank == 0:
            import oracle
            o = oracle.Oracle.from_scenario(scn)
        dom = domains.partition(scn, world)
        d = domains.DistDomain(scn, dom, device=0,
                               flags=tsim.FLAG_FUSED | tsim.FLAG_HASH | tsim.FLAG_LINK_WORK)
        assert d.host_staging and not d.native and len(d.peers) >= 1
        checked = 0
        for phase in range(2):
            for _ in range(steps // 20):
                t_from = d.t + 1
                d.step(20)
                hs = [None] * world
                dist.all_gather_object(hs, d.sim.history(t_from, 20)["hash"])
                if rank == 0:
                    oh = o.run_hashes(20)
                    tot = [sum(h[i] for h in hs) % 2**64 for i in range(20)]
                    bad = [t_from + i for i in range(20) if tot[i] != oh[i]]
                    assert not bad, f"{name}: per-step hash differs at t={bad[:5]}"
                    checked += 20
            v = d.vehicles()
            if rank == 0:
                vo = o.vehicles()
                for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
                    assert np.array_equal(vo[key], v[key]), (name, key, d.t)
            if phase == 0:
                new = d.rebalance()
                assert d.t == (o.t if rank == 0 else d.t)
                assert new.shape == dom.shape
        d.close()
        q.put((rank, "ok", checked))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-800:], 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,steps", [("config1", 300), ("portland", 200)])
def test_two_processes_one_gpu(name, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, name, steps, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = []
    import queue
    import time
    t0 = time.time()
    while len(res) < len(ps) and time.time() - t0 < 600:
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:  # a rank that died without reporting fails the test now
            dead = [p.exitcode for p in ps if p.exitcode not in (None, 0)]
            assert not dead, f"rank exited with {dead}"
    for p in ps:
        p.join(timeout=60)
    assert len(res) == len(ps), "ranks did not report"
    for rank, msg, checked in res:
        assert msg == "ok", (rank, msg)
    assert max(c for _, _, c in res) == 2 * steps
