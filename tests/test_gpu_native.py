"""The library's native exchange transport on one GPU:
ts_nccl_init / ts_exchange through DistDomain(native=True) with a single
rank (a one-domain partition: the exchange has no partners), bit-exact with
the oracle; bad ranks are rejected.  The multi-rank exchange itself needs
one GPU per rank."""
import socket

import numpy as np
import pytest

import oracle
import scenarios

pytestmark = pytest.mark.gpu

tsim = pytest.importorskip("paper_cs_0105004_b200")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_native_single_rank():
    import torch
    import torch.distributed as dist
    from paper_cs_0105004_b200 import domains
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda:0"))
    try:
        scn = scenarios.config("1")
        d = domains.DistDomain(scn, np.zeros(scn.n_nodes, np.int32), device=0,
                               flags=tsim.FLAG_FUSED | tsim.FLAG_HASH, native=True)
        assert d.native
        o = oracle.Oracle.from_scenario(scn)
        for _ in range(4):
            t_from = o.t + 1
            oh = o.run_hashes(50)
            d.step(50)
            assert list(d.sim.history(t_from, 50)["hash"]) == list(oh)
    finally:
        dist.destroy_process_group()


def test_nccl_init_rejects_bad_ranks():
    scn = scenarios.config("1")
    s = tsim.Sim.from_scenario(scn, flags=tsim.FLAG_FUSED)
    uid = tsim.nccl_unique_id()
    with pytest.raises(tsim.TsError):
        s.nccl_init(uid, 2, 0)  # one domain, two ranks
    with pytest.raises(tsim.TsError):
        s.nccl_init(uid, 1, 1)
