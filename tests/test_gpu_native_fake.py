"""The library's native multi-rank step (ts_nccl_init + ts_step with
neighbours: LC, exchange #1, move, exchange #2 inside the library, PAPER.md
:412-427 and :897-900) with real partners on one GPU.  libnccl cannot put
two ranks on one device, so the exchanges go through tests/fake_nccl.cpp
(TSIM_NCCL_LIB): every rank is a handle of one process on its own host
thread, each send / recv pair a stream-ordered device copy (no GPU-side
waiting).  Everything else -- the step loop, the phase order, the strip
packing and unpacking, the message offsets and sizes -- is the product
path `bench.py --gpus N` takes on N GPUs.  Bit-exact with the undivided
oracle at every step."""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = textwrap.dedent(r'''
    import sys, threading
    import numpy as np
    sys.path.insert(0, {root!r})
    import oracle, scenarios
    import paper_cs_0105004_b200 as tsim
    from paper_cs_0105004_b200 import domains

    scn = {scn}
    k, steps, chunk = {k}, {steps}, {chunk}
    dom = np.asarray(domains.partition(scn, k), np.int32)
    sims = []
    for me in range(k):
        s = tsim.Sim(p_slow=scn.p_slow, seed=scn.seed, flags=tsim.FLAG_FUSED | tsim.FLAG_HASH)
        s.load(scn)
        s.set_domain(k, dom, me)
        s.init(0)
        sims.append(s)
    assert sum(len(s.exchange_plan()) for s in sims) > 0, "no split links"
    uid = tsim.nccl_unique_id()
    errs = []
    barrier = threading.Barrier(k)

    def rank(me):
        try:
            s = sims[me]
            s.nccl_init(uid, k, me)
            s.exchange()          # the exchange after ts_init, then unpack
            s.phase(2)
            barrier.wait()
            done = 0
            while done < steps:   # whole steps with the native exchanges
                n = min(chunk, steps - done)
                s.step(n)
                done += n
        except Exception as e:  # noqa: BLE001
            errs.append(f"rank {{me}}: {{e!r}}")
            barrier.abort()

    th = [threading.Thread(target=rank, args=(me,)) for me in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    assert not errs, errs
    o = oracle.Oracle.from_scenario(scn)
    oh = o.run_hashes(steps)
    if steps <= 4000:  # (the per-step history ring holds 4,096 steps)
        hs = [s.history(1, steps)["hash"] for s in sims]
        gh = [sum(int(h[i]) for h in hs) & (2**64 - 1) for i in range(steps)]
        bad = [1 + i for i in range(steps) if gh[i] != oh[i]]
        assert not bad, f"per-step hash differs at t={{bad[:5]}}"
    tots = [s.totals() for s in sims]
    assert sum(t["active"] + t["pending"] + t["arrived"] for t in tots) == scn.n_vehicles
    assert sum(t["arrived"] for t in tots) == int((o.vehicles()["status"] == oracle.ARRIVED).sum())
    vo = o.vehicles()
    vg = domains.merge_vehicles([s.vehicles() for s in sims])
    for key in ("status", "link", "lane", "cell", "v", "cursor", "t_arrive"):
        assert np.array_equal(vo[key], vg[key]), key
    tm = sims[0].last_exchange_timing()
    print("ok", k, steps, sum(s.totals()["vehicle_updates"] for s in sims), tm)
''')


@pytest.fixture(scope="module")
def fake_nccl(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("fake_nccl") / "libfake_nccl.so")
    subprocess.run(["g++", "-O1", "-std=c++17", "-shared", "-fPIC",
                    os.path.join(ROOT, "tests", "fake_nccl.cpp"), "-I/usr/local/cuda/include",
                    "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-o", out], check=True)
    return out


@pytest.mark.parametrize("scn,k,steps,chunk", [
    ('scenarios.config("1")', 2, 300, 37),
    ('scenarios.config("1")', 4, 200, 50),
    ('scenarios.portland(n_nodes=600, n_edges=800, n_veh=6000, side_km=8.0, n_zones=16, seed=4, '
     'steps=300)', 3, 300, 100),
    ('scenarios.config("1")', 2, 5000, 5000),  # one call longer than the statistics ring
])
@pytest.mark.parametrize("overlap", [True, False])
def test_native_step_with_partners(fake_nccl, scn, k, steps, chunk, overlap):
    """overlap: exchange #1 on the side stream beside the node and row
    kernels (the default for domains with row and general tiles); False:
    TSIM_NO_XOVERLAP, every phase in stream order"""
    if not overlap and steps > 1000:
        pytest.skip("the long run once")
    env = dict(os.environ, TSIM_NCCL_LIB=fake_nccl)
    if not overlap:
        env["TSIM_NO_XOVERLAP"] = "1"
    code = CHILD.format(root=ROOT, scn=scn, k=k, steps=steps, chunk=chunk)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.startswith("ok"), r.stdout
