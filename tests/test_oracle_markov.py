"""The stochastic NaSch step against its exact Markov chain (SURVEY §8(c)
pin 5): on a tiny single-lane ring the stationary mean flow is computed by
enumerating every state (positions and velocities of the vehicles) and the
exact transition probabilities of the parallel update with braking
probability p (R15: accelerate, gap clamp, brake with
probability p if v > 0, move); a long oracle run (Philox draws, R3) must
reproduce it.  This pins the random-slowdown path for V > 1, which the
V = 1 closed form does not reach."""
import itertools

import numpy as np
import pytest

import oracle
import scenarios


def exact_stationary_flow(L, N, V, p):
    states = []
    for pos in itertools.combinations(range(L), N):
        for vel in itertools.product(range(V + 1), repeat=N):
            states.append((pos, vel))
    index = {s: i for i, s in enumerate(states)}
    P = np.zeros((len(states), len(states)))
    for i, (pos, vel) in enumerate(states):
        # deterministic part: v2 = min(v + 1, V, gap to the next vehicle)
        v2 = []
        for a in range(N):
            gap = (pos[(a + 1) % N] - pos[a] - 1) % L if N > 1 else L - 1
            v2.append(min(vel[a] + 1, V, gap))
        movers = [a for a in range(N) if v2[a] > 0]
        for brakes in itertools.product((0, 1), repeat=len(movers)):
            prob = 1.0
            v3 = list(v2)
            for a, b in zip(movers, brakes):
                prob *= p if b else 1.0 - p
                v3[a] -= b
            npos = [(pos[a] + v3[a]) % L for a in range(N)]
            order = sorted(range(N), key=lambda a: npos[a])
            key = (tuple(npos[a] for a in order), tuple(v3[a] for a in order))
            P[i, index[key]] += prob
    w, vec = np.linalg.eig(P.T)
    pi = np.real(vec[:, np.argmin(np.abs(w - 1.0))])
    pi = pi / pi.sum()
    # flow q = E[sum of velocities] / L in the stationary state
    return float(sum(pi[i] * sum(vel) for i, (_, vel) in enumerate(states))) / L


@pytest.mark.parametrize("L,N,V,p", [(10, 2, 5, 0.5), (10, 3, 2, 0.2), (11, 2, 3, 0.3)])
def test_stationary_flow_matches_markov_chain(L, N, V, p):
    q_exact = exact_stationary_flow(L, N, V, p)
    s = scenarios.ring(n_cells=L, lanes=1, n_veh=N, seed=11, vmax=V, v_init=0)
    s.p_slow = p
    o = oracle.Oracle.from_scenario(s)
    o.step(200)
    T = 60_000
    tot = 0
    for _ in range(T):
        o.step(1)
        tot += o.counters()["sum_v"]
    q_sim = tot / (T * L)
    # measured |q_sim - q_exact| <= 0.0011; a brake probability off by 0.05
    # moves q_exact by 0.012-0.037
    assert abs(q_sim - q_exact) < 0.004, (q_sim, q_exact)
