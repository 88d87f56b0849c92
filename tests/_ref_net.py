"""Independent one-step reference of the TRANSIMS CA step on small road
networks (tests only) -- the brute-force pin of the oracle's lane change
(R4-R7), intersection resolution (R8-R10) and move (R12, R15) rules.

Written from PAPER.md §3 (:320-362) and the readings of DESIGN.md §3 in a
representation different from the oracle's lane-cell grid: a vehicle LIST
(dict vid -> record), lanes searched by scanning the list.  It shares no
code with ``oracle/`` (only the pinned numpy Philox of ``tests/_ref.py``).

Network: dict with int arrays node_x, node_y (mm), link_from, link_to,
link_len_mm, link_lanes, link_vmax, link_class; routes: list of link lists.
Vehicle record: [link, lane, cell, v, cursor].
"""
import numpy as np

from tests._ref import brake_np

G_RANGE = 5  # interaction range / gap cap, PAPER.md:390-395 (R2)


class Net:
    def __init__(self, node_x, node_y, link_from, link_to, link_len_mm, link_lanes, link_vmax,
                 link_class, routes, D=10, G=5):
        self.nx = [int(a) for a in node_x]
        self.ny = [int(a) for a in node_y]
        self.frm = [int(a) for a in link_from]
        self.to = [int(a) for a in link_to]
        # R1: round half up in integer mm, at least one cell
        self.n = [max(1, (int(m) + 3750) // 7500) for m in link_len_mm]
        self.L = [int(a) for a in link_lanes]
        self.V = [int(a) for a in link_vmax]
        self.cls = [int(a) for a in link_class]
        self.routes = [list(map(int, r)) for r in routes]
        self.D, self.G = D, G
        self.incoming = {}
        for k, b in enumerate(self.to):
            self.incoming.setdefault(b, []).append(k)

    def turn(self, k, k2):
        """R7: 'T', 'L' or 'R' from the integer direction vectors"""
        ax, ay = self.nx[self.to[k]] - self.nx[self.frm[k]], self.ny[self.to[k]] - self.ny[self.frm[k]]
        bx, by = (self.nx[self.to[k2]] - self.nx[self.frm[k2]],
                  self.ny[self.to[k2]] - self.ny[self.frm[k2]])
        cross, dot = ax * by - ay * bx, ax * bx + ay * by
        if dot > 0 and abs(cross) <= dot:
            return "T"
        return "R" if cross < 0 else "L"  # a U-turn counts as left

    def lanes_ok(self, f, rec):
        """R7: set of lanes the vehicle may use on its current link"""
        k, cur = rec[0], rec[4]
        r = self.routes[f]
        L = self.L[k]
        if cur == len(r) - 1:
            return set(range(L))
        tt = self.turn(k, r[cur + 1])
        return {"T": set(range(L)), "R": {0}, "L": {L - 1}}[tt]

    def entry_lane(self, k, l, k2):
        """R8: T keeps the lane (clamped), R enters the curb lane, L the median"""
        tt = self.turn(k, k2)
        if tt == "T":
            return min(l, self.L[k2] - 1)
        return 0 if tt == "R" else self.L[k2] - 1


def _occupants(state):
    """(link, lane) -> {cell: vid}"""
    occ = {}
    for f, rec in state.items():
        occ.setdefault((rec[0], rec[1]), {})[rec[2]] = f
    return occ


def _free_ahead(occ, net, k, l, x):
    """consecutive empty cells after x in (k, l), stopping at the link end,
    at most 5 (R2)"""
    cells = occ.get((k, l), {})
    c = 0
    for j in range(1, G_RANGE + 1):
        if x + j > net.n[k] - 1 or (x + j) in cells:
            break
        c += 1
    return c


def _free_behind(occ, k, l, x):
    """consecutive empty cells before x, positions before the link start
    counting as empty, at most 5 (R2)"""
    cells = occ.get((k, l), {})
    c = 0
    for j in range(1, G_RANGE + 1):
        if x - j >= 0 and (x - j) in cells:
            break
        c += 1
    return c


def lane_change(net, state, t):
    """§LC on S0 = S(t) (R4-R7): returns S1"""
    occ = _occupants(state)
    d = 1 if t % 2 == 0 else -1
    new = {f: list(r) for f, r in state.items()}
    for f, rec in state.items():
        k, l, x, v, _ = rec
        l2 = l + d
        if l2 < 0 or l2 >= net.L[k] or x in occ.get((k, l2), {}):
            continue
        ok = net.lanes_ok(f, rec)
        Vk = net.V[k]
        if l not in ok:  # must reach its turn lane: only towards it
            want = min(ok) if min(ok) < l else max(ok)
            if (want - l) * d <= 0:
                continue
            dist = net.n[k] - 1 - x
            need_f, need_b = min(v + 1, Vk), Vk
            if dist < net.D:  # R6: accepted gaps shrink linearly, floored
                need_f, need_b = need_f * dist // net.D, need_b * dist // net.D
            if _free_ahead(occ, net, k, l2, x) >= need_f and _free_behind(occ, k, l2, x) >= need_b:
                new[f][1] = l2
        elif l2 in ok:  # R5: the other lane is faster and the gap behind suffices
            g = _free_ahead(occ, net, k, l, x)
            if g < v + 1 and _free_ahead(occ, net, k, l2, x) > g and _free_behind(occ, k, l2, x) >= Vk:
                new[f][1] = l2
    return new


def node_grants(net, state, t=0, signals=None):
    """§Node on S1 (R8-R10): {(k, l): entry space} for the
    front vehicle of every winning approach lane"""
    occ = _occupants(state)
    ext = {}
    for node, ins in net.incoming.items():
        top = max(net.cls[k] for k in ins)
        cands = []
        for k in ins:
            for l in range(net.L[k]):
                cells = occ.get((k, l), {})
                xs = [x for x in cells if x >= net.n[k] - G_RANGE]
                if not xs:
                    continue
                x = max(xs)
                f = cells[x]
                rec = state[f]
                r = net.routes[f]
                if rec[4] == len(r) - 1:
                    continue  # final link: exits, never crosses (R12)
                if not (net.n[k] - 1 - x < min(rec[3] + 1, net.V[k])):
                    continue
                k2 = r[rec[4] + 1]
                cands.append((0 if net.cls[k] == top else 1, k, l, k2, net.entry_lane(k, l, k2)))
        major_free = all(
            (x < net.n[j] - net.G)
            for j in ins if net.cls[j] == top
            for l in range(net.L[j]) for x in occ.get((j, l), {}))
        taken = set()
        for rank, k, l, k2, l2 in sorted(cands):
            if rank == 1 and not major_free:
                continue
            if (k2, l2) in taken:
                continue
            taken.add((k2, l2))
            cells = occ.get((k2, l2), {})
            e = 0
            while e < min(G_RANGE, net.n[k2]) and e not in cells:
                e += 1
            ext[(k, l)] = e
    return ext


def move(net, state, ext, t, seed, p):
    """§Move S1 -> S2 (R3, R12, R15): returns (S2, arrived
    vids)"""
    occ = _occupants(state)
    vids = np.array(sorted(state), dtype=np.int64)
    brake = dict(zip(vids.tolist(), brake_np(t, vids, seed, p).tolist())) if vids.size else {}
    new, arrived = {}, []
    for f, rec in state.items():
        k, l, x, v, cur = rec
        r = net.routes[f]
        ahead = [y for y in occ.get((k, l), {}) if y > x]
        if ahead:
            g = min(G_RANGE, min(ahead) - x - 1)
        elif cur == len(r) - 1:
            g = G_RANGE
        else:
            g = min(G_RANGE, net.n[k] - 1 - x + ext.get((k, l), 0))
        v2 = min(min(v + 1, net.V[k]), g)
        v3 = v2 - 1 if (v2 > 0 and brake[f]) else v2
        y = x + v3
        if y <= net.n[k] - 1:
            new[f] = [k, l, y, v3, cur]
        elif cur == len(r) - 1:
            arrived.append(f)
        else:
            k2 = r[cur + 1]
            new[f] = [k2, net.entry_lane(k, l, k2), y - net.n[k], v3, cur + 1]
    return new, arrived


def step(net, state, t, seed, p):
    """one whole step t -> t+1 without injection"""
    s1 = lane_change(net, state, t)
    ext = node_grants(net, s1, t)
    return move(net, s1, ext, t, seed, p)
