"""SPEC text formats of the network and plans files (SPEC.md "External
Interfaces"; load_network SPEC.md:46-54): pure host parsers of the C-ABI."""
import numpy as np
import pytest

from paper_cs_0105004_b200 import tsim as binding

NET = """# a 3-node chain and a signal
NODES
10 0 0
20 750 0      # 750 m east
30 1500 0.5
LINKS
100 10 20 750 2 5
200 20 30 75.0 1 5
300 20 10 750 2 5
TURNS
20 100 200 signal 25 35
20 300 200 yield
"""
PLANS = """1 0 3 100 200
7 12 0 300
# comment line
9 5 9 100
"""


def test_network_text_fields():
    n = binding.parse_network_text(NET)
    assert n["node_x_mm"].tolist() == [0, 750_000, 1_500_000]
    assert n["node_y_mm"].tolist() == [0, 0, 500]
    assert n["link_from"].tolist() == [0, 1, 1] and n["link_to"].tolist() == [1, 2, 0]
    assert n["link_len_mm"].tolist() == [750_000, 75_000, 750_000]
    assert n["link_lanes"].tolist() == [2, 1, 2] and n["link_class"].tolist() == [2, 1, 2]
    assert n["link_id"].tolist() == [100, 200, 300]
    # length 75.0 -> 10 cells (R1, round-half-up in mm)
    assert (n["link_len_mm"][1] + 3750) // 7500 == 10
    assert n["sig_node"].tolist() == [1] and n["sig_green"].tolist() == [35]
    assert n["sig_red"].tolist() == [25]


@pytest.mark.parametrize("bad,msg", [
    (NET.replace("200 20 30 75.0 1 5", "200 20 99 75.0 1 5"), "line 8: dangling node reference"),
    (NET.replace("75.0", "0"), "line 8: non-positive length"),
    (NET.replace("20 750 0", "20 750"), "line 4: NODES record"),
    ("LINKS\n1 1 2 10 1 5\n", "empty network"),
    ("NODES\n1 0 0\nLINKS\n1 1 2 10 1 5\n", "line 4: dangling node reference"),
    ("1 2 3\n", "line 1: record outside"),
    (NET.replace("100 10 20 750 2 5", "100 10 20 750 2 9"), "line 7: vmax"),
])
def test_network_text_errors(bad, msg):
    """parse error with line number, dangling node reference,
    non-positive length"""
    with pytest.raises(binding.TsError, match=msg):
        binding.parse_network_text(bad)


def test_plans_text():
    n = binding.parse_network_text(NET)
    off, route, dep, ent, vid = binding.parse_plans_text(PLANS, n["link_id"])
    assert off.tolist() == [0, 2, 3, 4]
    assert route.tolist() == [0, 1, 2, 0]
    assert dep.tolist() == [0, 12, 5] and ent.tolist() == [3, 0, 9] and vid.tolist() == [1, 7, 9]
    with pytest.raises(binding.TsError, match="line 1: unknown link id"):
        binding.parse_plans_text("1 0 0 555\n", n["link_id"])
    with pytest.raises(binding.TsError, match="line 2: negative departure"):
        binding.parse_plans_text("1 0 0 100\n2 -1 0 100\n", n["link_id"])


def test_round_trip_of_a_generated_grid():
    """SPEC invariant: a serialised network parses back to the same arrays"""
    import scenarios
    s = scenarios.config("1")
    lines = ["NODES"] + [f"{i} {x / 1000} {y / 1000}" for i, (x, y) in
                         enumerate(zip(s.node_x, s.node_y))]
    lines += ["LINKS"] + [f"{k} {a} {b} {ln / 1000} {la} {vm}" for k, (a, b, ln, la, vm) in
                          enumerate(zip(s.link_from, s.link_to, s.link_len_mm, s.link_lanes,
                                        s.link_vmax))]
    n = binding.parse_network_text("\n".join(lines))
    assert np.array_equal(n["node_x_mm"], s.node_x) and np.array_equal(n["node_y_mm"], s.node_y)
    assert np.array_equal(n["link_from"], s.link_from) and np.array_equal(n["link_to"], s.link_to)
    assert np.array_equal(n["link_len_mm"], s.link_len_mm)
