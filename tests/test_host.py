"""Host-side logic: types, validation, generators, arbitration (no GPU)."""

import numpy as np
import pytest

import paper_1508_06329_b200 as P
from conftest import load_json
from paper_1508_06329_b200.generate import gen_chordal_random, gen_dense_random, packed_sha256, remove_first_chord
from paper_1508_06329_b200.parallel import Arbitration


def c4():
    return P.Graph.from_edge_list(4, [(1, 2), (2, 3), (3, 4), (4, 1)])


def test_graph_construction_errors():
    with pytest.raises(P.InvalidVertex):
        P.Graph.from_edge_list(3, [(1, 4)])
    with pytest.raises(P.SelfLoop):
        P.Graph.from_edge_list(3, [(2, 2)])
    with pytest.raises(P.GraphTooLarge):
        P.Graph.from_edge_list(20001, [])
    g = P.Graph.from_edge_list(4, [(1, 2), (2, 1), (3, 4)])
    assert g.m == 2 and g.has_edge(2, 1) and not g.has_edge(1, 3)
    assert g.neighbors(1) == [2] and list(g.edges()) == [(1, 2), (3, 4)]


def test_vertex_ordering_validation():
    with pytest.raises(P.InvalidOrdering):
        P.VertexOrdering([1, 1, 2])
    with pytest.raises(P.InvalidOrdering):
        P.VertexOrdering([0, 1])
    o = P.VertexOrdering([3, 1, 2])
    assert o.pi(1) == 3 and o.pi_inv(3) == 1 and list(o) == [3, 1, 2]
    assert o.order0.tolist() == [2, 0, 1] and o.pos0.tolist() == [1, 2, 0]


def test_verdict_shape_enforced():
    with pytest.raises(ValueError):
        P.ChordalityVerdict(True)
    with pytest.raises(ValueError):
        P.ChordalityVerdict(False, peo=P.VertexOrdering([1]))


def test_bad_options_rejected_before_device():
    g = c4()
    with pytest.raises(ValueError):
        P.lexbfs_partition(g, method="bogus")
    with pytest.raises(ValueError):
        P.lexbfs_labels(g, method="bogus")
    with pytest.raises(ValueError):
        P.is_chordal(g, algo="mcs")
    with pytest.raises(ValueError):
        P.is_chordal(g, method="bogus")
    with pytest.raises(ValueError):
        P.parallel_lexbfs(g, Arbitration.fixed_priority(), backend="quantum")
    with pytest.raises(ValueError):
        P.parallel_lexbfs(g, Arbitration.fixed_priority(), backend="vector", audit=True)
    with pytest.raises(P.InvalidOrdering):
        P.is_peo(g, P.VertexOrdering([1, 2, 3]))
    with pytest.raises(ValueError):
        Arbitration.fixed_priority("sideways")


def test_lexlabel():
    with pytest.raises(ValueError):
        P.LexLabel((2, 2))
    assert P.LexLabel((3, 1)) < P.LexLabel((3, 2, 1)) < P.LexLabel((4,))


def test_arbitration_tie_rules():
    assert Arbitration.fixed_priority().choose("x", 0, 0, [3, 1, 2]) == 1
    assert Arbitration.fixed_priority("descending").choose("x", 0, 0, [3, 1, 2]) == 3
    a = Arbitration.seeded(5)
    assert a.choose("current", 0, 7, [1, 2, 3]) == a.choose("current", 0, 7, [3, 2, 1])
    assert Arbitration.seeded(1).tie_rule == 2 and Arbitration.fixed_priority().tie_rule == 0


def test_generators_match_reference_fingerprints():
    cfg = load_json("configs.json") if __import__("os").path.exists(
        __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "configs.json")) else {}
    if "4" not in cfg:
        pytest.skip("configs.json not generated")
    for rec in cfg["4"]["sample"][:16]:
        s = rec["seed"]
        g = gen_dense_random(512, 0.5, s) if s % 2 == 0 else gen_chordal_random(512, 8, s)
        assert packed_sha256(g._packed) == rec["packed_sha256"]
    if "1" in cfg:
        g = gen_chordal_random(1000, 8, 0)
        assert packed_sha256(g._packed) == cfg["1"]["chordal"]["packed_sha256"]
        h, e = remove_first_chord(g)
        assert list(e) == cfg["1"]["nonchordal"]["removed_edge"] == [1, 2]
        assert packed_sha256(h._packed) == cfg["1"]["nonchordal"]["packed_sha256"]


@pytest.mark.gpu
def test_scan_stats_formula_matches_reference_counts():
    """The reconstructed list-scan read count equals the reference's own count
    (the degrees, |LN| and parents come from the device; 600 more cases in
    test_gpu_left.py).  Expected values were produced by chordalkit's
    instrumented list method."""
    from paper_1508_06329_b200.peo import _list_scan_reads

    g = c4()
    o = P.VertexOrdering([1, 2, 4, 3])
    # reference: is_peo(c4, [1,2,4,3], stats=s, method="lists") -> ScanStats(reads=26, budget=32)
    assert _list_scan_reads(g, o, (2, 3, 1)) == 26
    k4 = P.Graph.from_edge_list(4, [(1, 2), (1, 3), (1, 4), (2, 3), (2, 4), (3, 4)])
    assert _list_scan_reads(k4, P.VertexOrdering([1, 2, 3, 4]), None) == 7 * 6
