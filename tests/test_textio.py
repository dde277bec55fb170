"""Text formats (textio.py): the C++ parser / writer against golden vectors
frozen from the reference (tests/golden/make_textio_golden.py) and the
reference's own test_textio.py cases.  Host code only: runs without a GPU."""

import base64
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1508_06329_b200 as P
from paper_1508_06329_b200.errors import GraphTooLarge, InvalidOrdering, ParseError
from paper_1508_06329_b200.textio import (
    parse_graph_text,
    parse_ordering_text,
    write_graph_text,
    write_ordering_text,
)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "textio.json")
CASES = json.load(open(GOLDEN))["cases"]


def _sha(packed) -> str:
    return hashlib.sha256(np.ascontiguousarray(packed).tobytes()).hexdigest()


def _run(case):
    raw = base64.b64decode(case["data"])
    try:
        if case["kind"] == "graph":
            g = parse_graph_text(raw, cap=case["cap"]) if case["cap"] is not None else parse_graph_text(raw)
            return {"ok": True, "n": g.n, "m": g.m, "sha": _sha(g._packed)}
        o = parse_ordering_text(raw, case["n"])
        return {"ok": True, "order": list(o.order)}
    except (ParseError, GraphTooLarge, InvalidOrdering) as e:
        return {"err": type(e).__name__, "msg": str(e), "line": getattr(e, "line", None)}


@pytest.mark.parametrize("i", range(len(CASES)))
def test_golden_case(i):
    """Same Graph (packed rows) or the same exception, message and line."""
    assert _run(CASES[i]) == CASES[i]["expect"]


def test_str_and_bytes_inputs_agree():
    for case in CASES:
        if case["kind"] != "graph" or "ok" not in case["expect"]:
            continue
        raw = base64.b64decode(case["data"])
        a = parse_graph_text(raw, cap=case["cap"]) if case["cap"] is not None else parse_graph_text(raw)
        b = parse_graph_text(raw.decode("utf-8"), cap=case["cap"]) if case["cap"] is not None else \
            parse_graph_text(raw.decode("utf-8"))
        assert a == b


# ---- the reference's own tests (pkg/tests/test_textio.py), restated ---------

def _c4():
    return P.Graph.from_edge_list(4, [(1, 2), (2, 3), (3, 4), (4, 1)])


def test_write_graph_golden():
    assert write_graph_text(_c4()) == "p 4 4\ne 1 2\ne 1 4\ne 2 3\ne 3 4\n"


def test_parse_graph_roundtrip_c4():
    assert parse_graph_text(write_graph_text(_c4())) == _c4()


def test_parse_accepts_comments_and_blank_lines():
    g = parse_graph_text("c a remark\n\np 3 1\nc another\ne 3 1\n")
    assert g.n == 3 and g.m == 1 and g.has_edge(1, 3)


def test_parse_error_reports_line_number():
    with pytest.raises(ParseError) as err:
        parse_graph_text("c hi\np 2 1\ne 1 3\n")
    assert err.value.line == 3 and "line 3" in str(err.value)


def test_parse_respects_cap():
    with pytest.raises(GraphTooLarge):
        parse_graph_text("p 100 0\n", cap=99)


def test_ordering_roundtrip_and_errors():
    o = P.VertexOrdering([1, 2, 4, 3])
    assert write_ordering_text(o) == "1 2 4 3\n"
    assert parse_ordering_text("1 2 4 3\n", 4) == o
    assert parse_ordering_text(b" 1\t2 4 3 ", 4) == o
    with pytest.raises(InvalidOrdering):
        parse_ordering_text("1 2 3\n", 4)
    with pytest.raises(InvalidOrdering):
        parse_ordering_text("1 2 4 4\n", 4)
    with pytest.raises(ParseError):
        parse_ordering_text("1 2 4 x\n", 4)


def test_graph_text_roundtrip_random():
    rng = np.random.default_rng(7)
    for n in list(range(0, 15)) + [63, 64, 65, 300]:
        for _ in range(3):
            pairs = [(u, v) for u in range(1, n + 1) for v in range(u + 1, n + 1)]
            k = int(rng.integers(0, len(pairs) + 1)) if pairs else 0
            idx = rng.choice(len(pairs), size=k, replace=False) if k else []
            g = P.Graph.from_edge_list(n, [pairs[i] for i in idx])
            t = write_graph_text(g)
            assert parse_graph_text(t) == g
