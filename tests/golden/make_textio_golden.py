"""Golden vectors for the text formats: run the REFERENCE (chordalkit.textio)
on a corpus of valid and broken inputs and freeze its results.

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_textio_golden.py

Writes tests/golden/textio.json: for every case the input (base64) and the
reference's outcome -- {"ok", n, m, sha256 of the packed rows} or
{exception class, message, line}.  Generated once in the build container (the
reference is not on the GPU box); tests/test_textio.py replays it against
paper_1508_06329_b200.textio.
"""
import base64
import hashlib
import json
import os
import random

import numpy as np
from chordalkit.errors import ChordalkitError
from chordalkit.graph import Graph
from chordalkit.textio import parse_graph_text, parse_ordering_text, write_graph_text

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "textio.json")


def sha(packed) -> str:
    return hashlib.sha256(np.ascontiguousarray(packed).tobytes()).hexdigest()


def outcome(fn):
    try:
        r = fn()
    except ChordalkitError as e:
        return {"err": type(e).__name__, "msg": str(e), "line": getattr(e, "line", None)}
    return r


def graph_case(raw: bytes, cap=None):
    def go():
        g = parse_graph_text(raw, cap=cap) if cap is not None else parse_graph_text(raw)
        return {"ok": True, "n": g.n, "m": g.m, "sha": sha(g._packed)}

    return {"kind": "graph", "data": base64.b64encode(raw).decode(), "cap": cap, "expect": outcome(go)}


def order_case(raw: bytes, n: int):
    def go():
        o = parse_ordering_text(raw, n)
        return {"ok": True, "order": list(o.order)}

    return {"kind": "ordering", "data": base64.b64encode(raw).decode(), "n": n, "expect": outcome(go)}


FIXED = [
    "", "e 1 2\n", "p 2\n", "p 2 x\n", "p -1 0\n", "p 2 1\ne 1 3\n", "p 2 1\ne 0 1\n", "p 3 1\ne 2 2\n",
    "p 3 2\ne 1 2\ne 2 1\n", "p 3 1\ne 1 2\ne 2 3\n", "p 3 2\ne 1 2\n", "p 3 1\nx 1 2\n", "p 3 1\ne 1 2 3\n",
    "p 3 1\ne 1 q\n", "c hi\np 2 1\ne 1 3\n", "c a remark\n\np 3 1\nc another\ne 3 1\n", "p 0 0\n", "p 1 0",
    "P 2 0\n", "p 2 0 0\n", "cats\np 2 1\ncomment\ne 1 2\n", "  p   3   1  \n\t e\t1\t3 \n",
    "p 3 1\r\ne 1 2\r\n", "p 3 1\re 1 2\r", "p 3 1\x0be 1 2\x0c", "p 3 1\x1ce 1 2\x1d", "p 3 1\x1ee 1 2\n",
    "p 3 1\x85e 1 2\n", "p 3 1 e 1 2 ", "p 3 1 e 1 2 ", "p 3 1\ne　1 2\n", "p 3 1\ne\x1f1\x1f2\n",
    "p 3 1\ne\xa01 2\n", "p 3 1\n　e 1 2 \n",
    "p +3 +1\ne +1 +002\n", "p 3 1\ne 0_1 2\n", "p 1_0 1\ne 1_0 9\n", "p 3 1\ne 1__2 3\n", "p 3 1\ne _1 2\n",
    "p 3 1\ne 1_ 2\n", "p 3 1\ne -1 2\n", "p 3 1\ne -0 2\n", "p 3 1\ne 4 -7\n", "p 3 1\ne 00003 1\n",
    "p 99999999999999999999999 0\n", "p 3 99999999999999999999999\ne 1 2\n",
    "p 3 1\ne 1 99999999999999999999999\n", "p 3 1\ne 1 1\n", "p 3 0\n\n\n", "p 3 2\ne 1 2\ne 1 2\ne 5 5\n",
    "p 3 1\ne 1 5\ne 1 2\n", "p 3 1\ne 3 1\nc trailing\n", "p 3 1\ne 1 2\np 3 1\n", "p 3 1 \ne 1 2\n",
    "\n\n  \n p 3 1\ne 1 2", "p 3 1\ne 1 2\n\n\nc\n", "p 3 -1\n", "p -0 0\n", "p 3 1\ne 1 2.0\n",
    "p 3 1\ne 1 0x2\n", "p 3 1\ne 1 2 \n", "p 4 4\ne 1 2\ne 1 4\ne 2 3\ne 3 4\n", "c \U0001F600 ok\np 1 0\n",
]


def main():
    rng = random.Random(1508)
    cases = [graph_case(t.encode("utf-8")) for t in FIXED]
    for raw in (b"p 2 1\ne 1 2\n\xff", b"\xc3\x28p 1 0\n", b"p 1 0\n\xe2\x82", b"p 2 1\ne 1 2\n\xed\xa0\x80\n"):
        cases.append(graph_case(raw))
    cases.append(graph_case(b"p 100 0\n", cap=99))
    cases.append(graph_case(b"p 99 0\n", cap=99))
    cases.append(graph_case(b"p 20001 0\n"))
    # round trips and mutations of random graphs
    for _ in range(160):
        n = rng.randint(0, 40)
        pairs = [(u, v) for u in range(1, n + 1) for v in range(u + 1, n + 1)]
        chosen = rng.sample(pairs, rng.randint(0, len(pairs))) if pairs else []
        g = Graph.from_edge_list(n, chosen)
        text = write_graph_text(g)
        lines = text.splitlines()
        mut = rng.randint(0, 9)
        if mut == 1 and len(lines) > 1:  # shuffled edges, mixed separators, comments, swapped ends
            body = lines[1:]
            rng.shuffle(body)
            seps = ["\n", "\r\n", "\r", "\x0b", "\x0c", "\x1c", " "]
            out = [lines[0]]
            for ln in body:
                if rng.random() < 0.2:
                    out.append("c " + "".join(rng.choice("abc xyz") for _ in range(5)))
                a, b_, c = ln.split()
                if rng.random() < 0.5:
                    b_, c = c, b_
                out.append(rng.choice([" ", "\t", "  ", "\xa0"]).join([a, b_, c]))
            text = "".join(x + rng.choice(seps) for x in out)
        elif mut == 2 and len(lines) > 1:  # duplicate one edge somewhere later
            i = rng.randint(1, len(lines) - 1)
            u, v = lines[i].split()[1:]
            lines.insert(rng.randint(i + 1, len(lines)), f"e {v} {u}")
            text = "\n".join(lines) + "\n"
        elif mut == 3 and len(lines) > 1:  # drop an edge
            del lines[rng.randint(1, len(lines) - 1)]
            text = "\n".join(lines) + "\n"
        elif mut == 4:  # extra edge, maybe invalid
            lines.insert(rng.randint(1, len(lines)), f"e {rng.randint(0, n + 1)} {rng.randint(0, n + 1)}")
            text = "\n".join(lines) + "\n"
        elif mut == 5 and len(lines) > 1:  # corrupt a field
            i = rng.randint(1, len(lines) - 1)
            f = lines[i].split()
            f[rng.randint(0, 2)] = rng.choice(["x", "1.5", "", "e", "--1", "+", "1_1", "0"])
            lines[i] = " ".join(f)
            text = "\n".join(lines) + "\n"
        elif mut == 6:  # header damage
            lines[0] = rng.choice([f"p {n}", f"p {n} {g.m + 1}", f"p {n + 1} {g.m}", f"q {n} {g.m}",
                                   f"p {n} {g.m} 1", f"p  {n}\t{g.m}  "])
            text = "\n".join(lines) + "\n"
        cases.append(graph_case(text.encode("utf-8")))
    for t, n in [("1 2 4 3\n", 4), (" 1\t2 4 3 ", 4), ("1 2 3\n", 4), ("1 2 4 4\n", 4), ("1 2 4 x\n", 4),
                 ("", 0), ("1", 1), ("1\n2\r\n3 4", 4), ("+1 02 3_0", 3), ("1 2 3 4 5", 4), ("0 1 2", 3),
                 ("3 2 1\n", 3), ("1 1.0", 2), ("2\u30001", 2)]:
        cases.append(order_case(t.encode("utf-8"), n))
    for _ in range(20):
        n = rng.randint(1, 50)
        perm = list(range(1, n + 1))
        rng.shuffle(perm)
        cases.append(order_case((" ".join(map(str, perm)) + "\n").encode(), n))
    with open(OUT, "w") as f:
        json.dump({"generator": "chordalkit.textio (reference) via tests/golden/make_textio_golden.py",
                   "cases": cases}, f, indent=0)
    print(len(cases), "cases ->", OUT)


if __name__ == "__main__":
    main()
