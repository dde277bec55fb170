"""Text ingest throughput: paper_1508_06329_b200.textio (C++) vs the reference
chordalkit.textio (Python) on the same text, when the reference is importable.

    python tools/textio_bench.py [n] [p]      (default G(4096, 0.5): 4.2 M edges)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1508_06329_b200.generate import gen_dense_random  # noqa: E402
from paper_1508_06329_b200.textio import parse_graph_text, write_graph_text  # noqa: E402


def best(fn, reps=3):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        t.append(time.perf_counter() - t0)
    return min(t), r


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    g = gen_dense_random(n, p, 0)
    tw, text = best(lambda: write_graph_text(g))
    raw = text.encode()
    tp, g2 = best(lambda: parse_graph_text(raw))
    assert g2 == g
    out = {"graph": f"gen_dense_random({n}, {p}, 0)", "m": g.m, "bytes": len(raw),
           "ours": {"parse_s": tp, "parse_MBps": len(raw) / tp / 1e6, "write_s": tw, "threads": 1}}
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref):
        sys.path.insert(0, ref)
        from chordalkit.textio import parse_graph_text as rparse, write_graph_text as rwrite

        trp, rg = best(lambda: rparse(raw), reps=1)
        trw, rtext = best(lambda: rwrite(rg), reps=1)
        assert rtext == text and (rg._packed == g2._packed).all()
        out["reference"] = {"parse_s": trp, "parse_MBps": len(raw) / trp / 1e6, "write_s": trw,
                            "threads": 1, "kind": "chordalkit.textio (Python)"}
        out["speedup_parse"] = trp / tp
        out["speedup_write"] = trw / tw
    print(json.dumps(out))


if __name__ == "__main__":
    main()
