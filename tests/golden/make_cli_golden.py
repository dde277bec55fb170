"""Golden outputs of the reference CLI's `gen` subcommand (chordalkit/cli.py:123-128):
sha256 of the graph text for every class at a few sizes and seeds.

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_cli_golden.py
"""
import hashlib
import json
import os

from chordalkit.bench import make_graph
from chordalkit.textio import write_graph_text

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli_gen.json")


def main():
    cases = []
    for cls, sizes, params in (("clique", (1, 5, 40), (None,)), ("dense", (7, 60, 300), (None, 0.1)),
                               ("sparse", (41, 100, 400), (None,)), ("tree", (1, 2, 3, 90, 700), (None,)),
                               ("chordal", (2, 30, 500), (None, 3.0))):
        for n in sizes:
            for param in params:
                for seed in (0, 4):
                    text = write_graph_text(make_graph(cls, n, seed, param))
                    cases.append({"cls": cls, "n": n, "param": param, "seed": seed,
                                  "sha256": hashlib.sha256(text.encode()).hexdigest(), "bytes": len(text)})
    json.dump({"generator": "chordalkit.bench.make_graph + write_graph_text (reference)", "cases": cases},
              open(OUT, "w"), indent=0)
    print(len(cases), "cases ->", OUT)


if __name__ == "__main__":
    main()
