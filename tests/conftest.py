import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (large configurations)")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_npz(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


class SmallCorpus:
    """Decoded random_small.npz: one record per graph."""

    def __init__(self):
        z = load_npz("random_small.npz")
        self.z = z
        ns = z["n"].astype(int)
        self.ns = ns
        self.off = z["packed_off"]
        self.voff = np.concatenate([[0], np.cumsum(ns)])

    def __len__(self):
        return len(self.ns)

    def packed(self, i):
        n = int(self.ns[i])
        w = (n + 7) // 8
        return self.z["packed"][self.off[i]:self.off[i + 1]].reshape(n, w)

    def vec(self, key, i):
        return self.z[key][self.voff[i]:self.voff[i + 1]]


@pytest.fixture(scope="session")
def small_corpus():
    return SmallCorpus()


def exhaustive_graph_packed(n, mask):
    import itertools

    pairs = list(itertools.combinations(range(n), 2))
    rows = np.zeros((n, n), dtype=bool)
    for i, (u, v) in enumerate(pairs):
        if mask >> i & 1:
            rows[u, v] = rows[v, u] = True
    return np.packbits(rows, axis=1, bitorder="little") if n else np.zeros((0, 0), np.uint8)


def named_packed(rec):
    n = rec["n"]
    rows = np.zeros((n, n), dtype=bool)
    for u, v in rec["edges"]:
        rows[u - 1, v - 1] = rows[v - 1, u - 1] = True
    return np.packbits(rows, axis=1, bitorder="little")


class LeftCorpus:
    """Decoded left_scan.npz (tests/golden/make_left_golden.py): one record per
    (graph, ordering) case with the reference's left_neighborhoods parents,
    |LN(v)|, is_peo verdict / witness and ScanStats reads / budget."""

    def __init__(self):
        z = load_npz("left_scan.npz")
        self.z = z
        self.ns = z["n"].astype(int)
        self.off = z["packed_off"]
        self.voff = np.concatenate([[0], np.cumsum(self.ns)])

    def __len__(self):
        return len(self.ns)

    def packed(self, i):
        n = int(self.ns[i])
        return self.z["packed"][self.off[i]:self.off[i + 1]].reshape(n, (n + 7) // 8)

    def vec(self, key, i):
        return self.z[key][self.voff[i]:self.voff[i + 1]]


@pytest.fixture(scope="session")
def left_corpus():
    return LeftCorpus()
