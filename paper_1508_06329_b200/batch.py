"""Batched chordality test over many small independent graphs.

The reference tests one graph per call (is_chordal, peo.py:177-202) and its
bench loops over graphs (bench.py:86-95); configuration 4 is 65,536 graphs of
512 vertices.  ``is_chordal_batch`` runs them all in one launch
(csrc/batch.cu: one warp-resident search per graph, adjacency staged in SMEM)
and returns per-graph verdicts identical to ``is_chordal`` on each graph.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native, ops
from .graph import VertexOrdering, device_stride, row_width
from .peo import ChordalityVerdict, WitnessTriple


@dataclass
class BatchVerdicts:
    """Per-graph results: ``chordal[b]``, 0-based ``orders0[b]`` and ``witness0[b]``."""

    chordal: np.ndarray
    orders0: np.ndarray
    witness0: np.ndarray

    def __len__(self) -> int:
        return int(self.chordal.size)

    def verdict(self, b: int) -> ChordalityVerdict:
        if self.chordal[b]:
            return ChordalityVerdict(True, peo=VertexOrdering._trusted(self.orders0[b]))
        v, p, z = (int(x) + 1 for x in self.witness0[b])
        return ChordalityVerdict(False, witness=WitnessTriple(v, p, z))


def stack_graphs(graphs, device=None):
    """Pack same-size graphs into one device tensor uint8[B, n, stride]."""
    torch = _native.require_cuda()
    graphs = list(graphs)
    if not graphs:
        raise ValueError("empty batch")
    n = int(graphs[0].n)
    if any(int(g.n) != n for g in graphs):
        raise ValueError("all graphs of a batch must have the same vertex count")
    stride, w = device_stride(n), row_width(n)
    host = np.zeros((len(graphs), n, stride), dtype=np.uint8)
    for b, g in enumerate(graphs):
        host[b, :, :w] = g._packed
    return torch.from_numpy(host).to(device or "cuda"), n, stride


def is_chordal_batch_device(adj, n: int, stride: int, stream=None):
    """Device form: adj uint8[B, n, stride] -> (orders int32[B,n], witness int32[B,3]) on device."""
    if n > _native.BATCH_MAX_N:
        from .errors import GraphTooLarge

        raise GraphTooLarge(f"batched kernel handles n <= {_native.BATCH_MAX_N}, got {n}")
    return ops.is_chordal_batch(adj, n, stride, stream)


def is_chordal_batch(graphs) -> BatchVerdicts:
    """is_chordal (LOWEST_INDEX) for every graph of the batch, in one launch."""
    adj, n, stride = stack_graphs(graphs)
    orders, wit = is_chordal_batch_device(adj, n, stride)
    w = wit.cpu().numpy()
    return BatchVerdicts(chordal=w[:, 0] < 0, orders0=orders.cpu().numpy(), witness0=w)
