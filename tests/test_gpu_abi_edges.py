"""C-ABI edge cases (GPU): padded host rows over dirty workspaces, empty
graphs in batches, understated edge counts.  Results are compared with the
oracle on the same inputs."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_1508_06329_b200 as P
from paper_1508_06329_b200 import _native, ops
from paper_1508_06329_b200.csr import CSRGraph, device_csr
from paper_1508_06329_b200.device import device_rows
from paper_1508_06329_b200.generate import chordal_random_edges, gen_chordal_random, remove_first_chord

pytestmark = pytest.mark.gpu


def _aligned_ws(nbytes, fill):
    ws = torch.full((nbytes + 256,), fill, dtype=torch.uint8, device="cuda")
    return ws, (ws.data_ptr() + 255) & ~255


def test_dense_host_ws_padded_rows_over_dirty_workspace():
    """row_bytes = 16 for n = 100 (ceil(n/8) = 13, device pitch 16): the pitch
    padding must be zeroed even though row_bytes == pitch; the workspace is
    pre-filled with 0xFF so stale bytes would show up as edges to vertices >= n."""
    cases = [(g, pitch) for g in (gen_chordal_random(100, 4, 1), remove_first_chord(gen_chordal_random(100, 4, 1))[0])
             for pitch in (16, 40)]  # 16: flat copy + device spread; 40 > device pitch: pitched copy
    for g, pitch in cases:
        n = g.n
        host = np.full((n, pitch), 0xFF, dtype=np.uint8)  # host pad bytes dirty too: never read
        host[:, :13] = g._packed
        wsb = int(_native.lib.chordal_dense_host_workspace_bytes(n, g.m))
        ws, wp = _aligned_ws(wsb, 0xFF)
        order = np.empty(n, dtype=np.int32)
        wit = np.empty(3, dtype=np.int32)
        flag = ctypes.c_int32(-1)
        rc = _native.lib.chordal_is_chordal_dense_host_ws(host.ctypes.data, n, pitch, g.m, 0, 0, order.ctypes.data,
                                                          wit.ctypes.data, ctypes.byref(flag), wp, wsb)
        assert rc == 0
        ok, o, w = oracle.is_chordal(np.ascontiguousarray(g._packed), n)
        assert bool(flag.value) == ok and order.tolist() == o.tolist()
        assert (None if ok else tuple(wit.tolist())) == w
        # the per-call form over pool memory
        order2 = np.empty(n, dtype=np.int32)
        wit2 = np.empty(3, dtype=np.int32)
        rc = _native.lib.chordal_is_chordal_dense_host(host.ctypes.data, n, pitch, 0, 0, order2.ctypes.data,
                                                       wit2.ctypes.data, ctypes.byref(flag))
        assert rc == 0 and order2.tolist() == o.tolist() and wit2.tolist() == wit.tolist()


def test_batch_host_padded_rows_dirty_host_padding():
    """Batch host entry with row_bytes = 16 > ceil(n/8) = 13 and 0xFF in the host
    pad bytes, over a dirty workspace: only the vertex bytes are copied."""
    gs = [gen_chordal_random(100, 4, s) if s % 3 else remove_first_chord(gen_chordal_random(100, 4, s))[0]
          for s in range(9)]
    for pitch in (13, 16, 40):  # 13 / 16: flat copy + device spread; 40 > device pitch: pitched copy
        host = np.full((9, 100, pitch), 0xFF, dtype=np.uint8)
        for b, g in enumerate(gs):
            host[b, :, :13] = g._packed
        clean = np.ascontiguousarray(host[:, :, :13])
        want_v, want_o, want_w = oracle.is_chordal_batch(clean, 100)
        wsb = int(_native.lib.chordal_batch_host_workspace_bytes(100, 4))
        ws, wp = _aligned_ws(wsb, 0xFF)
        orders = np.empty((9, 100), dtype=np.int32)
        wit = np.empty((9, 3), dtype=np.int32)
        assert _native.lib.chordal_is_chordal_batch_host_ws(host.ctypes.data, 9, 100, pitch, orders.ctypes.data,
                                                            wit.ctypes.data, 4, wp, wsb) == 0
        assert (orders == want_o).all() and (wit == want_w).all()
        assert _native.lib.chordal_is_chordal_batch_host(host.ctypes.data, 9, 100, pitch, orders.ctypes.data,
                                                         wit.ctypes.data, 4) == 0
        assert (orders == want_o).all() and (wit == want_w).all()


def test_empty_graphs_in_batches_are_chordal():
    wit = np.zeros((5, 3), dtype=np.int32)
    assert _native.lib.chordal_is_chordal_batch_host(None, 5, 0, 0, None, wit.ctypes.data, 0) == 0
    assert (wit == -1).all()
    adj = torch.zeros((5, 0, 16), dtype=torch.uint8, device="cuda")
    orders, w = ops.is_chordal_batch(adj, 0, 16)
    assert w.shape == (5, 3) and bool((w == -1).all())
    bv = P.is_chordal_batch([P.Graph.from_edge_list(0, [])] * 3)
    assert bv.chordal.all() and all(bv.verdict(b).chordal for b in range(3))


def test_understated_edge_count_is_rejected():
    """A caller m below the true edge count must not let the slot engine read
    past the buffers sized from it: EINVAL (ValueError) from both CSR routes."""
    n = 40000
    u, v = chordal_random_edges(n, 4, 1)
    g = P.Graph.from_edge_list(n, np.stack([u + 1, v + 1], 1), cap=n)
    c = CSRGraph.from_edges0(n, u, v)
    ip, ix = device_csr(c)
    with pytest.raises(ValueError):
        ops.lexbfs_csr(ip, ix, n, m=c.m // 2)
    order, pos, _ = ops.lexbfs_csr(ip, ix, n, m=c.m)  # the true m still works
    assert sorted(order.cpu().numpy().tolist()) == list(range(n))
    rows = device_rows(g)
    with pytest.raises(ValueError):
        ops.lexbfs(rows, m=c.m // 2)
