"""Synthetic inputs of the benchmark configurations, bit-identical to the reference.

These build the *inputs* of the hot path (they are not on it).  Each function
replays the reference generator's draws from the same named Philox4x64-10
stream (rng.py:18-21: key = mix64(seed, crc32(label))), so the same seed gives
the same graph as ``chordalkit.generate`` with the same numpy; the equality is
pinned by sha256 fixtures in tests/golden/ produced from the reference itself.

``gen_dense_random_device`` draws the identical dense graphs directly in HBM
(csrc/gen.cu) -- the batched configuration's 65,536 inputs are born on the GPU.
"""

from __future__ import annotations

import hashlib
import zlib

import numpy as np

from .errors import InvalidProbability, InvalidSize
from .graph import Graph, _check_size, row_width

_MASK64 = (1 << 64) - 1


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def stream_key(seed: int, label: str) -> int:
    """mix64(seed, crc32(label)) -- the Philox key of rng.stream (rng.py:18-21)."""
    h = _splitmix64(int(seed) & _MASK64)
    return _splitmix64(h ^ zlib.crc32(label.encode("ascii")))


def stream(seed: int, label: str = "") -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=stream_key(seed, label)))


def gen_clique(n: int, *, cap: int | None = None) -> Graph:
    """Complete graph K_n (generate.py:18-29)."""
    if n < 1:
        raise InvalidSize("clique needs at least one vertex")
    _check_size(n, cap)
    bits = np.ones((n, n), dtype=bool)
    np.fill_diagonal(bits, False)
    return Graph._from_packed(n, np.packbits(bits, axis=1, bitorder="little"))


def gen_dense_random(n: int, p: float, seed: int, *, cap: int | None = None) -> Graph:
    """G(n, p) with the reference's draw layout (generate.py:32-56), on the host."""
    if not 0.0 < p <= 1.0:
        raise InvalidProbability(f"edge probability must be in (0, 1], got {p}")
    _check_size(n, cap)
    w = row_width(n)
    packed = np.zeros((n, w), dtype=np.uint8)
    if n <= 1:
        return Graph._from_packed(n, packed)
    gen = stream(seed, "dense-random")
    col = np.arange(n, dtype=np.int64)
    for r0 in range(0, n, 1024):  # 1024-row blocks, one draw per cell, row-major
        r1 = min(r0 + 1024, n)
        upper = (gen.random((r1 - r0, n)) < p) & (col[None, :] > np.arange(r0, r1)[:, None])
        packed[r0:r1] |= np.packbits(upper, axis=1, bitorder="little")[:, :w]
        lower = np.packbits(upper.T, axis=1, bitorder="little")
        packed[:, r0 >> 3 : (r0 >> 3) + lower.shape[1]] |= lower
    return Graph._from_packed(n, packed)


def gen_dense_random_device(n: int, p: float, seeds, *, stride: int | None = None, out=None):
    """The same graphs drawn on the GPU: uint8[B, n, stride] for seeds seed0 + b*step.

    ``seeds`` is ``range``-like (start, step) or an int (one graph).
    """
    from . import _native, ops
    from .graph import device_stride

    torch = _native.require_cuda()
    if isinstance(seeds, int):
        seeds = range(seeds, seeds + 1)
    B = len(seeds)
    s = stride or device_stride(n)
    if out is None:
        out = torch.empty((B, n, s), dtype=torch.uint8, device="cuda")
    step = seeds.step if B > 1 else 1
    return ops.gen_dense_random(out, n, s, p, seeds.start, step)


def gen_chordal_random_device(n: int, k: int, seeds, *, stride: int | None = None, out=None):
    """gen_chordal_random drawn on the GPU (csrc/gen.cu): uint8[B, n, stride]."""
    from . import _native, ops
    from .graph import device_stride

    torch = _native.require_cuda()
    if isinstance(seeds, int):
        seeds = range(seeds, seeds + 1)
    B = len(seeds)
    s = stride or device_stride(n)
    if out is None:
        out = torch.empty((B, n, s), dtype=torch.uint8, device="cuda")
    step = seeds.step if B > 1 else 1
    return ops.gen_chordal_random(out, n, s, k, seeds.start, step)


def gen_chordal_random_csr_device(n: int, k: int, seed: int):
    """gen_chordal_random(n, k, seed) as device CSR (indptr int64[n+1], indices int32[2m]).

    The draws run on the GPU (one thread, csrc/gen.cu, bit-exact); the edge
    list is symmetrised and sorted with torch (input preparation, not the hot
    path).  This is how the N = 10^6 configuration is built without the 125 GB
    dense matrix the reference generator would allocate.
    """
    from . import _native
    from ._native import check, lib, ptr, stream_ptr

    torch = _native.require_cuda()
    cap = n * (k + 1) + 1
    u = torch.empty(cap, dtype=torch.int32, device="cuda")
    v = torch.empty(cap, dtype=torch.int32, device="cuda")
    m_t = torch.zeros(1, dtype=torch.int64, device="cuda")
    nbytes = int(lib.chordal_gen_chordal_random_scratch_bytes(1, n, k))
    scratch = torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")
    check(lib.chordal_gen_chordal_random_edges(n, k, seed, ptr(u), ptr(v), ptr(m_t), ptr(scratch), nbytes,
                                               stream_ptr()), "chordal_gen_chordal_random_edges")
    m = int(m_t.item())
    a = torch.cat([u[:m], v[:m]]).to(torch.int64)
    b = torch.cat([v[:m], u[:m]]).to(torch.int64)
    key = torch.unique(a * n + b)
    rows = key // n
    indptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    indptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    return indptr, (key % n).to(torch.int32)


def chordal_random_edges(n: int, k: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """0-based edge endpoints of gen_chordal_random (generate.py:118-155).

    Vertex i attaches to a random subset of a random earlier vertex j plus the
    clique j attached to; the draw sequence (integers(-1,2), integers(0,i),
    choice(size, want, replace=False)) is replayed call for call.
    """
    if n < 1:
        raise InvalidSize("need at least one vertex")
    if not 0 <= k < n:
        raise InvalidSize(f"attachment size must satisfy 0 <= k < n, got {k}")
    if k == 0 or n == 1:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64)
    gen = stream(seed, "chordal-random")
    attached: list[np.ndarray] = [np.empty(0, dtype=np.int64)]
    heads, tails = [], []
    for i in range(1, n):
        if k >= i:
            chosen = np.arange(i, dtype=np.int64)
        else:
            want = int(np.clip(k + gen.integers(-1, 2), 1, i))
            j = int(gen.integers(0, i))
            pool = np.append(attached[j], j)
            chosen = pool if want >= pool.size else pool[gen.choice(pool.size, size=want, replace=False)]
        attached.append(chosen)
        heads.append(np.full(chosen.size, i, dtype=np.int64))
        tails.append(chosen)
    return np.concatenate(heads), np.concatenate(tails)


def gen_chordal_random(n: int, k: int, seed: int, *, cap: int | None = None) -> Graph:
    """Random chordal graph by clique attachment (generate.py:118-155)."""
    if n < 1:
        raise InvalidSize("need at least one vertex")
    if not 0 <= k < n:
        raise InvalidSize(f"attachment size must satisfy 0 <= k < n, got {k}")
    _check_size(n, cap)
    u, v = chordal_random_edges(n, k, seed)
    if u.size == 0:
        return Graph(n, np.zeros((n, row_width(n)), dtype=np.uint8), 0)
    return Graph._from_numpy_edges(n, u + 1, v + 1)


def gen_sparse_random(n: int, seed: int, *, cap: int | None = None) -> Graph:
    """20n distinct uniform edges (generate.py:59-81): batches of endpoint pairs
    drawn from the "sparse-random" stream, self-loops dropped, first occurrences
    kept in draw order until 20n are collected."""
    if n < 41:
        raise InvalidSize(f"need n >= 41 so that 20n edges fit, got {n}")
    _check_size(n, cap)
    gen = stream(seed, "sparse-random")
    need = 20 * n
    taken: dict[int, None] = {}
    while len(taken) < need:
        batch = max(4096, 2 * (need - len(taken)))
        a = gen.integers(0, n, size=batch, dtype=np.int64)
        b = gen.integers(0, n, size=batch, dtype=np.int64)
        keep = a != b
        codes = np.minimum(a[keep], b[keep]) * n + np.maximum(a[keep], b[keep])
        for c in codes.tolist():
            if c not in taken:
                taken[c] = None
                if len(taken) == need:
                    break
    codes = np.fromiter(taken.keys(), dtype=np.int64, count=need)
    return Graph._from_numpy_edges(n, codes // n + 1, codes % n + 1)


def gen_tree(n: int, seed: int, *, cap: int | None = None) -> Graph:
    """Uniform labelled tree (generate.py:84-115): the Pruefer code of n-2 draws
    from the "tree" stream, decoded (the tree of a code is unique)."""
    import heapq

    if n < 1:
        raise InvalidSize("tree needs at least one vertex")
    _check_size(n, cap)
    if n == 1:
        return Graph.from_edge_list(1, [])
    if n == 2:
        return Graph.from_edge_list(2, [(1, 2)])
    code = stream(seed, "tree").integers(0, n, size=n - 2, dtype=np.int64)
    deg = np.ones(n, dtype=np.int64)
    np.add.at(deg, code, 1)
    leaves = [v for v in range(n) if deg[v] == 1]
    heapq.heapify(leaves)
    u = np.empty(n - 1, dtype=np.int64)
    v = np.empty(n - 1, dtype=np.int64)
    for i, c in enumerate(code.tolist()):
        leaf = heapq.heappop(leaves)
        u[i], v[i] = leaf, c
        deg[c] -= 1
        if deg[c] == 1:
            heapq.heappush(leaves, c)
    u[n - 2], v[n - 2] = heapq.heappop(leaves), heapq.heappop(leaves)
    return Graph._from_numpy_edges(n, u + 1, v + 1)


def remove_first_chord(g: Graph) -> tuple[Graph, tuple[int, int] | None]:
    """Drop the first edge u<v (edges() order) whose endpoints share two
    non-adjacent common neighbours; the copy then has a chordless 4-cycle.

    The rule that turns the chordal configuration graphs into their
    non-chordal twins.  Returns (graph, removed 1-based edge).
    """
    n = g.n
    packed = np.asarray(g._packed)

    def row(i):
        return np.unpackbits(packed[i], bitorder="little", count=n).astype(bool)

    for u in range(n):
        ru = row(u)
        for v in np.flatnonzero(ru[u + 1 :]) + u + 1:
            common = np.flatnonzero(ru & row(v))
            if common.size < 2:
                continue
            sub = np.unpackbits(packed[common], axis=1, bitorder="little", count=n)[:, common].astype(bool)
            if (~sub).sum() > common.size:  # some off-diagonal non-edge
                packed = np.array(g._packed, copy=True)
                packed[u, v >> 3] &= np.uint8(0xFF ^ (1 << (v & 7)))
                packed[v, u >> 3] &= np.uint8(0xFF ^ (1 << (u & 7)))
                return Graph(n, packed, g.m - 1), (u + 1, int(v) + 1)
    return g, None


def packed_sha256(packed: np.ndarray) -> str:
    """Fingerprint of the reference layout (n, ceil(n/8)) of a graph."""
    return hashlib.sha256(np.ascontiguousarray(packed, dtype=np.uint8).tobytes()).hexdigest()
