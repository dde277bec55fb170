"""CPU parity oracle for the chordality-test hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs (``cpu_baseline`` and ``--impl reference``) may import this module.  The
product package ``paper_1508_06329_b200`` never imports it and has no CPU
fallback.

The C restatement lives in ``chordal_oracle.c`` (each function cites the
reference file:line it restates); this module loads the compiled
``_build/liboracle.so`` with ctypes and exposes numpy-level helpers, all
0-based.  Parity pinning: ``tests/test_oracle_golden.py`` checks every helper
against fixtures produced by running the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile the oracle with the committed Makefile (idempotent)."""
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else os.environ.get("CC", "gcc")
    subprocess.run(["make", "-s", "-C", _HERE, f"CC={cc}"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "chordal_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_lexbfs_partition.argtypes = [P, i64, i64, P, P]
        L.oracle_lexbfs_partition_csr.argtypes = [P, P, i64, P]
        L.oracle_lexbfs_array.argtypes = [P, i64, i64, P, P]
        L.oracle_lexbfs_partition_seeded.argtypes = [P, i64, i64, ctypes.c_uint64, P]
        L.oracle_lexbfs_labels_seeded.argtypes = [P, i64, i64, ctypes.c_uint64, P]
        L.oracle_mcs_order.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_uint64, P]
        L.oracle_bfs_order.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_uint64, P]
        L.oracle_lexbfs_arbitrated.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_uint64, P]
        L.oracle_is_peo.argtypes = [P, i64, i64, P, P]
        L.oracle_is_peo_csr.argtypes = [P, P, i64, P, P]
        L.oracle_peo_lists_stats.argtypes = [P, P, i64, P, P, P, P, P]
        L.oracle_is_chordal_batch.argtypes = [P, i64, i64, i64, i64, P, P, P, ctypes.c_int]
        L.oracle_splitmix64.argtypes = [ctypes.c_uint64]
        L.oracle_splitmix64.restype = ctypes.c_uint64
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _rows(packed: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(packed, dtype=np.uint8)


def lexbfs_partition(packed: np.ndarray, n: int, members: np.ndarray | None = None) -> np.ndarray:
    """lexbfs_partition(method="linked") (search.py:515-532); 0-based order."""
    rows = _rows(packed)
    order = np.empty(n, dtype=np.int32)
    m = None if members is None else np.ascontiguousarray(members, dtype=np.int32)
    rc = lib().oracle_lexbfs_partition(_ptr(rows), n, rows.shape[1] if n else 0, _ptr(m), _ptr(order))
    if rc:
        raise MemoryError("oracle_lexbfs_partition")
    return order


def lexbfs_array(packed: np.ndarray, n: int, initial: np.ndarray | None = None) -> np.ndarray:
    """lexbfs_array (_arraylex.py:22-65); 0-based order."""
    rows = _rows(packed)
    order = np.empty(n, dtype=np.int32)
    ini = None if initial is None else np.ascontiguousarray(initial, dtype=np.int32)
    rc = lib().oracle_lexbfs_array(_ptr(rows), n, rows.shape[1] if n else 0, _ptr(ini), _ptr(order))
    if rc:
        raise MemoryError("oracle_lexbfs_array")
    return order


ARB_ASCENDING, ARB_DESCENDING, ARB_SEEDED = 0, 1, 2


def lexbfs_arbitrated(packed: np.ndarray, n: int, mode: int, seed: int = 0) -> np.ndarray:
    """parallel_lexbfs election rule (parallel/lexbfs.py:234-262); 0-based."""
    rows = _rows(packed)
    order = np.empty(n, dtype=np.int32)
    rc = lib().oracle_lexbfs_arbitrated(
        _ptr(rows), n, rows.shape[1] if n else 0, mode, seed & ((1 << 64) - 1), _ptr(order)
    )
    if rc:
        raise MemoryError("oracle_lexbfs_arbitrated")
    return order


def is_peo(packed: np.ndarray, n: int, order0: np.ndarray) -> tuple[bool, tuple[int, int, int] | None]:
    """is_peo (peo.py:72-149); witness 0-based (v, p, z) or None."""
    rows = _rows(packed)
    o = np.ascontiguousarray(order0, dtype=np.int32)
    w = np.full(3, -1, dtype=np.int32)
    rc = lib().oracle_is_peo(_ptr(rows), n, rows.shape[1] if n else 0, _ptr(o), _ptr(w))
    if rc < 0:
        raise MemoryError("oracle_is_peo")
    return (True, None) if rc == 1 else (False, (int(w[0]), int(w[1]), int(w[2])))


def lexbfs_linked_seeded(packed: np.ndarray, n: int, seed: int, variant: str) -> np.ndarray:
    """Seeded linked LexBFS: variant "partition" (search.py:515-532) or
    "labels" (search.py:283-310); 0-based order."""
    rows = np.ascontiguousarray(packed, dtype=np.uint8)
    order = np.empty(max(n, 1), dtype=np.int32)
    fn = lib().oracle_lexbfs_partition_seeded if variant == "partition" else lib().oracle_lexbfs_labels_seeded
    if fn(_ptr(rows), n, rows.shape[1] if n else 0, int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(order)):
        raise MemoryError("oracle seeded linked LexBFS")
    return order[:n]


def other_order(packed: np.ndarray, n: int, which: str, seed: int | None = None) -> np.ndarray:
    """mcs_order (search.py:113-145) or bfs_order (search.py:79-110); 0-based."""
    rows = np.ascontiguousarray(packed, dtype=np.uint8)
    order = np.empty(max(n, 1), dtype=np.int32)
    fn = lib().oracle_mcs_order if which == "mcs" else lib().oracle_bfs_order
    if fn(_ptr(rows), n, rows.shape[1] if n else 0, int(seed is not None), int(seed or 0) & 0xFFFFFFFFFFFFFFFF,
          _ptr(order)):
        raise MemoryError("oracle " + which)
    return order[:n]


def lexbfs_partition_csr(indptr: np.ndarray, indices: np.ndarray, n: int) -> np.ndarray:
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    order = np.empty(n, dtype=np.int32)
    if lib().oracle_lexbfs_partition_csr(_ptr(ip), _ptr(ix), n, _ptr(order)):
        raise MemoryError("oracle_lexbfs_partition_csr")
    return order


def is_peo_csr(indptr, indices, n: int, order0) -> tuple[bool, tuple[int, int, int] | None]:
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    o = np.ascontiguousarray(order0, dtype=np.int32)
    w = np.full(3, -1, dtype=np.int32)
    rc = lib().oracle_is_peo_csr(_ptr(ip), _ptr(ix), n, _ptr(o), _ptr(w))
    if rc < 0:
        raise MemoryError("oracle_is_peo_csr")
    return (True, None) if rc == 1 else (False, (int(w[0]), int(w[1]), int(w[2])))


def peo_lists_stats(indptr, indices, n: int, order0):
    """_is_peo_lists with its ScanStats count (peo.py:100-149):
    (ok, witness0|None, parent int32[n], ln_size int32[n], reads)."""
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int32)
    o = np.ascontiguousarray(order0, dtype=np.int32)
    w = np.full(3, -1, dtype=np.int32)
    parent = np.empty(max(n, 1), dtype=np.int32)
    lnsz = np.empty(max(n, 1), dtype=np.int32)
    reads = ctypes.c_int64()
    rc = lib().oracle_peo_lists_stats(_ptr(ip), _ptr(ix), n, _ptr(o), _ptr(w), _ptr(parent), _ptr(lnsz),
                                      ctypes.byref(reads))
    if rc < 0:
        raise MemoryError("oracle_peo_lists_stats")
    wit = None if rc == 1 else (int(w[0]), int(w[1]), int(w[2]))
    return rc == 1, wit, parent[:n], lnsz[:n], int(reads.value)


def csr_from_packed(packed: np.ndarray, n: int):
    """(indptr int64, indices int32) of packed rows (ascending neighbours)."""
    rows = np.unpackbits(np.asarray(packed, dtype=np.uint8), axis=1, bitorder="little", count=n).astype(bool) \
        if n else np.zeros((0, 0), bool)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(rows.sum(axis=1), out=indptr[1:])
    return indptr, (np.flatnonzero(rows.reshape(-1)) % max(n, 1)).astype(np.int32)


def is_chordal(packed: np.ndarray, n: int):
    """is_chordal (peo.py:177-202): (chordal, order0, witness0|None)."""
    order = lexbfs_partition(packed, n)
    ok, w = is_peo(packed, n, order)
    return ok, order, w


def is_chordal_batch(adj: np.ndarray, n: int, nthreads: int | None = None):
    """Batch of dense graphs ``adj[b, n, stride]``; returns (verdict, orders, witness)."""
    a = np.ascontiguousarray(adj, dtype=np.uint8)
    B = a.shape[0]
    orders = np.empty((B, n), dtype=np.int32)
    wit = np.full((B, 3), -1, dtype=np.int32)
    verdict = np.zeros(B, dtype=np.int32)
    nt = nthreads or lib().oracle_max_threads()
    rc = lib().oracle_is_chordal_batch(
        _ptr(a), B, n, a.shape[2], a.shape[1] * a.shape[2], _ptr(orders), _ptr(wit), _ptr(verdict), nt
    )
    if rc:
        raise MemoryError("oracle_is_chordal_batch")
    return verdict.astype(bool), orders, wit


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _gen_lib():
    L = lib()
    if not getattr(L, "_gen_bound", False):
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_gen_dense_random.argtypes = [i64, ctypes.c_double, ctypes.c_uint64, i64, P]
        L.oracle_gen_chordal_random.argtypes = [i64, i64, ctypes.c_uint64, i64, P]
        L.oracle_gen_config4_batch.argtypes = [i64, ctypes.c_double, i64, i64, i64, i64, P, ctypes.c_int]
        L._gen_bound = True
    return L


def gen_dense_random(n: int, p: float, seed: int, stride: int | None = None) -> np.ndarray:
    """gen_dense_random (generate.py:32-56) as packed rows uint8[n, stride]."""
    stride = stride or (n + 7) // 8
    out = np.empty((n, stride), dtype=np.uint8)
    _gen_lib().oracle_gen_dense_random(n, float(p), int(seed) & 0xFFFFFFFFFFFFFFFF, stride, _ptr(out))
    return out


def gen_chordal_random(n: int, k: int, seed: int, stride: int | None = None) -> np.ndarray:
    """gen_chordal_random (generate.py:118-155) as packed rows uint8[n, stride]."""
    stride = stride or (n + 7) // 8
    out = np.empty((n, stride), dtype=np.uint8)
    if _gen_lib().oracle_gen_chordal_random(n, k, int(seed) & 0xFFFFFFFFFFFFFFFF, stride, _ptr(out)):
        raise MemoryError("oracle_gen_chordal_random")
    return out


def gen_config4_batch(seed_lo: int, count: int, n: int = 512, p: float = 0.5, k: int = 8, stride: int = 64,
                      nthreads: int | None = None) -> np.ndarray:
    """Configuration 4's graphs of seeds [seed_lo, seed_lo + count): even seed
    gen_dense_random(n, p, s), odd seed gen_chordal_random(n, k, s); uint8[count, n, stride]."""
    out = np.empty((count, n, stride), dtype=np.uint8)
    rc = _gen_lib().oracle_gen_config4_batch(n, float(p), k, seed_lo, count, stride, _ptr(out),
                                             nthreads or max_threads())
    if rc:
        raise MemoryError("oracle_gen_config4_batch")
    return out


def lexbfs_certify(packed: np.ndarray, n: int, order0) -> tuple[int, int]:
    """LexBFS certificate of ``order0`` (pure Python, small n): replay the
    search with pivot i forced to order0[i], labels materialised as in the
    reference's debug mode (search.py:270-271: digit n - i appended at step i,
    _check_chain search.py:313-322: the chain's labels ascend to the class the
    pivot is taken from; parallel/lexbfs.py:82-129 audits the same set-list
    invariant).  Returns (first step whose pivot does not carry the largest
    label, first step whose pivot is not the smallest id among the vertices
    with the largest label), -1 for none."""
    rows = np.unpackbits(np.asarray(packed, dtype=np.uint8), axis=1, bitorder="little", count=n).astype(bool) \
        if n else np.zeros((0, 0), bool)
    adj = [np.flatnonzero(rows[v]).tolist() for v in range(n)]
    label: list[list[int]] = [[] for _ in range(n)]
    visited = [False] * n
    off = -1
    for i, x in enumerate(int(v) for v in order0):
        best = max(label[v] for v in range(n) if not visited[v])
        if label[x] != best:
            return i, (i if off < 0 else off)
        if off < 0 and x != min(v for v in range(n) if not visited[v] and label[v] == best):
            off = i
        visited[x] = True
        for y in adj[x]:
            if not visited[y]:
                label[y].append(n - i)
    return -1, off
