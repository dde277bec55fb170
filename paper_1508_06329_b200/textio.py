"""Plain-text graph and ordering formats (reference textio.py), parsed in C++.

Same functions, formats, exceptions and messages as the reference
(``textio.py:30-110``): ``parse_graph_text`` scans the text in
``libchordal_b200.so`` (``chordal_parse_graph_text``, csrc/textio.cpp) and
fills the packed rows of the returned ``Graph`` in the same pass;
``write_graph_text`` serialises in C++ as well.  Host code only (no GPU).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import GraphTooLarge, InvalidOrdering, ParseError
from .graph import DEFAULT_VERTEX_CAP, Graph, VertexOrdering, row_width

_ERR_CAP = 512


def _as_bytes(data: str | bytes) -> bytes:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return bytes(data)
    return data.encode("utf-8", "surrogatepass")


def _utf8_error(raw: bytes) -> ParseError:
    try:
        raw.decode("utf-8")
    except UnicodeDecodeError as e:  # the reference's message (textio.py:23-27)
        return ParseError(f"input is not valid UTF-8: {e}")
    return ParseError("input is not valid UTF-8")


def _raise(rc: int, raw: bytes, line: ctypes.c_int64, msg: ctypes.Array, cap: int) -> None:
    text = msg.value.decode("utf-8", "replace")
    if rc == _native.EUTF8:
        raise _utf8_error(raw)
    if rc == _native.EPARSE:
        raise ParseError(text, None if line.value < 0 else int(line.value))
    if rc == _native.ETOOLARGE:  # _check_size (graph.py:23-28)
        raise GraphTooLarge(f"n={text} exceeds the configured cap of {cap}")
    _native.check(rc, "chordal_parse_graph_text")


def parse_graph_text(data: str | bytes, *, cap: int | None = None) -> Graph:
    """Parse the edge-list text format into a Graph (textio.py:30-86)."""
    raw = _as_bytes(data)
    limit = DEFAULT_VERTEX_CAP if cap is None else int(cap)
    n, m, line = ctypes.c_int64(-1), ctypes.c_int64(-1), ctypes.c_int64(-1)
    msg = ctypes.create_string_buffer(_ERR_CAP)
    lib = _native.lib
    rc = lib.chordal_parse_graph_text(raw, len(raw), limit, ctypes.byref(n), ctypes.byref(m), None, 0,
                                      ctypes.byref(line), msg, _ERR_CAP)
    if rc != _native.OK:
        _raise(rc, raw, line, msg, limit)
    w = row_width(int(n.value))
    rows = np.zeros((int(n.value), w), dtype=np.uint8)
    rc = lib.chordal_parse_graph_text(raw, len(raw), limit, ctypes.byref(n), ctypes.byref(m),
                                      rows.ctypes.data if rows.size else None, w, ctypes.byref(line), msg, _ERR_CAP)
    if rc != _native.OK:
        _raise(rc, raw, line, msg, limit)
    rows.setflags(write=False)
    return Graph(int(n.value), rows, int(m.value))


def write_graph_text(g: Graph) -> str:
    """Serialize a Graph; edges come out u < v, ascending (textio.py:89-93)."""
    packed = np.ascontiguousarray(g._packed)
    n, w = int(g.n), int(packed.shape[1]) if packed.ndim == 2 else 0
    ptr = packed.ctypes.data if packed.size else None
    size = _native.lib.chordal_write_graph_text(ptr, n, w, int(g.m), None, 0)
    if size < 0:
        raise ValueError("chordal_write_graph_text: invalid graph rows")
    buf = ctypes.create_string_buffer(int(size))
    _native.lib.chordal_write_graph_text(ptr, n, w, int(g.m), buf, size)
    return buf.raw[:size].decode("ascii")


def parse_ordering_text(data: str | bytes, n: int) -> VertexOrdering:
    """Parse a one-line permutation of 1..n (textio.py:96-106)."""
    raw = _as_bytes(data)
    n = int(n)
    out = np.zeros(max(n, 1), dtype=np.int64)
    count, line = ctypes.c_int64(0), ctypes.c_int64(-1)
    msg = ctypes.create_string_buffer(_ERR_CAP)
    rc = _native.lib.chordal_parse_ordering_text(raw, len(raw), n, out.ctypes.data, ctypes.byref(count),
                                                 ctypes.byref(line), msg, _ERR_CAP)
    if rc == _native.EUTF8:
        raise _utf8_error(raw)
    if rc == _native.EPARSE:
        raise ParseError(msg.value.decode("utf-8", "replace"))
    _native.check(rc, "chordal_parse_ordering_text")
    if int(count.value) != n:
        raise InvalidOrdering(f"expected {n} entries, got {int(count.value)}")
    return VertexOrdering([int(x) for x in out[:n]])


def write_ordering_text(ordering: VertexOrdering) -> str:
    """One line of 1-based ids (textio.py:109-110)."""
    order0 = np.asarray(ordering.order0, dtype=np.int64)
    return " ".join(map(str, (order0 + 1).tolist())) + "\n"


__all__ = ["parse_graph_text", "write_graph_text", "parse_ordering_text", "write_ordering_text"]
