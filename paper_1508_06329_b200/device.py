"""HBM residency for graphs: padded bit rows as torch uint8 tensors.

PyTorch is used here only as the device-memory / stream allocator; all
compute happens in libchordal_b200.so.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _native
from .graph import Graph, device_stride, row_width


class DeviceRows:
    """Packed rows in HBM: ``data`` is uint8[n, stride], stride % 16 == 0."""

    __slots__ = ("n", "stride", "data", "m")

    def __init__(self, n: int, stride: int, data, m: int = -1):
        self.n = n
        self.stride = stride
        self.data = data
        self.m = m  # edge count if known (-1: the library counts it)

    @property
    def ptr(self) -> int:
        return int(self.data.data_ptr())


def upload_packed(packed: np.ndarray, n: int, device=None, stream=None, m: int = -1) -> DeviceRows:
    """Copy packed rows (n, ceil(n/8)) to the device with a 16-byte pitch."""
    torch = _native.require_cuda()
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    stride = device_stride(n)
    w = row_width(n)
    if n == 0:
        return DeviceRows(0, stride, torch.zeros((0, stride), dtype=torch.uint8, device=dev), 0)
    with warnings.catch_warnings():  # read-only source (Graph._packed); we never write it
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(np.ascontiguousarray(packed, dtype=np.uint8))
    if w == stride:
        data = host.to(dev, non_blocking=False)
    else:
        data = torch.zeros((n, stride), dtype=torch.uint8, device=dev)
        data[:, :w].copy_(host.to(dev))
    return DeviceRows(n, stride, data, m)


def device_rows(g) -> DeviceRows:
    """Rows of graph ``g`` in HBM; cached on this package's Graph objects.

    Foreign graphs (e.g. ``chordalkit.Graph``, which has no spare slot) are
    uploaded on every call.
    """
    torch = _native.require_cuda()
    own = isinstance(g, Graph)
    if own and g._dev is not None and g._dev.data.device.index == torch.cuda.current_device():
        return g._dev
    rows = upload_packed(g._packed, int(g.n), m=int(getattr(g, "m", -1)))
    if own:
        g._dev = rows
    return rows
