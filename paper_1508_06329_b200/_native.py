"""ctypes binding of libchordal_b200.so (declared in include/chordal_b200.h).

This is the only way the package computes anything: there is no CPU fallback.
If the shared library is missing the import fails loudly; if CUDA is not
available a call raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError, GraphTooLarge, InvalidOrdering

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libchordal_b200.so")

OK, EINVAL, ETOOLARGE, ECUDA, ENOMEM, EPARSE, EUTF8, ENCCL = 0, 1, 2, 3, 4, 5, 6, 7
TIE_ASCENDING, TIE_DESCENDING, TIE_SEEDED_ARB, TIE_SEEDED_PARTITION, TIE_SEEDED_LABELS = 0, 1, 2, 3, 4
DENSE_LEXBFS_MAX_N = 32768
BATCH_MAX_N = 1024

# name -> argtypes; restype is int unless listed in _RESTYPES
_P, _I64, _I32, _U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
_D, _SZ = ctypes.c_double, ctypes.c_size_t
SIGNATURES = {
    "chordal_abi_version": [],
    "chordal_strerror": [ctypes.c_int],
    "chordal_dense_workspace_bytes": [_I64, _I64],
    "chordal_lexbfs_dense": [_P, _I64, _I64, _I64, _I32, _U64, _P, _P, _P, _P, _SZ, _P],
    "chordal_lexbfs_certify_workspace_bytes": [_I64],
    "chordal_lexbfs_certify_dense": [_P, _I64, _I64, _I64, _P, _P, _P, _SZ, _P],
    "chordal_positions": [_P, _I64, _P, _P],
    "chordal_dense_nccl_workspace_bytes": [_I64, _I64],
    "chordal_is_chordal_dense_nccl": [_P, _I64, _I64, _I64, _I32, _U64, _I32, _P, _P, _P, _P, _P, _SZ, _P],
    "chordal_csr_nccl_workspace_bytes": [_I64, _I64],
    "chordal_is_chordal_csr_nccl": [_P, _P, _I64, _I64, _I32, _U64, _I32, _P, _P, _P, _P, _P, _SZ, _P],
    "chordal_key_init": [_P, _P],
    "chordal_peo_dense_key": [_P, _I64, _I64, _P, _P, _P, _I64, _I64, _P, _P],
    "chordal_peo_dense_witness": [_P, _I64, _I64, _P, _P, _P, _P],
    "chordal_peo_dense": [_P, _I64, _I64, _P, _P, _P, _P, _P, _P],
    "chordal_is_chordal_dense": [_P, _I64, _I64, _I64, _I32, _U64, _P, _P, _P, _SZ, _P, _P],
    "chordal_is_chordal_dense_host": [_P, _I64, _I64, _I32, _U64, _P, _P, _P],
    "chordal_dense_host_workspace_bytes": [_I64, _I64],
    "chordal_is_chordal_dense_host_ws": [_P, _I64, _I64, _I64, _I32, _U64, _P, _P, _P, _P, _SZ],
    "chordal_lexbfs_csr_workspace_bytes": [_I64, _I64],
    "chordal_lexbfs_csr": [_P, _P, _I64, _I64, _I32, _U64, _P, _P, _P, _P, _SZ, _P],
    "chordal_peo_csr_workspace_bytes": [_I64],
    "chordal_peo_csr_key": [_P, _P, _I64, _P, _P, _I64, _I64, _P, _P, _SZ, _P],
    "chordal_peo_csr_witness": [_P, _P, _I64, _P, _P, _P, _P],
    "chordal_peo_csr": [_P, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P],
    "chordal_dense_to_csr": [_P, _I64, _I64, _P, _P, _P],
    "chordal_left_dense": [_P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P],
    "chordal_left_csr": [_P, _P, _I64, _P, _P, _P, _P, _P],
    "chordal_permute_dense": [_P, _I64, _I64, _P, _P, _P],
    "chordal_is_chordal_batch": [_P, _I64, _I64, _I64, _P, _P, _P],
    "chordal_is_chordal_batch_host": [_P, _I64, _I64, _I64, _P, _P, _I64],
    "chordal_batch_host_workspace_bytes": [_I64, _I64],
    "chordal_is_chordal_batch_host_ws": [_P, _I64, _I64, _I64, _P, _P, _I64, _P, _SZ],
    "chordal_gen_dense_random": [_P, _I64, _I64, _I64, _D, _I64, _I64, _P],
    "chordal_edges_to_dense": [_P, _P, _I64, _P, _I64, _I64, _P],
    "chordal_gen_chordal_random_scratch_bytes": [_I64, _I64, _I64],
    "chordal_gen_chordal_random": [_P, _I64, _I64, _I64, _I64, _I64, _I64, _P, _SZ, _P],
    "chordal_gen_chordal_random_edges": [_I64, _I64, _I64, _P, _P, _P, _P, _SZ, _P],
    "chordal_mcs_dense": [_P, _I64, _I64, _I32, _U64, _P, _P, _P],
    "chordal_bfs_csr_workspace_bytes": [_I64],
    "chordal_bfs_dense": [_P, _I64, _I64, _I32, _U64, _P, _P, _P],
    "chordal_bfs_csr": [_P, _P, _I64, _I32, _U64, _P, _P, _P, _SZ, _P],
    "chordal_parse_graph_text": [_P, _I64, _I64, _P, _P, _P, _I64, _P, _P, _I64],
    "chordal_write_graph_text": [_P, _I64, _I64, _I64, _P, _I64],
    "chordal_parse_ordering_text": [_P, _I64, _I64, _P, _P, _P, _P, _I64],
}
_RESTYPES = {
    "chordal_strerror": ctypes.c_char_p,
    "chordal_gen_chordal_random_scratch_bytes": _SZ,
    "chordal_dense_workspace_bytes": _SZ,
    "chordal_lexbfs_certify_workspace_bytes": _SZ,
    "chordal_dense_nccl_workspace_bytes": _SZ,
    "chordal_csr_nccl_workspace_bytes": _SZ,
    "chordal_peo_csr_workspace_bytes": _SZ,
    "chordal_lexbfs_csr_workspace_bytes": _SZ,
    "chordal_write_graph_text": _I64,
    "chordal_bfs_csr_workspace_bytes": _SZ,
    "chordal_batch_host_workspace_bytes": _SZ,
    "chordal_dense_host_workspace_bytes": _SZ,
}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the package has no CPU fallback)"
    )

lib = ctypes.CDLL(LIB_PATH)
for _name, _args in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _RESTYPES.get(_name, ctypes.c_int)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def check(status: int, what: str) -> None:
    """Map a library status code onto the reference's exception types."""
    if status == OK:
        return
    msg = f"{what}: {lib.chordal_strerror(status).decode()}"
    if status == EINVAL:
        raise ValueError(msg)
    if status == ETOOLARGE:
        raise GraphTooLarge(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise DeviceError(msg)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("CUDA device not available: the chordality kernels run only on a GPU")
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr())


__all__ = ["lib", "check", "require_cuda", "stream_ptr", "ptr", "InvalidOrdering"]
