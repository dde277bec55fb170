"""The C-ABI library loads and exports every symbol include/chordal_b200.h declares.

No compute calls here (this runs without a GPU).
"""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "chordal_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|size_t|const char \*)\s*(chordal_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("chordal_lexbfs_dense", "chordal_peo_dense", "chordal_is_chordal_dense",
                 "chordal_is_chordal_dense_host", "chordal_is_chordal_batch", "chordal_peo_dense_key",
                 "chordal_peo_dense_witness", "chordal_parse_graph_text", "chordal_write_graph_text",
                 "chordal_mcs_dense", "chordal_bfs_csr", "chordal_lexbfs_csr"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1508_06329_b200 import _native

    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    # and the ctypes binding covers every declared entry point
    assert set(declared_functions()) <= set(_native.exported_symbols())


def test_library_is_sm100a():
    import subprocess

    from paper_1508_06329_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings():
    from paper_1508_06329_b200 import _native

    assert _native.lib.chordal_strerror(0) == b"ok"
    assert _native.lib.chordal_abi_version() == 3


def test_round2_entry_points_host_side():
    """Certificate / NCCL entry points: workspace sizes, argument validation that
    needs no device (NULL communicator / status), the ENCCL status string, and the
    communicator-pointer helper."""
    from paper_1508_06329_b200 import _native
    from paper_1508_06329_b200.distributed import _comm_ptr

    lib = _native.lib
    assert lib.chordal_lexbfs_certify_workspace_bytes(0) == 0
    assert lib.chordal_lexbfs_certify_workspace_bytes(1000) == 8000
    assert lib.chordal_strerror(_native.ENCCL).startswith(b"NCCL")
    d1, d2 = lib.chordal_dense_nccl_workspace_bytes(1000, 4000), lib.chordal_dense_nccl_workspace_bytes(2000, 4000)
    assert 0 < d1 < d2
    # n > 32768 dense: the CSR route's workspace grows with m
    assert lib.chordal_dense_nccl_workspace_bytes(40000, 10**6) > lib.chordal_dense_nccl_workspace_bytes(40000, 10**5)
    assert lib.chordal_csr_nccl_workspace_bytes(10**6, 8 * 10**6) > lib.chordal_csr_nccl_workspace_bytes(10**6, 10**6)
    # NULL communicator / status: rejected before anything touches a device
    assert lib.chordal_is_chordal_csr_nccl(None, None, 10, 5, 0, 0, 0, None, None, None, None, None, 0,
                                           None) == _native.EINVAL
    assert lib.chordal_lexbfs_certify_dense(None, 10, 16, 0, None, None, None, 0, None) == _native.EINVAL
    assert _comm_ptr(0x1234) == 0x1234
