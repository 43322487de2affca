"""The C-ABI library loads without a GPU and exports every symbol the header declares."""

import os
import re

from paper_2309_05884_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "symqoc_b200.h")


def test_header_symbols_exported():
    names = set(re.findall(r"\b(sqoc_\w+)\s*\(", open(HEADER).read()))
    assert names, "no declarations found"
    lib = _lib.load()
    for name in names:
        assert hasattr(lib, name), name
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)


def test_abi_version_and_limits():
    lib = _lib.load()
    assert lib.sqoc_abi_version() == 2
    assert lib.sqoc_tiny_max_dim() == 16


def test_create_rejects_bad_arguments():
    import ctypes

    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.sqoc_create(ctypes.byref(h), 0, 0, None, 2, None, None, 1, None, None, None, 10, 0.1, 1)
    assert rc == _lib.SQOC_ERR_ARG
    assert b"missing" in lib.sqoc_last_error()


def test_trotter_and_chunk_entry_points_reject_bad_arguments_without_a_gpu():
    import ctypes

    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.sqoc_trotter_create(ctypes.byref(h), 0, 13, 1.0, None, 0, 0.05, 0) == _lib.SQOC_ERR_ARG
    assert b"n <= 12" in lib.sqoc_last_error()
    cpl = (ctypes.c_double * 3)(0.2, 0.1, 0.1)
    assert lib.sqoc_trotter_create(ctypes.byref(h), 0, 4, 1.0, cpl, 3, 0.05, 0) == _lib.SQOC_ERR_ARG
    assert lib.sqoc_trotter_apply(None, None, 1, None, None, 1, 0, None) == _lib.SQOC_ERR_ARG
    assert lib.sqoc_trotter_replay(None, None, None, 1, 1, None, 0, None) == _lib.SQOC_ERR_ARG
    assert lib.sqoc_chunk_forward(None, None, None, 0, None) == _lib.SQOC_ERR_ARG
    assert lib.sqoc_chunk_backward(None, None, None, 1, 0, None, None, None, 0, None) == _lib.SQOC_ERR_ARG
    n = ctypes.c_longlong()
    assert lib.sqoc_chunk_size(None, ctypes.byref(n)) == _lib.SQOC_ERR_ARG
