"""ctypes binding of the C ABI (include/symqoc_b200.h).

The shared library is built in-tree by ``build.py`` (nvcc, sm_100a).  There is
no fallback: if the library or a GPU is missing, every product entry point
raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsymqoc_b200.so")

SQOC_OK = 0
SQOC_ERR_ARG = 1
SQOC_ERR_NONFINITE = 2
SQOC_ERR_CUDA = 3
SQOC_ERR_UNSUPPORTED = 4
SQOC_ERR_NCCL = 5
OBJ_STATE = 0
OBJ_GATE = 1
MEM_HOST = 0
MEM_DEVICE = 1

# name -> (restype, argtypes); the ABI surface tests check every name is exported
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_DP = ctypes.POINTER(ctypes.POINTER(ctypes.c_double))
_I = ctypes.c_int
SIGNATURES = {
    "sqoc_create": (_I, [ctypes.POINTER(_P), _I, _I, ctypes.POINTER(_I), _I, _DP, _DP, _I, _DP, _DP, _D, _I,
                         ctypes.c_double, _I]),
    "sqoc_eval": (_I, [_P, _P, _I, _P, _P, _P, _I, _P]),
    "sqoc_destroy": (_I, [_P]),
    "sqoc_state_gradient": (_I, [_I, _I, _D, _D, _D, _D, _D, _D, _D, _I, ctypes.c_double, _D, _D, _D]),
    "sqoc_last_launch_count": (_I, [_P]),
    "sqoc_set_timing": (_I, [_P, _I]),
    "sqoc_set_complex_gemm": (_I, [_I]),
    "sqoc_set_schedule": (_I, [_P, _I]),
    "sqoc_last_schedule": (_I, [_P]),
    "sqoc_set_tiny_schedule": (_I, [_P, _I]),
    "sqoc_last_tiny_schedule": (_I, [_P]),
    "sqoc_set_tiny_history": (_I, [_P, _I]),
    "sqoc_last_tiny_history": (_I, [_P]),
    "sqoc_set_tiny_cta_warps": (_I, [_P, _I]),
    "sqoc_last_plan": (_I, [_P, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "sqoc_set_norm_bounds": (_I, [_P, _D]),
    "sqoc_chunk_size": (_I, [_P, ctypes.POINTER(ctypes.c_longlong)]),
    "sqoc_chunk_forward": (_I, [_P, _P, _P, _I, _P]),
    "sqoc_chunk_backward": (_I, [_P, _P, _P, _I, _I, _P, _P, _P, _I, _P]),
    "sqoc_last_carry_stats": (_I, [_P, _D, ctypes.POINTER(_I)]),
    "sqoc_block_time_ms": (_I, [_P, _I, _D]),
    "sqoc_last_gemm_stats": (_I, [_P, _D, _D, ctypes.POINTER(_I)]),
    "sqoc_complex_gemm_mults": (_I, []),
    "sqoc_set_gemm_staging": (_I, [_I]),
    "sqoc_gemm_staging": (_I, []),
    "sqoc_tiny_max_dim": (_I, []),
    "sqoc_dn_basis_create": (_I, [ctypes.POINTER(_P), _I, _I]),
    "sqoc_basis_info": (_I, [_P, ctypes.POINTER(_I), _P, _P]),
    "sqoc_basis_nnz": (_I, [_P, _I, ctypes.POINTER(ctypes.c_longlong)]),
    "sqoc_basis_columns": (_I, [_P, _I, _P, _P, _P, _P]),
    "sqoc_basis_compress": (_I, [_P, _I, _P, _P, _P, _P]),
    "sqoc_basis_destroy": (_I, [_P]),
    "sqoc_trotter_create": (_I, [ctypes.POINTER(_P), _I, _I, ctypes.c_double, _P, _I, ctypes.c_double, _I]),
    "sqoc_trotter_apply": (_I, [_P, _P, _I, _P, _P, _I, _I, _P]),
    "sqoc_trotter_replay": (_I, [_P, _P, _P, _I, _I, _P, _I, _P]),
    "sqoc_trotter_last_launches": (_I, [_P]),
    "sqoc_trotter_destroy": (_I, [_P]),
    "sqoc_last_error": (ctypes.c_char_p, []),
    "sqoc_abi_version": (_I, []),
}

_lib = None


class EngineError(RuntimeError):
    pass


def load():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EngineError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    """Map SQOC status codes onto the reference's exception types."""
    if rc == SQOC_OK:
        return
    msg = f"{what}: {load().sqoc_last_error().decode(errors='replace')}"
    if rc == SQOC_ERR_ARG:
        raise ValueError(msg)
    if rc == SQOC_ERR_NONFINITE:
        raise FloatingPointError(msg)
    raise EngineError(msg)
