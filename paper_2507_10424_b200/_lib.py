"""ctypes loader for the in-tree libldpc.so (argument marshalling only; no fallback path)."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("LDPC_LIB") or os.path.join(HERE, "libldpc.so")  # LDPC_LIB: A/B builds

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U32 = ctypes.c_uint32

# name -> (restype, argtypes); mirrors include/ldpc.h one to one
SIGNATURES = {
    "ldpc_prepare_dense": (ctypes.c_int, [P, I32, I32, U32, P, ctypes.POINTER(P)]),
    "ldpc_prepare_coo": (ctypes.c_int, [P, P, I64, I32, I32, U32, P, ctypes.POINTER(P)]),
    "ldpc_decode": (ctypes.c_int, [P, P, I64, I32, P, P, P, P, P, P]),
    "ldpc_decode_host": (ctypes.c_int, [P, P, I64, I32, P, P, P, P, P, P]),
    "ldpc_info": (ctypes.c_int, [P, P, P, P, P, P]),
    "ldpc_get_graph": (ctypes.c_int, [P, P, P, P, P]),
    "ldpc_set_flags": (ctypes.c_int, [P, U32]),
    "ldpc_set_chunk": (ctypes.c_int, [P, I64]),
    "ldpc_set_check_every": (ctypes.c_int, [P, I32]),
    "ldpc_schedule": (ctypes.c_int, [P]),
    "ldpc_profile_enable": (ctypes.c_int, [P, ctypes.c_int]),
    "ldpc_profile_read": (ctypes.c_int, [P, P, P]),
    "ldpc_profile_reset": (ctypes.c_int, [P]),
    "ldpc_launch_count": (I64, [P]),
    "ldpc_stream_counters": (ctypes.c_int, [P, P]),
    "ldpc_destroy": (None, [P]),
    "ldpc_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "ldpc_abi_version": (ctypes.c_int, []),
}

_lib = None


def load():
    """Load libldpc.so.  Raises if it is missing: there is no CPU or eager fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(
            f"libldpc.so not found at {SO_PATH}; build it with `python -m paper_2507_10424_b200.build` "
            "(or __graft_entry__.build()).  There is no fallback decoder.")
    lib = ctypes.CDLL(SO_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
