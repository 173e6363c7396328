"""ctypes binding of include/ebic.h (libebic.so, built in-tree by build.py).

There is deliberately no fallback: if libebic.so is missing or cannot be
loaded, `lib()` raises, and every evaluating call in this package fails loudly.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .build import LIB_PATH

EBIC_OK = 0
EBIC_ERR_INVALID_ARGUMENT = 1
EBIC_ERR_CUDA = 2
EBIC_ERR_NO_MATRIX = 3
EBIC_ERR_CAPACITY = 4
EBIC_ERR_NOT_EXACT = 5
EBIC_ERR_NO_DEVICE = 6
EBIC_ERR_IO = 7

EBIC_STORE_AUTO = 0
EBIC_STORE_F32 = 1
EBIC_STORE_F64 = 2

# every function declared in include/ebic.h: name -> (restype, argtypes)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p
SIGNATURES = {
    "ebic_abi_version": (C.c_int, []),
    "ebic_last_error": (C.c_char_p, []),
    "ebic_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "ebic_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "ebic_ctx_destroy": (C.c_int, [_vp]),
    "ebic_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "ebic_ctx_sync": (C.c_int, [_vp]),
    "ebic_matrix_upload_f64": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_int)]),
    "ebic_matrix_upload_f32": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ebic_matrix_upload_device_f64": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_int)]),
    "ebic_matrix_upload_device_f32": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ebic_matrix_info": (C.c_int, [_vp, _u64p, _u64p, _u64p, C.POINTER(C.c_int), _u64p]),
    "ebic_matrix_free": (C.c_int, [_vp]),
    "ebic_eval_counts": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp]),
    "ebic_eval_counts_device": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp, _vp]),
    "ebic_eval_submit": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp, _u64p]),
    "ebic_eval_wait": (C.c_int, [_vp, C.c_uint64]),
    "ebic_support_rows": (C.c_int, [_vp, _vp, C.c_uint32, C.c_double, C.c_int, _vp, C.c_uint64, _u64p]),
    "ebic_support_rows_batch": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp, C.c_uint64, _vp]),
    "ebic_support_overlap_batch": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp, _vp]),
    "ebic_row_supports": (C.c_int, [_vp, C.c_uint64, _vp, C.c_uint32, C.c_double, C.c_int, C.POINTER(C.c_int)]),
    "ebic_fitness": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]),
    "ebic_ctx_launch_count": (C.c_int, [_vp, _u64p]),
    "ebic_ctx_set_slab_rows": (C.c_int, [_vp, C.c_uint32]),
    "ebic_ctx_set_path": (C.c_int, [_vp, C.c_int]),
    "ebic_matrix_index_stats": (C.c_int, [_vp, C.POINTER(C.c_int)] + [C.POINTER(C.c_uint64)] * 6),
    "ebic_ctx_set_pair_layout": (C.c_int, [_vp, C.c_int, C.c_int]),
    "ebic_ctx_set_table_budget": (C.c_int, [_vp, C.c_uint64]),
    "ebic_ctx_set_lazy_build": (C.c_int, [_vp, C.c_int]),
    "ebic_matrix_index_info": (C.c_int, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
    "ebic_tsv_read": (C.c_int, [C.c_char_p, C.c_int, _vp, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ebic_matrix_load_tsv": (C.c_int, [_vp, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ebic_xchg_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_uint64, _vp]),
    "ebic_xchg_open": (C.c_int, [_vp, _vp]),
    "ebic_xchg_open_local": (C.c_int, [_vp, _vp]),
    "ebic_xchg_window": (C.c_int, [_vp, C.POINTER(C.c_void_p)]),
    "ebic_xchg_destroy": (C.c_int, [_vp]),
    "ebic_eval_counts_rows_sum": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp, _vp]),
    "ebic_eval_counts_rows_sum_async": (C.c_int, [_vp, _vp, _vp, C.c_uint64, C.c_double, C.c_int, _vp, _vp]),
    "ebic_xchg_fence": (C.c_int, [_vp, _vp]),
    "ebic_matrix_prepare": (C.c_int, [_vp, C.c_double]),
    "ebic_matrix_build_info": (C.c_int, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
}

EBIC_PATH_AUTO = 0
EBIC_PATH_VALUE = 1
EBIC_PATH_PLANE = 2
EBIC_PATH_PLANE_U32 = 3
EBIC_PATH_TABLE = 4
EBIC_PATH_LAZY = 5
EBIC_IPC_HANDLE_BYTES = 64


class EbicError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"ebic status {status}: {message}")
        self.status = status


_lock = threading.Lock()
_lib = None


def lib_path() -> Path:
    return LIB_PATH


def lib():
    """Load libebic.so (raises if it is missing -- there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: the CUDA extension must be built "
                    "(python -m paper_2105_01196_b200.build or __graft_entry__.build())")
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().ebic_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    if status != EBIC_OK:
        raise EbicError(status, last_error())
