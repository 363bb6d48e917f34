"""ctypes binding of libmtnlg.so (the C ABI declared in include/*.h).

The product path has no fallback: if the library is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libmtnlg.so"
_lib = None


class GemmArgs(C.Structure):
    _fields_ = [
        ("a", C.c_void_p), ("lda", C.c_int64), ("a_batch_stride", C.c_int64), ("a_mn_major", C.c_int32),
        ("b", C.c_void_p), ("ldb", C.c_int64), ("b_batch_stride", C.c_int64), ("b_mn_major", C.c_int32),
        ("d", C.c_void_p), ("ldd", C.c_int64), ("d_batch_stride", C.c_int64),
        ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("batch", C.c_int64),
        ("alpha", C.c_float), ("epilogue", C.c_int32), ("causal", C.c_int32),
        ("bias", C.c_void_p), ("aux", C.c_void_p), ("ld_aux", C.c_int64), ("block_n", C.c_int32),
    ]


EPI_STORE_BF16, EPI_BIAS_GELU, EPI_GELU_BWD, EPI_STORE_F32, EPI_ACCUM_F32 = range(5)
CAUSAL_NONE, CAUSAL_SKIP_UPPER_TILES, CAUSAL_K_LE_M, CAUSAL_K_GE_M = range(4)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(f"native library {_LIB_PATH} is missing: run `python -m paper_2201_11990_b200.build`")
        _lib = C.CDLL(str(_LIB_PATH))
        _declare(_lib)
    return _lib


def _declare(L: C.CDLL) -> None:
    L.mt_gemm.argtypes = [C.POINTER(GemmArgs), C.c_void_p]
    L.mt_gemm.restype = C.c_int
