"""ctypes binding of libwect.so (include/wect.h).  Argument marshalling only: every
step of the computation runs in the library's CUDA kernels.  There is no CPU
fallback -- if the library or a GPU is missing, calls raise."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WECT_LIBWECT_OVERRIDE", os.path.join(HERE, "libwect.so"))  # dev experiments only

# wect_status
OK, EINVAL, ERANGE, EOVERFLOW, ECUDA, ENOMEM, ENOTSUP = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "WECT_OK", -1: "WECT_EINVAL", -2: "WECT_ERANGE", -3: "WECT_EOVERFLOW", -4: "WECT_ECUDA",
                -5: "WECT_ENOMEM", -6: "WECT_ENOTSUP"}
# wect_dtype
U8, I32, I64, F32, F64 = 1, 2, 3, 4, 5
# flags
VALIDATE, FP32_ONLY, TIME_MAIN, FREUDENTHAL = 1, 2, 4, 8

EXPORTS = ("wect_complex", "wect_images", "ecf_complex", "ecf_images", "wect_complex_backward", "ecf_complex_backward", "wect_maxheight", "wect_sync_status", "wect_last_error",
           "wect_repair_count", "wect_stats", "wect_abi_version")


class WectError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class wect_cells(ctypes.Structure):
    _fields_ = [("verts", ctypes.c_void_p), ("weights", ctypes.c_void_p), ("count", ctypes.c_int64),
                ("arity", ctypes.c_int32), ("dim", ctypes.c_int32)]


class wect_complex_desc(ctypes.Structure):
    _fields_ = [("coords", ctypes.c_void_p), ("k0", ctypes.c_int64), ("n", ctypes.c_int32),
                ("vweights", ctypes.c_void_p), ("cells", ctypes.POINTER(wect_cells)), ("ncell_dims", ctypes.c_int32),
                ("wdtype", ctypes.c_int)]


class wect_grid(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("d_begin", ctypes.c_int32), ("d_count", ctypes.c_int32),
                ("maxheight", ctypes.c_double), ("lo", ctypes.c_double), ("hi", ctypes.c_double),
                ("flags", ctypes.c_uint32)]


_L = None


def load() -> ctypes.CDLL:
    """Load libwect.so; raises ImportError if it was not built (no fallback)."""
    global _L
    if _L is not None:
        return _L
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.wect_complex.argtypes = [ctypes.POINTER(wect_complex_desc), vp, i32, ctypes.POINTER(wect_grid), vp, ctypes.c_int, vp]
    L.ecf_complex.argtypes = L.wect_complex.argtypes
    L.wect_images.argtypes = [vp, i64, i32, vp, vp, i32, ctypes.POINTER(wect_grid), vp, ctypes.c_int, vp]
    L.ecf_images.argtypes = [vp, i64, i32, vp, ctypes.POINTER(wect_grid), vp, ctypes.c_int, vp]
    L.wect_complex_backward.argtypes = [ctypes.POINTER(wect_complex_desc), vp, i32, ctypes.POINTER(wect_grid), vp, vp,
                                        vp, vp]
    L.ecf_complex_backward.argtypes = L.wect_complex_backward.argtypes
    L.wect_maxheight.argtypes = [vp, i64, i32, vp, i32, ctypes.POINTER(ctypes.c_double), vp]
    L.wect_sync_status.argtypes = [vp]
    L.wect_last_error.restype = ctypes.c_char_p
    L.wect_repair_count.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
    for f in ("wect_complex", "ecf_complex", "wect_images", "ecf_images", "wect_complex_backward", "ecf_complex_backward", "wect_maxheight", "wect_sync_status", "wect_repair_count"):
        getattr(L, f).restype = ctypes.c_int
    L.wect_stats.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                             ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    L.wect_stats.restype = ctypes.c_int
    L.wect_abi_version.restype = ctypes.c_int32
    _L = L
    return L


def check(status: int) -> None:
    if status != OK:
        raise WectError(status, load().wect_last_error().decode())
