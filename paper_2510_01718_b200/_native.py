"""ctypes binding of the C ABI in include/bd_kv_proj.h (libbd_kvproj.so, in-tree).

This is the Python side of the drop-in boundary: plain pointers, sizes and a
cudaStream_t cross it, no torch types.  Loading fails loudly (NativeLibraryError)
when the library is missing — there is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import NativeLibraryError, PrecisionError, ShapeError

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libbd_kvproj.so"
if os.environ.get("BD_LIB_PATH"):  # development aid: load an experimental build
    LIB_PATH = Path(os.environ["BD_LIB_PATH"])

# enum bd_dtype / bd_status / bd_mode / bd_tag  (include/bd_kv_proj.h)
BD_F32, BD_F64, BD_F16, BD_BF16 = 0, 1, 2, 3
BD_OK, BD_ERR_SHAPE, BD_ERR_DTYPE, BD_ERR_ALIGN, BD_ERR_CUDA, BD_ERR_ARG = 0, 1, 2, 3, 4, 5
BD_MODE_AUTO, BD_MODE_EXACT, BD_MODE_TC = 0, 1, 2
BD_MAX_GROUP = 4
ABI_VERSION = 6
BD_MAX_PEERS = 8
BD_OUT_TOKEN_MAJOR, BD_OUT_HEAD_MAJOR = 0, 1
BD_TAG_FIRST, BD_TAG_LAST = 0, 1

EXPORTED_SYMBOLS = (
    "bd_kv_proj",
    "bd_kv_proj_grouped",
    "bd_kv_proj_grouped_ex",
    "bd_kv_proj_grouped_allgather",
    "bd_kv_proj_grouped_rmsnorm",
    "bd_kv_proj_host",
    "bd_matmul",
    "bd_linear_forward",
    "bd_mla_attention",
    "bd_last_error",
    "bd_abi_version",
    "bd_launch_count",
)


class KvProblem(ctypes.Structure):
    """struct bd_kv_problem."""

    _fields_ = [
        ("x", ctypes.c_void_p),
        ("c", ctypes.c_void_p),
        ("out", ctypes.c_void_p),
        ("ldx", ctypes.c_int64),
        ("ldc", ctypes.c_int64),
        ("ldo", ctypes.c_int64),
        ("L", ctypes.c_int64),
        ("d", ctypes.c_int64),
        ("d_h", ctypes.c_int64),
        ("n_heads", ctypes.c_int64),
        ("mul_base", ctypes.c_int64),
        ("rep_base", ctypes.c_int64),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the C ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryError(
            f"{LIB_PATH} is missing; build it with `python -m paper_2510_01718_b200.build` "
            "(there is no CPU fallback)")
    try:
        lib = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
    i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    lib.bd_kv_proj.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, i64, i64, i64, ci, ci,
                               vp, vp]
    lib.bd_kv_proj.restype = ci
    lib.bd_kv_proj_grouped.argtypes = [ctypes.POINTER(KvProblem), ci, ci, ci, vp, vp]
    lib.bd_kv_proj_grouped.restype = ci
    lib.bd_kv_proj_grouped_ex.argtypes = [ctypes.POINTER(KvProblem), ci, ci, ci, ci, vp, vp]
    lib.bd_kv_proj_grouped_ex.restype = ci
    lib.bd_kv_proj_grouped_allgather.argtypes = [ctypes.POINTER(KvProblem), ci, ci, ci, ci, ci,
                                                 ctypes.POINTER(vp), vp, vp]
    lib.bd_kv_proj_grouped_allgather.restype = ci
    lib.bd_kv_proj_grouped_rmsnorm.argtypes = [ctypes.POINTER(KvProblem), ci, ci, ci, ci,
                                               ctypes.POINTER(vp), ctypes.c_float, vp, vp]
    lib.bd_kv_proj_grouped_rmsnorm.restype = ci
    lib.bd_kv_proj_host.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, ci, ci,
                                    ctypes.POINTER(ctypes.c_int)]
    lib.bd_kv_proj_host.restype = ci
    lib.bd_matmul.argtypes = [vp, i64, vp, i64, vp, i64, i64, i64, i64, ci, ci, vp, vp]
    lib.bd_matmul.restype = ci
    lib.bd_linear_forward.argtypes = [vp, i64, vp, i64, vp, i64, vp, i64, i64, i64, i64, i64, ci,
                                      ci, ci, vp, vp]
    lib.bd_linear_forward.restype = ci
    lib.bd_mla_attention.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, vp, i64, i64, vp, i64,
                                     i64, i64, i64, i64, i64, i64, ctypes.c_float, ci, ci, vp]
    lib.bd_mla_attention.restype = ci
    lib.bd_last_error.argtypes = []
    lib.bd_last_error.restype = ctypes.c_char_p
    lib.bd_abi_version.argtypes = []
    lib.bd_abi_version.restype = ci
    lib.bd_launch_count.argtypes = []
    lib.bd_launch_count.restype = ctypes.c_uint64
    if lib.bd_abi_version() != ABI_VERSION:
        raise NativeLibraryError(
            f"ABI mismatch: library {lib.bd_abi_version()} vs binding {ABI_VERSION}")
    _lib = lib
    return lib


def last_error() -> str:
    return load().bd_last_error().decode("utf-8", "replace")


def check(status: int, what: str) -> None:
    """Map a bd_status to the reference's exception types."""
    if status == BD_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == BD_ERR_SHAPE:
        raise ShapeError(msg)
    if status == BD_ERR_DTYPE:
        raise PrecisionError(msg)
    if status == BD_ERR_ALIGN:
        raise ShapeError(msg)
    if status == BD_ERR_ARG:
        raise ValueError(msg)
    raise NativeLibraryError(msg)


def launch_count() -> int:
    return int(load().bd_launch_count())
