"""ctypes binding of the C ABI declared in include/tatn_b200.h.

The shared library ``paper_2205_14135_b200/lib/libtatn_b200.so`` is built
in-tree by ``__graft_entry__.build()`` (or ``make -C paper_2205_14135_b200``).
There is no fallback: if the library is missing this module raises on import
of any compute entry point.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# TATN_B200_LIB may point at an alternative in-tree build (tuning experiments); default is the product library
LIB_PATH = Path(os.environ.get("TATN_B200_LIB", _PKG / "lib" / "libtatn_b200.so"))

ABI_VERSION = 4  # TATN_B200_ABI_VERSION (include/tatn_b200.h)

TATN_OK = 0
TATN_E_ARG = 1
TATN_E_SHAPE = 2
TATN_E_MASK = 3
TATN_E_UNSUPPORTED = 4
TATN_E_CUDA = 5
TATN_E_WORKSPACE = 6

TATN_DTYPE_BF16 = 0
TATN_DTYPE_FP16 = 1
TATN_DTYPE_FP32 = 2  # fp32 inputs (tf32 check mode); also a tatn_merge_partials output type

TATN_OUT_INPUT_DTYPE = 0
TATN_OUT_FP32 = 1

TATN_MASK_NONE = 0
TATN_MASK_CAUSAL = 1
TATN_MASK_KEY_PADDING = 2
TATN_MASK_CUSTOM = 3

# every symbol include/tatn_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTED_SYMBOLS = (
    "tatn_validate",
    "tatn_fwd_workspace_bytes",
    "tatn_fwd",
    "tatn_bwd_workspace_bytes",
    "tatn_bwd",
    "tatn_strerror",
    "tatn_abi_version",
    "tatn_last_launch_count",
    "tatn_profile_enable",
    "tatn_profile_read",
    "tatn_merge_partials",
)


class TatnAttnDesc(ctypes.Structure):
    """Mirror of ``tatn_attn_desc`` (include/tatn_b200.h)."""

    _fields_ = [
        ("B", ctypes.c_int32),
        ("H", ctypes.c_int32),
        ("Nq", ctypes.c_int32),
        ("Nk", ctypes.c_int32),
        ("d", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("q_str", ctypes.c_int64 * 3),
        ("k_str", ctypes.c_int64 * 3),
        ("v_str", ctypes.c_int64 * 3),
        ("o_str", ctypes.c_int64 * 3),
        ("tau", ctypes.c_float),
        ("mask_kind", ctypes.c_int32),
        ("valid_len", ctypes.c_void_p),
        ("block_grid", ctypes.c_void_p),
        ("br", ctypes.c_int32),
        ("bc", ctypes.c_int32),
        ("tr", ctypes.c_int32),
        ("tc", ctypes.c_int32),
        ("visited_bitmap", ctypes.c_void_p),
        ("p_drop", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("custom_mask", ctypes.c_void_p),
        ("custom_words", ctypes.c_int32),
        ("custom_bstride", ctypes.c_int64),
        ("k_offset", ctypes.c_int32),
        ("deterministic", ctypes.c_int32),
    ]


class TatnError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {strerror(status)} (status {status})")


_lib = None


def load() -> ctypes.CDLL:
    """Load the C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the attention path)"
        )
    lib = ctypes.CDLL(os.fspath(LIB_PATH))
    vp = ctypes.c_void_p
    pd = ctypes.POINTER(TatnAttnDesc)
    lib.tatn_validate.argtypes = [pd]
    lib.tatn_validate.restype = ctypes.c_int
    lib.tatn_fwd_workspace_bytes.argtypes = [pd]
    lib.tatn_fwd_workspace_bytes.restype = ctypes.c_size_t
    lib.tatn_fwd.argtypes = [pd, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.tatn_fwd.restype = ctypes.c_int
    lib.tatn_bwd_workspace_bytes.argtypes = [pd]
    lib.tatn_bwd_workspace_bytes.restype = ctypes.c_size_t
    lib.tatn_bwd.argtypes = [pd, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.tatn_bwd.restype = ctypes.c_int
    lib.tatn_strerror.argtypes = [ctypes.c_int]
    lib.tatn_strerror.restype = ctypes.c_char_p
    lib.tatn_abi_version.argtypes = []
    lib.tatn_abi_version.restype = ctypes.c_int
    if lib.tatn_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {lib.tatn_abi_version()} != {ABI_VERSION} (stale build?)")
    lib.tatn_last_launch_count.argtypes = []
    lib.tatn_last_launch_count.restype = ctypes.c_int
    if hasattr(lib, "tatn_debug_set_trace"):  # -DTATN_TRACE builds only
        lib.tatn_debug_set_trace.argtypes = [ctypes.c_void_p]
        lib.tatn_debug_set_trace.restype = ctypes.c_int
    lib.tatn_profile_enable.argtypes = [ctypes.c_int]
    lib.tatn_profile_enable.restype = ctypes.c_int
    lib.tatn_profile_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)]
    lib.tatn_profile_read.restype = ctypes.c_int
    i32 = ctypes.c_int32
    lib.tatn_merge_partials.argtypes = [i32, i32, i32, i32, i32, vp, vp, vp, i32, ctypes.POINTER(ctypes.c_int64), vp, vp]
    lib.tatn_merge_partials.restype = ctypes.c_int
    _lib = lib
    return lib


def profile_enable(on: bool) -> None:
    load().tatn_profile_enable(1 if on else 0)


def profile_read(which: int):
    """(total device ms, launches) of the main kernel (0 = forward K1, 1 = backward K3)."""
    ms = ctypes.c_double()
    n = ctypes.c_int()
    st = load().tatn_profile_read(which, ctypes.byref(ms), ctypes.byref(n))
    if st != TATN_OK:
        raise TatnError(st, "tatn_profile_read")
    return ms.value, n.value


def strerror(status: int) -> str:
    return load().tatn_strerror(status).decode()
