"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module. It wraps

* ``oracle/liboracle.so``      — the C restatement (tatn_oracle.c), always built
                                 by ``__graft_entry__.build()``; and
* ``oracle/_ref/libtatn_ref.so`` — the reference's own sources compiled by
                                 oracle/Makefile (present when built in the
                                 container that has /root/reference).

Every array is fp64, row-major, per (batch, head) slice, matching the
reference's per-head ``tatn::Matrix`` carrier (matrix.hpp:14-54).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libtatn_ref.so"

MASK_NONE, MASK_CAUSAL, MASK_KEY_PADDING = 0, 1, 2
MASK_CUSTOM = 3
MASK_CODES = {"none": MASK_NONE, "causal": MASK_CAUSAL, "key_padding": MASK_KEY_PADDING, "custom": MASK_CUSTOM}

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_ip = ctypes.POINTER(ctypes.c_int)
_u64p = ctypes.POINTER(ctypes.c_uint64)


class OrcCfg(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int),
        ("nk", ctypes.c_int),
        ("d", ctypes.c_int),
        ("tau", ctypes.c_double),
        ("mask_kind", ctypes.c_int),
        ("valid_len", ctypes.c_int),
        ("grid", ctypes.c_void_p),
        ("br", ctypes.c_int),
        ("bc", ctypes.c_int),
        ("tr", ctypes.c_int),
        ("tc", ctypes.c_int),
        ("p_drop", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("custom", ctypes.c_void_p),
        ("custom_stride", ctypes.c_longlong),
    ]


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


_lib = None
_ref = None


def build() -> None:
    """Compile oracle/liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", os.fspath(HERE)], check=True)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = ctypes.CDLL(os.fspath(LIB))
        pc = ctypes.POINTER(OrcCfg)
        L.orc_gaussian_matrix.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _dp]
        L.orc_dropout_scale.argtypes = [ctypes.c_uint64, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_double]
        L.orc_dropout_scale.restype = ctypes.c_double
        L.orc_forward_rows.argtypes = [pc, _dp, _dp, _dp, _dp, _dp, _ip, ctypes.c_int]
        L.orc_forward_rows.restype = ctypes.c_int
        L.orc_forward_batch.argtypes = [pc, ctypes.c_int, _ip, _dp, _dp, _dp, _dp, _dp, ctypes.c_int, ctypes.c_int]
        L.orc_forward_batch.restype = ctypes.c_int
        L.orc_backward_batch.argtypes = [pc, ctypes.c_int, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                         ctypes.c_int, ctypes.c_int]
        L.orc_backward_batch.restype = ctypes.c_int
        L.orc_backward_dq_rows.argtypes = [pc, _dp, _dp, _dp, _dp, _dp, _dp, _ip, ctypes.c_int, _dp]
        L.orc_backward_dq_rows.restype = ctypes.c_int
        L.orc_block_mask_butterfly.argtypes = [ctypes.c_int, ctypes.c_int, _u8p]
        L.orc_block_mask_butterfly.restype = ctypes.c_int
        L.orc_block_mask_local_global.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u8p]
        L.orc_block_mask_local_global.restype = ctypes.c_int
        u = ctypes.c_ulonglong
        L.orc_plan_tiles.argtypes = [u, u, u, ctypes.c_longlong, ctypes.c_longlong, ctypes.POINTER(u)]
        L.orc_plan_tiles.restype = ctypes.c_int
        for name in ("orc_predict_standard_forward_io", "orc_predict_standard_backward_io"):
            getattr(L, name).argtypes = [u, u, ctypes.POINTER(u)]
        for name in ("orc_predict_flash_forward_io", "orc_predict_flash_backward_io"):
            getattr(L, name).argtypes = [u, u, u, ctypes.POINTER(u)]
        for name in ("orc_predict_blocksparse_io", "orc_predict_blocksparse_backward_io"):
            getattr(L, name).argtypes = [u, u, u, u, ctypes.POINTER(u)]
        L.orc_flop_model.argtypes = [ctypes.c_int, u, u, u, u]
        L.orc_flop_model.restype = u
        L.orc_working_set_elems.argtypes = [u, u, u]
        L.orc_working_set_elems.restype = u
        _lib = L
    return _lib


def have_ref() -> bool:
    return REF_LIB.exists()


def ref() -> ctypes.CDLL:
    """The reference's own implementation (oracle/_ref); raises if not built."""
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference at build time)")
        R = ctypes.CDLL(os.fspath(REF_LIB))
        i, d_ = ctypes.c_int, ctypes.c_double
        R.ref_gaussian_matrix.argtypes = [i, i, ctypes.c_uint64, _dp]
        R.ref_standard_forward.argtypes = [i, i, i, d_, i, i, _u8p, i, i, i, d_, ctypes.c_uint64, _dp, _dp, _dp, _dp,
                                           _dp, _dp, _dp, _u64p]
        R.ref_standard_forward.restype = i
        R.ref_standard_backward.argtypes = [i, i, i, d_, i, i, _u8p, i, i, i, d_, ctypes.c_uint64, _dp, _dp, _dp, _dp,
                                            _dp, _dp, _dp, _u64p]
        R.ref_dropout_scale.argtypes = [ctypes.c_uint64, ctypes.c_longlong, ctypes.c_longlong, d_]
        R.ref_dropout_scale.restype = d_
        R.ref_standard_backward.restype = i
        R.ref_memeff_forward.argtypes = [i, i, i, d_, i, i, _dp, _dp, _dp, _dp, _dp]
        R.ref_memeff_forward.restype = i
        R.ref_memeff_backward.argtypes = [i, i, i, d_, i, i, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        R.ref_memeff_backward.restype = i
        R.ref_time_fwd_bwd.argtypes = [i, i, i, i, i, i]
        R.ref_time_fwd_bwd.restype = ctypes.c_double
        R.ref_write_matrix.argtypes = [ctypes.c_char_p, i, i, i, _dp]
        R.ref_write_matrix.restype = i
        R.ref_read_matrix.argtypes = [ctypes.c_char_p, i, ctypes.POINTER(i), ctypes.POINTER(i), _dp, ctypes.c_longlong]
        R.ref_read_matrix.restype = i
        _ref = R
    return _ref


# ----------------------------------------------------------------------------- inputs
def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """tatn::gaussian_matrix (random.cpp:25-30), restated in C."""
    out = np.empty((rows, cols), dtype=np.float64)
    lib().orc_gaussian_matrix(rows, cols, seed, _ptr(out))
    return out


def slice_seed(b: int, h: int, H: int, which: int) -> int:
    """seed = 1000 + 4*(b*H + h) + {0: Q, 1: K, 2: V, 3: dO}."""
    return 1000 + 4 * (b * H + h) + which


def gaussian_inputs(B: int, H: int, Nq: int, Nk: int, d: int):
    """Q, K, V, dO as [B, H, N, d] fp64 from the reference generator."""
    q = np.empty((B, H, Nq, d)); k = np.empty((B, H, Nk, d)); v = np.empty((B, H, Nk, d)); do = np.empty((B, H, Nq, d))
    for b in range(B):
        for h in range(H):
            q[b, h] = gaussian_matrix(Nq, d, slice_seed(b, h, H, 0))
            k[b, h] = gaussian_matrix(Nk, d, slice_seed(b, h, H, 1))
            v[b, h] = gaussian_matrix(Nk, d, slice_seed(b, h, H, 2))
            do[b, h] = gaussian_matrix(Nq, d, slice_seed(b, h, H, 3))
    return q, k, v, do


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp64 to bf16 / fp16 with round-to-nearest-even, returned as fp64."""
    if dtype == "fp16":
        return x.astype(np.float16).astype(np.float64)
    if dtype == "bf16":
        f = x.astype(np.float32)
        u = f.view(np.uint32).astype(np.uint64)
        nan = np.isnan(f)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        r = u.astype(np.uint32).view(np.float32).astype(np.float64)
        r[nan] = np.nan
        return r
    if dtype in ("fp32", "f32"):
        return x.astype(np.float32).astype(np.float64)
    raise ValueError(dtype)


# ----------------------------------------------------------------------------- attention
def _custom_u8(custom, shape):
    """Custom keep-mask (True/1 = keep) broadcast to `shape` as contiguous uint8 (kept alive by the caller)."""
    if custom is None:
        return None
    return np.ascontiguousarray(np.broadcast_to(np.asarray(custom).astype(np.uint8), shape))


def _cfg(Nq, Nk, d, tau, mask, valid_len, grid, br, bc, p_drop=0.0, seed=0, custom=None, custom_stride=0):
    c = OrcCfg()
    if custom is not None:
        c.custom, c.custom_stride = custom.ctypes.data, int(custom_stride)
    c.p_drop, c.seed = float(p_drop), int(seed)
    c.n, c.nk, c.d = Nq, Nk, d
    c.tau = tau if tau is not None else 1.0 / math.sqrt(d)
    c.mask_kind = MASK_CODES[mask] if isinstance(mask, str) else int(mask)
    c.valid_len = int(valid_len) if valid_len is not None else Nk
    if grid is not None:
        c.grid = grid.ctypes.data
        c.br, c.bc = br, bc
        c.tr, c.tc = grid.shape
    return c


def _contig(*arrs):
    return [np.ascontiguousarray(a, dtype=np.float64) for a in arrs]


def forward(q, k, v, tau=None, mask="none", valid_len=None, grid=None, br=128, bc=128, threads=None, p_drop=0.0, seed=0,
            custom=None):
    """O, LSE for q [B,H,Nq,d], k/v [B,H,Nk,d]. valid_len: per-batch array or scalar.
    Dropout: slice (b, h) uses seed + b*H + h, the C ABI's batched convention.
    custom (mask="custom"): keep-mask broadcastable to [B, H, Nq, Nk] (True = keep)."""
    q, k, v = _contig(q, k, v)
    B, H, Nq, d = q.shape
    Nk = k.shape[2]
    if grid is not None:
        grid = np.ascontiguousarray(grid, dtype=np.uint8)
    cu = _custom_u8(custom, (B, H, Nq, Nk))
    c = _cfg(Nq, Nk, d, tau, mask, None, grid, br, bc, p_drop, seed, cu, Nq * Nk)
    vl = None
    if valid_len is not None:
        vl = np.ascontiguousarray(np.broadcast_to(np.asarray(valid_len, dtype=np.int32).reshape(-1, 1), (B, H)).reshape(-1))
    o = np.empty_like(q)
    lse = np.empty((B, H, Nq))
    rc = lib().orc_forward_batch(ctypes.byref(c), B * H, _ptr(vl, _ip) if vl is not None else None, _ptr(q), _ptr(k),
                                 _ptr(v), _ptr(o), _ptr(lse), threads or os.cpu_count() or 1, 1)
    if rc != 0:
        raise RuntimeError("orc_forward_batch failed")
    return o, lse


def forward_rows(q, k, v, rows, tau=None, mask="none", valid_len=None, grid=None, br=128, bc=128, custom=None):
    """Forward on one slice (q [Nq,d]) restricted to the given query rows."""
    q, k, v = _contig(q, k, v)
    Nq, d = q.shape
    Nk = k.shape[0]
    if grid is not None:
        grid = np.ascontiguousarray(grid, dtype=np.uint8)
    cu = _custom_u8(custom, (Nq, Nk))
    c = _cfg(Nq, Nk, d, tau, mask, valid_len, grid, br, bc, custom=cu)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    o = np.zeros_like(q)
    lse = np.zeros(Nq)
    rc = lib().orc_forward_rows(ctypes.byref(c), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(rows, _ip),
                                len(rows))
    if rc != 0:
        raise RuntimeError("orc_forward_rows failed")
    return o[rows], lse[rows]


def backward_dq_rows(q, k, v, o_rows, do, lse_rows, rows, tau=None, mask="none", valid_len=None, grid=None, br=128,
                     bc=128, custom=None):
    """dQ for the given query rows of one slice; o_rows / lse_rows are those rows' forward outputs."""
    q, k, v, o_rows, do, lse_rows = _contig(q, k, v, o_rows, do, lse_rows)
    Nq, d = q.shape
    Nk = k.shape[0]
    if grid is not None:
        grid = np.ascontiguousarray(grid, dtype=np.uint8)
    cu = _custom_u8(custom, (Nq, Nk))
    c = _cfg(Nq, Nk, d, tau, mask, valid_len, grid, br, bc, custom=cu)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    out = np.empty((len(rows), d))
    lib().orc_backward_dq_rows(ctypes.byref(c), _ptr(q), _ptr(k), _ptr(v), _ptr(o_rows), _ptr(do), _ptr(lse_rows),
                               _ptr(rows, _ip), len(rows), _ptr(out))
    return out


def backward(q, k, v, o, do, lse, tau=None, mask="none", valid_len=None, grid=None, br=128, bc=128, threads=None, p_drop=0.0, seed=0,
             custom=None):
    """dQ, dK, dV from the saved (o, lse) — Algorithm 4 semantics in fp64."""
    q, k, v, o, do, lse = _contig(q, k, v, o, do, lse)
    B, H, Nq, d = q.shape
    Nk = k.shape[2]
    if grid is not None:
        grid = np.ascontiguousarray(grid, dtype=np.uint8)
    cu = _custom_u8(custom, (B, H, Nq, Nk))
    c = _cfg(Nq, Nk, d, tau, mask, None, grid, br, bc, p_drop, seed, cu, Nq * Nk)
    vl = None
    if valid_len is not None:
        vl = np.ascontiguousarray(np.broadcast_to(np.asarray(valid_len, dtype=np.int32).reshape(-1, 1), (B, H)).reshape(-1))
    dq = np.empty_like(q)
    dk = np.empty_like(k)
    dv = np.empty_like(v)
    rc = lib().orc_backward_batch(ctypes.byref(c), B * H, _ptr(vl, _ip) if vl is not None else None, _ptr(q), _ptr(k),
                                  _ptr(v), _ptr(o), _ptr(do), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                                  threads or os.cpu_count() or 1, 1)
    if rc != 0:
        raise RuntimeError("orc_backward_batch failed")
    return dq, dk, dv


def dropout_scale(seed: int, i: int, j: int, p: float) -> float:
    """tatn::dropout_scale (dropout.cpp:22-27), restated in C."""
    return float(lib().orc_dropout_scale(seed, i, j, p))


def dropout_mask(seed: int, rows: int, cols: int, p: float) -> np.ndarray:
    """tatn::dropout_mask_matrix (dropout.cpp:29-35) via the C restatement (vectorised over numpy)."""
    m = np.empty((rows, cols))
    for i in range(rows):
        for j in range(cols):
            m[i, j] = dropout_scale(seed, i, j, p)
    return m


# ----------------------------------------------------------------------------- block masks / plans / IO
def block_mask_butterfly(tr: int, tc: int) -> np.ndarray:
    g = np.empty((tr, tc), dtype=np.uint8)
    lib().orc_block_mask_butterfly(tr, tc, _ptr(g, _u8p))
    return g


def block_mask_local_global(window: int, globals_: int, tr: int, tc: int) -> np.ndarray:
    g = np.empty((tr, tc), dtype=np.uint8)
    lib().orc_block_mask_local_global(window, globals_, tr, tc, _ptr(g, _u8p))
    return g


def plan_tiles(n: int, d: int, m: int, br: int = 0, bc: int = 0):
    out = (ctypes.c_ulonglong * 6)()
    rc = lib().orc_plan_tiles(n, d, m, br, bc, out)
    keys = ("bc", "br", "tr", "tc", "m_capacity", "working_set")
    return rc, dict(zip(keys, list(out)))


def predict_io(kind: str, n: int, d: int, tc: int = 0, br: int = 0, visited: int = 0):
    out = (ctypes.c_ulonglong * 2)()
    L = lib()
    if kind == "standard_forward":
        L.orc_predict_standard_forward_io(n, d, out)
    elif kind == "standard_backward":
        L.orc_predict_standard_backward_io(n, d, out)
    elif kind == "flash_forward":
        L.orc_predict_flash_forward_io(n, d, tc, out)
    elif kind == "flash_backward":
        L.orc_predict_flash_backward_io(n, d, tc, out)
    elif kind == "blocksparse_forward":
        L.orc_predict_blocksparse_io(n, d, br, visited, out)
    elif kind == "blocksparse_backward":
        L.orc_predict_blocksparse_backward_io(n, d, br, visited, out)
    else:
        raise ValueError(kind)
    return int(out[0]), int(out[1])


def flop_model(algo: int, n: int, d: int, tr: int = 0, tc: int = 0) -> int:
    return int(lib().orc_flop_model(algo, n, d, tr, tc))


# ----------------------------------------------------------------------------- reference (oracle/_ref)
def ref_gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols))
    ref().ref_gaussian_matrix(rows, cols, seed, _ptr(out))
    return out


def ref_write_matrix(path, m: np.ndarray, binary: bool) -> None:
    """The reference's write_matrix_binary / write_matrix_csv (matrix_io.cpp:116-172)."""
    a = np.ascontiguousarray(m, dtype=np.float64)
    if ref().ref_write_matrix(os.fspath(path).encode(), int(binary), a.shape[0], a.shape[1], _ptr(a)) != 0:
        raise RuntimeError(f"reference matrix write failed: {path}")


def ref_read_matrix(path, binary: bool, capacity: int = 1 << 22) -> np.ndarray:
    """The reference's read_matrix_binary / read_matrix_csv; raises on the reference's errors."""
    out = np.empty(capacity, dtype=np.float64)
    r, c = ctypes.c_int(0), ctypes.c_int(0)
    st = ref().ref_read_matrix(os.fspath(path).encode(), int(binary), ctypes.byref(r), ctypes.byref(c), _ptr(out),
                               capacity)
    if st != 0:
        raise RuntimeError(f"reference matrix read failed ({st}): {path}")
    return out[: r.value * c.value].reshape(r.value, c.value).copy()


def ref_dropout_scale(seed: int, i: int, j: int, p: float) -> float:
    return float(ref().ref_dropout_scale(seed, i, j, p))


def ref_standard(q, k, v, do=None, tau=None, mask="none", valid_len=None, grid=None, br=128, bc=128, p_drop=0.0,
                 seed=0, custom=None):
    """The reference's standard_forward (+ standard_backward) on one slice.
    Returns dict with o, lse, m, l, fwd_counters (+ dq, dk, dv, bwd_counters).
    mask="custom": `custom` is the [n, nk] keep matrix (MaskSpec::custom_additive)."""
    q, k, v = _contig(q, k, v)
    n, d = q.shape
    nk = k.shape[0]
    tau = tau if tau is not None else 1.0 / math.sqrt(d)
    mk = MASK_CODES[mask] if isinstance(mask, str) else int(mask)
    vl = int(valid_len) if valid_len is not None else nk
    if mk == MASK_CUSTOM:
        grid = np.ascontiguousarray(np.broadcast_to(np.asarray(custom).astype(np.uint8), (n, nk)))
    g = np.ascontiguousarray(grid, dtype=np.uint8) if grid is not None else None
    tc = nk if mk == MASK_CUSTOM else (g.shape[1] if g is not None else 0)
    gp = _ptr(g, _u8p) if g is not None else None
    o = np.empty_like(q)
    lse = np.empty(n); m = np.empty(n); l = np.empty(n)
    ctr = np.zeros(3, dtype=np.uint64)
    R = ref()
    rc = R.ref_standard_forward(n, nk, d, tau, mk, vl, gp, br, bc, tc, p_drop, seed, _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                _ptr(lse), _ptr(m), _ptr(l), _ptr(ctr, _u64p))
    if rc != 0:
        raise ValueError("reference standard_forward threw")
    out = {"o": o, "lse": lse, "m": m, "l": l, "fwd_counters": ctr.copy()}
    if do is not None:
        (do,) = _contig(do)
        dq = np.empty_like(q); dk = np.empty_like(k); dv = np.empty_like(v)
        ctr2 = np.zeros(3, dtype=np.uint64)
        rc = R.ref_standard_backward(n, nk, d, tau, mk, vl, gp, br, bc, tc, p_drop, seed, _ptr(q), _ptr(k), _ptr(v),
                                     _ptr(do), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ctr2, _u64p))
        if rc != 0:
            raise ValueError("reference standard_backward threw")
        out.update(dq=dq, dk=dk, dv=dv, bwd_counters=ctr2)
    return out


def ref_time_fwd_bwd(nslices: int, n: int, d: int, mask: str, memeff: bool, threads: int) -> float:
    return float(ref().ref_time_fwd_bwd(nslices, n, d, MASK_CODES[mask], 1 if memeff else 0, threads))
