"""The C-ABI library loads, exports every symbol include/tatn_b200.h declares,
and rejects bad descriptors with the reference's error classes (CPU only: no
compute entry point is called)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2205_14135_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "tatn_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tatn_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_bound_symbols():
    assert declared_functions() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_exports_have_c_linkage():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in declared_functions():
        assert name in exported, f"{name} is not exported unmangled"


def test_abi_version_and_strerror():
    lib = _lib.load()
    assert lib.tatn_abi_version() == 4
    for code in range(7):
        assert _lib.strerror(code)
    assert _lib.strerror(99) == "unknown status"


def good_desc(**kw):
    d = _lib.TatnAttnDesc()
    d.B, d.H, d.Nq, d.Nk, d.d = 2, 3, 300, 300, 64
    d.dtype = _lib.TATN_DTYPE_BF16
    for name in ("q_str", "k_str", "v_str", "o_str"):
        getattr(d, name)[:] = (3 * 300 * 64, 300 * 64, 64)
    d.tau = 0.125
    d.mask_kind = _lib.TATN_MASK_NONE
    d.tr, d.tc = 3, 3
    for key, val in kw.items():
        setattr(d, key, val)
    return d


def validate(d):
    return _lib.load().tatn_validate(ctypes.byref(d))


def test_valid_descriptor_passes():
    assert validate(good_desc()) == _lib.TATN_OK
    assert validate(good_desc(d=128, dtype=_lib.TATN_DTYPE_FP16, mask_kind=_lib.TATN_MASK_CAUSAL)) == _lib.TATN_OK
    # ABI v4: fp32 inputs select the tf32 check mode
    assert validate(good_desc(dtype=_lib.TATN_DTYPE_FP32)) == _lib.TATN_OK
    assert validate(good_desc(d=128, dtype=_lib.TATN_DTYPE_FP32, out_dtype=_lib.TATN_OUT_FP32)) == _lib.TATN_OK


def test_forward_workspace():
    """ABI v4: the forward's work-item counter lives in a caller-owned 16-byte workspace (no
    global state in the library); too small / misaligned / missing workspaces are rejected
    before any device access."""
    lib = _lib.load()
    d = good_desc()
    assert lib.tatn_fwd_workspace_bytes(ctypes.byref(d)) == 16
    assert lib.tatn_fwd_workspace_bytes(ctypes.byref(good_desc(B=0))) == 0
    buf = (ctypes.c_uint8 * 64)()
    base = (ctypes.addressof(buf) + 15) // 16 * 16
    one = ctypes.c_void_p(base)  # never dereferenced: the calls fail validation first
    st = lib.tatn_fwd(ctypes.byref(d), one, one, one, one, one, None, 16, None)
    assert st == _lib.TATN_E_ARG
    st = lib.tatn_fwd(ctypes.byref(d), one, one, one, one, one, base, 8, None)
    assert st == _lib.TATN_E_WORKSPACE
    st = lib.tatn_fwd(ctypes.byref(d), one, one, one, one, one, base + 4, 16, None)
    assert st == _lib.TATN_E_ARG
    # tensor base pointers must be 16-byte aligned (TMA tiles, 16-byte vector accesses)
    odd = ctypes.c_void_p(base + 2)
    st = lib.tatn_fwd(ctypes.byref(d), one, odd, one, one, one, base, 16, None)
    assert st == _lib.TATN_E_ARG
    st = lib.tatn_bwd(ctypes.byref(d), one, one, odd, one, one, one, one, one, one, base, 1 << 30, None)
    assert st == _lib.TATN_E_ARG


@pytest.mark.parametrize(
    "kw, code",
    [
        (dict(B=0), _lib.TATN_E_SHAPE),
        (dict(Nq=0), _lib.TATN_E_SHAPE),
        (dict(H=65536), _lib.TATN_E_SHAPE),  # K2 / K4 grid dimension (rows, H, B)
        (dict(B=65536), _lib.TATN_E_SHAPE),
        (dict(Nk=301), _lib.TATN_E_SHAPE),  # more keys than n (reference.cpp:25-26)
        (dict(d=32), _lib.TATN_E_UNSUPPORTED),
        (dict(dtype=7), _lib.TATN_E_UNSUPPORTED),
        (dict(tau=0.0), _lib.TATN_E_ARG),  # tau must be finite and > 0 (attn_config.cpp:52)
        (dict(tau=float("inf")), _lib.TATN_E_ARG),
        (dict(tau=float("nan")), _lib.TATN_E_ARG),
        (dict(p_drop=1.0), _lib.TATN_E_ARG),  # p in [0, 1) (attn_config.cpp:54)
        (dict(p_drop=-0.1), _lib.TATN_E_ARG),
        (dict(mask_kind=3), _lib.TATN_E_ARG),  # Custom without its mask
        (dict(mask_kind=9), _lib.TATN_E_ARG),  # not a MaskKind
        (dict(mask_kind=_lib.TATN_MASK_KEY_PADDING), _lib.TATN_E_ARG),  # no valid_len
    ],
)
def test_invalid_descriptors(kw, code):
    assert validate(good_desc(**kw)) == code


def test_bad_strides_rejected():
    d = good_desc()
    d.q_str[2] = 65  # rows must be 16-byte aligned for TMA
    assert validate(d) == _lib.TATN_E_SHAPE


def test_block_grid_must_match_plan():
    buf = (ctypes.c_uint8 * 9)()
    d = good_desc(block_grid=ctypes.addressof(buf), br=128, bc=128, tr=3, tc=3)
    assert validate(d) == _lib.TATN_OK
    assert validate(good_desc(block_grid=ctypes.addressof(buf), br=64, bc=128, tr=3, tc=3)) == _lib.TATN_E_MASK
    assert validate(good_desc(block_grid=ctypes.addressof(buf), br=128, bc=128, tr=2, tc=3)) == _lib.TATN_E_MASK


def test_null_descriptor():
    assert _lib.load().tatn_validate(None) == _lib.TATN_E_ARG


def test_workspace_formula():
    lib = _lib.load()
    d = good_desc()
    rows = 2 * 3 * 384  # Nq padded to a multiple of 128
    assert lib.tatn_bwd_workspace_bytes(ctypes.byref(d)) == rows * 64 * 4 + 2 * rows * 4 + 16
    assert lib.tatn_bwd_workspace_bytes(ctypes.byref(good_desc(B=0))) == 0


def test_deterministic_workspace_and_flag():
    lib = _lib.load()
    d = good_desc()
    base = lib.tatn_bwd_workspace_bytes(ctypes.byref(d))
    d.deterministic = 1
    rows = 2 * 3 * 384
    assert lib.tatn_bwd_workspace_bytes(ctypes.byref(d)) == base + 3 * rows * 64 * 4  # tc = 3 key tiles
    assert validate(good_desc(deterministic=2)) == _lib.TATN_E_ARG


def test_custom_mask_descriptor():
    buf = (ctypes.c_uint32 * (300 * 12 + 4))()
    base = (ctypes.addressof(buf) + 15) // 16 * 16
    ok = good_desc(mask_kind=_lib.TATN_MASK_CUSTOM, custom_mask=base, custom_words=12)
    assert validate(ok) == _lib.TATN_OK
    # words must cover Nk (ceil(300/32) = 10, rounded to a multiple of 4 = 12) and be 16-byte multiples
    assert validate(good_desc(mask_kind=3, custom_mask=base, custom_words=8)) == _lib.TATN_E_MASK
    assert validate(good_desc(mask_kind=3, custom_mask=base, custom_words=10)) == _lib.TATN_E_MASK
    assert validate(good_desc(mask_kind=3, custom_mask=base + 4, custom_words=12)) == _lib.TATN_E_ARG
    # a per-batch stride smaller than one Nq x words mask overlaps
    assert validate(good_desc(mask_kind=3, custom_mask=base, custom_words=12, custom_bstride=100)) == _lib.TATN_E_MASK
    assert validate(good_desc(mask_kind=3, custom_mask=base, custom_words=12, custom_bstride=3600)) == _lib.TATN_OK
    # the backward workspace adds the transposed mask [B or 1][Nk][Nq_pad/32]
    lib = _lib.load()
    rows = 2 * 3 * 384
    base_ws = rows * 64 * 4 + 2 * rows * 4 + 16
    assert lib.tatn_bwd_workspace_bytes(ctypes.byref(ok)) == base_ws + 300 * 12 * 4
    per_b = good_desc(mask_kind=3, custom_mask=base, custom_words=12, custom_bstride=3600)
    assert lib.tatn_bwd_workspace_bytes(ctypes.byref(per_b)) == base_ws + 2 * 300 * 12 * 4


def test_custom_mask_width_covers_key_offset():
    """The kernels read word (k_offset + j) / 32 of each row: a key shard at k_offset needs
    4 * ceil((k_offset + Nk) / 128) words, not ceil(Nk / 32) (advisor finding, round 1)."""
    buf = (ctypes.c_uint32 * (1024 * 32 + 4))()
    base = (ctypes.addressof(buf) + 15) // 16 * 16
    kw = dict(B=1, H=1, Nq=1024, Nk=128, tr=8, tc=1, mask_kind=3, custom_mask=base)
    d = good_desc(**kw, k_offset=768, custom_words=4)
    for name in ("q_str", "k_str", "v_str", "o_str"):
        getattr(d, name)[:] = (1024 * 64, 1024 * 64, 64)
    assert validate(d) == _lib.TATN_E_MASK
    d.custom_words = 28  # 4 * ceil((768 + 128) / 128)
    assert validate(d) == _lib.TATN_OK
    d.custom_bstride = 1024 * 4  # a per-batch stride must hold Nq rows of the full width
    assert validate(d) == _lib.TATN_E_MASK
