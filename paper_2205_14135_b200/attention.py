"""Device-side batched API over the C ABI (torch tensors as device buffers).

This is the "batched device API" of SURVEY.md §8(b)(ii): the bench and the GPU
parity tests call it; it only packs a ``tatn_attn_desc`` and passes raw device
pointers plus the current CUDA stream to ``libtatn_b200.so``. PyTorch provides
memory and streams only — no attention math happens here.

Tensor layout: ``[B, H, N, d]`` with ``d`` contiguous (any b/h/n strides that
are multiples of 8 elements), dtype bf16 or fp16 (the throughput path) or fp32
(the tf32 check mode: fp32 outputs), on an sm_100 device.
LSE is ``[B, H, Nq]`` fp32 (natural log).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, replace
from typing import Optional

import torch

from . import _lib

MASK_KINDS = {
    "none": _lib.TATN_MASK_NONE,
    "causal": _lib.TATN_MASK_CAUSAL,
    "key_padding": _lib.TATN_MASK_KEY_PADDING,
    "custom": _lib.TATN_MASK_CUSTOM,
}


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.TATN_DTYPE_BF16
    if t.dtype == torch.float16:
        return _lib.TATN_DTYPE_FP16
    if t.dtype == torch.float32:
        return _lib.TATN_DTYPE_FP32
    raise TypeError(f"unsupported dtype {t.dtype}: the sm_100a path takes bf16, fp16 or fp32 (tf32 check mode)")


def out_dtype(q: torch.Tensor, spec: "AttnSpec") -> torch.dtype:
    """dtype of O / dQ / dK / dV: fp32 for fp32 inputs or spec.out_fp32, else the input dtype."""
    return torch.float32 if (spec.out_fp32 or q.dtype == torch.float32) else q.dtype


def _strides(t: torch.Tensor, name: str):
    if t.dim() != 4:
        raise ValueError(f"{name} must be [B, H, N, d], got shape {tuple(t.shape)}")
    if t.stride(3) != 1:
        raise ValueError(f"{name} must be contiguous in d")
    return (t.stride(0), t.stride(1), t.stride(2))


@dataclass
class AttnSpec:
    tau: Optional[float] = None
    mask: str = "none"
    valid_len: Optional[torch.Tensor] = None  # int32 [B] on device (key_padding)
    # block-sparse grid (tatn::BlockMask::grid, block_mask.hpp:14-24): uint8 [tr, tc] on the device over
    # blocks of block_size = (br, bc) rows x keys — any block size, e.g. the reference's default plan
    # (64, 256) at N = 1024, d = 64; (128, 128) is the kernels' native tile (no lowering)
    block_grid: Optional[torch.Tensor] = None
    block_size: tuple = (128, 128)
    visited: Optional[torch.Tensor] = None  # int32 [ceil(tr*tc/32)] on device, zeroed by caller
    out_fp32: bool = False  # write O / dQ / dK / dV in fp32 (no output rounding)
    p_drop: float = 0.0  # dropout probability in [0, 1) (reference's positional PRNG, dropout.cpp)
    seed: int = 0  # dropout seed; slice (b, h) uses seed + b*H + h
    k_offset: int = 0  # key shard: key j is global key k_offset + j (sequence parallel; multiple of 128)
    # dQ summed over key tiles in a fixed order (bit-reproducible; all-true grid == dense exactly);
    # the backward workspace grows by ceil(Nk/128) x the dQ accumulator
    deterministic: bool = False
    # mask="custom": bit-packed keep matrix from pack_custom_mask(), int32 [Nq, words] shared
    # by every slice or [B, Nq, words] per batch element (MaskSpec::custom_additive)
    custom: Optional[torch.Tensor] = None


def pack_custom_mask(keep: torch.Tensor) -> torch.Tensor:
    """Bit-pack a boolean keep matrix [..., Nq, Nk] (True = additive 0, False = -inf) into the
    C ABI's custom_mask layout: int32 words [..., Nq, words], bit (j & 31) of word j >> 5,
    words = ceil(Nk / 32) rounded up to a multiple of 4 (16-byte rows). Runs on keep's device."""
    if keep.dtype != torch.bool:
        keep = keep != 0
    *lead, nq, nk = keep.shape
    words = (nk + 127) // 128 * 4
    padded = torch.zeros(*lead, nq, words * 32, dtype=torch.int64, device=keep.device)
    padded[..., :nk] = keep.to(torch.int64)
    bits = padded.view(*lead, nq, words, 32) << torch.arange(32, device=keep.device, dtype=torch.int64)
    packed = bits.sum(-1)  # < 2^32
    return torch.where(packed >= 2**31, packed - 2**32, packed).to(torch.int32).contiguous()


def _check_vec(t, name, dtype, n, device):
    if t.dtype != dtype or t.dim() != 1 or t.numel() < n or not t.is_contiguous() or t.device != device:
        raise ValueError(f"{name} must be a contiguous {dtype} vector of >= {n} elements on {device}, got "
                         f"{t.dtype} {tuple(t.shape)} on {t.device}")


def _rect_sums(grid: torch.Tensor, br: int, bc: int, Nq: int, Nk: int):
    """Per 128 x 128 tile (I, J): the number of true blocks overlapping it and the number of blocks
    overlapping it (2-D prefix sums over the block grid)."""
    dev = grid.device
    tr, tc = (Nq + 127) // 128, (Nk + 127) // 128
    S = torch.zeros((grid.shape[0] + 1, grid.shape[1] + 1), dtype=torch.int64, device=dev)
    S[1:, 1:] = (grid != 0).to(torch.int64).cumsum(0).cumsum(1)
    I = torch.arange(tr, device=dev)
    J = torch.arange(tc, device=dev)
    r_lo, r_hi = (128 * I) // br, (torch.clamp(128 * I + 128, max=Nq) - 1) // br + 1
    c_lo, c_hi = (128 * J) // bc, (torch.clamp(128 * J + 128, max=Nk) - 1) // bc + 1
    rl, rh, cl, ch = r_lo[:, None], r_hi[:, None], c_lo[None, :], c_hi[None, :]
    true = S[rh, ch] - S[rl, ch] - S[rh, cl] + S[rl, cl]
    return true, (rh - rl) * (ch - cl)


def _block_keep_bits(grid: torch.Tensor, br: int, bc: int, Nq: int, Nk: int) -> torch.Tensor:
    """Bit-packed element keep matrix [Nq, words] of a block grid: bit j of row i = grid[i // br, j // bc]
    (compose_block_mask, block_mask.hpp:42-46), built per block row and gathered per query row."""
    dev = grid.device
    words = (Nk + 127) // 128 * 4
    j = torch.arange(words * 32, device=dev)
    colblk = torch.clamp(j // bc, max=grid.shape[1] - 1)
    per_blockrow = (grid[:, colblk] != 0) & (j < Nk)[None, :]  # [tr_b, words * 32]
    bits = per_blockrow.view(grid.shape[0], words, 32).to(torch.int64) << torch.arange(32, device=dev)
    packed = bits.sum(-1)
    packed = torch.where(packed >= 2**31, packed - 2**32, packed).to(torch.int32)
    return packed[torch.arange(Nq, device=dev) // br].contiguous()


def _base_keep_bits(spec: "AttnSpec", B: int, Nq: int, Nk: int, device) -> Optional[torch.Tensor]:
    """The base mask as keep bits [Nq, words] or [B, Nq, words] (None for mask='none')."""
    words = (Nk + 127) // 128 * 4
    w0 = torch.arange(words, device=device, dtype=torch.int64) * 32
    full = (1 << 32) - 1

    def prefix_bits(limit):  # keep keys j < limit (limit broadcast against w0)
        n = torch.clamp(limit - w0, 0, 32)
        v = torch.where(n >= 32, torch.full_like(n, full), (torch.ones_like(n) << n) - 1)
        return torch.where(v >= 2**31, v - 2**32, v).to(torch.int32)

    if spec.mask == "none":
        return None
    if spec.mask == "causal":  # keep k_offset + j <= i
        i = torch.arange(Nq, device=device, dtype=torch.int64)[:, None]
        return prefix_bits(i + 1 - int(spec.k_offset)).contiguous()
    if spec.mask == "key_padding":
        vl = spec.valid_len.to(torch.int64)[:, None, None] - int(spec.k_offset)
        return prefix_bits(vl).expand(B, Nq, words).contiguous()
    if spec.mask == "custom":
        return spec.custom
    raise ValueError(f"unknown mask kind {spec.mask!r}")


def lower_block_mask(spec: "AttnSpec", B: int, Nq: int, Nk: int) -> "AttnSpec":
    """A block grid at any block size (br, bc) -> the kernels' 128 x 128 tile grid (tile visited iff a
    true block overlaps it) plus, when some visited tile is only partly covered by true blocks, the
    blocks' element pattern intersected with the base mask as a Custom keep-bit mask (mask folded
    in: the result is exactly compose_block_mask(base, grid)). Cached on the spec."""
    br, bc = (int(x) for x in spec.block_size)
    if spec.block_grid is None or (br, bc) == (128, 128):
        return spec
    ptr = lambda t: t.data_ptr() if t is not None else 0
    key = (ptr(spec.block_grid), br, bc, B, Nq, Nk, spec.mask, spec.k_offset, ptr(spec.valid_len), ptr(spec.custom))
    cached = getattr(spec, "_lowered", None)
    if cached is None or cached[0] != key:  # the lowered grid / bits are cached; the spec's other fields are not
        g = spec.block_grid
        if br < 1 or bc < 1 or g.shape[0] * br < Nq or g.shape[1] * bc < Nk:
            raise ValueError(f"block grid {tuple(g.shape)} x ({br}, {bc}) does not cover Nq={Nq}, Nk={Nk}")
        true, total = _rect_sums(g, br, bc, Nq, Nk)
        tiles = (true > 0).to(torch.uint8).contiguous()
        bits = None
        if bool(((true > 0) & (true < total)).any()):  # partly covered tiles: element pattern needed
            bits = _block_keep_bits(g, br, bc, Nq, Nk)
            base = _base_keep_bits(spec, B, Nq, Nk, g.device)
            if base is not None:
                bits = (bits & base).contiguous()
        cached = (key, tiles, bits)
        object.__setattr__(spec, "_lowered", cached)
    _, tiles, bits = cached
    if bits is None:
        return replace(spec, block_grid=tiles, block_size=(128, 128))
    return replace(spec, block_grid=tiles, block_size=(128, 128), mask="custom", custom=bits, valid_len=None)


def check_shapes(q, k, v, o=None):
    """The buffer shapes a descriptor is built from must agree: q [B, H, Nq, d], k and v
    [B, H, Nk, d], o (if given) like q. The ABI sees only the descriptor, so a mismatch here would
    let the kernels read or write past a buffer."""
    for name, t in (("q", q), ("k", k), ("v", v)) + ((("o", o),) if o is not None else ()):
        if t.dim() != 4:
            raise ValueError(f"{name} must be [B, H, N, d], got shape {tuple(t.shape)}")
    B, H, Nq, d = q.shape
    Nk = k.shape[2]
    if tuple(k.shape) != (B, H, Nk, d):
        raise ValueError(f"k shape {tuple(k.shape)} does not match q {tuple(q.shape)} (expected [B, H, Nk, d])")
    if tuple(v.shape) != tuple(k.shape):
        raise ValueError(f"v shape {tuple(v.shape)} != k shape {tuple(k.shape)}")
    if o is not None and tuple(o.shape) != tuple(q.shape):
        raise ValueError(f"o shape {tuple(o.shape)} != q shape {tuple(q.shape)}")
    return B, H, Nq, Nk, d


def make_desc(q, k, v, o, spec: AttnSpec, check_o: bool = True) -> _lib.TatnAttnDesc:
    """Pack a tatn_attn_desc, checking every shape / dtype / device the ABI cannot see (a
    descriptor that disagrees with the buffers would let the kernels read or write out of
    bounds)."""
    B, H, Nq, Nk, d = check_shapes(q, k, v, o if check_o else None)
    for name, t in (("q", q), ("k", k), ("v", v)) + ((("o", o),) if check_o else ()):
        if t.device != q.device or t.device.type != "cuda":
            raise ValueError(f"{name} must be a CUDA tensor on {q.device}, got {t.device}")
    spec = lower_block_mask(spec, B, Nq, Nk)
    desc = _lib.TatnAttnDesc()
    desc.B, desc.H, desc.Nq, desc.Nk, desc.d = B, H, Nq, Nk, d
    desc.dtype = _dtype_code(q)
    for t in (k, v):
        if t.dtype != q.dtype:
            raise TypeError("q, k, v must share one dtype")
    out_dt = out_dtype(q, spec)
    if check_o and o.dtype != out_dt:
        raise TypeError(f"o must be {out_dt} (input {q.dtype}, out_fp32={spec.out_fp32})")
    desc.out_dtype = _lib.TATN_OUT_FP32 if spec.out_fp32 else _lib.TATN_OUT_INPUT_DTYPE
    desc.q_str[:] = _strides(q, "q")
    desc.k_str[:] = _strides(k, "k")
    desc.v_str[:] = _strides(v, "v")
    desc.o_str[:] = _strides(o, "o")
    desc.tau = float(spec.tau) if spec.tau is not None else 1.0 / math.sqrt(d)
    if spec.mask not in MASK_KINDS:
        raise ValueError(f"unknown mask kind {spec.mask!r}")
    desc.mask_kind = MASK_KINDS[spec.mask]
    if spec.valid_len is not None:
        _check_vec(spec.valid_len, "valid_len", torch.int32, B, q.device)
    elif spec.mask == "key_padding":
        raise ValueError("mask='key_padding' needs spec.valid_len (int32 [B] on the device)")
    desc.valid_len = spec.valid_len.data_ptr() if spec.valid_len is not None else None
    tr, tc = (Nq + 127) // 128, (Nk + 127) // 128
    if spec.block_grid is not None:
        g = spec.block_grid
        if g.dtype != torch.uint8 or g.dim() != 2 or not g.is_contiguous() or g.device != q.device:
            raise ValueError("block_grid must be a contiguous uint8 [tr, tc] tensor on q's device")
        desc.block_grid = spec.block_grid.data_ptr()
        desc.br = desc.bc = 128
        desc.tr, desc.tc = spec.block_grid.shape
    else:
        desc.block_grid = None
        desc.tr, desc.tc = tr, tc
    if spec.visited is not None:
        _check_vec(spec.visited, "visited", torch.int32, (tr * tc + 31) // 32, q.device)
    desc.visited_bitmap = spec.visited.data_ptr() if spec.visited is not None else None
    desc.p_drop = float(spec.p_drop)
    desc.seed = int(spec.seed) & 0xFFFFFFFFFFFFFFFF
    desc.k_offset = int(spec.k_offset)
    desc.deterministic = 1 if spec.deterministic else 0
    if spec.mask == "custom":
        cm = spec.custom
        if (cm is None or cm.dtype != torch.int32 or cm.dim() not in (2, 3) or not cm.is_contiguous()
                or cm.device != q.device):
            raise ValueError("mask='custom' needs spec.custom = pack_custom_mask(keep) ([Nq, w] or [B, Nq, w] int32)")
        if cm.shape[-2] != Nq or (cm.dim() == 3 and cm.shape[0] != B):
            raise ValueError(f"custom mask shape {tuple(cm.shape)} does not match B={B}, Nq={Nq}")
        desc.custom_mask = cm.data_ptr()
        desc.custom_words = cm.shape[-1]
        desc.custom_bstride = cm.stride(0) if cm.dim() == 3 else 0
    else:
        desc.custom_mask = None
    return desc


def _check(status: int, what: str):
    if status != _lib.TATN_OK:
        raise _lib.TatnError(status, what)


FWD_WORKSPACE_BYTES = 16  # tatn_fwd_workspace_bytes() of every valid descriptor


def fwd_workspace(device) -> torch.Tensor:
    """A zeroed forward workspace (the persistent kernels' work-item counter, ABI v4). Every
    tatn_fwd leaves it zero again, so one workspace serves any number of calls that do not run
    concurrently (one per stream / per concurrently replayed graph)."""
    return torch.zeros(FWD_WORKSPACE_BYTES, dtype=torch.uint8, device=device)


def flash_fwd(q, k, v, spec: Optional[AttnSpec] = None, out=None, lse=None, stream=None, workspace=None):
    """O, LSE = attention forward (kernel K1) on device tensors. `workspace`: a zeroed
    fwd_workspace() reused across sequential calls (default: a fresh one per call)."""
    spec = spec or AttnSpec()
    lib = _lib.load()
    B, H, Nq, d = q.shape
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype(q, spec), device=q.device)
    if lse is None:
        lse = torch.empty((B, H, Nq), dtype=torch.float32, device=q.device)
    if lse.dtype != torch.float32 or tuple(lse.shape) != (B, H, Nq) or not lse.is_contiguous() or lse.device != q.device:
        raise ValueError(f"lse must be a contiguous fp32 [B, H, Nq] = {(B, H, Nq)} tensor on {q.device}")
    desc = make_desc(q, k, v, out, spec)
    if workspace is None:
        workspace = fwd_workspace(q.device)
    if workspace.device != q.device or workspace.numel() < FWD_WORKSPACE_BYTES:
        raise ValueError("workspace must be a >= 16-byte fwd_workspace() on q's device")
    s = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    st = lib.tatn_fwd(ctypes.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                      lse.data_ptr(), workspace.data_ptr(), workspace.numel(), s)
    _check(st, "tatn_fwd")
    return out, lse


def bwd_workspace(q, k, v, spec: Optional[AttnSpec] = None) -> torch.Tensor:
    spec = spec or AttnSpec()
    lib = _lib.load()
    desc = make_desc(q, k, v, q, spec, check_o=False)
    n = lib.tatn_bwd_workspace_bytes(ctypes.byref(desc))
    if n == 0:
        _check(lib.tatn_validate(ctypes.byref(desc)), "tatn_bwd_workspace_bytes")
    return torch.empty(n, dtype=torch.uint8, device=q.device)


def flash_bwd(q, k, v, o, dO, lse, spec: Optional[AttnSpec] = None, dq=None, dk=None, dv=None,
              workspace=None, stream=None):
    """dQ, dK, dV = attention backward (kernels K2-K4) on device tensors."""
    spec = spec or AttnSpec()
    lib = _lib.load()
    if dO.dtype != q.dtype:
        raise TypeError("dO must have the input dtype")
    if tuple(dO.shape) != tuple(q.shape) or tuple(o.shape) != tuple(q.shape):
        raise ValueError(f"o {tuple(o.shape)} and dO {tuple(dO.shape)} must have q's shape {tuple(q.shape)}")
    B, H, Nq, _ = q.shape
    if lse.dtype != torch.float32 or tuple(lse.shape) != (B, H, Nq) or not lse.is_contiguous() or lse.device != q.device:
        raise ValueError(f"lse must be a contiguous fp32 [B, H, Nq] = {(B, H, Nq)} tensor on {q.device}")
    if dO.stride() != o.stride():
        fixed = torch.empty_strided(o.shape, o.stride(), dtype=dO.dtype, device=dO.device)
        fixed.copy_(dO)
        dO = fixed
    gdt = out_dtype(q, spec)
    mk = lambda t: torch.empty_strided(t.shape, t.stride(), dtype=gdt, device=t.device)
    dq = mk(q) if dq is None else dq
    dk = mk(k) if dk is None else dk
    dv = mk(v) if dv is None else dv
    for t in (dq, dk, dv):
        if t.dtype != gdt:
            raise TypeError(f"gradients must be {gdt}")
    if dq.stride() != q.stride() or dk.stride() != k.stride() or dv.stride() != v.stride():
        raise ValueError("dq/dk/dv must have the strides of q/k/v")
    desc = make_desc(q, k, v, o, spec)
    if workspace is None:
        workspace = bwd_workspace(q, k, v, spec)
    if workspace.device != q.device:
        raise ValueError("workspace must be on q's device")
    s = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
    st = lib.tatn_bwd(ctypes.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                      dO.data_ptr(), lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                      workspace.data_ptr(), workspace.numel(), s)
    _check(st, "tatn_bwd")
    return dq, dk, dv


def last_launch_count() -> int:
    return _lib.load().tatn_last_launch_count()


def merge_partials(o_parts: torch.Tensor, lse_parts: torch.Tensor, out: Optional[torch.Tensor] = None,
                   lse: Optional[torch.Tensor] = None, stream=None):
    """Combine R partial (O_r, LSE_r) over disjoint key shards into (O, LSE) with the
    reference's merge_stats algebra (softmax.cpp:62-83), on the device (tatn_merge_partials).
    o_parts: fp32 [R, B, H, Nq, d] contiguous; lse_parts: fp32 [R, B, H, Nq]. out: fp32 /
    bf16 / fp16 [B, H, Nq, d] (default fp32)."""
    lib = _lib.load()
    if o_parts.dtype != torch.float32 or lse_parts.dtype != torch.float32:
        raise TypeError("partials must be fp32 (tatn_fwd with out_fp32=True)")
    if not (o_parts.is_contiguous() and lse_parts.is_contiguous()):
        raise ValueError("partials must be contiguous [R, B, H, Nq, d] / [R, B, H, Nq]")
    R, B, H, Nq, d = o_parts.shape
    if tuple(lse_parts.shape) != (R, B, H, Nq):
        raise ValueError(f"lse_parts shape {tuple(lse_parts.shape)} != {(R, B, H, Nq)}")
    if out is None:
        out = torch.empty((B, H, Nq, d), dtype=torch.float32, device=o_parts.device)
    if lse is None:
        lse = torch.empty((B, H, Nq), dtype=torch.float32, device=o_parts.device)
    code = {torch.bfloat16: _lib.TATN_DTYPE_BF16, torch.float16: _lib.TATN_DTYPE_FP16,
            torch.float32: _lib.TATN_DTYPE_FP32}[out.dtype]
    st = (ctypes.c_int64 * 3)(*_strides(out, "out"))
    s = stream if stream is not None else torch.cuda.current_stream(o_parts.device).cuda_stream
    _check(lib.tatn_merge_partials(R, B, H, Nq, d, o_parts.data_ptr(), lse_parts.data_ptr(), out.data_ptr(), code,
                                   st, lse.data_ptr(), ctypes.c_void_p(s)), "tatn_merge_partials")
    return out, lse
