"""Tile plan and IO / FLOP closed forms of the reference (product side).

Restates, for the drop-in's bookkeeping and the bench's IO-complexity bound:
  * plan_tiles / working_set_elems          tile_plan.hpp:8-52 (tile_plan.cpp is absent)
  * predict_*_io, flop_model                 io_predict.hpp:12-106 (io_predict.cpp is absent)
All counts are in ELEMENTS, as the reference's MemoryModel counts them.
tests/test_iomodel.py pins these against the oracle and the reference's own
instrumented counters.
"""
from __future__ import annotations

from dataclasses import dataclass

SRAM_SLACK_FORWARD = 1.5   # kSramSlackForward (tile_plan.hpp:14)
SRAM_SLACK_BACKWARD = 3.0  # kSramSlackBackward (tile_plan.hpp:15)


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def working_set_elems(br: int, bc: int, d: int) -> int:
    """K/V blocks, Q/O blocks, one score buffer and six stat vectors (tile_plan.hpp:30-37)."""
    return 2 * bc * d + 2 * br * d + br * bc + 6 * br


def backward_working_set_elems(br: int, bc: int, d: int) -> int:
    return 4 * bc * d + 4 * br * d + 2 * br * bc + 3 * br


@dataclass
class TilePlan:
    bc: int
    br: int
    tr: int
    tc: int
    m_capacity: int
    working_set: int


def plan_tiles(n: int, d: int, m_capacity: int, br: int = 0, bc: int = 0) -> TilePlan:
    """Bc = ceil(M/4d), Br = min(Bc, d), both clamped to n (tile_plan.hpp:43-52).
    Raises ValueError like the reference's std::invalid_argument."""
    if m_capacity < 4 * d:
        raise ValueError(f"plan_tiles: M={m_capacity} < 4d={4 * d}")
    bc = bc or _cdiv(m_capacity, 4 * d)
    br = br or min(bc, d)
    bc, br = min(bc, n), min(br, n)
    ws = working_set_elems(br, bc, d)
    if ws > SRAM_SLACK_FORWARD * m_capacity:
        raise ValueError(f"plan_tiles: working set {ws} exceeds {SRAM_SLACK_FORWARD}*M")
    return TilePlan(bc, br, _cdiv(n, br), _cdiv(n, bc), m_capacity, ws)


def predict_standard_forward_io(n: int, d: int):
    return 3 * n * d + 4 * n * n, 2 * n * n + n * d


def predict_standard_backward_io(n: int, d: int):
    return 7 * n * n + 5 * n * d, 2 * n * n + 3 * n * d


def predict_flash_forward_io(n: int, d: int, plan: TilePlan):
    tc = plan.tc
    return 2 * n * d + tc * (2 * n * d + 2 * n), (n * d + 2 * n) + tc * (n * d + 2 * n)


def predict_flash_backward_io(n: int, d: int, plan: TilePlan):
    tc = plan.tc
    return 2 * n * d + tc * (4 * n * d + 2 * n), n * d + tc * n * d + 2 * n * d


def predict_blocksparse_io(n: int, d: int, plan: TilePlan, visited: int):
    br = plan.br
    return 2 * n * d + visited * (2 * br * d + 2 * br), (n * d + 2 * n) + visited * (br * d + 2 * br)


def predict_blocksparse_backward_io(n: int, d: int, plan: TilePlan, visited: int):
    br = plan.br
    return 2 * n * d + visited * (4 * br * d + 2 * br), n * d + visited * br * d + 2 * n * d


def flop_model(algo: str, n: int, d: int, plan: TilePlan = None) -> int:
    if algo == "standard_forward":
        return 4 * n * n * d + 5 * n * n
    if algo == "standard_backward":
        return 8 * n * n * d + 4 * n * n + 2 * n * d
    if algo == "flash_forward":
        return 4 * n * n * d + 5 * n * n + plan.tc * (2 * n * d + 7 * n)
    if algo == "flash_backward":
        return 10 * n * n * d + 5 * n * n + 4 * plan.tc * n * d + 2 * plan.tr * n * d
    raise ValueError(algo)


# ---------------------------------------------------------------------------- B200 figures
SMEM_BYTES_PER_CTA = 227 * 1024  # M = 227 KiB of SMEM


def theorem2_bound_bytes(n: int, d: int, elem_bytes: int, slices: int, backward: bool) -> int:
    """The paper's IO-complexity figure (Theorem 2 via the reference's closed forms) with
    M = one CTA's shared memory in elements, times the number of (b, h) slices, in bytes."""
    m = SMEM_BYTES_PER_CTA // elem_bytes
    plan = plan_tiles(n, d, m)
    r, w = (predict_flash_backward_io if backward else predict_flash_forward_io)(n, d, plan)
    return (r + w) * elem_bytes * slices


def compulsory_bytes(n: int, d: int, elem_bytes: int, slices: int, backward: bool, out_bytes: int = None) -> int:
    """Minimum DRAM traffic: read Q, K, V (+ O, dO, LSE) and write O, LSE (or dQ, dK, dV)."""
    out_bytes = out_bytes or elem_bytes
    e = n * d
    if not backward:
        return slices * (3 * e * elem_bytes + e * out_bytes + 4 * n)
    return slices * (4 * e * elem_bytes + e * out_bytes + 4 * n + 3 * e * out_bytes)
