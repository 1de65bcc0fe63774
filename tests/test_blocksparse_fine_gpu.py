"""GPU parity of block-sparse attention at the reference's own block sizes (BlockMask with any
br x bc, block_mask.hpp:14-24; blocksparse_forward requires bmask blocks == the plan's, SPEC.md:245,
whose default at N = 1024, d = 64 is br = 64, bc = 256, tile_plan.hpp:22-24). The grid is lowered
onto the kernels' 128 x 128 tiles (attention.lower_block_mask): the visited tiles must be exactly
those a true block overlaps, and the values must equal the reference semantics
(compose_block_mask: the fp64 oracle iterating the grid at (br, bc))."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import gpu_helpers as G
from paper_2205_14135_b200 import attention as A

pytestmark = pytest.mark.gpu


def expected_tiles(grid, br, bc, Nq, Nk):
    el = grid[np.arange(Nq)[:, None] // br, np.arange(Nk)[None, :] // bc] != 0
    tr, tc = (Nq + 127) // 128, (Nk + 127) // 128
    return np.array([[el[128 * i:128 * i + 128, 128 * j:128 * j + 128].any() for j in range(tc)] for i in range(tr)],
                    dtype=np.uint8)


CASES = [  # B, H, N, d, dtype, br, bc, pattern, mask
    (1, 2, 1024, 64, "bf16", 64, 256, "butterfly", "causal"),  # the reference's default plan
    (1, 2, 300, 128, "fp16", 16, 16, "local", "none"),
    (2, 2, 512, 64, "bf16", 32, 32, "random", "key_padding"),
    (1, 1, 200, 64, "bf16", 1, 1, "random", "none"),
    (1, 2, 384, 64, "fp32", 64, 64, "butterfly", "causal"),  # tf32 check mode
]


@pytest.mark.parametrize("B,H,N,d,dtype,br,bc,pattern,mask", CASES)
def test_fine_block_sparse_matches_reference_semantics(cuda_device, B, H, N, d, dtype, br, bc, pattern, mask):
    trb, tcb = (N + br - 1) // br, (N + bc - 1) // bc
    rng = np.random.default_rng(br + 13 * bc)
    if pattern == "butterfly":
        grid = O.block_mask_butterfly(trb, tcb)
    elif pattern == "local":
        grid = O.block_mask_local_global(1, 1, trb, tcb)
    else:
        grid = (rng.random((trb, tcb)) < 0.4).astype(np.uint8)
    grid = np.ascontiguousarray(grid, dtype=np.uint8)
    vl = np.array([N - 5, N // 3], np.int32)[:B] if mask == "key_padding" else None
    q, k, v, do = G.make_inputs(B, H, N, N, d, dtype)
    got = G.run_gpu(q, k, v, do, dtype, mask=mask, valid_len=vl, grid=grid, block_size=(br, bc), visited=True)
    ref = G.oracle_full(q, k, v, do, mask=mask, valid_len=vl, grid=grid, block_size=(br, bc))
    tiles = expected_tiles(grid, br, bc, N, N)
    assert np.array_equal(got["visited_fwd"], tiles)
    assert np.array_equal(got["visited_bwd"], tiles)
    tol = dict(max_abs=G.F32_MAX_ABS_STRESS, rel_l2=G.F32_REL_L2, scale_max_abs=True) if dtype == "fp32" else {}
    for key in ("o", "lse", "dq", "dk", "dv"):
        G.assert_close(key, got[key], ref[key], **tol)


def test_all_true_fine_grid_is_dense_bit_for_bit(cuda_device):
    """An all-true grid at br = bc = 64 covers every tile completely: it runs on the exact tile path
    and equals the dense engine bit for bit (flash.hpp:62-63) for O, LSE, dK, dV."""
    q, k, v, do = G.make_inputs(1, 2, 512, 512, 64, "bf16")
    grid = np.ones((8, 8), np.uint8)
    dense = G.run_gpu(q, k, v, do, "bf16", mask="causal")
    sparse = G.run_gpu(q, k, v, do, "bf16", mask="causal", grid=grid, block_size=(64, 64))
    for key in ("o", "lse", "dk", "dv"):
        assert np.array_equal(dense[key], sparse[key]), key
