"""Block masks at the reference's own block sizes (BlockMask with any br x bc, block_mask.hpp:14-24;
SPEC.md:245, :275) lowered onto the kernels' 128 x 128 tiles (attention.lower_block_mask), checked
on the CPU against a brute-force expansion: a tile is visited iff a true block overlaps it, and when a
visited tile is only partly covered the element keep bits are exactly compose_block_mask(base, grid)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2205_14135_b200 import attention as A


def brute(grid, br, bc, Nq, Nk):
    el = grid[np.arange(Nq)[:, None] // br, np.arange(Nk)[None, :] // bc] != 0
    tr, tc = (Nq + 127) // 128, (Nk + 127) // 128
    tiles = np.zeros((tr, tc), np.uint8)
    for i in range(tr):
        for j in range(tc):
            tiles[i, j] = el[128 * i:128 * i + 128, 128 * j:128 * j + 128].any()
    return el, tiles


def unpack(words, Nk):
    w = np.asarray(words).view(np.uint32)
    bits = (w[..., :, :, None] >> np.arange(32, dtype=np.uint32)) & 1
    return bits.reshape(*w.shape[:-1], -1)[..., :Nk].astype(bool)


CASES = [  # Nq, Nk, br, bc, pattern, base mask
    (1024, 1024, 64, 256, "butterfly", "causal"),  # the reference's default plan at N = 1024, d = 64
    (300, 300, 16, 16, "local", "none"),
    (160, 150, 1, 1, "random", "key_padding"),
    (200, 200, 200, 200, "random", "none"),  # one block covering everything
    (256, 256, 32, 64, "butterfly", "custom"),
    (512, 512, 256, 256, "butterfly", "causal"),  # multiples of 128: exact tiles, no element mask
]


@pytest.mark.parametrize("Nq,Nk,br,bc,pattern,base", CASES)
def test_lowering_matches_brute_force(Nq, Nk, br, bc, pattern, base):
    trb, tcb = (Nq + br - 1) // br, (Nk + bc - 1) // bc
    rng = np.random.default_rng(br * 7 + bc)
    if pattern == "butterfly":
        grid = O.block_mask_butterfly(trb, tcb)
    elif pattern == "local":
        grid = O.block_mask_local_global(1, 1, trb, tcb)
    else:
        grid = (rng.random((trb, tcb)) < 0.5).astype(np.uint8)
    spec = A.AttnSpec(mask=base, block_grid=torch.from_numpy(np.ascontiguousarray(grid, dtype=np.uint8)),
                      block_size=(br, bc))
    B = 2
    base_keep = np.ones((B, Nq, Nk), bool)
    if base == "causal":
        base_keep &= np.arange(Nk)[None, None, :] <= np.arange(Nq)[None, :, None]
    elif base == "key_padding":
        vl = np.array([Nk - 7, 3], np.int32)
        spec.valid_len = torch.from_numpy(vl)
        base_keep &= np.arange(Nk)[None, None, :] < vl[:, None, None]
    elif base == "custom":
        keep = rng.random((Nq, Nk)) < 0.7
        spec.custom = A.pack_custom_mask(torch.from_numpy(keep))
        base_keep &= keep[None]
    low = A.lower_block_mask(spec, B, Nq, Nk)
    el, tiles = brute(grid, br, bc, Nq, Nk)
    assert np.array_equal(low.block_grid.numpy(), tiles)
    assert low.block_size == (128, 128)
    exact = all(el[128 * i:128 * i + 128, 128 * j:128 * j + 128].all() or not tiles[i, j]
                for i in range(tiles.shape[0]) for j in range(tiles.shape[1]))
    if exact:
        assert low.mask == base  # the base mask stays; the tile grid is the whole story
    else:
        assert low.mask == "custom"
        got = unpack(low.custom.numpy(), Nk)
        want = el[None] & base_keep
        if got.ndim == 2:
            got = np.broadcast_to(got, want.shape)
        assert np.array_equal(got, want)
    again = A.lower_block_mask(spec, B, Nq, Nk)  # the lowered grid / bits are cached on the spec
    assert again.block_grid is low.block_grid and again.custom is low.custom


def test_lowering_is_identity_at_128():
    g = torch.ones((2, 2), dtype=torch.uint8)
    spec = A.AttnSpec(block_grid=g)
    assert A.lower_block_mask(spec, 1, 256, 256) is spec


def test_lowering_rejects_a_grid_that_does_not_cover():
    spec = A.AttnSpec(block_grid=torch.ones((3, 3), dtype=torch.uint8), block_size=(64, 64))
    with pytest.raises(ValueError):
        A.lower_block_mask(spec, 1, 256, 256)
