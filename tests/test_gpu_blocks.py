"""GPU parity of ssa_build_blocks against oracle O1: bit-exact perm, offsets C,
block coordinates, batch ranges and the compression->selection map; error codes."""
import numpy as np
import pytest

from conftest import random_coords

pytestmark = pytest.mark.gpu


def _cmp(coords, grid, batch, sizes):
    import torch
    import oracle as O
    from paper_2505_17412_b200 import ssa
    po = O.block_build(coords, grid, batch, *sizes)
    pg = ssa.ssa_build_blocks(torch.from_numpy(coords).cuda(), grid, batch, *sizes)
    assert np.array_equal(pg.perm().cpu().numpy(), po.perm)
    for lvl, name in enumerate(("cmp", "slc", "win", "q")):
        assert pg.n_blocks[lvl] == po.n_blocks(name)
        assert np.array_equal(pg.offsets(lvl).cpu().numpy(), po.offsets[name]), name
        assert np.array_equal(pg.block_coords(lvl).cpu().numpy(), po.block_coords[name]), name
        assert np.array_equal(pg.batch_blocks(lvl).cpu().numpy(), po.batch_blocks[name]), name
        fills = np.diff(po.offsets[name])
        assert pg.max_fill[lvl] == fills.max()
    assert np.array_equal(pg.cmp_to_slc().cpu().numpy(), po.cmp_to_slc)


@pytest.mark.parametrize("sizes", [(4, 8, 8, 8), (4, 4, 4, 4), (2, 8, 4, 1), (1, 2, 2, 2)])
def test_random_coords_bit_exact(sizes):
    rng = np.random.Generator(np.random.PCG64(11))
    c = random_coords(rng, 700, 24, batch=3)
    _cmp(c, (24, 24, 24), 3, sizes)


def test_shell_and_ragged_grid():
    from ssa_workload import config_coords
    c, grid, batch = config_coords("C2")
    _cmp(c, grid, batch, (4, 8, 8, 8))
    rng = np.random.Generator(np.random.PCG64(5))
    cells = rng.choice(13 * 7 * 10, size=300, replace=False)           # grid not a multiple of m
    c = np.stack([np.zeros(300), cells // 70, (cells // 10) % 7, cells % 10], 1).astype(np.int32)
    _cmp(c, (13, 7, 10), 1, (4, 8, 8, 8))


def test_single_token_and_empty_batch_item():
    c = np.array([[1, 5, 6, 7]], dtype=np.int32)       # batch item 0 is empty
    _cmp(c, (8, 8, 8), 2, (4, 8, 8, 8))


def test_error_codes():
    import torch
    from paper_2505_17412_b200 import ssa
    dup = torch.tensor([[0, 1, 1, 1], [0, 2, 2, 2], [0, 1, 1, 1]], dtype=torch.int32).cuda()
    with pytest.raises(ssa.SSAError) as e:
        ssa.ssa_build_blocks(dup, (8, 8, 8), 1, 4, 8, 8, 8)
    assert e.value.code == "SSA_ERR_DUP_COORD"
    oor = torch.tensor([[0, 8, 1, 1]], dtype=torch.int32).cuda()
    with pytest.raises(ssa.SSAError) as e:
        ssa.ssa_build_blocks(oor, (8, 8, 8), 1, 4, 8, 8, 8)
    assert e.value.code == "SSA_ERR_COORD_RANGE"
    ok = torch.tensor([[0, 1, 1, 1]], dtype=torch.int32).cuda()
    with pytest.raises(ssa.SSAError) as e:
        ssa.ssa_build_blocks(ok, (8, 8, 8), 1, 4, 6, 6, 6)
    assert e.value.code == "SSA_ERR_HIERARCHY"


def test_empty_input():
    """N = 0 is a documented argument error (include/ssa.h): raised cleanly, nothing launched."""
    import torch
    from paper_2505_17412_b200 import ssa
    c = torch.zeros((0, 4), dtype=torch.int32).cuda()
    with pytest.raises(ssa.SSAError) as e:
        ssa.ssa_build_blocks(c, (8, 8, 8), 1, 4, 8, 8, 8)
    assert e.value.code == "SSA_ERR_ARG"
    torch.cuda.synchronize()
    # the library stays usable afterwards
    one = torch.tensor([[0, 1, 2, 3]], dtype=torch.int32).cuda()
    assert ssa.ssa_build_blocks(one, (8, 8, 8), 1, 4, 8, 8, 8).n_blocks[0] == 1
