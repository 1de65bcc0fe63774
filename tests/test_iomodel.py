"""Product-side tile plan / IO closed forms (paper_2205_14135_b200/iomodel.py)
against the oracle restatement and SPEC known answers (CPU)."""
import pytest

from oracle import oracle as O
from paper_2205_14135_b200 import iomodel as M


@pytest.mark.parametrize("n,d,m", [(1024, 64, 65536), (1024, 64, 1024), (64, 16, 4096), (2048, 128, 116224),
                                   (16384, 128, 116224), (1, 1, 4)])
def test_plan_matches_oracle(n, d, m):
    rc, ref = O.plan_tiles(n, d, m)
    if rc == 0:
        p = M.plan_tiles(n, d, m)
        assert (p.bc, p.br, p.tr, p.tc, p.working_set) == (ref["bc"], ref["br"], ref["tr"], ref["tc"], ref["working_set"])
    else:
        with pytest.raises(ValueError):
            M.plan_tiles(n, d, m)


def test_spec_plan_example():
    p = M.plan_tiles(1024, 64, 65536)
    assert (p.bc, p.br, p.tc, p.tr) == (256, 64, 4, 16)


@pytest.mark.parametrize("n,d", [(1024, 64), (512, 64), (2048, 128)])
def test_io_closed_forms_match_oracle(n, d):
    plan = M.plan_tiles(n, d, 65536)
    assert M.predict_standard_forward_io(n, d) == O.predict_io("standard_forward", n, d)
    assert M.predict_standard_backward_io(n, d) == O.predict_io("standard_backward", n, d)
    assert M.predict_flash_forward_io(n, d, plan) == O.predict_io("flash_forward", n, d, tc=plan.tc)
    assert M.predict_flash_backward_io(n, d, plan) == O.predict_io("flash_backward", n, d, tc=plan.tc)
    v = plan.tr * plan.tc // 3
    assert M.predict_blocksparse_io(n, d, plan, v) == O.predict_io("blocksparse_forward", n, d, br=plan.br, visited=v)
    assert M.predict_blocksparse_backward_io(n, d, plan, v) == O.predict_io("blocksparse_backward", n, d,
                                                                              br=plan.br, visited=v)
    for algo, code in (("standard_forward", 0), ("standard_backward", 1), ("flash_forward", 2),
                       ("flash_backward", 3)):
        assert M.flop_model(algo, n, d, plan) == O.flop_model(code, n, d, plan.tr, plan.tc)


def test_spec_counter_anchor():
    assert M.predict_standard_forward_io(1024, 64) == (4390912, 2162688)


def test_theorem2_bound_examples():
    # C2 forward ~153.7 MB, C4 N=16K forward ~30.1 GB (M = 227 KiB / 2 B)
    c2 = M.theorem2_bound_bytes(1024, 64, 2, 8 * 12, backward=False)
    assert 150e6 < c2 < 157e6
    c4 = M.theorem2_bound_bytes(16384, 128, 2, 32, backward=False)
    assert 29e9 < c4 < 31e9
