"""Host-side checks of the Python device API (CPU: no compute call). The C ABI sees only the
descriptor, so the API must reject buffers that disagree with it (advisor finding, round 1: a
q [2,4,256,64] with k [1,1,128,64], v [1,1,64,128], o [1,1,8,64] built a descriptor the ABI
accepted, and the kernels would have read K/V and written O/LSE out of bounds)."""
import pytest
import torch

from paper_2205_14135_b200 import attention as A


def t(*shape, dtype=torch.bfloat16):
    return torch.zeros(shape, dtype=dtype)


def test_advisor_example_is_rejected():
    with pytest.raises(ValueError):
        A.check_shapes(t(2, 4, 256, 64), t(1, 1, 128, 64), t(1, 1, 64, 128), t(1, 1, 8, 64))


@pytest.mark.parametrize("q,k,v,o", [
    ((2, 4, 256, 64), (2, 4, 128, 32), (2, 4, 128, 32), None),   # head dim of k differs
    ((2, 4, 256, 64), (2, 3, 128, 64), (2, 3, 128, 64), None),   # heads differ
    ((2, 4, 256, 64), (2, 4, 128, 64), (2, 4, 127, 64), None),   # v rows differ from k
    ((2, 4, 256, 64), (2, 4, 128, 64), (2, 4, 128, 64), (2, 4, 255, 64)),  # o not like q
    ((2, 4, 256), (2, 4, 128, 64), (2, 4, 128, 64), None),       # not 4-D
])
def test_shape_mismatches_are_rejected(q, k, v, o):
    with pytest.raises(ValueError):
        A.check_shapes(t(*q), t(*k), t(*v), t(*o) if o else None)


def test_consistent_shapes_pass():
    assert A.check_shapes(t(2, 4, 256, 64), t(2, 4, 128, 64), t(2, 4, 128, 64), t(2, 4, 256, 64)) == (2, 4, 256, 128, 64)


def test_cpu_tensors_never_reach_the_abi():
    q = t(1, 1, 128, 64)
    with pytest.raises(ValueError, match="CUDA"):
        A.make_desc(q, q, q, q, A.AttnSpec())


def test_out_dtype_rules():
    spec = A.AttnSpec()
    assert A.out_dtype(t(1, 1, 8, 64), spec) == torch.bfloat16
    assert A.out_dtype(t(1, 1, 8, 64, dtype=torch.float32), spec) == torch.float32  # tf32 check mode
    assert A.out_dtype(t(1, 1, 8, 64), A.AttnSpec(out_fp32=True)) == torch.float32
