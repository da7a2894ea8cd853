"""K16 matmul_sq_tc (tcgen05 kind::tf32, the extra dense-contraction variant)
against the fp32 oracle. Seed-pattern inputs are small integers, exact in
TF32 with exact FP32 sums (n <= 8192: sum <= 8192 * 17^2 < 2^24), so the tensor
core result must equal the oracle bit for bit. On U[-1,1) inputs the stated
bound is the TF32 operand rounding: |C - A.B| <= 2^-10 * (|A|.|B|) elementwise
(each operand carries <= 2^-11 relative error; FP32 accumulation adds
<= n * 2^-24 * (|A|.|B|), below 2^-11 of it for n <= 8192)."""
import numpy as np
import pytest

from oracle import suite as oracle_suite
from tests._inputs import desc_io, make_inputs

pytestmark = pytest.mark.gpu


def _ids(n):
    tc = f"matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-{n}"
    ref = (f"matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-{n}"
           "__prefetch-False")
    return tc, ref


@pytest.fixture(scope="module")
def dev():
    from paper_1904_09538_b200.device import CudaDevice
    d = CudaDevice(0)
    yield d
    d.close()


@pytest.mark.parametrize("n", [256, 512, 768, 2048])
def test_tc_seed_pattern_bitwise(dev, n):
    tc, ref = _ids(n)
    d, io = desc_io(tc)
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0]
    d2, io2 = desc_io(ref)
    want = oracle_suite.run(d2, io2, ins)[0]
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("n", [256, 1024])
def test_tc_uniform_within_tf32_bound(dev, n):
    tc, _ = _ids(n)
    d, io = desc_io(tc)
    ins = make_inputs(d, io, "uniform", seed=7)
    got = dev.run(d, ins)[0].astype(np.float64).reshape(n, n)
    a = ins[0].astype(np.float64).reshape(n, n)
    b = ins[1].astype(np.float64).reshape(n, n)
    exact = a @ b
    bound = 2.0 ** -10 * (np.abs(a) @ np.abs(b))
    assert np.all(np.abs(got - exact) <= bound)
    # and it is a TF32 result, not an FP32 one: error well above FP32 rounding
    assert np.max(np.abs(got - exact) / bound) > 1e-3


def test_tc_rejects_unsupported_sizes(dev):
    from paper_1904_09538_b200 import PsError
    with pytest.raises(PsError, match="multiple of 256"):
        d, io = desc_io("matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-384")
        dev.run(d, make_inputs(d, io, "seed17"))
