"""K19 dg_diff_tc (DG as a tcgen05 kind::tf32 contraction, an extra dense-
contraction variant) against the fp32 oracle. Seed-pattern inputs are small
integers, exact in TF32, with FP32 sums < 2^24 (Np <= 128), so the result must
equal the oracle bit for bit — including partial 128-row tiles (rows past nel
masked, TMA zero fill) and Np that are not multiples of 32 (16, 48, zero-filled
K columns). On U[-1,1) inputs: |res - exact| <= 2^-10 * (|dm| . |u|)
elementwise (TF32 operand rounding, as for K16)."""
import numpy as np
import pytest

from oracle import suite as oracle_suite
from tests._inputs import desc_io, make_inputs

pytestmark = pytest.mark.gpu


def _id(nel, np_, nmat=3):
    return f"dg_diff_tc__dtype-float32__nelements-{nel}__nmatrices-{nmat}__nunit_nodes-{np_}"


@pytest.fixture(scope="module")
def dev():
    from paper_1904_09538_b200.device import CudaDevice
    d = CudaDevice(0)
    yield d
    d.close()


@pytest.mark.parametrize("np_", [16, 32, 48, 64, 96, 128])
@pytest.mark.parametrize("nel", [16, 1040, 40000])
def test_dg_tc_seed_pattern_bitwise(dev, nel, np_):
    d, io = desc_io(_id(nel, np_))
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0]
    want = oracle_suite.run(d, io, ins)[0]
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("nmat", [1, 2, 4])
def test_dg_tc_other_matrix_counts(dev, nmat):
    d, io = desc_io(_id(272, 64, nmat))
    ins = make_inputs(d, io, "seed17")
    np.testing.assert_array_equal(dev.run(d, ins)[0].view(np.uint32),
                                  oracle_suite.run(d, io, ins)[0].view(np.uint32))


@pytest.mark.parametrize("np_", [48, 128])
def test_dg_tc_uniform_within_tf32_bound(dev, np_):
    nel, nmat = 1040, 3
    d, io = desc_io(_id(nel, np_))
    ins = make_inputs(d, io, "uniform", seed=5)
    got = dev.run(d, ins)[0].astype(np.float64).reshape(nmat, nel, np_)
    dm = ins[0].astype(np.float64).reshape(nmat, np_, np_)
    u = ins[1].astype(np.float64).reshape(nel, np_)
    exact = np.einsum("mij,kj->mki", dm, u)
    bound = 2.0 ** -10 * np.einsum("mij,kj->mki", np.abs(dm), np.abs(u))
    assert np.all(np.abs(got - exact) <= bound)
    assert np.max(np.abs(got - exact) / bound) > 1e-3  # a TF32 result, not FP32


@pytest.mark.parametrize("np_,nmat", [(128, 4), (112, 3), (128, 1)])
def test_dg_tc_matrix_groups(dev, np_, nmat):
    # Np >= 112: the matrices do not all fit beside the u ring, so the grid
    # splits into one group of CTAs per matrix (each group streams all tiles)
    d, io = desc_io(_id(1040, np_, nmat))
    ins = make_inputs(d, io, "seed17")
    np.testing.assert_array_equal(dev.run(d, ins)[0].view(np.uint32),
                                  oracle_suite.run(d, io, ins)[0].view(np.uint32))


@pytest.mark.parametrize("nel,np_,nmat", [(1040, 128, 3), (40000, 112, 3), (272, 128, 4)])
def test_dg_tc_cta_pairs(dev, monkeypatch, nel, np_, nmat):
    # cta_group::2 path (opt-in, PS_DGTC_PAIR=1): M = 256 tiles, dm split by N
    monkeypatch.setenv("PS_DGTC_PAIR", "1")
    d, io = desc_io(_id(nel, np_, nmat))
    ins = make_inputs(d, io, "seed17")
    np.testing.assert_array_equal(dev.run(d, ins)[0].view(np.uint32),
                                  oracle_suite.run(d, io, ins)[0].view(np.uint32))


@pytest.mark.parametrize("np_", [16, 32])
def test_dg_tc_ring_wraps_bitwise(dev, np_):
    """enough tiles per persistent CTA (>= 10 x 148 x 128 rows)
    that the u ring (8 stages at Np = 16, 3 at Np = 32) and the 8-warp
    epilogue buffers wrap many times, so every empty-barrier phase is used."""
    nel = 148 * 128 * 10 + 48  # plus a partial last tile
    d, io = desc_io(_id(nel, np_))
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0]
    want = oracle_suite.run(d, io, ins)[0]
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
