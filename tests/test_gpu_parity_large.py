"""GPU parity at the BASELINE.json configuration sizes: the
sizes bench.py times, not only the small parity cases.

* matmul PF/noPF: full oracle at n = 2048; at n = 4096 and 8192 a sample of
  rows of c from the oracle (oracle.suite.matmul_rows: the same per-element
  fused multiply-add order), bitwise, seed-pattern and U[-1,1) inputs;
* matmul_sq_rm (keep a / b, PF / noPF) at n = 4096 against the work
  remover's sum (seed-pattern integers: every partial sum exact, so the
  order-free float64 sum is the bitwise answer);
* finite_diff and finite_diff_rm, both tiles, at n = 8176 (full oracle);
* DG, all four variants at nel = 10^5 and every padded Np of orders 1-7
  (16, 32, 48, 64, 96, 128), and their work-removed kernels at Np = 32;
  at the bench's nel = 10^6 every variant and K19 on sampled elements;
* gmem_pattern k = 1, 2 at E = 2^28 (1 GiB per array);
* the tcgen05 variant K16 at n = 8192 on sampled rows: bitwise on
  seed-pattern inputs, within the TF32 bound (fp64 reference rows) on U[-1,1).
"""
import numpy as np
import pytest

from oracle import suite as oracle_suite
from tests._inputs import desc_io, make_inputs

pytestmark = pytest.mark.gpu


def vid(gen, **args):
    return gen + "".join(f"__{k}-{args[k]}" for k in sorted(args))


@pytest.fixture(scope="module")
def dev():
    from paper_1904_09538_b200.device import CudaDevice
    d = CudaDevice(0)
    yield d
    d.trim()
    d.close()


def _bitwise(got, want, what):
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32), err_msg=what)


def _mm(n, pf):
    return vid("matmul_sq", dtype="float32", prefetch=pf, lsize_0=16, lsize_1=16,
               groups_fit="True", n=n)


@pytest.mark.parametrize("mode", ["seed17", "uniform"])
@pytest.mark.parametrize("pf", ["True", "False"])
def test_matmul_2048_full(dev, pf, mode):
    d, io = desc_io(_mm(2048, pf))
    ins = make_inputs(d, io, mode, seed=7)
    _bitwise(dev.run(d, ins)[0], oracle_suite.run(d, io, ins)[0], f"n=2048 {pf} {mode}")


@pytest.mark.parametrize("mode", ["seed17", "uniform"])
@pytest.mark.parametrize("pf", ["True", "False"])
@pytest.mark.parametrize("n", [4096, 8192])
def test_matmul_bench_sizes_sampled_rows(dev, n, pf, mode):
    d, io = desc_io(_mm(n, pf))
    ins = make_inputs(d, io, mode, seed=7)
    got = dev.run(d, ins)[0].reshape(n, n)
    rng = np.random.default_rng(n)
    # one row in every 16-row work-group band position, plus the edges
    rows = sorted(set(rng.choice(n, 48, replace=False).tolist()) | {0, 15, 16, n - 17, n - 1})
    for r in rows:
        _bitwise(got[r], oracle_suite.matmul_rows(d, ins, r, r + 1), f"n={n} {pf} {mode} row {r}")


@pytest.mark.parametrize("n", [1600, 2064, 6144])
def test_matmul_nopf_partial_panels(dev, n):
    """Work-group grids that are not a whole number of 64-column panels (100
    and 129 block columns) and the bench's 6144 (6 panels): every work-group
    still computes its own 16x16 block (sampled rows in every 16-row band
    position, both edges, full output of the b-column work-removed kernel)."""
    d, io = desc_io(_mm(n, "False"))
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0].reshape(n, n)
    rng = np.random.default_rng(n)
    rows = sorted(set(rng.choice(n, 24, replace=False).tolist()) | {0, 15, 16, n - 17, n - 1})
    for r in rows:
        _bitwise(got[r], oracle_suite.matmul_rows(d, ins, r, r + 1), f"n={n} row {r}")
    d, io = desc_io(vid("matmul_sq_rm", dtype="float32", prefetch="False", keep="b", lsize_0=16,
                        lsize_1=16, groups_fit="True", n=n))
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0].reshape(n, n)
    want = np.repeat(ins[0].astype(np.float64).reshape(n, n).sum(axis=0)[None, :], n, axis=0)
    np.testing.assert_array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("keep", ["a", "b"])
@pytest.mark.parametrize("pf", ["True", "False"])
def test_matmul_rm_4096(dev, pf, keep):
    n, T = 4096, 16
    d, io = desc_io(vid("matmul_sq_rm", dtype="float32", prefetch=pf, keep=keep, lsize_0=16,
                        lsize_1=16, groups_fit="True", n=n))
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0].reshape(n, n)
    x = ins[0].astype(np.float64).reshape(n, n)
    # transforms.cpp:317-514: tgt_read accumulates the kept loads of a
    # work-item in program order; integers < 2^24, so the sum is exact
    i = np.arange(n)
    if pf == "False":
        want = (np.repeat(x.sum(axis=1)[:, None], n, axis=1) if keep == "a"
                else np.repeat(x.sum(axis=0)[None, :], n, axis=0))
    elif keep == "a":  # a[i, 16 t + j % 16]
        want = x.reshape(n, n // T, T).sum(axis=1)[:, i % T]
    else:  # b[16 t + i % 16, j]
        want = x.reshape(n // T, T, n).sum(axis=0)[i % T, :]
    np.testing.assert_array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("mode", ["seed17", "uniform"])
@pytest.mark.parametrize("tile", ["16x16", "18x18"])
def test_fd_8176(dev, tile, mode):
    ids = [vid("finite_diff", dtype="float32", tile=tile, n=8176)]
    ids += [vid("finite_diff_rm", dtype="float32", tile=tile, keep=k, n=8176) for k in ("u", "res")]
    for v in ids:
        d, io = desc_io(v)
        ins = make_inputs(d, io, mode, seed=7)
        for g, w in zip(dev.run(d, ins), oracle_suite.run(d, io, ins)):
            _bitwise(g, w, f"{v} {mode}")


@pytest.mark.parametrize("n", [1680, 2800, 3360, 5600, 6272])
@pytest.mark.parametrize("tile", ["16x16", "18x18"])
def test_fd_validation_sizes(dev, tile, n):
    """The application-only FD sizes the bench measures for model selection."""
    v = vid("finite_diff", dtype="float32", tile=tile, n=n)
    d, io = desc_io(v)
    ins = make_inputs(d, io, "uniform", seed=7)
    _bitwise(dev.run(d, ins)[0], oracle_suite.run(d, io, ins)[0], v)


@pytest.mark.parametrize("mode", ["seed17", "uniform"])
@pytest.mark.parametrize("np_", [16, 32, 48, 64, 96, 128])
@pytest.mark.parametrize("variant", ["noPF", "uPF", "dmPF", "dmPFtrans"])
def test_dg_1e5(dev, variant, np_, mode):
    v = vid("dg_diff", dtype="float32", variant=variant, nelements=100000, nunit_nodes=np_,
            nmatrices=3)
    d, io = desc_io(v)
    ins = make_inputs(d, io, mode, seed=7)
    _bitwise(dev.run(d, ins)[0], oracle_suite.run(d, io, ins)[0], f"{v} {mode}")


@pytest.mark.parametrize("keep", ["u", "dm", "res"])
@pytest.mark.parametrize("variant", ["noPF", "uPF", "dmPF", "dmPFtrans"])
def test_dg_rm_1e5_np32(dev, variant, keep):
    v = vid("dg_diff_rm", dtype="float32", variant=variant, keep=keep, nelements=100000,
            nunit_nodes=32, nmatrices=3)
    d, io = desc_io(v)
    ins = make_inputs(d, io, "uniform", seed=7)
    _bitwise(dev.run(d, ins)[0], oracle_suite.run(d, io, ins)[0], v)


@pytest.mark.parametrize("k", [1, 2])
def test_gmem_2_28(dev, k):
    v = vid("gmem_pattern", n_input_arrays=k, nelements=1 << 28, dtype="float32", lsize_0=16,
            lsize_1=16, lid_stride_0=1, lid_stride_1=2048)
    d, io = desc_io(v)
    ins = make_inputs(d, io, "uniform", seed=7)
    _bitwise(dev.run(d, ins)[0], oracle_suite.run(d, io, ins)[0], v)


def test_tc_8192_sampled_rows(dev):
    n = 8192
    d, io = desc_io(f"matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-{n}")
    ref = desc_io(_mm(n, "False"))[0]
    rows = [0, 127, 128, 255, 256, 4095, 5000, n - 1]
    # seed pattern: integers <= 17, exact in TF32, sums < 2^24 -> bitwise
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0].reshape(n, n)
    for r in rows:
        _bitwise(got[r], oracle_suite.matmul_rows(ref, ins, r, r + 1), f"tc row {r}")
    # U[-1,1): |C - A.B| <= 2^-10 (|A|.|B|) (TF32 operand rounding)
    ins = make_inputs(d, io, "uniform", seed=7)
    got = dev.run(d, ins)[0].reshape(n, n).astype(np.float64)
    a = ins[0].astype(np.float64).reshape(n, n)
    b = ins[1].astype(np.float64).reshape(n, n)
    exact = a[rows] @ b
    bound = 2.0 ** -10 * (np.abs(a[rows]) @ np.abs(b))
    assert np.all(np.abs(got[rows] - exact) <= bound)


@pytest.mark.parametrize("np_", [16, 32, 48, 64, 96, 128])
@pytest.mark.parametrize("variant", ["noPF", "uPF", "dmPF", "dmPFtrans", "tc"])
def test_dg_1e6_sampled_elements(dev, variant, np_):
    """The bench's largest DG size (nel = 10^6) for every variant, K19
    included: seed-pattern inputs are small integers, so every partial sum is
    exact and res[m, k, i] = sum_j dm[m, i, j] u[k, j] in float64 at sampled
    elements k is the bitwise answer regardless of summation order."""
    nel, nmat = 1_000_000, 3
    if variant == "tc":
        v = f"dg_diff_tc__dtype-float32__nelements-{nel}__nmatrices-{nmat}__nunit_nodes-{np_}"
    else:
        v = vid("dg_diff", dtype="float32", variant=variant, nelements=nel, nunit_nodes=np_,
                nmatrices=nmat)
    d, io = desc_io(v)
    ins = make_inputs(d, io, "seed17")
    got = dev.run(d, ins)[0]
    dm = ins[0].astype(np.float64).reshape(nmat, np_, np_)
    trans = variant == "dmPFtrans"
    u = ins[1].astype(np.float64)
    u = u.reshape(np_, nel).T if trans else u.reshape(nel, np_)
    rng = np.random.default_rng(np_)
    ks = np.concatenate([rng.choice(nel, 500, replace=False), [0, 127, 128, nel - 1]])
    want = np.einsum("mij,kj->mki", dm, u[ks])  # [m, k, i]
    g = got.reshape(nmat, np_, nel)[:, :, ks].transpose(0, 2, 1) if trans else \
        got.reshape(nmat, nel, np_)[:, ks, :]
    np.testing.assert_array_equal(g.astype(np.float64), want)
