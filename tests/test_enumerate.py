"""Exact counts three ways (SPEC acceptance 1): the symbolic
counter, the CPU enumeration oracle (oracle.cpp:76-443 semantics) and the GPU
enumerator (csrc/cuda/enum.cu), through ps_enumerate."""
import pytest

from paper_1904_09538_b200 import host

SMALL = [
    "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-64__prefetch-True",
    "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-48__prefetch-False",
    "matmul_sq_rm__dtype-float32__groups_fit-True__keep-b__lsize_0-16__lsize_1-16__n-64__prefetch-True",
    "finite_diff__dtype-float32__n-56__tile-16x16",
    "finite_diff_rm__dtype-float32__keep-u__n-48__tile-18x18",
    "dg_diff__dtype-float32__nelements-32__nmatrices-3__nunit_nodes-32__variant-uPF",
    "dg_diff_rm__dtype-float32__keep-dm__nelements-32__nmatrices-3__nunit_nodes-16__variant-dmPFtrans",
    "gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16"
    "__n_input_arrays-2__nelements-65536",
    "flops_madd_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-16__lsize_0-16__lsize_1-16"
    "__m-2__nelements-1024",
    "lmem_shuffle__dtype-float32__lid_stride_0-1__lid_stride_1-16__lsize_0-16__lsize_1-16"
    "__m-3__nelements-1024",
    "barrier_knl__lid_stride_0-1__lid_stride_1-16__lsize_0-16__lsize_1-16__m-5__nelements-1024",
    "overlap_knl__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16"
    "__m-2__nelements-65536",
]

# bench-sized kernels, too large for the CPU enumerator in a test (up to 10^9 points)
LARGE = [
    "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-1024__prefetch-True",
    "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-1024__prefetch-False",
    "matmul_sq_rm__dtype-float32__groups_fit-True__keep-a__lsize_0-16__lsize_1-16__n-1024"
    "__prefetch-False",
    "finite_diff__dtype-float32__n-2240__tile-16x16",
    "finite_diff_rm__dtype-float32__keep-res__n-2240__tile-18x18",
    "dg_diff__dtype-float32__nelements-100000__nmatrices-3__nunit_nodes-64__variant-dmPFtrans",
    "dg_diff_rm__dtype-float32__keep-u__nelements-100000__nmatrices-3__nunit_nodes-64__variant-noPF",
]

KEYS = ("ops", "access_counts", "footprints", "barrier_local")


@pytest.mark.parametrize("vid", SMALL)
def test_symbolic_equals_cpu_enumeration(vid):
    s = host.enumerate_counts(vid, "symbolic")
    c = host.enumerate_counts(vid, "cpu")
    for k in KEYS:
        assert s[k] == c[k], k


@pytest.fixture(scope="module")
def dev():
    from paper_1904_09538_b200.device import CudaDevice
    d = CudaDevice(0)
    yield d
    d.close()


@pytest.mark.gpu
@pytest.mark.parametrize("vid", SMALL)
def test_gpu_enumeration_equals_cpu_enumeration(dev, vid):
    g = host.enumerate_counts(vid, "gpu", dev)
    c = host.enumerate_counts(vid, "cpu")
    assert g == c


@pytest.mark.gpu
@pytest.mark.parametrize("vid", LARGE)
def test_gpu_enumeration_equals_symbolic_at_bench_sizes(dev, vid):
    g = host.enumerate_counts(vid, "gpu", dev)
    s = host.enumerate_counts(vid, "symbolic")
    for k in KEYS:
        assert g[k] == s[k], k
