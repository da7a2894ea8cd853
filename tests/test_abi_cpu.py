"""C ABI without a GPU: the library loads, exports every entry point declared
in include/perfseer_b200.h, parses every catalog variant id and reports
errors instead of crashing."""
import ctypes as C

import pytest

from paper_1904_09538_b200 import PsError, _abi, desc_from_id, host, kernel_io


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    names = _abi.exported_symbols()
    assert len(names) >= 30
    for n in names:
        assert hasattr(L, n), n


@pytest.mark.parametrize("which", ["reference", "b200"])
def test_every_catalog_variant_parses_and_has_io(which):
    ids = [k for k, _ in host.catalog([], which=which)]
    assert len(ids) > 100
    for vid in ids:
        d = desc_from_id(vid)
        io = kernel_io(d)
        assert io.n_outputs >= 0 and io.elem_bytes in (4, 8)
        if d.gen == 1:
            assert io.bytes_global == io.elem_bytes * d.nelements * (d.n_inputs + 1)


def test_reference_filter_examples():
    # SPEC.md:497-499 / acceptance 5
    tags = ["matmul_sq", "dtype:float32", "prefetch:True", "lsize_0:16", "lsize_1:16",
            "groups_fit:True", "n:2048,2560,3072,3584"]
    assert len(host.catalog(tags, which="reference")) == 4
    assert len(host.catalog([t for t in tags if t != "prefetch:True"], which="reference")) == 8
    assert host.catalog(["matmul_sq", "finite_diff"], which="reference") == []
    both = host.catalog(["matmul_sq", "finite_diff"], match="intersect", which="reference")
    gens = {k.split("__")[0] for k, _ in both}
    assert gens == {"matmul_sq", "finite_diff"}


@pytest.mark.parametrize("bad", [
    "nonsense__n-16",
    "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-100__prefetch-True",
    "finite_diff__dtype-float32__n-15__tile-16x16",
    "gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16"
    "__n_input_arrays-3__nelements-65536",
    "flops_add_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16"
    "__lsize_1-16__m-0__nelements-32768",
    "dg_diff__dtype-float32__nelements-100__nmatrices-3__nunit_nodes-64__variant-uPF",
])
def test_invalid_descriptors_are_errors(bad):
    with pytest.raises(PsError):
        kernel_io(desc_from_id(bad))


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = C.c_void_p()
    rc = _abi.lib().ps_init(0, C.byref(ctx))
    assert rc != 0
    assert _abi.lib().ps_last_error()


def test_process_options_validate_their_values():
    import pytest as _pytest

    from paper_1904_09538_b200 import PsError, host
    for key, good in (("measure_queue_ahead", ("off", "on")),
                      ("launch_geometry", ("literal", "realised")),
                      ("partial_subgroups", ("round_up", "strict"))):
        for v in good:
            host.set_option(key, v)
        with _pytest.raises(PsError):
            host.set_option(key, "sometimes")
    with _pytest.raises(PsError):
        host.set_option("no_such_option", "on")


def test_trace_ranges_nest_without_a_profiler():
    from paper_1904_09538_b200.host import trace
    with trace("outer"):
        with trace("inner"):
            pass
