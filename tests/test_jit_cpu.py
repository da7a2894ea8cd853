"""K18 run-time specialisation (eval_jit.cu), host side: the generated CUDA
source for real workload tables compiles with NVRTC for sm_100a (no device
needed); the GPU tests check its bits against the interpreter and the CPU
tables."""
import numpy as np


def _tables(workload: str, model: str, tag: list[str], coords: dict):
    from paper_1904_09538_b200 import host, workloads as W
    from paper_1904_09538_b200.predict import PredictionTables
    wl = W.WORKLOADS[workload]
    text = wl.models[model]
    m = host.HostModel(text)
    rng = np.random.default_rng(5)
    params = list(rng.uniform(1e-13, 1e-11, len(m.params)))
    for i, c in enumerate(m.cost_params):
        if not c:
            params[i] = 20.0
    variants = [{"id": vid, "model": text, "params": params, "group": 0, "coords": coords}
                for vid, _ in host.catalog(tag)]
    return PredictionTables(variants)


def test_jit_source_compiles_for_every_application():
    from paper_1904_09538_b200 import host
    host.set_option("partial_subgroups", "round_up")  # the FD workload's 18x18 tiles
    try:
        _compile_all()
    finally:
        host.set_option("partial_subgroups", "strict")


def _compile_all():
    for workload, model, tag, coords in (
            ("matmul", "overlap3", ["matmul_sq", "n:1024"], {"n": 0}),
            ("fd", "ldst_g", ["finite_diff", "n:1120"], {"n": 1}),
            ("dg", "ldst_g", ["dg_diff", "nelements:10000", "nunit_nodes:64"],
             {"nelements": 2, "nunit_nodes": 3})):
        t = _tables(workload, model, tag, coords)
        src = t.jit_source()
        assert "ps_k18_jit" in src and "glibc_tanh" in src
        assert src.count("ps_model_") >= 2
        assert t.jit_compile() > 1000  # cubin bytes


def test_jit_option_validates():
    import pytest

    from paper_1904_09538_b200 import PsError, host
    host.set_option("k18_jit", "off")
    host.set_option("k18_jit", "on")
    with pytest.raises(PsError):
        host.set_option("k18_jit", "maybe")
