"""K18 batched prediction: GPU tables vs the CPU port of the same tables vs
the reference-API predict() (features via evaluate_feature), and ranking."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1904_09538_b200.device import CudaDevice
    d = CudaDevice(0)
    yield d
    d.close()


def _tables():
    from paper_1904_09538_b200 import host, workloads as W
    from paper_1904_09538_b200.predict import PredictionTables
    variants = []
    for name in ("linear", "overlap3"):
        text = W.MATMUL.models[name]
        m = host.HostModel(text)
        rng = np.random.default_rng(3)
        params = list(rng.uniform(1e-13, 1e-11, len(m.params)))
        for i, c in enumerate(m.cost_params):
            if not c:
                params[i] = 20.0
        for vid, _ in host.catalog(["matmul_sq", "n:1024"]):
            variants.append({"id": vid, "model": text, "params": params,
                             "group": 0 if name == "linear" else 1, "coords": {"n": 0}})
    return PredictionTables(variants), variants


def test_gpu_eval_matches_cpu_tables_and_reference_predict(dev):
    from paper_1904_09538_b200 import host
    from paper_1904_09538_b200.predict import c5_points
    t, variants = _tables()
    pts = c5_points(20000, seed=11)
    pg, ag, secs = t.eval_gpu(dev, pts)
    pc, ac = t.eval_cpu(pts, threads=4)
    # device tanh = glibc tanh and the same register program: the same bits
    np.testing.assert_array_equal(pg.view(np.uint64), pc.view(np.uint64))
    assert np.array_equal(ag, ac)
    assert secs > 0
    # reference-API predict() at a few points
    for j in range(5):
        n = int(pts[j, 0])
        for v, var in enumerate(variants):
            m = host.HostModel(var["model"])
            ref = m.predict_cpu(np.array(var["params"]), [var["id"].replace("n-1024", f"n-{n}")])[0]
            assert pg[j, v] == ref


def test_gpu_eval_into_pinned_buffers(dev):
    from paper_1904_09538_b200.predict import c5_points
    t, _ = _tables()
    pts = c5_points(5000, seed=2)
    pp, pred, arg, keep = t.pinned_buffers(len(pts))
    pp[:] = pts
    g1, a1, _ = t.eval_gpu(dev, pp, out=(pred, arg))
    assert g1 is pred and a1 is arg
    g2, a2, _ = t.eval_gpu(dev, pts)
    np.testing.assert_array_equal(np.array(g1), g2)
    np.testing.assert_array_equal(np.array(a1), a2)


def test_nontabulable_features_are_rejected():
    from paper_1904_09538_b200 import PsError
    from paper_1904_09538_b200.predict import PredictionTables
    # lstride constraint against a parameter: match flips with n -> error
    text = ("f_exec_wall_time_cuda_b200_0\n"
            "p_a * f_mem_access_global_float32_load_lstrides:{1:<1000} + p_b * f_sync_kernel_launch\n")
    vid = "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-512__prefetch-True"
    with pytest.raises(PsError, match="not tabulable"):
        PredictionTables([{"id": vid, "model": text, "params": [1.0, 1.0], "group": 0,
                           "coords": {"n": 0}}])


def test_gpu_eval_chunked_pipeline_matches_cpu(dev):
    """1e6 points: the chunked copy-in / evaluate / copy-out pipeline
    (several chunks on three streams, pinned buffers) returns the same bits
    as the CPU tables on a sample and the same bits as a smaller
    single-chunk call on its prefix."""
    from paper_1904_09538_b200.predict import c5_points
    t, _ = _tables()
    pts = c5_points(1_000_000, seed=5)
    pp, pred, arg, keep = t.pinned_buffers(len(pts))
    pp[:] = pts
    g, a, secs = t.eval_gpu(dev, pp, out=(pred, arg))
    g, a = np.array(g), np.array(a)
    assert secs > 0
    idx = np.r_[0:2000, 151_000:153_000, 303_000:305_000, 998_000:1_000_000]
    pc, ac = t.eval_cpu(pts[idx], threads=4)
    np.testing.assert_array_equal(g[idx].view(np.uint64), pc.view(np.uint64))
    assert np.array_equal(a[idx], ac)
    g1, a1, _ = t.eval_gpu(dev, pts[:100_000])
    np.testing.assert_array_equal(g[:100_000].view(np.uint64), np.asarray(g1).view(np.uint64))
    assert np.array_equal(a[:100_000], np.asarray(a1))


def test_jit_kernel_matches_interpreter_bitwise(dev):
    """The run-time specialised K18 kernel (default) against the table
    interpreter (option k18_jit off) on the same points: identical bits."""
    from paper_1904_09538_b200 import host
    from paper_1904_09538_b200.predict import c5_points
    t, _ = _tables()
    pts = c5_points(300_000, seed=9)
    assert t.prepare_gpu(dev) >= 0.0
    gj, aj, _ = t.eval_gpu(dev, pts)
    host.set_option("k18_jit", "off")
    try:
        gi, ai, _ = t.eval_gpu(dev, pts)
    finally:
        host.set_option("k18_jit", "on")
    np.testing.assert_array_equal(np.asarray(gj).view(np.uint64), np.asarray(gi).view(np.uint64))
    assert np.array_equal(np.asarray(aj), np.asarray(ai))


def test_large_variant_space_keeps_the_interpreter(dev):
    """A table set whose generated kernel source exceeds the JIT limit is
    evaluated by the table interpreter (no compile), with the same bits as
    the CPU tables."""
    from paper_1904_09538_b200 import host, workloads as W
    from paper_1904_09538_b200.predict import PredictionTables, c5_points
    text = W.MATMUL.models["ldst_g"]
    m = host.HostModel(text)
    vids = [v for v, _ in host.catalog(["matmul_sq", "n:1024"])]
    rng = np.random.default_rng(4)
    variants = []
    for k in range(240):
        params = list(rng.uniform(1e-13, 1e-11, len(m.params)))
        for i, c in enumerate(m.cost_params):
            if not c:
                params[i] = 20.0
        variants.append({"id": vids[k % len(vids)], "model": text, "params": params,
                         "group": k % 8, "coords": {"n": 0}})
    t = PredictionTables(variants)
    assert len(t.jit_source()) > (1 << 19)
    assert t.prepare_gpu(dev) == 0.0
    pts = c5_points(3000, seed=8)
    pg, ag, _ = t.eval_gpu(dev, pts)
    pc, ac = t.eval_cpu(pts, threads=4)
    np.testing.assert_array_equal(np.asarray(pg).view(np.uint64), pc.view(np.uint64))
    assert np.array_equal(np.asarray(ag), ac)
