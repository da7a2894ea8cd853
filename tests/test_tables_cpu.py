"""K18 tables on the host (ps_eval_cpu) against the reference-API predict()
(ps_predict_cpu, features through evaluate_feature) for all 8 application
variants, including the FD 18x18 rational sub-group counts."""
import numpy as np


def _variants(model="lsu", seed=5):
    import bench
    from paper_1904_09538_b200 import host, workloads
    parts, _ = bench.workload_kernels("all")
    rng = np.random.default_rng(seed)
    out = []
    for g, (wl, _cal, app) in enumerate(parts):
        m = host.HostModel(wl.models[model])
        params = list(rng.uniform(1e-13, 1e-11, len(m.params)))
        seen = set()
        for vid in app:
            key = workloads.variant_of(vid, wl.variant_keys)
            if key not in seen:
                seen.add(key)
                out.append({"id": vid, "model": wl.models[model], "params": params, "group": g,
                            "coords": wl.c5_coords})
    return out


def test_tables_equal_reference_predict_bitwise():
    import bench
    from paper_1904_09538_b200 import host
    from paper_1904_09538_b200.predict import PredictionTables, c5_points
    variants = _variants()
    t = PredictionTables(variants)
    assert t.nvar == 8 and t.ngroups == 3
    pts = c5_points(40, seed=3)
    pred, arg = t.eval_cpu(pts, threads=2)
    for j in range(len(pts)):
        for v, var in enumerate(variants):
            sizes = {k: int(pts[j, c]) for k, c in var["coords"].items()}
            ref = host.HostModel(var["model"]).predict_cpu(
                np.array(var["params"]), [bench._concrete(var["id"], sizes)])[0]
            assert pred[j, v] == ref, (var["id"], sizes)
    # winners: strict '<' first minimum in variant order, global indices
    for g in range(3):
        cols = [i for i, v in enumerate(variants) if v["group"] == g]
        want = [cols[int(np.argmin(pred[j, cols]))] for j in range(len(pts))]
        assert list(arg[:, g]) == want


def test_same_model_text_with_different_params_stays_distinct():
    """one model calibrated twice (e.g. on two machines) must keep
    both parameter vectors, not reuse the first."""
    from paper_1904_09538_b200.predict import PredictionTables, c5_points
    v = _variants("linear")[0]
    a = dict(v, params=[1e-12] * len(v["params"]))
    b = dict(v, params=[5e-12] * len(v["params"]), group=1)
    t = PredictionTables([a, b])
    pred, _ = t.eval_cpu(c5_points(4, seed=1))
    np.testing.assert_allclose(pred[:, 1] / pred[:, 0], 5.0, rtol=1e-12)


def test_tables_reject_out_of_range_groups_and_too_many_variants():
    import pytest

    from paper_1904_09538_b200 import PsError
    from paper_1904_09538_b200.predict import PredictionTables
    v = _variants("linear")[0]
    for g in (-1, 8):
        with pytest.raises(PsError, match="group"):
            PredictionTables([dict(v, group=g)])
    with pytest.raises(PsError, match="256 variants"):
        PredictionTables([v] * 257)


def test_tables_reject_models_deeper_than_the_device_stack():
    import pytest

    from paper_1904_09538_b200 import PsError
    from paper_1904_09538_b200.predict import PredictionTables
    v = _variants("linear")[0]
    # a right-nested sum of 80 distinct terms keeps ~80 partial values live
    terms = " + (".join(f"p_{i} * f_thread_groups" for i in range(80)) + ")" * 79
    text = "f_exec_wall_time_x\n" + terms + "\n"
    with pytest.raises(PsError, match="registers"):
        PredictionTables([dict(v, model=text, params=[1e-12] * 80)])
