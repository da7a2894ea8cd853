"""Held-out model selection (bench.headline / bench._errors): the headline
model is chosen on the workload's validation sizes only and scored on the
rest; the paper's per-variant linear/nonlinear choice follows the majority of
the work-removal diagnosis."""
from __future__ import annotations

import numpy as np


def _app():
    from paper_1904_09538_b200 import workloads
    wl = workloads.MATMUL
    ids = [f"matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-{n}"
           f"__prefetch-{pf}" for n in (512, 1024, 2048, 4096) for pf in ("True", "False")]
    return wl, ids


def test_errors_split_validation_and_test():
    import bench
    wl, app = _app()
    meas = np.ones(len(app))
    pred = np.array([1.1 if "n-1024" in k or "n-4096" in k else 1.3 for k in app])
    e = bench._errors(wl, app, pred, meas)
    assert abs(e["validation_geomean_rel_error"] - 0.1) < 1e-12
    assert abs(e["validation_mean_rel_error"] - 0.1) < 1e-12
    assert abs(e["test"]["geomean_rel_error_all"] - 0.3) < 1e-12
    assert e["test"]["rows"] == 4


def test_headline_uses_validation_error_only():
    import bench
    models = {
        # better on test, worse on validation: must NOT win
        "a": {"gpu_reference_fit": {"calibration_geomean_rel_error": 0.01,
                                    "validation_mean_rel_error": 0.20,
                                    "test": {"geomean_rel_error_all": 0.01}}},
        "b": {"gpu_multistart_fit": {"calibration_geomean_rel_error": 0.05,
                                     "validation_mean_rel_error": 0.10,
                                     "test": {"geomean_rel_error_all": 0.40}}},
        "c": {"gpu_multistart_fit": {"error": "diverged"}},
    }
    m, fit, rec = bench.headline(models)
    assert (m, fit) == ("b", "gpu_multistart_fit")
    # forcing a model falls back to its lowest calibration error
    m, fit, _ = bench.headline(models, "a")
    assert (m, fit) == ("a", "gpu_reference_fit")


def test_paper_selection_follows_majority_diagnosis():
    import bench
    from paper_1904_09538_b200 import host, workloads
    wl, app = _app()
    mean_s = {k: 1e-3 for k in app}
    fits = {}
    for name in ("linear", "nonlinear"):
        m = host.HostModel(wl.models[name])
        fits[name] = {"gpu_reference_fit": {"calibration_geomean_rel_error": 0.1,
                                            "params": {p: 1e-12 for p in m.params}}}
    diag = {"matmul": {"matmul_sq_prefetch-True": {"n=512": {"kind": "linear"},
                                                   "n=1024": {"kind": "linear"},
                                                   "n=2048": {"kind": "max_overlap"}},
                       "matmul_sq_prefetch-False": {"n=512": {"kind": "max_overlap"},
                                                    "n=1024": {"kind": "max_overlap"}}}}
    out = bench.paper_selection([(wl, [], app)], {"matmul": fits}, diag, mean_s)
    assert out["matmul"]["choice"] == {"matmul_sq_prefetch-True": "linear",
                                       "matmul_sq_prefetch-False": "nonlinear"}
    assert set(out["matmul"]["geomean_rel_error"]) == {"matmul_sq_prefetch-True",
                                                       "matmul_sq_prefetch-False"}


def test_per_variant_selection_ranks_first_then_error_on_validation_only():
    import bench
    wl, app = _app()  # matmul PF/noPF at n = 512, 1024, 2048, 4096; validation 1024, 4096
    meas = {k: (1.0 if "prefetch-True" in k else 1.2) for k in app}
    # candidate A: PF accurate everywhere, noPF 30% low on validation -> ranks wrong
    # candidate B: PF 8% high, noPF 5% high on validation (ranks right), awful on test
    pa = {k: meas[k] * (1.0 if "prefetch-True" in k else 0.7) for k in app}
    pb = {k: meas[k] * ((1.08 if "prefetch-True" in k else 1.05)
                        if ("n-1024" in k or "n-4096" in k) else 3.0) for k in app}
    bench.APP_PREDICTIONS.clear()
    bench.APP_PREDICTIONS[("matmul", "a", "gpu_reference_fit")] = pa
    bench.APP_PREDICTIONS[("matmul", "b", "gpu_multistart_fit")] = pb
    r = bench.select_per_variant(wl, app, meas)
    bench.APP_PREDICTIONS.clear()
    # PF: A (exact); noPF: B — the only way to rank n=1024/4096 right; the
    # test sizes (where B is off by 3x) never enter the choice
    assert r["assignment"] == {"matmul_sq_prefetch-True": "a/gpu_reference_fit",
                               "matmul_sq_prefetch-False": "b/gpu_multistart_fit"}
    assert r["validation_ranking_correct_gap_ge_2pct"] == "2/2"
    assert r["test"]["geomean_rel_error"]["matmul_sq_prefetch-False"] > 1.0


def test_selection_mean_is_not_fooled_by_one_exact_row():
    import bench
    wl, app = _app()
    meas = np.ones(len(app))
    # validation rows n=1024/4096: a is exact on two rows and 40% off on two;
    # b is 5% off on all four. The geomean prefers a, the mean prefers b.
    val = [i for i, k in enumerate(app) if "n-1024" in k or "n-4096" in k]
    pa, pb = np.ones(len(app)), np.full(len(app), 1.05)
    pa[val[0]] = pa[val[1]] = 1.0 + 1e-9
    pa[val[2]] = pa[val[3]] = 1.4
    ea, eb = bench._errors(wl, app, pa, meas), bench._errors(wl, app, pb, meas)
    assert ea["validation_geomean_rel_error"] < eb["validation_geomean_rel_error"]
    assert ea["validation_mean_rel_error"] > eb["validation_mean_rel_error"]
