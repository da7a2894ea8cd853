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
