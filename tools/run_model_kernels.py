"""Target command for ncu captures of the model-side kernels: K17 v2 (every
model of every workload on the committed round-2 measurement table, reference
mode + 7-start B200 mode, ONE ps_fit_lm_jobs launch) and K18 (batched
prediction, the 8 application variants at 10^6 points)."""
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1904_09538_b200 import host, workloads  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice, fit_lm_jobs  # noqa: E402
from paper_1904_09538_b200.predict import PredictionTables, c5_points  # noqa: E402

rows = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(open(ROOT / "profiles" / "r02_table_all.csv"))}
parts, _ = bench.workload_kernels("all")
wl_app = [app for _wl, _cal, app in parts]
with CudaDevice(0) as dev:
    jobs, keys = [], []
    for g, (wl, cal, app) in enumerate(parts):
        cal = [k for k in cal if k in rows]
        tc = np.array([rows[k] for k in cal])
        for mname, text in wl.models.items():
            m = host.HostModel(text)
            fc = m.feature_table(cal)
            fs = fc / tc[:, None]
            jobs.append({"model": m, "features": fs, "t": np.ones_like(tc),
                         "starts": m.initial_point(fs, np.ones_like(tc), scale=0)[None], "mode": 0})
            p0 = m.initial_point(fc, tc, scale=2)
            jobs.append({"model": m, "features": fc, "t": tc, "starts": np.stack([p0] * 7), "mode": 7})
            keys.append((g, wl, mname, m))
    res, ksec = fit_lm_jobs(dev, jobs)  # K17 v2: one launch
    print("K17", len(jobs), "jobs", f"{ksec * 1e3:.3f} ms", flush=True)
    variants = []
    for i, (g, wl, mname, m) in enumerate(keys):
        if mname != "lsu":
            continue
        params, stats = res[2 * i + 1]
        best = int(np.argmin([s["residual_norm"] for s in stats]))
        seen = set()
        for vid in wl_app[g]:
            key = workloads.variant_of(vid, wl.variant_keys)
            if key not in seen:
                seen.add(key)
                variants.append({"id": vid, "model": wl.models["lsu"], "params": list(params[best]),
                                 "group": g, "coords": wl.c5_coords})
    t = PredictionTables(variants)
    pred, arg, secs = t.eval_gpu(dev, c5_points(1_000_000))  # K18
    print("K18", pred.shape, f"{secs * 1e3:.3f} ms", flush=True)
