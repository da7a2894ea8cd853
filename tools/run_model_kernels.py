"""Target command for ncu captures of the model-side kernels: K17 (batched LM,
the DG lsu model on its round-1 calibration rows, 7 starts) and K18 (batched
prediction, the 8 application variants at 10^6 points), from the committed
round-1 measurement table (profiles/r01_table_all.csv)."""
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1904_09538_b200 import host, workloads  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice, fit_lm_batched  # noqa: E402
from paper_1904_09538_b200.predict import PredictionTables, c5_points  # noqa: E402

rows = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(open(ROOT / "profiles" / "r01_table_all.csv"))}
parts, _ = bench.workload_kernels("all")
with CudaDevice(0) as dev:
    variants = []
    for g, (wl, cal, app) in enumerate(parts):
        m = host.HostModel(wl.models["lsu"])
        cal = [k for k in cal if k in rows]
        fc = m.feature_table(cal)
        tc = np.array([rows[k] for k in cal])
        p0 = m.initial_point(fc, tc, scale=2)
        starts = np.stack([p0] * 7)
        params, stats = fit_lm_batched(dev, m, fc, tc, starts, mode=13)  # K17
        best = int(np.argmin([s["residual_norm"] for s in stats]))
        seen = set()
        for vid in app:
            key = workloads.variant_of(vid, wl.variant_keys)
            if key not in seen:
                seen.add(key)
                variants.append({"id": vid, "model": wl.models["lsu"], "params": list(params[best]),
                                 "group": g, "coords": wl.c5_coords})
        print(wl.name, "fit", stats[best]["status"], stats[best]["iterations"], flush=True)
    t = PredictionTables(variants)
    pred, arg, secs = t.eval_gpu(dev, c5_points(1_000_000))  # K18
    print("K18", pred.shape, f"{secs * 1e3:.3f} ms", flush=True)
