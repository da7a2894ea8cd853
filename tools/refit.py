"""Offline re-fit of a measurement table (bench.py --table) with the C++ port:
per-application predictions vs measurements and the worst calibration rows."""
import csv
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1904_09538_b200 import host  # noqa: E402

table = sys.argv[1]
wname = next((a for a in sys.argv[2:] if not a.startswith("--")), "matmul")
rows = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(open(table))}
parts, _ = bench.workload_kernels(wname)
dev = None
if "--gpu" in sys.argv:
    from paper_1904_09538_b200.device import CudaDevice
    dev = CudaDevice(0)
for wl, cal, app in parts:
    cal = [k for k in cal if k in rows]
    app = [k for k in app if k in rows]
    print(wl.name, json.dumps(bench.model_report(wl, cal, app, rows, dev), indent=1))
    if "--rows" not in sys.argv:
        continue
    for mname, text in wl.models.items():
        m = host.HostModel(text)
        tc = np.array([rows[k] for k in cal])
        p, _ = m.fit_cpu(m.feature_table(cal), tc, scale=True)
        print(mname, dict(zip(m.params, p)))
        for k, pr in zip(app, m.predict_cpu(p, app)):
            print(f"   {rows[k]*1e3:10.4f}  pred {pr*1e3:10.4f}  ratio {pr/rows[k]:.3f}  {k[-40:]}")
        for k, pr in sorted(zip(cal, m.predict_cpu(p, cal)), key=lambda x: -abs(x[1] / rows[x[0]] - 1))[:10]:
            print(f"   cal {rows[k]*1e3:10.4f}  pred {pr*1e3:10.4f}  ratio {pr/rows[k]:.3f}  {k[:90]}")
