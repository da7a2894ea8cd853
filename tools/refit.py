"""Offline re-fit of a measurement table (bench.py --table) with the C++ port:
prints per-application predictions vs measurements for each model."""
import csv
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1904_09538_b200 import host, workloads  # noqa: E402

table = sys.argv[1]
wname = sys.argv[2] if len(sys.argv) > 2 else "matmul"
rows = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(open(table))}
wl, cal, app = bench.workload_kernels(wname)
cal = [k for k in cal if k in rows]
app = [k for k in app if k in rows]
dev = None
if "--gpu" in sys.argv:
    from paper_1904_09538_b200.device import CudaDevice
    dev = CudaDevice(0)
rep = bench.model_report(wl, cal, app, rows, dev)
import json
print(json.dumps(rep, indent=1))
for mname, r in rep.items():
    r = r.get("gpu_multistart_fit", r["reference_fit"])
    if "params" not in r:
        continue
    m = host.HostModel(wl.models[mname])
    p = np.array([r["params"][n] for n in m.params])
    pred = m.predict_cpu(p, app)
    for k, pr in zip(app, pred):
        print(f"   {rows[k]*1e3:10.4f}  pred {pr*1e3:10.4f}  ratio {pr/rows[k]:.3f}  {k[-40:]}")
    # calibration residuals
    predc = m.predict_cpu(p, cal)
    worst = sorted(zip(cal, predc), key=lambda x: -abs(x[1] / rows[x[0]] - 1))[:8]
    for k, pr in worst:
        print(f"   cal {rows[k]*1e3:10.4f}  pred {pr*1e3:10.4f}  ratio {pr/rows[k]:.3f}  {k[:70]}")
