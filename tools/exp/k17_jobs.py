"""K17 v2 critical path: the bench's fit jobs on a measurement table, first
all in one launch (as the bench runs them), then each job alone, sorted by
its kernel time — the slowest CTA sets the launch time.

usage: python tools/exp/k17_jobs.py TABLE.csv [JOB]   (JOB e.g. dg/ldst_g/ref: that job alone)
"""
import csv
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1904_09538_b200 import host  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice, fit_lm_jobs  # noqa: E402

rows = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(open(sys.argv[1]))}
parts, _ = bench.workload_kernels("all")
jobs, names = [], []
for wl, cal, _app in parts:
    cal = [k for k in cal if k in rows]
    tc = np.array([rows[k] for k in cal])
    for mname, text in wl.models.items():
        m = host.HostModel(text)
        fc = m.feature_table(cal)
        fs, ts = fc / tc[:, None], np.ones_like(tc)
        jobs.append({"model": m, "features": fs, "t": ts,
                     "starts": m.initial_point(fs, ts, scale=0)[None], "mode": 0})
        names.append(f"{wl.name}/{mname}/ref")
        p0 = m.initial_point(fc, tc, scale=2)
        starts = [p0]
        edges = [i for i, c in enumerate(m.cost_params) if not c]
        for e in (bench.EDGE_STARTS if edges else ()):
            s_ = p0.copy()
            s_[edges] = e
            starts.append(s_)
        jobs.append({"model": m, "features": fc, "t": tc, "starts": np.stack(starts), "mode": 7})
        names.append(f"{wl.name}/{mname}/multi")

only = sys.argv[2] if len(sys.argv) > 2 else ""
with CudaDevice(0) as dev:
    if only:  # one job alone (an ncu target)
        r, s = fit_lm_jobs(dev, [jobs[names.index(only)]])
        print(only, f"{s * 1e3:.3f} ms", [st["iterations"] for st in r[0][1]])
        sys.exit(0)
    fit_lm_jobs(dev, jobs[:1])  # module load
    res, ksec = fit_lm_jobs(dev, jobs)
    print(f"all {len(jobs)} jobs in one launch: {ksec * 1e3:.2f} ms", flush=True)
    out = []
    for name, job in zip(names, jobs):
        r, s = fit_lm_jobs(dev, [job])
        its = [st["iterations"] for st in r[0][1]]
        out.append((s, name, len(job["starts"]), job["features"].shape, its,
                    [st["trials"] for st in r[0][1]]))
    for s, name, nb, shape, its, stat in sorted(out, reverse=True):
        print(f"  {s * 1e3:9.3f} ms  {name:28s} starts {nb}  rows x feats {shape}  "
              f"iterations {its} damped trials {stat}")
