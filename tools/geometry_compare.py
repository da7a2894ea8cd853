#!/usr/bin/env python
"""Launch-geometry fidelity: calibrate and predict
twice on one B200 — once with the realised launches (vectorised row sweeps
for the contiguous gmem/overlap streams, FD strips of R work-groups per CTA)
and once with the literal IR geometry (one CTA per work-group,
launch_geometry, transforms.cpp:242-275) for every kernel whose realisation
differs (gmem_pattern, overlap_knl, finite_diff, finite_diff_rm; matmul, DG
and the pattern microbenchmarks launch the literal geometry already) — and
report kernel-time ratios and each application's model error both ways.

    python tools/geometry_compare.py [--trials 20] [--out profiles/r02_geometry.json]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402

CHANGED = ("gmem_pattern", "overlap_knl", "finite_diff", "finite_diff_rm")


def sweep(dev, kernels, trials, warmup):
    out = {}
    for k in kernels:
        dev.prepare(k)
        out[k] = bench.summarize(dev.measure(k, trials=trials, warmup=warmup))[0]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "r02_geometry.json"))
    args = ap.parse_args()
    from paper_1904_09538_b200 import host
    from paper_1904_09538_b200.device import CudaDevice
    parts, kernels = bench.workload_kernels("all")
    changed = [k for k in kernels if k.split("__")[0] in CHANGED]
    dev = CudaDevice(0)
    host.set_option("launch_geometry", "realised")
    realised = sweep(dev, kernels, args.trials, args.warmup)
    host.set_option("launch_geometry", "literal")
    literal = dict(realised)
    literal.update(sweep(dev, changed, args.trials, args.warmup))
    host.set_option("launch_geometry", "realised")
    dev.trim()
    ratios = {}
    for k in changed:
        ratios.setdefault(k.split("__")[0], []).append(literal[k] / realised[k])
    report = {"trials": args.trials, "changed_kernels": len(changed),
              "literal_over_realised_time": {g: {"min": round(min(r), 3), "median": round(
                  float(np.median(r)), 3), "max": round(max(r), 3)} for g, r in ratios.items()},
              "applications": {}}
    for wl, cal, app in parts:
        rep = {}
        for name, table in (("realised", realised), ("literal", literal)):
            models = bench.model_report(wl, cal, app, table, dev)
            rep[name] = {}
            for mname, fits in models.items():
                f = fits.get("gpu_multistart_fit", {})
                if "geomean_rel_error" in f:
                    rep[name][mname] = {"geomean_rel_error": f["geomean_rel_error"],
                                        "all": f["geomean_rel_error_all"],
                                        "ranking_correct": f["ranking_correct"],
                                        "calibration_geomean_rel_error":
                                            f["calibration_geomean_rel_error"]}
        report["applications"][wl.name] = rep
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(report, indent=1) + "\n")
    with open(Path(args.out).with_suffix(".csv"), "w") as f:
        f.write("kernel,realised_s,literal_s\n")
        for k in changed:
            f.write(f"{k},{realised[k]!r},{literal[k]!r}\n")
    print(json.dumps(report["literal_over_realised_time"]))
    dev.close()


if __name__ == "__main__":
    main()
