"""Offline comparison of held-out model-selection rules over bench runs: the
fitted parameters of every (model, fit) candidate come from a run's detail
file, the measurements from its table; predictions are recomputed on the CPU
(the port's predict, bit-identical to K18). For each rule: the TEST-size
per-variant errors and the rankings (gap >= 2%) it would have reported.

usage: python tools/selection_eval.py TABLE.csv DETAIL.json [TABLE DETAIL ...]
"""
import csv
import itertools
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1904_09538_b200 import host, workloads  # noqa: E402


def rel(p, t):
    return abs(p - t) / t


def geo(xs):
    return math.exp(sum(math.log(max(x, 1e-12)) for x in xs) / len(xs))


def candidates(wl, app, detail):
    out = {}
    for mname, fits in detail["models"][wl.name].items():
        m = host.HostModel(wl.models[mname])
        for fname, f in fits.items():
            if not fname.startswith("gpu_") or "params" not in f:
                continue
            try:
                pr = m.predict_cpu([f["params"][n] for n in m.params], app)
            except Exception:
                continue
            out[(mname, fname)] = dict(zip(app, pr))
    return out


METRICS = {
    "geo": lambda es: geo(es),
    "mean": lambda es: sum(es) / len(es),
    "max": lambda es: max(es),
    "rms": lambda es: math.sqrt(sum(e * e for e in es) / len(es)),
}


def evaluate(wl, app, meas, cands, rule, metric):
    variant = {k: workloads.variant_of(k, wl.variant_keys) for k in app}
    is_val = {k: workloads.size_of(k, wl.size_keys) in wl.validation_sizes for k in app}
    val = [k for k in app if is_val[k]]
    variants = sorted(set(variant.values()))
    f = METRICS[metric]

    def verr(c, v):
        return f([rel(cands[c][k], meas[k]) for k in val if variant[k] == v])

    if rule == "single":
        best = min(cands, key=lambda c: f([rel(cands[c][k], meas[k]) for k in val]))
        asg = {v: best for v in variants}
    elif rule == "single_rank":
        def key(c):
            rows = [(k, cands[c][k], meas[k]) for k in val]
            ok = int(bench._rank(wl, rows)["ranking_correct_gap_ge_2pct"].split("/")[0])
            return (-ok, f([rel(cands[c][k], meas[k]) for k in val]))
        best = min(cands, key=key)
        asg = {v: best for v in variants}
    else:  # per-variant: rankings first, then worst variant error
        short = {v: sorted(cands, key=lambda c: verr(c, v))[:TOP] for v in variants}
        best = None
        for combo in itertools.product(*[short[v] for v in variants]):
            a = dict(zip(variants, combo))
            rows = [(k, cands[a[variant[k]]][k], meas[k]) for k in val]
            ok = int(bench._rank(wl, rows)["ranking_correct_gap_ge_2pct"].split("/")[0])
            key = (-ok, max(verr(a[v], v) for v in variants))
            if best is None or key < best[0]:
                best = (key, a)
        asg = best[1]
    rows = [(k, cands[asg[variant[k]]][k], meas[k]) for k in app]
    test = [r for r in rows if not is_val[r[0]]]
    return {"asg": sorted({f"{c[0]}/{c[1][4:9]}" for c in asg.values()}),
            "test_err": {v[-6:]: round(geo([rel(p, t) for k, p, t in test if variant[k] == v]), 3)
                         for v in variants},
            "all_err": {v[-6:]: round(geo([rel(p, t) for k, p, t in rows if variant[k] == v]), 3)
                        for v in variants},
            "rank": bench._rank(wl, rows)["ranking_correct_gap_ge_2pct"]}


TOP = None


def main():
    args = sys.argv[1:]
    for table, detail in zip(args[::2], args[1::2]):
        meas = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(open(table))}
        det = json.load(open(detail))
        parts, _ = bench.workload_kernels("all")
        print(f"=== {table}")
        for wl, _cal, app in parts:
            app = [k for k in app if k in meas]
            cands = candidates(wl, app, det)
            for rule in ("single", "single_rank", "per_variant"):
                for metric in ("geo", "mean", "max"):
                    r = evaluate(wl, app, meas, cands, rule, metric)
                    worst = max(r["all_err"].values())
                    print(f"  {wl.name:7s} {rule:12s} {metric:5s} rank {r['rank']:6s} "
                          f"worst_all {worst:.3f} test {r['test_err']} {r['asg']}")


if __name__ == "__main__":
    main()
