#!/usr/bin/env python
"""Per-kernel launch counts and time shares from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file ...`, ncu_capture.sh
launches): `python tools/launch_summary.py launches_all.csv > summary.csv`."""
import csv
import re
import sys


def main(path: str) -> None:
    tot: dict[str, list] = {}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        t = tot.setdefault(name, [0, 0])
        t[0] += 1
        t[1] += int(float(r["Metric Value"].replace(",", "")))
    all_ns = sum(v[1] for v in tot.values())
    w = csv.writer(sys.stdout, quoting=csv.QUOTE_NONNUMERIC)
    w.writerow(["kernel", "launches", "total_ns", "share_pct"])
    for k, (n, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        w.writerow([k, n, ns, round(100.0 * ns / all_ns, 2)])


if __name__ == "__main__":
    main(sys.argv[1])
