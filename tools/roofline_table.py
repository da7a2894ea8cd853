"""Per-kernel roofline report from a bench measurement table (bench.py --table):
for every suite kernel, its binding resource (paper_1904_09538_b200/rooflines.py),
achieved rate and fraction of that resource's peak, and the best fraction per
kernel family.

usage: python tools/roofline_table.py TABLE.csv [--clock-mhz 1965] [--csv OUT]
"""
import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1904_09538_b200.rooflines import best_per_family, rows_of  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("table")
    ap.add_argument("--clock-mhz", type=float, default=1965.0)
    ap.add_argument("--csv", default="")
    a = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {"hbm_gbs": 6556.5, "bf16_tflops": 1598.1}
    with open(a.table) as f:
        mean_s = {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(f)}
    rows = rows_of(mean_s, a.clock_mhz * 1e6, peaks)
    fam = best_per_family(rows)
    print(f"{'family':58s} {'bound':7s} {'achieved':>10s} {'peak':>9s} unit     frac")
    for key in sorted(fam):
        vid, bound, ach, peak, unit, frac, t = fam[key]
        print(f"{key[:58]:58s} {bound:7s} {ach:10.2f} {peak:9.2f} {unit:8s} {frac:5.3f}")
    if a.csv:
        with open(a.csv, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "bound", "achieved", "peak", "unit", "frac", "seconds"])
            for r in rows:
                w.writerow([r[0], r[1], f"{r[2]:.4g}", f"{r[3]:.4g}", r[4], f"{r[5]:.4f}", f"{r[6]:.6g}"])


if __name__ == "__main__":
    main()
