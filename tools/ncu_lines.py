#!/usr/bin/env python
"""Stall samples per CUDA source line of an ncu report with source
correlation (`ncu --import-source on`, code built with -lineinfo):
`python tools/ncu_lines.py REPORT.ncu-rep [top]`."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
agg, fname, line, src = {}, "?", "?", ""
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        continue
    if row[0]:  # a source line row
        line, src = row[0], row[1]
        continue
    try:  # a SASS row under the current source line
        n = int(row[4])
    except (IndexError, ValueError):
        continue
    a = agg.setdefault((fname, line), [0, src])
    a[0] += n
tot = sum(v[0] for v in agg.values()) or 1
for (f, ln), (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * n / tot:5.1f}%  {f}:{ln:>4}  {s.strip()[:90]}")
