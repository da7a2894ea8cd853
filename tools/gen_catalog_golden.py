#!/usr/bin/env python
"""Pin the bench's own catalog to the reference library.

Writes the input stream for oracle/ref_catalog.cpp — every kernel of the
`all` workload as perfseer-kernel/1 JSON (the port's ps_kernel_json) plus the
union of every workload model's feature ids — and, with --golden, runs the
UNMODIFIED reference build (oracle/_ref/ref_catalog) on it to produce
tests/golden/catalog_reference.jsonl. tests/test_catalog_pin.py runs the same
program linked against the port and requires identical output."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden" / "catalog_reference.jsonl"


def feature_ids() -> list[str]:
    from paper_1904_09538_b200 import host, workloads
    out: list[str] = []
    for wl in workloads.WORKLOADS.values():
        for text in wl.models.values():
            for f in host.HostModel(text).features:
                if f not in out:
                    out.append(f)
    return out


def input_stream() -> str:
    from paper_1904_09538_b200 import host
    ids = json.loads((ROOT / "tests" / "golden" / "workload_all.json").read_text())["kernels"]
    lines = [json.dumps({"features": feature_ids(), "sub_group_size": 32})]
    lines += [json.dumps(host.kernel_json(i)) for i in ids]
    return "\n".join(lines) + "\n"


def run(exe: Path) -> str:
    r = subprocess.run([str(exe)], input=input_stream(), capture_output=True, text=True, check=True)
    return r.stdout


if __name__ == "__main__":
    out = run(ROOT / "oracle" / "_ref" / "ref_catalog")
    GOLDEN.write_text(out)
    print(GOLDEN, len(out.splitlines()), "kernels", len(out) // 1024, "KiB")
