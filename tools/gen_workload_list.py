#!/usr/bin/env python
"""Write tests/golden/workload_<name>.json: the kernel ids of a bench workload
(calibration and application ids per application, and their union in sweep
order) as the B200 catalog expands them. bench.py --impl reference reads this
file so the reference arm runs the same workload without loading the product
library; tests/test_variants_cpu.py checks the file is current."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def workload_doc(name: str) -> dict:
    import bench
    parts, kernels = bench.workload_kernels(name)
    return {"workload": name,
            "applications": {wl.name: {"calibration": cal, "application": app}
                             for wl, cal, app in parts},
            "kernels": kernels}


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "all"
    out = ROOT / "tests" / "golden" / f"workload_{name}.json"
    out.write_text(json.dumps(workload_doc(name), indent=1) + "\n")
    print(out, len(workload_doc(name)["kernels"]))
