"""The oracle's own variant parsing (oracle/variants.py) and the committed
workload files (tests/golden/workload_*.json) that let bench.py's reference
arm run the same workload without loading the product library."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
WORKLOADS = ("all", "matmul", "fd", "dg")
EXTRA = [
    "matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-8192",
    "dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-32",
    "gmem_pattern__dtype-float64__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16"
    "__n_input_arrays-1__nelements-65536",
]


@pytest.mark.parametrize("name", WORKLOADS)
def test_workload_file_is_current(name):
    sys.path.insert(0, str(ROOT / "tools"))
    from gen_workload_list import workload_doc
    committed = json.loads((ROOT / "tests" / "golden" / f"workload_{name}.json").read_text())
    assert committed == workload_doc(name), (
        f"tests/golden/workload_{name}.json is stale: run tools/gen_workload_list.py {name}")


def test_oracle_variants_match_product():
    from oracle import variants
    from paper_1904_09538_b200 import desc_from_id, kernel_io
    ids = json.loads((ROOT / "tests" / "golden" / "workload_all.json").read_text())["kernels"]
    for vid in ids + EXTRA:
        a, b = variants.parse(vid), desc_from_id(vid)
        for name, _ in b._fields_:
            assert getattr(a, name) == getattr(b, name), (vid, name)
        ia, ib = variants.io_of(a), kernel_io(b)
        assert ia.elem_bytes == ib.elem_bytes
        assert ia.input_elems == list(ib.input_elems[:ib.n_inputs]), vid
        assert ia.output_elems == list(ib.output_elems[:ib.n_outputs]), vid
        assert ia.bytes_global == ib.bytes_global and ia.flops == ib.flops, vid


def test_bench_config_identical_across_arms():
    import bench
    parts, kernels = bench.workload_kernels("all")
    n_app = len({k for _, _, app in parts for k in app})
    ours = bench.bench_config("all", len(kernels), len(kernels) - n_app, n_app, 80, 1)
    doc = bench.workload_doc("all")
    apps = {k for a in doc["applications"].values() for k in a["application"]}
    ref = bench.bench_config("all", len(doc["kernels"]), len(doc["kernels"]) - len(apps),
                             len(apps), 80, 1)
    assert ours == ref


def test_reference_arm_does_not_load_product_library():
    code = (
        "import sys, json, io, contextlib; sys.argv=['bench.py','--impl','reference',"
        "'--workload','fd','--steps','1','--warmup','0']\n"
        "import bench\n"
        "buf = io.StringIO()\n"
        "with contextlib.redirect_stdout(buf): bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "assert 'libperfseer_b200' not in maps, 'product library mapped'\n"
        "assert not any(m.startswith('paper_1904_09538_b200') for m in sys.modules)\n"
        "line = json.loads(buf.getvalue().strip().splitlines()[-1])\n"
        "assert line['impl'] == 'reference' and line['value'] > 0\n"
        "assert line['config']['workload'] == 'fd'\n"
        "print('ok')\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]
