"""The bench's own catalog pinned to the reference library.

oracle/ref_catalog.cpp reads every kernel of the `all` workload as
perfseer-kernel/1 JSON (DG variants and their ten dg-* work-removed tags,
the gmem 18x18 pattern and the B200 ladders included — kernels the
reference's own generators cannot build) and prints kernel_hash, the full
symbolic counts (analyze, counting.cpp:697-715) and every workload model's
feature values (evaluate_feature, features.cpp:342-415, strict sub-groups).
tests/golden/catalog_reference.jsonl is that program linked against the
UNMODIFIED reference (tools/gen_catalog_golden.py); here the same program
linked against the port must print the same bytes. The only unpinned values
are the SURVEY A1 extension: FD 18x18 sub-group entries, for which the
reference raises (324 work-items is not a multiple of 32) and the bench uses
ceil(324/32) sub-groups per work-group."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
GOLDEN = ROOT / "tests" / "golden" / "catalog_reference.jsonl"


@pytest.fixture(scope="module")
def port_output() -> str:
    import gen_catalog_golden
    subprocess.run(["make", "-s", "-f", str(ROOT / "tests" / "refapi.mk"), "catalog"], check=True,
                   cwd=ROOT)
    return gen_catalog_golden.run(ROOT / "tests" / "_build" / "port_ref_catalog")


def test_port_equals_reference_on_the_bench_catalog(port_output):
    want = GOLDEN.read_text().splitlines()
    got = port_output.splitlines()
    assert len(got) == len(want) == 336
    for g, w in zip(got, want):
        assert g == w, f"{json.loads(w)['id']}: port differs from the reference"


def test_golden_is_current_when_the_reference_is_built():
    exe = ROOT / "oracle" / "_ref" / "ref_catalog"
    if not exe.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    import gen_catalog_golden
    assert gen_catalog_golden.run(exe) == GOLDEN.read_text()


def test_only_fd18_subgroup_entries_are_unpinned():
    """Every entry the reference refuses is an FD 18x18 sub-group count (A1);
    the round_up extension changes exactly those and nothing else."""
    import gen_catalog_golden
    from paper_1904_09538_b200 import host
    feats = gen_catalog_golden.feature_ids()
    rows = [json.loads(l) for l in GOLDEN.read_text().splitlines()]
    refused = {(r["id"], f) for r in rows for f, v in zip(feats, r["features"])
               if isinstance(v, str)}
    assert refused and all("18x18" in k for k, _ in refused)
    assert all("324 is not a multiple" in v for r in rows for v in r["features"]
               if isinstance(v, str))
    ids = [r["id"] for r in rows]
    try:
        host.set_option("partial_subgroups", "round_up")
        for j, f in enumerate(feats):
            m = host.HostModel(f"f_exec_wall_time_x\np_a * {f}\n")
            vals = m.feature_table(ids)[:, 0]
            for r, v in zip(rows, vals):
                ref = r["features"][j]
                if isinstance(ref, str):
                    assert np.isfinite(v) and v >= 0
                else:
                    assert v == ref, (r["id"], f)
    finally:
        host.set_option("partial_subgroups", "strict")
