"""Binding-resource classification of the suite kernels (rooflines.py, used by
bench.py's suite_rooflines) and the LPT estimate source (previous run)."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PEAKS = {"hbm_gbs": 6500.0, "bf16_tflops": 1600.0}
CLK = 1965e6


def _row(vid, t):
    from paper_1904_09538_b200.rooflines import rows_of
    return rows_of({vid: t}, CLK, PEAKS)[0]


def test_hbm_stream_fraction():
    vid = ("gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16"
           "__n_input_arrays-2__nelements-268435456")
    # 3 arrays x 2^28 x 4 B = 3.22 GB in 0.5 ms -> 6442 GB/s
    _, bound, ach, peak, unit, frac, _ = _row(vid, 0.5e-3)
    assert bound == "hbm" and unit == "GB/s" and peak == 6500.0
    assert math.isclose(ach, 3 * 2 ** 28 * 4 / 0.5e-3 / 1e9) and math.isclose(frac, ach / 6500.0)


def test_matmul_l1_operand_path():
    vid = "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-1024__prefetch-False"
    _, bound, ach, peak, unit, frac, _ = _row(vid, 1e-3)
    assert bound == "l1" and unit == "TB/s"
    assert math.isclose(ach, 8 * 1024 ** 3 / 1e-3 / 1e12)
    assert math.isclose(peak, 148 * 128 * CLK / 1e12)


def test_flops_and_latency_and_work_removed():
    base = "__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-64__nelements-1048576"
    _, b_add, a_add, p_add, _, _, _ = _row("flops_add_pattern" + base, 1e-3)
    _, b_madd, a_madd, _, _, _, _ = _row("flops_madd_pattern" + base, 1e-3)
    assert b_add == b_madd == "fp32" and math.isclose(a_add, a_madd)  # madd counted once per op
    assert math.isclose(a_add, (2048 * 64 + 31) * 1048576 / 1e-3 / 1e12)  # + the 31-add reduction
    bar = _row("barrier_knl__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16__m-256"
               "__nelements-2097152", 2e-4)
    assert bar[1] == "latency" and math.isnan(bar[5])
    rm = _row("dg_diff_rm__dtype-float32__keep-res__nelements-10000__nmatrices-3__nunit_nodes-64"
              "__variant-noPF", 1e-5)
    assert rm[1] == "wr" and math.isnan(rm[5])


def test_best_per_family_and_previous_run():
    from paper_1904_09538_b200.rooflines import best_per_family, rows_of
    mk = "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-{}__prefetch-True"
    rows = rows_of({mk.format(1024): 1e-3, mk.format(2048): 4e-3}, CLK, PEAKS)
    fam = best_per_family(rows)
    assert list(fam) == ["matmul_sq_prefetch-True"]
    assert fam["matmul_sq_prefetch-True"][0] == mk.format(2048)  # 2x the rate of n=1024
    import bench
    prev = bench.previous_run_seconds()
    assert len(prev) > 100 and all(t > 0 for t in prev.values())
