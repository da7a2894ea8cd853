"""Per-kernel roofline report from a bench measurement table (bench.py --table):
for every suite kernel, its binding resource, achieved rate and fraction of
that resource's peak, and the best fraction per kernel family.

  HBM       gmem_pattern, overlap_knl, finite_diff(_rm), dg_diff_tc: algorithmic bytes (ps_kernel_io.bytes_global) / time
            vs MEASURED_PEAKS.json hbm_gbs
  FP32      flops_*_pattern: 2048 m E ops (madd counted once) / time vs
            148 SMs x 128 lanes x clock
  shared    lmem_shuffle: bytes_shared / time vs 148 x 128 B/clk x clock
  L1 path   matmul_sq, dg_diff (one work-item per thread): IR operand loads per
            madd x 4 B / time vs 148 x 128 B/clk x clock
  tensor    matmul_sq_tc: 2 n^3 / time vs MEASURED bf16 / 2
  latency   barrier_knl, empty_knl: absolute (no throughput roofline)
  wr        matmul_sq_rm, dg_diff_rm: work-removed calibration kernels that
            time one access pattern of an application kernel as that kernel
            issues it (e.g. DG's res stores, stride Np across lanes), timed
            only (no roofline claim)

usage: python tools/roofline_table.py TABLE.csv [--clock-mhz 1965] [--csv OUT]
"""
import argparse
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1904_09538_b200 import desc_from_id, kernel_io  # noqa: E402

# IR operand loads (bytes) per madd through the L1/shared data path, one
# work-item per thread: matmul a + b; DG per variant (uPF reads u_fetch once
# per j for the nmat accumulators)
DG_BYTES_PER_MADD = {0: 8.0, 1: 4.0 + 4.0 / 3.0, 2: 8.0, 3: 8.0}


def classify(vid: str, d, io, t: float, clk_hz: float, peaks: dict) -> tuple[str, float, float, str]:
    sm = 148
    gen = vid.split("__")[0]
    if gen in ("gmem_pattern", "overlap_knl", "finite_diff", "finite_diff_rm", "dg_diff_tc"):
        return "hbm", io.bytes_global / t / 1e9, peaks["hbm_gbs"], "GB/s"
    if gen.startswith("flops_"):
        ops = io.flops / (2.0 if "madd" in gen else 1.0)
        return "fp32", ops / t / 1e12, sm * 128 * clk_hz / 1e12, "Tops/s"
    if gen == "lmem_shuffle":
        return "shared", io.bytes_shared / t / 1e12, sm * 128 * clk_hz / 1e12, "TB/s"
    if gen == "matmul_sq":
        return "l1", 8.0 * float(d.n) ** 3 / t / 1e12, sm * 128 * clk_hz / 1e12, "TB/s"
    if gen == "dg_diff":
        b = DG_BYTES_PER_MADD[int(d.dg_variant)] * io.flops / 2.0
        return "l1", b / t / 1e12, sm * 128 * clk_hz / 1e12, "TB/s"
    if gen == "matmul_sq_tc":
        return "tensor", io.flops / t / 1e12, peaks["bf16_tflops"] / 2.0, "TFLOP/s"
    if gen in ("barrier_knl", "empty_knl"):
        return "latency", t * 1e6, float("nan"), "us"
    # work-removed kernels (matmul_sq_rm, dg_diff_rm): timed for
    # calibration only, no throughput claim; bytes_global / time for reference
    return "wr", io.bytes_global / t / 1e9, float("nan"), "GB/s"


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("table")
    ap.add_argument("--clock-mhz", type=float, default=1965.0)
    ap.add_argument("--csv", default="")
    a = ap.parse_args()
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() \
        else {"hbm_gbs": 6556.5, "bf16_tflops": 1598.1}
    rows = []
    with open(a.table) as f:
        for r in csv.DictReader(f):
            vid, t = r["kernel"], float(r["mean_seconds"])
            d = desc_from_id(vid)
            io = kernel_io(d)
            bound, ach, peak, unit = classify(vid, d, io, t, a.clock_mhz * 1e6, peaks)
            rows.append((vid, bound, ach, peak, unit, ach / peak if peak == peak else float("nan"), t))
    fam: dict[str, tuple] = {}
    for vid, bound, ach, peak, unit, frac, t in rows:
        gen, *parts = vid.split("__")
        key = gen + "".join("_" + p for p in parts if p.split("-")[0] in ("variant", "prefetch", "tile", "keep",
                                                                       "n_input_arrays"))
        if frac == frac and (key not in fam or frac > fam[key][5]):
            fam[key] = (vid, bound, ach, peak, unit, frac, t)
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
