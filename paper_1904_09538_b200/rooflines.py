"""Binding-resource rooflines of the suite kernels (used by bench.py's
`suite_rooflines` and tools/roofline_table.py).

  HBM       gmem_pattern, overlap_knl, finite_diff(_rm), dg_diff_tc: algorithmic
            bytes (ps_kernel_io.bytes_global) / time vs measured HBM GB/s
  FP32      flops_*_pattern: 2048 m E ops (madd counted once) / time vs
            148 SMs x 128 lanes x clock
  shared    lmem_shuffle: bytes_shared / time vs 148 x 128 B/clk x clock
  L1 path   matmul_sq, dg_diff (one work-item per thread): IR operand loads per
            madd x 4 B / time vs 148 x 128 B/clk x clock
  tensor    matmul_sq_tc: 2 n^3 / time vs measured bf16 / 2
  latency   barrier_knl, empty_knl: absolute (no throughput roofline)
  wr        matmul_sq_rm, dg_diff_rm: work-removed calibration kernels that
            time one access pattern of an application kernel as that kernel
            issues it, timed only (no roofline claim)
"""
from __future__ import annotations

from . import desc_from_id, kernel_io

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
        # instructions: a madd is one FFMA (io.flops counts it as 2 flops)
        ops = io.flops - (2048.0 * float(d.m) * float(d.nelements) if "madd" in gen else 0.0)
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




FAMILY_KEYS = ("variant", "prefetch", "tile", "keep", "n_input_arrays")


def family_of(vid: str) -> str:
    gen, *parts = vid.split("__")
    return gen + "".join("_" + p for p in parts if p.split("-")[0] in FAMILY_KEYS)


def rows_of(mean_s: dict[str, float], clk_hz: float, peaks: dict) -> list[tuple]:
    """(kernel, bound, achieved, peak, unit, frac, seconds) per measured kernel."""
    out = []
    for vid, t in mean_s.items():
        d = desc_from_id(vid)
        io = kernel_io(d)
        bound, ach, peak, unit = classify(vid, d, io, t, clk_hz, peaks)
        out.append((vid, bound, ach, peak, unit, ach / peak if peak == peak else float("nan"), t))
    return out


def best_per_family(rows: list[tuple]) -> dict[str, tuple]:
    fam: dict[str, tuple] = {}
    for r in rows:
        key = family_of(r[0])
        if r[5] == r[5] and (key not in fam or r[5] > fam[key][5]):
            fam[key] = r
    return fam
