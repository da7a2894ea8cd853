"""Run-to-run spread of short kernels: FD 16x16 vs 18x18 at the small sizes,
each re-prepared (fresh device allocations) several times, 40 trials per
allocation. If the per-allocation means spread by more than the two tiles
differ, a ranking at that size is not a property of the tile.

usage: python tools/exp/fd_alloc.py
"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1904_09538_b200 import desc_from_id  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

sizes = (1120, 1680, 2240, 3360)
with CudaDevice(0) as dev:
    res = {(n, t): [] for n in sizes for t in ("16x16", "18x18")}
    for rep in range(6):
        dev.trim()  # drop every prepared variant: fresh allocations below
        pad = desc_from_id("gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16"
                           f"__lsize_1-16__n_input_arrays-1__nelements-{(rep + 1) * 1048576}")
        dev.prepare(pad)  # shifts the next allocations
        for n in sizes:
            for t in ("16x16", "18x18"):
                d = desc_from_id(f"finite_diff__dtype-float32__n-{n}__tile-{t}")
                dev.prepare(d)
                m, _ = dev.measure_summary(d, trials=40, warmup=3)
                res[(n, t)].append(m * 1e6)
    for n in sizes:
        a, b = res[(n, "16x16")], res[(n, "18x18")]
        print(f"n {n}: 16x16 {statistics.mean(a):7.3f} us (spread {min(a):.3f}-{max(a):.3f})  "
              f"18x18 {statistics.mean(b):7.3f} us (spread {min(b):.3f}-{max(b):.3f})  "
              f"18/16 per allocation {[round(y / x, 3) for x, y in zip(a, b)]}", flush=True)
