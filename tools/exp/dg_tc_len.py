"""K19 (dg_diff_tc) at Np = 16/32/64 over growing nel: launch time t against
the algorithmic bytes B, and the least-squares line t = t0 + B / BW — the
fixed per-launch cost t0 (launch, TMEM/barrier set-up, ring fill, store
drain) against the streaming rate BW. A short kernel at a high BW and a
visible t0 is launch-bound, not bandwidth-bound.

usage: python tools/exp/dg_tc_len.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

from paper_1904_09538_b200 import desc_from_id, kernel_io  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

with CudaDevice(0) as dev:
    for np_ in (16, 32, 64):
        rows = []
        for nel in (250_000, 500_000, 1_000_000, 2_000_000, 4_000_000):
            vid = f"dg_diff_tc__dtype-float32__nelements-{nel}__nmatrices-3__nunit_nodes-{np_}"
            io = kernel_io(desc_from_id(vid))
            dev.prepare(vid)
            dev.measure(vid, trials=3, warmup=2)
            t, _ = dev.measure_summary(vid, trials=20, warmup=2)
            rows.append((io.bytes_global, t))
            print(f"Np {np_:3d} nel {nel:8d}  {t * 1e6:9.2f} us  {io.bytes_global / t / 1e9:7.1f} GB/s",
                  flush=True)
            dev.trim()
        b = np.array([r[0] for r in rows], dtype=float)
        t = np.array([r[1] for r in rows])
        slope, t0 = np.polyfit(b, t, 1)
        print(f"Np {np_:3d}: t = {t0 * 1e6:.2f} us + B / {1 / slope / 1e9:.0f} GB/s", flush=True)
