"""Time K18 on 10^6 C5 points x the matmul variants (GPU vs CPU port)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_1904_09538_b200 import host, workloads as W  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402
from paper_1904_09538_b200.predict import PredictionTables, c5_points  # noqa: E402

variants = []
for g, name in enumerate(("linear", "overlap3")):
    text = W.MATMUL.models[name]
    m = host.HostModel(text)
    params = [1e-12] * len(m.params)
    for vid, _ in host.catalog(["matmul_sq", "n:1024"]):
        variants.append({"id": vid, "model": text, "params": params, "group": g, "coords": {"n": 0}})
t = PredictionTables(variants)
pts = c5_points(1_000_000)
with CudaDevice(0) as dev:
    t.eval_gpu(dev, pts[:1000])
    t0 = time.perf_counter()
    pg, ag, ks = t.eval_gpu(dev, pts)
    wall = time.perf_counter() - t0
t0 = time.perf_counter()
pc, ac = t.eval_cpu(pts[:100000], threads=8)
cpu = time.perf_counter() - t0
print(f"variants {t.nvar} points 1e6: gpu kernel {ks*1e3:.3f} ms ({1e6*t.nvar/ks:.3e} evals/s), "
      f"e2e {wall*1e3:.1f} ms; cpu(8 thr) 1e5 pts {cpu*1e3:.1f} ms ({1e5*t.nvar/cpu:.3e} evals/s); "
      f"max rel diff {np.max(np.abs(pg[:100000]-pc)/np.abs(pc)):.2e}")
