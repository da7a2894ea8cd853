"""K18 end to end through pinned buffers at 10^6 C5 points x the 8
application variants (each workload's ldst_g model, synthetic parameters):
specialised kernel vs table interpreter, kernel time and call time.

usage: python tools/exp/k18_e2e.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

from paper_1904_09538_b200 import host, workloads as W  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402
from paper_1904_09538_b200.predict import PredictionTables, c5_points  # noqa: E402

host.set_option("partial_subgroups", "round_up")
variants = []
for g, wl in enumerate((W.MATMUL, W.FD, W.DG)):
    text = wl.models["ldst_g"]
    m = host.HostModel(text)
    rng = np.random.default_rng(g)
    params = list(rng.uniform(1e-13, 1e-11, len(m.params)))
    for i, c in enumerate(m.cost_params):
        if not c:
            params[i] = 20.0
    tag = {"matmul": ["matmul_sq", "n:1024"], "fd": ["finite_diff", "n:1120"],
           "dg": ["dg_diff", "nelements:10000", "nunit_nodes:64"]}[wl.name]
    for vid, _ in host.catalog(tag):
        variants.append({"id": vid, "model": text, "params": params, "group": g,
                         "coords": wl.c5_coords})
t = PredictionTables(variants)
npts = 1_000_000
pts = c5_points(npts)
with CudaDevice(0) as dev:
    pp, pred, arg, keep = t.pinned_buffers(npts)
    pp[:] = pts
    for mode in ("on", "off", "on"):
        host.set_option("k18_jit", mode)
        jit_s = t.prepare_gpu(dev)
        t.eval_gpu(dev, pp, out=(pred, arg))
        ks, ws = [], []
        for _ in range(5):
            t0 = time.perf_counter()
            _, _, k = t.eval_gpu(dev, pp, out=(pred, arg))
            ws.append(time.perf_counter() - t0)
            ks.append(k)
        nev = npts * t.nvar
        print(f"k18_jit {mode:3s}: compile {jit_s:6.3f} s  kernel {min(ks) * 1e3:7.3f} ms "
              f"({nev / min(ks):.3e} evals/s)  call {min(ws) * 1e3:7.3f} ms ({nev / min(ws):.3e} evals/s)",
              flush=True)
