"""Trial timings with and without the queue-ahead kernel (ps_measure): the
bench's pattern (4 trials per call, 20 calls, other kernels between calls) on
the short kernels where host enqueue latency can land inside an event pair.

usage: python tools/exp/queue_ahead.py [--calls 20] [--per-call 4]
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1904_09538_b200 import _abi, host  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--calls", type=int, default=20)
ap.add_argument("--per-call", type=int, default=4)
a = ap.parse_args()

ids = [f"dg_diff__dtype-float32__nelements-10000__nmatrices-3__nunit_nodes-{np_}__variant-{v}"
       for np_ in (16, 64) for v in ("noPF", "uPF", "dmPF", "dmPFtrans")]
ids += [v for v, _ in host.catalog(["empty_knl"])][:2]
ids += ["finite_diff__dtype-float32__n-1120__tile-16x16",
        "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-512__prefetch-True"]

with CudaDevice(0) as dev:
    descs = [_abi.desc_from_id(v) for v in ids]
    for d in descs:
        dev.prepare(d)
    for mode in ("off", "on", "off", "on"):
        host.set_option("measure_queue_ahead", mode)
        times = {v: [] for v in ids}
        for _ in range(a.calls):
            for v, d in zip(ids, descs):
                times[v] += dev.measure(d, trials=a.per_call, warmup=0)
        print(f"--- queue_ahead {mode}")
        for v in ids:
            t = sorted(times[v])
            mean = sum(t) / len(t)
            print(f"  med {t[len(t) // 2] * 1e6:9.2f} us  mean {mean * 1e6:9.2f}  "
                  f"min {t[0] * 1e6:9.2f}  max {t[-1] * 1e6:9.2f}  "
                  f"cv {statistics.pstdev(t) / mean:6.3f}  {v[:90]}")
