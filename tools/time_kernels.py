"""Time suite kernels (inputs resident, CUDA events) and print achieved HBM
bandwidth from the algorithmic byte count (ps_kernel_io bytes_global).

usage: python tools/time_kernels.py VARIANT_ID [VARIANT_ID ...]
       python tools/time_kernels.py --tag finite_diff --tag finite_diff_rm
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_09538_b200 import _abi, host  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("ids", nargs="*")
ap.add_argument("--tag", action="append", default=[])
ap.add_argument("--trials", type=int, default=20)
ap.add_argument("--opt", action="append", default=[], help="key=value for ps_set_option")
a = ap.parse_args()
for kv in a.opt:
    k, _, v = kv.partition("=")
    host.set_option(k, v)
ids = list(a.ids)
for t in a.tag:
    ids += [v for v, _ in host.catalog([t])]
with CudaDevice(0) as dev:
    for vid in ids:
        io = _abi.kernel_io(_abi.desc_from_id(vid))
        dev.prepare(vid)
        mean, _ = dev.measure_summary(vid, a.trials)
        print(f"{mean * 1e3:10.4f} ms {io.bytes_global / mean / 1e9:8.0f} GB/s "
              f"{io.flops / mean / 1e12:7.2f} TF/s  {vid}", flush=True)
