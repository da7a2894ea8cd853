"""K16 with B read N-major (3-D TMA, b_major=MN, no transpose) vs the
transposed K-major path: parity on seed-pattern inputs and launch time."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402

from oracle import suite as oracle_suite  # noqa: E402
from paper_1904_09538_b200 import desc_from_id, kernel_io  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402
from tests._inputs import make_inputs  # noqa: E402

with CudaDevice(0) as dev:
    for n in (256, 512, 1024):
        d = desc_from_id(f"matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-{n}")
        io = kernel_io(d)
        ins = make_inputs(d, io, "seed17")
        outs = {}
        for mode in ("k", "mn"):
            os.environ["PS_TC_B"] = mode
            outs[mode] = dev.run(d, ins)[0]
        r = desc_from_id(f"matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-{n}__prefetch-False")
        want = oracle_suite.run(r, kernel_io(r), ins)[0]
        print(n, "k==oracle", np.array_equal(outs["k"].view(np.uint32), want.view(np.uint32)),
              "mn==oracle", np.array_equal(outs["mn"].view(np.uint32), want.view(np.uint32)),
              "mn nonzero", int(np.count_nonzero(outs["mn"])), flush=True)
    for n in (4096, 8192):
        vid = f"matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-{n}"
        dev.prepare(vid)
        for mode in ("k", "mn", "k", "mn"):
            os.environ["PS_TC_B"] = mode
            dev.measure(vid, trials=3, warmup=1)
            mean, _ = dev.measure_summary(vid, trials=10, warmup=2)
            print(n, mode, f"{mean*1e3:.4f} ms", f"{2*n**3/mean/1e12:.1f} TF/s", flush=True)
