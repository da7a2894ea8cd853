"""K16 CTA-pair (cta_group::2, 256x256 tiles) vs single-CTA kernel: parity on
seed-pattern inputs and launch time."""
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
        r = desc_from_id(f"matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-{n}__prefetch-False")
        want = oracle_suite.run(r, kernel_io(r), ins)[0]
        res = {}
        for mode in ("1", "0"):
            os.environ["PS_TC_PAIR"] = mode
            got = dev.run(d, ins)[0]
            res[mode] = (np.array_equal(got.view(np.uint32), want.view(np.uint32)), int(np.count_nonzero(got)))
        print(n, "pair", res["1"], "single", res["0"], flush=True)
    for n in (4096, 8192):
        vid = f"matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-{n}"
        dev.prepare(vid)
        for mode in ("1", "0", "1", "0"):
            os.environ["PS_TC_PAIR"] = mode
            dev.measure(vid, trials=3, warmup=1)
            mean, _ = dev.measure_summary(vid, trials=10, warmup=2)
            print(n, "pair" if mode == "1" else "single", f"{mean*1e3:.4f} ms", f"{2*n**3/mean/1e12:.1f} TF/s",
                  flush=True)
