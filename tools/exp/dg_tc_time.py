"""K19 dg_diff_tc vs the paper variants at nel = 1e6, every order's Np:
launch time, achieved HBM bandwidth (u in + res out + dm), TF/s."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1904_09538_b200 import desc_from_id, kernel_io  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

with CudaDevice(0) as dev:
    for np_ in (16, 32, 48, 64, 96, 128):
        row = []
        for name in ("dg_diff_tc", "uPF", "dmPFtrans"):
            vid = (f"dg_diff_tc__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-{np_}"
                   if name == "dg_diff_tc" else
                   f"dg_diff__dtype-float32__nelements-1000000__nmatrices-3__nunit_nodes-{np_}__variant-{name}")
            io = kernel_io(desc_from_id(vid))
            dev.prepare(vid)
            dev.measure(vid, trials=3, warmup=1)
            t, _ = dev.measure_summary(vid, trials=10, warmup=2)
            row.append(f"{name} {t*1e3:8.4f} ms {io.bytes_global/t/1e9:7.1f} GB/s {io.flops/t/1e12:6.1f} TF/s")
        print(f"Np {np_:3d} | " + " | ".join(row), flush=True)
