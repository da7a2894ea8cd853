"""dg_diff_tc achieved bandwidth vs nel (matrix stride in res) and Np."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1904_09538_b200 import desc_from_id, kernel_io  # noqa: E402
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

with CudaDevice(0) as dev:
    for np_ in (32, 48, 64):
        for nel in (1000000, 1000064, 1003520, 1048576, 999936):
            for nmat in (1, 3):
                vid = f"dg_diff_tc__dtype-float32__nelements-{nel}__nmatrices-{nmat}__nunit_nodes-{np_}"
                io = kernel_io(desc_from_id(vid))
                dev.prepare(vid)
                dev.measure(vid, trials=3, warmup=1)
                t, _ = dev.measure_summary(vid, trials=10, warmup=2)
                print(f"Np {np_:3d} nel {nel:8d} nmat {nmat}  {t*1e3:7.4f} ms  {io.bytes_global/t/1e9:7.1f} GB/s",
                      flush=True)
            dev.trim()
