"""Prepare one suite kernel (inputs resident) and launch it N times — the
target command for ncu captures (profiles/)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1904_09538_b200.device import CudaDevice  # noqa: E402

vid = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
with CudaDevice(0) as dev:
    dev.prepare(vid)
    dev.run_timed(vid, n)
    print("ran", vid, n)
