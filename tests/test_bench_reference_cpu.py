"""bench.py --impl reference under torchrun (the driver's reference arm at
N > 1): rank 0 alone times the CPU implementation of the path and prints one
JSON line; the other ranks exit 0 without work and without a GPU."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_two_ranks():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", "29593", "bench.py", "--impl", "reference",
         "--gpus", "2", "--workload", "fd", "--steps", "1", "--warmup", "3"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = lines[0]
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["steps"] == 1
    assert j["value"] > 0 and j["cpu_baseline"]["value"] == j["value"]
    assert j["cpu_baseline"]["kind"] in ("port", "reference")
    assert j["e2e"] == {"value": j["value"], "unit": j["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
