"""compute-sanitizer as a test target: memcheck over the smoke
path, the K17 v2 one-launch fit, K18 and the arena e2e pipeline; racecheck
and synccheck over the K17 v2 kernel (shared-memory Jacobian rows, the
warp-cooperative solve) and the shared-memory suite kernels."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

K17_K18 = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1904_09538_b200 import host, workloads
from paper_1904_09538_b200.device import CudaDevice, fit_lm_batched, fit_lm_jobs
from paper_1904_09538_b200.predict import PredictionTables, c5_points
rng = np.random.default_rng(1)
with CudaDevice(0) as dev:
    jobs = []
    for w in ("matmul", "dg"):
        wl = workloads.WORKLOADS[w]
        m = host.HostModel(wl.models["ldst"])
        F = np.exp(rng.uniform(0, 20, (40, len(m.features))))
        t = F @ rng.uniform(1e-13, 1e-11, len(m.features)) + 1e-5
        p0 = m.initial_point(F, t, scale=2)
        jobs.append({"model": m, "features": F, "t": t, "starts": np.stack([p0, p0]), "mode": 7})
        jobs.append({"model": m, "features": F / t[:, None], "t": np.ones_like(t), "mode": 0,
                     "starts": m.initial_point(F / t[:, None], np.ones_like(t), scale=0)[None]})
    res, _ = fit_lm_jobs(dev, jobs)
    # the round-1 K17 (postfix bytecode, forward-mode derivatives) as well
    j = jobs[0]
    fit_lm_batched(dev, j["model"], j["features"], j["t"], j["starts"], mode=13)
    vid = "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-1024__prefetch-True"
    m = host.HostModel(workloads.MATMUL.models["ldst"])
    t = PredictionTables([{"id": vid, "model": m.text, "params": list(res[0][0][0]), "group": 0,
                           "coords": {"n": 0}}])
    t.eval_gpu(dev, c5_points(2000))
print("ok")
'''


K18_CHUNKED = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1904_09538_b200 import host, workloads as W
from paper_1904_09538_b200.device import CudaDevice
from paper_1904_09538_b200.predict import PredictionTables, c5_points
host.set_option("partial_subgroups", "round_up")
variants = []
for g, wl in enumerate((W.MATMUL, W.FD, W.DG)):
    m = host.HostModel(wl.models["ldst"])
    tag = {"matmul": ["matmul_sq", "n:1024"], "fd": ["finite_diff", "n:1120"],
           "dg": ["dg_diff", "nelements:10000", "nunit_nodes:64"]}[wl.name]
    for vid, _ in host.catalog(tag):
        variants.append({"id": vid, "model": m.text, "params": [1e-12] * len(m.params),
                         "group": g, "coords": wl.c5_coords})
t = PredictionTables(variants)
pts = c5_points(500_000)
with CudaDevice(0) as dev:
    pp, pred, arg, keep = t.pinned_buffers(len(pts))
    pp[:] = pts
    t.eval_gpu(dev, pp, out=(pred, arg))
    pc, ac = t.eval_cpu(pts[-1000:], threads=4)
    assert np.array_equal(np.asarray(pred)[-1000:].view(np.uint64), pc.view(np.uint64))
print("ok")
'''


def _run(args, code=None, timeout=900):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, *args, sys.executable]
    cmd += ["-c", code] if code else []
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def test_memcheck_smoke():
    rc, out = _run(["--tool", "memcheck", "--error-exitcode", "9"],
                   "import __graft_entry__ as g; g.smoke()")
    assert rc == 0 and "ERROR SUMMARY: 0 errors" in out, out[-3000:]


def test_memcheck_k17_k18():
    rc, out = _run(["--tool", "memcheck", "--error-exitcode", "9"], K17_K18)
    assert rc == 0 and "ERROR SUMMARY: 0 errors" in out, out[-3000:]


@pytest.mark.parametrize("tool", ["racecheck", "synccheck"])
def test_shared_memory_checks_k17(tool):
    rc, out = _run(["--tool", tool, "--error-exitcode", "9"], K17_K18)
    assert rc == 0, out[-3000:]
    assert ("0 hazards" in out or "ERROR SUMMARY: 0 errors" in out), out[-3000:]


def test_memcheck_e2e_arena():
    rc, out = _run(["--tool", "memcheck", "--error-exitcode", "9"],
                   "import sys, pytest; sys.exit(pytest.main(['-q', '-x', '-p', 'no:cacheprovider', "
                   "'tests/test_gpu_e2e.py']))")
    assert rc == 0 and "ERROR SUMMARY: 0 errors" in out, out[-3000:]


def test_memcheck_k18_specialised_chunked():
    """The run-time compiled K18 kernels over the chunked three-stream
    pipeline (500k points, several chunks) under memcheck."""
    rc, out = _run(["--tool", "memcheck", "--error-exitcode", "9"], K18_CHUNKED)
    assert rc == 0 and "ERROR SUMMARY: 0 errors" in out, out[-3000:]
