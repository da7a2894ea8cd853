"""The reference's own unit tests and golden generator, compiled from
/root/reference/proj (read in place) against this repo's C++ host port.

Passing means: the port is a drop-in for the reference API (same types,
names, error classes) and reproduces its behaviour — every catalog kernel's
symbolic counts and feature values, the reference interpreter outputs and the
Levenberg-Marquardt fits are byte-identical to the reference's own output
(tests/golden/reference.json). Skipped where /root/reference is absent
(the GPU box)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/proj")
pytestmark = pytest.mark.skipif(not REF.is_dir(), reason="reference sources not present")

TESTS = ["test_poly", "test_lang", "test_ir", "test_counting", "test_features", "test_model"]


@pytest.fixture(scope="module")
def built():
    lib = ROOT / "paper_1904_09538_b200" / "libperfseer_b200.so"
    if not lib.exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_1904_09538_b200" / "csrc"), "-j8"], check=True)
    subprocess.run(["make", "-f", str(ROOT / "tests" / "refapi.mk"), "-j8"], check=True,
                   capture_output=True)
    return ROOT / "tests" / "_build"


@pytest.mark.parametrize("name", TESTS)
def test_reference_unit_tests_pass_against_port(built, name):
    r = subprocess.run([str(built / f"port_{name}")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


def test_port_reproduces_reference_goldens_byte_for_byte(built):
    r = subprocess.run([str(built / "port_gen_golden")], capture_output=True, timeout=300)
    assert r.returncode == 0, r.stderr.decode()
    golden = (ROOT / "tests" / "golden" / "reference.json").read_bytes()
    assert r.stdout == golden


def test_reference_cpu_baseline_runs():
    # the bench's cpu_baseline_reference: the unmodified reference library timed
    # on the host (oracle/ref_cpu_bench.cpp)
    import json
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "_ref/ref_cpu_bench"], check=True,
                   capture_output=True)
    r = subprocess.run([str(ROOT / "oracle" / "_ref" / "ref_cpu_bench"), "0.2", "2"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["kind"] == "reference" and j["threads"] == 2 and j["catalog_kernels"] == 172
    assert j["predict_evals_per_s"] > 0 and j["fits_per_s"] > 0 and j["analyze_kernels_per_s"] > 0
