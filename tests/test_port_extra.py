"""This repo's generators — the reference's ten plus the DG builders, which
have no reference implementation — checked symbolically against the port's
enumeration oracle at small admissible sizes (tests/port_extra.cpp), and
every B200 catalog id rebuilt from its variant id."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_symbolic_counts_equal_enumeration_for_all_generators():
    subprocess.run(["make", "-f", str(ROOT / "tests" / "refapi.mk"), "extra"], check=True,
                   capture_output=True)
    r = subprocess.run([str(ROOT / "tests" / "_build" / "port_extra")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout
