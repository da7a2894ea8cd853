"""K17 (batched LM on the GPU) against the reference-exact CPU fit on the
reference's own canned problems (tests/golden/reference.json 'fits')."""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = json.loads((Path(__file__).parent / "golden" / "reference.json").read_text())
FITS = [f for f in GOLDEN["fits"] if "params" in f]


@pytest.fixture(scope="module")
def dev():
    from paper_1904_09538_b200.device import CudaDevice
    d = CudaDevice(0)
    yield d
    d.close()


def _problem(case):
    from paper_1904_09538_b200 import host
    m = host.HostModel(case["output"] + "\n" + case["expression"] + "\n")
    F = np.array([r["features"] for r in case["rows"]], dtype=np.float64)
    t = np.array([r["output"] for r in case["rows"]], dtype=np.float64)
    if case["scaled"]:
        F = F / t[:, None]
        t = np.ones_like(t)
    return m, F, t


@pytest.mark.parametrize("case", FITS, ids=lambda c: c["name"])
def test_gpu_lm_ordered_matches_reference_fit(dev, case):
    from paper_1904_09538_b200.device import fit_lm_batched
    m, F, t = _problem(case)
    p0 = m.initial_point(F, t, scale=False)
    params, stats = fit_lm_batched(dev, m, F, t, p0[None, :], mode=0)
    ref = np.array(case["params"])
    assert stats[0]["iterations"] == case["iterations"] or not case["converged"]
    np.testing.assert_allclose(params[0], ref, rtol=1e-4, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("case", [c for c in FITS if c["converged"]], ids=lambda c: c["name"])
def test_gpu_lm_shuffle_mode_within_spec_tolerance(dev, case):
    from paper_1904_09538_b200.device import fit_lm_batched
    m, F, t = _problem(case)
    p0 = m.initial_point(F, t, scale=False)
    params, stats = fit_lm_batched(dev, m, F, t, np.stack([p0, p0]), mode=2)
    ref = np.array(case["params"])
    for b in range(2):
        np.testing.assert_allclose(params[b], ref, rtol=1e-4, atol=1e-9 * np.abs(ref).max())


def test_gpu_lm_multistart_batch_is_independent(dev):
    from paper_1904_09538_b200.device import fit_lm_batched
    case = next(c for c in FITS if c["name"] == "overlap_seed5")
    m, F, t = _problem(case)
    p0 = m.initial_point(F, t, scale=False)
    starts = np.stack([p0] + [np.where(np.array(m.params) == "p_edge", e, p0) for e in (3.0, 10.0)])
    params, stats = fit_lm_batched(dev, m, F, t, starts, mode=1)
    assert len(stats) == 3
    single, _ = fit_lm_batched(dev, m, F, t, starts[1:2], mode=1)
    np.testing.assert_array_equal(params[1], single[0])


def test_gpu_lm_rank_deficiency_is_an_error(dev):
    from paper_1904_09538_b200 import PsError, host
    from paper_1904_09538_b200.device import fit_lm_batched
    m = host.HostModel("f_exec_wall_time_d\np_a * f_thread_groups + p_b\n")
    with pytest.raises(PsError, match="rank deficiency"):
        fit_lm_batched(dev, m, np.ones((1, 1)), np.ones(1), np.ones((1, 2)))
