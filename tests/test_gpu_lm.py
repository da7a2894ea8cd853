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


def test_device_tanh_is_glibc_tanh(dev):
    """ps_math_tanh (the tanh inside K17/K18) returns the host libm's bits."""
    import ctypes as C
    import math

    from paper_1904_09538_b200._abi import check, lib
    rng = np.random.default_rng(11)
    mag = np.exp(rng.uniform(-25.0, np.log(60.0), 200_000))
    x = np.concatenate([mag * np.where(rng.random(mag.size) < 0.5, -1.0, 1.0),
                        [0.0, -0.0, 1e-300, 5e-324, 0.5 * math.log(2), 1.5 * math.log(2), 1.0, -1.0,
                         21.99, 22.0, 22.01, 40.0, -40.0, math.inf, -math.inf]])
    want = np.array([math.tanh(v) for v in x])
    got = np.empty_like(x)
    L = lib()
    L.ps_math_tanh.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double)]
    L.ps_math_tanh.restype = C.c_int
    check(L.ps_math_tanh(dev._ctx, x.ctypes.data_as(C.POINTER(C.c_double)), x.size,
                         got.ctypes.data_as(C.POINTER(C.c_double))))
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, f"{bad.size} mismatches, e.g. x={x[bad[:3]]}"


def _table_fits():
    """Every model of every workload on the committed round-1 sweep table."""
    import csv
    rows = {}
    with open(Path(__file__).resolve().parents[1] / "profiles" / "r01_table_all.csv") as f:
        for r in csv.DictReader(f):
            rows[r["kernel"]] = float(r["mean_seconds"])
    from paper_1904_09538_b200 import workloads
    cases = []
    for wl in workloads.WORKLOADS.values():
        for name in wl.models:
            cases.append((wl.name, name))
    return rows, cases


_ROWS, _CASES = _table_fits()


@pytest.mark.parametrize("case", _CASES, ids=lambda c: f"{c[0]}-{c[1]}")
def test_gpu_lm_reference_mode_on_real_table(dev, case):
    """K17 in reference mode (output-scaled rows, the
    reference's start, row-order sums, glibc tanh) against fit_model
    (model.cpp:485-606, the port verified bit-exact against the reference) on
    the round-1 B200 calibration table: identical parameters."""
    import bench
    from paper_1904_09538_b200 import host, workloads
    from paper_1904_09538_b200.device import fit_lm_batched
    wname, mname = case
    parts, _ = bench.workload_kernels(wname)
    wl, cal, _app = parts[0]
    cal = [k for k in cal if k in _ROWS]
    m = host.HostModel(wl.models[mname])
    fc = m.feature_table(cal)
    tc = np.array([_ROWS[k] for k in cal])
    try:
        p_ref, st = m.fit_cpu(fc, tc, scale=True)
    except Exception as e:  # the reference itself fails (e.g. divergence): nothing to match
        pytest.skip(f"fit_model raises: {e}")
    fs, ts = fc / tc[:, None], np.ones_like(tc)
    pg, sg = fit_lm_batched(dev, m, fs, ts, m.initial_point(fs, ts, scale=0)[None], mode=0)
    rel = np.max(np.abs(pg[0] - p_ref) / np.maximum(np.abs(p_ref), 1e-300))
    assert rel <= 1e-4, f"max relative parameter difference {rel:.3g}"
    assert sg[0]["iterations"] == st["iterations"]
    np.testing.assert_array_equal(pg[0], p_ref)


def test_lm_rejects_programs_deeper_than_the_device_stack(dev):
    import ctypes as C

    from paper_1904_09538_b200 import PsError
    from paper_1904_09538_b200._abi import Bytecode, FitOpts, FitStats, check, lib
    L = lib()
    depth = 60  # push p0 60 times, then 59 adds
    ops = np.array([(1 << 16) | 0] * depth + [3 << 16] * (depth - 1), dtype=np.int32)
    consts = np.zeros(1)
    bc = Bytecode(len(ops), 0, ops.ctypes.data_as(C.POINTER(C.c_int32)),
                  consts.ctypes.data_as(C.POINTER(C.c_double)))
    jac = (Bytecode * 1)(bc)
    f = np.ones((1, 4, 1))
    t = np.ones((1, 4))
    p = np.ones((1, 1))
    st = (FitStats * 1)()
    o = FitOpts(1e-3, 0.1, 10.0, 1e-10, 1e-10, 200, 0)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    L.ps_fit_lm_batched_ex.restype = C.c_int
    rc = L.ps_fit_lm_batched_ex(dev._ctx, C.byref(bc), jac, 1, 1, dp(f), dp(t), 4, 1, C.byref(o), 0,
                                dp(p), st)
    assert rc != 0 and b"stack" in L.ps_last_error()
    with pytest.raises(PsError):
        check(rc)


def test_lm_jobs_one_launch_reference_mode_bitwise(dev):
    """K17 v2 (ps_fit_lm_jobs): every model of every workload on the r01
    table in ONE launch, reference mode: bit-identical to fit_model."""
    import bench
    from paper_1904_09538_b200 import host, workloads
    from paper_1904_09538_b200.device import fit_lm_jobs
    jobs, refs = [], []
    for wname, mname in _CASES:
        parts, _ = bench.workload_kernels(wname)
        wl, cal, _app = parts[0]
        cal = [k for k in cal if k in _ROWS]
        m = host.HostModel(wl.models[mname])
        fc = m.feature_table(cal)
        tc = np.array([_ROWS[k] for k in cal])
        try:
            p_ref, st = m.fit_cpu(fc, tc, scale=True)
        except Exception:
            continue
        fs = fc / tc[:, None]
        jobs.append({"model": m, "features": fs, "t": np.ones_like(tc),
                     "starts": m.initial_point(fs, np.ones_like(tc), scale=0)[None], "mode": 0})
        refs.append((f"{wname}-{mname}", p_ref, st))
    res, secs = fit_lm_jobs(dev, jobs)
    assert secs > 0
    for (name, p_ref, st), (pg, sg) in zip(refs, res):
        assert sg[0]["iterations"] == st["iterations"], name
        np.testing.assert_array_equal(pg[0], p_ref, err_msg=name)


@pytest.mark.parametrize("case", FITS, ids=lambda c: c["name"])
def test_lm_jobs_golden_fits(dev, case):
    from paper_1904_09538_b200.device import fit_lm_jobs
    m, F, t = _problem(case)
    p0 = m.initial_point(F, t, scale=False)
    (params, stats), = fit_lm_jobs(dev, [{"model": m, "features": F, "t": t, "starts": p0[None],
                                          "mode": 0}])[0]
    ref = np.array(case["params"])
    assert stats[0]["iterations"] == case["iterations"] or not case["converged"]
    np.testing.assert_allclose(params[0], ref, rtol=1e-4, atol=1e-12 * np.abs(ref).max())


def test_lm_jobs_multistart_shuffle_matches_single_starts(dev):
    from paper_1904_09538_b200.device import fit_lm_jobs
    case = next(c for c in FITS if c["name"] == "overlap_seed5")
    m, F, t = _problem(case)
    p0 = m.initial_point(F, t, scale=False)
    starts = np.stack([p0] + [np.where(np.array(m.params) == "p_edge", e, p0) for e in (3.0, 10.0)])
    res, _ = fit_lm_jobs(dev, [{"model": m, "features": F, "t": t, "starts": starts, "mode": 7},
                               {"model": m, "features": F, "t": t, "starts": starts[1:2], "mode": 7}])
    np.testing.assert_array_equal(res[0][0][1], res[1][0][0])


def test_lm_jobs_rejects_bad_jobs(dev):
    from paper_1904_09538_b200 import PsError, host, workloads
    from paper_1904_09538_b200.device import fit_lm_jobs
    m = host.HostModel(workloads.MATMUL.models["linear"])
    F = np.ones((20, len(m.features)))
    good = {"model": m, "features": F, "t": np.ones(20), "starts": np.ones((1, len(m.params)))}
    # second job with the same model text but the wrong feature count
    bad = dict(good, features=np.ones((20, len(m.features) - 1)))
    with pytest.raises(PsError, match="features"):
        fit_lm_jobs(dev, [good, bad])
    with pytest.raises(PsError, match="rank deficiency"):
        fit_lm_jobs(dev, [dict(good, features=F[:3], t=np.ones(3))])
