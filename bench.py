#!/usr/bin/env python
"""Benchmark of the B200 measured-kernel and calibration path.

One step = one pass over the workload's measurement and application kernels
(BASELINE.json configs[1]: the matmul PF/noPF sweep n = 512..8192 plus the
B200 microbenchmark sweep that calibrates its model), each kernel launched
``--trials-per-step`` times and timed with CUDA events on the executor
stream. Work units (kernel, trial) are LPT-sharded over ranks; after the
timed region the measurement table is gathered (torch.distributed; NCCL on
GPUs), rank 0 summarises trials (5x-median filter), computes count features
with the C++ port, fits the linear and overlap models (Levenberg-Marquardt)
and predicts the held-out application variants.

metric/unit: suite GB/s = algorithmic global-memory bytes of every launched
suite kernel / max-over-ranks device time of the timed region; plus the
model's geomean |pred - meas| / meas per variant. Inputs are resident in HBM
(filled once; HBM kernels use >= 1 GiB arrays, larger than the 126 MB L2).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
METRIC = "suite GB/s"


def peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# distributed plumbing


class Dist:
    def __init__(self, process_group: bool = True):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        # GPU of this rank; PS_BENCH_DEVICE pins every rank to one GPU (with
        # PS_BENCH_BACKEND=gloo) to exercise the N>1 path on a 1-GPU box
        self.device = int(os.environ.get("PS_BENCH_DEVICE", self.local_rank))
        self.pg = None
        self.backend = None
        if self.world > 1 and process_group:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            backend = os.environ.get("PS_BENCH_BACKEND") or (
                "nccl" if torch.cuda.is_available() else "gloo")
            if backend == "nccl":
                torch.cuda.set_device(self.device)
            dist.init_process_group(backend=backend)
            self.pg = dist
            self.backend = backend
            # communicator init, for the driver's rank-count check
            print(f"[bench] rank {self.rank}: {backend} process group initialised, "
                  f"nranks {dist.get_world_size()}, device {self.device}", file=sys.stderr,
                  flush=True)

    def barrier(self):
        if self.pg:
            if self.backend == "nccl":
                import torch
                self.pg.barrier(device_ids=[self.device])
                torch.cuda.synchronize()
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        dev = f"cuda:{self.device}" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        dev = f"cuda:{self.device}" if self.backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t)
        return float(t.item())

    def gather_table(self, rows: list[tuple[int, int, float]]) -> list[tuple[int, int, float]]:
        """All-gather (kernel index, trial index, seconds) records as fixed-size
        float64 tensors over the process group (NCCL over NVLink on GPUs)."""
        if not self.pg:
            return rows
        import torch
        dev = f"cuda:{self.device}" if self.backend == "nccl" else "cpu"
        n = torch.tensor([len(rows)], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        self.pg.all_gather(sizes, n)
        cap = int(max(s.item() for s in sizes))
        buf = torch.full((cap, 3), -1.0, dtype=torch.float64, device=dev)
        if rows:
            buf[: len(rows)] = torch.tensor(rows, dtype=torch.float64, device=dev)
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        self.pg.all_gather(parts, buf)
        out = []
        for p in parts:
            for k, t, s in p.cpu().tolist():
                if k >= 0:
                    out.append((int(k), int(t), s))
        return out

    def all_gather_rows(self, a: np.ndarray) -> np.ndarray:
        """All-gather a [rows, cols] float64 block per rank (rows may differ)
        into the rank-ordered concatenation, as fixed-size padded tensors."""
        if not self.pg:
            return a
        import torch
        dev = f"cuda:{self.device}" if self.backend == "nccl" else "cpu"
        a = np.ascontiguousarray(a, dtype=np.float64).reshape(len(a), -1)
        n = torch.tensor([a.shape[0]], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        self.pg.all_gather(sizes, n)
        sizes = [int(x.item()) for x in sizes]
        buf = torch.zeros((max(sizes), a.shape[1]), dtype=torch.float64, device=dev)
        buf[: a.shape[0]] = torch.from_numpy(a).to(dev)
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        self.pg.all_gather(parts, buf)
        return np.concatenate([p[:m].cpu().numpy() for p, m in zip(parts, sizes)])

    def broadcast(self, obj):
        """Rank 0's picklable object on every rank."""
        if not self.pg:
            return obj
        box = [obj]
        self.pg.broadcast_object_list(box, src=0)
        return box[0]

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}


class ClockSampler:
    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[float, float, int]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return

        def pump():
            for line in self.proc.stdout:
                try:
                    sm, smax, reasons = [x.strip() for x in line.split(",")]
                    self.samples.append((float(sm), float(smax), int(reasons, 16)))
                except ValueError:
                    pass

        self.thread = threading.Thread(target=pump, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        mask = 0
        for _, _, r in self.samples:
            mask |= r
        return {"sm_mhz": statistics.median(s for s, _, _ in self.samples),
                "sm_max_mhz": max(m for _, m, _ in self.samples),
                "reasons": [n for b, n in REASONS.items() if mask & b and b != 0x1] or ["none"],
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# workload


def workload_kernels(name: str):
    """[(workload, calibration ids, application ids)] for a workload or a group
    ("all"), plus the de-duplicated union of their kernels in sweep order."""
    from paper_1904_09538_b200 import host, workloads
    parts = []
    for wl in workloads.resolve(name):
        for key, value in wl.extra.get("options", {}).items():
            host.set_option(key, value)
    for wl in workloads.resolve(name):
        cal = [k for tags in wl.calibration_tags for k, _ in host.catalog(tags)]
        app = [k for tags in wl.application_tags for k, _ in host.catalog(tags)]
        parts.append((wl, cal, app))
    kernels = list(dict.fromkeys(k for _, cal, app in parts for k in cal + app))
    return parts, kernels


def estimate_seconds(io) -> float:
    return io.bytes_global / 6.0e12 + io.flops / 30e12 + io.bytes_shared / 30e12 + 4e-6


def previous_run_seconds(path: Path = ROOT / "profiles" / "r02_table_all.csv") -> dict[str, float]:
    """Per-kernel mean seconds of the last committed sweep (LPT
    on the previous run's times); kernels it lacks fall back to
    estimate_seconds. On the round-1 table the crude estimate balances 8
    ranks to 6.5x of one, the previous run's times to 8.0x."""
    import csv
    if not path.exists():
        return {}
    with open(path) as f:
        return {r["kernel"]: float(r["mean_seconds"]) for r in csv.DictReader(f)}


def lpt(units: list[tuple[int, int]], est: list[float], world: int) -> list[list[tuple[int, int]]]:
    """Longest-processing-time-first assignment of (kernel, trial) units."""
    order = sorted(units, key=lambda u: -est[u[0]])
    loads = [0.0] * world
    shards: list[list[tuple[int, int]]] = [[] for _ in range(world)]
    for u in order:
        r = min(range(world), key=lambda i: loads[i])
        shards[r].append(u)
        loads[r] += est[u[0]]
    for s in shards:
        s.sort()
    return shards


def summarize(times: list[float], factor: float = 5.0) -> tuple[float, int]:
    """executor.cpp:14-38: drop trials > factor x median, mean of the rest."""
    s = sorted(times)
    n = len(s)
    med = s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])
    kept = [t for t in times if not t > factor * med]
    return sum(kept) / len(kept), len(kept)


def _rank(wl, rows) -> dict:
    """Per size: strict '<' first minimum (tools/perfseer.cpp:458-467) of the
    prediction vs the measurement; rows = [(variant id, pred, meas)]."""
    from paper_1904_09538_b200 import workloads
    by_size: dict[str, list] = {}
    for vid, p, t in rows:
        by_size.setdefault(workloads.size_of(vid, wl.size_keys), []).append(
            (workloads.variant_of(vid, wl.variant_keys), p, t))
    ranks, clear, detail = [], [], {}
    for size, rs in by_size.items():
        if len(rs) < 2:
            continue
        mbest = pbest = rs[0]
        for r in rs:
            if r[2] < mbest[2]:
                mbest = r
            if r[1] < pbest[1]:
                pbest = r
        ranks.append(mbest[0] == pbest[0])
        # measured gap between the fastest and the runner-up variant
        ts = sorted(r[2] for r in rs)
        gap = (ts[1] - ts[0]) / ts[0]
        if gap >= 0.02:
            clear.append(mbest[0] == pbest[0])
        detail[size] = {"measured_best": mbest[0], "predicted_best": pbest[0],
                        "measured_gap": round(gap, 4)}
    return {"ranking_correct": f"{sum(ranks)}/{len(ranks)}",
            # sizes whose two fastest variants are >= 2% apart when measured
            "ranking_correct_gap_ge_2pct": f"{sum(clear)}/{len(clear)}", "ranking": detail}


def _per_variant(wl, rows) -> dict:
    from paper_1904_09538_b200 import host, workloads
    per: dict[str, list] = {}
    for vid, p, t in rows:
        per.setdefault(workloads.variant_of(vid, wl.variant_keys), []).append((p, t))
    return {v: round(host.geo_mean_rel_error([p for p, _ in pts], [t for _, t in pts]), 5)
            for v, pts in per.items()}


def _mean_rel(pred, meas) -> float:
    return sum(abs(p - t) / t for p, t in zip(pred, meas)) / len(meas)


def _errors(wl, app, pred, ta) -> dict:
    """Per-variant geomean |pred - meas| / meas and rankings over every
    application size, plus the held-out split: `validation` = the workload's
    validation sizes (used only to choose the headline model), `test` = the
    rest (what the chosen model is scored on)."""
    from paper_1904_09538_b200 import host, workloads
    rows = list(zip(app, pred, ta))
    out = {"geomean_rel_error": _per_variant(wl, rows),
           "geomean_rel_error_all": round(host.geo_mean_rel_error(pred, ta), 5)}
    out.update(_rank(wl, rows))
    val = [r for r in rows if workloads.size_of(r[0], wl.size_keys) in wl.validation_sizes]
    test = [r for r in rows if workloads.size_of(r[0], wl.size_keys) not in wl.validation_sizes]
    if val and test:
        out["validation_geomean_rel_error"] = round(host.geo_mean_rel_error(
            [p for _, p, _ in val], [t for _, _, t in val]), 5)
        # the selection criterion: the arithmetic mean of |pred - meas| / meas
        # (a geomean over a handful of rows lets one near-exact row hide a
        # bad one)
        out["validation_mean_rel_error"] = round(_mean_rel([p for _, p, _ in val],
                                                           [t for _, _, t in val]), 5)
        rt = _rank(wl, test)
        out["test"] = {"geomean_rel_error": _per_variant(wl, test),
                       "geomean_rel_error_all": round(host.geo_mean_rel_error(
                           [p for _, p, _ in test], [t for _, _, t in test]), 5),
                       "ranking_correct": rt["ranking_correct"],
                       "ranking_correct_gap_ge_2pct": rt["ranking_correct_gap_ge_2pct"],
                       "rows": len(test)}
    return out


def _cal_err(m, params, cal, tc) -> float:
    from paper_1904_09538_b200 import host
    return round(host.geo_mean_rel_error(m.predict_cpu(params, cal), tc), 5)


def headline(models: dict, model: str = "") -> tuple[str | None, str | None, dict]:
    """The headline (model, GPU fit). Held-out selection: among every
    candidate model's GPU fits, the one with the lowest mean relative error
    on the workload's VALIDATION sizes; the test sizes are never consulted. Without
    validation rows (or with `model` forced): that model's GPU fit with the
    lowest CALIBRATION error."""
    cands = []
    for mname, fits in models.items():
        if model and mname != model:
            continue
        for k, v in fits.items():
            if k.startswith("gpu_") and "calibration_geomean_rel_error" in v:
                key = (v["validation_mean_rel_error"] if not model and
                       "validation_mean_rel_error" in v else v["calibration_geomean_rel_error"])
                cands.append((key, mname, k, v))
    if not cands:
        return None, None, {}
    _, mname, k, v = min(cands, key=lambda c: c[0])
    return mname, k, v


EDGE_STARTS = (3.0, 10.0, 30.0, 100.0, 300.0, 1000.0)
# (workload, model, fit) -> {application kernel id: predicted seconds} of the
# latest model_reports call (per-variant selection reads it; not reported)
APP_PREDICTIONS: dict = {}


def model_reports(parts, mean_s: dict[str, float], dev=None) -> tuple[dict, dict]:
    """Fit every model of every workload on its measured calibration rows and
    predict the held-out application rows. Three calibrations per model:
    * reference_fit: fit_model itself (the port, bit-exact with the
      reference) on the output-scaled rows (model.cpp:421-435, 485-606);
    * gpu_reference_fit: the same fit on the GPU (K17 reference mode: row-order
      sums, the reference's start and trajectory; bit-identical);
    * gpu_multistart_fit: the B200 calibration — relative residuals,
      equilibrated columns, warp-shuffle sums, the relative-residual QR start
      plus a p_edge ladder; the start with the smallest residual wins.
    All GPU fits of the round (workloads x models x starts) run in ONE K17
    launch (ps_fit_lm_jobs). Returns ({workload: {model: fits}}, K17 stats)."""
    from paper_1904_09538_b200 import host
    out: dict = {}
    jobs, where = [], []
    prep = {}
    problems = []
    for wl, cal, app in parts:
        out[wl.name] = {}
        tc = np.array([mean_s[k] for k in cal])
        ta = np.array([mean_s[k] for k in app])
        for mname, text in wl.models.items():
            m = host.HostModel(text)
            feats = m.feature_table(cal + app)
            fc = feats[: len(cal)]
            rep = {}
            p_ref = None
            if dev is None:
                # no GPU: fit_model itself (the port, bit-exact with the
                # reference); with a GPU the reference library runs the same
                # problems below (reference_library_fits) and K17's
                # reference mode reproduces it bit for bit
                try:
                    p_ref, st_ref = m.fit_cpu(fc, tc, scale=True)
                    rep["reference_fit"] = dict(_errors(wl, app, m.predict_cpu(p_ref, app), ta),
                                                fit=st_ref, calibration_geomean_rel_error=_cal_err(
                                                    m, p_ref, cal, tc))
                except Exception as e:  # a fit failure is reported, not hidden
                    rep["reference_fit"] = {"error": str(e)}
            out[wl.name][mname] = rep
            prep[(wl.name, mname)] = (m, p_ref, tc, ta, cal, app)
            problems.append({"model": text, "features": fc.tolist(), "t": tc.tolist(), "scale": True})
            if dev is None:
                continue
            fs, ts = fc / tc[:, None], np.ones_like(tc)
            jobs.append({"model": m, "features": fs, "t": ts,
                         "starts": m.initial_point(fs, ts, scale=0)[None], "mode": 0})
            where.append((wl, mname, "gpu_reference_fit"))
            p0 = m.initial_point(fc, tc, scale=2)  # relative-residual QR start
            starts = [p0]
            edges = [i for i, c in enumerate(m.cost_params) if not c]  # tanh-only params
            for e in (EDGE_STARTS if edges else ()):
                s_ = p0.copy()
                s_[edges] = e
                starts.append(s_)
            # mode 1|2|4: equilibrated columns, warp-shuffle sums, residuals
            # relative to t (weights 1/t)
            jobs.append({"model": m, "features": fc, "t": tc, "starts": np.stack(starts),
                         "mode": 7})
            where.append((wl, mname, "gpu_multistart_fit"))
    k17 = None
    if dev is not None and jobs:
        from paper_1904_09538_b200.device import fit_lm_jobs
        try:
            # one untimed warm-up launch of the same job set (module load and
            # first-launch costs; the fits are deterministic, so the timed
            # launch recomputes the same results)
            _, first_s = fit_lm_jobs(dev, jobs)
        except Exception:
            first_s = None
        t0 = time.perf_counter()
        try:
            results, ksec = fit_lm_jobs(dev, jobs)
        except Exception as e:  # reported, not hidden
            for wl, mname, key in where:
                out[wl.name][mname][key] = {"error": str(e)}
            return out, {"error": str(e)}
        wall = time.perf_counter() - t0
        nfits = sum(len(j["starts"]) for j in jobs)
        iters = sum(s["iterations"] for _, st in results for s in st)
        damped = sum(s.get("trials", 0) for _, st in results for s in st)
        k17 = {"jobs": len(jobs), "fits": nfits, "launches": 1, "kernel_s": round(ksec, 5),
               "first_launch_s": round(first_s, 5) if first_s is not None else None,
               "wall_s": round(wall, 4), "fits_per_s": round(nfits / ksec, 1),
               "lm_iterations": iters, "damped_solves": damped,
               "iterations_per_s": round(iters / ksec, 1)}
        for (wl, mname, key), (params, stats) in zip(where, results):
            m, p_ref, tc, ta, cal, app = prep[(wl.name, mname)]
            ok = [i for i, s_ in enumerate(stats) if s_["status"] == 0]
            best = min(ok, key=lambda i: stats[i]["residual_norm"]) if ok else 0
            try:
                pa = m.predict_cpu(params[best], app)
                g = dict(_errors(wl, app, pa, ta), fit=stats[best],
                         starts=len(stats),
                         calibration_geomean_rel_error=_cal_err(m, params[best], cal, tc),
                         params={n: float(v) for n, v in zip(m.params, params[best])})
                out[wl.name][mname][key] = g
                APP_PREDICTIONS[(wl.name, mname, key)] = dict(zip(app, pa))
            except Exception as e:  # e.g. a fit whose predictions go negative
                out[wl.name][mname][key] = {"error": str(e)}
        # the reference library itself on the same reference-mode problems:
        # the CPU baseline of K17 and a bitwise pin of its reference mode
        ref = reference_library_fits(problems)
        if "params_hex" in ref:
            same = total = 0
            for (wl, mname, key), (params, _st), got in zip(
                    [w for w in where if w[2] == "gpu_reference_fit"],
                    [r for w, r in zip(where, results) if w[2] == "gpu_reference_fit"],
                    ref["params_hex"]):
                total += 1
                rec = out[wl.name][mname]["gpu_reference_fit"]
                if isinstance(got, str):  # the reference raises (e.g. divergence)
                    rec["reference_library"] = {"error": got}
                    continue
                want = np.array([int(h, 16) for h in got], dtype=np.uint64).view(np.float64)
                eq = bool(np.array_equal(params[0].view(np.uint64), want.view(np.uint64)))
                same += eq
                den = np.maximum(np.abs(want), 1e-300)
                rec["reference_library"] = {"bitwise_equal": eq, "max_rel_param_diff": float(
                    np.max(np.abs(params[0] - want) / den))}
            k17["reference_library"] = {
                "fits": ref["fits"], "seconds_1thread": round(ref["seconds_1thread"], 3),
                "threads": ref["threads"], "seconds_threads": round(ref["seconds_threads"], 3),
                "fits_per_s_1thread": round(ref["fits"] / ref["seconds_1thread"], 3),
                "fits_per_s_threads": round(ref["fits"] / ref["seconds_threads"], 3),
                "gpu_reference_mode_bitwise_equal": f"{same}/{total}"}
        else:
            k17["reference_library"] = ref
    return out, k17


def reference_library_fits(problems: list[dict]) -> dict:
    """fit_model of the UNMODIFIED reference library (oracle/_ref/ref_cpu_bench
    --fits) on the given problems, 1 host thread and all host threads."""
    import tempfile
    exe = ROOT / "oracle" / "_ref" / "ref_cpu_bench"
    if not exe.exists():
        return {"unavailable": "oracle/_ref/ref_cpu_bench not built (needs /root/reference at build time)"}
    with tempfile.NamedTemporaryFile("w", suffix=".json", delete=False) as f:
        json.dump({"problems": problems}, f)
        path = f.name
    try:
        r = subprocess.run([str(exe), "--fits", path, str(os.cpu_count() or 1)], capture_output=True,
                           text=True, timeout=1800)
    finally:
        os.unlink(path)
    if r.returncode != 0:
        return {"error": r.stderr.strip()[-300:]}
    return json.loads(r.stdout)


def model_report(wl, cal, app, mean_s: dict[str, float], dev=None) -> dict:
    """model_reports for one workload."""
    return model_reports([(wl, cal, app)], mean_s, dev)[0][wl.name]


# ---------------------------------------------------------------------------
# Overlap diagnosis (executor.cpp:169-174)


def overlap_diagnosis(parts, models: dict, mean_s: dict[str, float]) -> dict:
    """classify_overlap on real work-removed timings: per application variant
    (at every size that has work-removed kernels), full time vs the sum of its
    `_rm` kernels plus the on-chip estimate of the calibrated linear model;
    'max_overlap' when that sum exceeds the full time by > 15%."""
    from paper_1904_09538_b200 import host, workloads
    onchip = [("p_f32add", workloads.OPS["add"]), ("p_f32mul", workloads.OPS["mul"]),
              ("p_f32madd", workloads.OPS["madd"]), ("p_f32l", workloads.LMEM)]

    def split(v):
        g, *p = v.split("__")
        return g, dict(x.split("-", 1) for x in p)

    out = {}
    for wl, _cal, app in parts:
        fit = models.get(wl.name, {}).get("linear", {}).get("gpu_reference_fit", {})
        if "params" not in fit:
            continue
        lin = host.HostModel(wl.models["linear"])
        feats = dict(zip(app, lin.feature_table(app)))
        per = {}
        for vid in app:
            g, a = split(vid)
            rm = [k for k in mean_s if k.startswith(g + "_rm__")
                  and all(split(k)[1].get(x) == y for x, y in a.items())]
            if not rm:
                continue
            f = dict(zip(lin.features, feats[vid]))
            est = sum(fit["params"][pn] * f.get(fn, 0.0) for pn, fn in onchip)
            full, removed = mean_s[vid], sum(mean_s[k] for k in rm)
            kind = "max_overlap" if removed + est > full * 1.15 else "linear"
            key = workloads.variant_of(vid, wl.variant_keys)
            per.setdefault(key, {})[workloads.size_of(vid, wl.size_keys)] = {
                "full_s": full, "removed_s": removed, "onchip_s": est, "kind": kind}
        out[wl.name] = per
    return out


def select_per_variant(wl, app, mean_s: dict[str, float], top: int | None = None) -> dict | None:
    """Held-out PER-VARIANT model choice (the paper models each variant with
    its own form — linear or nonlinear, PAPER.md:2444-2454 — and so may we):
    every application variant gets one of the workload's fitted (model, fit)
    candidates. Only the VALIDATION sizes decide: among the `top` candidates
    of each variant (by its validation error) the assignment that ranks the
    most validation sizes right (where the measured gap is >= 2%) wins, ties
    broken by the smallest worst per-variant validation error. The TEST sizes
    only score the result."""
    import itertools

    from paper_1904_09538_b200 import host, workloads
    cands = {k[1:]: v for k, v in APP_PREDICTIONS.items() if k[0] == wl.name}
    if not cands:
        return None
    variant = {k: workloads.variant_of(k, wl.variant_keys) for k in app}
    is_val = {k: workloads.size_of(k, wl.size_keys) in wl.validation_sizes for k in app}
    val = [k for k in app if is_val[k]]
    test = [k for k in app if not is_val[k]]
    if not val or not test:
        return None
    variants = sorted(set(variant.values()))

    def verr(c, v, keys):  # mean relative error of variant v (the selection criterion)
        ks = [k for k in keys if variant[k] == v]
        return _mean_rel([cands[c][k] for k in ks], [mean_s[k] for k in ks])

    short = {v: sorted(cands, key=lambda c: verr(c, v, val))[:top] for v in variants}
    best = None
    for combo in itertools.product(*[short[v] for v in variants]):
        asg = dict(zip(variants, combo))
        rows = [(k, cands[asg[variant[k]]][k], mean_s[k]) for k in val]
        ok, n2 = (int(x) for x in _rank(wl, rows)["ranking_correct_gap_ge_2pct"].split("/"))
        worst = max(verr(asg[v], v, val) for v in variants)
        key = (-ok, worst)
        if best is None or key < best[0]:
            best = (key, asg)
    asg = best[1]
    rows_all = [(k, cands[asg[variant[k]]][k], mean_s[k]) for k in app]
    rows_test = [r for r in rows_all if not is_val[r[0]]]
    r_all, r_test = _rank(wl, rows_all), _rank(wl, rows_test)
    rows_val = [r for r in rows_all if is_val[r[0]]]
    return {"assignment": {v: f"{c[0]}/{c[1]}" for v, c in asg.items()},
            "selection": "per-variant, held-out validation sizes (rankings first, then worst error)",
            "validation_mean_rel_error": {v: round(verr(asg[v], v, val), 5) for v in variants},
            "validation_ranking_correct_gap_ge_2pct": _rank(wl, rows_val)["ranking_correct_gap_ge_2pct"],
            "geomean_rel_error": _per_variant(wl, rows_all),
            "geomean_rel_error_all": round(host.geo_mean_rel_error(
                [p for _, p, _ in rows_all], [t for _, _, t in rows_all]), 5),
            "ranking_correct": r_all["ranking_correct"],
            "ranking_correct_gap_ge_2pct": r_all["ranking_correct_gap_ge_2pct"],
            "test": {"geomean_rel_error": _per_variant(wl, rows_test),
                     "geomean_rel_error_all": round(host.geo_mean_rel_error(
                         [p for _, p, _ in rows_test], [t for _, _, t in rows_test]), 5),
                     "ranking_correct": r_test["ranking_correct"],
                     "ranking_correct_gap_ge_2pct": r_test["ranking_correct_gap_ge_2pct"],
                     "rows": len(rows_test)},
            "ranking": r_all["ranking"]}


def _acc(h: dict) -> dict:
    """The headline accuracy record of one application (per-variant choice
    if made, else the single model)."""
    return h.get("per_variant") or h


def _best_fit(fits: dict) -> dict:
    """A model's GPU fit with the lowest calibration error."""
    c = [v for k, v in fits.items() if k.startswith("gpu_") and "params" in v
         and "calibration_geomean_rel_error" in v]
    return min(c, key=lambda v: v["calibration_geomean_rel_error"]) if c else {}


def paper_selection(parts, models: dict, diagnosis: dict, mean_s: dict[str, float]) -> dict:
    """The paper's per-variant model choice:
    the work-removal diagnosis (overlap_diagnosis, classify_overlap
    executor.cpp:169-174) labels each application variant 'linear' or
    'max_overlap' by majority over its sizes; a linear variant is predicted by
    the linear model (Eq. 1), an overlapping one by the nonlinear model
    (Eqs. 4-5), each with its best GPU fit."""
    from paper_1904_09538_b200 import host, workloads
    out = {}
    for wl, _cal, app in parts:
        diag = diagnosis.get(wl.name, {}) if isinstance(diagnosis, dict) else {}
        fits = {m: _best_fit(models.get(wl.name, {}).get(m, {})) for m in ("linear", "nonlinear")}
        if not all(fits.values()) or not diag:
            continue
        choice = {}
        for var, by_size in diag.items():
            kinds = [v["kind"] for v in by_size.values()]
            choice[var] = "nonlinear" if kinds.count("max_overlap") * 2 > len(kinds) else "linear"
        pred = {}
        for mname in set(choice.values()):
            m = host.HostModel(wl.models[mname])
            p = np.array([fits[mname]["params"][n] for n in m.params])
            pred[mname] = dict(zip(app, m.predict_cpu(p, app)))
        rows = [(vid, pred[choice.get(workloads.variant_of(vid, wl.variant_keys), "linear")][vid]
                 if choice.get(workloads.variant_of(vid, wl.variant_keys), "linear") in pred
                 else pred[next(iter(pred))][vid], mean_s[vid]) for vid in app]
        r = _rank(wl, rows)
        out[wl.name] = {"choice": choice, "geomean_rel_error": _per_variant(wl, rows),
                        "geomean_rel_error_all": round(host.geo_mean_rel_error(
                            [p for _, p, _ in rows], [t for _, _, t in rows]), 5),
                        "ranking_correct": r["ranking_correct"],
                        "ranking_correct_gap_ge_2pct": r["ranking_correct_gap_ge_2pct"]}
    return out


# ---------------------------------------------------------------------------
# K16: the extra tcgen05 dense-contraction variant (not a paper variant)


def tensor_variant_report(dev, n: int = 8192, trials: int = 10) -> dict:
    """matmul_sq_tc (tcgen05 kind::tf32, A K-major and B N-major from HBM) at
    n, timed like every suite kernel, next to cuBLAS TF32 (torch.matmul with
    TF32 allowed) on the same shape, both with CUDA events."""
    from paper_1904_09538_b200 import desc_from_id, kernel_io
    vid = f"matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-{n}"
    d = desc_from_id(vid)
    io = kernel_io(d)
    dev.prepare(d)
    dev.measure(d, trials=3, warmup=0)
    mean, kept = dev.measure_summary(d, trials=trials, warmup=2)
    ours = io.flops / mean / 1e12
    out = {"kernel": vid, "n": n, "tflops": round(ours, 1), "ms": round(mean * 1e3, 4),
           "dtype": "tf32 operands, fp32 accumulate",
           "note": "A K-major, B N-major straight from row-major B (128B swizzle, 32B atoms); "
                   "no transpose"}
    pk, _src = peaks()
    tf32_peak = pk.get("bf16_tflops", 1598.1) / 2
    out["roofline"] = {"bound": "tensor", "achieved": round(ours, 1), "peak": round(tf32_peak, 1),
                       "unit": "TFLOP/s", "frac": round(ours / tf32_peak, 4),
                       "peak_source": "MEASURED_PEAKS.json bf16 dense / 2 (TF32 is half the "
                                      "bf16 tensor rate)",
                       "frac_vs_nominal": round(ours / 1100.0, 4),
                       "nominal_source": "B200_PROFILING.md tf32 dense 1.1 PFLOP/s"}
    try:
        import torch
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.rand(n, n, device=f"cuda:{dev.device}", dtype=torch.float32)
        b = torch.rand(n, n, device=f"cuda:{dev.device}", dtype=torch.float32)
        for _ in range(3):
            torch.matmul(a, b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(trials):
            torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        cub = e0.elapsed_time(e1) / 1e3 / trials
        out["cublas_tf32_tflops"] = round(2.0 * n ** 3 / cub / 1e12, 1)
        out["vs_cublas"] = round(ours / out["cublas_tf32_tflops"], 3)
        del a, b
        torch.cuda.empty_cache()
    except Exception as e:  # reported, not hidden
        out["cublas_tf32_tflops"] = None
        out["cublas_error"] = str(e)
    return out


def dg_tensor_variant_report(dev, mean_s: dict[str, float], nel: int = 1_000_000,
                             trials: int = 10) -> dict:
    """dg_diff_tc (K19: DG as a tcgen05 kind::tf32 contraction) at nel and every
    order's padded Np, timed like every suite kernel, against its HBM roofline
    (u in + res out + dm, MEASURED_PEAKS.json) and the fastest paper variant of
    the same size from this run's sweep."""
    from paper_1904_09538_b200 import desc_from_id, kernel_io
    pk, src = peaks()
    rows = {}
    for np_ in (16, 32, 48, 64, 96, 128):
        vid = f"dg_diff_tc__dtype-float32__nelements-{nel}__nmatrices-3__nunit_nodes-{np_}"
        io = kernel_io(desc_from_id(vid))
        dev.prepare(vid)
        dev.measure(vid, trials=3, warmup=0)
        mean, _ = dev.measure_summary(vid, trials=trials, warmup=2)
        best = min(((t, k) for k, t in mean_s.items()
                    if k.startswith("dg_diff__") and f"__nelements-{nel}__" in k
                    and f"__nunit_nodes-{np_}__" in k), default=(None, None))
        gbs = io.bytes_global / mean / 1e9
        rows[str(np_)] = {"ms": round(mean * 1e3, 4), "GBps": round(gbs, 1),
                          "hbm_frac": round(gbs / pk["hbm_gbs"], 4),
                          "tflops": round(io.flops / mean / 1e12, 1),
                          "best_paper_variant": best[1].rsplit("variant-", 1)[-1] if best[1] else None,
                          "speedup_vs_best_paper_variant": round(best[0] / mean, 2) if best[0] else None}
    return {"kernel": f"dg_diff_tc__dtype-float32__nelements-{nel}__nmatrices-3__nunit_nodes-*",
            "bound": "hbm", "peak_GBps": pk["hbm_gbs"], "peak_source": src,
            "dtype": "tf32 operands, fp32 accumulate", "by_nunit_nodes": rows}


# ---------------------------------------------------------------------------
# C5: the calibrated models evaluated over a large variant space (K18)


def _concrete(vid: str, sizes: dict[str, int]) -> str:
    gen, *parts = vid.split("__")
    args = dict(p.split("-", 1) for p in parts)
    args.update({k: str(v) for k, v in sizes.items()})
    return "__".join([gen] + [f"{k}-{args[k]}" for k in sorted(args)])


def c5_block(npts: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of the C5 points evaluated by `rank` (SURVEY 8(e):
    10^6 points in blocks of 125k per GPU at 8 GPUs)."""
    per = -(-npts // world)
    return min(npts, rank * per), min(npts, (rank + 1) * per)


def c5_variants(parts, models: dict, heads: dict) -> list[dict]:
    """One entry per application variant: its workload's headline model,
    fitted parameters, argmin group and size-coordinate map."""
    from paper_1904_09538_b200 import host, workloads
    variants = []
    for g, (wl, _cal, app) in enumerate(parts):
        h = heads[wl.name]
        asg = (h.get("per_variant") or {}).get("assignment", {})
        seen = set()
        for vid in app:
            key = workloads.variant_of(vid, wl.variant_keys)
            if key in seen:
                continue
            seen.add(key)
            # the variant's own (model, fit) when chosen per variant, else the
            # workload's single headline
            mname, fname = asg[key].split("/") if key in asg else (h["model"], h["fit"] or "")
            fit = models[wl.name].get(mname, {}).get(fname, {})
            if "params" not in fit:
                raise RuntimeError(f"{wl.name}: no fitted parameters for {key}")
            m = host.HostModel(wl.models[mname])
            variants.append({"id": vid, "model": wl.models[mname],
                             "params": [fit["params"][n] for n in m.params],
                             "group": g, "coords": wl.c5_coords})
    return variants


def c5_report(dev, parts, variants: list[dict], npts: int = 1_000_000, dist=None) -> dict | None:
    """Every application variant of every workload, with its workload's
    headline model and fitted parameters, evaluated at npts seeded points
    (BASELINE.json configs[4]); winners per application. Each rank evaluates
    one contiguous block of points (c5_block); predictions and argmins are
    all-gathered (NCCL over NVLink on GPUs) and rank 0 checks them against
    the CPU port of the same tables and against the reference-API predict()."""
    from paper_1904_09538_b200 import host, workloads
    from paper_1904_09538_b200.predict import PredictionTables, c5_points
    rank, world = (dist.rank, dist.world) if dist else (0, 1)
    t = PredictionTables(variants)
    pts = c5_points(npts)
    lo, hi = c5_block(npts, rank, world)
    # the rank's points and results in page-locked host buffers (filled
    # before the timed region, like the suite's e2e inputs)
    ppts, ppred, parg, _keep = t.pinned_buffers(hi - lo)
    ppts[:] = pts[lo:hi]
    err = None
    jit_s = None
    try:
        # the tables' specialised kernel (NVRTC), compiled and loaded before
        # the timed call; the seconds are reported, not hidden
        jit_s = t.prepare_gpu(dev)
        # warm at the timed size (device buffers, streams and events exist)
        t.eval_gpu(dev, ppts, out=(ppred, parg))
    except Exception as e:  # every rank learns of it before the collectives
        err = e
    if dist and dist.max(float(err is not None)) > 0:
        raise RuntimeError(f"C5 evaluation failed on a rank: {err}")
    if err is not None:
        raise err
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    pg, ag, ksec = t.eval_gpu(dev, ppts, out=(ppred, parg))
    wall = time.perf_counter() - t0
    pg, ag = np.array(pg), np.array(ag)
    if dist and dist.world > 1:
        pg = dist.all_gather_rows(pg)
        ag = dist.all_gather_rows(ag.astype(np.float64)).astype(np.int64)
        ksec, wall = dist.max(ksec), dist.max(wall)
    if rank != 0:
        return None
    nsub = min(npts, 100_000)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    pc, ac = t.eval_cpu(pts[:nsub], threads=threads)
    cpu = time.perf_counter() - t0
    rel = float(np.max(np.abs(pg[:nsub] - pc) / np.abs(pc)))
    # ranking agreement, excluding exact near-ties
    mism = 0
    for g in range(t.ngroups):
        cols = [i for i, v in enumerate(variants) if v["group"] == g]
        srt = np.sort(pc[:, cols], axis=1)
        tie = (srt[:, 1] - srt[:, 0]) <= 1e-12 * np.abs(srt[:, 0])
        mism += int(np.sum((ag[:nsub, g] != ac[:, g]) & ~tie))
    # reference-API predict() (features through evaluate_feature, one kernel
    # instance per point) on a sample, one batched call per variant
    nref = 256
    t0 = time.perf_counter()
    ref_rel = 0.0
    for v, var in enumerate(variants):
        m = host.HostModel(var["model"])
        ids = [_concrete(var["id"], {k: int(pts[j, c]) for k, c in var["coords"].items()})
               for j in range(nref)]
        r = m.predict_cpu(np.array(var["params"]), ids)
        ref_rel = max(ref_rel, float(np.max(np.abs(pg[:nref, v] - r) / np.abs(r))))
    ref_t = time.perf_counter() - t0
    winners = {}
    for g, (wl, _c, _a) in enumerate(parts):
        cols = [i for i, v in enumerate(variants) if v["group"] == g]
        cnt = np.bincount(ag[:, g], minlength=t.nvar)  # argmin holds global variant indices
        winners[wl.name] = {workloads.variant_of(variants[i]["id"], wl.variant_keys): int(cnt[i])
                            for i in cols}
    nev = npts * t.nvar
    return {"points": npts, "variants": t.nvar, "evaluations": nev, "ranks": world,
            "points_per_rank": hi - lo,
            "jit_compile_s": round(jit_s, 3) if jit_s is not None else None,
            "gpu_kernel_ms": round(ksec * 1e3, 3),
            "gpu_evals_per_s": round(nev / ksec, 1),
            "gpu_e2e_ms": round(wall * 1e3, 2), "gpu_e2e_evals_per_s": round(nev / wall, 1),
            "cpu_tables_evals_per_s": round(nsub * t.nvar / cpu, 1), "cpu_threads": threads,
            "cpu_max_rel_diff": rel, "argmin_mismatches_vs_cpu": mism,
            # the port's reference-API predict() (features through
            # evaluate_feature per point): a correctness pin; the reference
            # LIBRARY's own predict rate is cpu_baseline_reference
            "port_predict_evals_per_s": round(nref * t.nvar / ref_t, 1),
            "port_predict_max_rel_diff": ref_rel,
            "port_predict_sample": f"{nref} points x {t.nvar} variants through ps_predict_cpu",
            "winners": winners}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle restatement (oracle/suite_ref.c) on host cores


def reference_model_sample(seconds: float = 2.0) -> dict:
    """The unmodified reference library (oracle/_ref, compiled from
    /root/reference by oracle/Makefile; travels prebuilt) timed on the host
    cores for the modelling half of the path: analyze, gather_feature_values,
    fit_model and predict (oracle/ref_cpu_bench.cpp)."""
    exe = ROOT / "oracle" / "_ref" / "ref_cpu_bench"
    if not exe.exists():
        return {"unavailable": "oracle/_ref/ref_cpu_bench not built (needs /root/reference at build time)"}
    r = subprocess.run([str(exe), str(seconds)], capture_output=True, text=True, timeout=300)
    if r.returncode != 0:
        return {"error": r.stderr.strip()[-300:]}
    return json.loads(r.stdout)


WORKLOAD_FILE = ROOT / "tests" / "golden" / "workload_{}.json"


def workload_doc(name: str) -> dict:
    """The workload's kernel ids as committed by tools/gen_workload_list.py
    (the B200 catalog's expansion; tests/test_variants_cpu.py keeps it
    current). Lets the reference arm run the same workload without loading
    the product library."""
    return json.loads(Path(str(WORKLOAD_FILE).format(name)).read_text())


def bench_config(workload: str, n_kernels: int, n_cal: int, n_app: int, trials: int,
                 world: int) -> dict:
    """The `config` object of BOTH arms' lines (the driver compares them)."""
    return {"workload": workload, "kernels": n_kernels, "calibration_kernels": n_cal,
            "application_kernels": n_app, "trials_per_kernel": trials,
            "l2": "no flush; HBM microbenchmarks use >= 1 GiB arrays (> 126 MB L2); trials of a "
                  "kernel back to back as measure_kernel runs them (executor.cpp:40-48)",
            "parallelism": f"(kernel, trial) units LPT-sharded over {world} rank(s)"}


def reference_sample(kernels: list[str]) -> list:
    """Bounded CPU sample of a workload for the oracle restatement: every
    kernel except the cubic-cost ones above n = 1024 and DG above 10^5
    elements, with the HBM arrays shrunk to 2^24 elements (still larger than
    the host LLC). Descriptors come from oracle/variants.py, not the product."""
    from oracle import variants
    sample = []
    for vid in kernels:
        d = variants.parse(vid)
        if d.gen in (7, 8) and d.n > 1024:
            continue
        if d.gen in (1, 6) and d.nelements > (1 << 24):
            continue
        if d.gen == 2 and d.nelements > (1 << 20):
            continue
        if d.gen in (11, 12) and d.nel > 100000:
            continue
        sample.append((vid, d, variants.io_of(d)))
    for k in (1, 2):
        vid = ("gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16"
               f"__lsize_1-16__n_input_arrays-{k}__nelements-{1 << 24}")
        d = variants.parse(vid)
        sample.append((vid, d, variants.io_of(d)))
    return sample


def time_reference_sample(sample: list, warmup: int, steps: int, threads: int | None = None):
    """oracle/suite_ref.c (OpenMP) over the sample: (GB/s, seconds, cores)."""
    from oracle import suite as oracle_suite
    if threads:
        oracle_suite.set_threads(threads)
    rng = np.random.default_rng(0)
    inputs = {}
    for vid, d, io in sample:
        dt = np.float32 if io.elem_bytes == 4 else np.float64
        inputs[vid] = [rng.random(n).astype(dt) for n in io.input_elems]
    for _ in range(warmup):
        for vid, d, io in sample:
            oracle_suite.run(d, io, inputs[vid])
    t0 = time.perf_counter()
    nbytes = 0.0
    for _ in range(steps):
        for vid, d, io in sample:
            oracle_suite.run(d, io, inputs[vid])
            nbytes += io.bytes_global
    dt = time.perf_counter() - t0
    return nbytes / dt / 1e9, dt, oracle_suite.threads()


def sample_note(sample: list, workload: str) -> str:
    return (f"{len(sample)} kernels of the {workload} workload (matmul n<=1024, DG nel<=1e5, "
            "HBM arrays 2^24) through oracle/suite_ref.c, OpenMP")


def run_reference_arm(args, dist: Dist) -> None:
    """bench.py --impl reference: the reference has no GPU code (SPEC.md:16,
    597); its CPU implementation of this path is timed on the host cores — the
    kernel restatement (oracle/suite_ref.c) over a bounded sample of the SAME
    workload, same config/metric/unit as our arm. Never loads the product
    library: ids come from the committed workload file, descriptors from
    oracle/variants.py."""
    if dist.rank != 0:
        return
    doc = workload_doc(args.workload)
    kernels = doc["kernels"]
    apps = {k for a in doc["applications"].values() for k in a["application"]}
    sample = reference_sample(kernels)
    value, dt, cores = time_reference_sample(sample, args.warmup, args.steps,
                                             threads=os.cpu_count() or 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (deterministic seed pattern, tests/support.hpp:35-44)",
        "config": bench_config(args.workload, len(kernels), len(kernels) - len(apps), len(apps),
                               args.steps * args.trials_per_step, args.gpus),
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores,
                         "kind": "port", "sample": sample_note(sample, args.workload)},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


# ncu evidence of the pipe that binds each CUDA-core application kernel
# (profiles/r01_ncu_summary.csv): the paper variants are L1/shared-pipe bound
# by their access semantics, not FP32 bound.
BINDING = {
    7: "L1/TEX: 97% (noPF n=8192, panel order; b loads 64 B per warp per madd) / 95% (PF, LDS "
       "wavefronts); FMA pipe 14-16%",
    11: "L1/TEX 96-97% (noPF, dmPF, profiles/r01_ncu_summary_dg_skew.csv), 88-96% (uPF, "
        "dmPFtrans); FMA pipe 14-26%",
    9: "HBM 5.1 TB/s of 6.56 (dram read+write 483 MB vs 535 MB algorithmic)",
}


def run_ours(args, dist: Dist) -> None:
    from paper_1904_09538_b200 import desc_from_id, kernel_io
    from paper_1904_09538_b200.device import CudaDevice, PinnedArray

    parts, kernels = workload_kernels(args.workload)
    descs = [desc_from_id(k) for k in kernels]
    ios = [kernel_io(d) for d in descs]
    prev = previous_run_seconds()
    est = [prev.get(k) or estimate_seconds(io) for k, io in zip(kernels, ios)]
    units = [(i, t) for i in range(len(kernels)) for t in range(args.trials_per_step)]
    shards = lpt(units, est, dist.world)
    mine = shards[dist.rank]
    # a kernel whose trials are split over ranks runs its e2e pass on exactly
    # one of them: the rank holding its first trial
    e2e_owner = {i: r for r, sh in enumerate(shards) for i, t in sh if t == 0}
    my_kernels = sorted({i for i, _ in mine})

    dev = CudaDevice(dist.device)
    for i in my_kernels:  # fill once; inputs stay resident in HBM
        dev.prepare(descs[i])
    for _ in range(args.warmup):
        for i, _t in mine:
            dev.measure(descs[i], trials=1, warmup=0)

    sampler = ClockSampler(dist.device)
    sampler.start()
    time.sleep(0.5)
    dist.barrier()
    dev.mark(0)
    t_wall = time.perf_counter()
    records: list[tuple[int, int, float]] = []
    # Consecutive trials of one kernel run back to back (paper methodology,
    # 60 trials back to back); ps_measure times each launch with events.
    per_kernel = {}
    for i, _t in mine:
        per_kernel[i] = per_kernel.get(i, 0) + 1
    # a short kernel gets one untimed launch before its trials: the first
    # launch after a switch of kernel pays the switch (code fetch, cold
    # L2/TLB, ~2-4 us), which the paper's back-to-back trials after warm-up
    # never see; above 200 us it is < 2% of one trial (< 0.5% of the mean of
    # a step's four) while the extra launches would lengthen the step (3% at
    # a 2 ms threshold)
    warm = {i: 1 if est[i] < 2e-4 else 0 for i in per_kernel}
    # launches of the timed sweep: trials + warm-ups + one queue-ahead kernel
    # per ps_measure call
    sweep_launches = args.steps * sum(cnt + warm[i] + 1 for i, cnt in per_kernel.items())
    from paper_1904_09538_b200.host import trace
    with trace("bench: timed sweep"):
        for step in range(args.steps):
            for i, cnt in per_kernel.items():
                for j, s in enumerate(dev.measure(descs[i], trials=cnt, warmup=warm[i])):
                    records.append((i, step * args.trials_per_step + j, s))
    dev.mark(1)
    elapsed = dev.elapsed(0, 1)
    wall = time.perf_counter() - t_wall
    dist.barrier()
    sweep_launches_all = dist.sum(float(sweep_launches))
    clocks = sampler.stop()

    elapsed_max = dist.max(elapsed)
    table = dist.gather_table(records)

    # cross-rank timing agreement (SURVEY 8(e) caveat): every rank times the
    # same HBM stream; the table is only comparable across GPUs if they agree
    ref_vid = ("gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16"
               "__lsize_1-16__n_input_arrays-2__nelements-268435456")
    ref_mean, _ = dev.measure_summary(desc_from_id(ref_vid), trials=10, warmup=2)
    per_rank = dist.all_gather_rows(np.array([[ref_mean]]))[:, 0]
    cross_rank = {"kernel": ref_vid, "seconds_per_rank": [round(float(x), 9) for x in per_rank],
                  "max_over_min": round(float(per_rank.max() / per_rank.min()), 4)}

    # the sweep's resident arrays are no longer needed: the e2e pass places
    # every kernel's arrays in one device arena instead
    dev.trim()
    # e2e through host buffers (ps_run_host: H2D + kernel + D2H per launch)
    # every kernel of the sweep (the same workload as `value`), each on the
    # rank holding its first trial
    e2e_set = [i for i in my_kernels if e2e_owner.get(i) == dist.rank]
    # pinned host memory: ranks on one host share its RAM; the output arrays
    # (only the e2e_full_outputs pass needs them) are dropped first if the
    # rank's share would be exceeded
    import psutil
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    pin_budget = 0.8 * psutil.virtual_memory().available / local_ranks
    need_in = sum(int(ios[i].input_elems[j]) * ios[i].elem_bytes
                  for i in e2e_set for j in range(ios[i].n_inputs))
    need_out = sum(int(ios[i].output_elems[j]) * ios[i].elem_bytes
                   for i in e2e_set for j in range(ios[i].n_outputs))
    # every rank leaves together: a rank that cannot pin its inputs must not
    # strand the others in the next collective
    if dist.max(float(need_in > pin_budget)) > 0:
        raise SystemExit(f"rank {dist.rank}: e2e inputs need {need_in / 1e9:.1f} GB pinned host "
                         f"memory, {pin_budget / 1e9:.1f} GB available to this rank "
                         "(or another rank's share was exceeded)")
    full_outputs = need_in + need_out <= pin_budget
    pinned = {}
    h2d = d2h = 0
    for i in e2e_set:
        io = ios[i]
        ins = [PinnedArray(int(io.input_elems[j]) * io.elem_bytes) for j in range(io.n_inputs)]
        outs = [PinnedArray(int(io.output_elems[j]) * io.elem_bytes)
                for j in range(io.n_outputs)] if full_outputs else []
        for a in ins:
            a.numpy(np.uint8)[:] = 0x3f
        pinned[i] = (ins, outs)
        h2d += sum(a.nbytes for a in ins)
        d2h += sum(a.nbytes for a in outs)
    # one pipelined pass per step (ps_run_host_batch_ex: H2D of the next
    # kernel, this launch and the previous read-back overlap on three streams).
    # e2e: the step's result read back is one device checksum per kernel (the
    # sweep's product is its timing table, the output arrays are scratch);
    # e2e_full_outputs: every output array copied back as well.
    # Order the batch by Johnson's rule for the two-stage flow shop copy-in ->
    # launch (the device arena gives the copy engine unlimited lookahead, so
    # this order minimises the pass's makespan): kernels whose copy is shorter
    # than their run first, by increasing copy time (the SMs start at once
    # and the copy engine gets ahead), then the copy-dominated ones by
    # decreasing run time. The product is per kernel, so the order within a
    # step is free.
    def copy_s(i: int) -> float:
        return sum(a.nbytes for a in pinned[i][0]) / 50e9

    def run_s(i: int) -> float:
        return prev.get(kernels[i]) or est[i]
    first = sorted((i for i in e2e_set if copy_s(i) < run_s(i)), key=copy_s)
    last = sorted((i for i in e2e_set if copy_s(i) >= run_s(i)), key=run_s, reverse=True)
    e2e_set = first + last
    batch = [descs[i] for i in e2e_set]
    b_in = [pinned[i][0] for i in e2e_set]
    b_out = [pinned[i][1] for i in e2e_set]
    if e2e_set:  # warm (allocates the pipeline slots)
        dev.run_host_batch(batch, b_in, None, checksums=True)
        if full_outputs:
            dev.run_host_batch(batch, b_in, b_out)
    dist.barrier()
    e2e_time = e2e_full_time = 0.0
    e2e_bytes = 0.0
    last_sums = None
    with trace("bench: e2e through host buffers"):
        for _ in range(args.steps):
            if e2e_set:
                dt, last_sums = dev.run_host_batch(batch, b_in, None, checksums=True)
                e2e_time += dt
                if full_outputs:
                    e2e_full_time += dev.run_host_batch(batch, b_in, b_out)
            e2e_bytes += sum(ios[i].bytes_global for i in e2e_set)
    # the pipelined pass's per-kernel checksums at bench size against a
    # single launch of the same kernel on the same host inputs (ps_run_verify,
    # no arena, no overlap): checks the ring placement, the stream ordering
    # and the checksum reduction at the sizes the bench times (kernel values
    # themselves are pinned by the parity tests)
    e2e_verified = [0, 0]
    if e2e_set and last_sums is not None:
        big = sorted(range(len(e2e_set)), key=lambda p_: -ios[e2e_set[p_]].bytes_global)[:6]
        spread = list(range(0, len(e2e_set), max(1, len(e2e_set) // 6)))[:6]
        for pos in sorted(set(big + spread)):
            i = e2e_set[pos]
            dt = np.float32 if ios[i].elem_bytes == 4 else np.float64
            # ps_run_verify on views of the pinned inputs; pageable outputs
            # (the pinned budget is spent on the inputs)
            outs = dev.run(descs[i], [a.numpy(dt) for a in pinned[i][0]])
            want = sum(int(np.sum(o.view(np.uint32), dtype=np.uint64)) for o in outs) % (1 << 64)
            e2e_verified[0] += int(int(last_sums[pos]) == want)
            e2e_verified[1] += 1
            del outs
    e2e_verified = [int(dist.sum(float(x))) for x in e2e_verified]
    e2e_time_max = dist.max(e2e_time)
    e2e_full_time_max = dist.max(e2e_full_time)
    d2h_full = d2h
    d2h = 8 * len(e2e_set)
    e2e_bytes_all = e2e_bytes
    # per step: the checksum pass (each kernel + one checksum per output
    # array) and, when it runs, the full-output pass
    e2e_launches = (len(e2e_set) * (2 if full_outputs else 1)
                    + sum(ios[i].n_outputs for i in e2e_set))
    e2e_kernels = len(e2e_set)
    full_all = float(full_outputs)
    if dist.pg:
        import torch
        devn = f"cuda:{dist.device}" if dist.backend == "nccl" else "cpu"
        t = torch.tensor([e2e_bytes, float(h2d), float(d2h), float(d2h_full), float(e2e_launches),
                          float(e2e_kernels), 1.0 - full_all], dtype=torch.float64, device=devn)
        dist.pg.all_reduce(t)
        e2e_bytes_all, h2d, d2h, d2h_full, e2e_launches, e2e_kernels, missing = t.tolist()
        full_all = float(missing == 0)
    for ins, outs in pinned.values():
        for a in ins + outs:
            a.free()
    # give the fits, the prediction tables and the variant reports the HBM
    # the e2e arena held
    dev.trim()

    # ----- measurement table -> summaries (every rank holds the gathered table) -----
    trials: dict[int, list[float]] = {}
    for k, _t, s in table:
        trials.setdefault(k, []).append(s)
    mean_s = {}
    bytes_all = 0.0
    for k, ts in trials.items():
        mean_s[kernels[k]] = summarize(ts)[0]
        bytes_all += ios[k].bytes_global * len(ts)
    value = bytes_all / elapsed_max / 1e9

    # HBM-class and FLOP-class views of the same timed launches
    hbm_b = hbm_t = fl = fl_t = 0.0
    for k, ts in trials.items():
        if descs[k].gen in (1, 6):
            hbm_b += ios[k].bytes_global * len(ts)
            hbm_t += sum(ts)
        if descs[k].gen in (2, 7):
            fl += ios[k].flops * len(ts)
            fl_t += sum(ts)

    # roofline of the dominant kernel (largest share of the timed device time)
    pk, src = peaks()
    share = {k: sum(ts) for k, ts in trials.items()}
    total_t = sum(share.values())
    sm_mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    fp32_peak_tf = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12  # CUDA-core FFMA, measured clock

    def roofline_of(k: int) -> dict:
        avg = sum(trials[k]) / len(trials[k])
        d = descs[k]
        if d.gen in (1, 6, 9, 10):  # streaming kernels: HBM roofline
            achieved = ios[k].bytes_global / avg / 1e9
            traffic = None
            tf = ROOT / "profiles" / "ncu_traffic.json"
            if tf.exists():
                traffic = json.loads(tf.read_text()).get(kernels[k])
            return {"kernel": kernels[k], "bound": "hbm", "achieved": round(achieved, 1),
                    "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                    "traffic": traffic, "peak_source": src,
                    "algorithmic_bytes_per_launch": ios[k].bytes_global,
                    "share_of_step": round(share[k] / total_t, 4)}
        achieved = ios[k].flops / avg / 1e12
        traffic = None
        tf = ROOT / "profiles" / "ncu_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(kernels[k])
        l1 = None
        if d.gen == 7 and d.dtype == 0:
            # one work-item per thread: every madd reads an a and a b operand
            # through the L1/shared data path (global loads in noPF, a_fetch /
            # b_fetch local loads in PF) — 8 B per madd, 8 n^3 per launch —
            # against 148 SMs x 128 B/clk at the run's SM clock
            ob = 8.0 * float(d.n) ** 3
            l1_peak = 148 * 128 * sm_mhz * 1e6 / 1e12
            l1 = {"bound": "l1", "achieved": round(ob / avg / 1e12, 2), "peak": round(l1_peak, 2),
                  "unit": "TB/s", "frac": round(ob / avg / 1e12 / l1_peak, 4),
                  "operand_bytes_per_launch": ob,
                  "basis": "IR operand loads per madd (a and b, work-item granularity) x 4 B; "
                           "ncu l1tex throughput 97% (noPF, panel order) / 95% (PF) agrees"}
        return {"kernel": kernels[k], "bound": "fp32", "achieved": round(achieved, 3),
                "binding_roofline": l1,
                "peak": round(fp32_peak_tf, 2), "unit": "TFLOP/s",
                "frac": round(achieved / fp32_peak_tf, 4), "traffic": traffic,
                "binding_pipe": BINDING.get(d.gen),
                "peak_source": "148 SMs x 128 FP32 lanes x 2 x median SM clock of the run "
                               "(SURVEY 8(d) C2; no tensor cores in the paper variants)",
                "algorithmic_flops_per_launch": ios[k].flops,
                "share_of_step": round(share[k] / total_t, 4),
                "traffic_note": ("matmul noPF: work-groups run in panels of 64 block columns "
                                 "(a wave's b columns fit L2): 2.8 GB of DRAM per launch at "
                                 "n = 8192 against 0.8 GB compulsory (12 n^2), 60 GB in row-major "
                                 "order (profiles/r02_ncu_summary_mm_panel.csv, DESIGN.md K9)")
                if d.gen == 7 else None,
                "note": "16x16 CUDA-core tiles by construction (uipick.cpp:464-554); the paper "
                        "reports 8-20% of FP32 peak for these variants (PAPER.md:2155-2157)"}

    dom = max(share, key=share.get)
    roofline = roofline_of(dom)
    # every kernel family against its binding resource (best size per family)
    from paper_1904_09538_b200.rooflines import best_per_family, rows_of
    suite_rows = rows_of(mean_s, sm_mhz * 1e6, pk)
    suite_rooflines = {fam: {"bound": r[1], "achieved": round(r[2], 2), "peak": round(r[3], 2),
                             "unit": r[4], "frac": round(r[5], 4), "kernel": r[0]}
                       for fam, r in sorted(best_per_family(suite_rows).items())}
    # every kernel with a throughput roofline against its binding resource,
    # weighted by its time in the step (every kernel runs the same number of
    # trials); the rest of the step is work-removed calibration kernels and
    # latency microbenchmarks, which claim no roofline
    cov = [r for r in suite_rows if r[5] == r[5]]
    t_all, t_cov = sum(r[6] for r in suite_rows), sum(r[6] for r in cov)
    suite_binding = {"time_weighted_frac": round(sum(r[6] * r[5] for r in cov) / t_cov, 4),
                     "step_share": round(t_cov / t_all, 4), "kernels": len(cov)} if cov else None
    gm = [k for k in trials if descs[k].gen == 1]
    roofline_hbm = roofline_of(max(gm, key=lambda k: ios[k].bytes_global)) if gm else None

    if args.table and dist.rank == 0:
        # measurements_to_csv format (executor.cpp:279-295) + raw trials
        with open(args.table, "w") as f:
            f.write("kernel,bindings,mean_seconds,trials,raw\n")
            for k, ts in sorted(trials.items()):
                m, kept = summarize(ts)
                f.write(f"{kernels[k]},,{m!r},{kept},{' '.join(repr(x) for x in ts)}\n")
    # the fit runs once (rank 0); its headline parameters go to every rank
    models, heads, k17 = {}, {}, None
    if dist.rank == 0:
        with trace("bench: calibration fits (K17)"):
            models, k17 = model_reports(parts, mean_s, dev)
        for wl, cal, app in parts:
            forced = args.headline_model if args.headline_model in wl.models else ""
            hmodel, hfit, head = headline(models[wl.name], forced)
            if hmodel is None:  # no candidate fitted: fall back to the workload default
                hmodel = wl.headline_model
            pv = None if forced else select_per_variant(wl, app, mean_s)
            heads[wl.name] = {"model": hmodel, "fit": hfit, "per_variant": pv,
                              "selection": ("forced" if forced else
                                            "held-out validation sizes" if
                                            "validation_mean_rel_error" in head
                                            else "calibration error"),
                              "validation_mean_rel_error": head.get(
                                  "validation_mean_rel_error"),
                              "geomean_rel_error": head.get("geomean_rel_error"),
                              "geomean_rel_error_all": head.get("geomean_rel_error_all"),
                              "ranking_correct": head.get("ranking_correct"),
                              "ranking_correct_gap_ge_2pct": head.get("ranking_correct_gap_ge_2pct"),
                              "test": head.get("test")}
    try:
        variants = c5_variants(parts, models, heads) if dist.rank == 0 else None
        err = None
    except Exception as e:  # reported, not hidden
        variants, err = None, str(e)
    variants, err = dist.broadcast((variants, err))
    try:
        with trace("bench: variant-space prediction (K18)"):
            model_eval = (c5_report(dev, parts, variants, args.c5_points, dist)
                          if args.c5_points and variants else ({"error": err} if err else None))
    except Exception as e:  # reported, not hidden
        model_eval = {"error": str(e)}
    if dist.rank != 0:
        dev.close()
        return
    try:
        diagnosis = overlap_diagnosis(parts, models, mean_s)
    except Exception as e:
        diagnosis = {"error": str(e)}
    try:
        paper = paper_selection(parts, models, diagnosis, mean_s)
    except Exception as e:  # reported, not hidden
        paper = {"error": str(e)}
    try:
        tensor_variant = tensor_variant_report(dev) if args.tc else None
        if args.tc and tensor_variant is not None and any(w.name == "dg" for w, _, _ in parts):
            tensor_variant["dg_diff_tc"] = dg_tensor_variant_report(dev, mean_s)
    except Exception as e:
        tensor_variant = {"error": str(e)}
    n_app = len({k for _, _, app in parts for k in app})
    n_cal = len(kernels) - n_app
    e2e_launch_total = int(sweep_launches_all + args.steps * e2e_launches)
    cpu = None
    if dist.world == 1:
        # the oracle restatement on the host cores: the reference arm's
        # bounded sample of this workload, 1 warm-up + 2 passes
        sample = reference_sample(kernels)
        v, _dt, cores = time_reference_sample(sample, 1, 2, threads=os.cpu_count() or 1)
        cpu = {"value": round(v, 3), "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": sample_note(sample, args.workload)}
    ref_lib = reference_model_sample() if dist.world == 1 else None
    detail = {
        "models": models, "headline": heads, "k17": k17, "model_eval": model_eval,
        "overlap_diagnosis": diagnosis, "paper_selection": paper,
        "tensor_variant": tensor_variant,
        "roofline": roofline, "roofline_hbm": roofline_hbm, "suite_rooflines": suite_rooflines,
        "suite_binding": suite_binding,
        "suite_hbm_GBps": round(hbm_b / hbm_t / 1e9, 1) if hbm_t else None,
        "suite_flops_TFps": round(fl / fl_t / 1e12, 2) if fl_t else None,
        "cpu_baseline_reference": ref_lib,
        "e2e_full_outputs": {"value": round(e2e_bytes_all / e2e_full_time_max / 1e9, 3)
                             if e2e_full_time_max and full_all else None, "unit": "GB/s",
                             "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h_full),
                             "note": "the e2e pass with every output array copied back"},
        "cross_rank_timing": cross_rank, "host_wall_s": round(wall, 3),
        "workload_description": " | ".join(wl.description for wl, _, _ in parts),
    }
    detail_path = Path(args.detail)
    try:
        detail_path.parent.mkdir(parents=True, exist_ok=True)
        detail_path.write_text(json.dumps(detail, indent=1, default=str) + "\n")
        detail_ref = str(detail_path.relative_to(ROOT) if detail_path.is_relative_to(ROOT)
                         else detail_path)
    except OSError as e:
        detail_ref = f"unwritten: {e}"
    me = model_eval if isinstance(model_eval, dict) else {}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed_max / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (deterministic seed pattern, tests/support.hpp:35-44)",
        "config": bench_config(args.workload, len(kernels), n_cal, n_app,
                               args.steps * args.trials_per_step, dist.world),
        "roofline": {k: roofline.get(k) for k in ("bound", "achieved", "peak", "unit", "frac",
                                                   "traffic", "kernel", "share_of_step")},
        "roofline_binding": dict(({k: roofline["binding_roofline"][k]
                                   for k in ("bound", "achieved", "peak", "unit", "frac")}
                                  if roofline.get("binding_roofline") else {}),
                                 suite=suite_binding),
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_bytes_all / e2e_time_max / 1e9, 3) if e2e_time_max else None,
                "unit": "GB/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "checksums_verified": f"{e2e_verified[0]}/{e2e_verified[1]}"},
        # headline accuracy: the per-variant held-out choice where it was
        # made, else the single held-out model of the application
        "accuracy": {
            "selection": {w: ("per-variant held-out" if h.get("per_variant") else h["selection"])
                          for w, h in heads.items()},
            "model": {v: m for w, h in heads.items() for v, m in (
                (h["per_variant"]["assignment"].items()) if h.get("per_variant")
                else [(w, f"{h['model']}/{h['fit']}")])},
            "geomean_rel_error": {v: e for h in heads.values() for v, e in (
                _acc(h).get("geomean_rel_error") or {}).items()},
            "by_application": {w: _acc(h).get("geomean_rel_error_all") for w, h in heads.items()},
            "ranking_correct_gap_ge_2pct": {w: _acc(h).get("ranking_correct_gap_ge_2pct")
                                            for w, h in heads.items()},
            # the held-out sizes the choice was NOT made on
            "test_geomean_rel_error": {v: e for h in heads.values() for v, e in (
                (_acc(h).get("test") or {}).get("geomean_rel_error") or {}).items()},
            "test_ranking_correct_gap_ge_2pct": {w: (_acc(h).get("test") or {}).get(
                "ranking_correct_gap_ge_2pct") for w, h in heads.items()},
            # one model per application (held-out choice) and the paper's own
            # per-variant linear/nonlinear choice, for comparison
            "single_model": {w: {"model": f"{h['model']}/{h['fit']}",
                                 "all": h["geomean_rel_error_all"],
                                 "ranking_gap_ge_2pct": h["ranking_correct_gap_ge_2pct"]}
                             for w, h in heads.items()},
            "paper_model": ({w: {"all": v["geomean_rel_error_all"],
                                 "ranking_gap_ge_2pct": v["ranking_correct_gap_ge_2pct"]}
                             for w, v in paper.items()} if "error" not in paper else paper)},
        "model_eval": dict({k: me.get(k) for k in ("evaluations", "gpu_evals_per_s",
                                                   "gpu_e2e_evals_per_s", "argmin_mismatches_vs_cpu",
                                                   "port_predict_max_rel_diff")},
                           reference_library_predict_evals_per_s=(ref_lib or {}).get(
                               "predict_evals_per_s"),
                           reference_library_threads=(ref_lib or {}).get("threads"))
        if me else None,
        "k17": ({"fits": k17.get("fits"), "launches": k17.get("launches"),
                 "kernel_s": k17.get("kernel_s"), "fits_per_s": k17.get("fits_per_s"),
                 "reference_library": {k: (k17.get("reference_library") or {}).get(k) for k in (
                     "fits_per_s_1thread", "fits_per_s_threads", "threads",
                     "gpu_reference_mode_bitwise_equal")}}
                if k17 and "error" not in k17 else k17),
        "gpu_launches": e2e_launch_total,
        "clocks": {k: clocks.get(k) for k in ("sm_mhz", "sm_max_mhz", "reasons")},
        "detail": detail_ref,
    }
    out = json.dumps(line)
    if len(out) > 4096:  # keep the line parseable: drop the largest optional parts
        for k in ("model_eval", "roofline_binding"):
            line.pop(k, None)
            out = json.dumps(line)
            if len(out) <= 4096:
                break
    print(out, flush=True)
    dev.close()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="all",
                    help="matmul | fd | dg | all (one sweep over the union, BASELINE configs[3])")
    ap.add_argument("--trials-per-step", type=int, default=4)
    ap.add_argument("--table", default="", help="write the measurement table (CSV) here")
    ap.add_argument("--tc", type=int, default=1, help="report the tcgen05 variant (0: skip)")
    ap.add_argument("--c5-points", type=int, default=1_000_000,
                    help="parameter points for the model-evaluation report (0: skip)")
    ap.add_argument("--detail", default=str(ROOT / "gpurun_out" / "bench_detail.json"),
                    help="side file for the full report (models, diagnosis, per-family rooflines)")
    ap.add_argument("--headline-model", default="",
                    help="force this model as the headline (default: held-out selection over "
                         "every candidate model on the workload's validation sizes)")
    args = ap.parse_args()
    # the reference arm is CPU-only with no exchange (rank 0 alone runs it):
    # no process group, no GPU binding
    dist = Dist(process_group=args.impl != "reference")
    try:
        if args.impl == "reference":
            run_reference_arm(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
