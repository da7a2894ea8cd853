"""Python face of the B200 executor: a ps_ctx per GPU behind the C ABI.

Mirrors perfseer::Executor (reference include/perfseer/executor.hpp:16-23):
``id()`` and ``measure(kernel_id, trials)`` returning per-trial seconds, plus
``measure_summary`` = measure_kernel + summarize (src/executor.cpp:14-48).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import KernelDesc, check, lib


def _desc(kernel) -> KernelDesc:
    if isinstance(kernel, KernelDesc):
        return kernel
    return _abi.desc_from_id(str(kernel))


class CudaDevice:
    """One GPU context. Not reentrant (executors are exclusive resources)."""

    def __init__(self, device: int = 0):
        self.device = device
        self._ctx = C.c_void_p()
        check(lib().ps_init(device, C.byref(self._ctx)))

    def id(self) -> str:
        return f"cuda_b200_{self.device}"

    def close(self) -> None:
        if self._ctx:
            lib().ps_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        sm, clk, l2, free = C.c_int(), C.c_int(), C.c_size_t(), C.c_size_t()
        check(lib().ps_device_info(self._ctx, C.byref(sm), C.byref(clk), C.byref(l2),
                                   C.byref(free)))
        return {"sm_count": sm.value, "sm_clock_khz": clk.value, "l2_bytes": l2.value,
                "free_bytes": free.value}

    def prepare(self, kernel, fill: int = _abi.PS_FILL_SEED17, seed: int = 0) -> None:
        check(lib().ps_prepare(self._ctx, C.byref(_desc(kernel)), fill, seed))

    def measure(self, kernel, trials: int = 60, warmup: int = 5) -> list[float]:
        d = _desc(kernel)
        out = (C.c_double * trials)()
        check(lib().ps_measure(self._ctx, C.byref(d), warmup, trials, out))
        return list(out)

    def measure_summary(self, kernel, trials: int = 60, warmup: int = 5,
                        filter_factor: float = 5.0) -> tuple[float, int]:
        d = _desc(kernel)
        mean, kept = C.c_double(), C.c_int()
        check(lib().ps_measure_summary(self._ctx, C.byref(d), warmup, trials, filter_factor,
                                       C.byref(mean), C.byref(kept)))
        return mean.value, kept.value

    def run_timed(self, kernel, launches: int) -> float:
        d = _desc(kernel)
        s = C.c_double()
        check(lib().ps_run_timed(self._ctx, C.byref(d), launches, C.byref(s)))
        return s.value

    def run(self, kernel, inputs: list[np.ndarray]) -> list[np.ndarray]:
        """Parity hook: host inputs -> one launch -> host outputs."""
        d = _desc(kernel)
        io = _abi.kernel_io(d)
        dt = np.float32 if io.elem_bytes == 4 else np.float64
        if len(inputs) != io.n_inputs:
            raise ValueError(f"kernel takes {io.n_inputs} inputs, got {len(inputs)}")
        ins = []
        for i, a in enumerate(inputs):
            a = np.ascontiguousarray(a, dtype=dt).reshape(-1)
            if a.size != io.input_elems[i]:
                raise ValueError(f"input {i}: expected {io.input_elems[i]} elements, got {a.size}")
            ins.append(a)
        outs = [np.empty(io.output_elems[i], dtype=dt) for i in range(io.n_outputs)]
        in_ptrs = (C.c_void_p * max(1, len(ins)))(*[a.ctypes.data for a in ins])
        out_ptrs = (C.c_void_p * max(1, len(outs)))(*[a.ctypes.data for a in outs])
        check(lib().ps_run_verify(self._ctx, C.byref(d), in_ptrs, len(ins), out_ptrs, len(outs)))
        return outs

    # -- timing helpers (events on the context stream) ---------------------
    def mark(self, slot: int) -> None:
        check(lib().ps_mark(self._ctx, slot))

    def elapsed(self, a: int, b: int) -> float:
        s = C.c_double()
        check(lib().ps_elapsed(self._ctx, a, b, C.byref(s)))
        return s.value

    def run_host(self, kernel, inputs: list["PinnedArray"], outputs: list["PinnedArray"]) -> float:
        """H2D + launch + D2H through caller-owned (pinned) host buffers; seconds."""
        d = _desc(kernel)
        ip = (C.c_void_p * max(1, len(inputs)))(*[a.ptr for a in inputs])
        op = (C.c_void_p * max(1, len(outputs)))(*[a.ptr for a in outputs])
        s = C.c_double()
        check(lib().ps_run_host(self._ctx, C.byref(d), ip, len(inputs), op, len(outputs),
                                C.byref(s)))
        return s.value


    def trim(self) -> None:
        """Release every resident variant and staging buffer (ps_trim)."""
        check(lib().ps_trim(self._ctx))

    def run_host_batch(self, kernels, inputs: list[list["PinnedArray"]],
                       outputs: list[list["PinnedArray"]] | None, checksums: bool = False):
        """A sweep through host data, pipelined (ps_run_host_batch_ex): H2D of
        the next kernel, this kernel's launch and D2H of the previous one
        overlap; seconds from the first copy in to the last copy out. With
        checksums=True the step's result is one device-computed checksum per
        kernel (wrapping sum of its output words), returned as
        (seconds, uint64 array); outputs may then be None (no array copies)."""
        ds = [_desc(k) for k in kernels]
        arr = (_abi.KernelDesc * max(1, len(ds)))(*ds)
        ip = [a.ptr for ins in inputs for a in ins]
        ipa = (C.c_void_p * max(1, len(ip)))(*ip)
        opa = None
        if outputs is not None:
            op = [a.ptr for outs in outputs for a in outs]
            opa = (C.c_void_p * max(1, len(op)))(*op)
        sums = np.zeros(max(1, len(ds)), dtype=np.uint64)
        sp = sums.ctypes.data_as(C.POINTER(C.c_uint64)) if checksums else None
        s = C.c_double()
        check(lib().ps_run_host_batch_ex(self._ctx, len(ds), arr, ipa, opa, sp, C.byref(s)))
        return (s.value, sums[:len(ds)]) if checksums else s.value


class PinnedArray:
    """Page-locked host buffer from ps_host_alloc, viewable as numpy."""

    def __init__(self, nbytes: int):
        self.nbytes = nbytes
        p = C.c_void_p()
        check(lib().ps_host_alloc(nbytes, C.byref(p)))
        self.ptr = p.value

    def numpy(self, dtype) -> np.ndarray:
        n = self.nbytes // np.dtype(dtype).itemsize
        buf = (C.c_char * self.nbytes).from_address(self.ptr)
        return np.frombuffer(buf, dtype=dtype, count=n)

    def free(self) -> None:
        if self.ptr:
            lib().ps_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def fit_lm_batched(dev: CudaDevice, model, features: np.ndarray, t: np.ndarray, p0: np.ndarray,
                   opts=None, mode: int = 0):
    """K17 on `dev`: nbatch independent LM fits of a HostModel.

    features: [nbatch, nr, nf] (or [nr, nf], shared by every start), t: [nbatch, nr]
    or [nr], p0: [nbatch, np]. Returns (params [nbatch, np], stats list)."""
    from ._abi import Bytecode, FitOpts, FitStats
    from .host import default_fit_opts
    L = lib()
    if not getattr(L, "_lm_declared", False):
        L.ps_fit_lm_batched_ex.argtypes = [C.c_void_p, C.POINTER(Bytecode), C.POINTER(Bytecode),
                                           C.c_int, C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.c_int, C.c_int,
                                           C.POINTER(FitOpts), C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(FitStats)]
        L.ps_fit_lm_batched_ex.restype = C.c_int
        L._lm_declared = True
    p0 = np.atleast_2d(np.asarray(p0, dtype=np.float64))
    nb, npar = p0.shape
    f = np.asarray(features, dtype=np.float64)
    if f.ndim == 2:
        f = np.broadcast_to(f, (nb,) + f.shape)
    tt = np.asarray(t, dtype=np.float64)
    if tt.ndim == 1:
        tt = np.broadcast_to(tt, (nb, tt.shape[0]))
    f = np.ascontiguousarray(f)
    tt = np.ascontiguousarray(tt)
    nr, nf = f.shape[1], f.shape[2]
    keep = []

    def bc(which):
        ops, consts, _ = model.bytecode(which)
        keep.extend([ops, consts])
        return Bytecode(len(ops), len(consts), ops.ctypes.data_as(C.POINTER(C.c_int32)),
                        consts.ctypes.data_as(C.POINTER(C.c_double)))

    mb = bc(-1)
    if mode & 8:  # forward-mode derivatives on the device: no derivative programs
        if model.bytecode(-1)[2] > 24:
            raise ValueError("model expression too deep for the device evaluator (stack > 24)")
        jac = None
    else:
        jac = (Bytecode * npar)(*[bc(i) for i in range(npar)])
    params = np.ascontiguousarray(p0.copy())
    stats = (FitStats * nb)()
    o = opts or default_fit_opts()
    dptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    check(L.ps_fit_lm_batched_ex(dev._ctx, C.byref(mb), jac, npar, nf, dptr(f), dptr(tt), nr, nb,
                                 C.byref(o), mode, dptr(params), stats))
    return params, [{"residual_norm": s.residual_norm, "iterations": s.iterations,
                     "converged": bool(s.converged), "status": s.status} for s in stats]


class LmJob(C.Structure):
    """ps_lm_job (include/perfseer_b200.h)."""
    _fields_ = [("model_text", C.c_char_p), ("nf", C.c_int32), ("nr", C.c_int32),
                ("nbatch", C.c_int32), ("mode", C.c_int32), ("shared_rows", C.c_int32),
                ("reserved", C.c_int32), ("features", C.POINTER(C.c_double)),
                ("t", C.POINTER(C.c_double)), ("opts", _abi.FitOpts),
                ("params_inout", C.POINTER(C.c_double)), ("stats", C.POINTER(_abi.FitStats))]


def fit_lm_jobs(dev: CudaDevice, jobs: list[dict]):
    """K17 v2: every fit in ONE launch (ps_fit_lm_jobs). Each job: {"model":
    HostModel, "features": [nr, nf], "t": [nr], "starts": [nbatch, np],
    "mode": bits (1 equilibrate, 2 shuffle sums, 4 relative residuals),
    "opts": FitOpts or None}. Returns ([(params [nbatch, np], stats list)],
    kernel seconds)."""
    from ._abi import FitStats
    from .host import default_fit_opts
    L = lib()
    if not getattr(L, "_lm_jobs_declared", False):
        L.ps_fit_lm_jobs.argtypes = [C.c_void_p, C.c_int, C.POINTER(LmJob), C.POINTER(C.c_double)]
        L.ps_fit_lm_jobs.restype = C.c_int
        L._lm_jobs_declared = True
    keep, arr, outs = [], (LmJob * len(jobs))(), []
    dptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for j, job in enumerate(jobs):
        m = job["model"]
        f = np.ascontiguousarray(job["features"], dtype=np.float64)
        t = np.ascontiguousarray(job["t"], dtype=np.float64)
        p = np.ascontiguousarray(np.atleast_2d(job["starts"]), dtype=np.float64).copy()
        st = (FitStats * p.shape[0])()
        text = m.text.encode()
        keep += [f, t, p, st, text]
        arr[j] = LmJob(text, f.shape[1], f.shape[0], p.shape[0], int(job.get("mode", 0)), 1, 0,
                       dptr(f), dptr(t), job.get("opts") or default_fit_opts(), dptr(p), st)
        outs.append((p, st))
    secs = C.c_double()
    check(L.ps_fit_lm_jobs(dev._ctx, len(jobs), arr, C.byref(secs)))
    res = [(p, [{"residual_norm": s.residual_norm, "iterations": s.iterations,
                 "converged": bool(s.converged), "status": s.status, "trials": s.trials}
                for s in st])
           for p, st in outs]
    return res, secs.value
