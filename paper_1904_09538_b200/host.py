"""Python face of the C++ host port (catalog, count features, reference-exact
fit, prediction) through the C ABI — the same calls a C/C++/cgo caller makes."""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._abi import FitOpts, FitStats, check, lib

_P = C.POINTER


def _declare() -> C.CDLL:
    L = lib()
    if getattr(L, "_host_declared", False):
        return L
    L.ps_catalog.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t,
                             _P(C.c_size_t)]
    L.ps_model_info.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, _P(C.c_size_t)]
    L.ps_kernel_json.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, _P(C.c_size_t)]
    L.ps_kernel_json.restype = C.c_int
    L.ps_model_program.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_size_t, _P(C.c_size_t)]
    L.ps_model_program.restype = C.c_int
    L.ps_feature_table.argtypes = [C.c_char_p, C.c_char_p, C.c_int, _P(C.c_double), C.c_int64]
    L.ps_fit_cpu.argtypes = [C.c_char_p, _P(C.c_double), _P(C.c_double), C.c_int, C.c_int,
                             _P(FitOpts), _P(C.c_double), _P(FitStats)]
    L.ps_initial_point.argtypes = [C.c_char_p, _P(C.c_double), _P(C.c_double), C.c_int, C.c_int,
                                   _P(C.c_double)]
    L.ps_predict_cpu.argtypes = [C.c_char_p, _P(C.c_double), C.c_char_p, C.c_int, _P(C.c_double),
                                 C.c_int64]
    L.ps_model_bytecode.argtypes = [C.c_char_p, C.c_int, _P(C.c_int32), C.c_int, _P(C.c_double),
                                    C.c_int, _P(C.c_int), _P(C.c_int), _P(C.c_int)]
    L.ps_geo_mean_rel_error.argtypes = [_P(C.c_double), _P(C.c_double), C.c_int, _P(C.c_double)]
    for n in ("ps_catalog", "ps_model_info", "ps_feature_table", "ps_fit_cpu", "ps_initial_point",
              "ps_predict_cpu", "ps_model_bytecode", "ps_geo_mean_rel_error"):
        getattr(L, n).restype = C.c_int
    L._host_declared = True
    return L


def _string_call(fn, *args) -> str:
    need = C.c_size_t(0)
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        rc = fn(*args, buf, cap, C.byref(need))
        if rc == 0:
            return buf.value.decode()
        if need.value > cap:
            cap = need.value
            continue
        check(rc)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_P(C.c_double))


def catalog(tags: list[str], match: str = "superset", which: str = "b200") -> list[tuple[str, dict]]:
    """[(variant_id, bindings)] from KernelCollection::generate."""
    L = _declare()
    text = _string_call(L.ps_catalog, which.encode(), "\n".join(tags).encode(), match.encode())
    out = []
    for line in text.splitlines():
        vid, _, b = line.partition("\t")
        bind = {}
        for item in filter(None, b.split(";")):
            k, _, v = item.partition("=")
            bind[k] = int(v)
        out.append((vid, bind))
    return out


def kernel_json(variant_id: str) -> dict:
    """{"id", "kernel" (perfseer-kernel/1), "bindings"} of a catalog variant."""
    import json
    L = _declare()
    return json.loads(_string_call(L.ps_kernel_json, variant_id.encode()))


class HostModel:
    """A parsed model (reference model-file text: output id line + expression)."""

    def __init__(self, text: str):
        self.text = text
        info = json.loads(_string_call(_declare().ps_model_info, text.encode()))
        self.output = info["output"]
        self.params: list[str] = info["params"]
        self.features: list[str] = info["features"]
        self.cost_params = info["cost_params"]

    def feature_table(self, variant_ids: list[str], sub_group_size: int = 32) -> np.ndarray:
        out = np.zeros((len(variant_ids), len(self.features)), dtype=np.float64)
        check(_declare().ps_feature_table(self.text.encode(), "\n".join(variant_ids).encode(),
                                          sub_group_size, _dptr(out), out.size))
        return out

    def fit_cpu(self, features: np.ndarray, t: np.ndarray, scale: bool = True,
                opts: FitOpts | None = None):
        f = np.ascontiguousarray(features, dtype=np.float64)
        tt = np.ascontiguousarray(t, dtype=np.float64)
        p = np.zeros(len(self.params), dtype=np.float64)
        st = FitStats()
        check(_declare().ps_fit_cpu(self.text.encode(), _dptr(f), _dptr(tt), len(tt), int(scale),
                                    C.byref(opts) if opts else None, _dptr(p), C.byref(st)))
        return p, {"residual_norm": st.residual_norm, "iterations": st.iterations,
                   "converged": bool(st.converged)}

    def initial_point(self, features: np.ndarray, t: np.ndarray, scale: int = 1) -> np.ndarray:
        """scale 0/1: the reference's start (model.cpp:439-481) on raw/output-scaled
        rows; 2: relative-residual QR start used by the B200 fit."""
        f = np.ascontiguousarray(features, dtype=np.float64)
        tt = np.ascontiguousarray(t, dtype=np.float64)
        p = np.zeros(len(self.params), dtype=np.float64)
        check(_declare().ps_initial_point(self.text.encode(), _dptr(f), _dptr(tt), len(tt),
                                          int(scale), _dptr(p)))
        return p

    def predict_cpu(self, params: np.ndarray, variant_ids: list[str], sub_group_size: int = 32):
        p = np.ascontiguousarray(params, dtype=np.float64)
        out = np.zeros(len(variant_ids), dtype=np.float64)
        check(_declare().ps_predict_cpu(self.text.encode(), _dptr(p),
                                        "\n".join(variant_ids).encode(), sub_group_size,
                                        _dptr(out), out.size))
        return out

    def program(self, with_jacobian: bool = True) -> dict:
        """The CSE'd straight-line program K17/K18 run (ps_model_program)."""
        return json.loads(_string_call(_declare().ps_model_program, self.text.encode(),
                                       int(with_jacobian)))

    def bytecode(self, which: int = -1):
        cap = 1 << 14
        while True:
            ops = np.zeros(cap, dtype=np.int32)
            consts = np.zeros(cap, dtype=np.float64)
            n_ops, n_consts, stack = C.c_int(), C.c_int(), C.c_int()
            rc = _declare().ps_model_bytecode(self.text.encode(), which,
                                              ops.ctypes.data_as(_P(C.c_int32)), cap, _dptr(consts),
                                              cap, C.byref(n_ops), C.byref(n_consts), C.byref(stack))
            if rc and max(n_ops.value, n_consts.value) > cap:
                cap = max(n_ops.value, n_consts.value)
                continue
            check(rc)
            return ops[: n_ops.value].copy(), consts[: n_consts.value].copy(), stack.value


def enumerate_counts(variant_id: str, mode: str = "symbolic", dev=None) -> dict:
    """Exact counts of a variant at its own bindings: mode "symbolic"
    (analyze), "cpu" (brute_force_count) or "gpu" (the enumerator on dev)."""
    L = _declare()
    L.ps_enumerate.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_char_p, C.c_size_t,
                               _P(C.c_size_t)]
    L.ps_enumerate.restype = C.c_int
    m = {"symbolic": 0, "cpu": 1, "gpu": 2}[mode]
    ctx = dev._ctx if dev is not None else None
    return json.loads(_string_call(L.ps_enumerate, ctx, variant_id.encode(), m))


def set_option(key: str, value: str) -> None:
    """ps_set_option, e.g. ("partial_subgroups", "round_up") for 18x18 tiles."""
    L = _declare()
    L.ps_set_option.argtypes = [C.c_char_p, C.c_char_p]
    L.ps_set_option.restype = C.c_int
    check(L.ps_set_option(key.encode(), value.encode()))


def default_fit_opts() -> FitOpts:
    """FitOptions defaults (reference model.hpp:71-80)."""
    return FitOpts(1e-3, 0.1, 10.0, 1e-10, 1e-10, 200, 0)


def geo_mean_rel_error(pred, meas) -> float:
    p = np.ascontiguousarray(pred, dtype=np.float64)
    m = np.ascontiguousarray(meas, dtype=np.float64)
    out = C.c_double()
    check(_declare().ps_geo_mean_rel_error(_dptr(p), _dptr(m), len(p), C.byref(out)))
    return out.value

def trace(name: str):
    """NVTX range over a pipeline stage (ps_trace_push/pop): `with trace("sweep"): ...`."""
    import contextlib

    @contextlib.contextmanager
    def _range():
        L = lib()
        L.ps_trace_push.argtypes = [C.c_char_p]
        L.ps_trace_push(name.encode())
        try:
            yield
        finally:
            L.ps_trace_pop()
    return _range()
