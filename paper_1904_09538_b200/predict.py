"""Batched prediction and ranking over a variant space (K18) through the C ABI.

A table set binds calibrated models to kernel variants (ps_tables_build);
``eval_gpu`` evaluates every variant at every parameter point on a B200 and
returns predictions plus the per-application winner; ``eval_cpu`` is the same
computation on host threads.
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from ._abi import check, lib

_P = C.POINTER


def _declare():
    L = lib()
    if getattr(L, "_k18_declared", False):
        return L
    L.ps_tables_build.argtypes = [C.c_char_p, _P(C.c_void_p)]
    L.ps_tables_info.argtypes = [C.c_void_p, _P(C.c_int), _P(C.c_int), _P(C.c_int64)]
    L.ps_tables_free.argtypes = [C.c_void_p]
    L.ps_eval_batched.argtypes = [C.c_void_p, C.c_void_p, _P(C.c_int64), C.c_int64,
                                  _P(C.c_double), _P(C.c_uint8), _P(C.c_double)]
    L.ps_eval_cpu.argtypes = [C.c_void_p, _P(C.c_int64), C.c_int64, _P(C.c_double),
                              _P(C.c_uint8), C.c_int]
    L.ps_eval_prepare.argtypes = [C.c_void_p, C.c_void_p, _P(C.c_double)]
    L.ps_eval_jit_source.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, _P(C.c_size_t)]
    L.ps_eval_jit_compile.argtypes = [C.c_void_p, _P(C.c_size_t)]
    for n in ("ps_tables_build", "ps_tables_info", "ps_tables_free", "ps_eval_batched",
              "ps_eval_cpu", "ps_eval_prepare", "ps_eval_jit_source", "ps_eval_jit_compile"):
        getattr(L, n).restype = C.c_int
    L._k18_declared = True
    return L


class PredictionTables:
    """variants: list of dicts {id, model (text), params (list), group, coords}."""

    def __init__(self, variants: list[dict]):
        L = _declare()
        self._h = C.c_void_p()
        check(L.ps_tables_build(json.dumps({"variants": variants}).encode(), C.byref(self._h)))
        nvar, ngroups, nterms = C.c_int(), C.c_int(), C.c_int64()
        check(L.ps_tables_info(self._h, C.byref(nvar), C.byref(ngroups), C.byref(nterms)))
        self.nvar, self.ngroups, self.nterms = nvar.value, ngroups.value, nterms.value
        self.ids = [v["id"] for v in variants]

    def close(self):
        if self._h:
            _declare().ps_tables_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _out(self, points: np.ndarray, out=None):
        pts = np.ascontiguousarray(points, dtype=np.int64)
        if pts.ndim != 2 or pts.shape[1] != 4:
            raise ValueError("points must be [npts, 4] int64")
        if out is not None:
            pred, arg = out
            if pred.shape != (pts.shape[0], self.nvar) or arg.shape != (pts.shape[0], self.ngroups):
                raise ValueError("output buffers do not match the point count")
            return pts, pred, arg
        pred = np.empty((pts.shape[0], self.nvar), dtype=np.float64)
        arg = np.empty((pts.shape[0], self.ngroups), dtype=np.uint8)
        return pts, pred, arg

    def pinned_buffers(self, npts: int):
        """Page-locked point and result buffers (ps_host_alloc) so the
        end-to-end path copies at PCIe speed: (points [npts, 4] int64,
        pred [npts, nvar] float64, argmin [npts, ngroups] uint8, keep-alive)."""
        from .device import PinnedArray
        bufs = [PinnedArray(max(1, npts * 4 * 8)), PinnedArray(max(1, npts * self.nvar * 8)),
                PinnedArray(max(1, npts * self.ngroups))]
        pts = bufs[0].numpy(np.int64)[: npts * 4].reshape(npts, 4)
        pred = bufs[1].numpy(np.float64)[: npts * self.nvar].reshape(npts, self.nvar)
        arg = bufs[2].numpy(np.uint8)[: npts * self.ngroups].reshape(npts, self.ngroups)
        return pts, pred, arg, bufs

    def prepare_gpu(self, dev) -> float:
        """Compile and load the tables' specialised K18 kernel on dev ahead of
        the first evaluation (NVRTC); returns the seconds this call spent (0
        when it was already loaded, or with the option k18_jit off)."""
        secs = C.c_double()
        check(_declare().ps_eval_prepare(dev._ctx, self._h, C.byref(secs)))
        return secs.value

    def jit_source(self) -> str:
        """The CUDA source of the tables' specialised kernel."""
        L, need = _declare(), C.c_size_t()
        L.ps_eval_jit_source(self._h, None, 0, C.byref(need))  # size query
        buf = C.create_string_buffer(need.value + 1)
        check(L.ps_eval_jit_source(self._h, buf, len(buf), C.byref(need)))
        return buf.value.decode()

    def jit_compile(self) -> int:
        """Compile the specialised kernel with NVRTC (no device); cubin bytes."""
        n = C.c_size_t()
        check(_declare().ps_eval_jit_compile(self._h, C.byref(n)))
        return n.value

    def eval_gpu(self, dev, points: np.ndarray, out=None):
        """K18 on dev. out = (pred, argmin) writes into caller buffers (e.g.
        from pinned_buffers) instead of fresh pageable arrays."""
        pts, pred, arg = self._out(points, out)
        secs = C.c_double()
        check(_declare().ps_eval_batched(dev._ctx, self._h, pts.ctypes.data_as(_P(C.c_int64)),
                                         pts.shape[0], pred.ctypes.data_as(_P(C.c_double)),
                                         arg.ctypes.data_as(_P(C.c_uint8)), C.byref(secs)))
        return pred, arg, secs.value

    def eval_cpu(self, points: np.ndarray, threads: int = 1):
        pts, pred, arg = self._out(points)
        check(_declare().ps_eval_cpu(self._h, pts.ctypes.data_as(_P(C.c_int64)), pts.shape[0],
                                     pred.ctypes.data_as(_P(C.c_double)),
                                     arg.ctypes.data_as(_P(C.c_uint8)), threads))
        return pred, arg


def c5_points(npts: int, seed: int = 7) -> np.ndarray:
    """BASELINE.json configs[4] parameter points: n_mm in 16Z
    within [512, 8192], n_fd in 112Z within [1120, 8176], nel in 16Z within
    [1e4, 1e6], DG order 1..7 as padded nodes per element."""
    rng = np.random.default_rng(seed)
    np_of_order = np.array([16, 16, 32, 48, 64, 96, 128])  # (k+1)(k+2)(k+3)/6 padded to 16
    p = np.empty((npts, 4), dtype=np.int64)
    p[:, 0] = 16 * rng.integers(512 // 16, 8192 // 16 + 1, npts)
    p[:, 1] = 112 * rng.integers(1120 // 112, 8176 // 112 + 1, npts)
    p[:, 2] = 16 * rng.integers(10000 // 16 + 1, 1000000 // 16 + 1, npts)
    p[:, 3] = np_of_order[rng.integers(0, 7, npts)]
    return p
