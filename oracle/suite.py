"""TEST INFRASTRUCTURE ONLY: ctypes face of oracle/suite_ref.c (the plain-C
restatement of every suite kernel) plus the reference fixture's input pattern.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB = _HERE / "_build" / "libsuite_ref.so"
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(_HERE), "restatement"], check=True,
                           capture_output=True)
        _lib = C.CDLL(str(LIB))
        _lib.ref_run.restype = C.c_int
        _lib.ref_run.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        _lib.ref_flops_value.restype = C.c_float
        _lib.ref_flops_value.argtypes = [C.c_int, C.c_int64]
        _lib.ref_threads.restype = C.c_int
        _lib.ref_matmul_rows.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int64, C.c_int64,
                                         C.c_void_p]
        _lib.ref_set_threads.argtypes = [C.c_int]
    return _lib


FNV_OFFSET = np.uint64(1469598103934665603)
FNV_PRIME = np.uint64(1099511628211)


def seed_values(array: str, n: int, dtype=np.float32) -> np.ndarray:
    """1 + (FNV1a(array) ^ flat) * prime % 17 — tests/support.hpp:35-44."""
    h = int(FNV_OFFSET)
    for ch in array.encode():
        h ^= ch
        h = (h * int(FNV_PRIME)) & 0xFFFFFFFFFFFFFFFF
    flat = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        v = (np.uint64(h) ^ flat) * FNV_PRIME
    return (1 + (v % np.uint64(17))).astype(dtype)


def uniform_values(n: int, seed: int, dtype=np.float32) -> np.ndarray:
    """U[-1, 1) with 24 random bits (exact in float32)."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 1 << 24, size=n) / 8388608.0 - 1.0).astype(dtype)


def run(desc, io, inputs: list[np.ndarray]) -> list[np.ndarray]:
    """Restated kernel on host arrays (same I/O layout as ps_run_verify)."""
    dt = np.float32 if io.elem_bytes == 4 else np.float64
    ins = [np.ascontiguousarray(a, dtype=dt).reshape(-1) for a in inputs]
    outs = [np.zeros(io.output_elems[i], dtype=dt) for i in range(io.n_outputs)]
    ip = (C.c_void_p * max(1, len(ins)))(*[a.ctypes.data for a in ins])
    op = (C.c_void_p * max(1, len(outs)))(*[a.ctypes.data for a in outs])
    rc = lib().ref_run(C.addressof(desc), ip, op)
    if rc:
        raise ValueError(f"oracle has no restatement for generator {desc.gen}")
    return outs


def matmul_rows(desc, inputs: list[np.ndarray], i0: int, i1: int) -> np.ndarray:
    """Rows [i0, i1) of the matmul oracle (same per-element fma order)."""
    dt = np.float32 if desc.dtype == 0 else np.float64
    ins = [np.ascontiguousarray(a, dtype=dt).reshape(-1) for a in inputs]
    out = np.zeros((i1 - i0) * desc.n, dtype=dt)
    ip = (C.c_void_p * 2)(*[a.ctypes.data for a in ins])
    lib().ref_matmul_rows(C.addressof(desc), ip, i0, i1, out.ctypes.data)
    return out


def threads() -> int:
    return lib().ref_threads()


def set_threads(n: int) -> None:
    lib().ref_set_threads(n)
