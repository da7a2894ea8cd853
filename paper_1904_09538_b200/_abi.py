"""ctypes binding of the C ABI in include/perfseer_b200.h.

This is the reference-side binding a Python caller uses (INTEGRATION.md shows
the same stub for other hosts). The product path loads the in-tree
``libperfseer_b200.so`` only; if it is missing the import fails loudly — there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libperfseer_b200.so"

PS_GEN = {
    "gmem_pattern": 1, "flops": 2, "lmem_shuffle": 3, "barrier_knl": 4, "empty_knl": 5,
    "overlap_knl": 6, "matmul_sq": 7, "matmul_sq_rm": 8, "finite_diff": 9,
    "finite_diff_rm": 10, "dg_diff": 11, "dg_diff_rm": 12, "matmul_sq_tc": 13,
}
PS_F32, PS_F64 = 0, 1
PS_FILL_SEED17, PS_FILL_UNIFORM = 0, 1
PS_MAX_ARRAYS = 4


class KernelDesc(C.Structure):
    _fields_ = [
        ("gen", C.c_int32), ("dtype", C.c_int32), ("op", C.c_int32), ("keep", C.c_int32),
        ("nelements", C.c_int64), ("lsize0", C.c_int64), ("lsize1", C.c_int64),
        ("lid_stride0", C.c_int64), ("lid_stride1", C.c_int64), ("n_inputs", C.c_int64),
        ("m", C.c_int64), ("num_groups", C.c_int64), ("n", C.c_int64),
        ("prefetch", C.c_int32), ("tile", C.c_int32), ("nel", C.c_int64), ("np", C.c_int64),
        ("nmat", C.c_int64), ("dg_variant", C.c_int32), ("reserved", C.c_int32),
    ]


class IoInfo(C.Structure):
    _fields_ = [
        ("n_inputs", C.c_int32), ("n_outputs", C.c_int32), ("elem_bytes", C.c_int32),
        ("reserved", C.c_int32), ("input_elems", C.c_int64 * PS_MAX_ARRAYS),
        ("output_elems", C.c_int64 * PS_MAX_ARRAYS), ("bytes_global", C.c_double),
        ("flops", C.c_double), ("bytes_shared", C.c_double),
    ]


class Bytecode(C.Structure):
    _fields_ = [("n_ops", C.c_int32), ("n_consts", C.c_int32),
                ("ops", C.POINTER(C.c_int32)), ("consts", C.POINTER(C.c_double))]


class FitOpts(C.Structure):
    _fields_ = [("lambda0", C.c_double), ("lambda_decrease", C.c_double),
                ("lambda_increase", C.c_double), ("step_tol", C.c_double),
                ("grad_tol", C.c_double), ("max_iterations", C.c_int32),
                ("nonnegative", C.c_int32)]


class FitStats(C.Structure):
    _fields_ = [("residual_norm", C.c_double), ("iterations", C.c_int32),
                ("converged", C.c_int32), ("status", C.c_int32), ("trials", C.c_int32)]


class PsError(RuntimeError):
    """A nonzero ps_* status; message from ps_last_error()."""


_lib = None


def lib() -> C.CDLL:
    """The loaded product library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                "paper_1904_09538_b200/csrc). There is no CPU fallback.")
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def _declare(L: C.CDLL) -> None:
    P = C.POINTER
    L.ps_last_error.restype = C.c_char_p
    L.ps_version.restype = C.c_char_p
    L.ps_desc_from_id.argtypes = [C.c_char_p, P(KernelDesc)]
    L.ps_kernel_io.argtypes = [P(KernelDesc), P(IoInfo)]
    L.ps_init.argtypes = [C.c_int, P(C.c_void_p)]
    L.ps_destroy.argtypes = [C.c_void_p]
    L.ps_device_info.argtypes = [C.c_void_p, P(C.c_int), P(C.c_int), P(C.c_size_t),
                                 P(C.c_size_t)]
    L.ps_prepare.argtypes = [C.c_void_p, P(KernelDesc), C.c_int, C.c_uint64]
    L.ps_measure.argtypes = [C.c_void_p, P(KernelDesc), C.c_int, C.c_int, P(C.c_double)]
    L.ps_measure_summary.argtypes = [C.c_void_p, P(KernelDesc), C.c_int, C.c_int, C.c_double,
                                     P(C.c_double), P(C.c_int)]
    L.ps_run_timed.argtypes = [C.c_void_p, P(KernelDesc), C.c_int, P(C.c_double)]
    L.ps_run_verify.argtypes = [C.c_void_p, P(KernelDesc), P(C.c_void_p), C.c_int,
                                P(C.c_void_p), C.c_int]
    L.ps_buffer.argtypes = [C.c_void_p, C.c_int, C.c_int, P(C.c_void_p), P(C.c_int64)]
    L.ps_fit_lm_batched.argtypes = [C.c_void_p, P(Bytecode), P(Bytecode), C.c_int, C.c_int,
                                    P(C.c_double), P(C.c_double), C.c_int, C.c_int,
                                    P(FitOpts), P(C.c_double), P(FitStats)]
    L.ps_run_host.argtypes = [C.c_void_p, P(KernelDesc), P(C.c_void_p), C.c_int, P(C.c_void_p),
                              C.c_int, P(C.c_double)]
    L.ps_run_host_batch.argtypes = [C.c_void_p, C.c_int, P(KernelDesc), P(C.c_void_p),
                                    P(C.c_void_p), P(C.c_double)]
    L.ps_run_host_batch_ex.argtypes = [C.c_void_p, C.c_int, P(KernelDesc), P(C.c_void_p),
                                       P(C.c_void_p), P(C.c_uint64), P(C.c_double)]
    L.ps_trim.argtypes = [C.c_void_p]
    L.ps_host_alloc.argtypes = [C.c_size_t, P(C.c_void_p)]
    L.ps_host_free.argtypes = [C.c_void_p]
    L.ps_mark.argtypes = [C.c_void_p, C.c_int]
    L.ps_elapsed.argtypes = [C.c_void_p, C.c_int, C.c_int, P(C.c_double)]
    for name in ("ps_run_host", "ps_run_host_batch", "ps_run_host_batch_ex", "ps_trim", "ps_host_alloc", "ps_host_free", "ps_mark", "ps_elapsed"):
        getattr(L, name).restype = C.c_int
    for name in ("ps_desc_from_id", "ps_kernel_io", "ps_init", "ps_destroy", "ps_device_info",
                 "ps_prepare", "ps_measure", "ps_measure_summary", "ps_run_timed",
                 "ps_run_verify", "ps_buffer", "ps_fit_lm_batched", "ps_eval_batched"):
        getattr(L, name).restype = C.c_int


def check(rc: int) -> None:
    if rc != 0:
        raise PsError(lib().ps_last_error().decode())


def desc_from_id(variant_id: str) -> KernelDesc:
    d = KernelDesc()
    check(lib().ps_desc_from_id(variant_id.encode(), C.byref(d)))
    return d


def kernel_io(desc: KernelDesc) -> IoInfo:
    io = IoInfo()
    check(lib().ps_kernel_io(C.byref(desc), C.byref(io)))
    return io


def exported_symbols() -> list[str]:
    """ps_* function names declared in include/perfseer_b200.h."""
    import re
    hdr = (_HERE.parent / "include" / "perfseer_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*) (ps_\w+)\(", hdr, re.M)))
