"""TEST INFRASTRUCTURE ONLY: variant-id parsing and array sizes for the oracle.

A pure-Python restatement of how a generated kernel's id
(``gen__arg-value__...``, reference ``variant_id`` uipick.cpp:149-154) names
its generator and bindings, and of the global arrays each generator reads and
writes (uipick.cpp:295-664; DG per PAPER.md:2354-2436). It lets the oracle and
``bench.py --impl reference`` describe and run a workload WITHOUT loading the
product library (``libperfseer_b200.so``): ``Desc`` has the byte layout of
``ps_kernel_desc`` (include/perfseer_b200.h), which ``oracle/suite_ref.c``
consumes. ``tests/test_variants_cpu.py`` checks every field against the
product's ``ps_desc_from_id`` / ``ps_kernel_io`` over the whole B200 catalog.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

GEN = {"gmem_pattern": 1, "flops_add_pattern": 2, "flops_mul_pattern": 2,
       "flops_madd_pattern": 2, "lmem_shuffle": 3, "barrier_knl": 4, "empty_knl": 5,
       "overlap_knl": 6, "matmul_sq": 7, "matmul_sq_rm": 8, "finite_diff": 9,
       "finite_diff_rm": 10, "dg_diff": 11, "dg_diff_rm": 12, "matmul_sq_tc": 13,
       "dg_diff_tc": 14}
OP = {"flops_add_pattern": 0, "flops_mul_pattern": 1, "flops_madd_pattern": 2}
KEEP = {"a": 1, "b": 2, "u": 3, "res": 4, "dm": 5}
DG_VARIANT = {"noPF": 0, "uPF": 1, "dmPF": 2, "dmPFtrans": 3}
PATTERN_GENS = (1, 2, 3, 4, 6)


class Desc(C.Structure):
    """Same layout as ps_kernel_desc (include/perfseer_b200.h)."""
    _fields_ = [
        ("gen", C.c_int32), ("dtype", C.c_int32), ("op", C.c_int32), ("keep", C.c_int32),
        ("nelements", C.c_int64), ("lsize0", C.c_int64), ("lsize1", C.c_int64),
        ("lid_stride0", C.c_int64), ("lid_stride1", C.c_int64), ("n_inputs", C.c_int64),
        ("m", C.c_int64), ("num_groups", C.c_int64), ("n", C.c_int64),
        ("prefetch", C.c_int32), ("tile", C.c_int32), ("nel", C.c_int64), ("np", C.c_int64),
        ("nmat", C.c_int64), ("dg_variant", C.c_int32), ("reserved", C.c_int32),
    ]


@dataclass
class Io:
    """Global arrays of one launch and its algorithmic work."""
    elem_bytes: int = 4
    input_elems: list = field(default_factory=list)
    output_elems: list = field(default_factory=list)
    bytes_global: float = 0.0
    flops: float = 0.0

    @property
    def n_inputs(self) -> int:
        return len(self.input_elems)

    @property
    def n_outputs(self) -> int:
        return len(self.output_elems)


def parse(variant_id: str) -> Desc:
    gen, *parts = variant_id.split("__")
    if gen not in GEN:
        raise ValueError(f"unknown generator '{gen}' in '{variant_id}'")
    args = {}
    for p in parts:
        k, sep, v = p.partition("-")
        if not sep:
            raise ValueError(f"malformed variant argument '{p}' in '{variant_id}'")
        args[k] = v
    d = Desc()
    d.gen = GEN[gen]
    dt = args.get("dtype", "float32")
    if dt not in ("float32", "float64"):
        raise ValueError(f"unsupported dtype '{dt}'")
    d.dtype = 0 if dt == "float32" else 1
    i = lambda k: int(args[k])  # noqa: E731
    if d.gen in PATTERN_GENS:
        d.nelements, d.lsize0, d.lsize1 = i("nelements"), i("lsize_0"), i("lsize_1")
        d.lid_stride0, d.lid_stride1 = i("lid_stride_0"), i("lid_stride_1")
        if d.gen == 1:
            d.n_inputs = i("n_input_arrays")
        else:
            d.m = i("m")
        if d.gen == 2:
            d.op = OP[gen]
    elif d.gen == 5:
        d.num_groups = i("num_groups")
    elif d.gen in (7, 8, 13):
        d.n, d.lsize0, d.lsize1 = i("n"), i("lsize_0"), i("lsize_1")
        if d.gen != 13:
            d.prefetch = {"True": 1, "true": 1, "1": 1, "False": 0, "false": 0, "0": 0}[
                args["prefetch"]]
        if d.gen == 8:
            d.keep = KEEP[args["keep"]]
    elif d.gen in (9, 10):
        d.n = i("n")
        d.tile = {"16x16": 16, "18x18": 18}[args["tile"]]
        if d.gen == 10:
            d.keep = KEEP[args["keep"]]
    else:  # DG
        d.nel, d.np, d.nmat = i("nelements"), i("nunit_nodes"), i("nmatrices")
        if d.gen != 14:
            d.dg_variant = DG_VARIANT[args["variant"]]
        if d.gen == 12:
            d.keep = KEEP[args["keep"]]
    return d


def io_of(d: Desc) -> Io:
    """Arrays and algorithmic work (bytes: every array touched once)."""
    eb = 8 if d.dtype == 1 else 4
    io = Io(elem_bytes=eb)
    E, m = d.nelements, d.m
    g = d.gen
    if g == 1:
        io.input_elems = [E] * d.n_inputs
        io.output_elems = [E]
        io.bytes_global = float(eb * E * (d.n_inputs + 1))
        io.flops = float(E * (d.n_inputs - 1))
    elif g == 2:
        io.output_elems = [E]
        io.bytes_global = float(eb * E)
        io.flops = E * (2048.0 * m * (2.0 if d.op == 2 else 1.0) + 31.0)
    elif g in (3, 4):
        io.output_elems = [E]
        io.bytes_global = float(eb * E)
    elif g == 6:
        io.input_elems, io.output_elems = [E], [E]
        io.bytes_global = 2.0 * eb * E
    elif g in (7, 13):
        n = d.n
        io.input_elems, io.output_elems = [n * n, n * n], [n * n]
        io.bytes_global = 3.0 * eb * n * n
        io.flops = 2.0 * n ** 3
    elif g == 8:
        io.input_elems, io.output_elems = [d.n * d.n], [d.n * d.n]
        io.bytes_global = 2.0 * eb * d.n * d.n
    elif g == 9:
        n = d.n
        io.input_elems, io.output_elems = [(n + 2) ** 2], [n * n]
        io.bytes_global = float(eb * ((n + 2) ** 2 + n * n))
        io.flops = 5.0 * n * n
    elif g == 10:
        n, I = d.n, d.tile - 2
        if d.keep == KEEP["u"]:
            dw = (n // I) * d.tile
            io.input_elems, io.output_elems = [(n + 2) ** 2], [dw * dw]
            io.bytes_global = float(eb * ((n + 2) ** 2 + dw * dw))
        else:
            io.output_elems = [n * n]
            io.bytes_global = float(eb * n * n)
    elif g in (11, 12, 14):
        dm, u, res = d.nmat * d.np * d.np, d.nel * d.np, d.nmat * d.nel * d.np
        if g != 12:
            io.input_elems, io.output_elems = [dm, u], [res]
            io.bytes_global = 4.0 * (dm + u + res)
            io.flops = 2.0 * d.nmat * d.nel * d.np * d.np
        elif d.keep == KEEP["res"]:
            io.output_elems = [res]
            io.bytes_global = 4.0 * res
        else:
            src = u if d.keep == KEEP["u"] else dm
            io.input_elems, io.output_elems = [src], [d.np * d.nel]
            io.bytes_global = 4.0 * (src + d.np * d.nel)
    return io
