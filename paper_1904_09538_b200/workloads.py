"""Calibration workloads: which measurement kernels calibrate which model, and
which application variants the calibrated model must predict.

Each workload follows the paper's Fig. 5 pairing of models, measurement
kernels and features and SURVEY Appendix C's model
expressions in the reference grammar; kernels come from the B200 catalog
(ps_catalog "b200", csrc/host/ps_catalog.cpp).
"""
from __future__ import annotations

from dataclasses import dataclass, field

OUTPUT = "f_exec_wall_time_cuda_b200_0"

# Feature ids (reference grammar, features.cpp:124-249).
G16 = "f_mem_access_global_float32_lstrides:{0:1;1:>1}_gstrides:{0:16;1:>16}_afr:1"
# the same AFR-1 pattern split by direction (the gmem microbenchmarks with 1
# and 2 input arrays separate a load from a store cost)
G16L = "f_mem_access_global_float32_load_lstrides:{0:1;1:>1}_gstrides:{0:16;1:>16}_afr:1"
G16S = "f_mem_access_global_float32_store_lstrides:{0:1;1:>1}_gstrides:{0:16;1:>16}_afr:1"
OPS = {"add": "f_op_float32_add", "mul": "f_op_float32_mul", "madd": "f_op_float32_madd"}
LMEM = "f_mem_access_local_float32"
BAR = "f_sync_barrier_local"
GROUPS = "f_thread_groups"
LAUNCH = "f_sync_kernel_launch"


def _tag(t: str) -> str:
    return f"f_mem_access_tag:{t}"


def _sum(terms: list[str]) -> str:
    return " + ".join(terms)


def linear_model(gmem: list[tuple[str, str]], onchip: list[tuple[str, str]]) -> str:
    """ovh + c_gmem + c_onchip (paper Eq. 1)."""
    ovh = [f"p_bar * {BAR} * {GROUPS}", f"p_group * {GROUPS}", f"p_launch * {LAUNCH}"]
    terms = ovh + [f"{p} * {f}" for p, f in gmem] + [f"{p} * {f}" for p, f in onchip]
    return OUTPUT + "\n" + _sum(terms) + "\n"


def overlap_model(gmem: list[tuple[str, str]], onchip: list[tuple[str, str]]) -> str:
    """ovh + cg*sstep(cg - co; p_edge) + co*sstep(co - cg; p_edge) (Eqs. 4-5)."""
    ovh = _sum([f"p_bar * {BAR} * {GROUPS}", f"p_group * {GROUPS}", f"p_launch * {LAUNCH}"])
    cg = "(" + _sum([f"{p} * {f}" for p, f in gmem]) + ")"
    co = "(" + _sum([f"{p} * {f}" for p, f in onchip]) + ")"
    return (OUTPUT + "\n" + ovh + f" + {cg} * sstep({cg} - {co}; p_edge) + "
            f"{co} * sstep({co} - {cg}; p_edge)\n")


def smooth_max(a: str, b: str, edge: str) -> str:
    """max(a, b) through the paper's tanh step (Eq. 5) on the NORMALISED
    difference (a - b) / (a + b): the step argument is dimensionless, so one
    p_edge is equally sharp for a 5 us and a 200 ms kernel (the paper's
    sstep(a - b) needs p_edge ~ 1/t)."""
    s = f"(({a}) + ({b}) + 1e-15)"  # + 1 fs: defined when both costs vanish
    return (f"({a}) * sstep((({a}) - ({b})) / {s}; {edge}) + "
            f"({b}) * sstep((({b}) - ({a})) / {s}; {edge})")


def sharp_max(a: str, b: str, k: float = 40.0) -> str:
    """smooth_max with a fixed sharpness k on the normalised difference: a 5%
    cost gap already selects the larger term to 99%, i.e. the sm_100 pipes
    (LSU/L1, shared, FMA) are taken to overlap completely; no edge parameter
    is fitted."""
    s = f"(({a}) + ({b}) + 1e-15)"
    return (f"({a}) * (tanh({k} * (({a}) - ({b})) / {s}) + 1) / 2 + "
            f"({b}) * (tanh({k} * (({b}) - ({a})) / {s}) + 1) / 2")


def max3_model(gmem: list[tuple[str, str]], ops: list[tuple[str, str]],
               lmem: list[tuple[str, str]], k: float = 40.0) -> str:
    """launch/group overhead + max(c_gmem, c_ops, c_lmem, c_barrier) with
    fixed-sharpness steps: on sm_100 the LSU/L1 path, the FMA pipe and the
    shared-memory pipe run concurrently, and a work-group waiting at a
    barrier costs nothing extra while other resident groups keep the binding
    pipe busy."""
    ovh = _sum([f"p_group * {GROUPS}", f"p_launch * {LAUNCH}"])
    cg = _sum([f"{p} * {f}" for p, f in gmem])
    cops = _sum([f"{p} * {f}" for p, f in ops])
    cl = _sum([f"{p} * {f}" for p, f in lmem])
    cb = f"p_bar * {BAR} * {GROUPS}"
    onchip = sharp_max(cops, sharp_max(cl, cb, k), k)
    return OUTPUT + "\n" + ovh + " + " + sharp_max(cg, onchip, k) + "\n"


def lsu_model(gmem: list[tuple[str, str]], ops: list[tuple[str, str]],
              lmem: list[tuple[str, str]], k: float = 40.0) -> str:
    """launch/group overhead + max(c_gmem + c_lmem, c_ops, c_barrier): on
    sm_100 global loads that hit L1 and shared-memory accesses are issued
    through the same LSU/MIO pipe and do not overlap each other; either
    overlaps the FP32 pipe."""
    ovh = _sum([f"p_group * {GROUPS}", f"p_launch * {LAUNCH}"])
    cmem = _sum([f"{p} * {f}" for p, f in gmem] + [f"{p} * {f}" for p, f in lmem])
    cops = _sum([f"{p} * {f}" for p, f in ops])
    cb = f"p_bar * {BAR} * {GROUPS}"
    return OUTPUT + "\n" + ovh + " + " + sharp_max(cmem, sharp_max(cops, cb, k), k) + "\n"


def lsu2_model(hbm: list[tuple[str, str]], tags: list[tuple[str, str]],
               ops: list[tuple[str, str]], lmem: list[tuple[str, str]], k: float = 40.0) -> str:
    """launch/group overhead + max(c_hbm, c_tags + c_lmem, c_ops, c_barrier):
    the generic AFR-1 streams (G16/G18) calibrated by the HBM
    microbenchmarks are DRAM-bandwidth cost and overlap everything on chip;
    the tagged application accesses (mostly L1/L2 hits, each calibrated by
    its work-removed kernel) share the LSU/MIO pipe with shared-memory
    accesses, so those two add; the FP32 pipe and barriers overlap both."""
    ovh = _sum([f"p_group * {GROUPS}", f"p_launch * {LAUNCH}"])
    ch = _sum([f"{p} * {f}" for p, f in hbm])
    cl = _sum([f"{p} * {f}" for p, f in tags] + [f"{p} * {f}" for p, f in lmem])
    cops = _sum([f"{p} * {f}" for p, f in ops])
    cb = f"p_bar * {BAR} * {GROUPS}"
    return (OUTPUT + "\n" + ovh + " + " +
            sharp_max(ch, sharp_max(cl, sharp_max(cops, cb, k), k), k) + "\n")


def ldst_model(loads: list[tuple[str, str]], stores: list[tuple[str, str]],
               ops: list[tuple[str, str]], lmem: list[tuple[str, str]], k: float = 40.0,
               group_pipe: bool = False) -> str:
    """launch (+ group) overhead + max(c_load + c_lmem, c_store, c_ops, c_barrier
    [, c_group]): on sm_100 loads and shared-memory accesses occupy the
    LSU/MIO pipe and L1, while global stores retire through the L2 write path
    without holding the loads up (the DG variants' uncoalesced res stores
    overlap their row loads: sum of the work-removed kernels >> full time);
    the FP32 pipe and barriers overlap both. With group_pipe the per-group
    launch cost is one more overlapping pipe instead of an additive term
    (the CTA scheduler issues new groups while resident ones run)."""
    cl = _sum([f"{p} * {f}" for p, f in loads] + [f"{p} * {f}" for p, f in lmem])
    cs = _sum([f"{p} * {f}" for p, f in stores])
    cops = _sum([f"{p} * {f}" for p, f in ops])
    cb = f"p_bar * {BAR} * {GROUPS}"
    cg = f"p_group * {GROUPS}"
    inner = sharp_max(cops, sharp_max(cb, cg, k) if group_pipe else cb, k)
    body = sharp_max(cl, sharp_max(cs, inner, k), k)
    ovh = f"p_launch * {LAUNCH}" + ("" if group_pipe else f" + {cg}")
    return OUTPUT + "\n" + ovh + " + " + body + "\n"


def overlap3_model(gmem: list[tuple[str, str]], ops: list[tuple[str, str]],
                   lmem: list[tuple[str, str]]) -> str:
    """ovh + max(c_gmem, max(c_ops, c_lmem)): the paper's overlap form with the
    on-chip cost itself split into the FP32 pipe and the shared-memory pipe,
    which on sm_100 issue concurrently (a kernel bound by LDS wavefronts hides
    its FFMAs, e.g. the PF matmul)."""
    ovh = _sum([f"p_bar * {BAR} * {GROUPS}", f"p_group * {GROUPS}", f"p_launch * {LAUNCH}"])
    cg = _sum([f"{p} * {f}" for p, f in gmem])
    cops = _sum([f"{p} * {f}" for p, f in ops])
    cl = _sum([f"{p} * {f}" for p, f in lmem])
    return OUTPUT + "\n" + ovh + " + " + smooth_max(cg, smooth_max(cops, cl, "p_edge2"), "p_edge") + "\n"


ONCHIP = [("p_f32add", OPS["add"]), ("p_f32mul", OPS["mul"]), ("p_f32madd", OPS["madd"]),
          ("p_f32l", LMEM)]

# Microbenchmark tag sets common to every application (ps_catalog "b200").
MICRO_TAGS = [
    ["gmem_pattern_16"],
    ["flops_add_pattern"], ["flops_mul_pattern"], ["flops_madd_pattern"],
    ["lmem_shuffle"], ["barrier_knl"], ["empty_knl"], ["overlap_knl"],
]


@dataclass
class Workload:
    name: str
    description: str
    calibration_tags: list[list[str]]
    application_tags: list[list[str]]
    models: dict[str, str]
    # variant identity for per-variant error: generator args except the size
    variant_keys: tuple[str, ...] = ("prefetch",)
    size_keys: tuple[str, ...] = ("n",)
    hbm_generators: tuple[str, ...] = ("gmem_pattern", "overlap_knl")
    extra: dict = field(default_factory=dict)
    # C5 point column of each size parameter (predict.c5_points)
    c5_coords: dict = field(default_factory=lambda: {"n": 0})
    # application sizes held out for model selection (workloads.size_of
    # strings): the headline model is the candidate with the lowest geomean
    # error on these, and its error is reported on the remaining sizes
    validation_sizes: tuple[str, ...] = ()
    # fallback headline when no validation sizes were measured
    headline_model: str = "lsu"


MATMUL_GMEM = [("p_g16", G16), ("p_mmPFa", _tag("mm-PF-a")), ("p_mmPFb", _tag("mm-PF-b")),
               ("p_mmnoPFa", _tag("mm-noPF-a")), ("p_mmnoPFb", _tag("mm-noPF-b"))]

MATMUL_LOADS = [("p_g16l", G16L)] + MATMUL_GMEM[1:]
MATMUL_STORES = [("p_g16s", G16S)]

MATMUL = Workload(
    name="matmul",
    description=("BASELINE.json configs[1]: square fp32 matmul, prefetch (PF) and no-prefetch "
                 "(noPF) 16x16 variants, n = 512..8192, model calibrated on B200 from the "
                 "microbenchmark sweep plus the mm-* work-removed kernels (PAPER.md:2145-2330)"),
    calibration_tags=MICRO_TAGS + [["matmul_sq_rm"]],
    application_tags=[["matmul_sq"]],
    models={"linear": linear_model(MATMUL_GMEM, ONCHIP),
            "nonlinear": overlap_model(MATMUL_GMEM, ONCHIP),
            "overlap3": overlap3_model(MATMUL_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "max3": max3_model(MATMUL_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "lsu": lsu_model(MATMUL_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "lsu2": lsu2_model(MATMUL_GMEM[:1], MATMUL_GMEM[1:], ONCHIP[:3], ONCHIP[3:]),
            "ldst": ldst_model(MATMUL_LOADS, MATMUL_STORES, ONCHIP[:3], ONCHIP[3:]),
            "ldst_g": ldst_model(MATMUL_LOADS, MATMUL_STORES, ONCHIP[:3], ONCHIP[3:],
                                 group_pipe=True)},
    variant_keys=("prefetch",),
    validation_sizes=("n=1024", "n=4096"),
    size_keys=("n",),
)

G18 = "f_mem_access_global_float32_lstrides:{0:1;1:>1}_gstrides:{0:18;1:>18}_afr:1"
FD_GMEM = [("p_g16", G16), ("p_g18", G18),
           ("p_fd16u", _tag("fd-16x16-u")), ("p_fd16res", _tag("fd-16x16-res")),
           ("p_fd18u", _tag("fd-18x18-u")), ("p_fd18res", _tag("fd-18x18-res"))]

# the 18x18 gmem benchmark has one input array only: its load and store counts
# are collinear, so G18 stays undirected (with the loads)
FD_LOADS = [("p_g16l", G16L), ("p_g18", G18), ("p_fd16u", _tag("fd-16x16-u")),
            ("p_fd18u", _tag("fd-18x18-u"))]
FD_STORES = [("p_g16s", G16S), ("p_fd16res", _tag("fd-16x16-res")),
             ("p_fd18res", _tag("fd-18x18-res"))]

FD = Workload(
    name="fd",
    description=("BASELINE.json configs[0]: five-point FD stencil, 16x16 and 18x18 tiles, "
                 "grids 1120^2..8176^2 (9 sizes), calibrated from the microbenchmark sweep (gmem 16x16 and "
                 "18x18 patterns) plus the fd-* work-removed kernels (PAPER.md:2560-2670); "
                 "18x18 sub-group counts use the ceil(324/32) extension (SURVEY A1)"),
    calibration_tags=MICRO_TAGS + [["gmem_pattern_18"], ["finite_diff_rm"]],
    application_tags=[["finite_diff"]],
    models={"linear": linear_model(FD_GMEM, ONCHIP),
            "nonlinear": overlap_model(FD_GMEM, ONCHIP),
            "max3": max3_model(FD_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "lsu": lsu_model(FD_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "lsu2": lsu2_model(FD_GMEM[:2], FD_GMEM[2:], ONCHIP[:3], ONCHIP[3:]),
            "ldst": ldst_model(FD_LOADS, FD_STORES, ONCHIP[:3], ONCHIP[3:]),
            "ldst_g": ldst_model(FD_LOADS, FD_STORES, ONCHIP[:3], ONCHIP[3:], group_pipe=True)},
    variant_keys=("tile",),
    # the five sizes between the four calibration sizes (ps_catalog.cpp)
    validation_sizes=("n=1680", "n=2800", "n=3360", "n=5600", "n=6272"),
    size_keys=("n",),
    extra={"options": {"partial_subgroups": "round_up"}},
    c5_coords={"n": 1},
)

DG_TAGS = ["dg-noPF-u", "dg-noPF-res", "dg-uPFnoPF-dm", "dg-uPF-u", "dg-uPF-res", "dg-dmPF-dm",
           "dg-dmPF-u", "dg-dmPF-res", "dg-dmPFtrans-u", "dg-dmPFtrans-res"]
DG_GMEM = [("p_g16", G16)] + [("p_" + t.replace("-", "_"), _tag(t)) for t in DG_TAGS]

DG_LOADS = [("p_g16l", G16L)] + [("p_" + t.replace("-", "_"), _tag(t)) for t in DG_TAGS
                                  if not t.endswith("-res")]
DG_STORES = [("p_g16s", G16S)] + [("p_" + t.replace("-", "_"), _tag(t)) for t in DG_TAGS
                                   if t.endswith("-res")]

DG = Workload(
    name="dg",
    description=("BASELINE.json configs[2]: DG differentiation res[m,k,i] = sum_j dm[m,i,j] u[k,j], "
                 "4 variants (noPF, uPF, dmPF, dmPFtrans), nmat=3, 3-D orders 1-7 (Np padded to "
                 "16, 32, 48, 64, 96, 128), nel 10^4..10^6, "
                 "calibrated from the microbenchmark sweep plus the 10 dg-* work-removed tags "
                 "(PAPER.md:2041-2050, 2354-2505)"),
    calibration_tags=MICRO_TAGS + [["dg_diff_rm"]],
    application_tags=[["dg_diff"]],
    models={"linear": linear_model(DG_GMEM, ONCHIP),
            "nonlinear": overlap_model(DG_GMEM, ONCHIP),
            "max3": max3_model(DG_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "lsu": lsu_model(DG_GMEM, ONCHIP[:3], ONCHIP[3:]),
            "lsu2": lsu2_model(DG_GMEM[:1], DG_GMEM[1:], ONCHIP[:3], ONCHIP[3:]),
            "ldst": ldst_model(DG_LOADS, DG_STORES, ONCHIP[:3], ONCHIP[3:]),
            "ldst_g": ldst_model(DG_LOADS, DG_STORES, ONCHIP[:3], ONCHIP[3:], group_pipe=True)},
    variant_keys=("variant",),
    validation_sizes=tuple(f"nelements=100000;nunit_nodes={n}" for n in (16, 32, 48, 64, 96, 128)),
    size_keys=("nelements", "nunit_nodes"),
    c5_coords={"nelements": 2, "nunit_nodes": 3},
)

WORKLOADS = {w.name: w for w in (MATMUL, FD, DG)}
# "all": one calibration sweep over the union of the three workloads' kernels
# (BASELINE.json configs[3]); every workload's models are fitted on its own rows
WORKLOAD_SETS = {"all": ["matmul", "fd", "dg"]}


def resolve(name: str) -> list[Workload]:
    if name in WORKLOAD_SETS:
        return [WORKLOADS[n] for n in WORKLOAD_SETS[name]]
    return [WORKLOADS[name]]


def variant_of(variant_id: str, keys: tuple[str, ...]) -> str:
    gen, *parts = variant_id.split("__")
    args = dict(p.split("-", 1) for p in parts)
    return gen + "".join(f"_{k}-{args[k]}" for k in keys if k in args)


def size_of(variant_id: str, keys: tuple[str, ...]) -> str:
    _, *parts = variant_id.split("__")
    args = dict(p.split("-", 1) for p in parts)
    return ";".join(f"{k}={args[k]}" for k in keys if k in args)
