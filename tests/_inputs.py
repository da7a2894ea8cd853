"""Shared input builders for parity tests (seed pattern keyed by array name)."""
from __future__ import annotations

import numpy as np

from oracle import suite as oracle_suite
from paper_1904_09538_b200 import _abi

INPUT_NAMES = {
    1: lambda d, i: "in0" if i == 0 else "in1",
    6: lambda d, i: "in0",
    7: lambda d, i: "a" if i == 0 else "b",
    8: lambda d, i: "a" if d.keep == 1 else "b",
    9: lambda d, i: "u",
    10: lambda d, i: "u",
    11: lambda d, i: "diff_mat" if i == 0 else "u",
    12: lambda d, i: "u" if d.keep == 3 else "diff_mat",
    13: lambda d, i: "a" if i == 0 else "b",
    14: lambda d, i: "diff_mat" if i == 0 else "u",
}


def make_inputs(desc, io, mode: str = "seed17", seed: int = 7) -> list[np.ndarray]:
    dt = np.float32 if io.elem_bytes == 4 else np.float64
    out = []
    for i in range(io.n_inputs):
        n = int(io.input_elems[i])
        if mode == "seed17":
            name = INPUT_NAMES[desc.gen](desc, i)
            out.append(oracle_suite.seed_values(name, n, dt))
        else:
            out.append(oracle_suite.uniform_values(n, seed + 1000 * i, dt))
    return out


def desc_io(variant_id: str):
    d = _abi.desc_from_id(variant_id)
    return d, _abi.kernel_io(d)
