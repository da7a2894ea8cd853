"""The straight-line model programs K17 and K18 execute (ps_model_program:
common subexpressions computed once, slots reused after their last use)
give the same bits as evaluating the reference's expression trees — the
model and every symbolic derivative (eval_expr / diff_expr, model.cpp:238-330)
— here through the postfix bytecode tree walk."""
from __future__ import annotations

import math

import numpy as np
import pytest


def _run_postfix(ops, consts, p, f):
    st = []
    for w in ops:
        code, arg = int(w) >> 16, int(w) & 0xffff
        if code == 0:
            st.append(consts[arg])
        elif code == 1:
            st.append(p[arg])
        elif code == 2:
            st.append(f[arg])
        elif code == 7:
            st[-1] = math.tanh(st[-1])
        else:
            b, a = st.pop(), st.pop()
            st.append(a + b if code == 3 else a - b if code == 4 else a * b if code == 5 else a / b)
    return st[0]


def _run_program(pr, p, f):
    s = [0.0] * pr["n_slots"]
    ins = pr["insns"]
    for i in range(0, len(ins), 2):
        op, d = ins[i] >> 16, ins[i] & 0xffff
        a, b = ins[i + 1] >> 16, ins[i + 1] & 0xffff
        if op == 0:
            v = pr["consts"][a]
        elif op == 1:
            v = p[a]
        elif op == 2:
            v = f[a]
        elif op == 7:
            v = math.tanh(s[a])
        else:
            x, y = s[a], s[b]
            v = x + y if op == 3 else x - y if op == 4 else x * y if op == 5 else x / y
        s[d] = v
    return [s[o] for o in pr["outputs"]]


def _cases():
    from paper_1904_09538_b200 import workloads
    return [(w.name, m) for w in workloads.WORKLOADS.values() for m in w.models]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c[0]}-{c[1]}")
def test_program_equals_tree_walk_bitwise(case):
    from paper_1904_09538_b200 import host, workloads
    wl = workloads.WORKLOADS[case[0]]
    m = host.HostModel(wl.models[case[1]])
    pr = m.program(with_jacobian=True)
    assert len(pr["outputs"]) == 1 + len(m.params)
    rng = np.random.default_rng(3)
    codes = [m.bytecode(-1)] + [m.bytecode(i) for i in range(len(m.params))]
    for _ in range(6):
        p = list(rng.uniform(1e-13, 1e-10, len(m.params)) * rng.choice([1, 1, -1], len(m.params)))
        f = list(np.exp(rng.uniform(0, 25, len(m.features))))
        got = _run_program(pr, p, f)
        want = [_run_postfix(ops, consts, p, f) for ops, consts, _ in codes]
        for g, w in zip(got, want):
            assert np.float64(g).tobytes() == np.float64(w).tobytes()


def test_program_shares_subexpressions():
    from paper_1904_09538_b200 import host, workloads
    m = host.HostModel(workloads.DG.models["ldst_g"])
    pr = m.program(True)
    tree_ops = sum(len(m.bytecode(i)[0]) for i in range(-1, len(m.params)))
    assert pr["n_nodes"] * 100 < tree_ops and pr["n_slots"] <= 64
