"""World-size-2 CPU (gloo) checks of the multi-GPU sweep plumbing in bench.py
(SURVEY 8(e)): LPT sharding of (kernel, trial) units, the fixed-size record
all-gather of the measurement table, and the max-over-ranks timing."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q) -> None:
    import sys
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    from paper_1904_09538_b200 import desc_from_id, kernel_io
    try:
        dist = bench.Dist()
        assert dist.world == world and dist.backend == "gloo"
        _, kernels = bench.workload_kernels("all")
        est = [bench.estimate_seconds(kernel_io(desc_from_id(k))) for k in kernels]
        trials = 3
        units = [(i, t) for i in range(len(kernels)) for t in range(trials)]
        mine = bench.lpt(units, est, world)[rank]
        # synthetic per-trial seconds, a pure function of the unit
        records = [(i, t, 1e-6 * (i + 1) + 1e-9 * t) for i, t in mine]
        table = dist.gather_table(records)
        load = sum(est[i] for i, _ in mine)
        mx = dist.max(load)
        total = dist.sum(float(len(mine)))  # launch counts add over ranks
        dist.barrier()
        # C5 prediction sharding: contiguous point blocks per rank, predictions
        # and argmins all-gathered; the fitted variants come from rank 0
        import numpy as np
        from paper_1904_09538_b200.predict import PredictionTables, c5_points
        model = ("f_exec_wall_time_cuda_b200_0\n"
                 "p_launch * f_sync_kernel_launch + p_madd * f_op_float32_madd"
                 " + p_l * f_mem_access_local_float32\n")
        base = "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-512__prefetch-"
        variants = [{"id": base + pf, "model": model, "params": [5e-6, 1e-12 * (1 + i), 2e-12],
                     "group": 0, "coords": {"n": 0}} for i, pf in enumerate(("True", "False"))]
        variants = dist.broadcast(variants if rank == 0 else None)
        t = PredictionTables(variants)
        pts = c5_points(1001)
        lo, hi = bench.c5_block(len(pts), rank, world)
        p, a = t.eval_cpu(pts[lo:hi])
        P = dist.all_gather_rows(p)
        A = dist.all_gather_rows(a.astype(np.float64)).astype(np.int64)
        fp, fa = t.eval_cpu(pts)
        c5 = (hi - lo, bool(np.array_equal(P, fp)), bool(np.array_equal(A, fa.astype(np.int64))))
        q.put((rank, len(mine), sorted(table), load, mx, len(units), c5, total))
        dist.close()
    except Exception as e:  # surfaced by the parent
        q.put((rank, "error", repr(e)))


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        item = q.get(timeout=240)
        out[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    for r, item in out.items():
        assert item[1] != "error", f"rank {r}: {item[2]}"
    return out


def test_every_unit_measured_exactly_once(results):
    r0, r1 = results[0], results[1]
    n_units = r0[5]
    assert r0[1] + r1[1] == n_units
    assert r0[1] > 0 and r1[1] > 0
    table = r0[2]
    assert table == r1[2], "all ranks see the same gathered table"
    assert len(table) == n_units
    assert len({(k, t) for k, t, _ in table}) == n_units
    for k, t, s in table:
        assert s == pytest.approx(1e-6 * (k + 1) + 1e-9 * t, rel=0, abs=0)


def test_max_over_ranks_and_lpt_balance(results):
    loads = [results[0][3], results[1][3]]
    assert results[0][4] == results[1][4] == max(loads)
    # LPT: the makespan is within one largest unit of the perfect split
    assert max(loads) - min(loads) <= max(loads) * 0.5


def test_c5_points_sharded_and_gathered(results):
    # 10^6 points in contiguous per-rank blocks, one all-gather
    n0, n1 = results[0][6][0], results[1][6][0]
    assert n0 + n1 == 1001 and abs(n0 - n1) <= 1
    for r in (0, 1):
        assert results[r][6][1], "gathered predictions equal the single-rank evaluation"
        assert results[r][6][2], "gathered argmins equal the single-rank evaluation"


def test_sum_over_ranks(results):
    # every rank sees the whole job's unit count
    n_units = results[0][5]
    assert all(item[7] == n_units for item in results.values())
