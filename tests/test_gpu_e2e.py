"""ps_run_host_batch (the pipelined end-to-end path through pinned host
buffers, used by bench.py's `e2e`): outputs equal the single-launch parity
hook bit for bit for a mixed batch (odd length, so both device slots are
reused and the last one is drained), and the batch reports positive time."""
import numpy as np
import pytest

from tests._inputs import desc_io, make_inputs

pytestmark = pytest.mark.gpu

IDS = [
    "gmem_pattern__dtype-float32__lid_stride_0-1__lid_stride_1-2048__lsize_0-16__lsize_1-16"
    "__n_input_arrays-2__nelements-1048576",
    "matmul_sq__dtype-float32__groups_fit-True__lsize_0-16__lsize_1-16__n-256__prefetch-True",
    "finite_diff__dtype-float32__n-1120__tile-16x16",
    "dg_diff__dtype-float32__nelements-4096__nmatrices-3__nunit_nodes-48__variant-noPF",
    "matmul_sq_tc__dtype-float32__lsize_0-16__lsize_1-16__n-512",
]


def test_batch_equals_single_launch():
    from paper_1904_09538_b200.device import CudaDevice, PinnedArray
    with CudaDevice(0) as dev:
        ins_all, outs_all, want = [], [], []
        for vid in IDS:
            d, io = desc_io(vid)
            ins = make_inputs(d, io, "seed17")
            want.append(dev.run(d, ins))
            pins = []
            for a in ins:
                p = PinnedArray(a.nbytes)
                p.numpy(a.dtype)[:] = a
                pins.append(p)
            ins_all.append(pins)
            outs_all.append([PinnedArray(int(io.output_elems[j]) * io.elem_bytes)
                             for j in range(io.n_outputs)])
        secs = dev.run_host_batch(IDS, ins_all, outs_all)
        assert secs > 0
        for vid, outs, w in zip(IDS, outs_all, want):
            for o, ref in zip(outs, w):
                got = o.numpy(ref.dtype)
                assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), vid
        for arrs in ins_all + outs_all:
            for a in arrs:
                a.free()


def test_batch_checksums_equal_host_sums_of_outputs():
    # the step's result without output copies: one device checksum per kernel
    from paper_1904_09538_b200.device import CudaDevice, PinnedArray
    with CudaDevice(0) as dev:
        ins_all, want = [], []
        for vid in IDS:
            d, io = desc_io(vid)
            ins = make_inputs(d, io, "seed17")
            outs = dev.run(d, ins)
            want.append(sum(int(np.sum(o.view(np.uint32), dtype=np.uint64)) for o in outs) % (1 << 64))
            pins = []
            for a in ins:
                p = PinnedArray(a.nbytes)
                p.numpy(a.dtype)[:] = a
                pins.append(p)
            ins_all.append(pins)
        secs, sums = dev.run_host_batch(IDS, ins_all, None, checksums=True)
        assert secs > 0
        assert [int(x) for x in sums] == want
        for arrs in ins_all:
            for a in arrs:
                a.free()


def test_batch_with_a_small_arena_reuses_regions_correctly(monkeypatch):
    """A device arena smaller than the batch: regions are reused as a ring and
    the copy-in of a kernel waits for the launch (and copy-out) of the kernel
    that last held its bytes — outputs still equal the single-launch hook."""
    from paper_1904_09538_b200.device import CudaDevice, PinnedArray
    ids = IDS * 3  # 15 kernels through an arena of ~2 of them
    monkeypatch.setenv("PS_E2E_ARENA_MB", "20")
    with CudaDevice(0) as dev:
        ins_all, outs_all, want = [], [], []
        for vid in ids:
            d, io = desc_io(vid)
            ins = make_inputs(d, io, "uniform", seed=len(ins_all))
            want.append(dev.run(d, ins))
            pins = []
            for a in ins:
                p = PinnedArray(a.nbytes)
                p.numpy(a.dtype)[:] = a
                pins.append(p)
            ins_all.append(pins)
            outs_all.append([PinnedArray(int(io.output_elems[j]) * io.elem_bytes)
                             for j in range(io.n_outputs)])
        for _ in range(2):
            assert dev.run_host_batch(ids, ins_all, outs_all) > 0
            for vid, outs, w in zip(ids, outs_all, want):
                for o, ref in zip(outs, w):
                    assert np.array_equal(o.numpy(ref.dtype).view(np.uint8), ref.view(np.uint8)), vid
        for arrs in ins_all + outs_all:
            for a in arrs:
                a.free()
