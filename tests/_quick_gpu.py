import time, json
from paper_1904_09538_b200.device import CudaDevice
from paper_1904_09538_b200 import desc_from_id, kernel_io
dev = CudaDevice(0)
print(dev.info())
def vid(gen, **a): return gen + "".join(f"__{k}-{a[k]}" for k in sorted(a))
PAT = dict(dtype="float32", lsize_0=16, lsize_1=16, lid_stride_0=1, lid_stride_1=2048)
cases = []
for k in (1,2):
    for E in (1<<28, 5<<27):
        cases.append(vid("gmem_pattern", n_input_arrays=k, nelements=E, **PAT))
for op in ("add","mul","madd"):
    cases.append(vid(f"flops_{op}_pattern", m=1024, nelements=1<<22, **PAT))
cases.append(vid("lmem_shuffle", m=1024, nelements=1<<22, **PAT))
cases.append(vid("barrier_knl", m=1024, nelements=1<<23, **{k:v for k,v in PAT.items() if k!='dtype'}))
cases.append(vid("empty_knl", num_groups=16))
cases.append(vid("empty_knl", num_groups=512))
for m in (0, 4, 16):
    cases.append(vid("overlap_knl", m=m, nelements=1<<28, **PAT))
for pf in ("True","False"):
    for n in (2048, 8192):
        cases.append(vid("matmul_sq", dtype="float32", prefetch=pf, lsize_0=16, lsize_1=16, groups_fit="True", n=n))
for tile, n in (("16x16", 8176), ("18x18", 8192)):
    cases.append(vid("finite_diff", dtype="float32", tile=tile, n=n))
for v in ("noPF","uPF","dmPF","dmPFtrans"):
    cases.append(vid("dg_diff", dtype="float32", variant=v, nelements=1000000 // 16 * 16, nunit_nodes=64, nmatrices=3))
for c in cases:
    d = desc_from_id(c); io = kernel_io(d)
    t, kept = dev.measure_summary(d, trials=20, warmup=3)
    print(json.dumps({"id": c[:90], "ms": round(t*1e3, 4), "GB/s": round(io.bytes_global/t/1e9,1), "TF/s": round(io.flops/t/1e12,2), "smemTB/s": round(io.bytes_shared/t/1e12,2)}))
