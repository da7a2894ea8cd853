"""Summarise `ncu --set full` reports (gpurun_out/ncu_<tag>.ncu-rep) into the
profiles/ CSV columns: duration, DRAM bytes, pipe and unit utilisation."""
import csv
import io
import subprocess
import sys

COLS = [("time_us", "gpu__time_duration.sum"),
        ("dram_read", "dram__bytes_read.sum"),
        ("dram_write", "dram__bytes_write.sum"),
        ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("fma_pipe_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        ("lds_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
        ("l1_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
        ("l2_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        ("regs", "launch__registers_per_thread")]


def summary(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    got = {}
    for name, metric in COLS:
        if metric in head:
            i = head.index(metric)
            got[name] = f"{vals[i]} {units[i]}".strip()
    got["kernel"] = vals[head.index("Kernel Name")] if "Kernel Name" in head else ""
    return got


if __name__ == "__main__":
    w = csv.writer(sys.stdout)
    w.writerow(["tag"] + [c for c, _ in COLS] + ["kernel"])
    for rep in sys.argv[1:]:
        tag = rep.rsplit("/", 1)[-1].replace("ncu_", "").replace(".ncu-rep", "")
        s = summary(rep)
        w.writerow([tag] + [s.get(c, "") for c, _ in COLS] + [s["kernel"]])
