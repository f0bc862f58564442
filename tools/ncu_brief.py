"""Brief per-kernel summary of an ncu report (the metrics the roofline notes cite).

usage: python tools/ncu_brief.py <report.ncu-rep> > profiles/<tag>_ncu_full.txt
"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
           "sm__cycles_elapsed.avg.per_second"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("----")
        print(f"  {'Kernel Name':<70} {r[hdr.index('Kernel Name')]}")
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"  {m:<70} {r[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
