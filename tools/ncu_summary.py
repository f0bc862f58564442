"""Summarise gpurun_out ncu artefacts into profiles/ (committed).

usage: python tools/ncu_summary.py <tag> <config>
  reads gpurun_out/launches_<tag>.csv and gpurun_out/prof_<tag>.ncu-rep
  writes profiles/<tag>_launches.txt, profiles/<tag>_ncu_full.csv, updates profiles/ncu_traffic.json
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = [("tell_kernel", "tell"), ("tell_update", "tell_update"), ("ask_kernel", "ask"),
        ("eval_warp", "eval_bbob"), ("eval_block", "eval_bbob"), ("rank_kernel", "rank"),
        ("mlp", "eval_mlp")]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
           "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def kind(name):
    for k, v in KIND:
        if k in name:
            return v
    return name.split("(")[0]


def launches(tag):
    p = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    rows = list(csv.reader(open(p)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ni, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        n = r[ni].split("(")[0]
        agg[n][0] += 1
        agg[n][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none ({tag}); cold-cache, "
           f"serialised: compare shares", f"{'kernel':58s} {'n':>5s} {'total_us':>10s} "
           f"{'avg_us':>9s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k[:58]:58s} {v[0]:5d} {v[1]/1e3:10.1f} {v[1]/v[0]/1e3:9.1f} {v[1]/tot:6.3f}")
    return "\n".join(out) + "\n"


def full(tag):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    cols = ["Kernel Name"] + [m for m in METRICS if m in hdr]
    out = [cols]
    for r in rows[2:]:
        out.append([r[hdr.index(c)] for c in cols])
    return out, units, hdr


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lp):
        open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w").write(launches(tag))
    rp = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    if os.path.exists(rp):
        out, units, hdr = full(tag)
        with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.csv"), "w") as f:
            csv.writer(f).writerows(out)
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        traffic = json.load(open(tp)) if os.path.exists(tp) else {}
        per = defaultdict(list)
        cols = out[0]
        for r in out[1:]:
            rd = float(r[cols.index("dram__bytes_read.sum")]) * (1e6 if "Mbyte" in units[hdr.index("dram__bytes_read.sum")] else 1)
            wr = float(r[cols.index("dram__bytes_write.sum")]) * (1e6 if "Mbyte" in units[hdr.index("dram__bytes_write.sum")] else 1)
            per[kind(r[0])].append(rd + wr)
        traffic[cfg] = {k: sum(v) / len(v) for k, v in per.items()}
        traffic[cfg]["_source"] = f"profiles/{tag}_ncu_full.csv (ncu --set full, bytes per launch)"
        json.dump(traffic, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
