"""Summarise an ncu report (details page) or a launch-list csv into profiles/.

  python tools/ncu_summary.py report.ncu-rep  > profiles/xxx.txt
  python tools/ncu_summary.py launches.csv    > profiles/xxx.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ("Duration", "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Achieved Occupancy", "Theoretical Occupancy", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Issued Instructions", "Eligible Warps Per Scheduler",
        "Active Warps Per Scheduler", "No Eligible")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64", "sm__pipe_fp64_cycles_active",
       "smsp__inst_executed_pipe_fp64", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared", "lts__t_sector_hit_rate",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg.per_second", "gpu__time_duration.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    kn, mn, mu, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    print("report:", path)
    seen = set()
    for r in rows[1:]:
        if len(r) <= mv:
            continue
        if r[mn] in KEYS and (r[kn], r[mn]) not in seen:
            seen.add((r[kn], r[mn]))
            print(f"  {r[kn][:60]:60s} | {r[mn]:40s} | {r[mv]:>14s} {r[mu]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hdr, units = rr[0], rr[1]
        for r in rr[2:]:
            print("  raw:", r[hdr.index("Kernel Name")][:60] if "Kernel Name" in hdr else "")
            for i, name in enumerate(hdr):
                if any(name.startswith(k) for k in RAW):
                    print(f"    {name:70s} {r[i]:>18s} {units[i]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]].append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print("launch list:", path, "(ncu, cold-cache serialised: compare shares)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k[:70]:70s} launches {len(v):5d}  total {sum(v):12.1f} us  share {sum(v) / tot:6.1%}  "
              f"avg {sum(v) / len(v):10.1f} us")


if __name__ == "__main__":
    p = sys.argv[1]
    rep(p) if p.endswith(".ncu-rep") else launches(p)
