#!/usr/bin/env python3
"""Summarise an ncu report: key SOL / occupancy / stall metrics and the top stalled SASS lines.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 20]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

KEYS = ["Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "L1/TEX Cache Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "SM Busy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy",
        "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Block Limit Registers",
        "Block Limit Shared Mem", "Grid Size"]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ni, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    kname = rows[1][hdr.index("Kernel Name")] if len(rows) > 1 else "?"
    print("kernel:", kname)
    for r in rows[1:]:
        if len(r) > vi and r[ni] in KEYS:
            print(f"  {r[ni]}: {r[vi]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        d = dict(zip(rr[0], rr[2]))
        pipes = [("ALU", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                 ("FMA", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                 ("issue", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 ("LSU shared wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")]
        print("  pipes (% of peak):", ", ".join(f"{n} {float(d[k]):.1f}" for n, k in pipes if d.get(k)))
        def num(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None
        rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        units = dict(zip(rr[0], rr[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if rd is not None and wr is not None:
            rb = rd * scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
            wb = wr * scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
            print(f"  dram bytes per launch: read {rb:.0f} + write {wb:.0f} = {rb + wb:.0f}")
        pre = "smsp__pcsamp_warps_issue_stalled_"
        st = {k[len(pre):]: float(v.replace(",", "")) for k, v in d.items()
              if k.startswith(pre) and not k.endswith("_not_issued") and v.replace(",", "").replace(".", "").isdigit()}
        tot_st = sum(st.values()) or 1.0
        print("  warp states (pc samples):", ", ".join(f"{k} {v / tot_st:.3f}"
                                                     for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:9]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = srows[2:]
    samp = ix["Warp Stall Sampling (All Samples)"]
    ex = ix["Instructions Executed"]
    tot = sum(int(r[samp] or 0) for r in data)
    texec = sum(int(r[ex] or 0) for r in data)
    mix = Counter()
    for r in data:
        op = r[ix["Source"]].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        mix[o.split(".")[0]] += int(r[ex] or 0)
    print(f"  instruction mix (of {texec} warp-instrs):",
          ", ".join(f"{k} {v / texec:.3f}" for k, v in mix.most_common(14)))
    print(f"  top stalled SASS (of {tot} samples):")
    for r in sorted(data, key=lambda r: -int(r[samp] or 0))[:top]:
        print(f"    {int(r[samp] or 0) / tot:6.3f}  {r[ix['Source']].strip()[:70]}")


if __name__ == "__main__":
    main()
