#!/usr/bin/env python3
"""Markdown table of a round's bench lines (profiles/README_rNN.md).

  python tools/round_table.py profiles/bench_r01_C{1,2,3,4,5}.json
"""
import json
import sys


def main():
    print("| config | kernel | ms/step | WPCU/s | comb cells/clk/SM | SURVEY frac | native (ceiling) | e2e WPCU/s |"
          " CPU reference WPCU/s (cores) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for f in sys.argv[1:]:
        d = json.loads(open(f).read().strip().split("\n")[-1])
        r = d.get("roofline") or {}
        kb = r.get("kernel_alu_bound") or {}
        cpu = d.get("cpu_baseline") or {}
        wl = d["config"]["workload"].split(":")[0]
        print(f"| {wl} | `{d.get('kernel', '')}` | {d['ms_per_step']:.4g} | {d['value']:.3e} | "
              f"{kb.get('cells_per_clk_per_sm', 0):.1f} | {r.get('frac', 0):.2f} | "
              f"{kb.get('frac', 0):.2f} ({kb.get('ceiling', 0):.1f}) | {d['e2e']['value']:.3e} | "
              f"{cpu.get('value', 0):.3e} ({cpu.get('cores', '-')}) |")


if __name__ == "__main__":
    main()
