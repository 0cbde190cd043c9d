#!/usr/bin/env python3
"""Per-kernel totals and shares of an ncu launch list (--metrics gpu__time_duration.sum --csv).

  python tools/ncu_launch_summary.py gpurun_out/r01b/launches_C2.csv "python bench.py ... (C2)"
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    what = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            k = r[ik].split("(")[0]
            t[k] += float(r[iv].replace(",", ""))   # ns
            n[k] += 1
    tot = sum(t.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none, {what}")
    print("cold-cache serialized per-launch times; compare SHARES, not absolutes")
    for k, v in sorted(t.items(), key=lambda x: -x[1]):
        print(f"{n[k]:4d} launches {v / 1e6:10.3f} ms total {v / 1e6 / n[k]:9.3f} ms/launch  share {v / tot:7.4f}  {k}")


if __name__ == "__main__":
    main()
