"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel totals and shares.

usage: python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/<round>_launches.txt
"""
import collections
import csv
import sys


def main(path, cmd):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hdr]
    kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn].split("(")[0].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        v = float(r[mv].replace(",", ""))
        unit = h[mv + 1] if False else None
        tot[name] += v
        cnt[name] += 1
    all_t = sum(tot.values())
    print(f"launch list: ncu --metrics gpu__time_duration.sum --clock-control none {cmd}")
    print("(per-launch times are serialised and cold-cache under ncu; the SHARE is what compares with bench.py)")
    print(f"{'launches':>8} {'total':>12} {'avg':>10}  {'share':>6}  kernel   (times in the report's unit, ns)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{cnt[k]:8d} {v:12.0f} {v / cnt[k]:10.1f}  {100 * v / all_t:5.2f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
