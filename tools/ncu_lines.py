"""Per-source-line instruction counts of an ncu report (source page, cuda+sass): top lines and per-region totals.

usage: python tools/ncu_lines.py <report.ncu-rep> [top_n]
"""
import collections
import csv
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg, stall, src = collections.Counter(), collections.Counter(), {}
    hdr = curfile = None
    for r in rows:
        if r and r[0] == "File Path":
            curfile = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) <= ie or not r[0]:
            continue
        key = (curfile, int(r[0]))
        src[key] = r[1].strip()[:90]
        try:
            agg[key] += int(r[ie] or 0)
            stall[key] += int(r[st] or 0)
        except ValueError:
            pass
    return agg, stall, src


if __name__ == "__main__":
    agg, stall, src = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    tot = sum(agg.values())
    print("total warp instructions", tot)
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
        print(f"{v:9d} {100 * v / tot:5.1f}% st={stall[k]:4d} {k[0]}:{k[1]} {src[k]}")
