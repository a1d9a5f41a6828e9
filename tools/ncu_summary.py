"""Summarise an ncu report of the fused pass kernel into profiles/ (text + json).

usage: python tools/ncu_summary.py gpurun_out/prof_<tag>.ncu-rep profiles/<round>_<tag>
"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    hdr, units, row = r[0], r[1], r[2]
    m = {h: (v, u) for h, u, v in zip(hdr, units, row)}
    summary = {"kernel": m.get("Kernel Name", ("?", ""))[0], "metrics": {k: m[k] for k in KEYS if k in m}}
    stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for h, (v, u) in m.items()
              if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and
              v.replace(".", "", 1).isdigit()]
    stalls.sort(key=lambda x: -x[1])
    summary["stall_samples"] = stalls[:12]
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    h2 = rows[1]
    i_src, i_ex = h2.index("Source"), h2.index("Instructions Executed")
    mix, total = collections.Counter(), 0
    for x in rows[2:]:
        if len(x) <= i_ex or not x[i_ex].isdigit():
            continue
        toks = x[i_src].strip().split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        mix[op] += int(x[i_ex])
        total += int(x[i_ex])
    summary["instruction_mix_pct"] = [(k, round(100 * v / total, 2)) for k, v in mix.most_common(20)]
    with open(out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    with open(out + ".txt", "w") as fh:
        fh.write(f"report: {rep}\nkernel: {summary['kernel']}\n")
        for k, (v, u) in summary["metrics"].items():
            fh.write(f"{k:70s} {v} {u}\n")
        fh.write("stall samples: " + ", ".join(f"{a}={b:.0f}" for a, b in stalls[:12]) + "\n")
        fh.write("instruction mix %: " + ", ".join(f"{a}={b}" for a, b in summary["instruction_mix_pct"]) + "\n")
    print(open(out + ".txt").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
