"""Markdown summary of an `ncu --set full` capture of K1 (raw page metrics +
stall reasons + the source-page instruction count per walk step).
usage: python tools/ncu_k1_summary.py REPORT.ncu-rep PLAIN_BENCH_LOG "title" > out.md"""
import csv
import io
import json
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "Duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM frequency"),
    ("smsp__inst_executed.sum", "Executed warp-instructions"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "Issue slots busy (%)"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe (IMAD) (%)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe (%)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe (%)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "Achieved occupancy (%)"),
    ("launch__registers_per_thread", "Registers per thread"),
    ("launch__occupancy_limit_registers", "Block limit (registers)"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "Active threads per warp-instruction"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(rep, plain, title):
    h, units, v = raw(rep)
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    line = [l for l in open(plain) if l.startswith("{")][-1]
    steps = json.loads(line)["walk_steps_per_step"]
    print(f"# {title}\n")
    print("| metric | value |\n|---|---|")
    for k, name in WANT:
        if k in d:
            print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
    inst = float(d["smsp__inst_executed.sum"].replace(",", ""))
    print(f"| walk steps in the launch (bench log) | {steps:,} |")
    print(f"| **warp-instructions per walk step** | **{inst / steps:.3f}** |")
    stalls = {k.split("stalled_")[1]: float(v.replace(",", "") or 0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
    print("\nWarp-state samples (all): " + ", ".join(f"{k} {100 * x / tot:.1f} %" for k, x in top))


if __name__ == "__main__":
    main(*sys.argv[1:4])
