"""Executed warp-instructions of one kernel in an ncu report, grouped by SASS
opcode (from the source page), per walk step and per 64 lane-steps (one warp
trip of two jumps with all lanes active). Not product code.
usage: python tools/ncu_opcode_mix.py REPORT.ncu-rep WALK_STEPS [TOP]"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(rep, steps, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    isrc, iex, ith = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    by, thr = Counter(), Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= iex or not r[iex].strip().isdigit():
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        by[op] += int(r[iex])
        thr[op] += int(r[ith])
    tot = sum(by.values())
    print(f"total {tot:.4g} warp-instr, {tot / steps:.3f} per walk step, {64 * tot / steps:.1f} per 64 lane-steps")
    for op, n in by.most_common(top):
        print(f"{op:24s} {64 * n / steps:7.2f} per 64 lane-steps  ({100 * n / tot:5.1f} %, {thr[op] / n:5.1f} thr)")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
