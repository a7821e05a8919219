"""Executed warp-instructions of one kernel per CUDA source line: joins the
ncu source page (per-SASS-address counts) with `nvdisasm -g` line info of the
same cubin. Not product code.
usage: python tools/ncu_line_mix.py REPORT.ncu-rep CUBIN MANGLED_NAME WALK_STEPS [TOP]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter, defaultdict


def line_map(cubin, fn):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    on, cur, m = False, None, {}
    for l in dis.splitlines():
        if l.startswith(fn + ":"):
            on = True
            continue
        if on and l.startswith(".text.") or (on and l.strip().startswith(".section")):
            break
        if not on:
            continue
        g = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if g:
            cur = f"{g.group(1).split('/')[-1]}:{g.group(2)}"
            continue
        g = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if g:
            m[int(g.group(1), 16)] = (cur, g.group(2))
    return m


def main(rep, cubin, fn, steps, top=40):
    lm = line_map(cubin, fn)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    iex = h.index("Instructions Executed")
    body = [r for r in rows[hdr + 1:] if len(r) > iex and r[iex].strip().isdigit()]
    base = int(body[0][0], 16)
    by, ops = Counter(), defaultdict(Counter)
    for r in body:
        off = int(r[0], 16) - base
        ln, ins = lm.get(off, ("?", r[1]))
        toks = ins.split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        n = int(r[iex])
        by[ln] += n
        ops[ln][op] += n
    tot = sum(by.values())
    print(f"{len(lm)} mapped SASS lines; {64 * tot / steps:.1f} warp-instr per 64 lane-steps")
    for ln, n in by.most_common(top):
        top_ops = ", ".join(f"{o} {64 * c / steps:.1f}" for o, c in ops[ln].most_common(5))
        print(f"{ln:22s} {64 * n / steps:7.2f}  [{top_ops}]")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]), int(sys.argv[5]) if len(sys.argv) > 5 else 40)
