"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list as a
markdown table (per kernel: launches, mean ms, share of the summed time)."""
import csv
import re
import sys
from collections import defaultdict


def main(path, title):
    rows = [l for l in open(path) if l.startswith('"')]
    r = csv.DictReader(rows)
    t = defaultdict(list)
    for x in r:
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", x["Kernel Name"]).strip()
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}[x["Metric Unit"].strip() or "ns"]
        t[name].append(float(x["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in t.values())
    print(f"# {title}\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold, serialised launches: "
          "compare shares, not absolute times)\n")
    print("| kernel | launches | mean ms | share |\n|---|---|---|---|")
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k[:110]}` | {len(v)} | {sum(v) / len(v):.3f} | {100 * sum(v) / tot:.2f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu launch list")
