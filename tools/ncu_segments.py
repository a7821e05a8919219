"""Dynamic profile of K1 from an ncu source page: contiguous SASS regions with
the same execution count, normalised per loop trip (the execution count of the
loop-top active test). Not product code.
usage: ncu -i REP --page source --csv --print-source sass > x.csv; python tools/ncu_segments.py x.csv [min_dyn]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
isrc, iex, ith = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
R = [r for r in rows[2:] if r[iex].isdigit()]
tot = sum(int(r[iex]) for r in R)
top = [int(r[iex]) for r in R if 'LOP3.LUT P' in r[isrc] and '0xff, RZ, 0xc0' in r[isrc]]
trips = max(top)
print(f"warp-instructions {tot:.4g}, loop trips {trips:.4g}, per trip {tot / trips:.1f}")
seg = []
cur = None
for i, r in enumerate(R):
    n = int(r[iex]) / trips
    if cur is None or abs(cur['n'] - n) > 0.15 * max(cur['n'], 0.05):
        cur = {'start': i, 'n': n, 'cnt': 0, 'sum': 0.0, 'thr': 0.0, 'ops': collections.Counter()}
        seg.append(cur)
    cur['cnt'] += 1
    cur['sum'] += n
    cur['thr'] += int(r[ith]) / trips
    t = r[isrc].split()
    op = t[1] if t[0].startswith('@') else t[0]
    cur['ops'][op.split('.')[0]] += 1
lim = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
for s in seg:
    if s['sum'] > lim:
        print(f"{s['start']:5d} exec/trip={s['n']:5.2f} len={s['cnt']:4d} dyn={s['sum']:7.1f} "
              f"thr={s['thr'] / s['sum']:5.1f}", dict(s['ops'].most_common(6)))
