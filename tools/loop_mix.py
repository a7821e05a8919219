"""Static opcode histogram of K1's walk loop body (from the loop top's active
test to the trip's WARPSYNC) in a tools/sass_fun.sh listing. Not product code.
usage: python tools/loop_mix.py LISTING [pattern ...]"""
import collections
import re
import sys

L = [l.rstrip() for l in open(sys.argv[1])]
a = [i for i, l in enumerate(L) if re.search(r'LOP3.LUT P\d, RZ, R\d+, 0xff, RZ, 0xc0', l)][0]
b = [i for i, l in enumerate(L) if 'WARPSYNC.ALL' in l and i > a][0]
body = L[a:b]
ops = [x.split()[1] if not x.split()[1].startswith('@') else x.split()[2] for x in body]
c = collections.Counter(ops)
print(len(body), c.most_common(50))
for pat in sys.argv[2:]:
    for l in body:
        if re.search(pat, l):
            print(l)
