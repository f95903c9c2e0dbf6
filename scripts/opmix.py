"""Opcode mix from `ncu -i REP --page source --csv --print-source sass` (one kernel):
warp instructions executed per opcode, ÷ UNITS.  usage: opmix.py export.csv [units]"""
import csv
import sys
from collections import Counter

units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
c = Counter()
ii = None
for r in csv.reader(open(sys.argv[1])):
    if "Instructions Executed" in r:
        ii = r.index("Instructions Executed")
        continue
    if ii is None or len(r) <= ii:
        continue
    src = r[1].strip()
    try:
        n = float(r[ii])
    except ValueError:
        continue
    if not src:
        continue
    t = src.split()
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += n
tot = sum(c.values())
for k, v in c.most_common(32):
    print(f"{k:10s} {v / units:9.1f} {100 * v / tot:5.1f}%")
print(f"total {tot / units:.1f} per unit")
