"""Per-source-line totals from `ncu -i REP --page source --csv --print-source cuda,sass`:
warp instructions executed (÷ UNITS) and stall samples, grouped by file:line.
usage: python scripts/src_lines.py export.csv [units] [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
inst = defaultdict(float)
samp = defaultdict(float)
text = {}
fname, cur, hdr = "?", None, None
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 8:
        continue
    if row[0] not in ("", "..."):
        cur = (fname, int(row[0]))
        text[cur] = row[1].strip()[:90]
        continue
    if cur is None or row[2] in ("", "..."):
        continue
    try:
        n = float(row[hdr.index("Instructions Executed")])
        s = float(row[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    inst[cur] += n
    samp[cur] += s
tot_i = sum(inst.values())
tot_s = sum(samp.values()) or 1
print(f"total warp inst {tot_i:.0f} ({tot_i / units:.1f} per unit); samples {tot_s:.0f}")
for k in sorted(inst, key=lambda k: -samp[k])[:top]:
    print(f"{k[0]}:{k[1]:5d} inst/unit {inst[k] / units:8.1f}  samp% {100 * samp[k] / tot_s:5.1f}  {text.get(k, '')}")
