"""Median per-kernel duration (us) from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import io
import statistics
import sys
from collections import defaultdict

txt = open(sys.argv[1]).read()
rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = defaultdict(list)
for r in rows[1:]:
    n = r[ki].split("(")[0].split("::")[-1]
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] in ("ns", "nsecond") else (v * 1000 if r[ui] in ("ms", "msecond") else v)
    d[n].append(v)
for n, vs in sorted(d.items(), key=lambda kv: -statistics.median(kv[1])):
    print(f"{n:44s} n={len(vs):3d} median {statistics.median(vs):9.2f} us")
