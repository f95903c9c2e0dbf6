"""Summarise a gpu_round.sh output directory into profiles/<tag>_summary.md
(ncu launch list shares, per-kernel ncu metrics, bench lines)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1]
src = os.path.join("gpurun_out", tag)
out = []
out.append(f"# Profile summary {tag}\n")
bj = os.path.join(src, "bench.json")
if os.path.exists(bj):
    d = json.loads(open(bj).read().strip().splitlines()[-1])
    out.append("## bench.py (default run)\n")
    out.append("```json\n" + json.dumps(d, indent=1) + "\n```\n")
rj = os.path.join(src, "bench_ref.json")
if os.path.exists(rj):
    lines = [l for l in open(rj).read().splitlines() if l.startswith("{")]
    if lines:
        out.append("## bench.py --impl reference (oracle)\n")
        out.append("```json\n" + lines[-1] + "\n```\n")
lc = os.path.join(src, "launches.csv")
if os.path.exists(lc) and '"ID"' in open(lc).read():
    txt = open(lc).read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("edffs::", "").replace("<unnamed>::", "")
        name = name.replace("unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
        seq.append((name, v))

    def table(items, title):
        tot, cnt = defaultdict(float), defaultdict(int)
        for name, v in items:
            tot[name] += v
            cnt[name] += 1
        s_ = sum(tot.values()) or 1.0
        out.append(title + "\n")
        out.append("| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
        for k in sorted(tot, key=lambda k: -tot[k]):
            out.append(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {100 * tot[k] / s_:.1f}% |")
        out.append("")
        return tot, cnt

    table(seq, "## ncu launch list, every captured launch (`--metrics gpu__time_duration.sum --clock-control none`, "
               "cold-cache, serialised)")
    gen = [i for i, (n, _) in enumerate(seq) if n == "generation_kernel"]
    if gen:
        a = gen[0]
        b = next((i for i in range(a, len(seq)) if seq[i][0] == "random_population_kernel"), len(seq))
        # run.best() after the timed steps decodes one chromosome with its schedule
        # (lane_decode_kernel<., 1>, preceded by its order kernel): not a step
        def is_sched(nm):
            if nm.startswith("lane_decode2_kernel"):
                return nm.endswith("<1>")
            if nm.startswith("lane_decode_kernel"):
                return nm.endswith(", 1>")
            if nm.startswith("evaluate_kernel"):
                return nm.split(",")[1].strip() == "1"
            return False
        sched = [i for i in range(a, b) if is_sched(seq[i][0])]
        if sched:
            b = sched[0] - 1
        ng = sum(1 for i in gen if a <= i < b)
        tot, cnt = table(seq[a:b], f"## GA step region of the same list ({ng} generations of the bench's GA: from "
                                   "the first generation_kernel up to run.best())")
        per_step = sum(tot.values()) / ng
        out.append(f"Per generation (sum of the region / generations): {per_step:.1f} us\n")
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__average_warp_latency_per_inst_issued.ratio"]
traffic = None
for rep in ("prof_eval", "prof_gen"):
    p = os.path.join(src, rep + ".ncu-rep")
    if not os.path.exists(p):
        continue
    raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    if rep == "prof_eval" and "dram__bytes_read.sum" in h:
        # one evaluate launch = the order + decode kernels of the capture
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += sum(float(r[i].replace(",", "")) * scale.get(units[i], 1.0) for r in rows[2:])
        def col(m):
            return [r[h.index(m)] for r in rows[2:]] if m in h else None
        traffic = {"kernels": [r[h.index("Kernel Name")].split("(")[0] for r in rows[2:]],
                   "issue_active_pct": col("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "alu_pipe_pct": col("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                   "duration_us": col("gpu__time_duration.sum"),
                   "inst_executed": col("smsp__inst_executed.sum"),
                   "thread_inst_per_inst": col("smsp__thread_inst_executed_per_inst_executed.ratio"),
                   "sm_cycles_per_second": col("sm__cycles_elapsed.avg.per_second"),
                   "dram_bytes_per_evaluate": tot, "population": 65536,
                   "source": f"ncu --set full, gpurun_out/{tag}/prof_eval.ncu-rep (scripts/prof_eval.py 65536)"}
    out.append(f"## ncu --set full: {rep}\n")
    out.append("| metric | " + " | ".join(r[h.index("Kernel Name")].split("(")[0][-40:] for r in rows[2:]) + " |")
    out.append("|---|" + "---|" * (len(rows) - 2))
    for w in want:
        if w in h:
            i = h.index(w)
            out.append(f"| {w} ({units[i]}) | " + " | ".join(r[i] for r in rows[2:]) + " |")
    out.append("")
if traffic is not None:
    json.dump(traffic, open(os.path.join("profiles", f"{tag}_traffic.json"), "w"), indent=1)
    out.append(f"DRAM traffic per evaluate launch (order + decode): {traffic['dram_bytes_per_evaluate'] / 1e6:.1f} MB\n")
dst = os.path.join("profiles", f"{tag}_summary.md")
open(dst, "w").write("\n".join(out) + "\n")
print(dst)
