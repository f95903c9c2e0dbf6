"""A/B timing helper (not the bench): config C, GA step (256 islands x 256,
CUDA events over N generations) and the evaluate launch alone, printed as one
JSON line.  usage: ab_time.py LABEL [generations] [evaluate launches]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod

label = sys.argv[1] if len(sys.argv) > 1 else "run"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 200
NE = int(sys.argv[3]) if len(sys.argv) > 3 else 100
torch.cuda.set_device(0)
wl = wlmod.config_C()
base = ffs.Instance.from_arrays(wl.original_instance(), device=0)
st0 = ffs.make_state(base, 0)
_, pstart, _, _, pcmax = ffs.decode_schedule(st0, wl.plan_x, wl.plan_y)
rs = wl.rs_from_makespan(wl.ratios[0], pcmax)
inst = ffs.Instance.from_arrays(wl.instance_at(0, [rs]), device=0)
st = ffs.make_state(inst, rs, wl.plan_x.astype(np.int32), pstart[: wl.n * wl.g])
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    run = ffs.Run(st, 16, 16, 256, G + 10, 10741, stream=stream)
    run.step(10)
torch.cuda.synchronize()
# clocks up: ~1.5 s of evaluates before anything is timed
import time
import pynvml
pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
KP0 = (st.K + 15) // 16 * 16
xw, yw = ffs.random_population(st, 65536, 7, stream=stream, row=KP0)
t_end = time.time() + 1.5
while time.time() < t_end:
    ffs.evaluate(st, xw, yw, stream=stream)
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(stream):
    e0.record(stream)
    run.step(G)
    e1.record(stream)
torch.cuda.synchronize()
ga_ms = e0.elapsed_time(e1) / G
K = st.K
KP = (K + 15) // 16 * 16
x, y = ffs.random_population(st, 65536, 10741, stream=stream, row=KP)
obj = torch.empty(65536, dtype=torch.int64, device="cuda")
T = torch.empty(65536, dtype=torch.int64, device="cuda")
M = torch.empty(65536, dtype=torch.int32, device="cuda")
for _ in range(3):
    ffs.evaluate(st, x, y, obj, T, M, stream=stream)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(NE)]
torch.cuda.synchronize()
for a, b in ev:
    a.record(stream)
    ffs.evaluate(st, x, y, obj, T, M, stream=stream)
    b.record(stream)
torch.cuda.synchronize()
t = [a.elapsed_time(b) for a, b in ev]
mhz = pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
print(json.dumps({"label": label, "sm_mhz": mhz, "ga_ms": round(ga_ms, 5), "eval_ms": round(statistics.median(t), 5),
                  "evals_per_s": round(65536 / ga_ms * 1e3 / 1e6, 2), "obj_sum": int(obj.sum().item())}))
