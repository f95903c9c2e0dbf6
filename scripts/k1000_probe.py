"""Diagnostic: config C's shape with all 100 jobs at RS = 0 (K = 1,000, every op pending):
state info and evaluate throughput on 65,536 padded-row chromosomes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod

wl = wlmod.gen_v1("Cs", 100, 10, 4, 10, seed=1903)
inst = ffs.Instance.from_arrays(wl.original_instance(), device=0)
st = ffs.make_state(inst, 0)
print(st.info())
KP = (st.K + 15) // 16 * 16
x, y = ffs.random_population(st, 65536, 1, row=KP)
ob = torch.empty(65536, dtype=torch.int64, device="cuda")
M = torch.empty(65536, dtype=torch.int32, device="cuda")
T = torch.empty(65536, dtype=torch.int64, device="cuda")
for _ in range(2):
    ffs.evaluate(st, x, y, ob, T, M)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    ffs.evaluate(st, x, y, ob, T, M)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print("K", st.K, "ms", round(dt * 1e3, 3), "M evals/s", round(65536 / dt / 1e6, 1))
print("makespan min/mean/max", int(M.min()), float(M.float().mean()), int(M.max()),
      "over cap", int((M > st.info()["horizon_cap"]).sum()))
