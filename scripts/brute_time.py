"""Time the GPU brute-force enumerator on gen-v1 instances at RS = 0."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod

for n, g, o, q in [(5, 2, 2, 2), (4, 3, 2, 3)]:
    wl = wlmod.gen_v1("bf", n, g, o, q, seed=12)
    inst = ffs.Instance.from_arrays(wl.original_instance())
    st = ffs.make_state(inst, 0)
    ffs.brute_force(st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    best, ev, bx, by = ffs.brute_force(st)
    dt = time.perf_counter() - t0
    print(f"n={n} g={g} o={o} K={st.K}: {ev} decodes in {dt:.3f}s = {ev / dt / 1e6:.1f} M/s, best {best}", flush=True)
