"""Host launch cost vs device time per GA generation (why the GA loop is not a
CUDA graph): config C (256 islands x 256) and config B's shape (64 islands x
128, first event).  Prints host microseconds to enqueue G generations
(run.step returns once they are queued) and the device time of the same
generations (CUDA events)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod


def state_of(wl):
    base = ffs.Instance.from_arrays(wl.original_instance(), device=0)
    st0 = ffs.make_state(base, 0)
    _, pstart, _, _, pcmax = ffs.decode_schedule(st0, wl.plan_x, wl.plan_y)
    rs = wl.rs_from_makespan(wl.ratios[0], pcmax)
    inst = ffs.Instance.from_arrays(wl.instance_at(0, [rs]), device=0)
    st = ffs.make_state(inst, rs, wl.plan_x.astype(np.int32), pstart[: wl.n * wl.g])
    st._keep = (base, st0, inst)
    return st


out = {}
for name, wl, shape in [("C", wlmod.config_C(), (16, 16, 256)), ("B", wlmod.config_B(), (16, 8, 64))]:
    st = state_of(wl)
    G = int(os.environ.get("GENS", "50"))
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        run = ffs.Run(st, shape[0], shape[1], shape[2], G + 20, 10741, stream=stream)
        run.step(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        h0 = time.perf_counter()
        run.step(G)
        h1 = time.perf_counter()
        e1.record(stream)
    torch.cuda.synchronize()
    out[name] = {"host_us_per_gen": round((h1 - h0) / G * 1e6, 2), "device_us_per_gen": round(e0.elapsed_time(e1) / G * 1e3, 2),
                 "launches_per_gen": run.info()["launches"] / (G + 20)}
print(json.dumps(out))
