import sys, os, time, statistics
sys.path.insert(0, os.getcwd())
import torch
from paper_1903_10741_b200 import ffs
from scripts.prof_eval import config_c_state
wl, st = config_c_state()
for rep in range(6):
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        run = ffs.Run(st, 16, 16, 256, 105, 10741, stream=stream)
        for _ in range(5): run.step(1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream); run.step(100); t1 = time.perf_counter(); e1.record(stream)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"rep {rep}: {e0.elapsed_time(e1)/100:.4f} ms/gen  host launch {1e3*(t1-t0):.2f} ms  wall {1e3*(t2-t0):.2f} ms", flush=True)
    del run
