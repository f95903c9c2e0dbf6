import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1903_10741_b200 import ffs
from scripts.prof_eval import config_c_state
wl, st = config_c_state()
K = st.K; KP = (K + 15) // 16 * 16
for total in [int(a) for a in sys.argv[1:]]:
    xs, ys = ffs.random_population(st, total, 10741, row=KP)
    torch.cuda.synchronize()
    print("gen ok", total, flush=True)
    ob = torch.empty(total, dtype=torch.int64, device="cuda")
    ffs.evaluate(st, xs, ys, ob)
    torch.cuda.synchronize()
    print("eval ok", total, ob[:3].tolist(), flush=True)
