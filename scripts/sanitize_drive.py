"""Small driver that launches every kernel of the library once or twice, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_drive.py

Covers: state staging, the lane path (order kernel with and without x
staging, both row layouts; decode modes 0/1/2; the LIST re-decode), the warp
path and the overflow fallback, random_population, the island GA (generation, replace,
migration, trace; config A and the config C shape; the binary64 trace), calls on
two streams, the brute force.  Checks nothing itself -- the tool does."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod


def state_of(arr, rs=0):
    inst = ffs.Instance.from_arrays(arr, device=0)
    st = ffs.make_state(inst, rs)
    st._keep = inst
    return st


def evals(st, n, pad):
    x, y = ffs.random_population(st, n, 7, row=(st.K + 15) // 16 * 16 if pad else 0)
    ffs.evaluate(st, x, y, with_schedule=True)


def main():
    torch.cuda.set_device(0)
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("all", "eval"):
        # mode 2 (Q = 1), K = 855-ish config C at 2 tiles of chromosomes, both row layouts
        wl = wlmod.config_C()
        st = state_of(wl.original_instance())
        for pad in (False, True):
            evals(st, 70, pad)
        # the unstaged order kernel (long rows)
        os.environ["FFS_ORDER_NO_XS"] = "1"
        st2 = state_of(wl.original_instance())
        del os.environ["FFS_ORDER_NO_XS"]
        for pad in (False, True):
            evals(st2, 40, pad)
        # mode 1 / mode 0 and the warp path with a tiny horizon (overflow fallback)
        wb = wlmod.config_B()
        arr = wb.original_instance()
        evals(state_of(arr), 100, False)
        arr1 = dict(arr, Q=np.full_like(arr["Q"], 1), q_max=40)
        evals(state_of(arr1), 100, False)
        os.environ["FFS_DISABLE_LANE"] = "1"
        st3 = state_of(arr)
        del os.environ["FFS_DISABLE_LANE"]
        st3.set_horizon_cap(64)
        evals(st3, 100, False)
        # lane path with a tiny horizon: first call -> general fallback (smem
        # profile), second -> LIST re-decode (the state has seen an overflow)
        st4 = state_of(arr)
        st4.set_horizon_cap(64)
        evals(st4, 100, False)
        evals(st4, 100, False)
        xh, yh = wlmod.random_chromosomes(300, st.K, wl.o, seed=5)
        ffs.evaluate_host(st, xh, yh)
    if which in ("all", "ga"):
        wa = wlmod.config_A2()
        st = state_of(wa.original_instance())
        run = ffs.Run(st, 4, 4, 4, 12, 10741)
        run.step(12)
        run.best()
        # config C shape (K = 1,000 at RS = 0): multi-word breeding loops, both
        # sides of the cut, migration every 2, the one-pass replacement + trace
        wc = wlmod.config_C()
        stc = state_of(wc.original_instance())
        runc = ffs.Run(stc, 16, 16, 2, 3, 10741, migration_interval=2)
        runc.step(3)
        runc.best()
        # binary64 objective (f3): the R33 sequential trace sums
        str_ = state_of(wa.original_instance())
        str_.set_objective_weight(0.37)
        runr = ffs.Run(str_, 4, 4, 4, 5, 7)
        runr.step(5)
        runr.best()
        # device calls on two streams sharing the state's scratch
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        x1, y1 = ffs.random_population(stc, 64, 1)
        torch.cuda.synchronize()   # the rows come from the default stream
        ffs.evaluate(stc, x1, y1, stream=s1)
        ffs.evaluate(stc, x1, y1, stream=s2)
    if which in ("all", "brute"):
        rng = np.random.default_rng(1)
        n, g, o = 3, 2, 2
        P = rng.integers(1, 4, size=(n, g, o)).astype(np.int32)
        Q = rng.integers(1, 3, size=(n, g, o)).astype(np.int32)
        R = np.zeros(n, np.int32)
        a = dict(n=n, n_prime=0, g=g, o=o, P=P, Q=Q, R=R, D=R + 4, q_max=3, wt=10)
        ffs.brute_force(state_of(a))
    torch.cuda.synchronize()
    print("sanitize driver done", which)


if __name__ == "__main__":
    main()
