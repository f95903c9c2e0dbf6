"""Fractional WT (Table 11): the CUDA path's binary64 objective
words against the oracle's or_objective_value, bit for bit; GA trajectories with
a fractional weight (x, y, objective, fitness, E_max, history and the trace
identical bit for bit -- the binary64 trace sum follows reading R33's order
on both sides); the Table 11 sweep driver against the oracle-driven sweep."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workflow
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx
from tests.gpu_util import both_event_ctx
from tests.test_gpu_ga import assert_same

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TABLE11_WT = workflow.TABLE11_WT


@pytest.mark.parametrize("cfg", ["A2", "B", "C"])
def test_real_objective_words(cfg, path):
    wl = {"A2": wlmod.config_A2, "B": wlmod.config_B, "C": wlmod.config_C}[cfg]()
    octx, st, arr = both_event_ctx(wl)
    count = {"A2": 1000, "B": 400, "C": 120}[cfg]
    x, y = wlmod.random_chromosomes(count, st.K, wl.o, seed=31)
    xd, yd = torch.as_tensor(x).to(DEV), torch.as_tensor(y).to(DEV)
    o_int, T, M, _ = ffs.evaluate(st, xd, yd)
    o_int = o_int.cpu().numpy().copy()
    for wt in TABLE11_WT + (0.0, 0.37, float(wl.wt)):
        st.set_objective_weight(wt)
        octx.set_real_weight(wt)
        obj, T2, M2, _ = ffs.evaluate(st, xd, yd)
        torch.cuda.synchronize()
        assert obj.dtype == torch.float64
        ov, oT, oM, _ = octx.evaluate_batch(x, y, nthreads=8)
        got = obj.cpu().numpy()
        assert (got.view(np.int64) == ov.view(np.int64)).all(), wt        # bit-identical binary64
        assert (T2.cpu().numpy() == oT).all() and (M2.cpu().numpy() == oM).all()
        if wt == float(wl.wt):
            assert (got == o_int.astype(np.float64)).all()
    oh, _, _ = ffs.evaluate_host(st, x, y)
    assert (oh.view(np.int64) == ov.view(np.int64)).all()


@pytest.mark.parametrize("cfg,w,h,islands,G,wt", [("A2", 4, 4, 4, 21, 0.37), ("B", 16, 8, 2, 11, 0.01),
                                                  ("B", 16, 8, 2, 11, 4.0), ("C", 16, 16, 4, 3, 0.37)])
def test_real_ga_trajectory(cfg, w, h, islands, G, wt, path):
    wl = {"A2": wlmod.config_A2, "B": wlmod.config_B, "C": wlmod.config_C}[cfg]()
    octx, st, arr = both_event_ctx(wl)
    st.set_objective_weight(wt)
    octx.set_real_weight(wt)
    seed = 2024
    ga = orc.GA(octx, w, h, islands, G, seed, nthreads=8)
    run = ffs.Run(st, w, h, islands, G, seed)
    ga.step()
    assert run.info()["emax"] == ga.emax
    for k in range(1, G + 1):
        ga.step()
        run.step(1)
        if k in (1, G // 2, G):
            gx, gy, gobj, gfit = run.population()
            ox, oy, oobj, ofit = ga.population()
            assert (gx == ox).all() and (gy == oy).all(), k
            assert (gobj.view(np.int64) == oobj.view(np.int64)).all(), k
            assert (gfit.view(np.int64) == ofit.view(np.int64)).all(), k
            hx, hy, hobj, hfit = run.history()
            px, py, pobj, pfit = ga.history()
            assert (hx == px).all() and (hobj == pobj).all() and (hfit == pfit).all(), k
    b = run.best()
    tmin, tsum = ga.trace()
    assert (b["trace_min"] == tmin).all()
    assert (np.asarray(b["trace_sum"]).view(np.int64) == np.asarray(tsum).view(np.int64)).all()
    r = octx.decode_genes(b["x"], b["y"])
    assert b["objective"] == r["value"]


def oracle_wt_sweep(wts, seeds, ratio, shape, G):
    out = {}
    for seed in seeds:
        wl = workflow.test3_workload(ratio, seed)
        c0 = orc.Ctx(fx.workload_instance(wl.original_instance()), 0)
        ga = orc.GA(c0, shape[0], shape[1], shape[2], G, seed, nthreads=8)
        for _ in range(G + 1):
            ga.step()
        hx, hy, hobj, hfit = ga.history()
        plan = c0.decode_genes(hx[int(np.argmax(hfit))], hy[int(np.argmax(hfit))])
        rs = wl.rs_from_makespan(ratio, plan["makespan"])
        arr = wl.instance_at(0, [rs])
        n_g = wl.n * wl.g
        for wt in wts:
            ctx = orc.Ctx(fx.workload_instance(arr), rs, plan["assign"][:n_g], plan["start"][:n_g])
            ctx.set_real_weight(wt)
            g2 = orc.GA(ctx, shape[0], shape[1], shape[2], G, seed + 1, nthreads=8)
            for _ in range(G + 1):
                g2.step()
            hx, hy, hobj, hfit = g2.history()
            b = int(np.argmax(hfit))
            r = ctx.decode_genes(hx[b], hy[b])
            out[(wt, seed)] = (rs, r["value"], r["sum_tardiness"], r["makespan"])
    return out


def test_wt_sweep_parity():
    wts, seeds, shape, G = (0.01, 0.7, 100.0), (1903, 11), (4, 4, 4), 11
    ref = oracle_wt_sweep(wts, seeds, 0.5, shape, G)
    rows = workflow.wt_sweep(wts=wts, seeds=seeds, ratio=0.5, shape=shape, generations=G)
    for row in rows:
        for run in row.runs:
            rs, v, T, M = ref[(row.wt, run["seed"])]
            assert run["rs"] == rs
            assert run["objective"] == v and run["sum_tardiness"] == T and run["makespan"] == M
