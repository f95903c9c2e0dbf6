"""Traditional static approach (Fig. 7): the CUDA
path on `ffs_static_state` against the oracle's static context, bit-exact --
decode/evaluate on Table 4 and configs A2/B/C (both decode paths), the
overflow fallback, and a GA trajectory."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx
from tests.gpu_util import both_event_ctx, check_gene_order, gpu_state
from tests.test_gpu_evaluate import compare, gpu_eval
from tests.test_gpu_ga import assert_same

pytestmark = pytest.mark.gpu


def test_table4_static_fig7(path):
    d, a = fx.table4_arrays()
    a = dict(a, wt=0)            # objective = C_max: the due dates are not printed
    oa, os_ = np.array(d["orig_assign"]), np.array(d["orig_start"])
    octx = orc.Ctx(fx.workload_instance(a), d["rs"], oa, os_, static=True)
    st = gpu_state(a, d["rs"], oa, os_, static=True)
    check_gene_order(octx, st)
    assert st.K == 6 and (st.cell_states()[: 6 * 3] != 0).all()
    x, y = wlmod.random_chromosomes(4096, st.K, 2, seed=17)
    compare(octx, st, x, y, n_sched=64)
    obj, T, M, _ = gpu_eval(st, x, y)
    assert M.min() == 1991                     # Fig. 7 caption
    assert (obj == M).all()


@pytest.mark.parametrize("cfg,count,nsched", [("A2", 2000, 100), ("B", 1000, 40), ("C", 400, 10)])
def test_static_configs(cfg, count, nsched, path):
    wl = {"A2": wlmod.config_A2, "B": wlmod.config_B, "C": wlmod.config_C}[cfg]()
    octx, st, arr = both_event_ctx(wl, static=True)
    check_gene_order(octx, st)
    assert st.K == (arr["n_prime"]) * wl.g
    x, y = wlmod.random_chromosomes(count, st.K, wl.o, seed=23)
    compare(octx, st, x, y, n_sched=nsched)
    # the merged schedule keeps every original op verbatim (SPEC invariant)
    _, _, _, S = gpu_eval(st, x[:4], y[:4], sched=True)
    n, g = arr["n"], wl.g
    for i in range(4):
        r = octx.decode_genes(x[i], y[i])
        assert (S[i][: n * g] == octx._os).all()
        assert octx.validate(r["assign"], r["start"])[0] == 0


def test_static_general_power(path):
    wl = wlmod.gen_v1("Sq", 24, 5, 3, 6, arrivals_per_event=[8], ratios=[0.4], power="u13", seed=6)
    octx, st, arr = both_event_ctx(wl, static=True)
    x, y = wlmod.random_chromosomes(500, st.K, wl.o, seed=8)
    compare(octx, st, x, y, n_sched=20)


def test_static_overflow_path(path):
    wl = wlmod.config_B()
    octx, st, arr = both_event_ctx(wl, static=True)
    x, y = wlmod.random_chromosomes(300, st.K, wl.o, seed=9)
    ref = gpu_eval(st, x, y, sched=True)
    st.set_horizon_cap(64)
    got = gpu_eval(st, x, y, sched=True)
    for u, v in zip(ref, got):
        assert (u == v).all()
    compare(octx, st, x[:60], y[:60], n_sched=10)
    st.set_horizon_cap(0)


@pytest.mark.parametrize("cfg,w,h,islands,G", [("A2", 4, 4, 4, 21), ("B", 16, 8, 2, 11)])
def test_static_ga_trajectory(cfg, w, h, islands, G, path):
    wl = {"A2": wlmod.config_A2, "B": wlmod.config_B}[cfg]()
    octx, st, arr = both_event_ctx(wl, static=True)
    seed = 4711
    ga = orc.GA(octx, w, h, islands, G, seed, nthreads=8)
    run = ffs.Run(st, w, h, islands, G, seed)
    ga.step()
    assert_same(run, ga, 0)
    for k in range(1, G + 1):
        ga.step()
        run.step(1)
    assert_same(run, ga, G)
    b = run.best()
    tmin, tsum = ga.trace()
    assert (b["trace_min"] == tmin).all() and (b["trace_sum"] == tsum).all()
    assert octx.validate(b["assign"], b["start"])[0] == 0
