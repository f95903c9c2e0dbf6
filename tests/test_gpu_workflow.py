"""Predictive-reactive workflow (config B: three arrival events) -- the CUDA
path (paper_1903_10741_b200.workflow) against the same workflow driven by the
oracle GA: every event's RS, K, best objective, merged schedule and trace must
be identical."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import workflow
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx

pytestmark = pytest.mark.gpu


def oracle_evolve(ctx, shape, G, seed, nthreads=8):
    w, h, islands = shape
    ga = orc.GA(ctx, w, h, islands, G, seed, nthreads=nthreads)
    for _ in range(G + 1):
        ga.step()
    hx, hy, hobj, hfit = ga.history()
    b = int(np.argmax(hfit))                    # ties -> lowest island (R28)
    r = ctx.decode_genes(hx[b], hy[b])
    tmin, tsum = ga.trace()
    return r, tmin, tsum


def oracle_workflow(wl, shape, G, seed, nthreads=8):
    out = []
    base = wl.original_instance()
    c0 = orc.Ctx(fx.workload_instance(base), 0)
    r, tmin, tsum = oracle_evolve(c0, shape, G, seed, nthreads)
    out.append((0, c0.K, r, tmin, tsum))
    c_plan = r["makespan"]
    rs_list = []
    assign, start = r["assign"], r["start"]
    for e in range(wl.n_events):
        rs = wl.rs_from_makespan(wl.ratios[e], c_plan)
        rs_list.append(rs)
        arr = wl.instance_at(e, rs_list)
        ctx = orc.Ctx(fx.workload_instance(arr), rs, assign, start)
        r, tmin, tsum = oracle_evolve(ctx, shape, G, seed + 1 + e, nthreads)
        assert ctx.validate(r["assign"], r["start"])[0] == 0      # Eqs. (4)-(10), frozen ops kept
        out.append((rs, ctx.K, r, tmin, tsum))
        assign, start = r["assign"], r["start"]
    return out


@pytest.mark.parametrize("shape,G", [((4, 2, 4), 12), ((8, 4, 2), 11)])
def test_config_b_workflow_parity(shape, G):
    wl = wlmod.config_B()
    ref = oracle_workflow(wl, shape, G, 10741)
    got = workflow.run_events(wl, shape=shape, generations=G, seed=10741)
    evs = [got.plan] + got.events
    assert len(evs) == len(ref) == 4
    for ev, (rs, K, r, tmin, tsum) in zip(evs, ref):
        assert ev.rs == rs and ev.K == K
        assert ev.objective == r["objective"] and ev.makespan == r["makespan"]
        assert ev.sum_tardiness == r["sum_tardiness"]
        assert (ev.start == r["start"]).all() and (ev.assign == r["assign"]).all()
        assert (ev.trace_min == tmin).all() and (ev.trace_sum == tsum).all()


def oracle_compare(ratios, seeds, shape, G):
    """The Table 10 comparison driven by the oracle GA."""
    from paper_1903_10741_b200.workflow import test3_workload
    out = {}
    for ratio in ratios:
        for seed in seeds:
            wl = test3_workload(ratio, seed)
            c0 = orc.Ctx(fx.workload_instance(wl.original_instance()), 0)
            plan, _, _ = oracle_evolve(c0, shape, G, seed)
            rs = wl.rs_from_makespan(ratio, plan["makespan"])
            arr = wl.instance_at(0, [rs])
            n_g = wl.n * wl.g
            for name, static in (("dynamic", False), ("static", True)):
                ctx = orc.Ctx(fx.workload_instance(arr), rs, plan["assign"][:n_g], plan["start"][:n_g],
                              static=static)
                r, tmin, _ = oracle_evolve(ctx, shape, G, seed + 1)
                assert ctx.validate(r["assign"], r["start"])[0] == 0
                out[(ratio, seed, name)] = (rs, ctx.K, r, tmin)
    return out


def test_policy_comparison_parity():
    """Dynamic vs static (Table 10 design): every run's RS, K, best objective,
    schedule and trace equal the oracle-driven comparison."""
    ratios, seeds, shape, G = (0.2, 0.6), (1903, 7), (4, 4, 4), 11
    ref = oracle_compare(ratios, seeds, shape, G)
    rows = workflow.compare_policies(ratios=ratios, seeds=seeds, shape=shape, generations=G)
    assert [r.ratio for r in rows] == list(ratios)
    for row in rows:
        assert row.n_prime == round(row.ratio * 10)
        for run in row.runs:
            for name in ("dynamic", "static"):
                rs, K, r, tmin = ref[(row.ratio, run["seed"], name)]
                ev = run[name + "_result"]
                assert run["rs"] == rs and ev.K == K
                assert ev.objective == r["objective"] and ev.makespan == r["makespan"]
                assert (ev.start == r["start"]).all() and (ev.assign == r["assign"]).all()
                assert (ev.trace_min == tmin).all()
            assert run["K_static"] == row.n_prime * 3
