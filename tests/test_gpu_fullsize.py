"""Parity at the BASELINE configurations as the bench runs them (VERDICT r1
"Next" item 2): element by element against the oracle, no sampling.

(a) config C's GA at the bench's launch configuration: 256 islands x 256
    (16x16 tiles, 65,536 cells: the breeding kernel's grid-stride path, a
    4-wave grid, replacement and trace over 256 islands) on a side stream,
    with migration every 2 generations so the ring runs inside the window;
    population, objectives, fitness, history elites and trace are compared
    with the oracle GA after every generation;
(b) every one of the 65,536 evaluations of a config-C population in the
    GA's padded-row layout: objective, sum T and C_max from the bench's
    launch, and the full schedule (start time of every operation) of every
    chromosome from the schedule-emitting launch;
(c) config B in full: plan + 3 arrival events x 100 generations at 64
    islands x 128 (16x8), every event's RS, K, best, merged schedule and
    trace.
The oracle runs on every host core (it is the slow side: ~1-2 min per test).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod
from tests.gpu_util import both_event_ctx, check_gene_order

pytestmark = pytest.mark.gpu
CORES = len(os.sched_getaffinity(0))
SEED = 10741


def _assert_same(run, ga, k):
    gx, gy, gobj, gfit = run.population()
    ox, oy, oobj, ofit = ga.population()
    bad = np.flatnonzero(gobj != oobj)
    assert bad.size == 0, f"gen {k}: objective mismatch at {bad[:8]}"
    assert (gfit == ofit).all(), f"gen {k}: fitness"
    assert (gx == ox).all(), f"gen {k}: X"
    assert (gy == oy).all(), f"gen {k}: Y"
    hx, hy, hobj, hfit = run.history()
    px, py, pobj, pfit = ga.history()
    assert (hobj == pobj).all() and (hfit == pfit).all(), f"gen {k}: history values"
    assert (hx == px).all() and (hy == py).all(), f"gen {k}: history chromosomes"


def test_config_c_ga_at_bench_launch():
    wl = wlmod.config_C()
    octx, st, _ = both_event_ctx(wl)
    check_gene_order(octx, st)
    w, h, islands, G = 16, 16, 256, 4
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        run = ffs.Run(st, w, h, islands, G, SEED, migration_interval=2, stream=stream)
    ga = orc.GA(octx, w, h, islands, G, SEED, migration_interval=2, nthreads=CORES)
    ga.step()
    torch.cuda.synchronize()
    assert run.info()["emax"] == ga.emax
    _assert_same(run, ga, 0)
    for k in range(1, G + 1):
        with torch.cuda.stream(stream):
            run.step(1)
        ga.step()
        torch.cuda.synchronize()
        _assert_same(run, ga, k)
    b = run.best()
    tmin, tsum = ga.trace()
    assert (b["trace_min"] == tmin).all() and (b["trace_sum"] == tsum).all()
    _, _, pobj, pfit = ga.history()
    assert b["objective"] == pobj[int(np.argmax(pfit))]
    assert octx.validate(b["assign"], b["start"])[0] == 0


def test_config_c_every_evaluation_and_schedule():
    wl = wlmod.config_C()
    octx, st, _ = both_event_ctx(wl)
    K = st.K
    KP = (K + 15) // 16 * 16
    n = 65536
    stream = torch.cuda.Stream()
    x, y = ffs.random_population(st, n, SEED, stream=stream, row=KP)       # the GA's row layout
    obj, T, M, _ = ffs.evaluate(st, x, y, stream=stream)                    # the bench's launch
    _, _, _, S = ffs.evaluate(st, x, y, with_schedule=True, stream=stream)  # schedule-emitting launch
    torch.cuda.synchronize()
    xs = x[:, :K].cpu().numpy()
    ys = y[:, :K].cpu().numpy()
    oo, oT, oM, oS = octx.evaluate_batch_schedule(xs, ys, nthreads=CORES)
    obj, T, M, S = obj.cpu().numpy(), T.cpu().numpy(), M.cpu().numpy(), S.cpu().numpy()
    assert (obj == oo).all(), np.flatnonzero(obj != oo)[:10]
    assert (T == oT).all() and (M == oM).all()
    bad = np.flatnonzero((S != oS).any(axis=1))
    assert bad.size == 0, f"{bad.size} schedules differ, first {bad[:8]}"


def test_config_b_in_full():
    from tests.test_gpu_workflow import oracle_workflow
    from paper_1903_10741_b200 import workflow
    wl = wlmod.config_B()
    shape, G = (16, 8, 64), 100
    ref = oracle_workflow(wl, shape, G, SEED, nthreads=CORES)
    got = workflow.run_events(wl, shape=shape, generations=G, seed=SEED)
    evs = [got.plan] + got.events
    assert len(evs) == len(ref) == 4
    for ev, (rs, K, r, tmin, tsum) in zip(evs, ref):
        assert ev.rs == rs and ev.K == K
        assert ev.objective == r["objective"] and ev.makespan == r["makespan"]
        assert ev.sum_tardiness == r["sum_tardiness"]
        assert (ev.start == r["start"]).all() and (ev.assign == r["assign"]).all()
        assert (ev.trace_min == tmin).all() and (ev.trace_sum == tsum).all()
