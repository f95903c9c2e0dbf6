"""The C-ABI's contracts (include/ffs.h) beyond the parity of its
results: the one-shot ffs_evolve, the K = 0 case, calls on several
streams, argument checks that keep the kernels safe, and the shard hooks."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx
from tests.gpu_util import both_event_ctx, gpu_state

pytestmark = pytest.mark.gpu


def test_evolve_one_shot_equals_stepwise():
    """ffs_evolve (one call, all generations) == ffs_evolve_begin + ffs_evolve_step
    + ffs_best, and both equal the oracle GA's trace and best."""
    wl = wlmod.config_A2()
    octx, st, _ = both_event_ctx(wl)
    G, seed = 23, 555
    a = ffs.Run(st, 4, 4, 4, G, seed)
    a.step(G)
    b = ffs.evolve(st, 4, 4, 4, G, seed)
    assert b.info()["generation"] == G
    for u, v in zip(a.population(), b.population()):
        assert (u == v).all()
    for u, v in zip(a.history(), b.history()):
        assert (u == v).all()
    ba, bb = a.best(), b.best()
    for k in ("x", "y", "assign", "start", "trace_min", "trace_sum"):
        assert (ba[k] == bb[k]).all(), k
    for k in ("objective", "sum_tardiness", "makespan"):
        assert ba[k] == bb[k], k
    ga = orc.GA(octx, 4, 4, 4, G, seed)
    for _ in range(G + 1):
        ga.step()
    tmin, tsum = ga.trace()
    assert (bb["trace_min"] == tmin).all() and (bb["trace_sum"] == tsum).all()
    r = octx.decode_genes(bb["x"], bb["y"])
    assert bb["objective"] == r["objective"] and (bb["start"] == r["start"]).all()


def _k0_state():
    """An instance frozen after its plan completed: every op COMPLETED, K = 0."""
    from tests.test_gpu_evaluate import edge_instance
    a, plan, rs = edge_instance("rs_end", 12345)
    octx = orc.Ctx(fx.workload_instance(a), rs, plan["assign"], plan["start"])
    st = gpu_state(a, rs, plan["assign"], plan["start"])
    assert octx.K == 0 and st.K == 0
    return octx, st, plan


@pytest.mark.parametrize("one_shot", [True, False])
def test_evolve_K0_returns_frozen_plan(one_shot):
    """with nothing pending the GA has nothing to evolve; the best is the
    frozen plan itself and the trace is empty."""
    octx, st, plan = _k0_state()
    run = ffs.Run(st, 2, 1, 1, 5, 7, one_shot=one_shot)
    if not one_shot:
        run.step(5)
    b = run.best()
    r = octx.decode(-np.ones(octx.cells, np.int32), -np.ones(octx.cells, np.int32))
    assert (b["start"] == plan["start"]).all() and (b["start"] == r["start"]).all()
    assert (b["assign"] == plan["assign"]).all()
    assert b["objective"] == r["objective"] and b["makespan"] == r["makespan"]
    assert b["sum_tardiness"] == r["sum_tardiness"]
    assert b["trace_min"].size == 0 and b["trace_sum"].size == 0
    assert b["x"].size == 0 and b["y"].size == 0


def test_calls_on_several_streams_share_the_state_safely():
    """Every device-pointer call on a state shares its scratch (overflow lists,
    the order->decode buffer): calls issued on different streams back to back,
    and a host-buffer call after a device call on another stream, give the
    single-stream results (the scratch is ordered across streams)."""
    wl = wlmod.config_C()
    octx, st, _ = both_event_ctx(wl)
    n = 20000
    xa, ya = ffs.random_population(st, n, 1)
    xb, yb = ffs.random_population(st, n, 2)
    ref_a = [t.clone() for t in ffs.evaluate(st, xa, ya)[:3]]
    ref_b = [t.clone() for t in ffs.evaluate(st, xb, yb)[:3]]
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        ga = ffs.evaluate(st, xa, ya, stream=s1)[:3]
        gb = ffs.evaluate(st, xb, yb, stream=s2)[:3]
        hb = ffs.evaluate_host(st, xb.cpu().numpy(), yb.cpu().numpy(), stream=s1)
        torch.cuda.synchronize()
        for u, v in zip(ga, ref_a):
            assert bool((u == v).all())
        for u, v in zip(gb, ref_b):
            assert bool((u == v).all())
        for u, v in zip(hb, ref_b):
            assert (u == v.cpu().numpy()).all()
    idx = np.arange(0, n, 997)
    oo, _, _, _ = octx.evaluate_batch(xa.cpu().numpy()[idx], ya.cpu().numpy()[idx], nthreads=8)
    assert (ref_a[0].cpu().numpy()[idx] == oo).all()


def test_objective_word_overflow_is_rejected():
    """WT large enough that WT * sum T + C_max could leave the 64-bit objective
    word (or make the E_max search run away) is refused at state creation and
    by ffs_state_set_objective_weight, which then leaves the state unchanged."""
    wl = wlmod.config_C()
    octx, st, arr = both_event_ctx(wl)
    big = dict(arr)
    big["wt"] = 10 ** 15
    with pytest.raises(ffs.FFSError) as ei:
        gpu_state(big, st.rs, *[np.asarray(v) for v in _plan(wl)])
    assert ei.value.status == 1
    with pytest.raises(ffs.FFSError):
        st.set_objective_weight(1e299)
    x, y = ffs.random_population(st, 64, 3)
    obj = ffs.evaluate(st, x, y)[0]
    oo, _, _, _ = octx.evaluate_batch(x.cpu().numpy(), y.cpu().numpy())
    assert (obj.cpu().numpy() == oo).all()          # still the integer WT = 100 objective


def _plan(wl):
    octx, arr, plan, rs = fx.oracle_event_ctx(wl)
    return plan["assign"][: wl.n * wl.g], plan["start"][: wl.n * wl.g]


@pytest.mark.parametrize("which", ["none", "allgather_only", "allreduce_only"])
def test_sharded_run_needs_both_hooks(which):
    """world > 1 without both collective hooks is refused (a missing
    allreduce would silently calibrate E_max per shard)."""
    wl = wlmod.config_A2()
    _, st, _ = both_event_ctx(wl)
    ar = ffs.ALLRED(lambda u, p, s: 0) if which == "allreduce_only" else ffs.ALLRED()
    ag = ffs.ALLGATHER(lambda u, a, b, n, s: 0) if which == "allgather_only" else ffs.ALLGATHER()
    cfg = ffs.GAConfig(4, 2, 4, 0, 2, ffs.XO_090, ffs.MUT_010, 10, 5, 1, 0, 2, ar, ag, None)
    h = C.c_void_p()
    rc = ffs.lib().ffs_evolve_begin(st.h, C.byref(cfg), C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                    C.byref(h))
    assert rc == 1 and not h.value
    assert b"hooks" in ffs.lib().ffs_last_error()


def test_checkpoint_restore_K0():
    """A K = 0 run (nothing pending) checkpoints and restores its
    (empty) state; another generation is refused; its best stays the frozen
    plan."""
    octx, st, plan = _k0_state()
    run = ffs.Run(st, 2, 1, 1, 5, 7)
    run.step(5)
    ck = run.checkpoint()
    other = ffs.Run(st, 2, 1, 1, 5, 7)
    other.restore(ck)
    bad = dict(ck, generation=3)
    with pytest.raises(ffs.FFSError):
        other.restore(bad)
    assert (other.best()["start"] == plan["start"]).all()
