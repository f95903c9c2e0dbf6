"""Whole-trajectory parity of the CUDA island GA with the oracle GA (same
Philox stream spec): population, objectives, fitness, history elites and
trace must be identical generation by generation."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod
from tests.gpu_util import both_event_ctx

pytestmark = pytest.mark.gpu


def assert_same(gpu_run, ga, k):
    gx, gy, gobj, gfit = gpu_run.population()
    ox, oy, oobj, ofit = ga.population()
    assert (gobj == oobj).all(), f"gen {k}: objective mismatch at {np.flatnonzero(gobj != oobj)[:8]}"
    assert (gfit == ofit).all(), f"gen {k}: fitness"
    assert (gx == ox).all(), f"gen {k}: X"
    assert (gy == oy).all(), f"gen {k}: Y"
    hx, hy, hobj, hfit = gpu_run.history()
    px, py, pobj, pfit = ga.history()
    assert (hobj == pobj).all() and (hfit == pfit).all() and (hx == px).all() and (hy == py).all(), k


@pytest.mark.parametrize("cfg,w,h,islands,G,every", [
    ("A2", 8, 8, 1, 50, 1),          # config A: one 8x8 island, 50 generations
    ("A2", 4, 4, 4, 30, 1),          # config A variant with ring migration
    ("B", 16, 8, 4, 12, 3),          # config B shape, 4 islands
    ("C", 16, 16, 2, 3, 1),          # config C shape, 2 islands, a few generations
])
def test_trajectory_parity(cfg, w, h, islands, G, every, path):
    wl = {"A2": wlmod.config_A2, "B": wlmod.config_B, "C": wlmod.config_C}[cfg]()
    octx, st, arr = both_event_ctx(wl)
    seed = 10741
    ga = orc.GA(octx, w, h, islands, G, seed, nthreads=8)
    run = ffs.Run(st, w, h, islands, G, seed)
    ga.step()
    assert run.info()["emax"] == ga.emax
    assert_same(run, ga, 0)
    for k in range(1, G + 1):
        ga.step()
        run.step(1)
        if k % every == 0 or k == G:
            assert_same(run, ga, k)
    b = run.best()
    tmin, tsum = ga.trace()
    assert (b["trace_min"] == tmin).all() and (b["trace_sum"] == tsum).all()
    assert (np.diff(b["trace_min"]) <= 0).all()
    # the best is the oracle's best history elite, decoded to a valid schedule
    _, _, pobj, pfit = ga.history()
    i = int(np.argmax(pfit))
    assert b["objective"] == pobj[i]
    nv, kinds = octx.validate(b["assign"], b["start"])
    assert nv == 0, kinds


def test_two_shard_run_equals_single_gpu_run():
    """Two shards of the product run (islands [0,2) and [2,4) of 4) driven by
    two host threads whose collective hooks exchange device buffers through a
    barrier: E_max allreduce + boundary-elite allgather every 10 generations
    must reproduce the single-run trajectory exactly (the ring crosses the
    shard boundary twice)."""
    import threading
    from paper_1903_10741_b200 import dist as fdist
    wl = wlmod.config_A2()
    octx, st, arr = both_event_ctx(wl)
    G, world = 21, 2
    full = ffs.Run(st, 4, 2, 4, G, 99)
    full.step(G)
    ref = full.population()
    ref_best = full.best()
    bar = threading.Barrier(world)
    slots = [None] * world

    def hooks(rank):
        def allreduce(user, ptr, stream):
            torch.cuda.synchronize()
            t = fdist._dev_view(ptr, 1, "<i8")
            slots[rank] = t.clone()
            bar.wait()
            m = torch.max(torch.stack([s_ for s_ in slots]))
            bar.wait()
            t.copy_(m.reshape(1))
            torch.cuda.synchronize()
            return 0

        def allgather(user, send, recv, nbytes, stream):
            torch.cuda.synchronize()
            slots[rank] = fdist._dev_view(send, nbytes, "|u1").clone()
            bar.wait()
            r = fdist._dev_view(recv, nbytes * world, "|u1")
            for k in range(world):
                r[k * nbytes:(k + 1) * nbytes].copy_(slots[k])
            torch.cuda.synchronize()
            bar.wait()
            return 0
        return allreduce, allgather

    out = [None] * world
    errs = []

    def drive(rank):
        try:
            b, e = fdist.shard(4, rank, world)
            s = torch.cuda.Stream()
            run = ffs.Run(st, 4, 2, 4, G, 99, island_begin=b, island_end=e, rank=rank, world=world,
                          hooks=hooks(rank), stream=s)
            run.step(G)
            out[rank] = (run.population(), run.best())
        except Exception as ex:  # pragma: no cover
            errs.append(ex)
            bar.abort()

    th = [threading.Thread(target=drive, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(4):
        assert (np.concatenate([out[0][0][k], out[1][0][k]]) == ref[k]).all(), k
    tmin = np.minimum(out[0][1]["trace_min"], out[1][1]["trace_min"])
    assert (tmin == ref_best["trace_min"]).all()
    assert (out[0][1]["trace_sum"] + out[1][1]["trace_sum"] == ref_best["trace_sum"]).all()


def test_trajectory_parity_long_jobs():
    """GA trajectory with G = 16 (3-step min-scan in the order kernel) and a
    row length that is not a multiple of the crossover's 8-gene words."""
    from paper_1903_10741_b200 import workload as wlmod
    wl = wlmod.gen_v1("G16ga", 9, 16, 3, 5, arrivals_per_event=[2], ratios=[0.3], seed=16)
    octx, st, _ = both_event_ctx(wl)
    G = 12
    run = ffs.Run(st, 4, 4, 4, G, 4242)
    run.step(G)
    ga = orc.GA(octx, 4, 4, 4, G, 4242)
    for _ in range(G + 1):
        ga.step()
    for u, v in zip(run.population(), ga.population()):
        assert (u == v).all()


@pytest.mark.parametrize("relist", ["on", "off"])
def test_trajectory_parity_through_overflows(relist, monkeypatch):
    """A tiny horizon makes many children overflow every generation: the GA's
    evaluations go through the overflow routes (the lane re-decode once the
    state has seen an overflow, then the general fallback; or the fallback
    alone) and the trajectory still equals the oracle's."""
    monkeypatch.delenv("FFS_RELIST_CAP", raising=False)
    if relist == "off":
        monkeypatch.setenv("FFS_RELIST_CAP", "0")
    wl = wlmod.config_B()
    octx, st, _ = both_event_ctx(wl)
    st.set_horizon_cap(64)
    G = 10
    run = ffs.Run(st, 16, 8, 4, G, 777)
    run.step(G)
    ga = orc.GA(octx, 16, 8, 4, G, 777, nthreads=8)
    for _ in range(G + 1):
        ga.step()
    for u, v in zip(run.population(), ga.population()):
        assert (u == v).all()
    tmin, tsum = ga.trace()
    b = run.best()
    assert (b["trace_min"] == tmin).all() and (b["trace_sum"] == tsum).all()


@pytest.mark.parametrize("k,wt", [(0, None), (7, None), (10, None), (12, None), (9, 0.37)])
def test_checkpoint_resume_is_bit_identical(k, wt, tmp_path):
    """Run.checkpoint() after generation k -> an .npz file -> a fresh run of the
    same configuration restores it (ffs_run_restore) and finishes: population,
    objective / fitness words, history elites, E_max, the best schedule and the
    whole trace equal the uninterrupted run's (k = 7 and 9 resume before the
    generation-10 migration, k = 10 right after it, k = 0 from the initial
    population; wt: fractional WT, binary64 words)."""
    wl = wlmod.config_A2()
    _, st, _ = both_event_ctx(wl)
    if wt is not None:
        st.set_objective_weight(wt)
    G, shape = 23, (4, 4, 4)
    full = ffs.Run(st, *shape, G, 10741)
    full.step(G)
    a = ffs.Run(st, *shape, G, 10741)
    a.step(k)
    ck = a.checkpoint()
    del a
    np.savez(tmp_path / "ck.npz", **ck)
    ck2 = dict(np.load(tmp_path / "ck.npz"))
    b = ffs.Run(st, *shape, G, 10741)
    b.restore(ck2)
    assert b.info()["generation"] == k
    b.step(G - k)
    for u, v in zip(full.population(), b.population()):   # 64-bit words compared as bit patterns
        u, v = np.asarray(u), np.asarray(v)
        if u.dtype.itemsize == 8:
            u, v = u.view(np.int64), v.view(np.int64)
        assert (u == v).all()
    for u, v in zip(full.history(), b.history()):
        u, v = np.asarray(u), np.asarray(v)
        if u.dtype.itemsize == 8:
            u, v = u.view(np.int64), v.view(np.int64)
        assert (u == v).all()
    fi, bi = full.info(), b.info()
    assert fi["generation"] == bi["generation"] == G and fi["emax"] == bi["emax"]
    fb, bb = full.best(), b.best()
    assert (fb["x"] == bb["x"]).all() and (fb["y"] == bb["y"]).all() and (fb["start"] == bb["start"]).all()
    assert (np.asarray(fb["trace_min"]).view(np.int64) == np.asarray(bb["trace_min"]).view(np.int64)).all()
    assert (np.asarray(fb["trace_sum"]).view(np.int64) == np.asarray(bb["trace_sum"]).view(np.int64)).all()


def test_restore_rejects_bad_generation():
    wl = wlmod.config_A2()
    _, st, _ = both_event_ctx(wl)
    r = ffs.Run(st, 4, 4, 2, 5, 1)
    ck = r.checkpoint()
    ck["generation"] = 6   # beyond the configured 5 generations
    ck["trace_min"] = ck["trace_sum"] = np.zeros(7, np.int64)
    with pytest.raises(ffs.FFSError):
        r.restore(ck)
    other = ffs.Run(st, 4, 4, 2, 5, 2)   # another seed: refused before any copy
    with pytest.raises(ValueError):
        r.restore(other.checkpoint())
    ck = r.checkpoint()
    ck["x"] = ck["x"][:-1]               # wrong size: refused before any copy
    with pytest.raises(ValueError):
        r.restore(ck)
