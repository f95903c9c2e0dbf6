"""Hand-derived goldens for the oracle's GA steps (tests/golden/ga_ops.json).

The paper prints no GA trajectory, and its Figs. 9, 10 and 13 are missing,
so each step the oracle GA runs is pinned on its own by a small case worked
out by hand, chosen so that a plausible slip fails it:
  * init ranks: a key tie (ties by gene index) and a key >= 2^31
    (unsigned comparison);
  * selection (R17, R18): N=S, self=N and E=W ties, wraps on every
    edge, a non-square tile (w/h transposition);
  * breeding (R13, R16, R19, R20): the pair order, the '<'
    thresholds (one draw exactly at the threshold), the cut mapping, the
    mutation after the crossover, the b >= a shift of the swap genes;
  * replacement (R21): strict improvement, an equal best (no update),
    ties of the best and of the worst to the lowest cell;
  * migration (R22): direction, synchronous snapshot (an import
    that beats the receiving island's own best), ring across a shard
    boundary through the allgather record;
  * trace.
The oracle GA calls exactly these functions (oracle/ffs_oracle.c ga_init /
ga_generation), so the GPU trajectory parity tests inherit the pins.
"""
import json
import os
import threading

import numpy as np
import pytest

from oracle import oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))
G = json.load(open(os.path.join(HERE, "golden", "ga_ops.json")))


def _ops_ctx():
    d = json.load(open(os.path.join(HERE, "golden", "operators.json")))["ctx"]
    n, g, o = d["n"], d["g"], d["o"]
    P = np.ones((n, g, o), np.int32)
    inst = orc.Instance(n, 0, g, o, P, P.copy(), np.zeros(n, np.int32), np.full(n, 100, np.int32),
                        d["q_max"], 1)
    return orc.Ctx(inst, d["rs"], np.array(d["orig_assign"]), np.array(d["orig_start"]))


def test_init_ranks():
    d = G["init_ranks"]
    assert orc.init_ranks(d["keys"]).tolist() == d["y"]


def test_select():
    for case in G["select"]:
        win = orc.select(np.array(case["fit"], np.float64).ravel(), case["w"], case["h"])
        assert win.tolist() == case["winner"], case["cite"]


def test_argmax_argmin_ties_lowest():
    lib = orc.lib()
    f = np.array([3.0, 7.0, 1.0, 7.0, 1.0])
    assert lib.or_argmax_fitness(orc._p(f), 5) == 1
    assert lib.or_argmin_fitness(orc._p(f), 5) == 2


def test_breed_one_island():
    d = G["breed"]
    ctx = _ops_ctx()
    assert ctx.K == 6 and ctx.pending_cells.tolist() == [1, 2, 5, 6, 7, 8]
    tile = d["w"] * d["h"]
    PX = np.array(d["parents_X"], np.int32).reshape(tile, ctx.cells)
    PY = np.array(d["parents_Y"], np.int32).reshape(tile, ctx.cells)
    mut_x = np.zeros((tile, ctx.K), np.uint32)     # o = 2: every draw flips the machine
    X, Y = orc.breed(ctx, d["w"], d["h"], PX, PY, d["winner"], d["xo_fire"], d["xo_cut"],
                     d["mut_fire"], d["mut_a"], d["mut_b"], mut_x)
    assert X.tolist() == np.array(d["children_X"]).reshape(tile, -1).tolist()
    assert Y.tolist() == np.array(d["children_Y"]).reshape(tile, -1).tolist()


def _pop(d, key="X"):
    X = np.ascontiguousarray(np.array(d[key], np.int32).reshape(-1, 1))
    fit = np.ascontiguousarray(np.array(d["fit"], np.float64).ravel())
    return X, X.copy(), d["emax"] - fit, fit


def test_replace():
    d = G["replace"]
    X, Y, obj, fit = _pop(d)
    HX = np.array(d["hist_X"], np.int32).reshape(-1, 1)
    hfit = np.array(d["hist_fit"], np.float64)
    HY, hobj = HX.copy(), d["emax"] - hfit
    orc.replace(d["tile"], X, Y, obj, fit, HX, HY, hobj, hfit)
    assert X.ravel().tolist() == np.ravel(d["X_after"]).tolist()
    assert (Y == X).all()
    assert fit.tolist() == np.ravel(d["fit_after"]).astype(float).tolist()
    assert (obj == d["emax"] - fit).all()
    assert HX.ravel().tolist() == d["hist_X_after"] and (HY == HX).all()
    assert hfit.tolist() == [float(v) for v in d["hist_fit_after"]]
    assert (hobj == d["emax"] - hfit).all()


def _check_migrated(d, X, Y, obj, fit):
    assert X.ravel().tolist() == np.ravel(d["X_after"]).tolist()
    assert (Y == X).all()
    assert fit.tolist() == np.ravel(d["fit_after"]).astype(float).tolist()
    assert (obj == d["emax"] - fit).all()


def test_migrate_single_shard():
    d = G["migrate"]
    X, Y, obj, fit = _pop(d)
    orc.migrate(len(d["X"]), d["tile"], X, Y, obj, fit)
    _check_migrated(d, X, Y, obj, fit)


@pytest.mark.parametrize("split", [0, 1])
def test_migrate_across_shard_boundary(split):
    """Shards (islands [0,2) + [2,3), or one island per rank at world 3) run
    concurrently with an allgather of their boundary records: the same ring
    as one shard; world 3 separates rank-1 from rank+1."""
    d = G["migrate"]
    sp = d["shard_splits"][split]
    tile, emax = d["tile"], d["emax"]
    world = len(sp["shards"])
    slots = [None] * world
    bar = threading.Barrier(world)
    sent = {}
    out = {}
    errs = []

    def run(rank):
        try:
            b, e = sp["shards"][rank]
            X = np.ascontiguousarray(np.array(d["X"][b:e], np.int32).reshape(-1, 1))
            fit = np.ascontiguousarray(np.array(d["fit"][b:e], np.float64).ravel())
            Y, obj = X.copy(), emax - fit

            def allgather(buf):
                sent[rank] = buf
                slots[rank] = buf
                bar.wait()
                res = list(slots)
                bar.wait()
                return res
            orc.migrate(e - b, tile, X, Y, obj, fit, rank=rank, world=world, allgather=allgather)
            out[rank] = (X, Y, obj, fit)
        except Exception as ex:  # pragma: no cover - surfaced below
            errs.append(ex)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in range(world):
        s = sp["sent"][r]
        assert sent[r] == orc.migration_record([s["X"]], [s["X"]], emax - s["fit"], s["fit"])
    X, Y, obj, fit = (np.concatenate([out[r][i] for r in range(world)]) for i in range(4))
    _check_migrated(d, X, Y, obj, fit)


def test_trace_stats():
    d = G["trace"]
    assert orc.trace_stats(d["obj"]) == (d["min"], d["sum"])
    d = G["trace_islands"]
    assert orc.trace_stats(d["obj"], d["tile"]) == (d["min"], d["sum"])
