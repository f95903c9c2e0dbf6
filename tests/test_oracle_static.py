"""Pins of the oracle's traditional static approach (
PAPER.md P:291 / P:313-317, Fig. 7; readings R29-R30).

* Table 4 in the static environment: the decoder-reachable optimum makespan
  over every arrival chromosome is 19.91 (Fig. 7 caption) -- with WT = 0
  the brute-force optimum IS the makespan, so the unprinted due dates do not
  enter.  A reading without the originals' power (R30) reaches 18.42 on the
  same enumeration (scratch check), so the pin separates the two.
* the freeze pattern: originals COMPLETED / RUNNING as in the printed Z, every
  other original op KEPT, arrivals are the only genes (K = n'g);
* decode == an independent exhaustive integer scan with the static initial
  conditions, on random instances; validate() (incl. the append check) holds;
* zero arrivals: K = 0 and the schedule is the original plan.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx
from tests.test_oracle_properties import random_ctx


def table4_static(wt=None):
    d, a = fx.table4_arrays()
    if wt is not None:
        a = dict(a, wt=wt)
    inst = orc.Instance(**a)
    return d, inst, orc.Ctx(inst, d["rs"], np.array(d["orig_assign"]), np.array(d["orig_start"]), static=True)


def test_table4_static_freeze_pattern():
    d, inst, ctx = table4_static()
    Zp = fx.printed_Z(d)
    assert ctx.K == d["n_prime"] * d["g"] == 6
    for j in range(d["n"] + d["n_prime"]):
        for s in range(d["g"]):
            z, st = Zp[j, s], ctx.states[j, s]
            if j >= d["n"]:
                assert st == orc.PENDING
            elif z == orc.Z_COMPLETED:
                assert st == orc.COMPLETED
            elif z == 0:
                assert st == orc.RUNNING
            else:                               # pending in the dynamic freeze -> held
                assert st == orc.KEPT
    x, y = wlmod.random_chromosomes(1, ctx.K, 2, 1)
    Z = ctx.order(ctx.to_matrix(x[0], y[0])[1])
    assert ((Z.reshape(ctx.states.shape) == orc.Z_KEPT) == (ctx.states == orc.KEPT)).all()


def test_fig7_static_optimum_makespan():
    """Fig. 7 caption: C_max = 19.91 for the optimized static schedule."""
    d, inst, ctx = table4_static(wt=0)
    best, count, bX, bZ = ctx.brute_force()
    assert count == 2 ** 6 * 20            # o^K * (6 choose 3) chain interleavings
    assert best == 1991
    r = ctx.decode(bX, None, Z=bZ)
    assert r["makespan"] == 1991
    assert ctx.validate(r["assign"], r["start"])[0] == 0


def _scan_static(inst, ctx, X, order_cells):
    """Independent statement of the static baseline: every original op keeps
    (machine, start); an arrival op starts at the first integer t >= max(RS,
    release / predecessor completion, end of every earlier op on its machine)
    where the power of all ops overlapping [t, t+p) stays <= Q_max."""
    g = inst.g
    placed = []                                  # (s, m, start, end, q)
    start = -np.ones(ctx.cells, np.int64)
    asg = -np.ones(ctx.cells, np.int64)
    for cell in range(ctx.cells):
        if ctx.states.ravel()[cell] != orc.PENDING:
            j, s = divmod(cell, g)
            m = int(ctx._oa[cell])
            start[cell], asg[cell] = ctx._os[cell], m
            placed.append((s, m, int(start[cell]), int(start[cell] + inst.P[j, s, m]), int(inst.Q[j, s, m])))
    for cell in order_cells:
        j, s = divmod(int(cell), g)
        m = int(X[cell])
        p, q = int(inst.P[j, s, m]), int(inst.Q[j, s, m])
        ready = inst.R[j] if s == 0 else start[cell - 1] + inst.P[j, s - 1, asg[cell - 1]]
        t = max([ctx.rs, int(ready)] + [e for (ss, mm, _, e, _) in placed if (ss, mm) == (s, m)])
        while any(sum(qq for (_, _, a, b, qq) in placed if a <= tau < b) + q > inst.q_max
                  for tau in range(t, t + p)):
            t += 1
        start[cell], asg[cell] = t, m
        placed.append((s, m, t, t + p, q))
    return asg, start


def static_ctx_from(inst, ctx):
    return orc.Ctx(inst, ctx.rs, ctx._oa, ctx._os, static=True)


@pytest.mark.parametrize("case", [(3, 2, 2, 2, 2, 1, 5), (4, 2, 3, 2, 3, 1, 5), (5, 3, 3, 2, 3, 3, 6),
                                  (4, 1, 2, 3, 2, 2, 9)])
def test_static_decode_equals_scan_and_is_valid(case):
    n, n_p, g, o, q_max, pw, pmax = case
    rng = np.random.default_rng(sum(case) * 7919 + len(case))
    for rep in range(4):
        inst, dctx, _ = random_ctx(rng, n, n_p, g, o, q_max, pw, pmax=pmax)
        ctx = static_ctx_from(inst, dctx)
        assert ctx.K == n_p * g
        assert (ctx.states[:n] != orc.PENDING).all() and (ctx.states[n:] == orc.PENDING).all()
        xs, ys = wlmod.random_chromosomes(10, ctx.K, o, int(rng.integers(1 << 30)))
        for x, y in zip(xs, ys):
            X, Y = ctx.to_matrix(x, y)
            r = ctx.decode(X, Y)
            Z = ctx.order(Y)
            order_cells = [int(np.flatnonzero(Z == k)[0]) for k in range(1, ctx.K + 1)]
            asg, st = _scan_static(inst, ctx, X, order_cells)
            assert (st == r["start"]).all() and (asg == r["assign"]).all()
            nv, kinds = ctx.validate(r["assign"], r["start"])
            assert nv == 0, kinds
            # originals verbatim (byte-equal to the plan, SPEC invariant)
            assert (r["assign"][: n * g] == ctx._oa).all() and (r["start"][: n * g] == ctx._os).all()


def test_static_validate_detects_append_violation():
    d, inst, ctx = table4_static()
    x, y = wlmod.random_chromosomes(1, ctx.K, 2, 5)
    r = ctx.decode_genes(x[0], y[0])
    assert ctx.validate(r["assign"], r["start"])[0] == 0
    # job 6 stage 0 forced before the last original op on its machine ends
    asg, st = r["assign"].copy(), r["start"].copy()
    c = 6 * 3
    m = asg[c]
    ends = [d["orig_start"][j][0] + 100 for j in range(6) if d["orig_assign"][j][0] == m]
    st[c] = max(ends) - 1
    assert ctx.validate(asg, st)[1] & 128
    # the dynamic context does not impose the append rule
    dctx = fx.table4_ctx()[2]
    assert not (dctx.validate(asg, st)[1] & 128)


def test_zero_arrivals_static_is_the_plan():
    rng = np.random.default_rng(3)
    inst, dctx, plan = random_ctx(rng, 4, 0, 3, 2, 3, rs_ratio=0.4)
    ctx = static_ctx_from(inst, dctx)
    assert ctx.K == 0
    r = ctx.decode(np.full(ctx.cells, -1, np.int32), np.full(ctx.cells, -1, np.int32))
    assert (r["start"] == plan["start"]).all() and (r["assign"] == plan["assign"]).all()
    assert r["makespan"] == plan["makespan"]


def test_static_requires_plan():
    d, a = fx.table4_arrays()
    with pytest.raises(Exception):
        orc.Ctx(orc.Instance(**a), 700, static=True)
