"""Pins of the oracle's fractional-WT objective (Table 11,
PAPER.md P:473-489; Eq. (1), Eq. (13), E_max rule P:375).

* an integer-valued real weight (WT = 100.0) reproduces the integer-objective
  GA bit for bit (the integer path is pinned by the paper's examples);
* WT = 0 gives C_max, the value is within one rounding of the exact rational
  WT*sum T + C_max and is non-decreasing in WT (Table 11's grid);
* E_max and Eq. (13) closed forms on fractional objectives;
* GA invariants with WT = 0.37: every stored objective is the decode's value,
  fitness = max(E_max - objective, 0), elitism keeps the best non-increasing.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx

TABLE11_WT = [0.01, 0.1, 0.4, 0.7, 1.0, 4.0, 7.0, 10.0, 100.0]       # Table 11


def test_emax_and_fitness_real_closed_forms():
    assert orc.emax_real([9.99]) == 10.0
    assert orc.emax_real([10.0]) == 100.0
    assert orc.emax_real([0.5, 99.5]) == 100.0
    assert orc.emax_real([99999.99]) == 1e5
    assert orc.emax_real([0.0]) == 10.0
    assert orc.fitness_real(99.75, 100.0) == 0.25
    assert orc.fitness_real(150.5, 100.0) == 0.0
    assert orc.fitness_real(100.0, 100.0) == 0.0


def test_value_rounding_and_monotone_in_wt():
    d, inst, ctx = fx.table4_ctx()
    r = ctx.decode(np.array(d["X"]), np.array(d["Y"]))
    T, M = r["sum_tardiness"], r["makespan"]
    assert M == 2042                                   # Fig. 8 caption
    prev = None
    for wt in [0.0] + TABLE11_WT:
        ctx.set_real_weight(wt)
        v = ctx.decode(np.array(d["X"]), np.array(d["Y"]))["value"]
        exact = Fraction(wt) * T + M
        assert abs(Fraction(v) - exact) <= abs(exact) * Fraction(2, 2 ** 52)
        if wt == 0.0:
            assert v == M
        if prev is not None:
            assert v >= prev
        prev = v


def test_integer_valued_real_weight_equals_integer_ga():
    wl = wlmod.config_A2()
    ctx_i, _, _, _ = fx.oracle_event_ctx(wl)
    ctx_r, _, _, _ = fx.oracle_event_ctx(wl)
    ctx_r.set_real_weight(float(wl.wt))
    G = 21
    gi = orc.GA(ctx_i, 4, 4, 4, G, 99)
    gr = orc.GA(ctx_r, 4, 4, 4, G, 99)
    for _ in range(G + 1):
        gi.step()
        gr.step()
        xi, yi, oi, fi = gi.population()
        xr, yr, orr, fr = gr.population()
        assert (xi == xr).all() and (yi == yr).all()
        assert (oi.astype(np.float64) == orr).all() and (fi.astype(np.float64) == fr).all()
    assert float(gi.emax) == gr.emax
    ti, si = gi.trace()
    tr, sr = gr.trace()
    assert (ti.astype(np.float64) == tr).all() and (si.astype(np.float64) == sr).all()


def test_fractional_ga_invariants():
    wl = wlmod.config_A2()
    ctx, _, _, _ = fx.oracle_event_ctx(wl)
    ctx.set_real_weight(0.37)
    G = 15
    ga = orc.GA(ctx, 4, 4, 2, G, 5)
    ga.step()
    E = ga.emax
    x, y, obj, fit = ga.population()
    assert E > obj.max() and E / 10 <= obj.max() or E == 10.0
    for k in range(G + 1):
        if k:
            ga.step()
        x, y, obj, fit = ga.population()
        for i in range(0, len(obj), 5):
            assert ctx.decode_genes(x[i], y[i])["value"] == obj[i]
        assert (fit == np.maximum(E - obj, 0.0)).all()
    tmin, tsum = ga.trace()
    assert (np.diff(tmin) <= 0).all()
    hx, hy, hobj, hfit = ga.history()
    assert (hfit == np.maximum(E - hobj, 0.0)).all()
    assert np.isclose(tsum[-1], obj.sum(), rtol=1e-12)
