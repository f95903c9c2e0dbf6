"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here is independent of the oracle's own formulas: paper-printed
values (Table 4, Figs. 8, 11, 12), hand-computed H3, Random123 KATs,
textbook special cases, brute force, and exhaustive integer scans.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import fixtures as fx

# --------------------------------------------------------------------------
# Philox4x32-10 known-answer vectors (Random123 kat_vectors)
# --------------------------------------------------------------------------
KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_kat(ctr, key, out):
    assert orc.philox(ctr, key).tolist() == out


# --------------------------------------------------------------------------
# Table 4 worked example
# --------------------------------------------------------------------------
def test_table4_freeze_matches_printed_Z_sentinels():
    d, inst, ctx = fx.table4_ctx()
    Zp = fx.printed_Z(d)
    assert ctx.K == 13                                   # 24 cells - r=11 frozen (R11)
    # z = C <-> COMPLETED, z = 0 <-> RUNNING, rank <-> PENDING
    expect = np.where(Zp == orc.Z_COMPLETED, orc.COMPLETED, np.where(Zp == 0, orc.RUNNING, orc.PENDING))
    assert (ctx.states == expect).all()
    # frozen cells are exactly the -1 cells of the printed X and Y
    X, Y = np.array(d["X"]), np.array(d["Y"])
    assert ((ctx.states != orc.PENDING) == (X == -1)).all()
    assert ((ctx.states != orc.PENDING) == (Y == -1)).all()
    # printed Y is a permutation of 1..K over the pending cells
    assert sorted(Y[Y > 0].tolist()) == list(range(1, 14))


def test_table4_decode_printed_Z_reproduces_fig8():
    d, inst, ctx = fx.table4_ctx()
    r = ctx.decode(np.array(d["X"]), np.array(d["Y"]), fx.printed_Z(d))
    st = r["start"].reshape(8, 3)
    # Fig. 8 caption: C_max = 20.42
    assert r["makespan"] == d["expected_makespan_with_printed_Z"] == 2042
    # j7s0 "is delayed until the completion of job 5 at stage 2"
    assert st[7, 0] == st[5, 2] + 300
    # it could not start at the completion of j2s0 on its machine
    assert st[7, 0] > 780
    # the decoded schedule is feasible (Eqs. (4)-(10)) and peak <= Q_max = 3
    n, kinds = ctx.validate(r["assign"], r["start"])
    assert n == 0, kinds
    peak = max(orc.power_at(inst, r["assign"], r["start"], t) for t in r["start"])
    assert peak == 3


def test_table4_greedy_order_and_one_swap_reading():
    """R1: the greedy reading of Algorithm 1 on the printed Y differs from the
    printed Z at ranks 4-7; swapping y_32 <-> y_60 reproduces the printed Z."""
    d, inst, ctx = fx.table4_ctx()
    Y = np.array(d["Y"])
    Zp = fx.printed_Z(d)
    Z = ctx.order(Y).reshape(8, 3)
    cells = lambda Zm: [int(np.flatnonzero(Zm.ravel() == k)[0]) for k in range(1, 14)]
    greedy = cells(Z)
    printed = cells(Zp)
    assert greedy != printed
    assert greedy[:3] == printed[:3] and greedy[7:] == printed[7:]
    Ys = Y.copy()
    Ys[3, 2], Ys[6, 0] = Ys[6, 0], Ys[3, 2]
    assert (ctx.order(Ys).reshape(8, 3) == Zp).all()
    # the greedy order also decodes to C_max 20.42
    assert ctx.decode(np.array(d["X"]), Y)["makespan"] == 2042


def test_table4_original_plan_is_a_decode_output():
    """Table 4's printed plan is decode(X = Table 4 machines, Y) at RS = 0."""
    d, a = fx.table4_arrays()
    n = d["n"]
    inst0 = orc.Instance(n, 0, a["g"], a["o"], a["P"][:n], a["Q"][:n], a["R"][:n], a["D"][:n],
                         a["q_max"], a["wt"])
    c0 = orc.Ctx(inst0, 0)
    assert c0.K == 18
    r = c0.decode(np.array(d["orig_assign"]), np.array(d["plan_Y_rs0"]))
    assert (r["start"].reshape(n, 3) == np.array(d["orig_start"])).all()
    assert c0.validate(r["assign"], r["start"])[0] == 0


# --------------------------------------------------------------------------
# H3: hand-computed instance
# --------------------------------------------------------------------------
def test_h3_hand_computed():
    d, inst, ctx = fx.h3()
    X, Y = np.array(d["X"]), np.array(d["Y"])
    Z = ctx.order(Y)
    order = [int(np.flatnonzero(Z == k)[0]) for k in range(1, ctx.K + 1)]
    assert order == d["expected_order_cells"]
    r = ctx.decode(X, Y)
    assert (r["start"].reshape(3, 2) == np.array(d["expected_start"])).all()
    assert r["sum_tardiness"] == d["expected_sum_tardiness"]
    assert r["makespan"] == d["expected_makespan"]
    assert r["objective"] == d["expected_objective"]
    assert r["counters"]["jumps"] == 1                      # only j0s1 is power-delayed


def test_h3_brute_force():
    d, inst, ctx = fx.h3()
    best, count, bx, bz = ctx.brute_force()
    assert count == d["brute_force_count"] == 2 ** 6 * 90
    assert best == d["brute_force_optimum"]
    # the witness decodes to the optimum and is feasible
    r = ctx.decode(bx, None, bz)
    assert r["objective"] == best and ctx.validate(r["assign"], r["start"])[0] == 0


# --------------------------------------------------------------------------
# GA operators: Fig. 11 and Fig. 12
# --------------------------------------------------------------------------
def test_fig11_crossover_and_correction():
    d, ctx = fx.operators_ctx()
    f = d["fig11"]
    assert ctx.K == 6
    XA2, YA2, XB2, YB2 = ctx.crossover(f["XA"], f["YA"], f["XB"], f["YB"], f["cut_row_major"])
    assert XA2.reshape(3, 3).tolist() == f["corrected_XA"]
    assert YA2.reshape(3, 3).tolist() == f["corrected_YA"]
    assert XB2.reshape(3, 3).tolist() == f["corrected_XB"]
    assert YB2.reshape(3, 3).tolist() == f["corrected_YB"]
    # correction alone maps the printed "After crossover" Y to the printed "Correction" Y
    assert ctx.repair(f["after_crossover_YA"]).reshape(3, 3).tolist() == f["corrected_YA"]
    assert ctx.repair(f["after_crossover_YB"]).reshape(3, 3).tolist() == f["corrected_YB"]


def test_fig12_mutation():
    d, ctx = fx.operators_ctx()
    f = d["fig12"]
    cells = ctx.pending_cells.tolist()
    ga, gb = (cells.index(c) for c in f["swap_cells_row_major"])
    for rx in (0, 123456789, 0xffffffff):     # o = 2: every draw flips the machine
        X2, Y2 = ctx.mutate(f["X"], f["Y"], [rx] * ctx.K, ga, gb)
        assert X2.reshape(3, 3).tolist() == f["X_after"]
        assert Y2.reshape(3, 3).tolist() == f["Y_after"]


def test_repair_is_identity_on_permutations():
    d, ctx = fx.operators_ctx()
    Y = np.array(d["fig11"]["YA"])
    assert (ctx.repair(Y) == Y.ravel()).all()


# --------------------------------------------------------------------------
# Eq. (13) and the E_max rule
# --------------------------------------------------------------------------
def test_emax_and_fitness():
    assert orc.emax([950, 432]) == 1000
    assert orc.emax([9]) == 10
    assert orc.emax([1000]) == 10000          # strict: "smaller than E_max"
    assert orc.emax([0]) == 10                # a starts at 1
    assert orc.fitness(18391, 100000) == 81609
    assert orc.fitness(10**5, 10**5) == 0     # clamp
    assert orc.fitness(10**6, 10**5) == 0
    assert orc.fitness(0, 1000) == 1000
