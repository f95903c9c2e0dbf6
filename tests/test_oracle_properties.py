"""Property pins of the oracle: exhaustive scans, textbook special cases,
brute force and the schedule invariants of Eqs. (4)-(10)."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx


def random_ctx(rng, n, n_prime, g, o, q_max, power_max=1, rs_ratio=None, pmax=5):
    """Random integer instance; the original plan is an oracle decode at RS=0
    of a random chromosome (any valid plan is a valid input)."""
    NJ = n + n_prime
    P = rng.integers(1, pmax + 1, size=(NJ, g, o)).astype(np.int32)
    Q = rng.integers(0 if power_max > 1 else 1, power_max + 1, size=(NJ, g, o)).astype(np.int32)
    R = rng.integers(0, 6, size=NJ).astype(np.int32)
    D = (R + rng.integers(0, 20, size=NJ)).astype(np.int32)
    q_max = max(int(q_max), int(Q.max()))
    inst0 = orc.Instance(n, 0, g, o, P[:n], Q[:n], R[:n], D[:n], q_max, 7)
    c0 = orc.Ctx(inst0, 0)
    x, y = wlmod.random_chromosomes(1, c0.K, o, int(rng.integers(1 << 30)))
    plan = c0.decode(*c0.to_matrix(x[0], y[0]))
    if rs_ratio is None:
        rs_ratio = rng.uniform(0.0, 0.9)
    rs = int(np.floor(rs_ratio * plan["makespan"]))
    R = R.copy()
    R[n:] = rs + rng.integers(0, 6, size=n_prime)
    D = (R + rng.integers(0, 20, size=NJ)).astype(np.int32)
    inst = orc.Instance(n, n_prime, g, o, P, Q, R, D, q_max, 7)
    ctx = orc.Ctx(inst, rs, plan["assign"][: n * g], plan["start"][: n * g])
    return inst, ctx, plan


def scan_decode(inst, ctx, X, order_cells):
    """Independent re-statement of Algorithm 2 by exhaustive integer scan:
    S = min{t >= t0 : for all tau in [t, t+p): Q_tau + q <= Q_max}."""
    g, o = inst.g, inst.o
    cells = ctx.cells
    start = -np.ones(cells, np.int64)
    comp = -np.ones(cells, np.int64)
    asg = -np.ones(cells, np.int64)
    ivs = []
    mfree = np.full((g, o), ctx.rs, np.int64)
    for cell in range(cells):
        if ctx.states.ravel()[cell] != orc.PENDING:
            j, s = divmod(cell, g)
            m = int(ctx._oa[cell])
            start[cell] = ctx._os[cell]
            comp[cell] = start[cell] + inst.P[j, s, m]
            asg[cell] = m
            if ctx.states.ravel()[cell] == orc.RUNNING:
                ivs.append((start[cell], comp[cell], int(inst.Q[j, s, m])))
                mfree[s, m] = max(mfree[s, m], comp[cell])
    for cell in order_cells:
        j, s = divmod(int(cell), g)
        m = int(X[cell])
        p, q = int(inst.P[j, s, m]), int(inst.Q[j, s, m])
        ready = inst.R[j] if s == 0 else comp[cell - 1]
        t = max(ctx.rs, ready, mfree[s, m])

        def level(tau):
            return sum(qq for (a, b, qq) in ivs if a <= tau < b)
        while any(level(tau) + q > inst.q_max for tau in range(t, t + p)):
            t += 1
        start[cell], comp[cell], asg[cell] = t, t + p, m
        ivs.append((t, t + p, q))
        mfree[s, m] = t + p
    return asg, start


def prefix_min_order(ctx, Y):
    """R1 shortcut used by the GPU: stable sort by (prefix-min of y over the
    job's pending stages, descending; stage ascending)."""
    Y = np.asarray(Y).ravel()
    keys = []
    g = ctx.inst.g
    for cell in ctx.pending_cells:
        j, s = divmod(int(cell), g)
        pm = min(Y[j * g + t] for t in range(s + 1) if ctx.states[j, t] == orc.PENDING)
        keys.append((-pm, s, int(cell)))
    return [c for (_, _, c) in sorted(keys)]


CASES = [  # n, n', g, o, q_max, power_max, pmax
    (3, 1, 2, 2, 2, 1, 5),
    (4, 2, 3, 2, 3, 1, 5),
    (5, 2, 3, 3, 2, 1, 5),
    (4, 0, 2, 2, 3, 3, 5),
    (6, 2, 4, 2, 4, 3, 5),
    (3, 3, 3, 1, 1, 1, 4),
    (2, 2, 1, 2, 2, 2, 9),
    (5, 3, 2, 3, 3, 2, 30),
]


@pytest.mark.parametrize("case", CASES)
def test_decode_equals_exhaustive_scan_and_is_valid(case):
    """Jump rule (R5) == earliest feasible integer start; Eqs. (4)-(10) hold."""
    n, n_p, g, o, q_max, pw, pmax = case
    rng = np.random.default_rng(hash(case) % (1 << 32))
    for rep in range(4):
        inst, ctx, _ = random_ctx(rng, n, n_p, g, o, q_max, pw, pmax=pmax)
        if ctx.K == 0:
            continue
        xs, ys = wlmod.random_chromosomes(12, ctx.K, o, int(rng.integers(1 << 30)))
        for x, y in zip(xs, ys):
            X, Y = ctx.to_matrix(x, y)
            r = ctx.decode(X, Y)
            Z = ctx.order(Y)
            order_cells = [int(np.flatnonzero(Z == k)[0]) for k in range(1, ctx.K + 1)]
            asg, st = scan_decode(inst, ctx, X, order_cells)
            assert (st == r["start"]).all() and (asg == r["assign"]).all()
            nv, kinds = ctx.validate(r["assign"], r["start"])
            assert nv == 0, kinds
            T, M, O = orc.objective(inst, r["assign"], r["start"])
            assert (T, M, O) == (r["sum_tardiness"], r["makespan"], r["objective"])


@pytest.mark.parametrize("seed", range(6))
def test_greedy_order_equals_prefix_min_sort(seed):
    rng = np.random.default_rng(100 + seed)
    inst, ctx, _ = random_ctx(rng, 7, 3, 4, 2, 3)
    for _ in range(40):
        x, y = wlmod.random_chromosomes(1, ctx.K, 2, int(rng.integers(1 << 30)))
        X, Y = ctx.to_matrix(x[0], y[0])
        Z = ctx.order(Y)
        greedy = [int(np.flatnonzero(Z == k)[0]) for k in range(1, ctx.K + 1)]
        assert greedy == prefix_min_order(ctx, Y)
        # ranks strictly increase with stage inside each job
        Zm = Z.reshape(ctx.states.shape)
        for j in range(Zm.shape[0]):
            pend = [Zm[j, s] for s in range(Zm.shape[1]) if ctx.states[j, s] == orc.PENDING]
            assert pend == sorted(pend)


def test_order_special_cases():
    """a single pending job ranks in stage order; two single-stage
    jobs with y = (2, 1) rank (1, 2)."""
    P = np.ones((1, 3, 1), np.int32)
    inst = orc.Instance(1, 0, 3, 1, P, P, np.zeros(1, np.int32), np.zeros(1, np.int32), 1, 1)
    ctx = orc.Ctx(inst, 0)
    assert ctx.order([3, 1, 2]).tolist() == [1, 2, 3]
    P = np.ones((2, 1, 1), np.int32)
    inst = orc.Instance(2, 0, 1, 1, P, P, np.zeros(2, np.int32), np.zeros(2, np.int32), 1, 1)
    assert orc.Ctx(inst, 0).order([2, 1]).tolist() == [1, 2]


def test_no_power_binding_is_plain_list_scheduling():
    """with Q_max >= sum of all powers the decode never delays and is
    the textbook list schedule S = max(RS, ready, machine free)."""
    rng = np.random.default_rng(7)
    for _ in range(10):
        inst, ctx, _ = random_ctx(rng, 5, 2, 3, 2, 10 ** 6)
        x, y = wlmod.random_chromosomes(1, ctx.K, 2, int(rng.integers(1 << 30)))
        X, Y = ctx.to_matrix(x[0], y[0])
        r = ctx.decode(X, Y)
        assert r["counters"]["jumps"] == 0
        Z = ctx.order(Y)
        g = inst.g
        comp = {}
        mfree = {}
        for cell in range(ctx.cells):
            if ctx.states.ravel()[cell] != orc.PENDING:
                j, s = divmod(cell, g)
                m = int(ctx._oa[cell])
                comp[cell] = int(ctx._os[cell]) + int(inst.P[j, s, m])
                if ctx.states.ravel()[cell] == orc.RUNNING:
                    mfree[(s, m)] = comp[cell]
        for k in range(1, ctx.K + 1):
            cell = int(np.flatnonzero(Z == k)[0])
            j, s = divmod(cell, g)
            m = int(X[cell])
            ready = int(inst.R[j]) if s == 0 else comp[cell - 1]
            S = max(ctx.rs, ready, mfree.get((s, m), ctx.rs))
            assert r["start"][cell] == S
            comp[cell] = S + int(inst.P[j, s, m])
            mfree[(s, m)] = comp[cell]


def test_single_machine_textbook():
    """g = o = 1, no power binding: jobs run back to back in descending y."""
    n = 6
    rng = np.random.default_rng(3)
    P = rng.integers(1, 6, size=(n, 1, 1)).astype(np.int32)
    Q = np.ones_like(P)
    R = rng.integers(0, 10, size=n).astype(np.int32)
    D = R + 3
    inst = orc.Instance(n, 0, 1, 1, P, Q, R, D, 1, 5)
    ctx = orc.Ctx(inst, 0)
    Y = (rng.permutation(n) + 1).astype(np.int32)
    r = ctx.decode(np.zeros(n, np.int32), Y)
    t = 0
    for j in np.argsort(-Y):
        t = max(t, int(R[j]))
        assert r["start"][j] == t
        t += int(P[j, 0, 0])
    assert r["makespan"] == t


def test_freeze_boundaries():
    """R7: completion == RS -> COMPLETED; start == RS -> PENDING; S < RS < C -> RUNNING."""
    P = np.full((3, 1, 3), 2, np.int32)
    Q = np.ones_like(P)
    inst = orc.Instance(3, 0, 1, 3, P, Q, np.zeros(3, np.int32), np.full(3, 9, np.int32), 3, 1)
    ctx = orc.Ctx(inst, 4, np.array([0, 1, 2]), np.array([2, 4, 3]))
    assert ctx.states.ravel().tolist() == [orc.COMPLETED, orc.PENDING, orc.RUNNING]
    ctx0 = orc.Ctx(inst, 0, np.array([0, 1, 2]), np.array([2, 4, 3]))
    assert (ctx0.states == orc.PENDING).all()


def test_infeasible_and_bad_plans_rejected():
    P = np.ones((2, 1, 1), np.int32)
    Q = np.full((2, 1, 1), 3, np.int32)
    inst = orc.Instance(2, 0, 1, 1, P, Q, np.zeros(2, np.int32), np.zeros(2, np.int32), 2, 1)
    with pytest.raises(orc.OracleError) as e:
        orc.Ctx(inst, 0)
    assert e.value.code == orc.ERR_INFEASIBLE
    Q = np.ones((2, 1, 1), np.int32)
    inst = orc.Instance(2, 0, 1, 1, P, Q, np.zeros(2, np.int32), np.zeros(2, np.int32), 2, 1)
    with pytest.raises(orc.OracleError) as e:       # two ops overlap on one machine (Eq. (6))
        orc.Ctx(inst, 1, np.array([0, 0]), np.array([0, 0]))
    assert e.value.code == orc.ERR_SCHEDULE


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 5, 11])
def test_brute_force_bounds_every_decode(seed):
    """The decoder-reachable optimum is <= every decoded chromosome and the
    enumeration count is o^K * K!/prod L_j!.  Seeds chosen so
    every instance has K <= 7 (K = 5..7): none is skipped."""
    rng = np.random.default_rng(50 + seed)
    inst, ctx, _ = random_ctx(rng, 3, 1, 2, 2, 2, rs_ratio=0.3)
    assert 5 <= ctx.K <= 7
    best, count, _, _ = ctx.brute_force()
    L = [int((ctx.states[j] == orc.PENDING).sum()) for j in range(ctx.states.shape[0])]
    from math import factorial
    orders = factorial(sum(L))
    for l in L:
        orders //= factorial(l)
    assert count == 2 ** ctx.K * orders
    xs, ys = wlmod.random_chromosomes(200, ctx.K, 2, seed)
    for x, y in zip(xs, ys):
        assert ctx.decode_genes(x, y)["objective"] >= best


def test_frozen_ops_untouched_and_validate_detects_violations():
    d, inst, ctx = fx.table4_ctx()
    r = ctx.decode(np.array(d["X"]), np.array(d["Y"]))
    st = r["start"].copy()
    st[0] += 1                       # move a COMPLETED op
    assert ctx.validate(r["assign"], st)[1] & 32
    st = r["start"].copy()
    st[3 * 3 + 1] = 600              # a pending op before RS (Eq. (10)), also Eq. (5)
    assert ctx.validate(r["assign"], st)[1] & 16
    asg = r["assign"].copy()
    st = r["start"].copy()
    # put j6s0 on j7s0's machine at the same start: Eq. (6)
    asg[6 * 3], st[6 * 3] = asg[7 * 3], st[7 * 3]
    assert ctx.validate(asg, st)[1] & 4
