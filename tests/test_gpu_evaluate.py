"""Bit-exact parity of the CUDA decode/evaluate (through the C-ABI) with the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx
from tests.gpu_util import both_event_ctx, check_gene_order, gpu_state

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def gpu_eval(st, x, y, sched=False):
    xd = torch.as_tensor(np.ascontiguousarray(x)).to(DEV)
    yd = torch.as_tensor(np.ascontiguousarray(y)).to(DEV)
    obj, T, M, S = ffs.evaluate(st, xd, yd, with_schedule=sched)
    torch.cuda.synchronize()
    return obj.cpu().numpy(), T.cpu().numpy(), M.cpu().numpy(), (S.cpu().numpy() if sched else None)


def compare(octx, st, x, y, n_sched=None):
    """Objective, sum T, C_max and the full schedule of EVERY chromosome (the
    schedule-emitting launch), and the values of the plain launch."""
    obj, T, M, S = gpu_eval(st, x, y, sched=True)
    obj2, T2, M2, _ = gpu_eval(st, x, y, sched=False)
    oo, oT, oM, oS = octx.evaluate_batch_schedule(x, y, nthreads=8)
    assert (obj == oo).all(), np.flatnonzero(obj != oo)[:10]
    assert (T == oT).all()
    assert (M == oM).all()
    assert (obj2 == oo).all() and (T2 == oT).all() and (M2 == oM).all()
    bad = np.flatnonzero((S != oS).any(axis=1))
    assert bad.size == 0, f"schedules differ at {bad[:10]}"


def test_table4_printed_chromosome():
    d, inst, octx = fx.table4_ctx()
    _, a = fx.table4_arrays()
    st = gpu_state(a, d["rs"], np.array(d["orig_assign"]), np.array(d["orig_start"]))
    check_gene_order(octx, st)
    x, y = octx.to_genes(np.array(d["X"]), np.array(d["Y"]))
    obj, T, M, S = gpu_eval(st, x[None], y[None], sched=True)
    assert M[0] == 2042                                       # Fig. 8 caption
    compare(octx, st, x[None], y[None])


def test_h3():
    d, inst, octx = fx.h3()
    a = dict(n=3, n_prime=0, g=2, o=2, P=np.array(d["P"]), Q=np.ones((3, 2, 2), np.int32),
             R=np.array(d["release"]), D=np.array(d["due"]), q_max=2, wt=10)
    st = gpu_state(a, 0)
    x, y = octx.to_genes(np.array(d["X"]), np.array(d["Y"]))
    obj, T, M, S = gpu_eval(st, x[None], y[None], sched=True)
    assert obj[0] == 27 and T[0] == 2 and M[0] == 7
    assert (S[0].reshape(3, 2) == np.array(d["expected_start"])).all()


@pytest.mark.parametrize("cfg,count,nsched", [("A2", 3000, 200), ("B", 1000, 50), ("C", 300, 10)])
def test_random_chromosomes_configs(cfg, count, nsched, path):
    wl = {"A2": wlmod.config_A2, "B": wlmod.config_B, "C": wlmod.config_C}[cfg]()
    octx, st, arr = both_event_ctx(wl)
    check_gene_order(octx, st)
    x, y = wlmod.random_chromosomes(count, st.K, wl.o, seed=7)
    compare(octx, st, x, y, n_sched=nsched)


def test_general_power_path(path):
    wl = wlmod.gen_v1("Cq", 30, 6, 3, 6, arrivals_per_event=[8], ratios=[0.3], power="u13", seed=5)
    octx, st, arr = both_event_ctx(wl)
    x, y = wlmod.random_chromosomes(500, st.K, wl.o, seed=8)
    compare(octx, st, x, y, n_sched=20)


@pytest.mark.parametrize("fb", ["relist", "relist_chain", "smem", "global"])
def test_overflow_path_is_exact(path, fb, monkeypatch):
    """A tiny in-SMEM horizon forces the overflow paths: mode 2's lane
    re-decode of the overflow list with a longer horizon (relist; capped at
    96 ticks so that some chromosomes go on to the general fallback:
    relist_chain), and the general fallback over the full proven horizon with
    its profile in shared memory, or in global memory (FFS_FALLBACK_GLOBAL)."""
    monkeypatch.delenv("FFS_RELIST_CAP", raising=False)
    monkeypatch.delenv("FFS_FALLBACK_GLOBAL", raising=False)
    if fb == "relist_chain":
        monkeypatch.setenv("FFS_RELIST_CAP", "96")
    elif fb in ("smem", "global"):
        monkeypatch.setenv("FFS_RELIST_CAP", "0")
    if fb == "global":
        monkeypatch.setenv("FFS_FALLBACK_GLOBAL", "1")
    wl = wlmod.config_B()
    octx, st, arr = both_event_ctx(wl)
    x, y = wlmod.random_chromosomes(400, st.K, wl.o, seed=9)
    ref = gpu_eval(st, x, y, sched=True)
    st.set_horizon_cap(64)
    assert st.info()["horizon_bound"] > 64
    # the first overflowing call goes to the general fallback; it sets the
    # state's sticky overflow flag, so the second one (relist*) re-decodes the
    # overflow list on the lane path first
    for _ in range(2):
        got = gpu_eval(st, x, y, sched=True)
        for u, v in zip(ref, got):
            assert (u == v).all()
    compare(octx, st, x[:100], y[:100], n_sched=20)
    st.set_horizon_cap(0)


def test_u16_profile_path():
    """Q_max > 255 selects the 16-bit power profile."""
    rng = np.random.default_rng(4)
    n, g, o = 12, 3, 3
    P = rng.integers(1, 6, size=(n, g, o)).astype(np.int32)
    Q = rng.integers(50, 200, size=(n, g, o)).astype(np.int32)
    R = rng.integers(0, 5, size=n).astype(np.int32)
    a = dict(n=n, n_prime=0, g=g, o=o, P=P, Q=Q, R=R, D=R + 10, q_max=400, wt=3)
    octx = orc.Ctx(fx.workload_instance(a), 0)
    st = gpu_state(a, 0)
    x, y = wlmod.random_chromosomes(300, st.K, o, seed=3)
    compare(octx, st, x, y, n_sched=30)


def edge_instance(case, seed):
    rng = np.random.default_rng(seed)
    n, g, o, qmax = 6, 3, 2, 2
    P = rng.integers(1, 4, size=(n, g, o)).astype(np.int32)
    Q = np.ones((n, g, o), np.int32)
    R = rng.integers(0, 4, size=n).astype(np.int32)
    D = R + 5
    if case == "o1":
        o, P, Q = 1, P[:, :, :1].copy(), Q[:, :, :1].copy()
    if case == "g1":
        g, P, Q = 1, P[:, :1].copy(), Q[:, :1].copy()
    if case == "qinf":
        qmax = 1000
    if case == "q0":
        Q = rng.integers(0, 2, size=P.shape).astype(np.int32)
    if case == "static_ties":
        P = np.ones_like(P)
        R = np.zeros(n, np.int32)
    a = dict(n=n, n_prime=0, g=g, o=o, P=P, Q=Q, R=R, D=D, q_max=qmax, wt=7)
    octx0 = orc.Ctx(fx.workload_instance(a), 0)
    xp, yp = wlmod.random_chromosomes(1, octx0.K, o, seed=1)
    plan = octx0.decode_genes(xp[0], yp[0])
    if case == "K1":   # freeze late enough that exactly one op remains pending
        ends = plan["start"] + P.reshape(-1, o)[np.arange(n * g), plan["assign"]]
        for t in range(int(max(ends)), -1, -1):
            if orc.Ctx(fx.workload_instance(a), t, plan["assign"], plan["start"]).K == 1:
                return a, plan, t
        return None
    rs = plan["makespan"] + 3 if case == "rs_end" else plan["makespan"] // 3
    return a, plan, rs


@pytest.mark.parametrize("case", ["K1", "o1", "g1", "qinf", "q0", "rs_end", "static_ties"])
def test_edge_cases(case, path):
    import zlib
    seed = zlib.crc32(case.encode())
    r = None
    while r is None:
        r = edge_instance(case, seed)
        seed += 1
    a, plan, rs = r
    o = a["o"]
    octx = orc.Ctx(fx.workload_instance(a), rs, plan["assign"], plan["start"])
    st = gpu_state(a, rs, plan["assign"], plan["start"])
    check_gene_order(octx, st)
    if case == "K1":
        assert octx.K == 1
    if octx.K == 0:
        x = np.zeros((4, 1), np.int8)
        y = np.ones((4, 1), np.int16)
        obj, T, M, S = gpu_eval(st, x[:, :0].copy(), y[:, :0].copy(), sched=True)
        r = octx.decode(-np.ones(octx.cells, np.int32), -np.ones(octx.cells, np.int32))
        assert (obj == r["objective"]).all() and (M == r["makespan"]).all()
        assert (S == r["start"]).all()
        return
    x, y = wlmod.random_chromosomes(200, st.K, o, seed=2)
    compare(octx, st, x, y, n_sched=50)


def test_random_population_matches_oracle_init():
    wl = wlmod.config_A2()
    octx, st, arr = both_event_ctx(wl)
    ga = orc.GA(octx, 4, 2, 3, 1, seed=10741)
    ga.step()
    ox, oy, oobj, _ = ga.population()
    xs, ys = [], []
    for I in range(3):
        x, y = ffs.random_population(st, 8, seed=10741, first_id=I << 20)
        xs.append(x.cpu().numpy())
        ys.append(y.cpu().numpy())
    assert (np.concatenate(xs) == ox).all() and (np.concatenate(ys) == oy).all()


def test_evaluate_host_matches_device():
    wl = wlmod.config_B()
    octx, st, arr = both_event_ctx(wl)
    x, y = wlmod.random_chromosomes(256, st.K, wl.o, seed=11)
    obj, T, M = ffs.evaluate_host(st, x, y)
    ref = gpu_eval(st, x, y)
    assert (obj == ref[0]).all() and (T == ref[1]).all() and (M == ref[2]).all()


def test_full_size_sampled_parity(path):
    """Config C at the bench's launch configuration (65,536 Philox chromosomes
    generated on the device); the oracle checks a sample one by one."""
    wl = wlmod.config_C()
    octx, st, arr = both_event_ctx(wl)
    x, y = ffs.random_population(st, 65536, seed=10741)
    obj, T, M, _ = ffs.evaluate(st, x, y)
    torch.cuda.synchronize()
    idx = np.random.default_rng(0).choice(65536, 48, replace=False)
    xs, ys = x.cpu().numpy()[idx], y.cpu().numpy()[idx]
    oo, oT, oM, _ = octx.evaluate_batch(xs, ys, nthreads=8)
    assert (obj.cpu().numpy()[idx] == oo).all()
    assert (T.cpu().numpy()[idx] == oT).all() and (M.cpu().numpy()[idx] == oM).all()
    # every chromosome is a valid permutation (device generator property)
    ysort = torch.sort(y.to(torch.int32), dim=1).values
    assert bool((ysort == torch.arange(1, st.K + 1, device=y.device, dtype=torch.int32)).all())


def test_config_e_million_sampled_parity():
    """Config E's sweep at 1e6 Philox chromosomes on the 100-job instance
    (padded rows, 8 chunks of 2^17 in one call, as bench.py's sweep): every
    chunk's first and last chromosome plus random ones against the oracle,
    one by one; every objective of the population is positive."""
    wl = wlmod.config_C()
    octx, st, arr = both_event_ctx(wl)
    KP = (st.K + 15) // 16 * 16
    n = 1_000_000
    x, y = ffs.random_population(st, n, seed=2024, row=KP)
    obj, T, M, _ = ffs.evaluate(st, x, y)
    torch.cuda.synchronize()
    chunk = 1 << 17
    edges = sorted({i for c in range(0, n, chunk) for i in (c, min(c + chunk, n) - 1)})
    idx = np.array(edges + list(np.random.default_rng(5).choice(n, 32, replace=False)))
    it = torch.as_tensor(idx, device=x.device)
    xs = x.index_select(0, it)[:, :st.K].cpu().numpy()
    ys = y.index_select(0, it)[:, :st.K].cpu().numpy()
    oo, oT, oM, _ = octx.evaluate_batch(np.ascontiguousarray(xs), np.ascontiguousarray(ys), nthreads=8)
    assert (obj.index_select(0, it).cpu().numpy() == oo).all()
    assert (T.index_select(0, it).cpu().numpy() == oT).all() and (M.index_select(0, it).cpu().numpy() == oM).all()
    assert bool((obj > 0).all())


def test_multi_chunk_equals_per_chunk():
    """Above 2^17 chromosomes the lane path runs in chunks (order + decode
    per chunk, the overflow counts reset by the first chunk's order kernel,
    kernels chained by programmatic dependent launch): a 140,000-chromosome
    call (padded rows, as the GA) equals the same rows evaluated in two
    separate calls, and the oracle on a sample across the chunk boundary."""
    wl = wlmod.config_C()
    octx, st, arr = both_event_ctx(wl)
    KP = (st.K + 15) // 16 * 16
    n = 140_000
    x, y = ffs.random_population(st, n, seed=77, row=KP)
    obj, T, M, _ = ffs.evaluate(st, x, y)
    cut = 131_072
    o1, T1, M1, _ = ffs.evaluate(st, x[:cut], y[:cut])
    o2, T2, M2, _ = ffs.evaluate(st, x[cut:], y[cut:])
    torch.cuda.synchronize()
    assert bool((obj == torch.cat([o1, o2])).all()) and bool((T == torch.cat([T1, T2])).all())
    assert bool((M == torch.cat([M1, M2])).all())
    idx = np.concatenate([np.arange(cut - 8, cut + 8), np.random.default_rng(3).choice(n, 16, replace=False)])
    xs, ys = x[:, :st.K].cpu().numpy()[idx], y[:, :st.K].cpu().numpy()[idx]
    oo, oT, oM, _ = octx.evaluate_batch(xs, ys, nthreads=8)
    assert (obj.cpu().numpy()[idx] == oo).all()
    assert (T.cpu().numpy()[idx] == oT).all() and (M.cpu().numpy()[idx] == oM).all()


@pytest.mark.parametrize("g,n,o,q_max", [(16, 12, 3, 5), (40, 5, 2, 4), (70, 3, 2, 3)])
def test_long_jobs(g, n, o, q_max, path):
    """Jobs with up to G pending genes span more lanes of the order kernel's
    tiles: G = 16 and 40 take the 3- and 5-step segmented min-scans (G <= 13
    takes 2), G = 70 lets one job cover a whole 128-gene tile boundary."""
    wl = wlmod.gen_v1(f"G{g}", n, g, o, q_max, arrivals_per_event=[2], ratios=[0.3], seed=g)
    octx, st, arr = both_event_ctx(wl)
    check_gene_order(octx, st)
    x, y = wlmod.random_chromosomes(300, st.K, wl.o, seed=13)
    compare(octx, st, x, y, n_sched=20)


@pytest.mark.parametrize("g,n,lane", [(70, 3, True), (70, 9, False), (128, 1, True)])
def test_order_key_bound(g, n, lane):
    """The order kernel keeps u = K - pm and g - g_L (< max_pending) in one u16
    per gene, u in the low ceil(log2 K) bits: the lane path is taken only when
    max_pending <= 2^(16 - ceil(log2 K)).  Jobs of 70 stages: at K <= 256 the
    offsets fit (the lane path, one job spanning tile boundaries), at K ~ 600
    they do not (the general kernel); jobs of 128 stages at 256 < K <= 512:
    max_pending = 128 = 2^7 exactly, every offset bit in use (lane path); all
    equal the oracle."""
    wl = wlmod.gen_v1(f"G{g}n{n}", n, g, 2, 3, arrivals_per_event=[2], ratios=[0.3], seed=g + n)
    octx, st, arr = both_event_ctx(wl)
    p = st.path()
    ub = max(1, (st.K - 1).bit_length())
    assert p["max_pending"] > 32 and p["lane_mode"] == 2
    if g == 128:
        assert p["max_pending"] == 128 and 256 < st.K <= 512
    assert p["lane_path"] == lane == (p["max_pending"] <= 2 ** (16 - ub))
    check_gene_order(octx, st)
    x, y = wlmod.random_chromosomes(200, st.K, wl.o, seed=23)
    compare(octx, st, x, y)


@pytest.mark.parametrize("q_max,power", [(4, "one"), (7, "u13")])
def test_long_processing_times_warp_path(q_max, power):
    """P_sm ~ U{9..40} (above the lane decoder's P <= 8): the warp-per-
    chromosome kernel with runs longer than one 32-tick ballot window
    (evaluate.cu multi-window run logic), uniform and general power."""
    wl = wlmod.gen_v1("Plong", 14, 5, 3, q_max, arrivals_per_event=[4], ratios=[0.3], seed=40 + q_max,
                      power=power, p_range=(9, 40))
    assert wl.P.min() >= 9 and wl.P.max() > 32
    octx, st, arr = both_event_ctx(wl)
    check_gene_order(octx, st)
    x, y = wlmod.random_chromosomes(400, st.K, wl.o, seed=19)
    compare(octx, st, x, y)


@pytest.mark.parametrize("n,g", [(16, 8), (32, 8), (43, 6), (16, 16), (65, 4)])
def test_tile_boundary_K(n, g, path):
    """Static problems (RS = 0, K = n g) with K = 128, 256, 258, 256, 260:
    full and partial 128-gene tiles, 256-entry prefix-sum steps and the last
    quad of ranks."""
    wl = wlmod.gen_v1(f"K{n * g}", n, g, 3, 6, seed=n + g)
    a = wl.original_instance()
    octx = orc.Ctx(fx.workload_instance(a), 0)
    st = gpu_state(a, 0)
    assert st.K == n * g
    x, y = wlmod.random_chromosomes(200, st.K, 3, seed=17)
    compare(octx, st, x, y, n_sched=20)


@pytest.mark.parametrize("pad", [0, 16])
def test_long_rows_K1000(pad, path):
    """K = 1000 (100 jobs x 10 stages, RS = 0): the order kernel's x staging
    does not fit beside its histograms, so the lane path takes the unstaged
    variant; compact and 16-padded (TMA) rows."""
    wl = wlmod.gen_v1("Cs", 100, 10, 4, 10, seed=1903)
    a = wl.original_instance()
    octx = orc.Ctx(fx.workload_instance(a), 0)
    st = gpu_state(a, 0)
    assert st.K == 1000
    x, y = wlmod.random_chromosomes(160, st.K, 4, seed=31)
    if pad:
        R = (st.K + pad - 1) // pad * pad
        xp = np.zeros((len(x), R), np.int8)
        yp = np.zeros((len(y), R), np.int16)
        xp[:, :st.K] = x
        yp[:, :st.K] = y
        got = gpu_eval(st, xp, yp)
        oo, oT, oM, _ = octx.evaluate_batch(x, y, nthreads=8)
        assert (got[0] == oo).all() and (got[1] == oT).all() and (got[2] == oM).all()
    else:
        compare(octx, st, x, y, n_sched=8)


@pytest.mark.parametrize("q,q_max", [(1, 20), (2, 40), (3, 50), (2, 9), (3, 40), (4, 7)])
def test_uniform_power(q, q_max, path):
    """Uniform Q = q: Q_max / q <= 15 takes mode 2 (headroom counted in ops of
    power q; (2, 9), (3, 40), (4, 7): fractional remainders of Q_max / q),
    larger ratios the byte-level mode 1."""
    wl = wlmod.gen_v1(f"U{q}", 20, 5, 3, q_max, arrivals_per_event=[5], ratios=[0.3], seed=40 + q)
    arr = wl.original_instance()
    arr = dict(arr, Q=np.full_like(arr["Q"], q))
    octx = orc.Ctx(fx.workload_instance(arr), 0)
    st = gpu_state(arr, 0)
    x, y = wlmod.random_chromosomes(300, st.K, wl.o, seed=19)
    compare(octx, st, x, y, n_sched=20)


@pytest.mark.parametrize("count", [16500, 33001])
def test_evaluate_host_chunked_pipeline(count):
    """ffs_evaluate_host splits large batches into 2 or 4 uneven chunks on two
    internal streams; results equal the device call."""
    wl = wlmod.config_A2()
    octx, st, arr = both_event_ctx(wl)
    x, y = wlmod.random_chromosomes(count, st.K, wl.o, seed=23)
    obj, T, M = ffs.evaluate_host(st, x, y)
    ref = gpu_eval(st, x, y)
    assert (obj == ref[0]).all() and (T == ref[1]).all() and (M == ref[2]).all()
    idx = np.random.default_rng(1).choice(count, 64, replace=False)
    oo, oT, oM, _ = octx.evaluate_batch(x[idx], y[idx])
    assert (obj[idx] == oo).all() and (T[idx] == oT).all() and (M[idx] == oM).all()


@pytest.mark.parametrize("pad", [16, 5])
def test_strided_rows_match_compact(pad, path):
    """ffs_evaluate_strided: rows padded to a multiple of 16 genes (TMA row
    staging) or by an odd amount (element loads) give the compact results."""
    wl = wlmod.config_B()
    octx, st, arr = both_event_ctx(wl)
    x, y = wlmod.random_chromosomes(700, st.K, wl.o, seed=29)
    R = (st.K + 15) // 16 * 16 if pad == 16 else st.K + pad
    xp = np.zeros((len(x), R), np.int8)
    yp = np.zeros((len(y), R), np.int16)
    xp[:, :st.K] = x
    yp[:, :st.K] = y
    ref = gpu_eval(st, x, y, sched=True)
    got = gpu_eval(st, xp, yp, sched=True)
    for u, v in zip(ref, got):
        assert (u == v).all()
    compare(octx, st, x[:60], y[:60], n_sched=10)


@pytest.mark.parametrize("R", [1024, 2048])
def test_wide_padded_rows_config_c(R, path):
    """Rows much wider than K (K = 855 in rows of 1,024 / 2,048 genes, 16-B
    aligned: the TMA row staging) -- the staging copies ceil16(K) genes, never
    the whole row, so it cannot overrun the per-warp slots."""
    wl = wlmod.config_C()
    octx, st, arr = both_event_ctx(wl)
    x, y = wlmod.random_chromosomes(200, st.K, wl.o, seed=31)
    xp = np.full((len(x), R), 3, np.int8)     # junk in the padding
    yp = np.full((len(y), R), 7, np.int16)
    xp[:, :st.K] = x
    yp[:, :st.K] = y
    got = gpu_eval(st, xp, yp, sched=True)
    oo, oT, oM, oS = octx.evaluate_batch_schedule(x, y, nthreads=8)
    assert (got[0] == oo).all() and (got[1] == oT).all() and (got[2] == oM).all()
    assert (got[3] == oS).all()


def test_random_population_strided_equals_compact():
    wl = wlmod.config_B()
    octx, st, arr = both_event_ctx(wl)
    x, y = ffs.random_population(st, 100, seed=77, first_id=5)
    R = st.K + 13
    xp, yp = ffs.random_population(st, 100, seed=77, first_id=5, row=R)
    assert (xp[:, :st.K] == x).all() and (yp[:, :st.K] == y).all()
    assert (xp[:, st.K:] == 0).all() and (yp[:, st.K:] == 0).all()


def test_strided_row_shorter_than_K_is_rejected():
    wl = wlmod.config_A2()
    octx, st, arr = both_event_ctx(wl)
    x = torch.zeros((4, st.K - 1), dtype=torch.int8, device=DEV)
    y = torch.zeros((4, st.K - 1), dtype=torch.int16, device=DEV)
    with pytest.raises(ffs.FFSError):
        ffs.evaluate(st, x, y)
    with pytest.raises(ffs.FFSError):
        ffs.random_population(st, 4, seed=1, row=st.K - 1)


def test_evaluate_host_long_rows_through_overflows():
    """K = 1,000 through ffs_evaluate_host (4 chunks on two streams): ~1% of
    the chromosomes overflow the lane horizon (416 ticks) and are re-decoded
    (the general fallback on the first call, the LIST re-decode after); the
    host results equal the device call and, on the overflowed chromosomes
    and a random sample, the oracle."""
    wl = wlmod.gen_v1("Cs", 100, 10, 4, 10, seed=1903)
    a = wl.original_instance()
    octx = orc.Ctx(fx.workload_instance(a), 0)
    st = gpu_state(a, 0)
    cap = st.info()["horizon_cap"]
    x, y = wlmod.random_chromosomes(33001, st.K, 4, seed=41)
    for _ in range(2):   # first call: fallback only; second: the state has seen an overflow
        obj, T, M = ffs.evaluate_host(st, x, y)
        ref = gpu_eval(st, x, y)
        assert (obj == ref[0]).all() and (T == ref[1]).all() and (M == ref[2]).all()
    over = np.flatnonzero(M > cap)
    assert len(over) > 0
    idx = np.concatenate([over[:48], np.random.default_rng(2).choice(len(x), 16, replace=False)])
    oo, oT, oM, _ = octx.evaluate_batch(x[idx], y[idx], nthreads=8)
    assert (obj[idx] == oo).all() and (T[idx] == oT).all() and (M[idx] == oM).all()
