"""GPU brute-force enumerator against the oracle's brute force:
same optimum over o^K x linear extensions, same enumeration count, and the
returned chromosome decodes (oracle) to that optimum; the Fig. 7 static
optimum; the GA never beats the exhaustive optimum."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from paper_1903_10741_b200 import workload as wlmod
from tests import fixtures as fx
from tests.gpu_util import gpu_state
from tests.test_oracle_properties import random_ctx

pytestmark = pytest.mark.gpu


def test_fig7_static_optimum_on_gpu(path):
    d, a = fx.table4_arrays()
    a = dict(a, wt=0)
    oa, os_ = np.array(d["orig_assign"]), np.array(d["orig_start"])
    st = gpu_state(a, d["rs"], oa, os_, static=True)
    best, ev, bx, by = ffs.brute_force(st)
    assert best == 1991 and ev == 2 ** 6 * 20          # Fig. 7 caption
    octx = orc.Ctx(fx.workload_instance(a), d["rs"], oa, os_, static=True)
    assert octx.decode_genes(bx, by)["objective"] == 1991


@pytest.mark.parametrize("case", [(3, 1, 2, 2, 2, 1, 5), (4, 2, 3, 2, 3, 1, 5), (3, 2, 2, 3, 2, 2, 6),
                                  (2, 2, 3, 2, 1, 1, 4)])
def test_brute_force_matches_oracle(case, path):
    n, n_p, g, o, q_max, pw, pmax = case
    rng = np.random.default_rng(sum(case) * 31 + 7)
    done = 0
    while done < 3:
        inst, octx, plan = random_ctx(rng, n, n_p, g, o, q_max, pw, pmax=pmax, rs_ratio=rng.uniform(0.1, 0.5))
        if octx.K == 0 or octx.K > (8 if o == 2 else 6):
            continue
        a = dict(n=inst.n, n_prime=inst.n_prime, g=inst.g, o=inst.o, P=inst.P, Q=inst.Q, R=inst.R, D=inst.D,
                 q_max=inst.q_max, wt=inst.wt)
        st = gpu_state(a, octx.rs, octx._oa, octx._os)
        best, ev, bx, by = ffs.brute_force(st)
        obest, oev, _, _ = octx.brute_force()
        assert (best, ev) == (obest, oev)
        assert octx.decode_genes(bx, by)["objective"] == best
        done += 1


def test_real_weight_brute_force(path):
    d, a = fx.table4_arrays()
    oa, os_ = np.array(d["orig_assign"]), np.array(d["orig_start"])
    st = gpu_state(a, d["rs"], oa, os_, static=True)
    st.set_objective_weight(0.37)
    best, ev, bx, by = ffs.brute_force(st)
    octx = orc.Ctx(fx.workload_instance(a), d["rs"], oa, os_, static=True)
    octx.set_real_weight(0.37)
    assert octx.decode_genes(bx, by)["value"] == best
    x, y = wlmod.random_chromosomes(3000, st.K, 2, seed=3)
    vals, _, _, _ = octx.evaluate_batch(x, y)
    assert best <= vals.min()


def test_limit_and_k0_errors():
    d, a = fx.table4_arrays()
    st = gpu_state(a, d["rs"], np.array(d["orig_assign"]), np.array(d["orig_start"]))
    with pytest.raises(ffs.FFSError):
        ffs.brute_force(st, limit=10 ** 6)          # K = 13: 2^13 * 21,621,600 decodes


def test_ga_never_beats_exhaustive_optimum():
    wl = wlmod.gen_v1("bf", 5, 2, 2, 2, seed=12)
    st = gpu_state(wl.original_instance(), 0)
    assert st.K == 10
    best, ev, _, _ = ffs.brute_force(st)
    assert ev == 2 ** 10 * 113400                    # 10!/(2!)^5 interleavings
    run = ffs.Run(st, 8, 8, 4, 40, 99)
    run.step(40)
    b = run.best()
    assert b["objective"] >= best
