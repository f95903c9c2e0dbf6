"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no freeze, order, decode,
objective or GA step): only random draws that follow the paper's
experimental data recipe (Table 5) in integer ticks, and the
workload configurations of BASELINE.json.  Both sides compute everything
else independently.

Recipe "gen-v1":
  * P_sm ~ U{1..5}, shared by every job: "P_0sm = P_1sm = ...";
    stored as [j][s][m].
  * Q == 1.  Variant power="u13": Q_jsm ~ U{1..3} exercises the
    general power path.
  * Pbar = sum_s mean_m P_sm.
  * original jobs: R_j ~ U{0..floor(Pbar)};
    every job: D_j = R_j + floor(Pbar * (1 + sigma_j)), sigma_j ~ U[0, 2).
  * arrival jobs of event e: R_j = RS_e + U{0..floor(Pbar)}.
  * the original plan is the decode, at RS = 0, of the recorded random
    chromosome (plan_x, plan_y) over the original jobs -- each side decodes it
    with its own decoder; RS_e = floor(ratio_e * C_max(plan)).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np


@dataclass
class Workload:
    name: str
    n: int                      # original jobs
    g: int
    o: int
    q_max: int
    wt: int
    P: np.ndarray               # [n_total, g, o] int32 (all jobs incl. every arrival)
    Q: np.ndarray               # [n_total, g, o] int32
    R_orig: np.ndarray          # [n] int32
    slack: np.ndarray           # [n_total] int32: D_j - R_j
    arr_offset: np.ndarray      # [n_arr] int32: R_j - RS_event
    arr_event: np.ndarray       # [n_arr] int32: event index of each arrival
    ratios: List[float]         # RS_e / C_max(plan) per event
    plan_x: np.ndarray          # [n*g] int8   machine of each original op
    plan_y: np.ndarray          # [n*g] int16  permutation of 1..n*g
    seed: int
    meta: dict = field(default_factory=dict)

    @property
    def n_events(self) -> int:
        return len(self.ratios)

    def jobs_at_event(self, e: int) -> int:
        """Jobs (originals + arrivals of events <= e) known at event e."""
        return self.n + int(np.sum(self.arr_event <= e))

    def original_instance(self):
        """Arrays of the static problem over the original jobs only (RS = 0)."""
        n = self.n
        R = self.R_orig.astype(np.int32)
        D = (R + self.slack[:n]).astype(np.int32)
        return dict(n=n, n_prime=0, g=self.g, o=self.o, P=self.P[:n].copy(), Q=self.Q[:n].copy(),
                    R=R, D=D, q_max=self.q_max, wt=self.wt)

    def instance_at(self, e: int, rs_list: Sequence[int], n_prev: int | None = None):
        """Instance of event e given the rescheduling points of events 0..e.

        Jobs of events < e are the 'original' jobs J of event e (their plan is
        the previous event's merged schedule, R26); arrivals of event e are J'.
        """
        NJ = self.jobs_at_event(e)
        n_orig = self.jobs_at_event(e - 1) if e > 0 else self.n
        R = np.zeros(NJ, dtype=np.int64)
        R[:self.n] = self.R_orig
        for a in range(NJ - self.n):
            R[self.n + a] = int(rs_list[self.arr_event[a]]) + int(self.arr_offset[a])
        D = R + self.slack[:NJ]
        return dict(n=n_orig, n_prime=NJ - n_orig, g=self.g, o=self.o, P=self.P[:NJ].copy(),
                    Q=self.Q[:NJ].copy(), R=R.astype(np.int32), D=D.astype(np.int32),
                    q_max=self.q_max, wt=self.wt)

    @staticmethod
    def rs_from_makespan(ratio: float, makespan: int) -> int:
        """RS = floor(ratio * C_max(original plan))."""
        return int(np.floor(ratio * makespan))


def gen_v1(name: str, n: int, g: int, o: int, q_max: int, *, arrivals_per_event: Sequence[int] = (),
           ratios: Sequence[float] = (), wt: int = 100, seed: int = 1903, power: str = "one",
           p_range: Sequence[int] = (1, 5)) -> Workload:
    """p_range: P_sm ~ U{lo..hi}; the paper's (1, 5) by default (Table 5)."""
    rng = np.random.default_rng(seed)
    Psm = rng.integers(int(p_range[0]), int(p_range[1]) + 1, size=(g, o))   # U{1..5}
    n_arr = int(sum(arrivals_per_event))
    NT = n + n_arr
    P = np.broadcast_to(Psm, (NT, g, o)).astype(np.int32).copy()
    if power == "one":
        Q = np.ones((NT, g, o), dtype=np.int32)                         # Q = 1
    elif power == "u13":
        Q = rng.integers(1, 4, size=(NT, g, o)).astype(np.int32)
    else:
        raise ValueError(power)
    pbar = float(Psm.mean(axis=1).sum())
    fp = int(np.floor(pbar))
    R_orig = rng.integers(0, fp + 1, size=n).astype(np.int32)           # U[0, Pbar]
    sigma = rng.uniform(0.0, 2.0, size=NT)                              # sigma ~ U[0, 2]
    slack = np.floor(pbar * (1.0 + sigma)).astype(np.int32)             # D - R = Pbar (1 + sigma)
    arr_offset = rng.integers(0, fp + 1, size=n_arr).astype(np.int32)
    arr_event = np.repeat(np.arange(len(arrivals_per_event)), arrivals_per_event).astype(np.int32)
    plan_x = rng.integers(0, o, size=n * g).astype(np.int8)
    plan_y = (rng.permutation(n * g) + 1).astype(np.int16)
    return Workload(name=name, n=n, g=g, o=o, q_max=q_max, wt=wt, P=P, Q=Q, R_orig=R_orig,
                    slack=slack, arr_offset=arr_offset, arr_event=arr_event, ratios=list(ratios),
                    plan_x=plan_x, plan_y=plan_y, seed=seed, meta=dict(pbar=pbar))


def random_chromosomes(count: int, K: int, o: int, seed: int):
    """count random compact chromosomes: x ~ U{0..o-1}, y = random permutation of 1..K."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, o, size=(count, K)).astype(np.int8)
    y = (np.argsort(rng.random((count, K)), axis=1) + 1).astype(np.int16)
    return x, y


# ---------------------------------------------------------------------------
# BASELINE.json configurations; GA shapes per config.
# ---------------------------------------------------------------------------
def config_A2(seed: int = 1903) -> Workload:
    """Config A (ii): gen-v1(n=6, g=3, o=2, Q_max=3) + 2 arrivals at ratio 0.45."""
    return gen_v1("A2", 6, 3, 2, 3, arrivals_per_event=[2], ratios=[0.45], seed=seed)


def config_B(seed: int = 1903) -> Workload:
    """Config B: gen-v1(n=30, g=5, o=3, Q_max=5), 3 events at 0.25/0.50/0.75, 7 arrivals each."""
    return gen_v1("B", 30, 5, 3, 5, arrivals_per_event=[7, 7, 7], ratios=[0.25, 0.50, 0.75],
                  seed=seed)


def config_C(seed: int = 1903, power: str = "one") -> Workload:
    """Config C: gen-v1(n=80 + n'=20 at ratio 0.25, g=10, o=4, Q_max=10) -- the 100-job config."""
    return gen_v1("C", 80, 10, 4, 10, arrivals_per_event=[20], ratios=[0.25], seed=seed, power=power)


GA_SHAPES = {
    # name: (island_w, island_h, islands, generations)
    "A": (8, 8, 1, 50),
    "B": (16, 8, 64, 100),
    "C": (16, 16, 256, 100),
    "D": (16, 16, 2048, 100),
}
