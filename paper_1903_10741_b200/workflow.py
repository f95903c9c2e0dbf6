"""Predictive-reactive complete rescheduling (§4.1, Fig. 2).

Host glue over the C-ABI: plan the original jobs (island GA at RS = 0), then for
every new-job-arrival event e freeze the current plan at RS_e
(`ffs_reschedule_state`), re-optimise every pending operation of the original
jobs together with the new jobs (`ffs_evolve`), and merge the frozen part with
the best schedule found (`ffs_best`): that merged plan is the "original plan"
of the next event (reading R26).  RS_e = floor(ratio_e * C_max(original plan))
(P:373-375).  Every step of the method runs in the sm_100a library; this module
only sequences calls.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import ffs
from .workload import Workload


@dataclass
class EventResult:
    event: int
    rs: int
    K: int
    objective: int
    sum_tardiness: int
    makespan: int
    assign: np.ndarray
    start: np.ndarray
    trace_min: np.ndarray
    trace_sum: np.ndarray
    seconds: float


@dataclass
class WorkflowResult:
    plan: EventResult
    events: List[EventResult] = field(default_factory=list)


def _evolve(st, shape, generations, seed, stream=None) -> EventResult:
    w, h, islands = shape
    t0 = time.perf_counter()
    run = ffs.Run(st, w, h, islands, generations, seed, stream=stream)
    run.step(generations)
    b = run.best()
    dt = time.perf_counter() - t0
    return EventResult(event=-1, rs=st.rs, K=st.K, objective=b["objective"], sum_tardiness=b["sum_tardiness"],
                       makespan=b["makespan"], assign=b["assign"], start=b["start"], trace_min=b["trace_min"],
                       trace_sum=b["trace_sum"], seconds=dt)


def run_events(wl: Workload, shape=(16, 8, 64), generations: int = 100, seed: int = 10741,
               device: int = 0, stream=None) -> WorkflowResult:
    """Config B workflow: plan at RS = 0, then one rescheduling per event."""
    base = ffs.Instance.from_arrays(wl.original_instance(), device=device)
    st0 = ffs.make_state(base, 0)
    plan = _evolve(st0, shape, generations, seed, stream)
    plan.event = 0
    res = WorkflowResult(plan=plan)
    c_plan = plan.makespan
    rs_list: List[int] = []
    cur_assign, cur_start = plan.assign, plan.start
    keep = [base, st0]
    for e in range(wl.n_events):
        rs = wl.rs_from_makespan(wl.ratios[e], c_plan)
        rs_list.append(rs)
        arr = wl.instance_at(e, rs_list)
        inst = ffs.Instance.from_arrays(arr, device=device)
        st = ffs.make_state(inst, rs, cur_assign, cur_start)
        ev = _evolve(st, shape, generations, seed + 1 + e, stream) if st.K > 0 else None
        if ev is None:   # nothing pending: the frozen plan stands
            assign, start, obj, T, M = ffs.decode_schedule(st, np.zeros(0, np.int8), np.zeros(0, np.int16))
            ev = EventResult(-1, rs, 0, obj, T, M, assign, start, np.zeros(0, np.int64), np.zeros(0, np.int64), 0.0)
        ev.event = e + 1
        res.events.append(ev)
        cur_assign, cur_start = ev.assign, ev.start
        keep += [inst, st]
    return res


# ---------------------------------------------------------------------------
# Dynamic vs static comparison (Table 10 design)
# ---------------------------------------------------------------------------
@dataclass
class PolicyRow:
    ratio: float
    n_prime: int
    static_mean: float
    dynamic_mean: float
    improvement_ratio: float
    runs: List[dict]


def test3_workload(ratio: float, seed: int, n: int = 10, g: int = 3, o: int = 2, q_max: int = 4) -> Workload:
    """Test 3's instance (10 original jobs, 3 stages, 2 machines, Q_max 4)
    with n' = round(ratio * n) arrivals (reading R31)."""
    from .workload import gen_v1
    return gen_v1("T10", n, g, o, q_max, arrivals_per_event=[int(round(ratio * n))], ratios=[ratio], seed=seed)


def compare_policies(ratios=(0.2, 0.4, 0.6, 0.8), seeds=(1903,), shape=(8, 8, 64), generations: int = 100,
                     device: int = 0, make_workload=test3_workload, stream=None) -> List[PolicyRow]:
    """For every seed: plan the original jobs (island GA at RS = 0, the
    "original schedule of an optimized solution", Fig. 6); for every ratio take
    RS = floor(ratio * C_max(plan)), then optimise the same arrivals with the
    predictive-reactive policy (ffs_reschedule_state) and with the traditional
    static policy (ffs_static_state), same GA seed.  improvement ratio =
    mean static objective / mean dynamic objective (Table 10's last column)."""
    rows = []
    plans = {}
    for ratio in ratios:
        runs = []
        for seed in seeds:
            wl = make_workload(ratio, seed)
            base_arr = wl.original_instance()
            key = (seed, base_arr["P"].tobytes(), base_arr["R"].tobytes(), base_arr["D"].tobytes())
            if key not in plans:
                base = ffs.Instance.from_arrays(base_arr, device=device)
                st0 = ffs.make_state(base, 0)
                plans[key] = (_evolve(st0, shape, generations, seed, stream), base, st0)
            plan = plans[key][0]
            rs = wl.rs_from_makespan(ratio, plan.makespan)
            arr = wl.instance_at(0, [rs])
            inst = ffs.Instance.from_arrays(arr, device=device)
            n_g = wl.n * wl.g
            res = {}
            for name, static in (("dynamic", False), ("static", True)):
                st = ffs.make_state(inst, rs, plan.assign[:n_g], plan.start[:n_g], static=static)
                ev = _evolve(st, shape, generations, seed + 1, stream)
                res[name] = ev
            runs.append(dict(seed=seed, rs=rs, plan_makespan=plan.makespan, K_dynamic=res["dynamic"].K,
                             K_static=res["static"].K, dynamic=res["dynamic"].objective,
                             static=res["static"].objective, dynamic_result=res["dynamic"],
                             static_result=res["static"]))
        sm = float(np.mean([r["static"] for r in runs]))
        dm = float(np.mean([r["dynamic"] for r in runs]))
        rows.append(PolicyRow(ratio=ratio, n_prime=int(wl.arr_event.size), static_mean=sm, dynamic_mean=dm,
                              improvement_ratio=sm / dm if dm > 0 else float("inf"), runs=runs))
    return rows


# ---------------------------------------------------------------------------
# WT sensitivity (Table 11)
# ---------------------------------------------------------------------------
TABLE11_WT = (0.01, 0.1, 0.4, 0.7, 1.0, 4.0, 7.0, 10.0, 100.0)


@dataclass
class WeightRow:
    wt: float
    tardiness_mean: float
    makespan_mean: float
    objective_mean: float
    runs: List[dict]


def wt_sweep(wts=TABLE11_WT, seeds=(1903,), ratio: float = 0.5, shape=(8, 8, 64), generations: int = 100,
             device: int = 0, make_workload=test3_workload, stream=None) -> List[WeightRow]:
    """For every seed: plan the originals with the instance's integer WT (GA at
    RS = 0), freeze at RS = floor(ratio * C_max) (reading R32), then for every
    WT of the grid re-optimise with the fractional objective
    fl(fl(WT * sum T) + C_max) (ffs_state_set_objective_weight) and record the
    best schedule's sum T, C_max and objective (Table 11's columns)."""
    rows = []
    ctxs = []
    for seed in seeds:
        wl = make_workload(ratio, seed)
        base = ffs.Instance.from_arrays(wl.original_instance(), device=device)
        st0 = ffs.make_state(base, 0)
        plan = _evolve(st0, shape, generations, seed, stream)
        rs = wl.rs_from_makespan(ratio, plan.makespan)
        inst = ffs.Instance.from_arrays(wl.instance_at(0, [rs]), device=device)
        n_g = wl.n * wl.g
        ctxs.append((seed, rs, inst, plan.assign[:n_g], plan.start[:n_g], base, st0))
    for wt in wts:
        runs = []
        for seed, rs, inst, oa, os_, _, _ in ctxs:
            st = ffs.make_state(inst, rs, oa, os_)
            st.set_objective_weight(wt)
            ev = _evolve(st, shape, generations, seed + 1, stream)
            runs.append(dict(seed=seed, rs=rs, K=ev.K, objective=ev.objective, sum_tardiness=ev.sum_tardiness,
                             makespan=ev.makespan, result=ev))
        rows.append(WeightRow(wt=float(wt), tardiness_mean=float(np.mean([r["sum_tardiness"] for r in runs])),
                              makespan_mean=float(np.mean([r["makespan"] for r in runs])),
                              objective_mean=float(np.mean([r["objective"] for r in runs])), runs=runs))
    return rows
