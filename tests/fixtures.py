"""Golden fixtures (tests/golden/*.json) as oracle instances.  Test-only."""
import json
import os

import numpy as np

from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def table4_arrays():
    d = load("table4.json")
    NJ, g, o = d["n"] + d["n_prime"], d["g"], d["o"]
    P = np.zeros((NJ, g, o), np.int32)
    for s in range(g):
        P[:, s, :] = d["proc_time_per_stage"][s]
    Q = np.full((NJ, g, o), d["power"], np.int32)
    R = np.array(d["release"], np.int32)
    D = R + 1200  # assumption, see fixture ("due_assumed")
    return d, dict(n=d["n"], n_prime=d["n_prime"], g=g, o=o, P=P, Q=Q, R=R, D=D,
                   q_max=d["q_max"], wt=d["wt"])


def table4_ctx():
    d, a = table4_arrays()
    inst = orc.Instance(**a)
    return d, inst, orc.Ctx(inst, d["rs"], np.array(d["orig_assign"]), np.array(d["orig_start"]))


def printed_Z(d):
    return np.array([[orc.Z_COMPLETED if v == "C" else v for v in row] for row in d["Z_printed"]],
                    np.int32)


def h3():
    d = load("h3.json")
    NJ, g, o = d["n"], d["g"], d["o"]
    P = np.array(d["P"], np.int32)
    Q = np.full((NJ, g, o), d["Q"], np.int32)
    inst = orc.Instance(d["n"], 0, g, o, P, Q, np.array(d["release"], np.int32),
                        np.array(d["due"], np.int32), d["q_max"], d["wt"])
    return d, inst, orc.Ctx(inst, 0)


def operators_ctx():
    d = load("operators.json")
    c = d["ctx"]
    n, g, o = c["n"], c["g"], c["o"]
    P = np.ones((n, g, o), np.int32)
    Q = np.ones((n, g, o), np.int32)
    R = np.zeros(n, np.int32)
    D = np.full(n, 10, np.int32)
    inst = orc.Instance(n, 0, g, o, P, Q, R, D, c["q_max"], 100)
    return d, orc.Ctx(inst, c["rs"], np.array(c["orig_assign"]), np.array(c["orig_start"]))


def workload_instance(arrs):
    return orc.Instance(arrs["n"], arrs["n_prime"], arrs["g"], arrs["o"], arrs["P"], arrs["Q"],
                        arrs["R"], arrs["D"], arrs["q_max"], arrs["wt"])


def oracle_event_ctx(wl, e=0, static=False):
    """Oracle-side construction of a workload's rescheduling context at event 0:
    decode the recorded plan chromosome at RS = 0 with the ORACLE, take
    RS = floor(ratio * C_max), freeze (static=True: the traditional static
    approach's context instead)."""
    base = wl.original_instance()
    c0 = orc.Ctx(workload_instance(base), 0)
    X, Y = c0.to_matrix(wl.plan_x, wl.plan_y)
    plan = c0.decode(X, Y)
    rs = wl.rs_from_makespan(wl.ratios[0], plan["makespan"])
    arr = wl.instance_at(0, [rs])
    ctx = orc.Ctx(workload_instance(arr), rs, plan["assign"][: wl.n * wl.g],
                  plan["start"][: wl.n * wl.g], static=static)
    return ctx, arr, plan, rs
