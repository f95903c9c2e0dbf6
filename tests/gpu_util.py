"""Helpers shared by the GPU parity tests (test-only)."""
import numpy as np

from oracle import oracle as orc
from paper_1903_10741_b200 import ffs
from tests import fixtures as fx


def gpu_state(arrs, rs, oa=None, os_=None, device=0, static=False):
    inst = ffs.Instance.from_arrays(arrs, device=device)
    st = ffs.make_state(inst, rs, oa, os_, static=static)
    st._inst_ref = inst
    return st


def both_event_ctx(wl, static=False):
    """Each side builds the event-0 context independently (plan decode on its
    own decoder); the plans must agree exactly."""
    octx, arr, oplan, ors = fx.oracle_event_ctx(wl, static=static)
    base = wl.original_instance()
    st0 = gpu_state(base, 0)
    assign, start, obj, T, M = ffs.decode_schedule(st0, wl.plan_x, wl.plan_y)
    rs = wl.rs_from_makespan(wl.ratios[0], M)
    assert rs == ors and M == oplan["makespan"]
    assert (start == oplan["start"]).all() and (assign == oplan["assign"]).all()
    arr_g = wl.instance_at(0, [rs])
    st = gpu_state(arr_g, rs, assign[: wl.n * wl.g], start[: wl.n * wl.g], static=static)
    return octx, st, arr


def check_gene_order(octx, st):
    jj, ss = st.genes()
    g = octx.inst.g
    assert st.K == octx.K
    assert (jj * g + ss == octx.pending_cells).all()
    assert (st.cell_states().reshape(octx.states.shape) == octx.states).all()
