"""Thin Python binding of the C-ABI (include/ffs.h) -- argument marshalling only.

Every step of the hot path runs in libffs.so's sm_100a kernels.  PyTorch is
used only for device memory and streams.  There is no fallback: importing
works without a GPU (for the build check), but every call requires the
compiled library and a CUDA device and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

OK = 0
STATUS = {0: "FFS_OK", 1: "FFS_ERR_INVALID_ARG", 2: "FFS_ERR_INFEASIBLE", 3: "FFS_ERR_INVALID_SCHEDULE",
          4: "FFS_ERR_CUDA", 5: "FFS_ERR_OOM", 6: "FFS_ERR_COMM"}

XO_090 = 3865470566   # floor(0.9 * 2^32), crossover rate of P:395
MUT_010 = 429496729   # floor(0.1 * 2^32), mutation rate of P:395

# every entry point declared in include/ffs.h
EXPORTS = [
    "ffs_last_error", "ffs_version", "ffs_instance_create", "ffs_instance_destroy",
    "ffs_reschedule_state", "ffs_static_state", "ffs_state_genes", "ffs_state_cells", "ffs_state_cut_table",
    "ffs_state_set_horizon_cap", "ffs_state_set_objective_weight", "ffs_state_info", "ffs_state_path", "ffs_state_destroy", "ffs_evaluate",
    "ffs_evaluate_host", "ffs_evaluate_strided", "ffs_brute_force", "ffs_random_population", "ffs_random_population_strided", "ffs_evolve_begin", "ffs_evolve_step",
    "ffs_evolve", "ffs_best", "ffs_run_population", "ffs_run_history", "ffs_run_info", "ffs_run_restore",
    "ffs_run_destroy",
]


class FFSError(RuntimeError):
    def __init__(self, status, what, msg):
        super().__init__(f"{what}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class _Desc(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_prime", C.c_int32), ("g", C.c_int32), ("o", C.c_int32),
                ("proc_time", C.POINTER(C.c_int32)), ("power", C.POINTER(C.c_int32)),
                ("release", C.POINTER(C.c_int32)), ("due", C.POINTER(C.c_int32)),
                ("q_max", C.c_int32), ("wt", C.c_int64)]


ALLRED = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class GAConfig(C.Structure):
    _fields_ = [("island_w", C.c_int32), ("island_h", C.c_int32), ("islands_total", C.c_int32),
                ("island_begin", C.c_int32), ("island_end", C.c_int32),
                ("xo_threshold", C.c_uint32), ("mut_threshold", C.c_uint32),
                ("migration_interval", C.c_int32), ("generations", C.c_int32),
                ("seed", C.c_uint64), ("rank", C.c_int32), ("world", C.c_int32),
                ("allreduce_max_i64", ALLRED), ("allgather", ALLGATHER), ("user", C.c_void_p)]


_lib = None


def lib():
    """Load libffs.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_build.LIB):
            raise ImportError(f"{_build.LIB} is missing: the sm_100a library must be built "
                              "(python -m paper_1903_10741_b200.build); there is no CPU fallback")
        L = C.CDLL(_build.LIB)
        P = C.c_void_p
        sig = {
            "ffs_last_error": ([], C.c_char_p), "ffs_version": ([], C.c_char_p),
            "ffs_instance_create": ([C.POINTER(_Desc), C.c_int, P], C.c_int),
            "ffs_instance_destroy": ([P], None),
            "ffs_reschedule_state": ([P, C.c_int32, P, P, P, P], C.c_int),
            "ffs_static_state": ([P, C.c_int32, P, P, P, P], C.c_int),
            "ffs_state_genes": ([P, P, P], C.c_int), "ffs_state_cells": ([P, P], C.c_int),
            "ffs_state_cut_table": ([P, P], C.c_int),
            "ffs_state_set_horizon_cap": ([P, C.c_int32], C.c_int),
            "ffs_state_set_objective_weight": ([P, C.c_double], C.c_int),
            "ffs_brute_force": ([P, C.c_int64, P, P, P, P, P], C.c_int),
            "ffs_state_info": ([P, P, P, P, P, P], C.c_int), "ffs_state_path": ([P, P, P, P], C.c_int), "ffs_state_destroy": ([P], None),
            "ffs_evaluate": ([P, C.c_int64, P, P, P, P, P, P, P], C.c_int),
            "ffs_evaluate_host": ([P, C.c_int64, P, P, P, P, P, P], C.c_int),
            "ffs_evaluate_strided": ([P, C.c_int64, P, P, C.c_int64, P, P, P, P, P], C.c_int),
            "ffs_random_population": ([P, C.c_int64, C.c_uint64, C.c_int64, P, P, P], C.c_int),
            "ffs_random_population_strided": ([P, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, P, P, P], C.c_int),
            "ffs_evolve_begin": ([P, C.POINTER(GAConfig), P, P], C.c_int),
            "ffs_evolve_step": ([P, C.c_int32], C.c_int),
            "ffs_evolve": ([P, C.POINTER(GAConfig), P, P], C.c_int),
            "ffs_best": ([P, P, P, P, P, P, P, P, P, P], C.c_int),
            "ffs_run_population": ([P, P, P, P, P], C.c_int),
            "ffs_run_history": ([P, P, P, P, P], C.c_int),
            "ffs_run_info": ([P, P, P, P, P], C.c_int), "ffs_run_destroy": ([P], None),
            "ffs_run_restore": ([P, C.c_int32, P, P, P, P, P, P, P, P, C.c_int64, P, P], C.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st, what):
    if st != OK:
        raise FFSError(st, what, lib().ffs_last_error().decode())


def _np_ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _dev_ptr(t, dtype, numel, what):
    import torch
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{what}: expected a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous() or t.numel() < numel:
        raise TypeError(f"{what}: expected contiguous {dtype} with >= {numel} elements")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _on(stream):
    """Context placing torch allocations (and their fills) on the stream the
    library call is issued on, so they are ordered with it."""
    import contextlib
    import torch
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


class Instance:
    """EDFFS instance (Table 2) in integer ticks, uploaded to `device`."""

    def __init__(self, n, n_prime, g, o, P, Q, R, D, q_max, wt, device=0):
        self._a = [np.ascontiguousarray(np.asarray(v, dtype=np.int32)).ravel() for v in (P, Q, R, D)]
        ptr = [a.ctypes.data_as(C.POINTER(C.c_int32)) for a in self._a]
        desc = _Desc(int(n), int(n_prime), int(g), int(o), ptr[0], ptr[1], ptr[2], ptr[3], int(q_max), int(wt))
        h = C.c_void_p()
        _check(lib().ffs_instance_create(C.byref(desc), int(device), C.byref(h)), "ffs_instance_create")
        self.h = h
        self.n, self.n_prime, self.g, self.o = int(n), int(n_prime), int(g), int(o)
        self.NJ = self.n + self.n_prime
        self.q_max, self.wt, self.device = int(q_max), int(wt), int(device)

    @classmethod
    def from_arrays(cls, a: dict, device=0):
        return cls(a["n"], a["n_prime"], a["g"], a["o"], a["P"], a["Q"], a["R"], a["D"], a["q_max"], a["wt"],
                   device=device)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ffs_instance_destroy(self.h)
            self.h = None


class State:
    """Frozen rescheduling context at RS (ffs_reschedule_state), or with
    static=True the traditional static approach (ffs_static_state)."""

    def __init__(self, inst: Instance, rs: int, orig_assign=None, orig_start=None, static: bool = False):
        self.inst = inst
        self.static = bool(static)
        oa = None if orig_assign is None else np.ascontiguousarray(np.asarray(orig_assign, np.int32)).ravel()
        os_ = None if orig_start is None else np.ascontiguousarray(np.asarray(orig_start, np.int32)).ravel()
        h = C.c_void_p()
        K = C.c_int32()
        fn = "ffs_static_state" if static else "ffs_reschedule_state"
        _check(getattr(lib(), fn)(inst.h, int(rs), _np_ptr(oa), _np_ptr(os_), C.byref(h), C.byref(K)), fn)
        self.h = h
        self.K = K.value
        self.rs = int(rs)
        self.real_wt = None
        self.cells = inst.NJ * inst.g

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ffs_state_destroy(self.h)
            self.h = None

    def genes(self):
        j = np.zeros(max(self.K, 1), np.int32)
        s = np.zeros(max(self.K, 1), np.int32)
        _check(lib().ffs_state_genes(self.h, _np_ptr(j), _np_ptr(s)), "ffs_state_genes")
        return j[:self.K], s[:self.K]

    def cell_states(self):
        c = np.zeros(self.cells, np.int32)
        _check(lib().ffs_state_cells(self.h, _np_ptr(c)), "ffs_state_cells")
        return c

    def cut_table(self):
        c = np.zeros(self.cells + 1, np.int32)
        _check(lib().ffs_state_cut_table(self.h, _np_ptr(c)), "ffs_state_cut_table")
        return c

    def set_objective_weight(self, wt: float):
        """Fractional WT (Table 11): objectives/fitness become binary64."""
        _check(lib().ffs_state_set_objective_weight(self.h, C.c_double(float(wt))),
               "ffs_state_set_objective_weight")
        self.real_wt = float(wt)

    def set_horizon_cap(self, cap: int):
        _check(lib().ffs_state_set_horizon_cap(self.h, int(cap)), "ffs_state_set_horizon_cap")

    def info(self):
        v = [C.c_int32() for _ in range(5)]
        _check(lib().ffs_state_info(self.h, *[C.byref(x) for x in v]), "ffs_state_info")
        return dict(K=v[0].value, cells=v[1].value, horizon_cap=v[2].value, horizon_bound=v[3].value,
                    smem_bytes=v[4].value)

    def path(self):
        v = [C.c_int32() for _ in range(3)]
        _check(lib().ffs_state_path(self.h, *[C.byref(x) for x in v]), "ffs_state_path")
        return dict(lane_path=bool(v[0].value), lane_mode=v[1].value, max_pending=v[2].value)


def evaluate(state: State, x, y, objective=None, total_tardiness=None, makespan=None, start_out=None,
             with_schedule=False, stream=None):
    """Decode + evaluate device chromosomes x:int8[count,R], y:int16[count,R]
    (R = K, or a padded row R > K: ffs_evaluate_strided)."""
    import torch
    count = x.shape[0] if x.dim() == 2 else (x.numel() // max(state.K, 1))
    row = x.shape[1] if (x.dim() == 2 and x.shape[1] != state.K) else 0
    dev = x.device
    with _on(stream):
        if objective is None:
            objective = torch.empty(count, dtype=torch.int64, device=dev)
        if total_tardiness is None:
            total_tardiness = torch.empty(count, dtype=torch.int64, device=dev)
        if makespan is None:
            makespan = torch.empty(count, dtype=torch.int32, device=dev)
        if with_schedule and start_out is None:
            start_out = torch.empty((count, state.cells), dtype=torch.int32, device=dev)
    n = count * (row or state.K)
    _check(lib().ffs_evaluate_strided(state.h, count, _dev_ptr(x, torch.int8, n, "x"),
                                      _dev_ptr(y, torch.int16, n, "y"), row,
                                      _dev_ptr(objective, torch.int64, count, "objective"),
                                      _dev_ptr(total_tardiness, torch.int64, count, "total_tardiness"),
                                      _dev_ptr(makespan, torch.int32, count, "makespan"),
                                      _dev_ptr(start_out, torch.int32, count * state.cells, "start_out"),
                                      _stream(stream)), "ffs_evaluate_strided")
    if state.real_wt is not None:
        objective = objective.view(torch.float64)
    return objective, total_tardiness, makespan, start_out


def evaluate_host(state: State, x: np.ndarray, y: np.ndarray, stream=None):
    """Same as evaluate() with host buffers (copies inside the call)."""
    x = np.ascontiguousarray(x, dtype=np.int8)
    y = np.ascontiguousarray(y, dtype=np.int16)
    count = x.shape[0]
    obj = np.zeros(count, np.int64)
    T = np.zeros(count, np.int64)
    M = np.zeros(count, np.int32)
    _check(lib().ffs_evaluate_host(state.h, count, _np_ptr(x), _np_ptr(y), _np_ptr(obj), _np_ptr(T), _np_ptr(M),
                                   _stream(stream)), "ffs_evaluate_host")
    return _words(state, obj), T, M


def _words(state: State, a: np.ndarray) -> np.ndarray:
    """64-bit objective words as values: int64, or binary64 in real-WT mode."""
    return a.view(np.float64) if state.real_wt is not None else a


def evaluate_host_into(state: State, x: np.ndarray, y: np.ndarray, obj: np.ndarray, T: np.ndarray,
                       M: np.ndarray, stream=None):
    """evaluate_host() into caller-provided (e.g. pinned) host buffers."""
    _check(lib().ffs_evaluate_host(state.h, x.shape[0], _np_ptr(x), _np_ptr(y), _np_ptr(obj), _np_ptr(T),
                                   _np_ptr(M), _stream(stream)), "ffs_evaluate_host")


def brute_force(state: State, limit: int = 1 << 34, stream=None):
    """Exhaustive ground truth over o^K x linear extensions (ffs_brute_force):
    returns (best objective, evaluated, best x [K], best y [K])."""
    K = state.K
    best, ev = C.c_int64(), C.c_int64()
    bx = np.zeros(max(K, 1), np.int8)
    by = np.zeros(max(K, 1), np.int16)
    _check(lib().ffs_brute_force(state.h, int(limit), C.byref(best), C.byref(ev), _np_ptr(bx), _np_ptr(by),
                                 _stream(stream)), "ffs_brute_force")
    b = best.value
    if state.real_wt is not None:
        b = float(np.array([b], np.int64).view(np.float64)[0])
    return b, ev.value, bx[:K], by[:K]


def random_population(state: State, count: int, seed: int, first_id: int = 0, device=None, stream=None,
                      row: int = 0):
    """Counter-based random chromosomes on the device: [count, K], or
    rows of `row` genes (zero padding; ffs_random_population_strided)."""
    import torch
    dev = torch.device("cuda", state.inst.device) if device is None else device
    R = row if row else state.K
    alloc = torch.zeros if R != state.K else torch.empty
    with _on(stream):   # the zero fill must precede the kernel on its stream
        x = alloc((count, R), dtype=torch.int8, device=dev)
        y = alloc((count, R), dtype=torch.int16, device=dev)
    _check(lib().ffs_random_population_strided(state.h, count, int(seed), int(first_id), int(row),
                                               C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), _stream(stream)),
           "ffs_random_population_strided")
    return x, y


def decode_schedule(state: State, x_genes, y_genes):
    """Decode ONE chromosome on the GPU and return its merged schedule (host):
    assign/start [(n+n')*g], objective, sum T, C_max."""
    import torch
    dev = torch.device("cuda", state.inst.device)
    x = torch.as_tensor(np.asarray(x_genes, np.int8).reshape(1, -1)).to(dev)
    y = torch.as_tensor(np.asarray(y_genes, np.int16).reshape(1, -1)).to(dev)
    if state.K == 0:
        x = torch.zeros((1, 1), dtype=torch.int8, device=dev)
        y = torch.ones((1, 1), dtype=torch.int16, device=dev)
    obj, T, M, st = evaluate(state, x, y, with_schedule=True)
    torch.cuda.synchronize(dev)
    start = st[0].cpu().numpy()
    cs = state.cell_states()
    assign = -np.ones(state.cells, np.int32)
    jj, ss = state.genes()
    g = state.inst.g
    frozen = getattr(state, "frozen_assign", None)
    if frozen is not None:
        assign[cs != 0] = frozen[cs != 0]
    for k in range(state.K):
        assign[jj[k] * g + ss[k]] = int(np.asarray(x_genes).ravel()[k])
    return assign, start, int(obj.item()), int(T.item()), int(M.item())


def make_state(inst: Instance, rs: int, orig_assign=None, orig_start=None, static: bool = False) -> State:
    """State plus the frozen assignment kept for merged-schedule assembly."""
    st = State(inst, rs, orig_assign, orig_start, static=static)
    fa = -np.ones(st.cells, np.int32)
    if orig_assign is not None:
        oa = np.asarray(orig_assign, np.int32).ravel()
        fa[: oa.size] = oa
    st.frozen_assign = fa
    return st


def evolve(state: State, island_w: int, island_h: int, islands_total: int, generations: int, seed: int,
           **kw) -> "Run":
    """The one-shot call ffs_evolve: every generation of the island GA of one
    rescheduling point, returned as a finished Run (read it with best())."""
    return Run(state, island_w, island_h, islands_total, generations, seed, one_shot=True, **kw)


def trace_rows(best: dict, population: int):
    """RunTrace rows: (generation, best objective, mean objective)
    for k = 0..G from a Run.best() / dist.global_best() record: best = the
    minimum objective of generation k's population (after replacement and
    migration), mean = the sum of its objectives / population (the integer
    sum is exact; one division; binary64 sums in fractional-WT mode)."""
    tmin = np.asarray(best["trace_min"])
    tsum = np.asarray(best["trace_sum"])
    return [(k, tmin[k].item(), float(tsum[k]) / float(population)) for k in range(len(tmin))]


def write_trace_csv(path, best: dict, population: int):
    """The trace as CSV `generation,best_objective,mean_objective`."""
    with open(path, "w") as f:
        f.write("generation,best_objective,mean_objective\n")
        for k, b, m in trace_rows(best, population):
            f.write(f"{k},{b},{m!r}\n")


class Run:
    """Island GA of one rescheduling point (ffs_evolve_begin / _step / ffs_best).

    hooks: optional (allreduce_max_i64, allgather) Python callables with the
    C signatures of ffs_ga_config (see paper_1903_10741_b200.dist).
    """

    def __init__(self, state: State, island_w: int, island_h: int, islands_total: int, generations: int,
                 seed: int, island_begin: int = 0, island_end: int | None = None, xo_threshold: int = XO_090,
                 mut_threshold: int = MUT_010, migration_interval: int = 10, rank: int = 0, world: int = 1,
                 hooks=None, stream=None, one_shot: bool = False):
        self.state = state
        island_end = islands_total if island_end is None else island_end
        ar, ag = (ALLRED(), ALLGATHER()) if hooks is None else (ALLRED(hooks[0]), ALLGATHER(hooks[1]))
        self._keep = (ar, ag)
        self.cfg = GAConfig(island_w, island_h, islands_total, island_begin, island_end, xo_threshold,
                            mut_threshold, migration_interval, generations, seed, rank, world, ar, ag, None)
        self.generations = generations
        self.tile = island_w * island_h
        self.nisl = island_end - island_begin
        self.nloc = self.nisl * self.tile
        self._stream = stream
        h = C.c_void_p()
        # one_shot: ffs_evolve (all generations, synchronised) instead of ffs_evolve_begin
        fn = "ffs_evolve" if one_shot else "ffs_evolve_begin"
        _check(getattr(lib(), fn)(state.h, C.byref(self.cfg), _stream(stream), C.byref(h)), fn)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ffs_run_destroy(self.h)
            self.h = None

    def step(self, generations: int = 1):
        _check(lib().ffs_evolve_step(self.h, int(generations)), "ffs_evolve_step")

    def info(self):
        g = C.c_int32()
        e = C.c_int64()
        ev = C.c_int64()
        nl = C.c_int32()
        _check(lib().ffs_run_info(self.h, C.byref(g), C.byref(e), C.byref(ev), C.byref(nl)), "ffs_run_info")
        emax = e.value
        if self.state.real_wt is not None:
            emax = float(np.array([emax], np.int64).view(np.float64)[0])
        return dict(generation=g.value, emax=emax, evaluations=ev.value, launches=nl.value)

    def population(self):
        K = self.state.K
        x = np.zeros((self.nloc, K), np.int8)
        y = np.zeros((self.nloc, K), np.int16)
        obj = np.zeros(self.nloc, np.int64)
        fit = np.zeros(self.nloc, np.int64)
        _check(lib().ffs_run_population(self.h, _np_ptr(x), _np_ptr(y), _np_ptr(obj), _np_ptr(fit)),
               "ffs_run_population")
        return x, y, _words(self.state, obj), _words(self.state, fit)

    def history(self):
        K = self.state.K
        x = np.zeros((self.nisl, K), np.int8)
        y = np.zeros((self.nisl, K), np.int16)
        obj = np.zeros(self.nisl, np.int64)
        fit = np.zeros(self.nisl, np.int64)
        _check(lib().ffs_run_history(self.h, _np_ptr(x), _np_ptr(y), _np_ptr(obj), _np_ptr(fit)), "ffs_run_history")
        return x, y, _words(self.state, obj), _words(self.state, fit)

    def checkpoint(self) -> dict:
        """Everything ffs_run_restore needs to continue this run bit-identically
        (numpy arrays; objective/fitness/trace as raw 64-bit words)."""
        K = self.state.K
        x = np.zeros((self.nloc, K), np.int8)
        y = np.zeros((self.nloc, K), np.int16)
        obj = np.zeros(self.nloc, np.int64)
        fit = np.zeros(self.nloc, np.int64)
        _check(lib().ffs_run_population(self.h, _np_ptr(x), _np_ptr(y), _np_ptr(obj), _np_ptr(fit)),
               "ffs_run_population")
        hx = np.zeros((self.nisl, K), np.int8)
        hy = np.zeros((self.nisl, K), np.int16)
        hobj = np.zeros(self.nisl, np.int64)
        hfit = np.zeros(self.nisl, np.int64)
        _check(lib().ffs_run_history(self.h, _np_ptr(hx), _np_ptr(hy), _np_ptr(hobj), _np_ptr(hfit)),
               "ffs_run_history")
        g, e = C.c_int32(), C.c_int64()
        _check(lib().ffs_run_info(self.h, C.byref(g), C.byref(e), None, None), "ffs_run_info")
        b = self.best()
        words = lambda a: np.ascontiguousarray(np.asarray(a)).view(np.int64)
        c = self.cfg
        config = np.array([K, c.island_w, c.island_h, c.islands_total, c.island_begin, c.island_end,
                           c.migration_interval, c.seed & 0x7FFFFFFFFFFFFFFF, c.xo_threshold, c.mut_threshold], np.int64)
        return dict(generation=g.value, emax=e.value, x=x, y=y, objective=obj, fitness=fit, hx=hx, hy=hy,
                    hobj=hobj, hfit=hfit, trace_min=words(b["trace_min"]), trace_sum=words(b["trace_sum"]),
                    config=config)

    def restore(self, ck: dict):
        """Load a checkpoint() of a run with the same configuration (ffs_run_restore);
        step() then continues at generation ck['generation'] + 1."""
        g = int(ck["generation"])
        K = self.state.K
        c = self.cfg
        mine = np.array([K, c.island_w, c.island_h, c.islands_total, c.island_begin, c.island_end,
                         c.migration_interval, c.seed & 0x7FFFFFFFFFFFFFFF, c.xo_threshold, c.mut_threshold], np.int64)
        if "config" in ck and not np.array_equal(np.asarray(ck["config"]), mine):
            raise ValueError("checkpoint of a run with another configuration (K, shape, shard, interval, seed, rates)")
        if K == 0:   # nothing evolves: only the generation counter must agree
            _check(lib().ffs_run_restore(self.h, g, None, None, None, None, None, None, None, None, 0, None, None),
                   "ffs_run_restore")
            return
        want = {"x": ((self.nloc, K), np.int8), "y": ((self.nloc, K), np.int16), "objective": ((self.nloc,), np.int64),
                "fitness": ((self.nloc,), np.int64), "hx": ((self.nisl, K), np.int8), "hy": ((self.nisl, K), np.int16),
                "hobj": ((self.nisl,), np.int64), "hfit": ((self.nisl,), np.int64),
                "trace_min": ((max(g + 1, 1),), np.int64), "trace_sum": ((max(g + 1, 1),), np.int64)}
        arr = {}
        for k, (shape, dt) in want.items():
            a = np.ascontiguousarray(ck[k])
            if a.dtype.itemsize != np.dtype(dt).itemsize or a.size != int(np.prod(shape)):
                raise ValueError(f"checkpoint array {k}: {a.dtype}{a.shape}, expected {np.dtype(dt)}{shape}")
            arr[k] = a.view(dt).reshape(shape)
        _check(lib().ffs_run_restore(self.h, g, *[_np_ptr(arr[k]) for k in ("x", "y", "objective", "fitness", "hx",
                                                                             "hy", "hobj", "hfit")],
                                     int(ck["emax"]), _np_ptr(arr["trace_min"]), _np_ptr(arr["trace_sum"])),
               "ffs_run_restore")

    def best(self):
        K, cells = self.state.K, self.state.cells
        x = np.zeros(max(K, 1), np.int8)
        y = np.zeros(max(K, 1), np.int16)
        assign = np.zeros(cells, np.int32)
        start = np.zeros(cells, np.int32)
        obj, T, M = C.c_int64(), C.c_int64(), C.c_int32()
        g = self.info()["generation"]
        tmin = np.zeros(max(g + 1, 1), np.int64)
        tsum = np.zeros(max(g + 1, 1), np.int64)
        _check(lib().ffs_best(self.h, _np_ptr(x), _np_ptr(y), _np_ptr(assign), _np_ptr(start), C.byref(obj),
                              C.byref(T), C.byref(M), _np_ptr(tmin), _np_ptr(tsum)), "ffs_best")
        objective = obj.value
        if self.state.real_wt is not None:
            objective = float(np.array([objective], np.int64).view(np.float64)[0])
        return dict(x=x[:K], y=y[:K], assign=assign, start=start, objective=objective, sum_tardiness=T.value,
                    makespan=M.value, trace_min=_words(self.state, tmin[:g + 1]),
                    trace_sum=_words(self.state, tsum[:g + 1]))
