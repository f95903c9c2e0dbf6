"""ctypes wrapper of the C ORACLE (oracle/ffs_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / ``--impl reference`` leg may import this module.
It shares nothing with the CUDA path (paper_1903_10741_b200/); the product
never imports it.

Notation follows PAPER.md: X, Y, Z are (n+n') x g matrices (row-major, -1 on
frozen cells) -- Eqs. (10)-(12).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "ffs_oracle.c")
LIB = os.path.join(HERE, "libffs_oracle.so")

PENDING, RUNNING, COMPLETED, KEPT = 0, 1, 2, 3
Z_COMPLETED = -2
Z_KEPT = -4
OK, ERR_ARG, ERR_INFEASIBLE, ERR_SCHEDULE, ERR_LIMIT = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no GPU, no shared code)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "ffs_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-Wall", "-Wextra", "-Wno-unused-parameter",
                               "-shared", "-fPIC", "-o", LIB, SRC, "-lpthread"])
    return LIB


class _Inst(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_prime", C.c_int32), ("g", C.c_int32), ("o", C.c_int32),
                ("P", C.POINTER(C.c_int32)), ("Q", C.POINTER(C.c_int32)),
                ("R", C.POINTER(C.c_int32)), ("D", C.POINTER(C.c_int32)),
                ("q_max", C.c_int32), ("wt", C.c_int64)]


class _Cnt(C.Structure):
    _fields_ = [("dispatches", C.c_int64), ("checks", C.c_int64),
                ("jumps", C.c_int64), ("updates", C.c_int64)]


_ALLRED = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double))
_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class _Draws(C.Structure):
    _fields_ = [("xo_threshold", C.c_uint32), ("mut_threshold", C.c_uint32),
                ("xo_fire", C.c_void_p), ("xo_cut", C.c_void_p), ("mut_fire", C.c_void_p),
                ("mut_a", C.c_void_p), ("mut_b", C.c_void_p), ("mut_x", C.c_void_p)]


class _GaCfg(C.Structure):
    _fields_ = [("island_w", C.c_int32), ("island_h", C.c_int32), ("islands_total", C.c_int32),
                ("island_begin", C.c_int32), ("island_end", C.c_int32),
                ("xo_threshold", C.c_uint32), ("mut_threshold", C.c_uint32),
                ("migration_interval", C.c_int32), ("generations", C.c_int32),
                ("seed", C.c_uint64), ("nthreads", C.c_int32),
                ("allreduce_max", _ALLRED), ("allgather", _ALLGATHER),
                ("rank", C.c_int32), ("world", C.c_int32), ("user", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        _lib.or_ctx_create.argtypes = [C.POINTER(_Inst), C.c_int32, P, P, C.POINTER(P)]
        _lib.or_ctx_create_static.argtypes = [C.POINTER(_Inst), C.c_int32, P, P, C.POINTER(P)]
        _lib.or_ctx_destroy.argtypes = [P]
        _lib.or_ctx_K.argtypes = [P]
        _lib.or_ctx_cells.argtypes = [P]
        _lib.or_ctx_states.argtypes = [P, P]
        _lib.or_ctx_pending_cells.argtypes = [P, P]
        _lib.or_order.argtypes = [P, P, P]
        _lib.or_decode.argtypes = [P, P, P, P, P, P, P, P, P, C.POINTER(_Cnt)]
        _lib.or_objective.argtypes = [C.POINTER(_Inst), P, P, P, P, P]
        _lib.or_validate.argtypes = [P, P, P, P]
        _lib.or_power_at.argtypes = [C.POINTER(_Inst), P, P, C.c_int64]
        _lib.or_power_at.restype = C.c_int64
        _lib.or_emax.argtypes = [P, C.c_int64]
        _lib.or_emax.restype = C.c_int64
        _lib.or_fitness.argtypes = [C.c_int64, C.c_int64]
        _lib.or_fitness.restype = C.c_int64
        _lib.or_emax_real.argtypes = [P, C.c_int64]
        _lib.or_emax_real.restype = C.c_double
        _lib.or_fitness_real.argtypes = [C.c_double, C.c_double]
        _lib.or_fitness_real.restype = C.c_double
        _lib.or_ctx_set_real_weight.argtypes = [P, C.c_double]
        _lib.or_objective_value.argtypes = [P, C.c_int64, C.c_int64]
        _lib.or_objective_value.restype = C.c_double
        _lib.or_brute_force.argtypes = [P, C.c_int64, P, P, P, P]
        _lib.or_philox4x32_10.argtypes = [P, P, P]
        _lib.or_repair.argtypes = [P, P]
        _lib.or_crossover.argtypes = [P, P, P, P, P, C.c_int32, P, P, P, P]
        _lib.or_mutate.argtypes = [P, P, P, P, C.c_int32, C.c_int32]
        _lib.or_ga_create.argtypes = [P, C.POINTER(_GaCfg), C.POINTER(P)]
        _lib.or_ga_step.argtypes = [P]
        _lib.or_ga_generation.argtypes = [P]
        _lib.or_ga_emax.argtypes = [P]
        _lib.or_ga_emax.restype = C.c_double
        _lib.or_ga_population.argtypes = [P, P, P, P, P]
        _lib.or_ga_trace.argtypes = [P, P, P]
        _lib.or_ga_history.argtypes = [P, P, P, P, P]
        _lib.or_ga_destroy.argtypes = [P]
        _lib.or_evaluate_batch.argtypes = [P, C.c_int64, P, P, P, P, P, P, C.c_int32, C.POINTER(_Cnt)]
        _lib.or_evaluate_batch_schedule.argtypes = [P, C.c_int64, P, P, P, P, P, P, C.c_int32]
        _lib.or_init_ranks.argtypes = [C.c_int32, P, P]
        _lib.or_argmax_fitness.argtypes = [P, C.c_int32]
        _lib.or_argmin_fitness.argtypes = [P, C.c_int32]
        _lib.or_select.argtypes = [P, C.c_int32, C.c_int32, P]
        _lib.or_breed.argtypes = [P, C.c_int32, C.c_int32, P, P, P, C.POINTER(_Draws), P, P]
        _lib.or_replace.argtypes = [C.c_int32, C.c_int32, C.c_int32, P, P, P, P, P, P, P, P]
        _lib.or_migrate.argtypes = [C.c_int32, C.c_int32, C.c_int32, P, P, P, P, C.c_int32, C.c_int32,
                                    _ALLGATHER, P]
        _lib.or_trace_stats.argtypes = [P, C.c_int64, C.c_int32, P, P]
    return _lib


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


@dataclass
class Instance:
    """EDFFS instance in integer ticks (Table 2)."""
    n: int
    n_prime: int
    g: int
    o: int
    P: np.ndarray      # [(n+n'), g, o]
    Q: np.ndarray      # [(n+n'), g, o]
    R: np.ndarray      # [n+n']
    D: np.ndarray      # [n+n']
    q_max: int
    wt: int

    def _c(self):
        self._keep = [_i32(self.P).ravel(), _i32(self.Q).ravel(), _i32(self.R), _i32(self.D)]
        ptr = [a.ctypes.data_as(C.POINTER(C.c_int32)) for a in self._keep]
        return _Inst(self.n, self.n_prime, self.g, self.o, ptr[0], ptr[1], ptr[2], ptr[3],
                     int(self.q_max), int(self.wt))


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with status {code}")
        self.code = code


def _chk(st, what):
    if st != OK:
        raise OracleError(st, what)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def emax(objectives) -> int:
    a = np.ascontiguousarray(np.asarray(objectives, dtype=np.int64))
    return int(lib().or_emax(_p(a), len(a)))


def fitness(objective: int, e_max: int) -> int:
    return int(lib().or_fitness(int(objective), int(e_max)))


def emax_real(objectives) -> float:
    a = np.ascontiguousarray(np.asarray(objectives, dtype=np.float64))
    return float(lib().or_emax_real(_p(a), len(a)))


def fitness_real(objective: float, e_max: float) -> float:
    return float(lib().or_fitness_real(float(objective), float(e_max)))


def _values(a, real):
    """GA values are binary64 in the oracle: int64 view for the integer objective."""
    if real:
        return a
    assert np.all(np.abs(a) < 2.0 ** 53) and np.all(a == np.floor(a))
    return a.astype(np.int64)


def objective(inst: Instance, assign, start):
    ci = inst._c()
    a, s = _i32(assign).ravel(), _i32(start).ravel()
    T, M, O = C.c_int64(), C.c_int64(), C.c_int64()
    lib().or_objective(C.byref(ci), _p(a), _p(s), C.byref(T), C.byref(M), C.byref(O))
    return T.value, M.value, O.value


def power_at(inst: Instance, assign, start, t) -> int:
    ci = inst._c()
    a, s = _i32(assign).ravel(), _i32(start).ravel()
    return int(lib().or_power_at(C.byref(ci), _p(a), _p(s), int(t)))


class Ctx:
    """Frozen rescheduling context at RS (Algorithm 1 frozen branch)."""

    def __init__(self, inst: Instance, rs: int, orig_assign=None, orig_start=None, static: bool = False):
        """static=True: the traditional static approach (Fig. 7) --
        the originals keep their whole plan, only the new jobs are genes."""
        self.inst = inst
        self.static = bool(static)
        self.real_wt = None
        self._ci = inst._c()
        self._oa = None if orig_assign is None else _i32(orig_assign).ravel()
        self._os = None if orig_start is None else _i32(orig_start).ravel()
        h = C.c_void_p()
        create = lib().or_ctx_create_static if static else lib().or_ctx_create
        _chk(create(C.byref(self._ci), int(rs), _p(self._oa), _p(self._os), C.byref(h)), "ctx_create")
        self.h = h
        self.rs = int(rs)
        self.K = lib().or_ctx_K(h)
        self.cells = lib().or_ctx_cells(h)
        st = np.zeros(self.cells, dtype=np.int32)
        lib().or_ctx_states(h, _p(st))
        self.states = st.reshape(inst.n + inst.n_prime, inst.g)
        pc = np.zeros(max(self.K, 1), dtype=np.int32)
        lib().or_ctx_pending_cells(h, _p(pc))
        self.pending_cells = pc[:self.K].copy()

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_ctx_destroy(self.h)
            self.h = None

    def set_real_weight(self, wt: float):
        """Fractional WT (Table 11): Eq. (1) in binary64 from now on."""
        _chk(lib().or_ctx_set_real_weight(self.h, float(wt)), "set_real_weight")
        self.real_wt = float(wt)

    def objective_value(self, sum_tardiness: int, makespan: int):
        v = float(lib().or_objective_value(self.h, int(sum_tardiness), int(makespan)))
        return v if self.real_wt is not None else int(v)

    # compact canonical genes <-> paper matrices
    def to_matrix(self, x_genes, y_genes):
        X = -np.ones(self.cells, dtype=np.int32)
        Y = -np.ones(self.cells, dtype=np.int32)
        X[self.pending_cells] = np.asarray(x_genes, dtype=np.int32)
        Y[self.pending_cells] = np.asarray(y_genes, dtype=np.int32)
        return X, Y

    def to_genes(self, X, Y):
        X = np.asarray(X).ravel()
        Y = np.asarray(Y).ravel()
        return X[self.pending_cells].astype(np.int8), Y[self.pending_cells].astype(np.int16)

    def order(self, Y):
        Yc = _i32(Y).ravel()
        Z = np.zeros(self.cells, dtype=np.int32)
        _chk(lib().or_order(self.h, _p(Yc), _p(Z)), "order")
        return Z

    def decode(self, X, Y=None, Z=None):
        Xc = _i32(X).ravel()
        Yc = None if Y is None else _i32(Y).ravel()
        Zc = None if Z is None else _i32(Z).ravel()
        asg = np.zeros(self.cells, dtype=np.int32)
        st = np.zeros(self.cells, dtype=np.int32)
        T, M, O = C.c_int64(), C.c_int64(), C.c_int64()
        cnt = _Cnt()
        _chk(lib().or_decode(self.h, _p(Xc), _p(Yc), _p(Zc), _p(asg), _p(st), C.byref(T),
                             C.byref(M), C.byref(O), C.byref(cnt)), "decode")
        return dict(assign=asg, start=st, sum_tardiness=T.value, makespan=M.value,
                    objective=O.value, value=self.objective_value(T.value, M.value),
                    counters=dict(dispatches=cnt.dispatches, checks=cnt.checks,
                                  jumps=cnt.jumps, updates=cnt.updates))

    def decode_genes(self, x_genes, y_genes):
        X, Y = self.to_matrix(x_genes, y_genes)
        return self.decode(X, Y)

    def validate(self, assign, start):
        a, s = _i32(assign).ravel(), _i32(start).ravel()
        kinds = C.c_int32()
        n = lib().or_validate(self.h, _p(a), _p(s), C.byref(kinds))
        return n, kinds.value

    def brute_force(self, limit=10**7):
        best = C.c_int64()
        ev = C.c_int64()
        bx = np.zeros(self.cells, dtype=np.int32)
        bz = np.zeros(self.cells, dtype=np.int32)
        _chk(lib().or_brute_force(self.h, int(limit), C.byref(best), C.byref(ev), _p(bx), _p(bz)),
             "brute_force")
        return best.value, ev.value, bx, bz

    def repair(self, Y):
        Yc = _i32(Y).ravel().copy()
        lib().or_repair(self.h, _p(Yc))
        return Yc

    def crossover(self, XA, YA, XB, YB, p):
        ins = [_i32(a).ravel() for a in (XA, YA, XB, YB)]
        outs = [np.zeros(self.cells, dtype=np.int32) for _ in range(4)]
        lib().or_crossover(self.h, *[_p(a) for a in ins], int(p), *[_p(a) for a in outs])
        return outs

    def mutate(self, X, Y, rx, gene_a, gene_b):
        Xc, Yc = _i32(X).ravel().copy(), _i32(Y).ravel().copy()
        r = None if rx is None else np.ascontiguousarray(np.asarray(rx, dtype=np.uint32))
        lib().or_mutate(self.h, _p(Xc), _p(Yc), _p(r), int(gene_a), int(gene_b))
        return Xc, Yc

    def evaluate_batch(self, x, y, nthreads=1):
        """Decode + evaluate compact chromosomes x[count,K] int8, y[count,K] int16."""
        x = np.ascontiguousarray(x, dtype=np.int8)
        y = np.ascontiguousarray(y, dtype=np.int16)
        count = x.shape[0]
        obj = np.zeros(count, dtype=np.int64)
        T = np.zeros(count, dtype=np.int64)
        M = np.zeros(count, dtype=np.int64)
        val = np.zeros(count, dtype=np.float64)
        cnt = _Cnt()
        _chk(lib().or_evaluate_batch(self.h, count, _p(x), _p(y), _p(obj), _p(T), _p(M), _p(val),
                                     int(nthreads), C.byref(cnt)), "evaluate_batch")
        if self.real_wt is not None:       # Eq. (1) with the real weight, binary64
            obj = val
        return obj, T, M, dict(dispatches=cnt.dispatches, checks=cnt.checks, jumps=cnt.jumps,
                               updates=cnt.updates)

    def evaluate_batch_schedule(self, x, y, nthreads=1):
        """evaluate_batch plus every chromosome's merged start times [count, cells]."""
        x = np.ascontiguousarray(x, dtype=np.int8)
        y = np.ascontiguousarray(y, dtype=np.int16)
        count = x.shape[0]
        obj = np.zeros(count, dtype=np.int64)
        T = np.zeros(count, dtype=np.int64)
        M = np.zeros(count, dtype=np.int64)
        S = np.zeros((count, self.cells), dtype=np.int32)
        _chk(lib().or_evaluate_batch_schedule(self.h, count, _p(x), _p(y), _p(obj), _p(T), _p(M), _p(S),
                                              int(nthreads)), "evaluate_batch_schedule")
        return obj, T, M, S


# ---- single GA steps (the functions the oracle GA itself runs) ----
def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def init_ranks(keys):
    """Generation-0 priorities: y = 1 + rank of the key (ties by index)."""
    k = _u32(keys)
    y = np.zeros(len(k), dtype=np.int32)
    lib().or_init_ranks(len(k), _p(k), _p(y))
    return y


def select(fit_tile, w, h):
    """Asteroid selection on one island tile: winner index per cell."""
    f = _f64(fit_tile).ravel()
    assert f.size == w * h
    win = np.zeros(w * h, dtype=np.int32)
    lib().or_select(_p(f), int(w), int(h), _p(win))
    return win


def breed(ctx: "Ctx", w, h, PX, PY, winner, xo_fire, xo_cut, mut_fire, mut_a, mut_b, mut_x,
          xo_threshold=None, mut_threshold=None):
    """One island's crossover + correction and mutation with explicit draws."""
    tile = w * h
    px, py = _i32(PX).reshape(tile, ctx.cells), _i32(PY).reshape(tile, ctx.cells)
    arrs = [_i32(winner), _u32(xo_fire), _u32(xo_cut), _u32(mut_fire), _u32(mut_a), _u32(mut_b),
            _u32(mut_x).reshape(tile * max(ctx.K, 1))]
    d = _Draws(XO_090 if xo_threshold is None else xo_threshold,
               MUT_010 if mut_threshold is None else mut_threshold,
               *[a.ctypes.data for a in arrs[1:]])
    X = np.zeros((tile, ctx.cells), dtype=np.int32)
    Y = np.zeros((tile, ctx.cells), dtype=np.int32)
    lib().or_breed(ctx.h, int(w), int(h), _p(px), _p(py), _p(arrs[0]), C.byref(d), _p(X), _p(Y))
    return X, Y


def replace(tile, X, Y, obj, fit, HX, HY, hobj, hfit):
    """Elitist replacement over len(hfit) islands; arrays updated in place."""
    nisl = len(hfit)
    cells = X.shape[-1]
    for a, dt in ((X, np.int32), (Y, np.int32), (HX, np.int32), (HY, np.int32),
                  (obj, np.float64), (fit, np.float64), (hobj, np.float64), (hfit, np.float64)):
        assert a.dtype == dt and a.flags.c_contiguous
    lib().or_replace(nisl, int(tile), int(cells), _p(X), _p(Y), _p(obj), _p(fit), _p(HX), _p(HY),
                     _p(hobj), _p(hfit))


def migrate(nisl, tile, X, Y, obj, fit, rank=0, world=1, allgather=None):
    """Synchronous ring migration of one shard's islands, in place.
    allgather(bytes) -> list of per-rank bytes (rank-major)."""
    cells = X.shape[-1]
    for a, dt in ((X, np.int32), (Y, np.int32), (obj, np.float64), (fit, np.float64)):
        assert a.dtype == dt and a.flags.c_contiguous
    ag = _ALLGATHER()
    if allgather is not None:
        def _ag(user, send, recv, nbytes):
            joined = b"".join(allgather(C.string_at(send, nbytes)))
            C.memmove(recv, joined, len(joined))
            return 0
        ag = _ALLGATHER(_ag)
    _chk(lib().or_migrate(int(nisl), int(tile), int(cells), _p(X), _p(Y), _p(obj), _p(fit),
                          int(rank), int(world), ag, None), "migrate")


def migration_record(x, y, obj, fit):
    """The cross-shard record of or_migrate: X[cells] int32, Y[cells] int32, obj, fit."""
    return (_i32(x).tobytes() + _i32(y).tobytes() + np.float64(obj).tobytes()
            + np.float64(fit).tobytes())


def trace_stats(obj, tile=None):
    """(min, sum) over islands of `tile` cells (default: one island), R33."""
    o = _f64(obj)
    tile = len(o) if tile is None else int(tile)
    assert len(o) % tile == 0
    mn, sm = C.c_double(), C.c_double()
    lib().or_trace_stats(_p(o), len(o) // tile, tile, C.byref(mn), C.byref(sm))
    return mn.value, sm.value


XO_090 = 3865470566   # floor(0.9 * 2^32)
MUT_010 = 429496729   # floor(0.1 * 2^32)


class GA:
    """Literal island GA of one rescheduling point (shard-aware)."""

    def __init__(self, ctx: Ctx, island_w, island_h, islands_total, generations, seed,
                 island_begin=0, island_end=None, xo_threshold=XO_090, mut_threshold=MUT_010,
                 migration_interval=10, nthreads=1, allreduce_max=None, allgather=None,
                 rank=0, world=1):
        self.ctx = ctx
        island_end = islands_total if island_end is None else island_end
        self._cb = []
        ar = _ALLRED()
        ag = _ALLGATHER()
        if allreduce_max is not None:
            def _ar(user, ptr):
                ptr[0] = float(allreduce_max(float(ptr[0])))
                return 0
            ar = _ALLRED(_ar)
        if allgather is not None:
            def _ag(user, send, recv, nbytes):
                buf = C.string_at(send, nbytes)
                out = allgather(buf)  # list of bytes, rank-major
                joined = b"".join(out)
                C.memmove(recv, joined, len(joined))
                return 0
            ag = _ALLGATHER(_ag)
        self._cb = [ar, ag]
        self.cfg = _GaCfg(island_w, island_h, islands_total, island_begin, island_end,
                          xo_threshold, mut_threshold, migration_interval, generations, seed,
                          nthreads, ar, ag, rank, world, None)
        h = C.c_void_p()
        _chk(lib().or_ga_create(ctx.h, C.byref(self.cfg), C.byref(h)), "ga_create")
        self.h = h
        self.generations = generations
        self.nloc = (island_end - island_begin) * island_w * island_h
        self.nisl = island_end - island_begin

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_ga_destroy(self.h)
            self.h = None

    def step(self):
        _chk(lib().or_ga_step(self.h), "ga_step")

    @property
    def generation(self):
        return lib().or_ga_generation(self.h)

    @property
    def real(self):
        return self.ctx.real_wt is not None

    @property
    def emax(self):
        e = float(lib().or_ga_emax(self.h))
        return e if self.real else int(e)

    def population(self):
        K = self.ctx.K
        x = np.zeros((self.nloc, K), dtype=np.int8)
        y = np.zeros((self.nloc, K), dtype=np.int16)
        obj = np.zeros(self.nloc, dtype=np.float64)
        fit = np.zeros(self.nloc, dtype=np.float64)
        lib().or_ga_population(self.h, _p(x), _p(y), _p(obj), _p(fit))
        return x, y, _values(obj, self.real), _values(fit, self.real)

    def history(self):
        K = self.ctx.K
        x = np.zeros((self.nisl, K), dtype=np.int8)
        y = np.zeros((self.nisl, K), dtype=np.int16)
        obj = np.zeros(self.nisl, dtype=np.float64)
        fit = np.zeros(self.nisl, dtype=np.float64)
        lib().or_ga_history(self.h, _p(x), _p(y), _p(obj), _p(fit))
        return x, y, _values(obj, self.real), _values(fit, self.real)

    def trace(self):
        tmin = np.zeros(self.generations + 1, dtype=np.float64)
        tsum = np.zeros(self.generations + 1, dtype=np.float64)
        lib().or_ga_trace(self.h, _p(tmin), _p(tsum))
        return _values(tmin, self.real), _values(tsum, self.real)
