/*
 * ffs_oracle.h -- CPU ORACLE for arXiv 1903.10741 (Luo, Fujimura, El Baz).
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1903_10741_b200/csrc, include/ffs.h); neither includes the other.
 *
 * Plain, slow, literal C99.  Everything is written in the paper's notation:
 * matrices X(k), Y(k), Z(k) are (n+n') x g, row-major, -1 marks a frozen cell
 * (Eqs. (10)-(12)).  Times and powers are integer ticks
 * (reading R10).  Citations: "P:n" = PAPER.md line n.
 *
 * Parity pins (tests/test_oracle_*.py): Table 4 freeze + decode,
 * Table 4 original plan as a decode output, hand-computed H3
 * instance, Fig. 11 crossover/correction, Fig. 12 mutation
 * (P:355-359), Eq. (13) + E_max rule examples, Philox Random123 KATs,
 * brute force over all (X, order) on tiny instances, exhaustive integer scan
 * for the delay rule, schedule invariants Eqs. (4)-(10).
 * GA steps (init ranks, selection, breeding order, replacement, ring
 * migration across a shard boundary, trace): hand-derived goldens
 * (tests/golden/ga_ops.json).  The GA trajectory as a
 * whole has no printed value in the paper; it is the composition of those
 * pinned steps.
 */
#ifndef FFS_ORACLE_H
#define FFS_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* operation states at the rescheduling point (Algorithm 1) */
#define OR_PENDING   0
#define OR_RUNNING   1   /* z_js = 0  */
#define OR_COMPLETED 2   /* z_js = C  */
#define OR_KEPT      3   /* static baseline only: original op held at its plan */

/* rescheduling policies */
#define OR_DYNAMIC 0     /* predictive-reactive complete rescheduling (Fig. 8) */
#define OR_STATIC  1     /* traditional static approach (Fig. 7)                */

#define OR_OK 0
#define OR_ERR_ARG 1
#define OR_ERR_INFEASIBLE 2
#define OR_ERR_SCHEDULE 3
#define OR_ERR_LIMIT 4

typedef struct {
  int32_t n, n_prime, g, o;      /* Table 2 */
  const int32_t *P;              /* P_jsm  [(n+n')*g*o] */
  const int32_t *Q;              /* Q_jsm  [(n+n')*g*o] */
  const int32_t *R;              /* R_j    [n+n'] */
  const int32_t *D;              /* D_j    [n+n'] */
  int32_t q_max;                 /* Q_max */
  int64_t wt;                    /* WT, integer (reading R25) */
} or_instance;

typedef struct or_ctx or_ctx;    /* instance + frozen rescheduling context */

/* Counters of the literal algorithm (instrumentation for the roofline's
 * algorithmic-op count). */
typedef struct {
  int64_t dispatches;   /* operations assigned by Algorithm 2            */
  int64_t checks;       /* instants at which Q_t + Q_js <= Q_max is tested */
  int64_t jumps;        /* "delayed until finishing job i' at stage s'"  */
  int64_t updates;      /* profile intervals committed                   */
} or_counters;

/* Freeze at RS (Algorithm 1 frozen branch; Eq. (10)).
 * orig_assign/orig_start: [n*g] plan of the original jobs, or NULL (then
 * every original op is PENDING, the static problem).  Validates the plan
 * (Eqs. (4)-(7)) and the power precondition. */
int or_ctx_create(const or_instance *inst, int32_t rs, const int32_t *orig_assign,
                  const int32_t *orig_start, or_ctx **out);
/* Traditional static approach (Fig. 7): the
 * original jobs keep their whole plan (OR_KEPT for the ops still pending at
 * RS), only the new jobs' ops are genes (K = n'*g).  KEPT ops hold their
 * machine and draw power over their planned interval, so every arrival op
 * starts after the last original op on its machine (R29) within Q_max (R30).
 * The plan is required when n > 0. */
int or_ctx_create_static(const or_instance *inst, int32_t rs, const int32_t *orig_assign,
                         const int32_t *orig_start, or_ctx **out);
void or_ctx_destroy(or_ctx *c);
int32_t or_ctx_K(const or_ctx *c);
int32_t or_ctx_cells(const or_ctx *c);
/* state per cell [(n+n')*g]: OR_PENDING/OR_RUNNING/OR_COMPLETED/OR_KEPT */
void or_ctx_states(const or_ctx *c, int32_t *state);
/* canonical gene order: the pending cells in row-major order [K] */
void or_ctx_pending_cells(const or_ctx *c, int32_t *cell_of_gene);

/* Algorithm 1, greedy reading (DESIGN R1): Z[(n+n')*g] gets
 * 0 for RUNNING, -2 for COMPLETED (the paper's "C"), -4 for KEPT, rank
 * 1..K otherwise. */
int or_order(const or_ctx *c, const int32_t *Y, int32_t *Z);

/* Algorithm 2 decode of one chromosome.
 * X, Y: [(n+n')*g] matrices (-1 on frozen cells).
 * Z: optional rank matrix to decode with instead of Algorithm 1 (used for
 *    the paper's printed Z and by brute force); NULL = or_order(Y).
 * assign/start: optional [(n+n')*g] merged schedule (frozen cells copied).
 * Objective Eqs. (1)-(3) over all jobs J u J'. */
int or_decode(const or_ctx *c, const int32_t *X, const int32_t *Y, const int32_t *Z,
              int32_t *assign, int32_t *start, int64_t *sum_tardiness,
              int64_t *makespan, int64_t *objective, or_counters *cnt);

/* Eqs. (1)-(3) on a full schedule [(n+n')*g]. */
void or_objective(const or_instance *inst, const int32_t *assign, const int32_t *start,
                  int64_t *sum_tardiness, int64_t *makespan, int64_t *objective);

/* Constraint check, Eqs. (4)-(10) + frozen ops unchanged.  Returns the
 * number of violations; kinds (bitmask, may be NULL): 1 Eq4, 2 Eq5, 4 Eq6,
 * 8 Eq7, 16 Eq10, 32 frozen op moved, 64 machine index out of range,
 * 128 (static policy) a new op starts before an original op on its machine ends. */
int or_validate(const or_ctx *c, const int32_t *assign, const int32_t *start, int32_t *kinds);

/* Power profile level Q_t at instant t (Eqs. (8)-(9)) of a full schedule. */
int64_t or_power_at(const or_instance *inst, const int32_t *assign, const int32_t *start,
                    int64_t t);

/* E_max = 10^a, a >= 1, smallest with every objective < E_max. */
int64_t or_emax(const int64_t *objectives, int64_t count);
/* Eq. (13): max(E_max - objective, 0). */
int64_t or_fitness(int64_t objective, int64_t emax);
/* the same two rules over binary64 values (used by the GA; exact for the
 * integer objective below 2^53, and the fractional-WT objective of Table 11) */
double or_emax_real(const double *objectives, int64_t count);
double or_fitness_real(double objective, double emax);

/* Fractional WT (Table 11): switch the context to
 * Eq. (1) with a real weight wt >= 0.  or_objective_value then returns
 * fl(fl(WT * sum T) + C_max) (two binary64 roundings, no FMA); without the
 * switch it returns the exact integer objective of the instance's WT. */
int or_ctx_set_real_weight(or_ctx *c, double wt);
double or_objective_value(const or_ctx *c, int64_t sum_tardiness, int64_t makespan);

/* Brute force over every X in [0,o-1]^K and every linear extension of the
 * job chains (the decoder-reachable set), decoding each order directly.
 * Fails with OR_ERR_LIMIT if o^K * #orders > limit. */
int or_brute_force(const or_ctx *c, int64_t limit, int64_t *best_objective,
                   int64_t *evaluated, int32_t *best_X, int32_t *best_Z);

/* Philox4x32-10 (Random123), DESIGN.md "RNG". */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* ---- GA operators on single chromosomes (paper notation) ---- */
/* Correction (Fig. 11): keep first occurrence (row-major), replace
 * later duplicates with the missing values 1..K in ascending order. */
void or_repair(const or_ctx *c, int32_t *Y);
/* Neighbouring paired crossover at row-major cut p (Fig. 11): children
 * swap every cell at position >= p, then each child's Y is corrected. */
void or_crossover(const or_ctx *c, const int32_t *XA, const int32_t *YA,
                  const int32_t *XB, const int32_t *YB, int32_t p,
                  int32_t *XA2, int32_t *YA2, int32_t *XB2, int32_t *YB2);
/* Mutation body (Fig. 12) with explicit draws: rx[K] per gene
 * (x <- (x + 1 + floor(rx*(o-1)/2^32)) mod o), then swap Y at genes a, b. */
void or_mutate(const or_ctx *c, int32_t *X, int32_t *Y, const uint32_t *rx,
               int32_t gene_a, int32_t gene_b);

/* ---- GA steps on one generation; the GA below runs
 * exactly these functions, so their goldens (tests/golden/ga_ops.json) pin
 * the trajectory's operators.  Fitness/objective values are binary64. ---- */
/* y of gene gi = 1 + rank of keys[gi] ascending, ties by gene index */
void or_init_ranks(int32_t K, const uint32_t *keys, int32_t *y);
/* largest / smallest fitness, ties -> lowest index */
int32_t or_argmax_fitness(const double *fit, int32_t n);
int32_t or_argmin_fitness(const double *fit, int32_t n);
/* asteroid selection on one island tile fit[h*w] (R17, R18) */
void or_select(const double *fit, int32_t w, int32_t h, int32_t *winner);
/* the draws one island's breeding consumes */
typedef struct {
  uint32_t xo_threshold, mut_threshold;
  const uint32_t *xo_fire, *xo_cut;             /* [tile/2], pair = row*(w/2)+c   */
  const uint32_t *mut_fire, *mut_a, *mut_b;     /* [tile]                         */
  const uint32_t *mut_x;                        /* [tile*K], row i read iff cell i mutates */
} or_breed_draws;
/* crossover + correction of the winner pairs, then mutation (
 * R13-R16, R19, R20).  PX/PY: island snapshot [tile*cells]; X/Y: new cells. */
void or_breed(const or_ctx *c, int32_t w, int32_t h, const int32_t *PX, const int32_t *PY,
              const int32_t *winner, const or_breed_draws *d, int32_t *X, int32_t *Y);
/* elitist replacement over nisl islands of `tile` cells of `cells` ints (R21) */
void or_replace(int32_t nisl, int32_t tile, int32_t cells, int32_t *X, int32_t *Y,
                double *obj, double *fit, int32_t *HX, int32_t *HY, double *hobj, double *hfit);
/* synchronous single-ring migration of this shard's nisl islands (
 * R22); cross-shard record = X[cells] int32, Y[cells] int32, obj, fit */
int or_migrate(int32_t nisl, int32_t tile, int32_t cells, int32_t *X, int32_t *Y,
               double *obj, double *fit, int32_t rank, int32_t world,
               int (*allgather)(void *user, const void *send, void *recv, size_t bytes_per_rank),
               void *user);
/* trace: min objective and sum over nisl islands of `tile` cells, each
 * island in cell order, then islands in order (R33) */
void or_trace_stats(const double *obj, int64_t nisl, int32_t tile, double *mn, double *sum);

/* ---- the island GA of one rescheduling point ---- */
typedef struct {
  int32_t island_w, island_h;         /* island tile (row-major cells)        */
  int32_t islands_total;              /* global island count                  */
  int32_t island_begin, island_end;   /* this shard                           */
  uint32_t xo_threshold;              /* fire iff u < thr; 0.9 -> 3865470566  */
  uint32_t mut_threshold;             /* 0.1 -> 429496729                     */
  int32_t migration_interval;         /* 10                           */
  int32_t generations;                /* G                                    */
  uint64_t seed;
  int32_t nthreads;                   /* evaluation threads (timing only)     */
  /* shard exchange (NULL when single shard): global max of a binary64
   * objective; allgather of bytes_per_rank from every shard into recv
   * (rank-major) */
  int (*allreduce_max)(void *user, double *val);
  int (*allgather)(void *user, const void *send, void *recv, size_t bytes_per_rank);
  int32_t rank, world;
  void *user;
} or_ga_cfg;

typedef struct or_run or_run;
int or_ga_create(const or_ctx *c, const or_ga_cfg *cfg, or_run **out);
/* gen 0 (init + evaluate + E_max + history) when the run is fresh, else one
 * generation k = done+1 (select, crossover, mutate, evaluate, replace,
 * migrate, trace). */
int or_ga_step(or_run *r);
int32_t or_ga_generation(const or_run *r);
/* The GA keeps objectives (or_objective_value) and fitness in binary64. */
double or_ga_emax(const or_run *r);
/* local shard population as compact genes (canonical order) [cells_local*K] */
void or_ga_population(const or_run *r, int8_t *x, int16_t *y, double *obj, double *fit);
/* local trace: per generation min objective and sum of objectives (summed
 * per island in cell order, then islands in order, R33) [G+1] */
void or_ga_trace(const or_run *r, double *tmin, double *tsum);
/* per-island history elites of the shard: [islands_local*K] + obj/fit */
void or_ga_history(const or_run *r, int8_t *x, int16_t *y, double *obj, double *fit);
void or_ga_destroy(or_run *r);

/* batch evaluation of compact chromosomes, nthreads workers; objective is
 * the integer-WT Eq. (1), value (may be NULL) or_objective_value */
int or_evaluate_batch(const or_ctx *c, int64_t count, const int8_t *x, const int16_t *y,
                      int64_t *objective, int64_t *sum_tardiness, int64_t *makespan,
                      double *value, int32_t nthreads, or_counters *cnt);

/* the same with each chromosome's merged schedule start[count*cells]
 * (Algorithm 2's start times, frozen cells copied) -- or_decode per row */
int or_evaluate_batch_schedule(const or_ctx *c, int64_t count, const int8_t *x, const int16_t *y,
                               int64_t *objective, int64_t *sum_tardiness, int64_t *makespan,
                               int32_t *start, int32_t nthreads);

#ifdef __cplusplus
}
#endif
#endif
