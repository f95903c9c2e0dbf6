/*
 * ffs.h -- C-ABI of the B200-native decode/evaluate + island GA for the
 * energy-efficient dynamic flexible flow shop (EDFFS) of
 * Luo, Fujimura, El Baz, arXiv 1903.10741 ("the paper", PAPER.md).
 *
 * Citations "P:n" are PAPER.md line numbers; readings "Rn" are listed in
 * DESIGN.md ("Readings").  Implemented only by hand-written sm_100a CUDA
 * (paper_1903_10741_b200/csrc); there is no CPU fallback.
 *
 * Conventions (all calls):
 *  - Integer time ticks and integer power (R10).  Instance arrays are
 *    row-major [j][s][m] (job, stage, stage-local machine) as in Table 2
 *    (P:92-130).  Jobs 0..n-1 are the original jobs J, n..n+n'-1 the new
 *    arrival jobs J'.
 *  - Status return only; out-parameters are written only on FFS_OK.
 *    ffs_last_error() returns a thread-local message for the last non-OK
 *    status of the calling thread.
 *  - Ownership: every input array is copied during the call; the caller
 *    keeps ownership of its arrays.  Handles are caller-owned and released
 *    with the matching *_destroy.  An ffs_state must not outlive its
 *    ffs_instance; an ffs_run must not outlive its ffs_state.
 *  - Device pointers are plain CUDA global-memory pointers on the
 *    instance's device (e.g. torch tensor data_ptr()); `cuda_stream` is a
 *    cudaStream_t (NULL = legacy default stream).  Device-pointer calls are
 *    stream-ordered and asynchronous: asynchronous CUDA faults surface as
 *    FFS_ERR_CUDA at the next synchronising call.
 *  - One host thread per handle at a time.
 */
#ifndef FFS_H
#define FFS_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FFS_API __attribute__((visibility("default")))
#else
#define FFS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FFS_OK = 0,
  FFS_ERR_INVALID_ARG = 1,      /* null pointer, bad size/range, D_j < R_j, P <= 0, Q < 0,
                                   a limit of this implementation exceeded (see below)   */
  FFS_ERR_INFEASIBLE = 2,       /* some Q_jsm > Q_max (no start can ever satisfy Eq. (7)),
                                   or the RUNNING ops at RS already exceed Q_max         */
  FFS_ERR_INVALID_SCHEDULE = 3, /* original plan misses an op or violates Eqs. (4)-(7)   */
  FFS_ERR_CUDA = 4,             /* CUDA runtime / launch / asynchronous kernel error     */
  FFS_ERR_OOM = 5,              /* device allocation failed                              */
  FFS_ERR_COMM = 6              /* a collective hook returned non-zero                   */
} ffs_status;

/* Message of the last non-OK status on this thread ("" if none). */
FFS_API const char *ffs_last_error(void);
/* Library version string. */
FFS_API const char *ffs_version(void);

typedef struct ffs_instance ffs_instance;  /* instance data + device copy            */
typedef struct ffs_state ffs_state;        /* frozen context at RS + staged tables   */
typedef struct ffs_run ffs_run;            /* island-GA population, elites, trace    */

/* ------------------------------------------------------------------------
 * Instance (Table 2; conditions of Table 1).
 * Limits of this implementation: n+n' <= 65535, g*o <= 4096, o <= 127,
 * P_jsm in [1, 65535], Q_jsm in [0, 65535], Q_max <= 65535, R_j >= 0,
 * every derived time below 2^30 ticks.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t n;                  /* original jobs J                     */
  int32_t n_prime;            /* new arrival jobs J'                 */
  int32_t g;                  /* stages S                            */
  int32_t o;                  /* machines per stage M                */
  const int32_t *proc_time;   /* P_jsm [(n+n')*g*o], > 0             */
  const int32_t *power;       /* Q_jsm [(n+n')*g*o], >= 0            */
  const int32_t *release;     /* R_j [n+n']                          */
  const int32_t *due;         /* D_j [n+n'], D_j >= R_j              */
  int32_t q_max;              /* Q_max, power's peak (Eq. (7))        */
  int64_t wt;                 /* WT >= 0, weight of total tardiness (Eq. (1)); integer (R25) */
} ffs_instance_desc;

/* Copy host arrays, validate, upload to `cuda_device`. */
FFS_API ffs_status ffs_instance_create(const ffs_instance_desc *d, int cuda_device, ffs_instance **out);
FFS_API void ffs_instance_destroy(ffs_instance *inst);

/* ------------------------------------------------------------------------
 * Freeze at the rescheduling point RS (Algorithm 1 frozen branch,
 * P:245-255; Eq. (10); predictive-reactive complete rescheduling
 * P:164).  For every original op with plan machine M, start S and
 * completion C = S + P_jsM:  RUNNING iff S < RS < C (z_js = 0),
 * COMPLETED iff C <= RS (z_js = C), otherwise PENDING (R7).  Every op of a
 * new job is PENDING.  RUNNING ops keep their machine and draw power until
 * C (R3).
 *   orig_assign, orig_start: host [n*g] plan of the original jobs, row-major
 *     [j][s]; both NULL means "no plan": every op is PENDING (static problem).
 *   K_out: number of pending ops = genes per chromosome (g(n+n') - r, R11).
 * The canonical gene order is the pending cells in row-major order
 * (job-major, stage-minor); ffs_state_genes reports it.
 * Errors: FFS_ERR_INVALID_SCHEDULE if the plan violates Eqs. (4)-(7);
 * FFS_ERR_INVALID_ARG if WT * sum T + C_max could reach 1e17 (the 64-bit
 * objective word and its E_max = 10^a, must stay below 2^63).
 * ---------------------------------------------------------------------- */
FFS_API ffs_status ffs_reschedule_state(const ffs_instance *inst, int32_t rs, const int32_t *orig_assign,
                                const int32_t *orig_start, ffs_state **out, int32_t *K_out);
/* ------------------------------------------------------------------------
 * Traditional static approach ("they could only be scheduled after
 * completing the operations of the original schedule at each stage",
 * P:313-317 Fig. 7).  Same freeze rule as
 * ffs_reschedule_state for RUNNING / COMPLETED ops, but every other original
 * op is KEPT at its plan (cell state 3) instead of becoming pending: only the
 * arrivals' ops are genes (K = n'*g).  KEPT ops hold their machine and draw
 * power over their planned interval, so every arrival op starts after the last
 * original op on its machine (reading R29) and shares Q_max with them (R30).
 * The same ffs_evaluate / ffs_evolve / ffs_best run on the returned state.
 *   orig_assign, orig_start: host [n*g] plan, required when n > 0.
 * Errors: FFS_ERR_INVALID_ARG without a plan, FFS_ERR_INVALID_SCHEDULE if the
 * plan violates Eqs. (4)-(7).
 * ---------------------------------------------------------------------- */
FFS_API ffs_status ffs_static_state(const ffs_instance *inst, int32_t rs, const int32_t *orig_assign,
                                    const int32_t *orig_start, ffs_state **out, int32_t *K_out);
/* Host [K] arrays: job and stage of each gene (either may be NULL). */
FFS_API ffs_status ffs_state_genes(const ffs_state *st, int32_t *gene_job, int32_t *gene_stage);
/* Host [(n+n')*g]: 0 pending, 1 running, 2 completed, 3 kept (static policy). */
FFS_API ffs_status ffs_state_cells(const ffs_state *st, int32_t *cell_state);
/* Number of cells with row-major position < p, for p in [0, (n+n')*g]:
 * the compact cut of a row-major crossover point (R13).  Host [cells+1]. */
FFS_API ffs_status ffs_state_cut_table(const ffs_state *st, int32_t *pending_before);
/* Horizon capacity (time slots) of the in-SMEM power profile.  A chromosome
 * whose schedule outgrows it is re-decoded exactly, with identical results:
 * (uniform power, once the state has seen an overflow) first by the lane
 * decoder over a longer horizon, then by the warp-per-chromosome fallback over
 * the proven bound (its profile in shared memory when it fits, else global
 * memory).  cap <= 0 restores the automatic choice.  (Testing/tuning knob.) */
FFS_API ffs_status ffs_state_set_horizon_cap(ffs_state *st, int32_t cap);
FFS_API ffs_status ffs_state_info(const ffs_state *st, int32_t *K, int32_t *cells, int32_t *horizon_cap,
                          int32_t *horizon_bound, int32_t *smem_bytes_per_cta);
/* Which decode path ffs_evaluate takes for this state (diagnostic; host
 * pointers, each may be NULL): *lane_path = 1 for the lane path (order kernel
 * + lane-per-chromosome decode: P <= 8, Q_max <= 127, the order kernel's
 * shared memory fits, and every job's pending genes fit the order kernel's
 * u16 gene key: max_pending <= 2^(16 - ceil(log2 K))), else 0 (the general
 * warp-per-chromosome kernel, same results); *lane_mode = the lane decoder's
 * profile mode (2: uniform power, headroom bit planes; 0/1: byte levels);
 * *max_pending = the most pending genes of one job. */
FFS_API ffs_status ffs_state_path(const ffs_state *st, int32_t *lane_path, int32_t *lane_mode, int32_t *max_pending);
FFS_API void ffs_state_destroy(ffs_state *st);

/* ------------------------------------------------------------------------
 * Fractional WT (Table 11).  Switches the state to
 * Eq. (1) with a real weight: objective = fl(fl(WT * sum T_j) + C_max) in
 * IEEE-754 binary64 (two roundings, no fused multiply-add), fitness (Eq. (13))
 * = max(E_max - objective, +0) and E_max = the smallest 10^a above
 * every initial objective, all in binary64.  From then on every `objective`,
 * `fitness`, E_max and trace word of ffs_evaluate / ffs_evaluate_host /
 * ffs_run_* / ffs_best is the 64-bit pattern of that double (reinterpret it);
 * the trace sum is a fixed-order binary64 sum.  Decoding does not depend on
 * WT.  wt: finite, >= 0.  Call before ffs_evolve_begin; a run keeps the mode
 * it started with only if the state is not switched again while it runs.
 * Errors: FFS_ERR_INVALID_ARG for a negative or non-finite wt, or one for
 * which WT * sum T + C_max could reach 1e300 (the state is then unchanged).
 * ---------------------------------------------------------------------- */
FFS_API ffs_status ffs_state_set_objective_weight(ffs_state *st, double wt);

/* ------------------------------------------------------------------------
 * Decode + evaluate (Algorithm 1; Algorithm 2, P:273-289;
 * Eqs. (1)-(3)).  Algorithm 1 runs one WARP per chromosome (a
 * counting sort, order_warp_kernel); Algorithm 2 runs one LANE per chromosome
 * (lane_decode*_kernel: its per-dispatch work is scalar and sequential) when
 * the instance fits the lane decoder (P <= 8, Q_max <= 127, ...), else one
 * warp per chromosome with a 32-tick ballot window (evaluate_kernel); the
 * results are identical.
 * Streams: every device-pointer call on a state shares the state's scratch
 * (overflow lists, the order->decode buffer); a call issued on another stream
 * than the previous call is ordered after it (event), so calls on several
 * streams are correct but do not overlap each other.
 *   x: device int8  [count*K], machine of each gene, in [0, o-1] (X(k))
 *   y: device int16 [count*K], priorities: a permutation of 1..K per
 *      chromosome, larger = earlier (Y(k)).  Not validated.
 *   objective:       device int64 [count], WT*sum T_j + C_max     (may be NULL;
 *                    binary64 bit patterns after ffs_state_set_objective_weight)
 *   total_tardiness: device int64 [count], sum_j T_j over J u J'   (may be NULL)
 *   makespan:        device int32 [count], C_max                   (may be NULL)
 *   start_out:       device int32 [count*(n+n')*g], S_js of the merged schedule
 *                    (frozen ops keep their plan start)           (may be NULL)
 * ---------------------------------------------------------------------- */
FFS_API ffs_status ffs_evaluate(const ffs_state *st, int64_t count, const int8_t *x, const int16_t *y,
                        int64_t *objective, int64_t *total_tardiness, int32_t *makespan,
                        int32_t *start_out, void *cuda_stream);
/* Same with a row stride: chromosome c's genes are x[c*row .. c*row+K) and
 * y[c*row .. c*row+K) (row = 0 means K).  row >= K; with row % 16 == 0 and
 * 16-byte aligned x, y the order kernel stages whole rows by TMA bulk copies
 * (the GA's own padded population layout).  Errors: FFS_ERR_INVALID_ARG for
 * 0 < row < K; otherwise as ffs_evaluate. */
FFS_API ffs_status ffs_evaluate_strided(const ffs_state *st, int64_t count, const int8_t *x, const int16_t *y,
                                        int64_t row, int64_t *objective, int64_t *total_tardiness,
                                        int32_t *makespan, int32_t *start_out, void *cuda_stream);
/* Same with HOST buffers (pageable or pinned): copies in, evaluates, copies
 * out, synchronises.  Ordered after earlier work on cuda_stream.  Large
 * batches run as a pipeline of up to 4 chunks on two internal streams (chunk
 * i's host->device copy overlaps chunk i-1's decode and result copy-out);
 * results are identical to ffs_evaluate.  Used for end-to-end timing. */
FFS_API ffs_status ffs_evaluate_host(const ffs_state *st, int64_t count, const int8_t *x, const int16_t *y,
                             int64_t *objective, int64_t *total_tardiness, int32_t *makespan,
                             void *cuda_stream);
/* ------------------------------------------------------------------------
 * Brute force over the decoder-reachable set:
 * every X in [0, o-1]^K times every linear extension of the job chains (the
 * orders Algorithm 1 can produce; o^K * K!/prod_j L_j! of them,
 * L_j = pending ops of job j), each decoded by the ffs_evaluate kernels.
 * Enumeration index i = order_rank * o^K + x_rank (x_rank = K base-o digits,
 * gene g = digit g; order_rank = multinomial rank, jobs ascending); the
 * chromosome of an order has y = K - position.  Ties -> lowest index.
 *   limit: maximum number of decodes; FFS_ERR_INVALID_ARG beyond it, for
 *          K = 0, K > 64 or more than 64 jobs with pending ops.
 *   best_objective: host, the minimum objective word (binary64 pattern in
 *          real-WT mode); evaluated: host, the number of decodes;
 *   best_x [K], best_y [K]: host, a chromosome reaching it (may be NULL).
 * Synchronises `cuda_stream`.
 * ---------------------------------------------------------------------- */
FFS_API ffs_status ffs_brute_force(const ffs_state *st, int64_t limit, int64_t *best_objective, int64_t *evaluated,
                                   int8_t *best_x, int16_t *best_y, void *cuda_stream);
/* Counter-based random chromosomes (the GA's initialisation operator,
 * P:227): chromosome id -> island id>>20, individual id&(2^20-1); device
 * x [count*K], y [count*K]. */
FFS_API ffs_status ffs_random_population(const ffs_state *st, int64_t count, uint64_t seed, int64_t first_id,
                                 int8_t *x, int16_t *y, void *cuda_stream);
/* Same into rows of `row` genes (row >= K; genes K..row-1 untouched): the
 * padded layout of ffs_evaluate_strided.  row = 0 means K. */
FFS_API ffs_status ffs_random_population_strided(const ffs_state *st, int64_t count, uint64_t seed,
                                                 int64_t first_id, int64_t row, int8_t *x, int16_t *y,
                                                 void *cuda_stream);

/* ------------------------------------------------------------------------
 * Island GA of one rescheduling point.
 * Population layout: global island I owns cells I*island_w*island_h + i,
 * i row-major in the island tile.  This process holds islands
 * [island_begin, island_end).  The random stream is keyed by
 * (seed, purpose, island, generation, individual, gene), so a shard never
 * changes a draw.
 * Collective hooks: NULL when islands_total == island_end - island_begin.
 *   allreduce_max_i64: replace *dev_val (device int64) by its max over all
 *     processes, stream-ordered on `stream`.  Return 0 on success.
 *   allgather: gather bytes_per_rank from every process into recv_dev
 *     (rank-major), stream-ordered.  Return 0 on success.
 * ---------------------------------------------------------------------- */
typedef struct {
  int32_t island_w, island_h;           /* tile; island_w even (pairs, R19)           */
  int32_t islands_total;                /* global island count                         */
  int32_t island_begin, island_end;     /* this process's shard                        */
  uint32_t xo_threshold;                /* crossover iff u32 < thr; 0.9 -> 3865470566  */
  uint32_t mut_threshold;               /* mutation iff u32 < thr; 0.1 -> 429496729    */
  int32_t migration_interval;           /* 10                           */
  int32_t generations;                  /* G                                           */
  uint64_t seed;
  int32_t rank, world;                  /* position of this shard in the ring          */
  int (*allreduce_max_i64)(void *user, int64_t *dev_val, void *stream);
  int (*allgather)(void *user, const void *send_dev, void *recv_dev, size_t bytes_per_rank,
                   void *stream);
  void *user;
} ffs_ga_config;

/* Generation 0: initialise, evaluate, E_max (global via the
 * allreduce hook, R23), fitness (Eq. (13)), per-island history elite.
 * Errors: FFS_ERR_INVALID_ARG for a bad tile/shard/rank, or world > 1
 * without BOTH hooks. */
FFS_API ffs_status ffs_evolve_begin(ffs_state *st, const ffs_ga_config *cfg, void *cuda_stream, ffs_run **out);
/* Run `generations` more generations (selection, crossover + correction,
 * mutation, evaluation, elitist replacement, ring migration every
 * migration_interval, trace).  Asynchronous except around hook calls. */
FFS_API ffs_status ffs_evolve_step(ffs_run *run, int32_t generations);
/* begin + step(cfg->generations) + synchronise.  K == 0: returns a run whose
 * best is the frozen plan and whose trace is empty. */
FFS_API ffs_status ffs_evolve(ffs_state *st, const ffs_ga_config *cfg, void *cuda_stream, ffs_run **out);
/* Best-in-history of THIS SHARD (ties -> lowest island) and its decoded,
 * merged schedule.  Host outputs, any may be NULL:
 *   x [K], y [K], assign/start [(n+n')*g], trace_min/trace_sum [G+1] (local
 *   shard: min objective and sum of objectives per generation).
 * Sharded runs: the global best of the ring and the global trace
 * are the reduction of every shard's ffs_best over the process group --
 * min objective, ties -> lowest rank (= lowest global island), trace min of
 * mins and sum of sums (paper_1903_10741_b200.dist.global_best). */
FFS_API ffs_status ffs_best(ffs_run *run, int8_t *x, int16_t *y, int32_t *assign, int32_t *start,
                    int64_t *objective, int64_t *total_tardiness, int32_t *makespan,
                    int64_t *trace_min, int64_t *trace_sum);
/* Host copies of the shard population (cells_local*K genes), its
 * objective/fitness, the per-island history elites, E_max and generation. */
FFS_API ffs_status ffs_run_population(ffs_run *run, int8_t *x, int16_t *y, int64_t *objective, int64_t *fitness);
FFS_API ffs_status ffs_run_history(ffs_run *run, int8_t *x, int16_t *y, int64_t *objective, int64_t *fitness);
FFS_API ffs_status ffs_run_info(const ffs_run *run, int32_t *generation, int64_t *emax, int64_t *evaluations,
                        int32_t *kernel_launches);
/* Checkpoint / resume.  A checkpoint of a run after generation k is what the
 * calls above return: ffs_run_population (x, y, objective, fitness words),
 * ffs_run_history (the per-island elites), ffs_run_info (k, E_max word) and
 * ffs_best's trace_min / trace_sum [k+1].  ffs_run_restore loads such a
 * checkpoint into a run created by ffs_evolve_begin with the SAME
 * ffs_ga_config (shape, shard, seed, thresholds, interval, generations >= k;
 * the state must be the same rescheduling point), after which
 * ffs_evolve_step continues at generation k+1 exactly as the uninterrupted
 * run does: every random draw is keyed by (seed, island, generation,
 * individual, gene) and the rest of the run's state is a function of the
 * restored arrays.  Host buffers (copied synchronously), all required when
 * K > 0: x, y [cells_local*K], objective, fitness [cells_local], hx, hy
 * [islands_local*K], hobj, hfit [islands_local], trace_min, trace_sum [k+1];
 * emax = the E_max word.  0 <= generation <= cfg.generations, else
 * FFS_ERR_INVALID_ARG.  K = 0 (nothing evolves): only generation == the run's
 * own counter is accepted; the arrays are not read.  The chromosomes are not
 * re-validated (a checkpoint carries the run's own permutations). */
FFS_API ffs_status ffs_run_restore(ffs_run *run, int32_t generation, const int8_t *x, const int16_t *y,
                           const int64_t *objective, const int64_t *fitness, const int8_t *hx,
                           const int16_t *hy, const int64_t *hobj, const int64_t *hfit, int64_t emax,
                           const int64_t *trace_min, const int64_t *trace_sum);
FFS_API void ffs_run_destroy(ffs_run *run);

#ifdef __cplusplus
}
#endif
#endif /* FFS_H */
