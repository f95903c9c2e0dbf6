/*
 * ffs_oracle.c -- CPU ORACLE for arXiv 1903.10741.  See ffs_oracle.h.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT CODE: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It shares
 * nothing with the CUDA path.  Deliberately plain: no blocking, no fusion,
 * no incremental data structures -- each function follows the paper's
 * statement in its order and notation so that it can be checked by eye.
 *
 * Readings of the paper used here are numbered R1..R26 in DESIGN.md
 * ("Readings") and cited inline.
 */
#include "ffs_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define Z_COMPLETED (-2)   /* the paper's "C" in Z(k) */
#define Z_UNRANKED  (-3)
#define Z_KEPT      (-4)   /* static baseline: original op held at its plan */

struct or_ctx {
  or_instance in;
  int32_t *Pbuf, *Qbuf, *Rbuf, *Dbuf;
  int32_t rs;
  int32_t NJ, cells, K;
  int32_t *state;      /* [cells] OR_PENDING / OR_RUNNING / OR_COMPLETED / OR_KEPT */
  int32_t policy;      /* OR_DYNAMIC or OR_STATIC                         */
  int32_t real_wt;     /* 1: Eq. (1) with the real weight wt_real (Table 11) */
  double wt_real;
  int32_t *fassign;    /* [cells] frozen machine (plan), -1 when pending  */
  int32_t *fstart;     /* [cells] frozen start (plan), -1 when pending    */
  int32_t *gene_cell;  /* [K] pending cells in row-major order            */
  int32_t *cell_gene;  /* [cells] gene index or -1                         */
};

/* ------------------------------------------------------------------ */
/* small helpers                                                       */
/* ------------------------------------------------------------------ */
static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

static int32_t Pjsm(const or_instance *in, int j, int s, int m) {
  return in->P[((int64_t)j * in->g + s) * in->o + m];
}
static int32_t Qjsm(const or_instance *in, int j, int s, int m) {
  return in->Q[((int64_t)j * in->g + s) * in->o + m];
}

/* one committed processing interval [start, end) drawing power q (Eq. (9)) */
typedef struct { int64_t start, end; int64_t q; } interval;

/* Q_t of Eq. (8) at instant t: sum of q over intervals with start <= t < end */
static int64_t level_at(const interval *iv, int n, int64_t t) {
  int64_t L = 0;
  for (int i = 0; i < n; ++i)
    if (iv[i].start <= t && t < iv[i].end) L += iv[i].q;
  return L;
}

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., Random123)                            */
/* ------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += W0; k1 += W1; }
    uint64_t p0 = (uint64_t)M0 * c0;
    uint64_t p1 = (uint64_t)M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* draw word `word` of block `block` for purpose/individual/generation/island
 * (ctr = (purpose<<24 | block, individual, k, island)). */
static uint32_t draw(uint64_t seed, uint32_t purpose, uint32_t block, uint32_t word,
                     uint32_t individual, uint32_t k, uint32_t island) {
  uint32_t ctr[4] = {(purpose << 24) | block, individual, k, island};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  or_philox4x32_10(ctr, key, out);
  return out[word];
}
/* floor(u * n / 2^32) */
static uint32_t bounded(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * n) >> 32); }

/* ------------------------------------------------------------------ */
/* Instance / plan checks                                              */
/* ------------------------------------------------------------------ */
static int check_instance(const or_instance *in) {
  if (!in || in->n < 0 || in->n_prime < 0 || in->n + in->n_prime < 1 || in->g < 1 || in->o < 1)
    return OR_ERR_ARG;
  if (!in->P || !in->Q || !in->R || !in->D || in->wt < 0) return OR_ERR_ARG;
  int NJ = in->n + in->n_prime;
  for (int j = 0; j < NJ; ++j) {
    if (in->D[j] < in->R[j] || in->R[j] < 0) return OR_ERR_ARG;
    for (int s = 0; s < in->g; ++s)
      for (int m = 0; m < in->o; ++m) {
        if (Pjsm(in, j, s, m) <= 0 || Qjsm(in, j, s, m) < 0) return OR_ERR_ARG;
        if (Qjsm(in, j, s, m) > in->q_max) return OR_ERR_INFEASIBLE;
      }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Freeze at RS (Algorithm 1 frozen branch)                 */
/* ------------------------------------------------------------------ */
static int ctx_create(const or_instance *inst, int32_t rs, const int32_t *orig_assign,
                      const int32_t *orig_start, int32_t policy, or_ctx **out) {
  int st = check_instance(inst);
  if (st != OR_OK) return st;
  if (rs < 0 || !out) return OR_ERR_ARG;
  if (policy == OR_STATIC && inst->n > 0 && !(orig_assign && orig_start)) return OR_ERR_ARG;
  int NJ = inst->n + inst->n_prime, g = inst->g, o = inst->o;
  int cells = NJ * g;
  or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
  c->in = *inst;
  size_t tab = (size_t)cells * o;
  c->Pbuf = (int32_t *)malloc(tab * sizeof(int32_t));
  c->Qbuf = (int32_t *)malloc(tab * sizeof(int32_t));
  c->Rbuf = (int32_t *)malloc(NJ * sizeof(int32_t));
  c->Dbuf = (int32_t *)malloc(NJ * sizeof(int32_t));
  memcpy(c->Pbuf, inst->P, tab * sizeof(int32_t));
  memcpy(c->Qbuf, inst->Q, tab * sizeof(int32_t));
  memcpy(c->Rbuf, inst->R, NJ * sizeof(int32_t));
  memcpy(c->Dbuf, inst->D, NJ * sizeof(int32_t));
  c->in.P = c->Pbuf; c->in.Q = c->Qbuf; c->in.R = c->Rbuf; c->in.D = c->Dbuf;
  c->rs = rs; c->NJ = NJ; c->cells = cells; c->policy = policy;
  c->state = (int32_t *)malloc(cells * sizeof(int32_t));
  c->fassign = (int32_t *)malloc(cells * sizeof(int32_t));
  c->fstart = (int32_t *)malloc(cells * sizeof(int32_t));
  c->cell_gene = (int32_t *)malloc(cells * sizeof(int32_t));
  c->gene_cell = (int32_t *)malloc((cells + 1) * sizeof(int32_t));

  const or_instance *in = &c->in;
  if (orig_assign && orig_start) {
    /* the original plan must itself satisfy Eqs. (4)-(7) over J */
    for (int j = 0; j < inst->n; ++j)
      for (int s = 0; s < g; ++s) {
        int32_t m = orig_assign[j * g + s];
        if (m < 0 || m >= o || orig_start[j * g + s] < 0) { or_ctx_destroy(c); return OR_ERR_SCHEDULE; }
      }
    for (int j = 0; j < inst->n; ++j) {
      if (orig_start[j * g] < in->R[j]) { or_ctx_destroy(c); return OR_ERR_SCHEDULE; } /* Eq. (4) */
      for (int s = 1; s < g; ++s) {
        int64_t prevC = (int64_t)orig_start[j * g + s - 1] + Pjsm(in, j, s - 1, orig_assign[j * g + s - 1]);
        if (orig_start[j * g + s] < prevC) { or_ctx_destroy(c); return OR_ERR_SCHEDULE; } /* Eq. (5) */
      }
    }
    for (int a = 0; a < inst->n * g; ++a)      /* Eq. (6), read symmetrically (R-M7) */
      for (int b = a + 1; b < inst->n * g; ++b) {
        int ja = a / g, sa = a % g, jb = b / g, sb = b % g;
        if (sa != sb || orig_assign[a] != orig_assign[b]) continue;
        int64_t ea = (int64_t)orig_start[a] + Pjsm(in, ja, sa, orig_assign[a]);
        int64_t eb = (int64_t)orig_start[b] + Pjsm(in, jb, sb, orig_assign[b]);
        if (orig_start[a] < eb && orig_start[b] < ea) { or_ctx_destroy(c); return OR_ERR_SCHEDULE; }
      }
    for (int a = 0; a < inst->n * g; ++a) {    /* Eq. (7) at every start instant */
      int64_t t = orig_start[a], L = 0;
      for (int b = 0; b < inst->n * g; ++b) {
        int jb = b / g, sb = b % g;
        int64_t e = (int64_t)orig_start[b] + Pjsm(in, jb, sb, orig_assign[b]);
        if (orig_start[b] <= t && t < e) L += Qjsm(in, jb, sb, orig_assign[b]);
      }
      if (L > in->q_max) { or_ctx_destroy(c); return OR_ERR_SCHEDULE; }
    }
  }

  /* Case rules and Algorithm 1's frozen branch:
   * RUNNING iff S_js < RS < S_js + P (z = 0); COMPLETED iff it finished by
   * RS (z = C); everything else, and every op of a new job, is PENDING.
   * Boundaries per R7: C == RS -> COMPLETED, S == RS -> PENDING. */
  int64_t running_power = 0;
  for (int j = 0; j < NJ; ++j)
    for (int s = 0; s < g; ++s) {
      int cell = j * g + s;
      c->state[cell] = OR_PENDING;
      c->fassign[cell] = -1;
      c->fstart[cell] = -1;
      if (j < inst->n && orig_assign && orig_start) {
        int32_t m = orig_assign[cell];
        int64_t S = orig_start[cell];
        int64_t C = S + Pjsm(in, j, s, m);
        if (S < rs && rs < C) {
          c->state[cell] = OR_RUNNING;
          running_power += Qjsm(in, j, s, m);
        } else if (C <= rs) {
          c->state[cell] = OR_COMPLETED;
        } else if (policy == OR_STATIC) {
          /* traditional static approach (Fig. 7): the original
           * jobs keep their schedule in full */
          c->state[cell] = OR_KEPT;
        }
        if (c->state[cell] != OR_PENDING) { c->fassign[cell] = m; c->fstart[cell] = (int32_t)S; }
      }
    }
  if (running_power > in->q_max) { or_ctx_destroy(c); return OR_ERR_INFEASIBLE; }
  /* canonical gene order: pending cells row-major (job-major, stage-minor) */
  int K = 0;
  for (int cell = 0; cell < cells; ++cell) {
    if (c->state[cell] == OR_PENDING) { c->cell_gene[cell] = K; c->gene_cell[K++] = cell; }
    else c->cell_gene[cell] = -1;
  }
  c->K = K;
  *out = c;
  return OR_OK;
}

int or_ctx_create(const or_instance *inst, int32_t rs, const int32_t *orig_assign,
                  const int32_t *orig_start, or_ctx **out) {
  return ctx_create(inst, rs, orig_assign, orig_start, OR_DYNAMIC, out);
}

int or_ctx_create_static(const or_instance *inst, int32_t rs, const int32_t *orig_assign,
                         const int32_t *orig_start, or_ctx **out) {
  return ctx_create(inst, rs, orig_assign, orig_start, OR_STATIC, out);
}

void or_ctx_destroy(or_ctx *c) {
  if (!c) return;
  free(c->Pbuf); free(c->Qbuf); free(c->Rbuf); free(c->Dbuf);
  free(c->state); free(c->fassign); free(c->fstart); free(c->cell_gene); free(c->gene_cell);
  free(c);
}
int32_t or_ctx_K(const or_ctx *c) { return c->K; }
int32_t or_ctx_cells(const or_ctx *c) { return c->cells; }
void or_ctx_states(const or_ctx *c, int32_t *state) { memcpy(state, c->state, c->cells * sizeof(int32_t)); }
void or_ctx_pending_cells(const or_ctx *c, int32_t *cg) { memcpy(cg, c->gene_cell, c->K * sizeof(int32_t)); }

/* ------------------------------------------------------------------ */
/* Algorithm 1                                             */
/* ------------------------------------------------------------------ */
/* Greedy reading (R1): the stage rule (s < s'' => earlier) is kept
 * absolutely by only ranking ops whose predecessor is frozen or already
 * ranked; among those eligible ops the y rule (larger y => earlier) picks
 * the next rank.  y is unique, so there are no ties. */
int or_order(const or_ctx *c, const int32_t *Y, int32_t *Z) {
  int g = c->in.g;
  for (int cell = 0; cell < c->cells; ++cell) {
    if (c->state[cell] == OR_RUNNING) Z[cell] = 0;
    else if (c->state[cell] == OR_COMPLETED) Z[cell] = Z_COMPLETED;
    else if (c->state[cell] == OR_KEPT) Z[cell] = Z_KEPT;
    else Z[cell] = Z_UNRANKED;
  }
  for (int rank = 1; rank <= c->K; ++rank) {
    int best = -1;
    for (int cell = 0; cell < c->cells; ++cell) {
      if (c->state[cell] != OR_PENDING || Z[cell] != Z_UNRANKED) continue;
      int s = cell % g;
      int pred_ok = (s == 0) || c->state[cell - 1] != OR_PENDING || Z[cell - 1] != Z_UNRANKED;
      if (!pred_ok) continue;
      if (best < 0 || Y[cell] > Y[best]) best = cell;
    }
    if (best < 0) return OR_ERR_ARG;
    Z[best] = rank;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Algorithm 2: the decoding rule                          */
/* ------------------------------------------------------------------ */
int or_decode(const or_ctx *c, const int32_t *X, const int32_t *Y, const int32_t *Zin,
              int32_t *assign_out, int32_t *start_out, int64_t *sumT_out,
              int64_t *cmax_out, int64_t *obj_out, or_counters *cnt) {
  const or_instance *in = &c->in;
  int g = in->g, o = in->o, cells = c->cells, K = c->K;
  int64_t rs = c->rs;
  int32_t *Z = (int32_t *)malloc(cells * sizeof(int32_t));
  int32_t *byrank = (int32_t *)malloc((K + 1) * sizeof(int32_t));
  int32_t *asg = (int32_t *)malloc(cells * sizeof(int32_t));
  int64_t *S = (int64_t *)malloc(cells * sizeof(int64_t));
  int64_t *C = (int64_t *)malloc(cells * sizeof(int64_t));
  int64_t *mfree = (int64_t *)malloc((size_t)g * o * sizeof(int64_t));
  interval *iv = (interval *)malloc((cells + 1) * sizeof(interval));
  int64_t *cand = (int64_t *)malloc((cells + 2) * sizeof(int64_t));
  int niv = 0, st = OR_OK;

  if (Zin) memcpy(Z, Zin, cells * sizeof(int32_t));
  else if ((st = or_order(c, Y, Z)) != OR_OK) goto done;
  for (int r = 0; r <= K; ++r) byrank[r] = -1;
  for (int cell = 0; cell < cells; ++cell)
    if (c->state[cell] == OR_PENDING) {
      if (Z[cell] < 1 || Z[cell] > K || byrank[Z[cell]] >= 0) { st = OR_ERR_ARG; goto done; }
      byrank[Z[cell]] = cell;
    }

  /* frozen operations keep their plan; RUNNING ones occupy their machine and
   * draw power until completion (R3); COMPLETED ones are over by RS.  In the
   * static baseline the KEPT original ops do the same over their planned
   * interval, so an arrival op waits for the last original op on its machine
   * ("only be scheduled after completing the operations of the original
   * schedule", reading R29) and shares Q_max with them (R30). */
  for (int s = 0; s < g; ++s)
    for (int m = 0; m < o; ++m) mfree[s * o + m] = rs;
  for (int cell = 0; cell < cells; ++cell) {
    asg[cell] = -1; S[cell] = -1; C[cell] = -1;
    if (c->state[cell] == OR_PENDING) continue;
    int j = cell / g, s = cell % g, m = c->fassign[cell];
    asg[cell] = m;
    S[cell] = c->fstart[cell];
    C[cell] = S[cell] + Pjsm(in, j, s, m);
    if (c->state[cell] == OR_RUNNING || c->state[cell] == OR_KEPT) {
      iv[niv].start = S[cell]; iv[niv].end = C[cell]; iv[niv].q = Qjsm(in, j, s, m); ++niv;
      mfree[s * o + m] = max64(mfree[s * o + m], C[cell]);
    }
  }

  for (int r = 1; r <= K; ++r) {
    int cell = byrank[r];
    int j = cell / g, s = cell % g, m = X[cell];
    if (m < 0 || m >= o) { st = OR_ERR_ARG; goto done; }
    int64_t p = Pjsm(in, j, s, m), q = Qjsm(in, j, s, m);
    /* earliest start allowed by Eq. (10) RS <= S (R8), Eq. (4) release /
     * Eq. (5) predecessor completion, and the machine's previous operation
     * in Z order (append-only R6) */
    int64_t ready = (s == 0) ? (int64_t)in->R[j] : C[cell - 1];
    int64_t t = max64(max64(rs, ready), mfree[s * o + m]);
    if (cnt) cnt->dispatches++;
    for (;;) {
      /* if Q_max >= Q_t + Q_jsm over the whole processing interval (R2):
       * level can only rise at an interval start, so test t and every start
       * inside (t, t+p) in ascending order */
      int nc = 0;
      cand[nc++] = t;
      for (int i = 0; i < niv; ++i)
        if (iv[i].start > t && iv[i].start < t + p) cand[nc++] = iv[i].start;
      for (int a = 1; a < nc; ++a)            /* insertion sort */
        for (int b = a; b > 1 && cand[b - 1] > cand[b]; --b) {
          int64_t tmp = cand[b]; cand[b] = cand[b - 1]; cand[b - 1] = tmp;
        }
      int64_t viol = -1;
      for (int a = 0; a < nc; ++a) {
        if (cnt) cnt->checks++;
        if (level_at(iv, niv, cand[a]) + q > in->q_max) { viol = cand[a]; break; }
      }
      if (viol < 0) break;
      /* "needs be delayed ... until finishing job i' at stage s'", the
       * earliest finished one among the operations processing at that
       * period (R5) */
      int64_t e = -1;
      for (int i = 0; i < niv; ++i)
        if (iv[i].start <= viol && viol < iv[i].end && (e < 0 || iv[i].end < e)) e = iv[i].end;
      t = e;
      if (cnt) cnt->jumps++;
    }
    asg[cell] = m; S[cell] = t; C[cell] = t + p;
    iv[niv].start = t; iv[niv].end = t + p; iv[niv].q = q; ++niv;
    mfree[s * o + m] = t + p;
    if (cnt) cnt->updates++;
  }

  {
    /* Eqs. (1)-(3) over every job of J u J' (R9) */
    int64_t sumT = 0, cmax = 0;
    for (int j = 0; j < c->NJ; ++j) {
      int64_t Cj = C[j * g + g - 1];
      int64_t Tj = Cj - in->D[j];
      if (Tj < 0) Tj = 0;
      sumT += Tj;
      if (Cj > cmax) cmax = Cj;
    }
    if (sumT_out) *sumT_out = sumT;
    if (cmax_out) *cmax_out = cmax;
    if (obj_out) *obj_out = in->wt * sumT + cmax;
  }
  if (assign_out) memcpy(assign_out, asg, cells * sizeof(int32_t));
  if (start_out)
    for (int cell = 0; cell < cells; ++cell) start_out[cell] = (int32_t)S[cell];
done:
  free(Z); free(byrank); free(asg); free(S); free(C); free(mfree); free(iv); free(cand);
  return st;
}

void or_objective(const or_instance *in, const int32_t *assign, const int32_t *start,
                  int64_t *sumT_out, int64_t *cmax_out, int64_t *obj_out) {
  int g = in->g, NJ = in->n + in->n_prime;
  int64_t sumT = 0, cmax = 0;
  for (int j = 0; j < NJ; ++j) {
    int cell = j * g + g - 1;
    int64_t Cj = (int64_t)start[cell] + Pjsm(in, j, g - 1, assign[cell]);  /* Eq. (2)/(3) */
    int64_t Tj = Cj - in->D[j];
    sumT += Tj > 0 ? Tj : 0;
    if (Cj > cmax) cmax = Cj;
  }
  *sumT_out = sumT; *cmax_out = cmax; *obj_out = in->wt * sumT + cmax;      /* Eq. (1) */
}

int64_t or_power_at(const or_instance *in, const int32_t *assign, const int32_t *start, int64_t t) {
  int g = in->g, NJ = in->n + in->n_prime;
  int64_t L = 0;
  for (int cell = 0; cell < NJ * g; ++cell) {
    int j = cell / g, s = cell % g;
    int64_t e = (int64_t)start[cell] + Pjsm(in, j, s, assign[cell]);
    if (start[cell] <= t && t < e) L += Qjsm(in, j, s, assign[cell]);   /* Eqs. (8)-(9) */
  }
  return L;
}

int or_validate(const or_ctx *c, const int32_t *assign, const int32_t *start, int32_t *kinds_out) {
  const or_instance *in = &c->in;
  int g = in->g, o = in->o, cells = c->cells, nviol = 0, kinds = 0;
  for (int cell = 0; cell < cells; ++cell)
    if (assign[cell] < 0 || assign[cell] >= o) { ++nviol; kinds |= 64; }
  if (kinds & 64) { if (kinds_out) *kinds_out = kinds; return nviol; }
  for (int j = 0; j < c->NJ; ++j) {
    if (start[j * g] < in->R[j]) { ++nviol; kinds |= 1; }                    /* Eq. (4) */
    for (int s = 1; s < g; ++s) {
      int64_t prevC = (int64_t)start[j * g + s - 1] + Pjsm(in, j, s - 1, assign[j * g + s - 1]);
      if (start[j * g + s] < prevC) { ++nviol; kinds |= 2; }                 /* Eq. (5) */
    }
  }
  for (int a = 0; a < cells; ++a)
    for (int b = a + 1; b < cells; ++b) {                                    /* Eq. (6) */
      int sa = a % g, sb = b % g;
      if (sa != sb || assign[a] != assign[b]) continue;
      int64_t ea = (int64_t)start[a] + Pjsm(in, a / g, sa, assign[a]);
      int64_t eb = (int64_t)start[b] + Pjsm(in, b / g, sb, assign[b]);
      if (start[a] < eb && start[b] < ea) { ++nviol; kinds |= 4; }
    }
  for (int a = 0; a < cells; ++a)                                            /* Eq. (7) */
    if (or_power_at(in, assign, start, start[a]) > in->q_max) { ++nviol; kinds |= 8; }
  for (int cell = 0; cell < cells; ++cell) {
    if (c->state[cell] == OR_PENDING) {
      if (start[cell] < c->rs) { ++nviol; kinds |= 16; }                     /* Eq. (10) */
    } else if (assign[cell] != c->fassign[cell] || start[cell] != c->fstart[cell]) {
      ++nviol; kinds |= 32;
    }
  }
  if (c->policy == OR_STATIC)     /* arrivals after the originals on each machine (R29) */
    for (int a = 0; a < cells; ++a) {
      if (c->state[a] != OR_PENDING) continue;
      for (int b = 0; b < cells; ++b) {
        if (c->state[b] == OR_PENDING || b % g != a % g || c->fassign[b] != assign[a]) continue;
        if (start[a] < (int64_t)c->fstart[b] + Pjsm(in, b / g, b % g, c->fassign[b])) { ++nviol; kinds |= 128; }
      }
    }
  if (kinds_out) *kinds_out = kinds;
  return nviol;
}

/* ------------------------------------------------------------------ */
/* Eq. (13) and the E_max rule                      */
/* ------------------------------------------------------------------ */
int64_t or_emax(const int64_t *objectives, int64_t count) {
  /* "a is kept increasing from 1 until all individuals' initial objective
   * function values are smaller than E_max" */
  int64_t E = 10;
  for (;;) {
    int all_smaller = 1;
    for (int64_t i = 0; i < count; ++i)
      if (!(objectives[i] < E)) { all_smaller = 0; break; }
    if (all_smaller) return E;
    E *= 10;
  }
}
int64_t or_fitness(int64_t objective, int64_t emax) {
  int64_t f = emax - objective;
  return f > 0 ? f : 0;
}

/* The same two rules over binary64 values (fractional WT, Table 11; exact for
 * integer values below 2^53).  Powers of ten are exact in binary64 up to 1e22. */
double or_emax_real(const double *objectives, int64_t count) {
  double E = 10.0;
  for (;;) {
    int all_smaller = 1;
    for (int64_t i = 0; i < count; ++i)
      if (!(objectives[i] < E)) { all_smaller = 0; break; }
    if (all_smaller) return E;
    E *= 10.0;
  }
}
double or_fitness_real(double objective, double emax) {
  double f = emax - objective;
  return f > 0.0 ? f : 0.0;
}

/* Eq. (1) as a binary64 value in the context's weight mode:
 * integer WT (R25): the exact integer WT*sum T + C_max; real WT (Table 11,
 * P:473-489): fl(fl(WT * sum T) + C_max), two roundings, no fused
 * multiply-add (the library is built with -ffp-contract=off). */
double or_objective_value(const or_ctx *c, int64_t sum_tardiness, int64_t makespan) {
  if (!c->real_wt) return (double)(c->in.wt * sum_tardiness + makespan);
  double weighted = (double)sum_tardiness * c->wt_real;
  return weighted + (double)makespan;
}

int or_ctx_set_real_weight(or_ctx *c, double wt) {
  if (!c || !(wt >= 0.0) || wt > 1e300) return OR_ERR_ARG;
  c->real_wt = 1;
  c->wt_real = wt;
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Brute force over the decoder-reachable set                          */
/* ------------------------------------------------------------------ */
typedef struct {
  const or_ctx *c;
  int32_t *X, *Z, *bestX, *bestZ;
  int64_t best, evaluated;
  int32_t *next_stage;  /* per job: next pending stage to rank */
} bf_state;

static void bf_all_X(bf_state *b) {
  const or_ctx *c = b->c;
  int K = c->K, o = c->in.o;
  int32_t *digit = (int32_t *)calloc(K + 1, sizeof(int32_t));
  for (;;) {
    for (int gi = 0; gi < K; ++gi) b->X[c->gene_cell[gi]] = digit[gi];
    int64_t obj;
    or_decode(c, b->X, NULL, b->Z, NULL, NULL, NULL, NULL, &obj, NULL);
    b->evaluated++;
    if (b->best < 0 || obj < b->best) {
      b->best = obj;
      if (b->bestX) memcpy(b->bestX, b->X, c->cells * sizeof(int32_t));
      if (b->bestZ) memcpy(b->bestZ, b->Z, c->cells * sizeof(int32_t));
    }
    int gi = 0;
    while (gi < K && ++digit[gi] == o) digit[gi++] = 0;
    if (gi == K) break;
  }
  free(digit);
}

static void bf_orders(bf_state *b, int rank) {
  const or_ctx *c = b->c;
  int g = c->in.g;
  if (rank > c->K) { bf_all_X(b); return; }
  for (int j = 0; j < c->NJ; ++j) {
    int s = b->next_stage[j];
    if (s >= g) continue;
    b->Z[j * g + s] = rank;
    b->next_stage[j]++;
    bf_orders(b, rank + 1);
    b->next_stage[j]--;
    b->Z[j * g + s] = Z_UNRANKED;
  }
}

int or_brute_force(const or_ctx *c, int64_t limit, int64_t *best_objective,
                   int64_t *evaluated, int32_t *best_X, int32_t *best_Z) {
  int g = c->in.g, K = c->K;
  /* search size o^K * K! / prod_j L_j! */
  double size = 1.0;
  for (int i = 0; i < K; ++i) size *= c->in.o;
  double orders = 1.0;
  int idx = 1;
  for (int j = 0; j < c->NJ; ++j) {
    int L = 0;
    for (int s = 0; s < g; ++s) L += c->state[j * g + s] == OR_PENDING;
    for (int k = 1; k <= L; ++k) { orders *= (double)idx++; orders /= k; }
  }
  size *= orders;
  if (size > (double)limit) return OR_ERR_LIMIT;
  bf_state b;
  b.c = c; b.best = -1; b.evaluated = 0; b.bestX = best_X; b.bestZ = best_Z;
  b.X = (int32_t *)malloc(c->cells * sizeof(int32_t));
  b.Z = (int32_t *)malloc(c->cells * sizeof(int32_t));
  b.next_stage = (int32_t *)malloc(c->NJ * sizeof(int32_t));
  for (int cell = 0; cell < c->cells; ++cell) {
    b.X[cell] = -1;
    b.Z[cell] = c->state[cell] == OR_RUNNING ? 0 : c->state[cell] == OR_COMPLETED ? Z_COMPLETED
              : c->state[cell] == OR_KEPT ? Z_KEPT : Z_UNRANKED;
  }
  for (int j = 0; j < c->NJ; ++j) {
    int s = 0;
    while (s < g && c->state[j * g + s] != OR_PENDING) ++s;
    b.next_stage[j] = s;
  }
  bf_orders(&b, 1);
  *best_objective = b.best;
  *evaluated = b.evaluated;
  free(b.X); free(b.Z); free(b.next_stage);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* GA operators                                            */
/* ------------------------------------------------------------------ */
void or_repair(const or_ctx *c, int32_t *Y) {
  /* "a correction step is required to replace the duplicate values by the
   * missing values in ascending order" (R14) */
  int K = c->K;
  char *seen = (char *)calloc(K + 2, 1);
  char *dup = (char *)calloc(c->cells, 1);
  for (int cell = 0; cell < c->cells; ++cell) {       /* row-major scan */
    if (c->state[cell] != OR_PENDING) continue;
    int v = Y[cell];
    if (v >= 1 && v <= K && !seen[v]) seen[v] = 1;  /* first occurrence kept */
    else dup[cell] = 1;
  }
  int next_missing = 1;
  for (int cell = 0; cell < c->cells; ++cell) {
    if (!dup[cell]) continue;
    while (seen[next_missing]) ++next_missing;
    Y[cell] = next_missing;
    seen[next_missing] = 1;
  }
  free(seen); free(dup);
}

void or_crossover(const or_ctx *c, const int32_t *XA, const int32_t *YA,
                  const int32_t *XB, const int32_t *YB, int32_t p,
                  int32_t *XA2, int32_t *YA2, int32_t *XB2, int32_t *YB2) {
  /* "a 2D single point crossover is executed for the target machine matrix
   * and the priority matrix respectively": one row-major cut p,
   * shared by X and Y (R13); cells at position >= p are exchanged. */
  for (int cell = 0; cell < c->cells; ++cell) {
    if (cell < p) { XA2[cell] = XA[cell]; YA2[cell] = YA[cell]; XB2[cell] = XB[cell]; YB2[cell] = YB[cell]; }
    else          { XA2[cell] = XB[cell]; YA2[cell] = YB[cell]; XB2[cell] = XA[cell]; YB2[cell] = YA[cell]; }
  }
  or_repair(c, YA2);
  or_repair(c, YB2);
}

void or_mutate(const or_ctx *c, int32_t *X, int32_t *Y, const uint32_t *rx,
               int32_t gene_a, int32_t gene_b) {
  /* "The non-negative elements of the target machine matrix ... are
   * replaced by random values in the range, apart from the original ones.
   * Regarding the priority matrix, two non-negative elements are chosen
   * randomly to exchange the values." (R15) */
  int o = c->in.o, K = c->K;
  if (o >= 2 && rx)
    for (int gi = 0; gi < K; ++gi) {
      int cell = c->gene_cell[gi];
      X[cell] = (X[cell] + 1 + (int32_t)bounded(rx[gi], (uint32_t)(o - 1))) % o;
    }
  if (K >= 2 && gene_a >= 0 && gene_b >= 0 && gene_a != gene_b) {
    int ca = c->gene_cell[gene_a], cb = c->gene_cell[gene_b];
    int32_t t = Y[ca]; Y[ca] = Y[cb]; Y[cb] = t;
  }
}

/* Generation-0 priorities: "y_js(k) is also generated randomly from
 * the range starting from 1 to the amount of unassigned operations ... and
 * the value of each element is unique".  Each gene draws a random key; y of
 * gene gi = 1 + the number of genes h whose key is smaller, or equal with
 * h < gi (ties by gene index), i.e. the rank of the key. */
void or_init_ranks(int32_t K, const uint32_t *keys, int32_t *y) {
  for (int gi = 0; gi < K; ++gi) {
    int rank = 0;
    for (int h = 0; h < K; ++h)
      if (keys[h] < keys[gi] || (keys[h] == keys[gi] && h < gi)) ++rank;
    y[gi] = rank + 1;
  }
}

/* largest fitness, ties -> lowest index (R21, R28) */
int32_t or_argmax_fitness(const double *fit, int32_t n) {
  int32_t b = 0;
  for (int32_t i = 1; i < n; ++i) if (fit[i] > fit[b]) b = i;
  return b;
}
/* smallest fitness, ties -> lowest index (R21) */
int32_t or_argmin_fitness(const double *fit, int32_t n) {
  int32_t w = 0;
  for (int32_t i = 1; i < n; ++i) if (fit[i] < fit[w]) w = i;
  return w;
}

/* Local asteroid selection: "every individual compares its fitness
 * with its four neighbours ... the individual with the largest fitness
 * replaces it".  Tournament over self, N, S, E, W, torus inside the island
 * tile (R17), strictly larger wins so ties go to the earlier of that order
 * (R18).  fit: one island tile [h*w] row-major; winner[cell] = tile index. */
void or_select(const double *fit, int32_t w, int32_t h, int32_t *winner) {
  for (int row = 0; row < h; ++row)
    for (int col = 0; col < w; ++col) {
      int nb[5] = {row * w + col,                      /* self */
                   ((row + h - 1) % h) * w + col,      /* N: row above */
                   ((row + 1) % h) * w + col,          /* S: row below */
                   row * w + (col + 1) % w,            /* E: next column */
                   row * w + (col + w - 1) % w};       /* W: previous column */
      int best = nb[0];
      for (int t = 1; t < 5; ++t) if (fit[nb[t]] > fit[best]) best = nb[t];
      winner[row * w + col] = best;
    }
}

/* One island's breeding from the selected winners (R19, R20):
 * cells (r,2c) and (r,2c+1) of the winner grid pair up; the pair's crossover
 * fires iff xo_fire < xo_threshold (R16) at row-major cut
 * p = 1 + floor(xo_cut * (cells-1) / 2^32) (R13), else both winners are copied;
 * then every cell i mutates iff mut_fire[i] < mut_threshold, with gene draws
 * mut_x[i*K ..] and the Y swap of genes a = floor(mut_a*K/2^32),
 * b = floor(mut_b*(K-1)/2^32) (+1 if b >= a).
 * PX/PY: the island's snapshot [tile*cells]; X/Y: its new cells. */
void or_breed(const or_ctx *c, int32_t w, int32_t h, const int32_t *PX, const int32_t *PY,
              const int32_t *winner, const or_breed_draws *d, int32_t *X, int32_t *Y) {
  int K = c->K, o = c->in.o, cells = c->cells, tile = w * h;
  for (int row = 0; row < h; ++row)
    for (int cp = 0; cp < w / 2; ++cp) {
      int a = row * w + 2 * cp, b = a + 1, pair = row * (w / 2) + cp;
      const int32_t *XA = PX + (size_t)winner[a] * cells, *YA = PY + (size_t)winner[a] * cells;
      const int32_t *XB = PX + (size_t)winner[b] * cells, *YB = PY + (size_t)winner[b] * cells;
      if (d->xo_fire[pair] < d->xo_threshold) {
        int32_t p = 1 + (int32_t)bounded(d->xo_cut[pair], (uint32_t)(cells - 1));
        or_crossover(c, XA, YA, XB, YB, p, X + (size_t)a * cells, Y + (size_t)a * cells,
                     X + (size_t)b * cells, Y + (size_t)b * cells);
      } else {
        memcpy(X + (size_t)a * cells, XA, cells * sizeof(int32_t));
        memcpy(Y + (size_t)a * cells, YA, cells * sizeof(int32_t));
        memcpy(X + (size_t)b * cells, XB, cells * sizeof(int32_t));
        memcpy(Y + (size_t)b * cells, YB, cells * sizeof(int32_t));
      }
    }
  for (int i = 0; i < tile; ++i) {
    if (d->mut_fire[i] >= d->mut_threshold) continue;
    int32_t ga = -1, gb = -1;
    if (K >= 2) {
      ga = (int32_t)bounded(d->mut_a[i], (uint32_t)K);
      gb = (int32_t)bounded(d->mut_b[i], (uint32_t)(K - 1));
      if (gb >= ga) ++gb;
    }
    or_mutate(c, X + (size_t)i * cells, Y + (size_t)i * cells,
              o >= 2 ? d->mut_x + (size_t)i * K : NULL, ga, gb);
  }
}

/* Elitist replacement: "the best individual in history of each
 * island replaces the worst individual of the current generation".  Per
 * island: the history is updated from the evaluated cells only when their
 * best fitness is strictly larger (lowest index among equals); then the
 * worst cell (smallest fitness, lowest index) takes the history elite (R21).
 * X/Y [nisl*tile*cells], obj/fit [nisl*tile]; HX/HY [nisl*cells], hobj/hfit [nisl]. */
void or_replace(int32_t nisl, int32_t tile, int32_t cells, int32_t *X, int32_t *Y,
                double *obj, double *fit, int32_t *HX, int32_t *HY, double *hobj, double *hfit) {
  for (int li = 0; li < nisl; ++li) {
    size_t base = (size_t)li * tile;
    size_t b = base + or_argmax_fitness(fit + base, tile);
    if (fit[b] > hfit[li]) {
      memcpy(HX + (size_t)li * cells, X + b * cells, cells * sizeof(int32_t));
      memcpy(HY + (size_t)li * cells, Y + b * cells, cells * sizeof(int32_t));
      hobj[li] = obj[b]; hfit[li] = fit[b];
    }
    size_t wst = base + or_argmin_fitness(fit + base, tile);
    memcpy(X + wst * cells, HX + (size_t)li * cells, cells * sizeof(int32_t));
    memcpy(Y + wst * cells, HY + (size_t)li * cells, cells * sizeof(int32_t));
    obj[wst] = hobj[li]; fit[wst] = hfit[li];
  }
}

/* Single-ring migration: "the best individual of each island
 * replaces the worst individual of its neighbouring island" on a single
 * ring.  Synchronous (R22): every island's best and worst are found first,
 * then island I's worst takes the best of island I-1 (mod islands_total).
 * This shard holds nisl consecutive islands; its first island receives the
 * last island of the previous shard (rank-1 mod world) through `allgather`
 * (one record per rank: X[cells] int32, Y[cells] int32, obj, fit binary64);
 * world == 1 (or no allgather) closes the ring inside the shard. */
int or_migrate(int32_t nisl, int32_t tile, int32_t cells, int32_t *X, int32_t *Y,
               double *obj, double *fit, int32_t rank, int32_t world,
               int (*allgather)(void *user, const void *send, void *recv, size_t bytes_per_rank),
               void *user) {
  size_t rec = (size_t)cells * 2 * sizeof(int32_t) + 2 * sizeof(double);
  char *donors = (char *)malloc(rec * nisl);
  int *worst = (int *)malloc(nisl * sizeof(int));
  for (int li = 0; li < nisl; ++li) {       /* snapshot first: synchronous */
    size_t base = (size_t)li * tile;
    size_t b = base + or_argmax_fitness(fit + base, tile);
    char *d = donors + rec * li;
    memcpy(d, X + b * cells, cells * sizeof(int32_t));
    memcpy(d + cells * sizeof(int32_t), Y + b * cells, cells * sizeof(int32_t));
    memcpy(d + cells * 2 * sizeof(int32_t), &obj[b], sizeof(double));
    memcpy(d + cells * 2 * sizeof(int32_t) + sizeof(double), &fit[b], sizeof(double));
    worst[li] = (int)(base + or_argmin_fitness(fit + base, tile));
  }
  char *incoming = (char *)malloc(rec);
  int st = OR_OK;
  if (allgather && world > 1) {
    char *all = (char *)malloc(rec * world);
    if (allgather(user, donors + rec * (nisl - 1), all, rec) != 0) st = OR_ERR_ARG;
    memcpy(incoming, all + rec * ((rank + world - 1) % world), rec);
    free(all);
  } else {
    memcpy(incoming, donors + rec * (nisl - 1), rec);
  }
  if (st == OR_OK)
    for (int li = 0; li < nisl; ++li) {
      const char *src = li == 0 ? incoming : donors + rec * (li - 1);
      size_t wst = (size_t)worst[li];
      memcpy(X + wst * cells, src, cells * sizeof(int32_t));
      memcpy(Y + wst * cells, src + cells * sizeof(int32_t), cells * sizeof(int32_t));
      memcpy(&obj[wst], src + cells * 2 * sizeof(int32_t), sizeof(double));
      memcpy(&fit[wst], src + cells * 2 * sizeof(int32_t) + sizeof(double), sizeof(double));
    }
  free(donors); free(worst); free(incoming);
  return st;
}

/* Per-generation trace: smallest objective and the sum of all
 * objectives of nisl islands of `tile` cells.  The sum (R33) is taken island
 * by island: each island's objectives in cell order, then the island sums in
 * island order (exact for the integer objective; for the binary64 objective
 * of f3 it fixes the rounding). */
void or_trace_stats(const double *obj, int64_t nisl, int32_t tile, double *mn, double *sum) {
  double m = obj[0], s = 0.0;
  for (int64_t li = 0; li < nisl; ++li) {
    double p = 0.0;
    for (int32_t i = 0; i < tile; ++i) {
      double v = obj[li * tile + i];
      if (v < m) m = v;
      p += v;
    }
    s += p;
  }
  *mn = m; *sum = s;
}

/* ------------------------------------------------------------------ */
/* threaded evaluation (for baseline timing; results are per-cell)     */
/* ------------------------------------------------------------------ */
typedef struct {
  const or_ctx *c;
  int64_t begin, end;
  const int32_t *Xs, *Ys;        /* matrix form [count*cells] or NULL */
  const int8_t *xc; const int16_t *yc;   /* compact form [count*K]  */
  int64_t *obj, *sumT, *cmax;
  double *value;                 /* Eq. (1) in the context's weight mode */
  int32_t *start;                /* optional merged schedule [count*cells] */
  or_counters cnt;
  int status;
} eval_job;

static void *eval_worker(void *arg) {
  eval_job *w = (eval_job *)arg;
  const or_ctx *c = w->c;
  int32_t *X = NULL, *Y = NULL;
  if (!w->Xs) {
    X = (int32_t *)malloc(c->cells * sizeof(int32_t));
    Y = (int32_t *)malloc(c->cells * sizeof(int32_t));
    for (int cell = 0; cell < c->cells; ++cell) { X[cell] = -1; Y[cell] = -1; }
  }
  for (int64_t i = w->begin; i < w->end; ++i) {
    const int32_t *Xi, *Yi;
    if (w->Xs) { Xi = w->Xs + i * c->cells; Yi = w->Ys + i * c->cells; }
    else {
      for (int gi = 0; gi < c->K; ++gi) {
        X[c->gene_cell[gi]] = w->xc[i * c->K + gi];
        Y[c->gene_cell[gi]] = w->yc[i * c->K + gi];
      }
      Xi = X; Yi = Y;
    }
    int64_t T, M, O;
    int32_t *Si = w->start ? w->start + i * c->cells : NULL;
    int st = or_decode(c, Xi, Yi, NULL, NULL, Si, &T, &M, &O, &w->cnt);
    if (st != OR_OK) { w->status = st; break; }
    if (w->obj) w->obj[i] = O;
    if (w->sumT) w->sumT[i] = T;
    if (w->cmax) w->cmax[i] = M;
    if (w->value) w->value[i] = or_objective_value(c, T, M);
  }
  free(X); free(Y);
  return NULL;
}

static int run_eval(const or_ctx *c, int64_t count, const int32_t *Xs, const int32_t *Ys,
                    const int8_t *xc, const int16_t *yc, int64_t *obj, int64_t *sumT,
                    int64_t *cmax, double *value, int32_t *start, int nthreads, or_counters *cnt) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > count) nthreads = count > 0 ? (int)count : 1;
  eval_job *jobs = (eval_job *)calloc(nthreads, sizeof(eval_job));
  pthread_t *th = (pthread_t *)calloc(nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {           /* static partition */
    jobs[t].c = c;
    jobs[t].begin = count * t / nthreads;
    jobs[t].end = count * (t + 1) / nthreads;
    jobs[t].Xs = Xs; jobs[t].Ys = Ys; jobs[t].xc = xc; jobs[t].yc = yc;
    jobs[t].obj = obj; jobs[t].sumT = sumT; jobs[t].cmax = cmax; jobs[t].value = value;
    jobs[t].start = start;
  }
  if (nthreads == 1) eval_worker(&jobs[0]);
  else {
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, eval_worker, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  int st = OR_OK;
  for (int t = 0; t < nthreads; ++t) {
    if (jobs[t].status != OR_OK) st = jobs[t].status;
    if (cnt) {
      cnt->dispatches += jobs[t].cnt.dispatches; cnt->checks += jobs[t].cnt.checks;
      cnt->jumps += jobs[t].cnt.jumps; cnt->updates += jobs[t].cnt.updates;
    }
  }
  free(jobs); free(th);
  return st;
}

int or_evaluate_batch(const or_ctx *c, int64_t count, const int8_t *x, const int16_t *y,
                      int64_t *objective, int64_t *sum_tardiness, int64_t *makespan,
                      double *value, int32_t nthreads, or_counters *cnt) {
  return run_eval(c, count, NULL, NULL, x, y, objective, sum_tardiness, makespan, value, NULL, nthreads, cnt);
}

int or_evaluate_batch_schedule(const or_ctx *c, int64_t count, const int8_t *x, const int16_t *y,
                               int64_t *objective, int64_t *sum_tardiness, int64_t *makespan,
                               int32_t *start, int32_t nthreads) {
  return run_eval(c, count, NULL, NULL, x, y, objective, sum_tardiness, makespan, NULL, start, nthreads, NULL);
}

/* ------------------------------------------------------------------ */
/* The hybrid island GA (R13-R23)                */
/* ------------------------------------------------------------------ */
struct or_run {
  const or_ctx *c;
  or_ga_cfg cfg;
  int32_t tile, nisl, nloc;          /* cells per island, local islands, local cells */
  int32_t gen;                       /* last completed generation (-1 = fresh) */
  /* objective / fitness values are binary64: exact for the integer
   * objective (< 2^53), and the real-WT objective of Table 11 */
  double emax;
  int32_t *X, *Y;                    /* [nloc*cells] */
  double *obj, *fit;                 /* [nloc] */
  int32_t *HX, *HY;                  /* history elites [nisl*cells] */
  double *hobj, *hfit;
  double *tmin, *tsum;               /* [G+1] local trace */
};

int or_ga_create(const or_ctx *c, const or_ga_cfg *cfg, or_run **out) {
  if (cfg->island_w < 2 || (cfg->island_w & 1) || cfg->island_h < 1) return OR_ERR_ARG;
  if (cfg->island_begin < 0 || cfg->island_end > cfg->islands_total ||
      cfg->island_begin >= cfg->island_end || cfg->generations < 0 || cfg->migration_interval < 1)
    return OR_ERR_ARG;
  or_run *r = (or_run *)calloc(1, sizeof(or_run));
  r->c = c; r->cfg = *cfg;
  r->tile = cfg->island_w * cfg->island_h;
  r->nisl = cfg->island_end - cfg->island_begin;
  r->nloc = r->nisl * r->tile;
  r->gen = -1;
  size_t cells = c->cells;
  r->X = (int32_t *)malloc((size_t)r->nloc * cells * sizeof(int32_t));
  r->Y = (int32_t *)malloc((size_t)r->nloc * cells * sizeof(int32_t));
  r->obj = (double *)malloc(r->nloc * sizeof(double));
  r->fit = (double *)malloc(r->nloc * sizeof(double));
  r->HX = (int32_t *)malloc((size_t)r->nisl * cells * sizeof(int32_t));
  r->HY = (int32_t *)malloc((size_t)r->nisl * cells * sizeof(int32_t));
  r->hobj = (double *)malloc(r->nisl * sizeof(double));
  r->hfit = (double *)malloc(r->nisl * sizeof(double));
  r->tmin = (double *)calloc(cfg->generations + 1, sizeof(double));
  r->tsum = (double *)calloc(cfg->generations + 1, sizeof(double));
  *out = r;
  return OR_OK;
}

void or_ga_destroy(or_run *r) {
  if (!r) return;
  free(r->X); free(r->Y); free(r->obj); free(r->fit); free(r->HX); free(r->HY);
  free(r->hobj); free(r->hfit); free(r->tmin); free(r->tsum); free(r);
}

static int32_t *cellX(or_run *r, int idx) { return r->X + (size_t)idx * r->c->cells; }
static int32_t *cellY(or_run *r, int idx) { return r->Y + (size_t)idx * r->c->cells; }

static void evaluate_population(or_run *r) {
  run_eval(r->c, r->nloc, r->X, r->Y, NULL, NULL, NULL, NULL, NULL, r->obj, NULL, r->cfg.nthreads, NULL);
  for (int i = 0; i < r->nloc; ++i) r->fit[i] = or_fitness_real(r->obj[i], r->emax);
}

static void record_trace(or_run *r, int k) {
  or_trace_stats(r->obj, r->nisl, r->tile, &r->tmin[k], &r->tsum[k]);
}

static void set_history(or_run *r, int li, int idx) {
  size_t cells = r->c->cells;
  memcpy(r->HX + li * cells, cellX(r, idx), cells * sizeof(int32_t));
  memcpy(r->HY + li * cells, cellY(r, idx), cells * sizeof(int32_t));
  r->hobj[li] = r->obj[idx]; r->hfit[li] = r->fit[idx];
}

static int ga_init(or_run *r) {
  const or_ctx *c = r->c;
  int K = c->K, o = c->in.o;
  uint64_t seed = r->cfg.seed;
  uint32_t *keys = (uint32_t *)malloc((K + 1) * sizeof(uint32_t));
  int32_t *y = (int32_t *)malloc((K + 1) * sizeof(int32_t));
  for (int li = 0; li < r->nisl; ++li) {
    uint32_t I = (uint32_t)(r->cfg.island_begin + li);
    for (int i = 0; i < r->tile; ++i) {
      int32_t *X = cellX(r, li * r->tile + i), *Y = cellY(r, li * r->tile + i);
      for (int cell = 0; cell < c->cells; ++cell) { X[cell] = -1; Y[cell] = -1; }
      /* "x_js(k) is equal to a random integer representing the target
       * machine"; y from the rank of a random key (or_init_ranks) */
      for (int gi = 0; gi < K; ++gi) {
        X[c->gene_cell[gi]] = (int32_t)bounded(draw(seed, 1, gi / 4, gi % 4, i, 0, I), (uint32_t)o);
        keys[gi] = draw(seed, 2, gi / 4, gi % 4, i, 0, I);
      }
      or_init_ranks(K, keys, y);
      for (int gi = 0; gi < K; ++gi) Y[c->gene_cell[gi]] = y[gi];
    }
  }
  free(keys); free(y);
  /* E_max from every individual's initial objective (R23: global) */
  r->emax = 10.0;   /* placeholder so evaluate_population computes fitness */
  evaluate_population(r);
  double mx = r->obj[0];
  for (int i = 1; i < r->nloc; ++i) if (r->obj[i] > mx) mx = r->obj[i];
  if (r->cfg.allreduce_max && r->cfg.allreduce_max(r->cfg.user, &mx) != 0) return OR_ERR_ARG;
  r->emax = or_emax_real(&mx, 1);
  for (int i = 0; i < r->nloc; ++i) r->fit[i] = or_fitness_real(r->obj[i], r->emax);
  /* generation 0: each island's history elite = its best cell (R27) */
  for (int li = 0; li < r->nisl; ++li)
    set_history(r, li, li * r->tile + or_argmax_fitness(r->fit + (size_t)li * r->tile, r->tile));
  record_trace(r, 0);
  r->gen = 0;
  return OR_OK;
}

static int ga_generation(or_run *r, int k) {
  const or_ctx *c = r->c;
  int K = c->K, cells = c->cells;
  int w = r->cfg.island_w, h = r->cfg.island_h, tile = r->tile;
  uint64_t seed = r->cfg.seed;
  size_t bytes = (size_t)r->nloc * cells * sizeof(int32_t);
  /* snapshot of generation k-1 (synchronous update, R18) */
  int32_t *PX = (int32_t *)malloc(bytes), *PY = (int32_t *)malloc(bytes);
  double *Pfit = (double *)malloc(r->nloc * sizeof(double));
  memcpy(PX, r->X, bytes); memcpy(PY, r->Y, bytes);
  memcpy(Pfit, r->fit, r->nloc * sizeof(double));
  int32_t *winner = (int32_t *)malloc(tile * sizeof(int32_t));
  uint32_t *xo_fire = (uint32_t *)malloc((tile / 2) * sizeof(uint32_t));
  uint32_t *xo_cut = (uint32_t *)malloc((tile / 2) * sizeof(uint32_t));
  uint32_t *mut_fire = (uint32_t *)malloc(tile * sizeof(uint32_t));
  uint32_t *mut_a = (uint32_t *)malloc(tile * sizeof(uint32_t));
  uint32_t *mut_b = (uint32_t *)malloc(tile * sizeof(uint32_t));
  uint32_t *mut_x = (uint32_t *)calloc((size_t)tile * (K + 1), sizeof(uint32_t));
  or_breed_draws d = {r->cfg.xo_threshold, r->cfg.mut_threshold, xo_fire, xo_cut,
                      mut_fire, mut_a, mut_b, mut_x};

  for (int li = 0; li < r->nisl; ++li) {
    uint32_t I = (uint32_t)(r->cfg.island_begin + li);
    size_t base = (size_t)li * tile;
    /* a6: selection on the snapshot */
    or_select(Pfit + base, w, h, winner);
    /* the pair's draws are keyed by its left cell, the mutation's by the
     * cell */
    for (int row = 0; row < h; ++row)
      for (int cp = 0; cp < w / 2; ++cp) {
        uint32_t a = (uint32_t)(row * w + 2 * cp);
        xo_fire[row * (w / 2) + cp] = draw(seed, 3, 0, 0, a, (uint32_t)k, I);
        xo_cut[row * (w / 2) + cp] = draw(seed, 3, 0, 1, a, (uint32_t)k, I);
      }
    for (int i = 0; i < tile; ++i) {
      mut_fire[i] = draw(seed, 4, 0, 0, (uint32_t)i, (uint32_t)k, I);
      mut_a[i] = draw(seed, 4, 0, 1, (uint32_t)i, (uint32_t)k, I);
      mut_b[i] = draw(seed, 4, 0, 2, (uint32_t)i, (uint32_t)k, I);
      if (mut_fire[i] < r->cfg.mut_threshold)   /* gene draws only where read */
        for (int gi = 0; gi < K; ++gi)
          mut_x[(size_t)i * K + gi] = draw(seed, 5, gi / 4, gi % 4, (uint32_t)i, (uint32_t)k, I);
    }
    /* a7 + a8: crossover + correction, then mutation */
    or_breed(c, w, h, PX + base * cells, PY + base * cells, winner, &d,
             cellX(r, (int)base), cellY(r, (int)base));
  }
  free(PX); free(PY); free(Pfit); free(winner);
  free(xo_fire); free(xo_cut); free(mut_fire); free(mut_a); free(mut_b); free(mut_x);

  evaluate_population(r);

  /* a9: elitist replacement */
  or_replace(r->nisl, tile, cells, r->X, r->Y, r->obj, r->fit, r->HX, r->HY, r->hobj, r->hfit);

  /* a10: single-ring migration every migration_interval generations */
  if (k % r->cfg.migration_interval == 0 && r->cfg.islands_total >= 2) {
    int st = or_migrate(r->nisl, tile, cells, r->X, r->Y, r->obj, r->fit, r->cfg.rank,
                        r->cfg.world, r->cfg.allgather, r->cfg.user);
    if (st != OR_OK) return st;
  }
  record_trace(r, k);
  r->gen = k;
  return OR_OK;
}

int or_ga_step(or_run *r) {
  if (r->c->K == 0) return OR_ERR_ARG;
  if (r->gen < 0) return ga_init(r);
  if (r->gen >= r->cfg.generations) return OR_ERR_ARG;
  return ga_generation(r, r->gen + 1);
}
int32_t or_ga_generation(const or_run *r) { return r->gen; }
double or_ga_emax(const or_run *r) { return r->emax; }

void or_ga_population(const or_run *r, int8_t *x, int16_t *y, double *obj, double *fit) {
  const or_ctx *c = r->c;
  for (int i = 0; i < r->nloc; ++i)
    for (int gi = 0; gi < c->K; ++gi) {
      int cell = c->gene_cell[gi];
      if (x) x[(size_t)i * c->K + gi] = (int8_t)r->X[(size_t)i * c->cells + cell];
      if (y) y[(size_t)i * c->K + gi] = (int16_t)r->Y[(size_t)i * c->cells + cell];
    }
  if (obj) memcpy(obj, r->obj, r->nloc * sizeof(double));
  if (fit) memcpy(fit, r->fit, r->nloc * sizeof(double));
}

void or_ga_history(const or_run *r, int8_t *x, int16_t *y, double *obj, double *fit) {
  const or_ctx *c = r->c;
  for (int li = 0; li < r->nisl; ++li)
    for (int gi = 0; gi < c->K; ++gi) {
      int cell = c->gene_cell[gi];
      if (x) x[(size_t)li * c->K + gi] = (int8_t)r->HX[(size_t)li * c->cells + cell];
      if (y) y[(size_t)li * c->K + gi] = (int16_t)r->HY[(size_t)li * c->cells + cell];
    }
  if (obj) memcpy(obj, r->hobj, r->nisl * sizeof(double));
  if (fit) memcpy(fit, r->hfit, r->nisl * sizeof(double));
}

void or_ga_trace(const or_run *r, double *tmin, double *tsum) {
  int n = r->cfg.generations + 1;
  if (tmin) memcpy(tmin, r->tmin, n * sizeof(double));
  if (tsum) memcpy(tsum, r->tsum, n * sizeof(double));
}
