// evaluate.cu -- population-wide decode + evaluate on sm_100a.
//
// One warp per chromosome (persistent grid, chromosomes strided over warps).
// Per CTA: the frozen rescheduling state ("image": P/Q table, gene table,
// machine-free and job-ready times, initial power profile, due dates) is
// staged into shared memory once with cp.async.bulk (TMA) + mbarrier.
// Per warp (shared memory):
//   ord[K]   rank-ordered (gene | machine << 16)      -- Algorithm 1
//   cnt[K]   per-priority segment counts / rank starts (aliased with below)
//   level[h] integer power profile Q_t, one slot per tick after RS (Eq. (8))
//   ready[NJ], mfree[G*O]
// Algorithm 1 (greedy reading R1) is evaluated as a stable sort
// by (prefix-min of y over the job's pending stages desc, stage asc):
// segmented warp scans + a counting sort, O(K/32) warp steps.
// Algorithm 2 is evaluated as "earliest power-feasible start
// >= t0" (R5): a 32-slot window of the profile is tested with one ballot,
// runs of p feasible slots are found with shifts/ands on the ballot mask.
#include <climits>

#include "device_util.cuh"

namespace edffs {
namespace {

using namespace dev;

template <typename LVL>
struct WarpMem {
  uint32_t *ord;
  uint32_t *lbits;
  uint16_t *cnt;
  LVL *level;
  int32_t *ready;
  int32_t *mfree;
};

// per-warp region layout (must match State::build_image's size computation)
template <typename LVL>
__device__ __forceinline__ WarpMem<LVL> carve(unsigned char *base, const ImageHdr &h, bool level_in_smem,
                                              int32_t hcap) {
  auto r16 = [](uint32_t v) { return (v + 15u) & ~15u; };
  WarpMem<LVL> w;
  uint32_t K = (uint32_t)h.K, nt = (K + 31u) / 32u;
  w.ord = (uint32_t *)base;
  base += r16(4u * K);
  w.lbits = (uint32_t *)base;
  base += r16(4u * nt);
  w.cnt = (uint16_t *)base;  // union U
  unsigned char *u = base;
  if (level_in_smem) {
    w.level = (LVL *)u;
    u += r16((uint32_t)hcap * sizeof(LVL));
  } else {
    w.level = nullptr;
  }
  w.ready = (int32_t *)u;
  u += r16(4u * (uint32_t)h.NJ);
  w.mfree = (int32_t *)u;
  return w;
}

// Algorithm 2 for one chromosome.  Returns false when the schedule outgrows
// the profile capacity (the chromosome is then re-decoded by the overflow
// path).  Times are relative to RS.
template <typename LVL, bool SCHED>
__device__ __forceinline__ bool decode(const ImageHdr &h, const unsigned char *img, WarpMem<LVL> &w,
                                       int32_t hcap, int lane, int32_t *__restrict__ start_row) {
  const int K = h.K, G = h.G, O = h.O, NJ = h.NJ, qmax = h.q_max;
  const uint32_t *pq = (const uint32_t *)(img + h.off_pq);
  const uint32_t *ginfo = (const uint32_t *)(img + h.off_ginfo);
  // initial profile (RUNNING ops, R3), ready and machine-free times
  {
    const uint32_t *l0 = (const uint32_t *)(img + h.off_lvl0);
    uint32_t *lw = (uint32_t *)w.level;
    int words = (int)(((int64_t)hcap * (int64_t)sizeof(LVL)) >> 2);
    for (int i = lane; i < words; i += 32) lw[i] = i < h.lvl_words0 ? l0[i] : 0u;
    const int32_t *r0 = (const int32_t *)(img + h.off_ready0);
    const int32_t *m0 = (const int32_t *)(img + h.off_mfree0);
    for (int i = lane; i < NJ; i += 32) w.ready[i] = r0[i];
    for (int i = lane; i < G * O; i += 32) w.mfree[i] = m0[i];
  }
  __syncwarp();
  for (int r = 0; r < K; ++r) {
    uint32_t e = w.ord[r];
    int g = (int)(e & 0xFFFFu);
    int m = (int)((e >> 16) & 0xFFu);
    m = m < O ? m : O - 1;                       // unvalidated input: stay in bounds
    uint32_t gi = ginfo[g < K ? g : 0];
    int j = (int)(gi & 0xFFFFu), s = (int)(gi >> 16);
    uint32_t pqv = pq[(j * G + s) * O + m];
    int p = (int)(pqv & 0xFFFFu), q = (int)(pqv >> 16);
    int mi = s * O + m;
    // t0 = max(RS, release / predecessor completion, machine free) (Eqs. (4),
    // (5), (10); append-only machine sequencing R6)
    int t0 = max(w.ready[j], w.mfree[mi]);
    int thr = qmax - q;
    // earliest t >= t0 with Q_tau + q <= Q_max for all tau in [t, t+p) (R2, R5)
    int c = t0, run = 0, S;
    for (;;) {
      int idx = c + lane;
      int lv = idx < hcap ? (int)w.level[idx] : 0;
      uint32_t b = __ballot_sync(FULL, lv <= thr);
      int first0 = __clz(__brev(~b));
      if (run + first0 >= p) {
        S = c - run;
        break;
      }
      if (p <= 32) {
        uint32_t f = runs_ge(b, p);
        if (f) {
          S = c + __ffs(f) - 1;
          break;
        }
      }
      run = b == FULL ? run + 32 : __clz(~b);
      c += 32;
    }
    int C = S + p;
    if (C > hcap) return false;
    __syncwarp();   // every lane's reads of level / ready / mfree above precede the commit
    for (int k = lane; k < p; k += 32) w.level[S + k] = (LVL)(w.level[S + k] + q);
    w.ready[j] = C;  // every lane stores the same value: no cross-lane hazard
    w.mfree[mi] = C;
    if (SCHED && lane == 0) start_row[j * G + s] = S + h.rs;
    __syncwarp();
  }
  return true;
}

template <typename LVL, bool SCHED, bool FALLBACK>
__global__ void __launch_bounds__(1024, 1) evaluate_kernel(EvalArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  pdl_trigger();
  pdl_wait();
  // the overflow fallback is launched unconditionally (no host round trip);
  // with an empty list every block leaves before staging the image
  if (FALLBACK && *(volatile const int32_t *)a.ovf == 0) return;
  const uint32_t img_bytes = ((const ImageHdr *)a.image)->image_bytes;
  stage_image(smem, a.image, img_bytes, &bar);
  const ImageHdr &h = *(const ImageHdr *)smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  WarpMem<LVL> w = carve<LVL>(smem + img_bytes + (size_t)warp * a.per_warp_bytes, h, !FALLBACK || a.lvl_smem,
                              a.h_cap);
  if (FALLBACK && !a.lvl_smem) w.level = (LVL *)a.lvl_global + (size_t)gw * (size_t)a.h_cap;
  const int64_t count = FALLBACK ? (int64_t)a.ovf[0] : a.count;
  const int K = h.K;
  for (int64_t i = gw; i < count; i += nw) {
    const int64_t c = FALLBACK ? (int64_t)a.ovf[1 + i] : i;
    const int64_t row = a.row > 0 ? a.row : K;
    const int8_t *xr = a.x + c * row;
    const int16_t *yr = a.y + c * row;
    int32_t *srow = SCHED ? a.start_out + c * h.cells : nullptr;
    if (SCHED)
      for (int k = lane; k < h.cells; k += 32) srow[k] = a.fstart[k];
    build_order<0>(h, smem, OrderMem{w.ord, w.lbits, w.cnt}, xr, yr, lane);
    bool ok = decode<LVL, SCHED>(h, smem, w, a.h_cap, lane, srow);
    if (!ok) {
      if (lane == 0) {
        int pos = atomicAdd(&a.ovf[0], 1);
        a.ovf[1 + pos] = (int32_t)c;
      }
      __syncwarp();
      continue;
    }
    // Eqs. (1)-(3) over every job (R9): frozen jobs are constants of the state
    int64_t T = 0;
    int cm = h.frozen_cmax;
    const int32_t *pj = (const int32_t *)(smem + h.off_pjob);
    const int32_t *pd = (const int32_t *)(smem + h.off_pdue);
    for (int k = lane; k < h.n_pjobs; k += 32) {
      int Cr = w.ready[pj[k]];
      int tj = Cr - pd[k];
      if (tj > 0) T += tj;
      cm = max(cm, Cr + h.rs);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      T += __shfl_xor_sync(FULL, T, d);
      cm = max(cm, __shfl_xor_sync(FULL, cm, d));
    }
    T += h.frozen_T;
    if (lane == 0) {
      const int64_t obj = objective_word(h.real_wt, h.wt, h.wt_f, T, cm);
      if (a.obj) a.obj[c] = obj;
      if (a.tard) a.tard[c] = T;
      if (a.cmax) a.cmax[c] = cm;
      if (a.fit) a.fit[c] = fitness_word(h.real_wt, *a.emax, obj);   // Eq. (13)
    }
    __syncwarp();
  }
}

// Counter-based random chromosomes: x ~ U{0..o-1}, y = 1 + rank of a random
// key (ties by gene index).  Warp per chromosome; ranks by a bitonic sort of
// the keys in shared memory (rank_keys_warp).
__global__ void __launch_bounds__(256) random_population_kernel(int32_t K, int32_t NP, int32_t O, int64_t count,
                                                                uint64_t seed, int64_t first_id, int64_t row,
                                                                int8_t *x, int16_t *y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long *buf = (unsigned long long *)smem + (size_t)warp * NP;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; c < count; c += nw) {
    const int64_t id = first_id + c;
    const uint32_t island = (uint32_t)(id >> 20), indiv = (uint32_t)(id & 0xFFFFF);
    for (int g = lane; g < K; g += 32) {
      u32x4 rx = philox((RNG_INIT_X << 24) | (uint32_t)(g >> 2), indiv, 0u, island, k0, k1);
      u32x4 ry = philox((RNG_INIT_Y << 24) | (uint32_t)(g >> 2), indiv, 0u, island, k0, k1);
      x[c * row + g] = (int8_t)bounded(word_of(rx, g & 3), (uint32_t)O);
      buf[g] = ((unsigned long long)word_of(ry, g & 3) << 32) | (uint32_t)g;
    }
    rank_keys_warp(buf, K, NP, lane, y + c * row);
  }
}

template <typename LVL, bool SCHED, bool FB>
ffs_status set_smem_attr(size_t bytes) {
  return ensure_smem_attr((const void *)evaluate_kernel<LVL, SCHED, FB>, bytes);
}

template <typename LVL, bool SCHED>
ffs_status launch_typed(const State &st, const EvalArgs &a0, OvfScratch &scr, cudaStream_t s,
                        int *launches) {
  EvalArgs a = a0;
  a.ovf = scr.list;
  if (!(a.count > 0 && st.lane_ok)) {   // the lane path's first order launch resets them
    FFS_CUDA(cudaMemsetAsync(scr.list, 0, sizeof(int32_t), s));
    FFS_CUDA(cudaMemsetAsync(scr.list2, 0, sizeof(int32_t), s));
  }
  // mode 2's lane path re-decodes its overflow list itself (lane_hcap2) once
  // this state has been seen to overflow (the sticky mapped flag, read
  // without synchronising: an overflow not yet visible here is still caught
  // by the general fallback); the fallback then takes what is left (list2).
  // Decided once per call: both launches below follow the same decision.
  const bool relist = st.lane_ok && st.lane_hcap2 > st.lane_hcap && st.ovf_seen_host &&
                      *(volatile const int32_t *)st.ovf_seen_host != 0;
  a.relist = relist ? 1 : 0;
  a.ovf_seen = st.ovf_seen_dev;
  if (a.count > 0 && st.lane_ok) {
    ffs_status e = launch_lane(st, a, scr, s, launches);
    if (e != FFS_OK) return e;
  } else if (a.count > 0) {
    int64_t need_ctas = (a.count + st.warps_per_cta - 1) / st.warps_per_cta;
    int64_t grid = (int64_t)st.num_sms * st.ctas_per_sm;
    if (need_ctas < grid) grid = need_ctas;
    a.h_cap = st.h_cap;
    a.per_warp_bytes = (int32_t)st.per_warp_bytes;
    ffs_status e = set_smem_attr<LVL, SCHED, false>(st.smem_bytes);
    if (e != FFS_OK) return e;
    FFS_CUDA(launch_pdl(evaluate_kernel<LVL, SCHED, false>, dim3((unsigned)grid), dim3(st.warps_per_cta * 32),
                        st.smem_bytes, s, a));
    if (launches) ++*launches;
  }
  if ((st.lane_ok ? (relist ? st.lane_hcap2 : st.lane_hcap) : st.h_cap) < st.h_bound && a.count > 0) {
    // overflow path: profile of the full proven horizon
    if (relist) a.ovf = scr.list2;
    a.h_cap = st.h_bound;
    a.per_warp_bytes = (int32_t)st.fb_per_warp_bytes;
    a.lvl_global = scr.level;
    a.lvl_smem = st.fb_level_smem ? 1 : 0;
    ffs_status e = set_smem_attr<LVL, SCHED, true>(st.fb_smem_bytes);
    if (e != FFS_OK) return e;
    FFS_CUDA(launch_pdl(evaluate_kernel<LVL, SCHED, true>, dim3((unsigned)st.num_sms), dim3(st.fb_warps_per_cta * 32),
                        st.fb_smem_bytes, s, a));
    if (launches) ++*launches;
  }
  return FFS_OK;
}

}  // namespace

ffs_status launch_evaluate(const State &st, const EvalArgs &a, OvfScratch &scr, cudaStream_t s,
                           int *launches) {
  int64_t fb_warps = (int64_t)st.num_sms * st.fb_warps_per_cta;
  const int32_t cap = st.lane_ok ? st.lane_hcap : st.h_cap;
  ffs_status e = scr.ensure(a.count, cap < st.h_bound && !st.fb_level_smem ? fb_warps * st.h_bound * st.lvl_bytes : 0);
  if (e != FFS_OK) return e;
  const bool sched = a.start_out != nullptr;
  if (st.lvl_bytes == 1)
    return sched ? launch_typed<uint8_t, true>(st, a, scr, s, launches)
                 : launch_typed<uint8_t, false>(st, a, scr, s, launches);
  return sched ? launch_typed<uint16_t, true>(st, a, scr, s, launches)
               : launch_typed<uint16_t, false>(st, a, scr, s, launches);
}

ffs_status launch_random_population(const State &st, int64_t count, uint64_t seed, int64_t first_id, int64_t row,
                                    int8_t *x, int16_t *y, cudaStream_t s) {
  if (count <= 0 || st.K == 0) return FFS_OK;
  int NP = 64;
  while (NP < st.K) NP <<= 1;
  const int warps = (int)std::min<size_t>(8, (size_t)kSmemLimit / ((size_t)NP * 8));
  if (warps < 1) return fail(FFS_ERR_INVALID_ARG, "K too large for random_population");
  size_t smem = (size_t)warps * NP * 8;
  if (smem > 48 * 1024) {
    ffs_status e = ensure_smem_attr((const void *)random_population_kernel, smem);
    if (e != FFS_OK) return e;
  }
  int64_t grid = (count + warps - 1) / warps;
  int64_t cap = (int64_t)st.num_sms * 8;
  if (grid > cap) grid = cap;
  random_population_kernel<<<(unsigned)grid, warps * 32, smem, s>>>(st.K, NP, st.inst->o, count, seed, first_id,
                                                                    row, x, y);
  FFS_CUDA(cudaGetLastError());
  return FFS_OK;
}

}  // namespace edffs
