// state.cu -- instance creation and the freeze at RS (host), device image.
//
// Freeze (Algorithm 1 frozen branch): an original op with plan
// (M, S, C = S + P_jsM) is RUNNING iff S < RS < C, COMPLETED iff C <= RS,
// else PENDING (reading R7); every op of a new job is PENDING.  RUNNING ops
// keep their machine busy and draw power until C (R3).
#include <algorithm>
#include <map>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ffs_common.cuh"

namespace edffs {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
ffs_status fail(ffs_status st, const std::string &msg) {
  set_error(msg);
  return st;
}
ffs_status cuda_fail(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? FFS_ERR_OOM : FFS_ERR_CUDA;
}

ffs_status OvfScratch::alloc(void **p, size_t bytes) {
  if (pooled) FFS_CUDA(cudaMallocAsync(p, bytes, pool));
  else FFS_CUDA(cudaMalloc(p, bytes));
  return FFS_OK;
}
void OvfScratch::free_(void *p) {
  if (!p) return;
  if (pooled) cudaFreeAsync(p, pool);
  else cudaFree(p);
}

ffs_status OvfScratch::ensure(int64_t count, int64_t level_bytes_needed) {
  if (count + 1 > cap) {
    free_(list);
    list = nullptr;
    int64_t c = std::max<int64_t>(count + 1, 1024);
    ffs_status e = alloc((void **)&list, (size_t)2 * c * sizeof(int32_t));
    if (e != FFS_OK) return e;
    list2 = list + c;
    cap = c;
  }
  if (level_bytes_needed > level_bytes) {
    free_(level);
    level = nullptr;
    ffs_status e = alloc(&level, (size_t)level_bytes_needed);
    if (e != FFS_OK) return e;
    level_bytes = level_bytes_needed;
  }
  return FFS_OK;
}

ffs_status launch_evaluate_shared(State &st, const EvalArgs &a, cudaStream_t s) {
  OvfScratch &scr = st.scratch;
  if (!scr.done) FFS_CUDA(cudaEventCreateWithFlags(&scr.done, cudaEventDisableTiming));
  else if (scr.used && scr.last != s) FFS_CUDA(cudaStreamWaitEvent(s, scr.done, 0));
  ffs_status e = launch_evaluate(st, a, scr, s, nullptr);
  if (e != FFS_OK) return e;
  FFS_CUDA(cudaEventRecord(scr.done, s));
  scr.last = s;
  scr.used = true;
  return FFS_OK;
}

void OvfScratch::release() {
  free_(list);
  free_(level);
  free_(ordg);
  list = nullptr;
  list2 = nullptr;
  level = nullptr;
  ordg = nullptr;
  cap = 0;
  level_bytes = 0;
  ordg_elems = 0;
}

ffs_status ensure_smem_attr(const void *kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  FFS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t &d = done[{kernel, dev}];
  if (bytes > d) {
    FFS_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    d = bytes;
  }
  return FFS_OK;
}

void pool_keep(int dev) {
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

static uint32_t r16(uint64_t v) { return (uint32_t)((v + 15) & ~(uint64_t)15); }

// Build the staged image for the current h_cap and choose launch geometry.
ffs_status State::build_image() {
  const Instance &in = *inst;
  const int NJ = in.NJ, G = in.g, O = in.o;
  // --- per-job pending info
  std::vector<int32_t> first_pending(NJ, G);
  for (int j = 0; j < NJ; ++j)
    for (int s = 0; s < G; ++s)
      if (cell_state[j * G + s] == 0) {
        first_pending[j] = s;
        break;
      }
  auto Pof = [&](int j, int s, int m) { return in.P[((size_t)j * G + s) * O + m]; };
  auto Qof = [&](int j, int s, int m) { return in.Q[((size_t)j * G + s) * O + m]; };
  auto comp = [&](int j, int s) {  // completion of a frozen op (plan)
    int cell = j * G + s;
    return (int64_t)fstart[cell] + Pof(j, s, fassign[cell]);
  };
  std::vector<int32_t> ready0(NJ, 0), mfree0((size_t)G * O, 0);
  std::vector<int32_t> pjob, pdue;
  int64_t frozen_T = 0;
  int64_t frozen_cmax = 0;
  int64_t base = 0;
  for (int j = 0; j < NJ; ++j) {
    int s0 = first_pending[j];
    if (s0 < G) {
      // earliest start of the job's first pending op: Eq. (10) RS, Eq. (4) R_j or
      // Eq. (5) completion of the frozen predecessor (R8)
      int64_t t = s0 == 0 ? (int64_t)in.R[j] : comp(j, s0 - 1);
      t = std::max<int64_t>(t, rs);
      ready0[j] = (int32_t)(t - rs);
      base = std::max<int64_t>(base, t - rs);
      pjob.push_back(j);
      pdue.push_back((int32_t)((int64_t)in.D[j] - rs));
    } else {
      int64_t Cj = comp(j, G - 1);  // Eqs. (2)-(3) over J u J' (R9)
      frozen_T += std::max<int64_t>(Cj - in.D[j], 0);
      frozen_cmax = std::max(frozen_cmax, Cj);
    }
  }
  // machine free times and the initial profile from the frozen ops that end
  // after RS: RUNNING ones (R3) and, in the static policy, KEPT ones (R29, R30)
  int64_t Lr = 0;
  struct FrozenIv { int64_t a, c; int32_t q; };      // [a, c) relative to RS
  std::vector<FrozenIv> running;
  for (int j = 0; j < NJ; ++j)
    for (int s = 0; s < G; ++s) {
      int cell = j * G + s;
      if (cell_state[cell] != 1 && cell_state[cell] != 3) continue;
      int m = fassign[cell];
      int64_t Crel = comp(j, s) - rs;
      int64_t Srel = std::max<int64_t>((int64_t)fstart[cell] - rs, 0);
      mfree0[(size_t)s * O + m] = (int32_t)std::max<int64_t>(mfree0[(size_t)s * O + m], Crel);
      base = std::max(base, Crel);
      running.push_back({Srel, Crel, Qof(j, s, m)});
      Lr = std::max(Lr, Crel);
    }
  int64_t sum_p = 0;
  for (int k = 0; k < K; ++k) {
    int j = gene_job[k], s = gene_stage[k];
    int mx = 0;
    for (int m = 0; m < O; ++m) mx = std::max(mx, Pof(j, s, m));
    sum_p += mx;
  }
  // every completion is <= base + sum of the pending ops' longest P
  int64_t hb = base + sum_p + 1;
  hb = (hb + 31) / 32 * 32;
  if (hb >= (int64_t)1 << 30) return fail(FFS_ERR_INVALID_ARG, "time horizon exceeds 2^30 ticks");
  h_bound = (int32_t)hb;
  {
    // every objective stays inside its 64-bit word with room for E_max = 10^a
    // (P:375): C_j <= Cb, sum T <= NJ * Cb, so WT * sum T + C_max < 1e17
    // (integer: E_max <= 1e18 < 2^63) or < 1e300 (binary64, f3)
    const double Cb = (double)std::max<int64_t>((int64_t)rs + hb, frozen_cmax);
    const double objmax = (real_wt ? wt_f : (double)in.wt) * (double)NJ * Cb + Cb;
    if (!(objmax < (real_wt ? 1e300 : 1e17)))
      return fail(FFS_ERR_INVALID_ARG, "WT too large: WT * sum T + C_max could overflow the objective word");
  }

  // --- image layout
  const int nt = (K + 31) / 32;
  uint32_t off = r16(sizeof(ImageHdr));
  ImageHdr H;
  std::memset(&H, 0, sizeof(H));
  H.K = K; H.NJ = NJ; H.G = G; H.O = O; H.rs = rs; H.q_max = in.q_max;
  H.n_pjobs = (int32_t)pjob.size();
  H.wt = in.wt; H.real_wt = real_wt; H.wt_f = wt_f; H.frozen_T = frozen_T; H.frozen_cmax = (int32_t)frozen_cmax; H.cells = cells;
  int32_t qmin = in.q_max, qmaxv = 0, pmax = 0;
  for (size_t i = 0; i < in.Q.size(); ++i) {
    qmin = std::min(qmin, in.Q[i]);
    qmaxv = std::max(qmaxv, in.Q[i]);
    pmax = std::max(pmax, in.P[i]);
  }
  const bool uq = qmin == qmaxv;
  // lane decode profile: nibble headroom when every Q_jsm == 1 and Q_max <= 15
  // mode 2 when every op draws the same power q and at most 15 of them fit
  // under Q_max: the limit is then "at most Q_max / q ops at once" and the
  // headroom counts ops (q = 1 is the paper's Table 5 setting)
  const int lmode = (uq && qmin >= 1 && in.q_max / qmin <= 15 && NJ <= 6144 && G * O <= 768) ? 2 : (uq ? 1 : 0);
  // lane-decode prefix (staged by the lane kernels), then warp-path tables
  H.lane_mode = lmode;
  H.lane_units = lmode == 2 ? in.q_max / qmin : 0;
  // mode 2: 5 words (4 headroom bit planes + blocked bits) per 32 ticks;
  // modes 0/1 take the byte profile lvl0 instead
  H.hn_words0 = lmode == 2 ? (int32_t)(5 * ((Lr + 31) / 32)) : 0;
  H.bn_words0 = 0;
  H.off_hn0 = off; off += r16((uint64_t)H.hn_words0 * 4);
  H.off_bn0 = off; off += r16((uint64_t)H.bn_words0 * 4);
  // mode 2: indexed by gene (g * O + machine: the order kernel's ranks need no
  // per-gene table); modes 0/1: by cell ((j * G + s) * O + machine)
  H.off_pqt = off; off += r16((uint64_t)(lmode == 2 ? K : NJ * G) * O * 4);
  H.off_ready16 = off; off += r16((uint64_t)((NJ + 1) / 2) * 4);
  H.off_mfree16 = off; off += r16((uint64_t)((G * O + 1) / 2) * 4);
  int64_t lvl_bytes0 = Lr * lvl_bytes;
  H.lvl_words0 = (int32_t)((lvl_bytes0 + 3) / 4);
  H.off_lvl0 = off; off += r16((uint64_t)H.lvl_words0 * 4);
  H.off_pjob = off; off += r16((uint64_t)pjob.size() * 4);
  H.off_pdue = off; off += r16((uint64_t)pjob.size() * 4);
  H.lane_image_bytes = off;
  H.off_head = off; off += r16((uint64_t)nt * 4);
  H.off_pq = off; off += r16((uint64_t)NJ * G * O * 4);
  H.off_ginfo = off; off += r16((uint64_t)K * 4);
  H.off_ready0 = off; off += r16((uint64_t)NJ * 4);
  H.off_mfree0 = off; off += r16((uint64_t)G * O * 4);
  H.thr_min = in.q_max - qmin;
  H.uniform_q = uq;
  H.image_bytes = off;
  image_host.assign(off, 0);
  uint8_t *img = image_host.data();
  std::memcpy(img, &H, sizeof(H));
  uint32_t *pq = (uint32_t *)(img + H.off_pq);
  for (size_t i = 0; i < (size_t)NJ * G * O; ++i) pq[i] = (uint32_t)in.P[i] | ((uint32_t)in.Q[i] << 16);
  uint32_t *gi = (uint32_t *)(img + H.off_ginfo);
  uint32_t *hd = (uint32_t *)(img + H.off_head);
  for (int k = 0; k < K; ++k) {
    gi[k] = (uint32_t)gene_job[k] | ((uint32_t)gene_stage[k] << 16);
    if (k == 0 || gene_job[k - 1] != gene_job[k]) hd[k >> 5] |= 1u << (k & 31);
  }
  std::memcpy(img + H.off_ready0, ready0.data(), (size_t)NJ * 4);
  std::memcpy(img + H.off_mfree0, mfree0.data(), (size_t)G * O * 4);
  for (int64_t t = 0; t < Lr; ++t) {
    int64_t L = 0;
    for (auto &rq : running)
      if (rq.a <= t && t < rq.c) L += rq.q;
    if (lvl_bytes == 1) img[H.off_lvl0 + t] = (uint8_t)L;
    else ((uint16_t *)(img + H.off_lvl0))[t] = (uint16_t)L;
  }
  {
    uint32_t *pl = (uint32_t *)(img + H.off_hn0);
    for (int64_t t = 0; t < (int64_t)(H.hn_words0 / 5) * 32; ++t) {
      int64_t L = 0;
      for (auto &rq : running)
        if (rq.a <= t && t < rq.c) L += rq.q;
      const int64_t hr = std::max<int64_t>(0, (in.q_max - L) / std::max(qmin, 1));   // in ops of power q
      uint32_t *w = pl + 5 * (t >> 5);
      for (int b = 0; b < 4; ++b)
        if ((hr >> b) & 1) w[b] |= 1u << (t & 31);
      if (hr == 0) w[4] |= 1u << (t & 31);
    }
  }
  if (!pjob.empty()) {
    std::memcpy(img + H.off_pjob, pjob.data(), pjob.size() * 4);
    std::memcpy(img + H.off_pdue, pdue.data(), pdue.size() * 4);
  }
  {
    uint32_t *pqt = (uint32_t *)(img + H.off_pqt);
    if (lmode == 2) {
      // everything the lane decoder needs about the op of gene k on machine m,
      // precomputed: shift of the job's 10-bit ready field [0:5] | of the
      // machine's field [5:10] | ready word j/3 [10:21] | machine word mi/3
      // [21:29] | p-1 [29:32]
      for (int k = 0; k < K; ++k)
        for (int m = 0; m < O; ++m) {
          const int j = gene_job[k], so = gene_stage[k] * O + m;
          const uint32_t pv = (uint32_t)in.P[(size_t)j * G * O + so];
          pqt[(size_t)k * O + m] = (uint32_t)((j % 3) * 10) | ((uint32_t)((so % 3) * 10) << 5) |
                                   ((uint32_t)(j / 3) << 10) | ((uint32_t)(so / 3) << 21) | ((pv - 1) << 29);
        }
    } else {
      for (int j = 0; j < NJ; ++j)
        for (int so = 0; so < G * O; ++so) {
          const size_t i = (size_t)j * G * O + so;
          pqt[i] = ((uint32_t)in.P[i] & 0xFFu) | (((uint32_t)in.Q[i] & 0xFFu) << 8) | ((uint32_t)j << 16);
        }
    }
    if (lmode == 2) {   // three 10-bit times per word (times >= 1023 overflow to the fallback anyway)
      uint32_t *r10 = (uint32_t *)(img + H.off_ready16);
      for (int j = 0; j < NJ; ++j) r10[j / 3] |= (uint32_t)std::min<int32_t>(ready0[j], 1023) << ((j % 3) * 10);
      uint32_t *m10 = (uint32_t *)(img + H.off_mfree16);
      for (int i = 0; i < G * O; ++i) m10[i / 3] |= (uint32_t)std::min<int32_t>(mfree0[i], 1023) << ((i % 3) * 10);
    } else {
      uint16_t *r16p = (uint16_t *)(img + H.off_ready16);
      for (int j = 0; j < NJ; ++j) r16p[j] = (uint16_t)std::min<int32_t>(ready0[j], 65535);
      uint16_t *m16p = (uint16_t *)(img + H.off_mfree16);
      for (int i = 0; i < G * O; ++i) m16p[i] = (uint16_t)std::min<int32_t>(mfree0[i], 65535);
    }
  }

  // --- geometry: profile capacity and warps per CTA
  auto per_warp = [&](int64_t hcap, bool lvl_smem) -> uint64_t {
    uint64_t u_level = (lvl_smem ? r16((uint64_t)hcap * lvl_bytes) : 0) + r16((uint64_t)NJ * 4) +
                       r16((uint64_t)G * O * 4);
    uint64_t u = std::max<uint64_t>(r16((uint64_t)K * 2), u_level);
    return r16((uint64_t)K * 4) + r16((uint64_t)nt * 4) + u;
  };
  const int64_t budget = kSmemLimit - (int64_t)H.image_bytes - 256;
  if (budget < (int64_t)per_warp(32, true))
    return fail(FFS_ERR_INVALID_ARG, "instance too large: state image + one warp exceed shared memory");
  int64_t hcap;
  if (h_cap_user > 0) {
    hcap = std::min<int64_t>(((int64_t)h_cap_user + 31) / 32 * 32, h_bound);
  } else {
    // largest capacity that keeps 32 resident warps, at least 512 slots, at
    // most the proven bound h_bound
    int64_t fixed = (int64_t)per_warp(0, true);
    int64_t h32 = (budget / kMaxWarpsPerCta - fixed) / lvl_bytes;
    h32 = h32 / 32 * 32;
    hcap = std::min<int64_t>(h_bound, std::max<int64_t>(h32, 512));
  }
  while (hcap > 32 && (int64_t)per_warp(hcap, true) > budget) hcap -= 32;
  h_cap = (int32_t)hcap;
  per_warp_bytes = per_warp(hcap, true);
  warps_per_cta = (int)std::min<int64_t>(kMaxWarpsPerCta, budget / (int64_t)per_warp_bytes);
  smem_bytes = H.image_bytes + (size_t)warps_per_cta * per_warp_bytes;
  // overflow fallback over the proven horizon h_bound: its profile in shared
  // memory when a warp's copy fits (the usual case: ~4.5 KB at config C's
  // K = 1,000), else in global memory
  fb_level_smem = !fb_global_forced && (int64_t)per_warp(h_bound, true) <= budget;
  fb_per_warp_bytes = per_warp(fb_level_smem ? h_bound : 0, fb_level_smem);
  fb_warps_per_cta = (int)std::max<int64_t>(1, std::min<int64_t>(8, budget / (int64_t)fb_per_warp_bytes));
  fb_smem_bytes = H.image_bytes + (size_t)fb_warps_per_cta * fb_per_warp_bytes;

  // --- lane-decode path (one lane per chromosome): eligibility and geometry
  max_pending = 0;
  for (int k = 0, run = 0; k < K; ++k) {   // longest run of one job's pending genes
    run = (k > 0 && gene_job[k] == gene_job[k - 1]) ? run + 1 : 1;
    max_pending = std::max(max_pending, run);
  }
  lane_ok = !lane_disabled && K >= 1 && in.q_max <= 127 && pmax <= 8 && (int64_t)NJ * G * O <= 65536 && lvl_bytes == 1;
  if (lane_ok) {
    const int64_t lbudget = kSmemLimit - (int64_t)H.lane_image_bytes - 3072;   // static smem: mask tables + mbarrier
    const int64_t fixed_words = lmode == 2 ? (NJ + 2) / 3 + (G * O + 2) / 3 : (NJ + 1) / 2 + (G * O + 1) / 2;
    auto words = [&](int64_t hc) {   // + 2 sentinel words of `blocked` (+ mode 2: one dummy plane group)
      return lmode == 2 ? fixed_words + 5 * (hc / 32) + 3 : fixed_words + hc / 4 + hc / 32 + 2;
    };
    // horizon: the proven bound if it fits, else as large as keeps >= 8
    // warps (overflowing chromosomes are re-decoded exactly by the fallback)
    int64_t hc = h_bound;
    const int target_warps = lmode == 2 ? 14 : 8;
    if (words(hc) * 128 * target_warps > lbudget)
      hc = std::max<int64_t>(128, (lbudget / (128 * target_warps) - fixed_words - 3) * 32 / (lmode == 2 ? 5 : 9) /
                                      32 * 32);
    if (h_cap_user > 0) hc = std::min<int64_t>(hc, ((int64_t)h_cap_user + 31) / 32 * 32);
    hc = std::min<int64_t>(hc, lmode == 2 ? 992 : 65504);   // 10-bit times in mode 2
    int warps = (int)std::min<int64_t>(16, lbudget / (words(hc) * 128));
    // order kernel: 32 warps, per warp hist[K] u16 + ord[K] u16 (stride 8*odd)
    ord_hist_bytes = (size_t)((K + 511) / 512 * 512) * 2;                              // u16 [K], steps of 512
    ord_stride = ((size_t)(K + 1) * 2 + 7) / 8 * 8;                                    // ord [K] + dummy slot
    if ((ord_stride / 8) % 2 == 0) ord_stride += 8;
    {
      const size_t ntl = (size_t)(K + 127) / 128;
      ord_smem = 32 * (ord_hist_bytes + ord_stride + ((ntl * 128 * 2 + 15) & ~(size_t)15)) +   // per warp
                 ntl * 128 * 4 * 2 + ntl * 32 * 4 * 2;                                           // gtab, mtab, dtab, btab
      ord_xs_bytes = 32 * ntl * 128;   // per-warp x staging, when it fits
      ord_xs = !ord_xs_disabled && ord_smem + ord_xs_bytes + 2048 <= (size_t)kSmemLimit;
    }
    ord_ctas_per_sm = 1;  // 32 warps x <= 64 registers
    // the order kernel keeps u = K - pm (< K) and g - g_L (< max_pending) in
    // one u16 per gene (keys y << 16 | g, y <= K < 2^15)
    ord_ubits = 1;
    while ((1 << ord_ubits) < K) ++ord_ubits;
    const bool ord_fits = ord_ubits <= 15 && max_pending <= (1 << (16 - ord_ubits));
    if (!ord_fits || warps < 2 || hc < 32 || ord_smem + 2048 > (size_t)kSmemLimit) {   // + static smem
      lane_ok = false;
    } else {
      lane_hcap = (int32_t)hc;
      lane_wpt = (int32_t)words(hc);
      lane_warps_per_cta = warps;
      lane_smem = H.lane_image_bytes + (size_t)warps * lane_wpt * 128;
      lane_ctas_per_sm = 1;
      // mode 2: chromosomes that overflow this horizon are re-decoded by the
      // same lane kernel over the overflow list, with the longest horizon
      // that keeps 4 warps (<= h_bound, <= 992: 10-bit times)
      lane_hcap2 = 0;
      if (lmode == 2 && hc < h_bound && hc < 992 && relist_cap != 0) {
        int64_t h2 = std::min<int64_t>({(h_bound + 31) / 32 * 32, 992,
                                        (lbudget / (128 * 4) - fixed_words - 3) / 5 * 32});
        if (relist_cap > 0) h2 = std::min<int64_t>(h2, ((int64_t)relist_cap + 31) / 32 * 32);
        if (h2 > hc) {
          lane_hcap2 = (int32_t)h2;
          lane_wpt2 = (int32_t)words(h2);
          lane_warps2 = (int)std::min<int64_t>(8, lbudget / (words(h2) * 128));
          lane_smem2 = H.lane_image_bytes + (size_t)lane_warps2 * lane_wpt2 * 128;
        }
      }
    }
  }

  // --- upload
  cudaSetDevice(in.dev);
  if (image_dev) cudaFree(image_dev);
  image_dev = nullptr;
  FFS_CUDA(cudaMalloc(&image_dev, image_host.size()));
  FFS_CUDA(cudaMemcpy(image_dev, image_host.data(), image_host.size(), cudaMemcpyHostToDevice));
  int dev = in.dev;
  FFS_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  // one CTA of up to 32 warps per SM, or more CTAs if they fit
  ctas_per_sm = (int)std::max<int64_t>(1, std::min<int64_t>(64 / warps_per_cta,
                                                           (int64_t)(kSmemLimit + 1024) / (int64_t)(smem_bytes + 1024)));
  return FFS_OK;
}

}  // namespace edffs

using namespace edffs;

extern "C" {

const char *ffs_last_error(void) { return g_last_error.c_str(); }
const char *ffs_version(void) { return "ffs-b200 0.1 (sm_100a)"; }

ffs_status ffs_instance_create(const ffs_instance_desc *d, int cuda_device, ffs_instance **out) {
  if (!d || !out) return fail(FFS_ERR_INVALID_ARG, "null argument");
  if (d->n < 0 || d->n_prime < 0 || d->n + d->n_prime < 1 || d->g < 1 || d->o < 1)
    return fail(FFS_ERR_INVALID_ARG, "sizes: need n, n' >= 0, n + n' >= 1, g >= 1, o >= 1");
  if (d->n + d->n_prime > 65535 || d->o > 127 || (int64_t)d->g * d->o > 4096)
    return fail(FFS_ERR_INVALID_ARG, "limits: n + n' <= 65535, o <= 127, g*o <= 4096");
  if (!d->proc_time || !d->power || !d->release || !d->due) return fail(FFS_ERR_INVALID_ARG, "null array");
  if (d->wt < 0) return fail(FFS_ERR_INVALID_ARG, "WT must be >= 0");
  if (d->q_max < 0 || d->q_max > 65535) return fail(FFS_ERR_INVALID_ARG, "Q_max must be in [0, 65535]");
  const int NJ = d->n + d->n_prime;
  const size_t tab = (size_t)NJ * d->g * d->o;
  for (size_t i = 0; i < tab; ++i) {
    if (d->proc_time[i] < 1 || d->proc_time[i] > 65535)
      return fail(FFS_ERR_INVALID_ARG, "P_jsm must be in [1, 65535]");
    if (d->power[i] < 0 || d->power[i] > 65535) return fail(FFS_ERR_INVALID_ARG, "Q_jsm must be in [0, 65535]");
  }
  for (int j = 0; j < NJ; ++j)
    if (d->release[j] < 0 || d->due[j] < d->release[j])
      return fail(FFS_ERR_INVALID_ARG, "need 0 <= R_j <= D_j");
  for (size_t i = 0; i < tab; ++i)
    if (d->power[i] > d->q_max)
      return fail(FFS_ERR_INFEASIBLE, "some Q_jsm > Q_max: no start satisfies Eq. (7)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev)
    return fail(FFS_ERR_CUDA, "no such CUDA device");
  ffs_instance *h = new ffs_instance();
  Instance &in = h->v;
  in.dev = cuda_device;
  in.n = d->n; in.np = d->n_prime; in.g = d->g; in.o = d->o; in.NJ = NJ;
  in.q_max = d->q_max; in.wt = d->wt;
  in.P.assign(d->proc_time, d->proc_time + tab);
  in.Q.assign(d->power, d->power + tab);
  in.R.assign(d->release, d->release + NJ);
  in.D.assign(d->due, d->due + NJ);
  *out = h;
  return FFS_OK;
}

void ffs_instance_destroy(ffs_instance *inst) { delete inst; }

// policy 0: predictive-reactive complete rescheduling (freeze at RS, every
// other op pending); policy 1: traditional static approach (P:313-315,
// Fig. 7): every original op keeps its plan (cell state 3 = KEPT for those
// not over or running at RS), only the arrivals' ops are genes.
static ffs_status make_state(const ffs_instance *ih, int32_t rs, const int32_t *orig_assign,
                             const int32_t *orig_start, int policy, ffs_state **out, int32_t *K_out) {
  if (!ih || !out) return fail(FFS_ERR_INVALID_ARG, "null argument");
  if (rs < 0) return fail(FFS_ERR_INVALID_ARG, "RS must be >= 0");
  if ((orig_assign == nullptr) != (orig_start == nullptr))
    return fail(FFS_ERR_INVALID_ARG, "orig_assign and orig_start must both be given or both NULL");
  if (policy == 1 && ih->v.n > 0 && !orig_assign)
    return fail(FFS_ERR_INVALID_ARG, "the static policy needs the original plan");
  const Instance &in = ih->v;
  const int G = in.g, O = in.o, n = in.n, NJ = in.NJ;
  auto Pof = [&](int j, int s, int m) { return (int64_t)in.P[((size_t)j * G + s) * O + m]; };
  auto Qof = [&](int j, int s, int m) { return (int64_t)in.Q[((size_t)j * G + s) * O + m]; };
  if (orig_assign) {
    // the plan of the original jobs must satisfy Eqs. (4)-(7)
    for (int c = 0; c < n * G; ++c)
      if (orig_assign[c] < 0 || orig_assign[c] >= O || orig_start[c] < 0)
        return fail(FFS_ERR_INVALID_SCHEDULE, "original plan: machine out of range or negative start");
    std::vector<std::pair<int64_t, int64_t>> ev;  // per-(s,m) intervals check via sort
    for (int j = 0; j < n; ++j) {
      if (orig_start[j * G] < in.R[j]) return fail(FFS_ERR_INVALID_SCHEDULE, "original plan violates Eq. (4)");
      for (int s = 1; s < G; ++s)
        if (orig_start[j * G + s] < orig_start[j * G + s - 1] + Pof(j, s - 1, orig_assign[j * G + s - 1]))
          return fail(FFS_ERR_INVALID_SCHEDULE, "original plan violates Eq. (5)");
    }
    for (int s = 0; s < G; ++s)
      for (int m = 0; m < O; ++m) {
        std::vector<std::pair<int64_t, int64_t>> iv;
        for (int j = 0; j < n; ++j)
          if (orig_assign[j * G + s] == m)
            iv.push_back({orig_start[j * G + s], orig_start[j * G + s] + Pof(j, s, m)});
        std::sort(iv.begin(), iv.end());
        for (size_t k = 1; k < iv.size(); ++k)
          if (iv[k].first < iv[k - 1].second)
            return fail(FFS_ERR_INVALID_SCHEDULE, "original plan violates Eq. (6)");
      }
    // Eq. (7): sweep of +q at starts, -q at completions (completions first)
    std::vector<std::pair<int64_t, int64_t>> sweep;
    for (int j = 0; j < n; ++j)
      for (int s = 0; s < G; ++s) {
        int m = orig_assign[j * G + s];
        int64_t S = orig_start[j * G + s];
        sweep.push_back({S, Qof(j, s, m)});
        sweep.push_back({S + Pof(j, s, m), -Qof(j, s, m)});
      }
    std::sort(sweep.begin(), sweep.end());
    int64_t L = 0;
    for (auto &e : sweep) {
      L += e.second;
      if (L > in.q_max) return fail(FFS_ERR_INVALID_SCHEDULE, "original plan violates Eq. (7)");
    }
  }
  ffs_state *h = new ffs_state();
  State &st = h->v;
  st.inst = &in;
  st.rs = rs;
  st.cells = NJ * G;
  st.cell_state.assign(st.cells, 0);
  st.fassign.assign(st.cells, -1);
  st.fstart.assign(st.cells, -1);
  int64_t running_q = 0;
  for (int j = 0; j < n && orig_assign; ++j)
    for (int s = 0; s < G; ++s) {
      int c = j * G + s, m = orig_assign[c];
      int64_t S = orig_start[c], C = S + Pof(j, s, m);
      int stt = (S < rs && rs < C) ? 1 : (C <= rs ? 2 : (policy == 1 ? 3 : 0));
      st.cell_state[c] = stt;
      if (stt) {
        st.fassign[c] = m;
        st.fstart[c] = (int32_t)S;
      }
      if (stt == 1) running_q += Qof(j, s, m);
    }
  if (running_q > in.q_max) {
    delete h;
    return fail(FFS_ERR_INFEASIBLE, "RUNNING operations at RS exceed Q_max");
  }
  st.pend_before.assign(st.cells + 1, 0);
  for (int c = 0; c < st.cells; ++c) {
    st.pend_before[c + 1] = st.pend_before[c] + (st.cell_state[c] == 0);
    if (st.cell_state[c] == 0) {
      st.gene_cell.push_back(c);
      st.gene_job.push_back(c / G);
      st.gene_stage.push_back(c % G);
    }
  }
  st.K = (int32_t)st.gene_cell.size();
  if (st.K > 32767) {
    delete h;
    return fail(FFS_ERR_INVALID_ARG, "K (pending ops) must be <= 32767 (int16 priorities)");
  }
  st.lvl_bytes = in.q_max <= 255 ? 1 : 2;
  st.lane_disabled = getenv("FFS_DISABLE_LANE") != nullptr;
  st.ord_xs_disabled = getenv("FFS_ORDER_NO_XS") != nullptr;   // test hook: unstaged order kernel
  st.fb_global_forced = getenv("FFS_FALLBACK_GLOBAL") != nullptr;   // test hook: global-memory fallback profile
  if (const char *rc = getenv("FFS_RELIST_CAP")) st.relist_cap = atoi(rc);   // test hook: 0 = no re-decode
  cudaSetDevice(in.dev);
  ffs_status e = st.build_image();
  if (e != FFS_OK) {
    delete h;
    return e;
  }
  std::vector<uint32_t> gbase(std::max(st.K, 1));
  for (int k = 0; k < st.K; ++k) gbase[k] = (uint32_t)((st.gene_job[k] * G + st.gene_stage[k]) * O);
  cudaError_t ce = cudaMalloc(&st.gbase_dev, gbase.size() * 4);
  if (ce == cudaSuccess) ce = cudaMemcpy(st.gbase_dev, gbase.data(), gbase.size() * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMalloc(&st.fstart_dev, (size_t)st.cells * 4);
  if (ce == cudaSuccess) ce = cudaMemcpy(st.fstart_dev, st.fstart.data(), (size_t)st.cells * 4, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess) ce = cudaMalloc(&st.cut_dev, (size_t)(st.cells + 1) * 4);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(st.cut_dev, st.pend_before.data(), (size_t)(st.cells + 1) * 4, cudaMemcpyHostToDevice);
  // sticky "a lane decode overflowed" flag in mapped host memory: set by the
  // device (rare path), read by the host without synchronising (launch_typed)
  if (ce == cudaSuccess) ce = cudaHostAlloc((void **)&st.ovf_seen_host, 4, cudaHostAllocMapped);
  if (ce == cudaSuccess) {
    *(volatile int32_t *)st.ovf_seen_host = 0;
    ce = cudaHostGetDevicePointer((void **)&st.ovf_seen_dev, st.ovf_seen_host, 0);
  }
  if (ce != cudaSuccess) {
    ffs_state_destroy(h);
    return cuda_fail(ce, "state upload");
  }
  *out = h;
  if (K_out) *K_out = st.K;
  return FFS_OK;
}

ffs_status ffs_reschedule_state(const ffs_instance *ih, int32_t rs, const int32_t *orig_assign,
                                const int32_t *orig_start, ffs_state **out, int32_t *K_out) {
  return make_state(ih, rs, orig_assign, orig_start, 0, out, K_out);
}

ffs_status ffs_static_state(const ffs_instance *ih, int32_t rs, const int32_t *orig_assign,
                            const int32_t *orig_start, ffs_state **out, int32_t *K_out) {
  return make_state(ih, rs, orig_assign, orig_start, 1, out, K_out);
}

ffs_status ffs_state_genes(const ffs_state *h, int32_t *gene_job, int32_t *gene_stage) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null state");
  if (gene_job) std::copy(h->v.gene_job.begin(), h->v.gene_job.end(), gene_job);
  if (gene_stage) std::copy(h->v.gene_stage.begin(), h->v.gene_stage.end(), gene_stage);
  return FFS_OK;
}

ffs_status ffs_state_cells(const ffs_state *h, int32_t *cell_state) {
  if (!h || !cell_state) return fail(FFS_ERR_INVALID_ARG, "null argument");
  std::copy(h->v.cell_state.begin(), h->v.cell_state.end(), cell_state);
  return FFS_OK;
}

ffs_status ffs_state_cut_table(const ffs_state *h, int32_t *pb) {
  if (!h || !pb) return fail(FFS_ERR_INVALID_ARG, "null argument");
  std::copy(h->v.pend_before.begin(), h->v.pend_before.end(), pb);
  return FFS_OK;
}

ffs_status ffs_state_set_horizon_cap(ffs_state *h, int32_t cap) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null state");
  h->v.h_cap_user = cap > 0 ? cap : 0;
  cudaSetDevice(h->v.inst->dev);
  return h->v.build_image();
}

ffs_status ffs_state_set_objective_weight(ffs_state *h, double wt) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null state");
  if (!(wt >= 0.0) || wt > 1e300) return fail(FFS_ERR_INVALID_ARG, "WT must be finite and >= 0");
  const int32_t old_real = h->v.real_wt;
  const double old_wt = h->v.wt_f;
  h->v.real_wt = 1;
  h->v.wt_f = wt;
  cudaSetDevice(h->v.inst->dev);
  ffs_status e = h->v.build_image();
  if (e != FFS_OK) {   // keep the state as it was
    std::string msg = ffs_last_error();
    h->v.real_wt = old_real;
    h->v.wt_f = old_wt;
    h->v.build_image();
    return fail(e, msg.c_str());
  }
  return FFS_OK;
}

ffs_status ffs_state_info(const ffs_state *h, int32_t *K, int32_t *cells, int32_t *hcap, int32_t *hb,
                          int32_t *smem) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null state");
  if (K) *K = h->v.K;
  if (cells) *cells = h->v.cells;
  if (hcap) *hcap = h->v.lane_ok ? h->v.lane_hcap : h->v.h_cap;
  if (hb) *hb = h->v.h_bound;
  if (smem) *smem = (int32_t)(h->v.lane_ok ? h->v.lane_smem : h->v.smem_bytes);
  return FFS_OK;
}

ffs_status ffs_state_path(const ffs_state *h, int32_t *lane_path, int32_t *lane_mode, int32_t *max_pending) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null state");
  if (lane_path) *lane_path = h->v.lane_ok ? 1 : 0;
  if (lane_mode) *lane_mode = ((const ImageHdr *)h->v.image_host.data())->lane_mode;
  if (max_pending) *max_pending = h->v.max_pending;
  return FFS_OK;
}

void ffs_state_destroy(ffs_state *h) {
  if (!h) return;
  State &st = h->v;
  if (st.image_dev) cudaFree(st.image_dev);
  if (st.fstart_dev) cudaFree(st.fstart_dev);
  if (st.cut_dev) cudaFree(st.cut_dev);
  if (st.gbase_dev) cudaFree(st.gbase_dev);
  if (st.ovf_seen_host) cudaFreeHost(st.ovf_seen_host);
  st.scratch.release();
  if (st.scratch.done) cudaEventDestroy(st.scratch.done);
  st.stage.release();
  st.stage.release_streams();
  delete h;
}

ffs_status ffs_evaluate(const ffs_state *h, int64_t count, const int8_t *x, const int16_t *y, int64_t *objective,
                        int64_t *total_tardiness, int32_t *makespan, int32_t *start_out, void *stream) {
  return ffs_evaluate_strided(h, count, x, y, 0, objective, total_tardiness, makespan, start_out, stream);
}

ffs_status ffs_evaluate_strided(const ffs_state *h, int64_t count, const int8_t *x, const int16_t *y, int64_t row,
                                int64_t *objective, int64_t *total_tardiness, int32_t *makespan, int32_t *start_out,
                                void *stream) {
  if (!h || count < 0) return fail(FFS_ERR_INVALID_ARG, "bad state or count");
  if (row != 0 && row < h->v.K) return fail(FFS_ERR_INVALID_ARG, "row stride must be 0 or >= K");
  if (count > 0 && h->v.K > 0 && (!x || !y)) return fail(FFS_ERR_INVALID_ARG, "null chromosome arrays");
  if (count > ((int64_t)1 << 31) - 2) return fail(FFS_ERR_INVALID_ARG, "count must be < 2^31");
  State &st = const_cast<State &>(h->v);
  cudaSetDevice(st.inst->dev);
  EvalArgs a{};
  a.image = st.image_dev;
  a.count = count;
  a.x = x;
  a.y = y;
  a.obj = objective;
  a.tard = total_tardiness;
  a.cmax = makespan;
  a.start_out = start_out;
  a.fstart = st.fstart_dev;
  a.row = row;
  return launch_evaluate_shared(st, a, (cudaStream_t)stream);
}

ffs_status ffs_evaluate_host(const ffs_state *h, int64_t count, const int8_t *x, const int16_t *y,
                             int64_t *objective, int64_t *total_tardiness, int32_t *makespan, void *stream) {
  if (!h || count < 0) return fail(FFS_ERR_INVALID_ARG, "bad state or count");
  State &st = const_cast<State &>(h->v);
  cudaSetDevice(st.inst->dev);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t gb = (size_t)count * st.K;
  // persistent device staging (grow-only), owned by the state
  HostStage &hs = st.stage;
  if (count > hs.cap || gb > hs.gene_cap) {
    hs.release();
    const size_t c = (size_t)std::max<int64_t>(count, 1), g = std::max<size_t>(gb, 1);
    FFS_CUDA(cudaMalloc(&hs.x, g));
    FFS_CUDA(cudaMalloc(&hs.y, g * 2));
    FFS_CUDA(cudaMalloc(&hs.obj, c * 8));
    FFS_CUDA(cudaMalloc(&hs.T, c * 8));
    FFS_CUDA(cudaMalloc(&hs.M, c * 4));
    hs.cap = (int64_t)c;
    hs.gene_cap = g;
  }
  if (!hs.copy) {
    FFS_CUDA(cudaStreamCreateWithFlags(&hs.copy, cudaStreamNonBlocking));
    FFS_CUDA(cudaStreamCreateWithFlags(&hs.comp, cudaStreamNonBlocking));
    for (cudaEvent_t &e : hs.ev) FFS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // Chunked pipeline: chunk i's host->device copy (copy stream) overlaps chunk
  // i-1's decode and its results' device->host copy (compute stream); the
  // call is ordered after earlier work on `stream` and synchronous on return.
  const int K = st.K;
  const int nch = count >= 4 * 8192 ? 4 : (count >= 2 * 8192 ? 2 : 1);
  FFS_CUDA(cudaEventRecord(hs.ev[8], s));
  FFS_CUDA(cudaStreamWaitEvent(hs.copy, hs.ev[8], 0));
  FFS_CUDA(cudaStreamWaitEvent(hs.comp, hs.ev[8], 0));
  for (int c = 0; c < nch; ++c) {
    const int64_t a0 = count * c / nch, n = count * (c + 1) / nch - a0;
    const size_t g0 = (size_t)a0 * K, gn = (size_t)n * K;
    if (gn) {
      FFS_CUDA(cudaMemcpyAsync(hs.x + g0, x + g0, gn, cudaMemcpyHostToDevice, hs.copy));
      FFS_CUDA(cudaMemcpyAsync(hs.y + g0, y + g0, gn * 2, cudaMemcpyHostToDevice, hs.copy));
    }
    FFS_CUDA(cudaEventRecord(hs.ev[c], hs.copy));
    FFS_CUDA(cudaStreamWaitEvent(hs.comp, hs.ev[c], 0));
    t_plain_launches = 1;   // the chunk's first kernel follows the copy-stream event: plain order
    ffs_status rc = ffs_evaluate(h, n, hs.x + g0, hs.y + g0, hs.obj + a0, hs.T + a0, hs.M + a0, nullptr, hs.comp);
    t_plain_launches = 0;
    if (rc != FFS_OK) return rc;
    if (objective)
      FFS_CUDA(cudaMemcpyAsync(objective + a0, hs.obj + a0, (size_t)n * 8, cudaMemcpyDeviceToHost, hs.comp));
    if (total_tardiness)
      FFS_CUDA(cudaMemcpyAsync(total_tardiness + a0, hs.T + a0, (size_t)n * 8, cudaMemcpyDeviceToHost, hs.comp));
    if (makespan)
      FFS_CUDA(cudaMemcpyAsync(makespan + a0, hs.M + a0, (size_t)n * 4, cudaMemcpyDeviceToHost, hs.comp));
  }
  FFS_CUDA(cudaEventRecord(hs.ev[8], hs.comp));
  FFS_CUDA(cudaStreamWaitEvent(s, hs.ev[8], 0));
  FFS_CUDA(cudaStreamSynchronize(hs.comp));
  return FFS_OK;
}

ffs_status ffs_random_population(const ffs_state *h, int64_t count, uint64_t seed, int64_t first_id, int8_t *x,
                                 int16_t *y, void *stream) {
  return ffs_random_population_strided(h, count, seed, first_id, 0, x, y, stream);
}

ffs_status ffs_random_population_strided(const ffs_state *h, int64_t count, uint64_t seed, int64_t first_id,
                                         int64_t row, int8_t *x, int16_t *y, void *stream) {
  if (!h || count < 0 || first_id < 0) return fail(FFS_ERR_INVALID_ARG, "bad arguments");
  if (row != 0 && row < h->v.K) return fail(FFS_ERR_INVALID_ARG, "row stride must be 0 or >= K");
  if (count > 0 && h->v.K > 0 && (!x || !y)) return fail(FFS_ERR_INVALID_ARG, "null output arrays");
  cudaSetDevice(h->v.inst->dev);
  return launch_random_population(h->v, count, seed, first_id, row > 0 ? row : h->v.K, x, y, (cudaStream_t)stream);
}

}  // extern "C"
