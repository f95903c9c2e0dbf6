// lane.cu -- the fast evaluate path: Algorithm 1 by a warp per chromosome
// (order_kernel), then Algorithm 2 by ONE LANE per chromosome
// (lane_decode_kernel), 32 chromosomes per warp.
//
// Why: Algorithm 2 is a dependent chain of K dispatches per chromosome whose
// per-dispatch work is scalar (t0 lookups, a window test, a commit).  With a
// warp per chromosome 31 lanes duplicate that scalar work (measured: 96 warp
// instructions per dispatch, 87% issue-active).  Here every lane decodes its
// own chromosome, so one warp instruction advances 32 chromosomes.
//
// Data layout
//   ordg  (global) [tile][ceil(K/4)][32 lanes][4]  u16 P/Q-table index of the
//         op at each rank, 4 ranks per lane per 8-byte load (coalesced 256 B)
//   per-thread state in shared memory, LANE-INTERLEAVED 32-bit words (word w
//   of lane l at (w*32 + l)*4: data-dependent accesses never bank-conflict):
//     ready[j]  u16 pairs  earliest start of job j's next op (rel. to RS)
//     mfree[m]  u16 pairs  machine free time (append-only sequencing, R6)
//     level[t]  u8 x4      Q_t per tick after RS (Eq. (8))
//     blocked   1 bit/tick level > Q_max - min Q: no op fits (exact)
// Feasibility (R2, R5): the earliest t >= t0 with p consecutive un-blocked
// ticks is found on a 32-tick window of the blocked bitmap (shift/and run
// test); ops with q > min Q also verify the window's bytes.  Commit adds q to
// p level bytes (byte-SIMD, no carries: Q_max <= 127) and refreshes the
// blocked bits of the touched words.
#include "device_util.cuh"

namespace edffs {
namespace {

using namespace dev;

__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// bit i set iff bits i..i+p-1 of b are set, 1 <= p <= 32 (no divergence on p)
__device__ __forceinline__ uint32_t runs_var(uint32_t b, int p) {
  uint32_t f2 = b & (b >> 1), f4 = f2 & (f2 >> 2), f8 = f4 & (f4 >> 4), f16 = f8 & (f8 >> 8);
  uint32_t f32 = f16 & (f16 >> 16);
  int lg = 31 - __clz(p);
  uint32_t fk = lg == 0 ? b : lg == 1 ? f2 : lg == 2 ? f4 : lg == 3 ? f8 : lg == 4 ? f16 : f32;
  return fk & (fk >> (p - (1 << lg)));
}

// ---------------------------------------------------------------------------
// Algorithm 1: one warp per chromosome, 32 chromosomes ("tile") per CTA pass;
// the tile's orders are written transposed (lane-interleaved) to ordg.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024, 1) order_kernel(EvalArgs a, uint32_t ord_stride, uint32_t ord_per_warp,
                                                        uint16_t *ordg) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t img_bytes = ((const ImageHdr *)a.image)->image_bytes;
  stage_image(smem, a.image, img_bytes, &bar);
  const ImageHdr &h = *(const ImageHdr *)smem;
  const int K = h.K, nt = (K + 31) >> 5, KQ = (K + 3) >> 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  unsigned char *ordbase = smem + img_bytes;
  unsigned char *scr = ordbase + 32 * ord_stride + (size_t)warp * ord_per_warp;
  OrderMem om;
  om.lbits = (uint32_t *)scr;
  om.cnt = (uint16_t *)(scr + ((4u * nt + 15u) & ~15u));
  const int64_t ntile = (a.count + 31) / 32;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    for (int cc = warp; cc < 32; cc += nwarps) {
      const int64_t c = tile * 32 + cc;
      if (c < a.count) {
        om.ord = ordbase + cc * ord_stride;
        const int64_t gc = a.first + c;
        build_order<1>(h, smem, om, a.x + gc * K, a.y + gc * K, lane);
      }
    }
    __syncthreads();
    // transposed write: element (q, cc, k) = order of chromosome cc at rank 4q + k
    uint16_t *dst = ordg + tile * (int64_t)KQ * 128;
    for (int idx = threadIdx.x; idx < KQ * 32; idx += blockDim.x) {
      const int qd = idx >> 5, cc = idx & 31;
      const uint16_t *src = (const uint16_t *)(ordbase + cc * ord_stride);
      uint16_t v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int r = 4 * qd + k;
        v[k] = r < K ? src[r] : (uint16_t)0;
      }
      uint2 pk;
      pk.x = (uint32_t)v[0] | ((uint32_t)v[1] << 16);
      pk.y = (uint32_t)v[2] | ((uint32_t)v[3] << 16);
      *(uint2 *)(dst + (size_t)idx * 4) = pk;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Algorithm 2 + Eqs. (1)-(3), (13): one lane per chromosome.
// ---------------------------------------------------------------------------
struct LaneCtx {
  uint32_t base;         // shared address of this lane's word 0
  int RW, MW, LW, BW;    // words: ready, mfree, level, blocked
  int hcap;
};
__device__ __forceinline__ uint32_t waddr(const LaneCtx &L, int w) { return L.base + ((uint32_t)w << 7); }

// earliest start >= t with p free ticks; general==true also checks q > min Q
// against the level bytes (threshold thr = Q_max - q)
__device__ __noinline__ int lane_search(const LaneCtx L, int t, int p, int thr, bool general) {
  const int LB = L.RW + L.MW, BB = LB + L.LW;
  const uint32_t KT = (uint32_t)(0x7F - thr) * 0x01010101u;
  for (;;) {
    const int bw = t >> 5;
    uint32_t b0 = bw < L.BW ? lds(waddr(L, BB + bw)) : 0u;
    uint32_t b1 = bw + 1 < L.BW ? lds(waddr(L, BB + bw + 1)) : 0u;
    uint32_t fr = ~__funnelshift_r(b0, b1, t & 31);
    uint32_t f = runs_var(fr, p);
    if (f == 0u) {
      t += 33 - p;
      continue;
    }
    const int cand = t + __ffs(f) - 1;
    if (!general) return cand;
    int bad = -1;
    for (int w = cand >> 2; w <= (cand + p - 1) >> 2 && bad < 0; ++w) {
      const int lo = max(cand - 4 * w, 0), hi = min(cand + p - 4 * w, 4);
      const uint32_t bm = (0xFFFFFFFFu << (lo << 3)) & (0xFFFFFFFFu >> ((4 - hi) << 3));
      const uint32_t v = w < L.LW ? lds(waddr(L, LB + w)) : 0u;
      const uint32_t fl = (v + KT) & 0x80808080u & bm;
      if (fl) bad = 4 * w + ((__ffs(fl) - 1) >> 3);
    }
    if (bad < 0) return cand;
    t = bad + 1;
  }
}

template <bool UQ, bool SCHED>
__global__ void __launch_bounds__(256, 1) lane_decode_kernel(EvalArgs a, int32_t lane_wpt) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t img_bytes = ((const ImageHdr *)a.image)->image_bytes;
  stage_image(smem, a.image, img_bytes, &bar);
  const ImageHdr &h = *(const ImageHdr *)smem;
  const int K = h.K, KQ = (K + 3) >> 2, GO = h.G * h.O;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  LaneCtx L;
  L.base = smem_u32(smem + img_bytes + (size_t)warp * lane_wpt * 128) + lane * 4;
  L.RW = (h.NJ + 1) >> 1;
  L.MW = (GO + 1) >> 1;
  L.hcap = a.h_cap;
  L.LW = a.h_cap >> 2;
  L.BW = a.h_cap >> 5;
  const int LB = L.RW + L.MW, BB = LB + L.LW;
  const uint32_t *pqt = (const uint32_t *)(smem + h.off_pqt);
  const uint32_t *r16 = (const uint32_t *)(smem + h.off_ready16);
  const uint32_t *m16 = (const uint32_t *)(smem + h.off_mfree16);
  const uint32_t *lv0 = (const uint32_t *)(smem + h.off_lvl0);
  const uint32_t KM = (uint32_t)(0x7F - h.thr_min) * 0x01010101u;
  const int qmin = h.q_max - h.thr_min;
  const int64_t ntile = (a.count + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; tile < ntile; tile += nw) {
    const int64_t c = tile * 32 + lane;
    const bool active = c < a.count;
    const int64_t gc = a.first + c;
    // --- initial state: ready/machine times, profile of the RUNNING ops
    for (int w = 0; w < L.RW; ++w) sts(waddr(L, w), r16[w]);
    for (int w = 0; w < L.MW; ++w) sts(waddr(L, L.RW + w), m16[w]);
    for (int w = 0; w < L.LW; ++w) sts(waddr(L, LB + w), w < h.lvl_words0 ? lv0[w] : 0u);
    for (int w = 0; w < L.BW; ++w) {
      uint32_t bits = 0;
      for (int k = 0; k < 8; ++k) {
        int lw = 8 * w + k;
        if (lw < h.lvl_words0) bits |= (((((lv0[lw] + KM) & 0x80808080u) * 0x00204081u) >> 28) << (4 * k));
      }
      sts(waddr(L, BB + w), bits);
    }
    int32_t *srow = nullptr;
    if (SCHED && active) {
      srow = a.start_out + gc * h.cells;
      for (int k = 0; k < h.cells; ++k) srow[k] = a.fstart[k];
    }
    bool ovf = false;
    const uint2 *op = (const uint2 *)(a.ordg + tile * (int64_t)KQ * 128) + lane;
    uint2 cur = active ? op[0] : make_uint2(0, 0);
    uint2 nxt = (active && KQ > 1) ? op[32] : make_uint2(0, 0);
    for (int qd = 0; qd < KQ; ++qd) {
      uint2 pre = (active && qd + 2 < KQ) ? op[(size_t)(qd + 2) * 32] : make_uint2(0, 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int r = 4 * qd + k;
        const uint32_t e = (k < 2 ? (k == 0 ? cur.x : cur.x >> 16) : (k == 2 ? cur.y : cur.y >> 16)) & 0xFFFFu;
        if (active && !ovf && r < K) {
          const uint32_t tv = pqt[e];
          const int p = (int)(tv & 0xFFu), q = (int)((tv >> 8) & 0xFFu), j = (int)(tv >> 16);
          const int mi = (int)e - j * GO;
          const uint32_t ra = waddr(L, j >> 1), ma = waddr(L, L.RW + (mi >> 1));
          const uint32_t rw = lds(ra), mw = lds(ma);
          const int rsh = (j & 1) << 4, msh = (mi & 1) << 4;
          // t0 = max(RS, release / predecessor completion, machine free)
          const int t0 = max((int)((rw >> rsh) & 0xFFFFu), (int)((mw >> msh) & 0xFFFFu));
          const int bw = t0 >> 5;
          const uint32_t b0 = bw < L.BW ? lds(waddr(L, BB + bw)) : 0u;
          const uint32_t b1 = bw + 1 < L.BW ? lds(waddr(L, BB + bw + 1)) : 0u;
          const uint32_t win = __funnelshift_r(b0, b1, t0 & 31);
          const uint32_t pm = 0xFFFFFFFFu >> (32 - p);
          int S = t0;
          if ((win & pm) != 0u || (!UQ && q != qmin)) S = lane_search(L, t0, p, h.q_max - q, !UQ && q != qmin);
          const int C = S + p;
          if (C > L.hcap) {
            ovf = true;
          } else {
            // commit: level += q on [S, C), refresh blocked bits
            const uint32_t QQ = (uint32_t)q * 0x01010101u;
            const int w0 = S >> 2, w1 = (C - 1) >> 2, bw0 = S >> 5;
            uint64_t acc = 0;
            for (int w = w0; w <= w1; ++w) {
              const int lo = max(S - 4 * w, 0), hi = min(C - 4 * w, 4);
              const uint32_t bm = (0xFFFFFFFFu << (lo << 3)) & (0xFFFFFFFFu >> ((4 - hi) << 3));
              const uint32_t la = waddr(L, LB + w);
              const uint32_t v = lds(la) + (QQ & bm);
              sts(la, v);
              const uint32_t nib = (((v + KM) & 0x80808080u) * 0x00204081u) >> 28;
              acc |= (uint64_t)nib << ((w - (bw0 << 3)) << 2);
            }
            const uint32_t ba = waddr(L, BB + bw0);
            sts(ba, lds(ba) | (uint32_t)acc);
            if (acc >> 32) sts(ba + 128, lds(ba + 128) | (uint32_t)(acc >> 32));
            sts(ra, (rw & ~(0xFFFFu << rsh)) | ((uint32_t)C << rsh));
            sts(ma, (mw & ~(0xFFFFu << msh)) | ((uint32_t)C << msh));
            if (SCHED) srow[e / h.O] = S + h.rs;
          }
        }
      }
      cur = nxt;
      nxt = pre;
    }
    if (!active) continue;
    if (ovf) {
      int pos = atomicAdd(&a.ovf[0], 1);
      a.ovf[1 + pos] = (int32_t)gc;
      continue;
    }
    // Eqs. (1)-(3) over every job (R9); frozen jobs are constants of the state
    const int32_t *pj = (const int32_t *)(smem + h.off_pjob);
    const int32_t *pd = (const int32_t *)(smem + h.off_pdue);
    int64_t T = 0;
    int cm = h.frozen_cmax;
    for (int k = 0; k < h.n_pjobs; ++k) {
      const int j = pj[k];
      const int Cr = (int)((lds(waddr(L, j >> 1)) >> ((j & 1) << 4)) & 0xFFFFu);
      const int tj = Cr - pd[k];
      T += tj > 0 ? tj : 0;
      cm = max(cm, Cr + h.rs);
    }
    T += h.frozen_T;
    const int64_t obj = h.wt * T + (int64_t)cm;
    if (a.obj) a.obj[gc] = obj;
    if (a.tard) a.tard[gc] = T;
    if (a.cmax) a.cmax[gc] = cm;
    if (a.fit) {  // Eq. (13)
      int64_t f = *a.emax - obj;
      a.fit[gc] = f > 0 ? f : 0;
    }
  }
}

template <typename KERN>
ffs_status smem_attr(KERN k, size_t bytes, size_t &done) {
  if (bytes > done) {
    FFS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done = bytes;
  }
  return FFS_OK;
}

}  // namespace

ffs_status launch_lane(const State &st, const EvalArgs &a0, OvfScratch &scr, cudaStream_t s, int *launches) {
  const int K = st.K, KQ = (K + 3) / 4;
  const int64_t chunk_max = (int64_t)1 << 17;
  const int64_t chunk = std::min<int64_t>((a0.count + 31) / 32 * 32, chunk_max);
  const int64_t elems = chunk / 32 * (int64_t)KQ * 128;
  if (elems > scr.ordg_elems) {
    if (scr.ordg) cudaFree(scr.ordg);
    scr.ordg = nullptr;
    FFS_CUDA(cudaMalloc(&scr.ordg, (size_t)elems * 2));
    scr.ordg_elems = elems;
  }
  static size_t a_ord = 0, a_l00 = 0, a_l01 = 0, a_l10 = 0, a_l11 = 0;
  ffs_status e = smem_attr(order_kernel, st.ord_smem, a_ord);
  if (e != FFS_OK) return e;
  const bool uq = ((const ImageHdr *)st.image_host.data())->uniform_q != 0;
  const bool sched = a0.start_out != nullptr;
  if (uq && sched) e = smem_attr(lane_decode_kernel<true, true>, st.lane_smem, a_l11);
  else if (uq) e = smem_attr(lane_decode_kernel<true, false>, st.lane_smem, a_l10);
  else if (sched) e = smem_attr(lane_decode_kernel<false, true>, st.lane_smem, a_l01);
  else e = smem_attr(lane_decode_kernel<false, false>, st.lane_smem, a_l00);
  if (e != FFS_OK) return e;
  const int ord_ctas_per_sm = (int)std::max<size_t>(1, (kSmemLimit + 1024) / (st.ord_smem + 1024));
  for (int64_t first = 0; first < a0.count; first += chunk) {
    EvalArgs a = a0;
    a.first = first;
    a.count = std::min<int64_t>(chunk, a0.count - first);
    a.ordg = scr.ordg;
    a.h_cap = st.lane_hcap;
    a.ovf = scr.list;
    const int64_t ntile = (a.count + 31) / 32;
    int64_t og = std::min<int64_t>(ntile, (int64_t)st.num_sms * ord_ctas_per_sm);
    order_kernel<<<(unsigned)og, st.ord_warps * 32, st.ord_smem, s>>>(a, st.ord_stride, (uint32_t)st.ord_per_warp,
                                                                      scr.ordg);
    FFS_CUDA(cudaGetLastError());
    const int64_t wpc = st.lane_warps_per_cta;
    int64_t lg = std::min<int64_t>((ntile + wpc - 1) / wpc, (int64_t)st.num_sms * st.lane_ctas_per_sm);
    const unsigned thr = (unsigned)(wpc * 32);
    if (uq && sched) lane_decode_kernel<true, true><<<(unsigned)lg, thr, st.lane_smem, s>>>(a, st.lane_wpt);
    else if (uq) lane_decode_kernel<true, false><<<(unsigned)lg, thr, st.lane_smem, s>>>(a, st.lane_wpt);
    else if (sched) lane_decode_kernel<false, true><<<(unsigned)lg, thr, st.lane_smem, s>>>(a, st.lane_wpt);
    else lane_decode_kernel<false, false><<<(unsigned)lg, thr, st.lane_smem, s>>>(a, st.lane_wpt);
    FFS_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
  }
  return FFS_OK;
}

}  // namespace edffs
