// lane.cu -- the fast evaluate path.  Algorithm 1 (order_warp_kernel): ONE
// WARP per chromosome (the sort is parallel work); Algorithm 2 (the decode
// kernels): ONE LANE per chromosome, 32 chromosomes per warp (its per-op work
// is a scalar dependent chain; with a warp per chromosome 31 lanes duplicated
// it: 96 warp instructions per dispatched op at 87% issue).
//
// Layouts
//   per-thread arrays live in shared memory LANE-INTERLEAVED: 32-bit word w of
//   lane l sits at (w*32 + l)*4, so data-dependent indices never bank-conflict.
//   ordg (global) [tile][ceil(K/4)][32 lanes][4] u16: P/Q-table index of the op
//   at each rank (4 ranks per lane per 8-byte load, 256 B per warp, coalesced).
// Algorithm 1 (greedy reading R1) = stable sort by (prefix-min of y
// over the job's pending stages desc, stage asc): a counting sort by the
// prefix minimum -- see order_warp_kernel.
// Algorithm 2 (R2, R5):
//   lane_decode2_kernel  every Q == 1, Q_max <= 15 (the paper's Table 5
//     setting): 10-bit job / machine times, headroom Q_max - Q_t as bit planes
//     in 8-tick groups, blocked bits, software-pipelined dispatches (below)
//   lane_decode_kernel (modes 0/1) otherwise: per lane
//     ready[j]  u16 pairs  earliest start of job j's next op (rel. to RS)
//     mfree[m]  u16 pairs  machine free time (append-only sequencing, R6)
//     level[t]  u8 x4      Q_t per tick + bias, bias = 0x7F - (Q_max - min Q):
//                          bit 7 of a byte  <=>  Q_t > Q_max - min Q
//     blocked   1 bit/tick copy of those bits: no op fits at that tick
//   The earliest t >= t0 with p un-blocked ticks is found on a 32-tick window
//   of `blocked` (run test by shifts/ands); ops with q > min Q verify the
//   bytes.  Commit adds q to p bytes (byte SIMD, no carries since Q_max <=
//   127) and ORs their bit-7 flags into `blocked`.
#include <type_traits>

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
[[maybe_unused]] __device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}
[[maybe_unused]] __device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
// predicated shared u16 store / load (no branch, no reconvergence barrier)
__device__ __forceinline__ void sts16_if(bool p, uint32_t a, uint32_t v) {   // a: shared-window address
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.u16 [%0], %1;\n}\n" ::"r"(a),
               "h"((unsigned short)v), "r"((uint32_t)p)
               : "memory");
}
// keep a staged value in a register (no rematerialisation on the critical path)
__device__ __forceinline__ void pin(uint32_t &v) { asm volatile("" : "+r"(v)); }
__device__ __forceinline__ void pin(int &v) { asm volatile("" : "+r"(v)); }
// zero-extended halves by one byte permute each (opaque to the compiler, so a
// table address becomes one shift-add instead of mask + shift + add)
__device__ __forceinline__ uint32_t lo16(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x4410;" : "=r"(r) : "r"(w));
  return r;
}
__device__ __forceinline__ uint32_t hi16(uint32_t w) {
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, 0x4432;" : "=r"(r) : "r"(w));
  return r;
}
// lane-interleaved u16 element v: word v/2, half v%2
[[maybe_unused]] __device__ __forceinline__ uint32_t h16addr(uint32_t base, uint32_t v) {
  return base + ((v >> 1) << 7) + ((v & 1u) << 1);
}

// bit i set iff bits i..i+p-1 of b are set, 1 <= p <= 32 (no divergence on p)
__device__ __forceinline__ uint32_t runs_var(uint32_t b, int p) {
  uint32_t f2 = b & (b >> 1), f4 = f2 & (f2 >> 2), f8 = f4 & (f4 >> 4), f16 = f8 & (f8 >> 8);
  uint32_t f32 = f16 & (f16 >> 16);
  int lg = 31 - __clz(p);
  uint32_t fk = lg == 0 ? b : lg == 1 ? f2 : lg == 2 ? f4 : lg == 3 ? f8 : lg == 4 ? f16 : f32;
  return fk & (fk >> (p - (1 << lg)));
}

// the four bit-7 byte flags of v packed into a nibble
__device__ __forceinline__ uint32_t flag_nibble(uint32_t v) {
  return ((v & 0x80808080u) * 0x00204081u) >> 28;
}

// ---------------------------------------------------------------------------
// Algorithm 1: one WARP per chromosome (4 genes per lane per 128-gene tile),
// 32 chromosomes per CTA; the CTA writes the tile's orders lane-interleaved.
//   pass A  (pm(g), g_L(g)) = min of the keys y << 16 | g over the job's
//           pending stages <= s (segmented warp scan, segments start at each
//           job's first pending gene): pm = the prefix minimum of y, g_L =
//           the gene holding it (the run's leader, a new prefix minimum);
//           the run's last gene stores hist[u] = g - g_L + 1, u = K - pm
//   pass C  start[u] = #genes with u' < u (exclusive prefix sum)
//   pass D  rank(g) = start[u(g)] + (g - g_L(g)); ord[rank] = the op's table
//           index (mode 2: g * O + machine; modes 0/1: cell base + machine)
// ---------------------------------------------------------------------------
struct OrdArgs {
  const int8_t *x;
  const int16_t *y;
  int64_t first, count;
  int64_t row;             // genes between chromosomes (>= K)
  int32_t vec;             // row % 16 == 0 and 16-B aligned bases: TMA bulk row staging
  int32_t K;
  const uint32_t *head;    // [ceil(K/32)] bit g: first pending gene of its job
  const uint32_t *gbase;   // [K] (j*G + s)*O (cell-indexed tables, modes 0/1; unused when GIDX)
  uint16_t *ordg;
  uint32_t hist_bytes;     // per warp
  uint32_t ord_stride;     // bytes between staged ord arrays (8 * odd)
  uint32_t pm_bytes;       // per warp, K u16 rounded to 16 B
  int32_t *zero0, *zero1;  // first chunk: the overflow lists' counts to reset (else null)
  int32_t ubits;           // pass A/D key: u = K - pm in the low ubits, g - g_L above (2^ubits >= K)
  int32_t O;               // machines per stage (GIDX: table index g * O + machine)
};

// prefix minima of the lane's four genes given the running min before the tile.
// A job's pending genes (<= G of them, consecutive) span at most
// floor((G+2)/4) + 1 lanes, so the segmented scan needs only SCAN doubling
// steps with 2^SCAN > that span - 1 (SCAN = 2 for G <= 13).  The segment
// structure is the same for every chromosome, so it comes from two CTA-wide
// tables built once per launch: M = the quad's per-gene reset masks (all ones
// iff the gene starts a segment: a job's first pending gene, or padding), and
// dsc = the lane's scan-step enables (bit i: combine with lane - 2^i) and, in
// bit 31, "a segment starts in an earlier lane of this tile".  A reset is an
// OR with all ones before an unsigned min (the keys y << 16 | g and the
// running minima are below 2^31 (y <= K < 2^15); padding keys are all ones),
// so no compare / select per gene.
template <int SCAN>
__device__ __forceinline__ void pm_quad(const int y[4], const uint4 M, uint32_t dsc, uint32_t carry, uint32_t Z,
                                        int pm[4]) {
  // v = min over the lane's genes from its last segment start (or all four)
  uint32_t v = (uint32_t)y[0];
  v = umin(v | M.y, (uint32_t)y[1]);
  v = umin(v | M.z, (uint32_t)y[2]);
  v = umin(v | M.w, (uint32_t)y[3]);
#pragma unroll
  for (int i = 0; i < SCAN; ++i) {
    const uint32_t vn = __shfl_up_sync(FULL, v, 1 << i);
    if ((dsc >> i) & 1u) v = umin(v, vn);
  }
  // exclusive value for the lane: min over lanes [s_prev, lane-1], plus the
  // carry when no segment starts before the lane in this tile (Z: lane 0)
  const uint32_t vex = __shfl_up_sync(FULL, v, 1);
  uint32_t run = umin(vex | Z, carry | (uint32_t)((int32_t)dsc >> 31));
  run = umin(run | M.x, (uint32_t)y[0]);
  pm[0] = (int)run;
  run = umin(run | M.y, (uint32_t)y[1]);
  pm[1] = (int)run;
  run = umin(run | M.z, (uint32_t)y[2]);
  pm[2] = (int)run;
  run = umin(run | M.w, (uint32_t)y[3]);
  pm[3] = (int)run;
}

// BULK: the row was staged in shared memory (the genes g0..g0+3 are one 8-byte
// word).  FULL: every gene of the tile is < K (no bounds tests).  y is in
// [1, K] (a permutation), so the halves need no sign extension; genes past
// the end read as INT_MAX (their own segments, see the reset masks).
template <bool BULK, bool FULL = false>
__device__ __forceinline__ void load_quad(const int16_t *yr, int K, int g0, int y[4]) {
  if (BULK) {
    const uint2 w = *(const uint2 *)(yr + g0);
    const int v[4] = {(int)(w.x & 0xFFFFu), (int)(w.x >> 16), (int)(w.y & 0xFFFFu), (int)(w.y >> 16)};
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = (FULL || g0 + k < K) ? v[k] : INT_MAX;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = (FULL || g0 + k < K) ? (int)__ldg(yr + g0 + k) : INT_MAX;
  }
}

__device__ __forceinline__ void load_xquad(const int8_t *xr, int K, int g0, uint32_t &xw) {
  xw = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (g0 + k < K) xw |= (uint32_t)(uint8_t)__ldg(xr + g0 + k) << (8 * k);
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// BULK (row % 16 == 0, 16-B aligned bases -- the GA's padded population):
// each warp stages its chromosome's whole y row into pmv
// with one TMA bulk copy (one elected lane, per-warp mbarrier) instead of
// per-lane global loads; pass A then reads y from shared memory and writes
// the prefix minima over it in place.
// XS: the warp also stages the chromosome's machines (x row) in shared memory
// during pass A (TMA under BULK); without it (long rows whose staging would
// not fit in 227 KB) pass D reads them from global memory one tile ahead.
template <bool BULK, int SCAN, bool XS, bool GIDX>
__global__ void __launch_bounds__(1024, 1) order_warp_kernel(OrdArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int K = a.K, KQ = (K + 3) >> 2, NT = (K + 127) >> 7;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *hist = (uint32_t *)(smem + (size_t)warp * a.hist_bytes);          // u16 pairs
  uint16_t *h16 = (uint16_t *)hist;
  uint16_t *pmv = (uint16_t *)(smem + (size_t)32 * a.hist_bytes + (size_t)32 * a.ord_stride +
                               (size_t)warp * a.pm_bytes);                      // [K] y, then (g - g_L) << ub | (2^ub - pm)
  unsigned char *ordb = smem + (size_t)32 * a.hist_bytes;
  uint16_t *ord = (uint16_t *)(ordb + (size_t)warp * a.ord_stride);
  const uint32_t h16s = smem_u32(h16), ords = smem_u32(ord);   // shared-window addresses
  // CTA-shared tables (the same for every chromosome): per-gene table base,
  // segment reset masks and per-lane scan descriptors (pm_quad); and (XS)
  // per-warp staging of the chromosome's machines
  unsigned char *tail = smem + (size_t)32 * (a.hist_bytes + a.ord_stride + a.pm_bytes);
  // gene table (pass D's strided reads hit 32 distinct banks)
  uint32_t *gtab = (uint32_t *)tail;
  uint32_t *mtab = gtab + 128 * NT;
  uint32_t *dtab = mtab + 128 * NT;
  uint32_t *btab = dtab + 32 * NT;   // per (tile, lane): byte k = 0xFF iff gene k of the quad starts a segment
  uint8_t *xs = (uint8_t *)(btab + 32 * NT) + (size_t)warp * 128 * NT;   // XS only
  if (!GIDX)   // GIDX: the rank's op is g * O + machine (mode 2's gene-indexed table)
    for (int i = threadIdx.x; i < K; i += blockDim.x) gtab[i] = __ldg(a.gbase + i);
  for (int i = threadIdx.x; i < 128 * NT; i += blockDim.x)
    mtab[i] = (i >= K || ((__ldg(a.head + (i >> 5)) >> (i & 31)) & 1u)) ? 0xFFFFFFFFu : 0u;
  __syncthreads();
  for (int t = warp; t < NT; t += 32) {
    const uint4 m = *(const uint4 *)(mtab + (t << 7) + 4 * lane);
    const uint32_t hb = __ballot_sync(FULL, (m.x | m.y | m.z | m.w) != 0u);   // lanes holding a segment start
    const uint32_t below = hb & (0xFFFFFFFFu >> (31 - lane));
    const int s0 = below ? 31 - __clz(below) : -1;
    uint32_t dsc = (hb & ((1u << lane) - 1u)) ? 0x80000000u : 0u;
    // bit 30: the gene after the lane's quad starts a job, or is past K
    const int gn = (t << 7) + 4 * lane + 4;
    if (gn >= 128 * NT || mtab[gn] != 0u) dsc |= 0x40000000u;
    btab[(t << 5) + lane] = (m.x & 0xFFu) | (m.y & 0xFF00u) | (m.z & 0xFF0000u) | (m.w & 0xFF000000u);
#pragma unroll
    for (int i = 0; i < 5; ++i)
      if (lane - (1 << i) >= s0 && lane >= (1 << i)) dsc |= 1u << i;
    dtab[(t << 5) + lane] = dsc;
  }
  const uint32_t Z = lane == 0 ? 0xFFFFFFFFu : 0u;
  for (int r = K + lane; r < 4 * KQ; r += 32) ord[r] = 0;   // padding ranks (never ranked)
  pdl_trigger();
  pdl_wait();   // the tables above are state constants; x, y and ordg are not
  // the call's overflow counts start at 0 (here rather than by a memset node,
  // so the launch chain stays kernel-to-kernel; earlier readers are done)
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.zero0) {
    *a.zero0 = 0;
    *a.zero1 = 0;
  }
  __shared__ __align__(8) uint64_t obar[32];
  const uint32_t bar = smem_u32(&obar[warp]);
  uint32_t phase = 0;
  if (BULK && lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntile = (a.count + 31) / 32;
  // BULK: one elected lane stages the warp's chromosome of tile `tl` (y row
  // into pmv, x row into xs) by TMA bulk copies on the warp's mbarrier --
  // ceil16(K) genes of the row (<= row: row % 16 == 0 and row >= K), never the
  // whole row (the smem slots are sized from K, 128 * ceil(K/128)).  The copy
  // of the warp's NEXT chromosome is issued as soon as pass D has consumed
  // pmv / xs, so it lands during the CTA's write-out of the current tile.
  auto stage_row = [&](const int64_t tl) {
    const int64_t cc = tl * 32 + warp;
    if (!BULK || lane != 0 || tl >= ntile || cc >= a.count) return;
    const uint32_t kc = ((uint32_t)K + 15u) & ~15u;
    const uint32_t yb = kc * 2u, xb = XS ? kc : 0u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // after the previous row's generic accesses
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(yb + xb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(pmv)),
                 "l"(a.y + (a.first + cc) * a.row), "r"(yb), "r"(bar)
                 : "memory");
    if (XS)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(xs)),
                   "l"(a.x + (a.first + cc) * a.row), "r"(xb), "r"(bar)
                   : "memory");
  };
  stage_row(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int64_t c = tile * 32 + warp;
    if (c < a.count) {
      const int16_t *yr = a.y + (a.first + c) * a.row;
      const int8_t *xr = a.x + (a.first + c) * a.row;
      // hist/start are indexed by u = K - pm (descending prefix minimum)
      for (int i = lane; i < ((K + 511) >> 9) << 6; i += 32) ((uint4 *)hist)[i] = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
      if (BULK) {
        while (!mbar_try(bar, phase)) {
        }
        phase ^= 1u;
      }
      // ---- pass A: prefix minima over packed keys (y << 16 | g): the minimum
      // carries its own gene, so every gene knows its run's leader g_L
      // (y is a permutation: the minimum is unique).  A run = a leader (new
      // prefix minimum) and the non-leaders after it in its job, all at
      // u = K - pm; its LAST gene (the next gene leads a run or starts a job)
      // stores the run length g - g_L + 1 into hist[u] -- one plain u16
      // store per run, no atomics.  pmv keeps u | (g - g_L) << ub per gene.
      uint32_t carry = 0xFFFFFFFFu;
      uint32_t umul = 1u << a.ubits;
      pin(umul);   // multiplies (fma pipe), not shifts
      const uint32_t hK2 = h16s + 2u * (uint32_t)K;
      // software pipeline (global loads): tile t+1's genes are loaded while
      // tile t is scanned
      int yq[4];
      uint32_t xq = 0, ynq = 0;
      if (!BULK) {
        load_quad<false>(yr, K, 4 * lane, yq);
        ynq = 4 * lane + 4 < K ? (uint32_t)__ldg(yr + 4 * lane + 4) : 0u;
        if (XS) load_xquad(xr, K, 4 * lane, xq);
      }
      auto tileA = [&](const int t, auto fullc) {
        constexpr bool FT = decltype(fullc)::value;   // every gene of the tile < K
        const int g0 = (t << 7) + 4 * lane;
        // keys y << 16 | g (padding: all ones); yn = y of the gene after the
        // quad (only read when it continues the job)
        uint32_t yp[4], yn;
        if (BULK) {
          const uint2 w = *(const uint2 *)(pmv + g0);
          yp[0] = __byte_perm(w.x, (uint32_t)g0, 0x1054);
          yp[1] = __byte_perm(w.x, (uint32_t)(g0 + 1), 0x3254);
          yp[2] = __byte_perm(w.y, (uint32_t)(g0 + 2), 0x1054);
          yp[3] = __byte_perm(w.y, (uint32_t)(g0 + 3), 0x3254);
          // lane 31's successor is the next tile's first gene, not yet overwritten
          const uint32_t nt = t + 1 < NT ? (uint32_t)pmv[(t + 1) << 7] : 0u;
          const uint32_t dn = __shfl_down_sync(FULL, w.x & 0xFFFFu, 1);
          yn = lane == 31 ? nt : dn;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) yp[k] = ((uint32_t)yq[k] << 16) | (uint32_t)(g0 + k);
          yn = ynq;
          if (XS) *(uint32_t *)(xs + g0) = xq;
          if (t + 1 < NT) {
            load_quad<false>(yr, K, g0 + 128, yq);
            ynq = g0 + 132 < K ? (uint32_t)__ldg(yr + g0 + 132) : 0u;
            if (XS) load_xquad(xr, K, g0 + 128, xq);
          }
        }
        if (!FT) {
#pragma unroll
          for (int k = 0; k < 4; ++k) yp[k] = g0 + k < K ? yp[k] : 0xFFFFFFFFu;
        }
        int rp[4];
        const uint32_t dsc = dtab[(t << 5) + lane];
        const uint32_t bf = btab[(t << 5) + lane];   // reset masks by sign-replicating byte permutes
        const uint4 M = make_uint4(__byte_perm(bf, 0u, 0x8888u), __byte_perm(bf, 0u, 0x9999u),
                                   __byte_perm(bf, 0u, 0xAAAAu), __byte_perm(bf, 0u, 0xBBBBu));
        pm_quad<SCAN>((const int *)yp, M, dsc, carry, Z, rp);
        // the gene after gene k leads a run (a new minimum, or a job's first
        // pending gene: its reset makes it its own minimum); after the quad:
        // dsc bit 30 (job start or past K) or y below the running minimum
        bool last[4];
#pragma unroll
        for (int k = 0; k < 3; ++k) last[k] = (uint32_t)rp[k + 1] == yp[k + 1];
        last[3] = ((dsc >> 30) & 1u) || (yn << 16) < (uint32_t)rp[3];
        uint32_t pk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t pm = (uint32_t)rp[k] >> 16;
          const uint32_t o1 = (uint32_t)(g0 + k + 1) - ((uint32_t)rp[k] & 0xFFFFu);   // g - g_L + 1
          pk[k] = o1 * umul - pm;   // (g - g_L) << ub | (2^ub - pm), 2^ub - pm = u + 2^ub - K
          sts16_if((FT || g0 + k < K) && last[k], hK2 - 2u * pm, o1);   // hist[u], u = K - pm
        }
        *(uint2 *)(pmv + g0) = make_uint2(__byte_perm(pk[0], pk[1], 0x5410), __byte_perm(pk[2], pk[3], 0x5410));
        carry = __shfl_sync(FULL, (uint32_t)rp[3], 31);
      };
      for (int t = 0; t + 1 < NT; ++t) tileA(t, std::true_type{});
      tileA(NT - 1, std::false_type{});
      __syncwarp();
      // ---- pass C: start[u] = #genes with u' < u (exclusive prefix over u),
      // 16 counts (u16 pairs) per lane per step of 512 (entries >= K are
      // written but never read); W * 0x10001 puts a pair's sum in the high half
      uint32_t acc = 0;
      for (int ub = 0; ub < K; ub += 512) {   // warp-uniform trip count (shuffles inside)
        const int u0 = ub + 16 * lane;
        uint4 wa = *(const uint4 *)(h16 + u0), wb = *(const uint4 *)(h16 + u0 + 8);   // 32-byte aligned
        const uint32_t W[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
        uint32_t ex[8], run = 0;                      // exclusive in-lane prefix of the pair sums
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          ex[i] = run;
          run += (W[i] * 0x10001u) >> 16;
        }
        const uint32_t sum = run;
        uint32_t incl = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t n = __shfl_up_sync(FULL, incl, d);
          if (lane >= d) incl += n;
        }
        const uint32_t e0 = acc + incl - sum;         // exclusive start of the lane's 16 counts
        uint32_t O[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {   // start of count 2i = e, of count 2i+1 = e + count 2i
          const uint32_t e = e0 + ex[i];
          O[i] = e | ((e + (W[i] & 0xFFFFu)) << 16);
        }
        *(uint4 *)(h16 + u0) = make_uint4(O[0], O[1], O[2], O[3]);
        *(uint4 *)(h16 + u0 + 8) = make_uint4(O[4], O[5], O[6], O[7]);
        acc += __shfl_sync(FULL, incl, 31);
      }
      __syncwarp();
      // ---- pass D: rank(g) = start[u(g)] + (g - g_L): per gene, no cross-lane work
      // the lane's four machines of tile t (!XS): one aligned word of a padded
      // row (BULK), else bytes; loaded one tile ahead to hide the latency
      // Genes are STRIDED here (lane l takes genes 128t + 32k + l), so the 32
      // lanes of one access hold consecutive genes: a run's genes read the
      // same start[u] (broadcast) and write consecutive ranks, which keeps the
      // gathers and the scatter nearly free of bank conflicts.
      // The lane's four machines of tile t (!XS): bytes of the x row, loaded
      // one tile ahead to hide the latency.
      uint32_t xnext[4] = {0u, 0u, 0u, 0u};
      auto loadx = [&](const int t) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int g = (t << 7) + 32 * k + lane;
          xnext[k] = g < K ? (uint32_t)(uint8_t)__ldg(xr + g) : 0u;
        }
      };
      if (!XS) loadx(0);
      const uint32_t umask = umul - 1u, hbase = hK2 - 2u * umul;   // start[u] at hbase + 2 (u + 2^ub - K)
      auto tileD = [&](const int t, auto fullc) {
        constexpr bool FT = decltype(fullc)::value;   // every gene of the tile < K
        const int gb = (t << 7) + lane;
        uint32_t xk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) xk[k] = XS ? (uint32_t)xs[gb + 32 * k] : xnext[k];
        if (!XS && t + 1 < NT) loadx(t + 1);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int g = gb + 32 * k;
          const bool ok = FT || g < K;
          const uint32_t pk = pmv[g];
          const uint32_t st = ok ? lds16(hbase + 2u * (pk & umask)) : 0u;
          const uint32_t rank = st + (pk >> a.ubits);
          const uint32_t e = GIDX ? (uint32_t)g * (uint32_t)a.O + xk[k] : gtab[g] + xk[k];
          if (FT)
            ord[rank] = (uint16_t)e;
          else
            sts16_if(ok, ords + 2u * rank, e);
        }
      };
      for (int t = 0; t + 1 < NT; ++t) tileD(t, std::true_type{});
      tileD(NT - 1, std::false_type{});
      if (BULK) {   // pmv / xs are consumed: stage the warp's next chromosome
        __syncwarp();
        stage_row(tile + gridDim.x);
      }
    }
    // lane-interleaved write-out: element (q, cc) = ranks 4q..4q+3 of chromosome
    // cc, at dst[32 q + cc].  Four independent groups of 8 warps (named
    // barriers 1..4, 256 threads): group G moves chromosomes 8G..8G+7, i.e.
    // bytes 64G..64G+63 (two whole sectors) of every 256-byte quad row; its
    // thread t moves chromosome 8G + t%8's quads q = t/8, t/8 + 32, ...
    // (conflict-free: the staged arrays are an odd number of 8-byte words
    // apart).  Ranks >= K hold the zeros written at kernel start.
    {
      const int grp = warp >> 3, t = ((warp & 7) << 5) | lane;
      const int cc = (grp << 3) | (t & 7);
      asm volatile("bar.sync %0, 256;" ::"r"(grp + 1) : "memory");
      if (cc < a.count - tile * 32) {
        const unsigned char *src = ordb + (size_t)cc * a.ord_stride + (size_t)(t >> 3) * 8;
        uint2 *dst = (uint2 *)(a.ordg + tile * (int64_t)KQ * 128) + (t >> 3) * 32 + cc;
#pragma unroll 2
        for (int qd = t >> 3; qd < KQ; qd += 32) {
          *dst = *(const uint2 *)src;
          src += 256;
          dst += 1024;
        }
      }
      asm volatile("bar.sync %0, 256;" ::"r"(grp + 1) : "memory");
    }
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

// Slow path (window miss, or q > min Q): earliest start >= t with p ticks
// that are un-blocked and, for general q, whose biased bytes b satisfy
// b + (q - qmin) < 0x80  (i.e. Q_t + q <= Q_max).
__device__ __noinline__ int lane_search(const LaneCtx L, int t, int p, int dq, uint32_t bias4) {
  const int LB = L.RW + L.MW, BB = LB + L.LW;
  const uint32_t KT = (uint32_t)dq * 0x01010101u;
  for (;;) {
    const int bw = t >> 5;
    uint32_t b0 = bw < L.BW ? lds(waddr(L, BB + bw)) : 0u;
    uint32_t b1 = bw + 1 < L.BW ? lds(waddr(L, BB + bw + 1)) : 0u;
    uint32_t f = runs_var(~__funnelshift_r(b0, b1, t & 31), p);
    if (f == 0u) {
      t += 33 - p;
      continue;
    }
    const int cand = t + __ffs(f) - 1;
    if (dq == 0) return cand;
    int bad = -1;
    for (int w = cand >> 2; w <= (cand + p - 1) >> 2 && bad < 0; ++w) {
      const int lo = max(cand - 4 * w, 0), hi = min(cand + p - 4 * w, 4);
      const uint32_t bm = (0xFFFFFFFFu << (lo << 3)) & (0xFFFFFFFFu >> ((4 - hi) << 3));
      const uint32_t v = w < L.LW ? lds(waddr(L, LB + w)) : bias4;
      const uint32_t fl = (v + KT) & 0x80808080u & bm;
      if (fl) bad = 4 * w + ((__ffs(fl) - 1) >> 3);
    }
    if (bad < 0) return cand;
    t = bad + 1;
  }
}

// Per-op constants that do not depend on the decode state (software-pipelined
// one op ahead): table fields, ready/machine word addresses, and the masks of
// the branch-free run test for this p (1 <= p <= 8).
struct OpA {
  uint32_t e, ra, ma, QQ, M1, M2, M4;
  int p, q, rsh, msh, sft;
};
__device__ __forceinline__ OpA stage_a(const uint32_t *pqt, const LaneCtx &L, int GO, uint32_t e) {
  OpA A;
  const uint32_t tv = pqt[e];
  A.e = e;
  A.p = (int)(tv & 0xFFu);
  A.q = (int)((tv >> 8) & 0xFFu);
  const int j = (int)(tv >> 16);
  const int mi = (int)e - j * GO;
  A.ra = waddr(L, j >> 1);
  A.ma = waddr(L, L.RW + (mi >> 1));
  A.rsh = (j & 1) << 4;
  A.msh = (mi & 1) << 4;
  A.QQ = (uint32_t)A.q * 0x01010101u;
  const int pp = max(A.p, 1);
  A.M1 = (uint32_t)((pp - 2) >> 31);   // skip the >=2 doubling step when p < 2
  A.M2 = (uint32_t)((pp - 4) >> 31);
  A.M4 = (uint32_t)((pp - 8) >> 31);
  A.sft = pp - (1 << (31 - __clz(pp)));
  return A;
}

// first run of p free ticks: doubling masks (bit i set iff bits i..i+p-1 set)
__device__ __forceinline__ uint32_t run_test(uint32_t f, const OpA &A) {
  f &= (f >> 1) | A.M1;
  f &= (f >> 2) | A.M2;
  f &= (f >> 4) | A.M4;
  return f & (f >> A.sft);
}

// MODE 0: byte levels, general Q; MODE 1: byte levels, uniform Q (every
// Q == 1 with Q_max <= 15 is mode 2: lane_decode2_kernel below).
template <int MODE, bool SCHED>
__global__ void __launch_bounds__(512, 1) lane_decode_kernel(EvalArgs a, int32_t lane_wpt) {
  static_assert(MODE == 0 || MODE == 1, "mode 2 has its own kernel");
  constexpr bool UQ = MODE != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint4 cmask[32];    // byte masks of [S, S+p) over words S/4 .. S/4+2, by (S%4, p-1)
  if (threadIdx.x < 32) {
    const int lo = threadIdx.x >> 3, ee = lo + (threadIdx.x & 7) + 1;
    uint4 m;
    m.x = (0xFFFFFFFFu << (lo << 3)) & (0xFFFFFFFFu >> ((4 - min(ee, 4)) << 3));
    m.y = ee > 4 ? 0xFFFFFFFFu >> ((4 - min(ee - 4, 4)) << 3) : 0u;
    m.z = ee > 8 ? 0xFFFFFFFFu >> ((12 - ee) << 3) : 0u;
    m.w = 0u;
    cmask[threadIdx.x] = m;
  }
  const uint32_t img_bytes = ((const ImageHdr *)a.image)->lane_image_bytes;
  stage_image(smem, a.image, img_bytes, &bar);
  pdl_trigger();
  pdl_wait();
  uint32_t cm_base = smem_u32(cmask);
  pin(cm_base);
  const ImageHdr &h = *(const ImageHdr *)smem;
  const int K = h.K, KQ = (K + 3) >> 2, GO = h.G * h.O;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  LaneCtx L;
  L.base = smem_u32(smem + img_bytes + (size_t)warp * lane_wpt * 128) + lane * 4;
  L.RW = (h.NJ + 1) >> 1;
  L.MW = (GO + 1) >> 1;
  constexpr uint32_t TM = 0xFFFFu;   // time field mask (u16 pairs)
  L.hcap = a.h_cap;
  L.LW = a.h_cap >> 2;
  L.BW = a.h_cap >> 5;
  const int LB = L.RW + L.MW, BB = LB + L.LW;
  const uint32_t *pqt = (const uint32_t *)(smem + h.off_pqt);
  const uint32_t *r16 = (const uint32_t *)(smem + h.off_ready16);
  const uint32_t *m16 = (const uint32_t *)(smem + h.off_mfree16);
  const uint32_t *lv0 = (const uint32_t *)(smem + h.off_lvl0);
  const int qmin = h.q_max - h.thr_min, lvw0 = h.lvl_words0;
  const uint32_t bias4 = (uint32_t)(0x7F - h.thr_min) * 0x01010101u;
  int hcap = L.hcap, BW = L.BW;
  pin(hcap);
  pin(BW);
  const int64_t ntile = (a.count + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; tile < ntile; tile += nw) {
    const int64_t c = tile * 32 + lane;
    const bool active = c < a.count;
    const int64_t gc = a.first + c;
    // --- initial state: ready/machine times, profile of the RUNNING ops
    for (int w = 0; w < L.RW; ++w) sts(waddr(L, w), r16[w]);
    for (int w = 0; w < L.MW; ++w) sts(waddr(L, L.RW + w), m16[w]);
    for (int w = 0; w < L.LW; ++w) sts(waddr(L, LB + w), (w < lvw0 ? lv0[w] : 0u) + bias4);
    for (int w = 0; w < BW; ++w) {
      uint32_t bits = 0;
      for (int k = 0; k < 8 && 8 * w + k < lvw0; ++k) bits |= flag_nibble(lv0[8 * w + k] + bias4) << (4 * k);
      sts(waddr(L, BB + w), bits);
    }
    sts(waddr(L, BB + BW), 0u);
    sts(waddr(L, BB + BW + 1), 0u);
    int32_t *srow = nullptr;
    if (SCHED && active) {
      srow = a.start_out + gc * h.cells;
      for (int k = 0; k < h.cells; ++k) srow[k] = a.fstart[k];
    }
    bool live = active;            // false when inactive or overflowed
    bool ovf = false;
    int kq_pref = active ? KQ : 0;   // prefetch bound (0 for inactive lanes): one 32-bit compare per quad
    pin(kq_pref);                    // (not re-derived from the 64-bit c < count)
    const uint2 *op = (const uint2 *)(a.ordg + tile * (int64_t)KQ * 128) + lane;
    // software pipeline: the next op's table lookup and every p-dependent
    // constant (stage A) is computed while the current op runs (B..E)
    uint2 cur = active ? op[0] : make_uint2(0, 0);
    uint2 nxt = (active && KQ > 1) ? op[32] : make_uint2(0, 0);
    OpA nA = stage_a(pqt, L, GO, cur.x & 0xFFFFu);
    for (int qd = 0; qd < KQ; ++qd) {
      const uint2 pre = qd + 2 < kq_pref ? op[(size_t)(qd + 2) * 32] : make_uint2(0, 0);
      const int nk = min(4, K - 4 * qd);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const OpA A = nA;
        {   // stage A of rank 4*qd + k + 1
          const uint32_t en = k == 0 ? cur.x >> 16 : k == 1 ? cur.y : k == 2 ? cur.y >> 16 : nxt.x;
          nA = stage_a(pqt, L, GO, 4 * qd + k + 1 < K ? en & 0xFFFFu : 0u);
        }
        if (live && k < nk) {
          // B: t0 = max(RS, release / predecessor completion, machine free)
          const uint32_t rw = lds(A.ra), mw = lds(A.ma);
          const int t0 = max((int)((rw >> A.rsh) & TM), (int)((mw >> A.msh) & TM));
          // C: first run of p un-blocked ticks in the 32-tick window at t0
          //    (blocked words BW, BW+1 are zero sentinels: no bounds test)
          const uint32_t bwa = waddr(L, BB + min(t0 >> 5, BW));
          uint32_t f = run_test(~__funnelshift_r(lds(bwa), lds(bwa + 128), t0 & 31), A);
          int S;
          if (UQ) {
            // window miss: slide by 33 - p ticks (a run starting in the last
            // p - 1 ticks of the window was not testable) with the same masks;
            // the zero sentinel words past the horizon end the loop
            int t = t0;
            while (f == 0u) {
              t += 33 - A.p;
              const uint32_t bwb = waddr(L, BB + min(t >> 5, BW));
              f = run_test(~__funnelshift_r(lds(bwb), lds(bwb + 128), t & 31), A);
            }
            S = t + __ffs(f) - 1;
          } else {
            S = t0 + __ffs(f) - 1;
            if (f == 0u || A.q != qmin) S = lane_search(L, t0, A.p, A.q - qmin, bias4);
          }
          const int C = S + A.p;
          if (C > hcap) {
            ovf = true;
            live = false;
          } else {
            // E: job / machine times (the next op's loads follow in program order)
            sts(A.ra, (rw & ~(TM << A.rsh)) | ((uint32_t)C << A.rsh));
            sts(A.ma, (mw & ~(TM << A.msh)) | ((uint32_t)C << A.msh));
            // D: level += q on [S, C) (<= 3 words, p <= 8), refresh blocked bits
            const int w0 = S >> 2;
            uint4 mk;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(mk.x), "=r"(mk.y), "=r"(mk.z), "=r"(mk.w)
                         : "r"(cm_base + ((((S & 3) << 3) + A.p - 1) << 4)));
            const uint32_t a0 = waddr(L, LB + w0);
            const uint32_t ba = waddr(L, BB + (w0 >> 3));
            const uint32_t B0 = lds(ba);
            const uint32_t v0 = lds(a0) + (A.QQ & mk.x);
            const uint32_t v1 = lds(a0 + 128) + (A.QQ & mk.y);
            const uint32_t v2 = lds(a0 + 256) + (A.QQ & mk.z);
            sts(a0, v0);
            sts(a0 + 128, v1);
            sts(a0 + 256, v2);
            // flags of untouched words are already in `blocked`: OR-ing them is harmless
            const uint32_t nib = flag_nibble(v0) | (flag_nibble(v1) << 4) | (flag_nibble(v2) << 8);
            const int sh = (w0 & 7) << 2;
            sts(ba, B0 | (nib << sh));
            const uint32_t spill = sh ? nib >> (32 - sh) : 0u;
            if ((w0 >> 3) + 1 < BW) sts(ba + 128, lds(ba + 128) | spill);   // stay inside this lane's words
            if (SCHED) srow[A.e / h.O] = S + h.rs;
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
      const int Cr = (int)((lds(waddr(L, j >> 1)) >> ((j & 1) << 4)) & TM);
      const int tj = Cr - pd[k];
      T += tj > 0 ? tj : 0;
      cm = max(cm, Cr + h.rs);
    }
    T += h.frozen_T;
    const int64_t obj = objective_word(h.real_wt, h.wt, h.wt_f, T, cm);
    if (a.obj) a.obj[gc] = obj;
    if (a.tard) a.tard[gc] = T;
    if (a.cmax) a.cmax[gc] = cm;
    if (a.fit) a.fit[gc] = fitness_word(h.real_wt, *a.emax, obj);   // Eq. (13)
  }
}

// ---------------------------------------------------------------------------
// Mode 2 (every Q_jsm == 1, Q_max <= 15: the paper's Table 5 setting), one
// lane per chromosome, SOFTWARE-PIPELINED across dispatches:
//   iteration r:  commit-1 of op r (job / machine times)
//                 load op r+1's job / machine words
//                 commit-2 of op r (headroom planes, blocked bits)
//                 stage A of op r+2 (table fields, run-test shifts)
//                 search of op r+1 (earliest power-feasible start)
// so op r+1's t0 arithmetic overlaps op r's plane update; op r+1's blocked
// words are read after op r's stores (program order of the shared accesses).
// Bit order is REVERSED (tick t at bit 31 - t%32 of word t/32): the earliest
// run is the highest set bit of the run mask, found by one clz.  The two
// sentinel words past the horizon are BLOCKED, so a run found in the first
// window always ends inside the horizon (C <= hcap); only the window-slide
// path can overflow.
// ---------------------------------------------------------------------------
struct Op2 {
  uint32_t ra, ma;        // shared addresses of the job's ready word and the machine word
  uint32_t rsh, msh;      // wrap-shift amounts of the two 10-bit fields (low 5 bits)
  uint32_t rmul, mmul;    // 1 << rsh, 1 << msh: field updates by IMAD (fma pipe)
  uint32_t m1n, m2, m4;   // run-test multipliers: -(1 << s1), 1 << s2, 1 << s4
  uint32_t top;           // the p ticks of an interval starting a 16-tick window: bits 15..16-p
  int pm1;                // p - 1
  uint32_t e;             // table index (SCHED: cell = e / O)
};

// The integer ALU pipe (LOP3/SHF/IADD3/SEL/...) issues every other cycle per
// SMSP and bounds this kernel; multiplies by powers of two run on the fma
// pipe, so left shifts by per-op amounts are written as IMADs.
__device__ __forceinline__ Op2 stage2(uint32_t pqt_s, uint32_t lbase, uint32_t mbase, uint32_t pt_base,
                                      uint32_t e) {
  // host-packed: rsh[0:5] | msh[5:10] | ready word[10:21] | machine word[21:29] | p-1[29:32]
  const uint32_t tv = lds(pqt_s + 4u * e);
  Op2 A;
  A.e = e;
  A.rsh = tv;
  A.msh = tv >> 5;
  // 2^shift by a wrap funnel shift (no mask), kept opaque so the compiler
  // does not turn the field updates' multiplies back into alu-pipe shifts
  A.rmul = __funnelshift_l(0u, 1u, tv);
  A.mmul = __funnelshift_l(0u, 1u, tv >> 5);
  pin(A.rmul);
  pin(A.mmul);
  A.ra = lbase + ((tv >> 3) & 0x3FF80u);
  A.ma = mbase + ((tv >> 14) & 0x7F80u);
  const uint32_t pm1 = tv >> 29;
  A.pm1 = (int)pm1;
  uint4 pt;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(pt.x), "=r"(pt.y), "=r"(pt.z), "=r"(pt.w)
               : "r"(pt_base + (pm1 << 4)));
  A.m1n = pt.x;
  A.m2 = pt.y;
  A.m4 = pt.z;
  A.top = pt.w;
  return A;
}

// runs of p free ticks in the window w of blocked bits (reversed order): bit
// i set iff the ticks of bits i, i-1, .., i-p+1 are free.  ~w * m = w * (-m) - m.
__device__ __forceinline__ uint32_t runs2(uint32_t w, const Op2 &A) {
  uint32_t f = ~w & (w * A.m1n + A.m1n);
  f &= f * A.m2;
  f &= f * A.m4;
  return f;
}

// the overflow path's reset of a lane's job / machine times (out of line: it
// is rare, and inlining it into every unrolled dispatch bloats the loop)
__device__ __noinline__ void reset_fields(uint32_t lbase, int n) {
  for (int w = 0; w < n; ++w) sts(lbase + ((uint32_t)w << 7), 0u);
}

// Earliest start >= t0 of p free ticks (reversed bit order).  Overflow (no
// run inside the horizon, rare path): the lane's result is void (sgn = -1,
// the fallback re-decodes the chromosome) and its job / machine times are
// reset to 0, so it goes on with every later access inside its own words and
// every field update non-negative; the op is committed at 0.
__device__ __forceinline__ int search2(const Op2 &A, int t0, uint32_t bb_base, int hcap, uint32_t lbase,
                                       int nfield_words, uint32_t &rw, uint32_t &mw, uint32_t &rf, uint32_t &mf,
                                       int &sgn) {
  uint32_t q = (uint32_t)t0 >> 5;
  pin(q);   // shift + IMAD, not shift-left + mask + add
  const uint32_t wa = bb_base + q * 128u;
  uint32_t f = runs2(__funnelshift_l(lds(wa + 128), lds(wa), (uint32_t)t0), A);
  int t = t0;
  if (f == 0u) {
    // window miss: slide by 33 - p ticks (a run starting in the last p - 1
    // ticks of the window was not testable); blocked sentinels end it
    do {
      t += 32 - A.pm1;
      if (t + A.pm1 >= hcap) {
        reset_fields(lbase, nfield_words);
        rw = mw = rf = mf = 0u;
        sgn = -1;
        return 0;
      }
      const uint32_t wb = bb_base + ((uint32_t)(t >> 5) << 7);
      f = runs2(__funnelshift_l(lds(wb + 128), lds(wb), (uint32_t)t), A);
    } while (f == 0u);
  }
  return t + __clz(f);
}

// Headroom Q_max - Q_t (every Q == 1) of 8 ticks in one word: byte b
// = bit plane b, tick i of the group at bit 7 - i.  Decrement by one on the
// ticks of the 8-bit mask m (each has headroom >= 1): plane b flips where m
// and every lower plane is 0 (borrow chain), i.e. under m & AND_{b'<b} ~h_b'.
__device__ __forceinline__ uint32_t dec8(uint32_t W, uint32_t mrep) {   // mrep: mask in all four bytes
  // byte b of W<<8, W<<16, W<<24 holds planes b-1, b-2, b-3 (zero-filled), so
  // ~(W<<8 | W<<16 | W<<24) is AND_{b'<b} ~h_b' in byte b; the shifts are
  // multiplies (fma pipe)
  const uint32_t lower = (W * 0x100u) | (W * 0x10000u) | (W * 0x1000000u);
  return W ^ (mrep & ~lower);
}
// blocked flags (headroom 0 <=> every plane 0) of two groups, tick i at bit
// 7 - i: group N0 in byte 0, group N1 in byte 2
__device__ __forceinline__ uint32_t blk2(uint32_t N0, uint32_t N1) {
  const uint32_t z = __byte_perm(N0, N1, 0x5410) | __byte_perm(N0, N1, 0x7632);   // planes 0|2, 1|3
  uint32_t r;   // ~(z | z >> 8) in one LOP3
  asm("lop3.b32 %0, %1, %2, 0, 0x03;" : "=r"(r) : "r"(z), "r"(z >> 8));
  return r;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts8m1(uint32_t a, uint32_t v) {   // byte at a - 1
  asm volatile("st.shared.u8 [%0+-1], %1;" ::"r"(a), "r"(v) : "memory");
}

// min(field, cap) for the three 10-bit fields of a word
__device__ __forceinline__ uint32_t clamp3(uint32_t w, uint32_t cap) {
  uint32_t o = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) o |= min((w >> (10 * i)) & 0x3FFu, cap) << (10 * i);
  return o;
}

// LIST: the re-decode of the chunk's overflow list a.ovf (chromosome ids;
// entries of other chunks are skipped) with a longer horizon a.h_cap; what
// still overflows goes to a.ovf2 for the general fallback.
template <bool SCHED, bool LIST>
__global__ void __launch_bounds__(512, 1) lane_decode2_kernel(EvalArgs a, int32_t lane_wpt) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  pdl_trigger();
  if (LIST) {
    pdl_wait();
    if (*(volatile const int32_t *)a.ovf == 0) return;   // nothing listed: before staging
  }
  __shared__ uint4 ptab[8];      // by p-1: run-test multipliers (-2^a, 2^b, 2^c), p ticks at bits 15..16-p
  if (threadIdx.x < 8) {
    const int p = threadIdx.x + 1;
    const uint32_t sa = p >= 2 ? 1u : 0u;
    const uint32_t sb = p >= 4 ? 2u : (p == 3 ? 1u : 0u);
    const uint32_t sc = p >= 5 ? (uint32_t)(p - 4) : 0u;
    ptab[threadIdx.x] = make_uint4(0u - (1u << sa), 1u << sb, 1u << sc, ((1u << p) - 1u) << (16 - p));
  }
  const uint32_t img_bytes = ((const ImageHdr *)a.image)->lane_image_bytes;
  stage_image(smem, a.image, img_bytes, &bar);   // the state image: a constant of the state
  uint32_t pt_base = smem_u32(ptab);
  pin(pt_base);
  const ImageHdr &h = *(const ImageHdr *)smem;
  const int K = h.K, KQ = (K + 3) >> 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t lbase = smem_u32(smem + img_bytes + (size_t)warp * lane_wpt * 128) + lane * 4;
  const int RW = (h.NJ + 2) / 3, MW = (h.G * h.O + 2) / 3;
  const int hcap = a.h_cap, BW = hcap >> 5;
  const int LB = RW + MW, BB = LB + 4 * BW + 1;   // 4 plane words per 32 ticks + one dummy group
  uint32_t mbase = lbase + ((uint32_t)RW << 7), pl_base = lbase + ((uint32_t)LB << 7),
           bb_base = lbase + ((uint32_t)BB << 7);
  pin(mbase);
  pin(pl_base);
  pin(bb_base);
  const uint32_t bb3 = bb_base + 3u;
  uint32_t pqt_s = smem_u32(smem + h.off_pqt);
  pin(pqt_s);
  const uint32_t *r10 = (const uint32_t *)(smem + h.off_ready16);
  const uint32_t *m10 = (const uint32_t *)(smem + h.off_mfree16);
  const uint32_t *pl0 = (const uint32_t *)(smem + h.off_hn0);   // initial planes, 5 words per tick-word
  const int64_t nunits = LIST ? (int64_t)*(volatile const int32_t *)a.ovf : a.count;
  const int64_t ntile = (nunits + 31) / 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  // LIST: a short list, one warp per SM first (its chain runs alone)
  const int64_t tile0 = LIST ? (int64_t)warp * gridDim.x + blockIdx.x : (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  bool waited = LIST;
  for (int64_t tile = tile0; tile < ntile; tile += nw) {
    int64_t c = tile * 32 + lane, gc = a.first + c;
    bool active = c < a.count;
    if (LIST) {
      gc = c < nunits ? (int64_t)a.ovf[1 + c] : -1;
      c = gc - a.first;
      active = gc >= 0 && c >= 0 && c < a.count;
      if (!active) c = 0;
    }
    // --- initial state: times clamped to the horizon (an op that cannot start
    // before it overflows either way), RUNNING ops' headroom, sentinels
    for (int w = 0; w < RW; ++w) sts(lbase + ((uint32_t)w << 7), clamp3(r10[w], (uint32_t)hcap));
    for (int w = 0; w < MW; ++w) sts(mbase + ((uint32_t)w << 7), clamp3(m10[w], (uint32_t)hcap));
    {
      // host image: per 32 ticks four plane words + blocked word, tick t at bit t%32
      const uint32_t qm = (uint32_t)h.lane_units;   // headroom of an empty tick, in ops
      for (int tw = 0; tw < BW; ++tw) {
        const bool init = 5 * tw < h.hn_words0;
        uint32_t pr[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) pr[b] = init ? __brev(pl0[5 * tw + b]) : (((qm >> b) & 1u) ? 0xFFFFFFFFu : 0u);
        // group k (ticks 32tw + 8k ..) = byte 3-k of every reversed plane
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t sel = 3u - (uint32_t)k;
          const uint32_t lo = __byte_perm(pr[0], pr[1], sel | ((sel + 4u) << 4));
          const uint32_t hi = __byte_perm(pr[2], pr[3], sel | ((sel + 4u) << 4));
          sts(pl_base + ((uint32_t)(4 * tw + k) << 7), __byte_perm(lo, hi, 0x5410));
        }
        sts(bb_base + ((uint32_t)tw << 7), init ? __brev(pl0[5 * tw + 4]) : 0u);
      }
      sts(pl_base + ((uint32_t)(4 * BW) << 7), 0u);   // dummy group past the horizon: blocked
      sts(bb_base + ((uint32_t)BW << 7), 0xFFFFFFFFu);
      sts(bb_base + ((uint32_t)(BW + 1) << 7), 0xFFFFFFFFu);
    }
    // the lane state above comes from the image; ordg, x and the outputs
    // belong to earlier kernels (first tile: its initialisation overlapped
    // the predecessor's drain)
    if (!LIST && !waited) {
      pdl_wait();
      waited = true;
    }
    int32_t *srow = nullptr;
    if (SCHED && active) {
      srow = a.start_out + gc * h.cells;
      for (int k = 0; k < h.cells; ++k) srow[k] = a.fstart[k];
    }
    // the chromosome's ranks: lane c % 32 of ordg tile c / 32
    int kq_pref = active ? KQ : 0;   // prefetch bound (0 for inactive lanes): one 32-bit compare per quad
    pin(kq_pref);                    // (not re-derived from the 64-bit c < count)
    const uint2 *op = (const uint2 *)(a.ordg + (c >> 5) * (int64_t)KQ * 128) + (c & 31);
    uint2 cur = active ? op[0] : make_uint2(0, 0);
    uint2 nxt = (active && KQ > 1) ? op[32] : make_uint2(0, 0);
    // prologue: ops 0 and 1 staged, op 0 searched
    Op2 A = stage2(pqt_s, lbase, mbase, pt_base, lo16(cur.x));
    Op2 An = stage2(pqt_s, lbase, mbase, pt_base, K > 1 ? hi16(cur.x) : 0u);
    uint32_t rw = lds(A.ra), mw = lds(A.ma);
    uint32_t rf = __funnelshift_r(rw, 0u, A.rsh) & 0x3FFu, mf = __funnelshift_r(mw, 0u, A.msh) & 0x3FFu;
    int sgn = 0;
    int S = search2(A, (int)max(rf, mf), bb_base, hcap, lbase, RW + MW, rw, mw, rf, mf, sgn);
    // one pipelined step: commit op r (A, S, rw, mw), load + search op r+1 (An),
    // stage op r+2 (table index e2); MORE: op r+1 exists
    auto step = [&](const int r, const uint32_t e2, const bool more) {
      // commit-1 of op r: job / machine times, field += (C - field) << shift
      const int Sx = S;
      const uint32_t C = (uint32_t)Sx + (uint32_t)A.pm1 + 1u;
      sts(A.ra, rw + (C - rf) * A.rmul);
      sts(A.ma, mw + (C - mf) * A.mmul);
      if (more) {
        rw = lds(An.ra);
        mw = lds(An.ma);
      }
      // commit-2 of op r: headroom of the 8-tick groups w = S/8 and w+1, their
      // blocked bytes (byte 3 - w%4 of blocked word w/4)
      {
        const uint32_t w = (uint32_t)Sx >> 3;
        const uint32_t m16 = A.top >> ((uint32_t)Sx & 7u);   // ticks 8w.. at bits 15..
        const uint32_t pa = pl_base + (w << 7);
        const uint32_t W0 = lds(pa), W1 = lds(pa + 128);
        const uint32_t N0 = dec8(W0, __byte_perm(m16, 0u, 0x1111)), N1 = dec8(W1, __byte_perm(m16, 0u, 0x0000));
        sts(pa, N0);
        sts(pa + 128, N1);
        // group v's blocked byte: word v/4, byte 3 - v%4, i.e. bb_base + 128 q
        // + 3 - (v - 4q) = 132 q + (bb_base + 3 - v) with q = v/4 (one IMAD);
        // group w+1 at 132 q' + (bb_base + 3 - w) - 1, q' = (S + 8) / 32
        uint32_t q = (uint32_t)Sx >> 5, q2 = ((uint32_t)Sx + 8u) >> 5;
        pin(q);
        pin(q2);
        const uint32_t tq = bb3 - w;
        const uint32_t bk = blk2(N0, N1);
        sts8(q * 132u + tq, bk);
        sts8m1(q2 * 132u + tq, bk >> 16);
      }
      if (SCHED && active) {   // gene-indexed table: the op's cell from the image's gene info
        const uint32_t gi = __ldg((const uint32_t *)((const unsigned char *)a.image + h.off_ginfo) + A.e / h.O);
        srow[(gi & 0xFFFFu) * h.G + (gi >> 16)] = Sx + h.rs;
      }
      // stage A of op r+2 (ranks >= K carry the padding index 0: harmless)
      const Op2 A2 = stage2(pqt_s, lbase, mbase, pt_base, e2);
      A = An;
      An = A2;
      // search of op r+1
      if (more) {
        rf = __funnelshift_r(rw, 0u, A.rsh) & 0x3FFu;
        mf = __funnelshift_r(mw, 0u, A.msh) & 0x3FFu;
        S = search2(A, (int)max(rf, mf), bb_base, hcap, lbase, RW + MW, rw, mw, rf, mf, sgn);
      }
    };
    // main loop: whole quads whose every op has a successor (no exits inside)
    int qd = 0;
    for (; 4 * qd + 4 < K; ++qd) {
      const uint2 pre = qd + 2 < kq_pref ? op[(size_t)(qd + 2) * 32] : make_uint2(0, 0);
      step(4 * qd + 0, lo16(cur.y), true);
      step(4 * qd + 1, hi16(cur.y), true);
      step(4 * qd + 2, lo16(nxt.x), true);
      step(4 * qd + 3, hi16(nxt.x), true);
      cur = nxt;
      nxt = pre;
    }
    // tail: the last 1..4 ops
    for (int r = 4 * qd; r < K; ++r) {
      const int k = r & 3;
      const uint32_t e2 = k == 0 ? lo16(cur.y) : k == 1 ? hi16(cur.y) : k == 2 ? lo16(nxt.x) : hi16(nxt.x);
      step(r, e2, r + 1 < K);
    }
    if (!active) continue;
    if (sgn < 0) {
      int32_t *ol = LIST ? a.ovf2 : a.ovf;
      int pos = atomicAdd(&ol[0], 1);
      ol[1 + pos] = (int32_t)gc;
      if (!LIST && a.ovf_seen) *(volatile int32_t *)a.ovf_seen = 1;
      continue;
    }
    // Eqs. (1)-(3) over every job (R9); frozen jobs are constants of the state
    const int32_t *pj = (const int32_t *)(smem + h.off_pjob);
    const int32_t *pd = (const int32_t *)(smem + h.off_pdue);
    int64_t T = 0;
    int cm = h.frozen_cmax;
    for (int k = 0; k < h.n_pjobs; ++k) {
      const int j = pj[k];
      const int wj = (j * 0xAAAB) >> 17;
      const int Cr = (int)((lds(lbase + ((uint32_t)wj << 7)) >> ((j - 3 * wj) * 10)) & 0x3FFu);
      const int tj = Cr - pd[k];
      T += tj > 0 ? tj : 0;
      cm = max(cm, Cr + h.rs);
    }
    T += h.frozen_T;
    const int64_t obj = objective_word(h.real_wt, h.wt, h.wt_f, T, cm);
    if (a.obj) a.obj[gc] = obj;
    if (a.tard) a.tard[gc] = T;
    if (a.cmax) a.cmax[gc] = cm;
    if (a.fit) a.fit[gc] = fitness_word(h.real_wt, *a.emax, obj);   // Eq. (13)
  }
  if (!waited) pdl_wait();   // warps without a tile: the grid still completes after its predecessor
}

template <typename KERN>
ffs_status smem_attr(KERN k, size_t bytes) {
  return ensure_smem_attr((const void *)k, bytes);
}

}  // namespace

ffs_status launch_lane(const State &st, const EvalArgs &a0, OvfScratch &scr, cudaStream_t s, int *launches) {
  const int K = st.K, KQ = (K + 3) / 4;
  const int64_t chunk_max = (int64_t)1 << 17;
  const int64_t chunk = std::min<int64_t>((a0.count + 31) / 32 * 32, chunk_max);
  const int64_t elems = chunk / 32 * (int64_t)KQ * 128;
  if (elems > scr.ordg_elems) {
    scr.free_(scr.ordg);
    scr.ordg = nullptr;
    ffs_status ea = scr.alloc((void **)&scr.ordg, (size_t)elems * 2);
    if (ea != FFS_OK) return ea;
    scr.ordg_elems = elems;
  }
  // the segmented min-scan's doubling steps: 2^SCAN > lanes a job's pending
  // genes can span - 1 (pm_quad)
  const int span = (st.max_pending + 2) / 4 + 1;
  const int scan = span <= 4 ? 2 : span <= 8 ? 3 : 5;
  // [GIDX][scan 2/3/5][XS][BULK]
#define OKS(G, S) {{order_warp_kernel<false, S, false, G>, order_warp_kernel<true, S, false, G>}, \
                   {order_warp_kernel<false, S, true, G>, order_warp_kernel<true, S, true, G>}}
  static void (*const okerns[2][3][2][2])(OrdArgs) = {{OKS(false, 2), OKS(false, 3), OKS(false, 5)},
                                                       {OKS(true, 2), OKS(true, 3), OKS(true, 5)}};
#undef OKS
  const int mode = ((const ImageHdr *)st.image_host.data())->lane_mode;
  const int si = scan == 2 ? 0 : scan == 3 ? 1 : 2, xi = st.ord_xs ? 1 : 0, gi = mode == 2 ? 1 : 0;
  void (*okern)(OrdArgs) = okerns[gi][si][xi][0], (*okern_v)(OrdArgs) = okerns[gi][si][xi][1];
  const size_t osm = st.ord_smem + (st.ord_xs ? st.ord_xs_bytes : 0);
  ffs_status e = smem_attr(okern, osm);
  if (e == FFS_OK) e = smem_attr(okern_v, osm);
  if (e != FFS_OK) return e;
  const bool sched = a0.start_out != nullptr;
  void (*kern)(EvalArgs, int32_t) =
      mode == 2 ? (sched ? lane_decode2_kernel<true, false> : lane_decode2_kernel<false, false>)
      : mode == 1 ? (sched ? lane_decode_kernel<1, true> : lane_decode_kernel<1, false>)
                  : (sched ? lane_decode_kernel<0, true> : lane_decode_kernel<0, false>);
  e = smem_attr(kern, st.lane_smem);
  if (e != FFS_OK) return e;
  // mode 2: the overflow list's re-decode with the longer horizon lane_hcap2
  const bool relist = mode == 2 && a0.relist;
  void (*kern2)(EvalArgs, int32_t) = sched ? lane_decode2_kernel<true, true> : lane_decode2_kernel<false, true>;
  if (relist) {
    e = smem_attr(kern2, st.lane_smem2);
    if (e != FFS_OK) return e;
  }
  for (int64_t first = 0; first < a0.count; first += chunk) {
    EvalArgs a = a0;
    a.first = first;
    a.count = std::min<int64_t>(chunk, a0.count - first);
    a.ordg = scr.ordg;
    a.h_cap = st.lane_hcap;
    a.ovf = scr.list;
    const int64_t ntile = (a.count + 31) / 32;
    OrdArgs oa;
    oa.x = a0.x;
    oa.y = a0.y;
    oa.first = first;
    oa.count = a.count;
    oa.row = a0.row > 0 ? a0.row : K;
    oa.vec = (oa.row % 16 == 0) && ((uintptr_t)a0.x % 16 == 0) && ((uintptr_t)a0.y % 16 == 0);
    oa.K = K;
    oa.head = (const uint32_t *)((const unsigned char *)st.image_dev +
                                 ((const ImageHdr *)st.image_host.data())->off_head);
    oa.gbase = st.gbase_dev;
    oa.ordg = scr.ordg;
    oa.hist_bytes = (uint32_t)st.ord_hist_bytes;
    oa.ord_stride = (uint32_t)st.ord_stride;
    oa.pm_bytes = (uint32_t)(((size_t)(K + 127) / 128 * 128 * 2 + 15) & ~(size_t)15);
    oa.ubits = st.ord_ubits;
    oa.O = st.inst->o;
    oa.zero0 = first == 0 ? scr.list : nullptr;
    oa.zero1 = first == 0 ? scr.list2 : nullptr;
    int64_t og = std::min<int64_t>(ntile, (int64_t)st.num_sms * st.ord_ctas_per_sm);
    FFS_CUDA(launch_pdl(oa.vec ? okern_v : okern, dim3((unsigned)og), dim3(1024), osm, s, oa));
    const int64_t wpc = st.lane_warps_per_cta;
    int64_t lg = std::min<int64_t>((ntile + wpc - 1) / wpc, (int64_t)st.num_sms * st.lane_ctas_per_sm);
    const unsigned thr = (unsigned)(wpc * 32);
    FFS_CUDA(launch_pdl(kern, dim3((unsigned)lg), dim3(thr), st.lane_smem, s, a, st.lane_wpt));
    if (launches) *launches += 2;
    if (relist) {   // launched unconditionally (no host round trip); empty list: every CTA leaves at once
      EvalArgs b = a;
      b.h_cap = st.lane_hcap2;
      b.ovf2 = scr.list2;
      FFS_CUDA(launch_pdl(kern2, dim3((unsigned)st.num_sms), dim3((unsigned)(st.lane_warps2 * 32)), st.lane_smem2, s,
                          b, st.lane_wpt2));
      if (launches) *launches += 1;
    }
  }
  return FFS_OK;
}

}  // namespace edffs
