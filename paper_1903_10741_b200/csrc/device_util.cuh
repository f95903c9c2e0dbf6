// device_util.cuh -- device helpers shared by the evaluate kernels:
// TMA staging of the state image, warp scans, and Algorithm 1 (order).
#pragma once
#include <climits>

#include "ffs_common.cuh"

namespace edffs {
namespace dev {

constexpr uint32_t FULL = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Stage the state image global -> shared with the bulk-copy engine (TMA).
__device__ __forceinline__ void stage_image(unsigned char *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(dst + off)),
          "l"((const char *)src + off), "r"(n), "r"(smem_u32(bar))
          : "memory");
    }
  }
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// bit i of the result is set iff bits i .. i+p-1 of b are all set (p <= 32,
// bits above 31 count as clear)
__device__ __forceinline__ uint32_t runs_ge(uint32_t b, int p) {
  int k = 1;
  while (2 * k <= p) {
    b &= b >> k;
    k <<= 1;
  }
  if (k < p) b &= b >> (p - k);
  return b;
}

// Segmented inclusive min-scan over the 32 lanes (segments start at `head`),
// continued from `carry` when no head precedes the lane in this tile.
__device__ __forceinline__ int seg_min_scan(int v, bool head, int carry, int lane) {
  uint32_t f = head;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int vn = __shfl_up_sync(FULL, v, d);
    uint32_t fn = __shfl_up_sync(FULL, f, d);
    if (lane >= d) {
      if (!f) v = min(v, vn);
      f |= fn;
    }
  }
  if (!f) v = min(v, carry);
  return v;
}

// Algorithm 1 for one chromosome: fills ord[0..K) in rank order with
//   MODE 0: (gene | x << 16)                 (u32, warp-decode path)
//   MODE 1: (j*G + s)*O + x  = P/Q table index  (u16, lane-decode path)
struct OrderMem {
  void *ord;
  uint32_t *lbits;
  uint16_t *cnt;
};
template <int MODE>
__device__ __forceinline__ void build_order(const ImageHdr &h, const unsigned char *img, OrderMem w,
                                            const int8_t *__restrict__ xr, const int16_t *__restrict__ yr,
                                            int lane) {
  const int K = h.K, nt = (K + 31) >> 5;
  const uint32_t *head = (const uint32_t *)(img + h.off_head);
  // Pass A: pm(g) = min y over the job's pending stages <= s; leaders are the
  // genes with pm(g) == y(g) (new prefix minima: the eligible op with the
  // largest y among its job's remaining ops starts a run).
  int carry = INT_MAX;
  for (int t = 0; t < nt; ++t) {
    int g = (t << 5) + lane;
    bool valid = g < K;
    int yv = valid ? (int)__ldg(yr + g) : INT_MAX;
    bool hd = !valid || ((head[t] >> lane) & 1u);
    int pm = seg_min_scan(yv, hd, carry, lane);
    uint32_t lb = __ballot_sync(FULL, valid && pm == yv);
    if (lane == 0) w.lbits[t] = lb;
    carry = __shfl_sync(FULL, pm, 31);
  }
  __syncwarp();
  // Pass B: cnt[y(l) - 1] = length of leader l's run (genes until the next
  // leader in gene order); 0 for non-leaders.  y is a permutation of 1..K,
  // so every slot is written exactly once.
  for (int t = 0; t < nt; ++t) {
    int g = (t << 5) + lane;
    if (g < K) {
      int yv = (int)__ldg(yr + g);
      uint32_t lb = w.lbits[t];
      int cv = 0;
      if ((lb >> lane) & 1u) {
        uint32_t m = lane == 31 ? 0u : (lb & (FULL << (lane + 1)));
        int tt = t;
        while (m == 0u && ++tt < nt) m = w.lbits[tt];
        int next = m == 0u ? K : (tt << 5) + __ffs(m) - 1;
        cv = next - g;
      }
      unsigned yi = (unsigned)(yv - 1);
      if (yi < (unsigned)K) w.cnt[yi] = (uint16_t)cv;
    }
  }
  __syncwarp();
  // Pass C: exclusive suffix sum over priorities: cnt[v] <- #genes with pm > v+1
  int acc = 0;
  for (int t = 0; t < nt; ++t) {
    int v = K - 1 - ((t << 5) + lane);
    bool valid = v >= 0;
    int cv = valid ? (int)w.cnt[v] : 0;
    int incl = cv;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int n = __shfl_up_sync(FULL, incl, d);
      if (lane >= d) incl += n;
    }
    if (valid) w.cnt[v] = (uint16_t)(acc + incl - cv);
    acc += __shfl_sync(FULL, incl, 31);
  }
  __syncwarp();
  // Pass D: rank(g) = start[pm(g)] + (g - leader(g)); scatter.
  carry = INT_MAX;
  int carry_lp = -1;
  for (int t = 0; t < nt; ++t) {
    int g = (t << 5) + lane;
    bool valid = g < K;
    int yv = valid ? (int)__ldg(yr + g) : INT_MAX;
    int xv = valid ? (int)__ldg(xr + g) : 0;
    bool hd = !valid || ((head[t] >> lane) & 1u);
    int pm = seg_min_scan(yv, hd, carry, lane);
    int lp = ((w.lbits[t] >> lane) & 1u) ? g : -1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int n = __shfl_up_sync(FULL, lp, d);
      if (lane >= d) lp = max(lp, n);
    }
    lp = max(lp, carry_lp);
    if (valid) {
      unsigned pi = (unsigned)(pm - 1);
      int rank = (pi < (unsigned)K ? (int)w.cnt[pi] : 0) + (g - lp);
      if ((unsigned)rank < (unsigned)K) {
        if (MODE == 0) {
          ((uint32_t *)w.ord)[rank] = (uint32_t)g | ((uint32_t)(xv & 0xFF) << 16);
        } else {
          uint32_t gi = ((const uint32_t *)(img + h.off_ginfo))[g];
          int m = xv < h.O ? (xv > 0 ? xv : 0) : h.O - 1;
          ((uint16_t *)w.ord)[rank] = (uint16_t)(((int)(gi & 0xFFFFu) * h.G + (int)(gi >> 16)) * h.O + m);
        }
      }
    }
    carry = __shfl_sync(FULL, pm, 31);
    carry_lp = __shfl_sync(FULL, lp, 31);
  }
  __syncwarp();
}


}  // namespace dev
}  // namespace edffs
