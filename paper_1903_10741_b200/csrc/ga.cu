// ga.cu -- island GA of one rescheduling point on sm_100a.
//
// Population: global island I owns cells I*tile + i (i row-major in the
// island tile, tile = island_w * island_h); SoA device buffers x int8[cell][KP],
// y int16[cell][KP] (rows padded to KP = K rounded up to 16 genes, so every
// row is 16-B aligned and moves with 16-B vector accesses), obj/fit
// int64[cell], double-buffered across generations (synchronous update from
// the previous generation's snapshot, R18).
// Per generation (operator order R20):
//   generation_kernel  warp per horizontal pair: asteroid selection,
//                      neighbouring paired crossover + correction,
//                      mutation                     -> next buffer
//   evaluate           decode + objective + fitness (Eq. (13))
//   replace_kernel     CTA per island: elitist replacement
//   donor/import       ring migration every migration_interval,
//                      allgather hook across processes
//   trace              min objective and sum of objectives: per-island partials in
//                      replace_kernel (import_kernel on migration generations),
//                      reduced by the last island block to finish
// Random draws: Philox4x32-10 keyed by the seed, counter
// (purpose << 24 | block, individual, generation, island) -- DESIGN.md "RNG".
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "ffs_common.cuh"

namespace edffs {

struct Run {
  State *st = nullptr;
  ffs_ga_config cfg{};
  cudaStream_t s = nullptr;
  int tile = 0, nisl = 0, K = 0, cells = 0;
  int64_t row = 0;                  // KP: padded genes per population / history row
  int64_t nloc = 0;
  int gen = -1;
  int cur = 0;
  int8_t *x[2] = {nullptr, nullptr};
  int16_t *y[2] = {nullptr, nullptr};
  int64_t *obj[2] = {nullptr, nullptr};
  int64_t *fit[2] = {nullptr, nullptr};
  int8_t *hx = nullptr;
  int16_t *hy = nullptr;
  int64_t *hobj = nullptr, *hfit = nullptr;
  int32_t *worst_idx = nullptr;
  unsigned char *donor = nullptr, *recv = nullptr;
  size_t rec = 0;
  int64_t *scal = nullptr;          // [0] emax, [1] max objective
  int64_t *tmin = nullptr, *tsum = nullptr;
  int64_t *parts = nullptr;         // [islands][2] per-island trace partials
  int64_t *best_v = nullptr;        // ffs_best: objective, sum T of the decoded elite
  int32_t *best_s = nullptr;        // ffs_best: its schedule [cells] + C_max
  unsigned *tcounter = nullptr;     // islands finished in the current trace
  OvfScratch scr;
  int64_t evaluations = 0;
  int launches = 0;
  std::vector<void *> allocs;
  // buffers are stream-ordered allocations from the default memory pool (kept
  // cached across runs: creating and destroying runs in a workflow does not
  // synchronise the device)
  ~Run() {
    for (void *p : allocs) cudaFreeAsync(p, s);
    scr.release();
  }
  template <typename T>
  ffs_status alloc(T **p, size_t n) {
    void *q = nullptr;
    FFS_CUDA(cudaMallocAsync(&q, std::max<size_t>(n, 1) * sizeof(T), s));
    allocs.push_back(q);
    *p = (T *)q;
    return FFS_OK;
  }
};

namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;

// ---- initialisation: x ~ U{0..o-1}, y = 1 + rank of a random key
// (warp per chromosome; the ranks by a bitonic sort in shared memory, NP u64
// per warp)
__global__ void __launch_bounds__(256) init_kernel(int32_t K, int32_t NP, int64_t row, int32_t O, int64_t count,
                                                   int32_t tile, int32_t island0, uint64_t seed, int8_t *x,
                                                   int16_t *y) {
  extern __shared__ __align__(16) unsigned long long keys_all[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long *buf = keys_all + (size_t)warp * NP;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; c < count; c += nw) {
    const uint32_t island = (uint32_t)(island0 + c / tile), indiv = (uint32_t)(c % tile);
    for (int g = lane; g < K; g += 32) {
      u32x4 rx = philox((RNG_INIT_X << 24) | (uint32_t)(g >> 2), indiv, 0u, island, k0, k1);
      u32x4 ry = philox((RNG_INIT_Y << 24) | (uint32_t)(g >> 2), indiv, 0u, island, k0, k1);
      x[c * row + g] = (int8_t)bounded(word_of(rx, g & 3), (uint32_t)O);
      buf[g] = ((unsigned long long)word_of(ry, g & 3) << 32) | (uint32_t)g;
    }
    rank_keys_warp(buf, K, NP, lane, y + c * row);
  }
}

// ---- E_max = 10^a, a >= 1, smallest with every initial objective < E_max
__global__ void max_kernel(const int64_t *obj, int64_t n, int64_t *out) {
  __shared__ long long sm[32];
  long long m = LLONG_MIN;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = max(m, (long long)obj[i]);
  for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(FULL, m, d));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : LLONG_MIN;
    for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(FULL, m, d));
    if (threadIdx.x == 0) *out = m;
  }
}

__global__ void emax_fitness_kernel(int64_t *scal, const int64_t *obj, int64_t *fit, int64_t n, int real) {
  int64_t E;
  if (real) {   // binary64 words (f3); powers of ten are exact up to 1e22
    const double mx = __longlong_as_double(scal[1]);
    double e = 10.0;
    for (int a = 1; a < 308 && e <= mx; ++a) e *= 10.0;   // bounded: objectives < 1e300 (state check)
    E = __double_as_longlong(e);
  } else {
    const int64_t mx = scal[1];
    E = 10;
    for (int a = 1; a < 18 && E <= mx; ++a) E *= 10;     // bounded: objectives < 1e17 (state check)
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) scal[0] = E;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    fit[i] = fitness_word(real, E, obj[i]);       // Eq. (13)
}

// ---- block helpers: argmax / argmin of fitness inside one island (ties -> lowest index)
__device__ __forceinline__ void better_max(int64_t &f, int &i, int64_t f2, int i2) {
  if (f2 > f || (f2 == f && i2 < i)) { f = f2; i = i2; }
}
__device__ __forceinline__ void better_min(int64_t &f, int &i, int64_t f2, int i2) {
  if (f2 < f || (f2 == f && i2 < i)) { f = f2; i = i2; }
}
__device__ void island_best_worst(const int64_t *fit, int tile, int &best, int &worst) {
  __shared__ long long sfb[32], sfw[32];
  __shared__ int sib[32], siw[32];
  int64_t fb = LLONG_MIN, fw = LLONG_MAX;
  int ib = INT_MAX, iw = INT_MAX;
  for (int i = threadIdx.x; i < tile; i += blockDim.x) {
    better_max(fb, ib, fit[i], i);
    better_min(fw, iw, fit[i], i);
  }
  for (int d = 16; d > 0; d >>= 1) {
    better_max(fb, ib, __shfl_xor_sync(FULL, fb, d), __shfl_xor_sync(FULL, ib, d));
    better_min(fw, iw, __shfl_xor_sync(FULL, fw, d), __shfl_xor_sync(FULL, iw, d));
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sfb[w] = fb; sib[w] = ib; sfw[w] = fw; siw[w] = iw; }
  __syncthreads();
  if (threadIdx.x < 32) {
    int nw = blockDim.x >> 5;
    fb = threadIdx.x < nw ? sfb[threadIdx.x] : LLONG_MIN;
    ib = threadIdx.x < nw ? sib[threadIdx.x] : INT_MAX;
    fw = threadIdx.x < nw ? sfw[threadIdx.x] : LLONG_MAX;
    iw = threadIdx.x < nw ? siw[threadIdx.x] : INT_MAX;
    for (int d = 16; d > 0; d >>= 1) {
      better_max(fb, ib, __shfl_xor_sync(FULL, fb, d), __shfl_xor_sync(FULL, ib, d));
      better_min(fw, iw, __shfl_xor_sync(FULL, fw, d), __shfl_xor_sync(FULL, iw, d));
    }
    if (threadIdx.x == 0) { sib[0] = ib; siw[0] = iw; }
  }
  __syncthreads();
  best = sib[0];
  worst = siw[0];
  __syncthreads();
}

__device__ __forceinline__ void copy_bytes(unsigned char *dst, const unsigned char *src, size_t n) {
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
// a padded population / history row (x: row bytes, y: 2*row bytes; 16-B aligned)
__device__ __forceinline__ void copy_row(int8_t *dx, int16_t *dy, const int8_t *sx, const int16_t *sy, int64_t row) {
  const int nx = (int)(row >> 4), ny = (int)(row >> 3);
  for (int i = threadIdx.x; i < nx + ny; i += blockDim.x) {
    if (i < nx) ((uint4 *)dx)[i] = ((const uint4 *)sx)[i];
    else ((uint4 *)dy)[i - nx] = ((const uint4 *)sy)[i - nx];
  }
}

// history elite record per island; generation 0 sets it unconditionally
__global__ void history_init_kernel(int64_t row, int tile, const int8_t *x, const int16_t *y, const int64_t *obj,
                                    const int64_t *fit, int8_t *hx, int16_t *hy, int64_t *hobj, int64_t *hfit) {
  const int li = blockIdx.x;
  const int64_t base = (int64_t)li * tile;
  int b, w;
  island_best_worst(fit + base, tile, b, w);
  const int64_t c = base + b;
  copy_row(hx + (int64_t)li * row, hy + (int64_t)li * row, x + c * row, y + c * row, row);
  if (threadIdx.x == 0) { hobj[li] = obj[c]; hfit[li] = fit[c]; }
}

// elitist replacement (R21): strict improvement updates the history;
// the island's worst cell is overwritten by the history elite.
struct TraceArgs {
  int64_t *parts;
  unsigned *counter;
  int64_t *tmin, *tsum;
  int k, real, nisl, on;
};

__device__ void island_trace(const int64_t *obj_isl, int tile, int real, int li, int nisl, int64_t *parts,
                             unsigned *counter, int64_t *tmin, int64_t *tsum, int k);

__device__ void block_min_sum(const int64_t *v, int64_t n, int real, long long &mn, long long &sm);

// one pass over an island's cells for the integer objective: best / worst
// fitness (ties -> lowest index), the worst cell's objective, and the island's
// objective min and sum (the trace partial before replacement)
__device__ void island_scan(const int64_t *fit, const int64_t *obj, int tile, int &best, int &worst, long long &ow,
                            long long &omin, long long &osum) {
  __shared__ long long sfb[32], sfw[32], sow[32], smn[32], ssm[32];
  __shared__ int sib[32], siw[32];
  int64_t fb = LLONG_MIN, fw = LLONG_MAX;
  int ib = INT_MAX, iw = INT_MAX;
  long long o_w = 0, mn = LLONG_MAX, sm = 0;
  for (int i = threadIdx.x; i < tile; i += blockDim.x) {
    const int64_t f = fit[i];
    const long long o = obj[i];
    better_max(fb, ib, f, i);
    if (f < fw || (f == fw && i < iw)) { fw = f; iw = i; o_w = o; }
    mn = min(mn, o);
    sm += o;
  }
  for (int d = 16; d > 0; d >>= 1) {
    better_max(fb, ib, __shfl_xor_sync(FULL, fb, d), __shfl_xor_sync(FULL, ib, d));
    const int64_t f2 = __shfl_xor_sync(FULL, fw, d);
    const int i2 = __shfl_xor_sync(FULL, iw, d);
    const long long o2 = __shfl_xor_sync(FULL, o_w, d);
    if (f2 < fw || (f2 == fw && i2 < iw)) { fw = f2; iw = i2; o_w = o2; }
    mn = min(mn, __shfl_xor_sync(FULL, mn, d));
    sm += __shfl_xor_sync(FULL, sm, d);
  }
  const int wp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sfb[wp] = fb; sib[wp] = ib; sfw[wp] = fw; siw[wp] = iw; sow[wp] = o_w; smn[wp] = mn; ssm[wp] = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      better_max(fb, ib, sfb[k], sib[k]);
      if (sfw[k] < fw || (sfw[k] == fw && siw[k] < iw)) { fw = sfw[k]; iw = siw[k]; o_w = sow[k]; }
      mn = min(mn, smn[k]);
      sm += ssm[k];
    }
    sib[0] = ib; siw[0] = iw; sow[0] = o_w; smn[0] = mn; ssm[0] = sm;
  }
  __syncthreads();
  best = sib[0];
  worst = siw[0];
  ow = sow[0];
  omin = smn[0];
  osum = ssm[0];
  __syncthreads();
}

// the island's trace partial is final: publish it; the last island block
// (ticket) reduces the partials in island order into trace[k]
__device__ void trace_publish(long long mn, long long sm, int real, int li, int nisl, int64_t *parts,
                              unsigned *counter, int64_t *tmin, int64_t *tsum, int k) {
  __shared__ unsigned ticket;
  if (threadIdx.x == 0) {
    parts[2 * li] = mn;
    parts[2 * li + 1] = sm;
    __threadfence();
    ticket = atomicAdd(counter, 1u);
  }
  __syncthreads();
  if (ticket != (unsigned)(nisl - 1)) return;
  __threadfence();
  block_min_sum(parts, nisl, real, mn, sm);
  if (threadIdx.x == 0) {
    tmin[k] = mn;
    tsum[k] = sm;
    *counter = 0u;
  }
}

__global__ void replace_kernel(int64_t row, int tile, int8_t *x, int16_t *y, int64_t *obj, int64_t *fit, int8_t *hx,
                               int16_t *hy, int64_t *hobj, int64_t *hfit, TraceArgs tr) {
  pdl_trigger();
  pdl_wait();
  const int li = blockIdx.x;
  const int64_t base = (int64_t)li * tile;
  __shared__ long long s_hist[2];   // the island's elite record: fitness, objective (before this generation)
  if (threadIdx.x == 0) {
    s_hist[0] = hfit[li];
    s_hist[1] = hobj[li];
  }
  // integer objective with the trace due now: one pass gives the trace partial
  // too (the worst cell's objective w_o is replaced by the elite's e_o <= w_o,
  // Eq. (13) being decreasing: min' = min(min, e_o), sum' = sum - w_o + e_o);
  // binary64 (f3) keeps R33's sequential sum over the updated cells below
  const bool fused = tr.on && !tr.real;
  int b, w;
  long long ow = 0, omin = 0, osum = 0;
  if (fused) island_scan(fit + base, obj + base, tile, b, w, ow, omin, osum);
  else island_best_worst(fit + base, tile, b, w);   // (their barriers publish s_hist)
  const int64_t cb = base + b, cw = base + w;
  int8_t *hxr = hx + (int64_t)li * row;
  int16_t *hyr = hy + (int64_t)li * row;
  const int64_t fb = fit[cb];
  const bool upd = fb > s_hist[0];   // strict improvement (R21)
  // one pass: worst <- (upd ? best : elite), elite <- best when upd (the old
  // two-pass order, elite first then worst <- elite, gives the same rows)
  {
    const int8_t *sx = upd ? x + cb * row : hxr;
    const int16_t *sy = upd ? y + cb * row : hyr;
    int8_t *dx = x + cw * row;
    int16_t *dy = y + cw * row;
    const int nx = (int)(row >> 4), ny = (int)(row >> 3);
    for (int i = threadIdx.x; i < nx + ny; i += blockDim.x) {
      if (i < nx) {
        const uint4 v = ((const uint4 *)sx)[i];
        ((uint4 *)dx)[i] = v;
        if (upd) ((uint4 *)hxr)[i] = v;
      } else {
        const uint4 v = ((const uint4 *)sy)[i - nx];
        ((uint4 *)dy)[i - nx] = v;
        if (upd) ((uint4 *)hyr)[i - nx] = v;
      }
    }
  }
  const int64_t ob = upd ? obj[cb] : (int64_t)s_hist[1];
  if (threadIdx.x == 0) {
    const int64_t fv = upd ? fb : (int64_t)s_hist[0];
    if (upd) {
      hobj[li] = ob;
      hfit[li] = fv;
    }
    obj[cw] = ob;
    fit[cw] = fv;
  }
  if (fused) {   // no migration this generation: the trace is final now
    trace_publish(min(omin, (long long)ob), osum - ow + (long long)ob, 0, li, tr.nisl, tr.parts, tr.counter,
                  tr.tmin, tr.tsum, tr.k);
  } else if (tr.on) {
    __syncthreads();
    island_trace(obj + base, tile, tr.real, li, tr.nisl, tr.parts, tr.counter, tr.tmin, tr.tsum, tr.k);
  }
}

// ring migration, part 1: snapshot every island's best (after replacement)
// and remember its worst cell (R22)
__global__ void donor_kernel(int K, int64_t row, int tile, size_t rec, const int8_t *x, const int16_t *y,
                             const int64_t *obj, const int64_t *fit, unsigned char *donor, int32_t *worst_idx) {
  pdl_trigger();
  pdl_wait();
  const int li = blockIdx.x;
  const int64_t base = (int64_t)li * tile;
  int b, w;
  island_best_worst(fit + base, tile, b, w);
  const int64_t cb = base + b;
  unsigned char *d = donor + (size_t)li * rec;   // compact record: x[K] y[K] obj fit
  copy_bytes(d, (const unsigned char *)(x + cb * row), (size_t)K);
  copy_bytes(d + K, (const unsigned char *)(y + cb * row), (size_t)K * 2);
  if (threadIdx.x == 0) {
    int64_t o = obj[cb], f = fit[cb];
    memcpy(d + 3 * (size_t)K, &o, 8);
    memcpy(d + 3 * (size_t)K + 8, &f, 8);
    worst_idx[li] = (int32_t)(base + w);
  }
}

// part 2: island li's worst cell <- best of island li-1; island 0 of the shard
// <- `incoming` (the last island of the previous shard, or of this shard)
__global__ void import_kernel(int K, int64_t row, int tile, size_t rec, const unsigned char *donor,
                              const unsigned char *incoming, const int32_t *worst_idx, int8_t *x, int16_t *y,
                              int64_t *obj, int64_t *fit, TraceArgs tr) {
  pdl_trigger();
  pdl_wait();
  const int li = blockIdx.x;
  const unsigned char *src = li == 0 ? incoming : donor + (size_t)(li - 1) * rec;
  const int64_t cw = worst_idx[li];
  copy_bytes((unsigned char *)(x + cw * row), src, (size_t)K);
  copy_bytes((unsigned char *)(y + cw * row), src + K, (size_t)K * 2);
  if (threadIdx.x == 0) {
    int64_t o, f;
    memcpy(&o, src + 3 * (size_t)K, 8);
    memcpy(&f, src + 3 * (size_t)K + 8, 8);
    obj[cw] = o;
    fit[cw] = f;
  }
  __syncthreads();
  island_trace(obj + (int64_t)li * tile, tile, tr.real, li, tr.nisl, tr.parts, tr.counter, tr.tmin, tr.tsum, tr.k);
}

// trace[k] = (min objective, sum of objectives).  Real-WT words (f3): the min
// works on the words (non-negative doubles); the sum is the binary64 sum of
// reading R33 -- each island's objectives in cell order, then the island sums
// in island order -- the oracle's order, so the trace is bit-identical (the
// integer sum is exact in any order and stays a parallel tree).
// Block reduction of (min, sum) over v[0..n) (all threads get the result).
__device__ void block_min_sum(const int64_t *v, int64_t n, int real, long long &mn, long long &sm) {
  __shared__ long long smin[32], ssum[32];
  mn = LLONG_MAX;
  long long si = 0;
  double sd = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {   // L2 loads: partials written by other blocks
    const long long a = __ldcg((const long long *)v + 2 * i), b = __ldcg((const long long *)v + 2 * i + 1);
    mn = min(mn, a);
    if (real) sd += __longlong_as_double(b);
    else si += b;
  }
  for (int d = 16; d > 0; d >>= 1) {
    mn = min(mn, __shfl_xor_sync(FULL, mn, d));
    if (real) sd += __shfl_xor_sync(FULL, sd, d);
    else si += __shfl_xor_sync(FULL, si, d);
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = mn;
    ssum[threadIdx.x >> 5] = real ? __double_as_longlong(sd) : si;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    mn = threadIdx.x < nw ? smin[threadIdx.x] : LLONG_MAX;
    long long s2 = threadIdx.x < nw ? ssum[threadIdx.x] : 0;
    double d2 = threadIdx.x < nw ? __longlong_as_double(ssum[threadIdx.x]) : 0.0;
    for (int d = 16; d > 0; d >>= 1) {
      mn = min(mn, __shfl_xor_sync(FULL, mn, d));
      if (real) d2 += __shfl_xor_sync(FULL, d2, d);
      else s2 += __shfl_xor_sync(FULL, s2, d);
    }
    if (threadIdx.x == 0) {
      if (real) {   // R33: island sums in island order
        d2 = 0.0;
        for (int64_t i = 0; i < n; ++i) d2 += __longlong_as_double(__ldcg((const long long *)v + 2 * i + 1));
      }
      smin[0] = mn;
      ssum[0] = real ? __double_as_longlong(d2) : s2;
    }
  }
  __syncthreads();
  mn = smin[0];
  sm = ssum[0];
  __syncthreads();
}

// Island partial (min, sum) of the final objectives of generation k into
// parts[li]; the last island block to finish (ticket counter) reduces the
// partials in island order into trace[k] and re-arms the counter.
__device__ void island_trace(const int64_t *obj_isl, int tile, int real, int li, int nisl, int64_t *parts,
                             unsigned *counter, int64_t *tmin, int64_t *tsum, int k) {
  __shared__ unsigned ticket;
  long long mn, sm;
  // per-island reduction over the objective words (min and sum of the same values)
  {
    __shared__ long long smin[32], ssum[32];
    mn = LLONG_MAX;
    long long si = 0;
    double sd = 0.0;
    for (int i = threadIdx.x; i < tile; i += blockDim.x) {
      const long long o = obj_isl[i];
      mn = min(mn, o);
      if (real) sd += __longlong_as_double(o);
      else si += o;
    }
    for (int d = 16; d > 0; d >>= 1) {
      mn = min(mn, __shfl_xor_sync(FULL, mn, d));
      if (real) sd += __shfl_xor_sync(FULL, sd, d);
      else si += __shfl_xor_sync(FULL, si, d);
    }
    if ((threadIdx.x & 31) == 0) {
      smin[threadIdx.x >> 5] = mn;
      ssum[threadIdx.x >> 5] = real ? __double_as_longlong(sd) : si;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int nw = blockDim.x >> 5;
      long long m0 = LLONG_MAX, s0 = 0;
      double d0 = 0.0;
      for (int w = 0; w < nw; ++w) {
        m0 = min(m0, smin[w]);
        if (!real) s0 += ssum[w];
      }
      if (real)   // R33: the island's objectives in cell order
        for (int i = 0; i < tile; ++i) d0 += __longlong_as_double(obj_isl[i]);
      parts[2 * li] = m0;
      parts[2 * li + 1] = real ? __double_as_longlong(d0) : s0;
      __threadfence();
      ticket = atomicAdd(counter, 1u);
    }
    __syncthreads();
  }
  if (ticket != (unsigned)(nisl - 1)) return;
  __threadfence();
  block_min_sum(parts, nisl, real, mn, sm);
  if (threadIdx.x == 0) {
    tmin[k] = mn;
    tsum[k] = sm;
    *counter = 0u;
  }
}

// trace of generation 0 (after the history initialisation): one block per island
__global__ void trace0_kernel(const int64_t *obj, int tile, int real, int nisl, int64_t *parts, unsigned *counter,
                              int64_t *tmin, int64_t *tsum) {
  island_trace(obj + (int64_t)blockIdx.x * tile, tile, real, blockIdx.x, nisl, parts, counter, tmin, tsum, 0);
}

// ---- one generation's breeding for one horizontal pair (a, b = a + 1)
struct GenArgs {
  int32_t K, O, cells, w, h, tile, island0, k;
  int32_t half_sh, wh_sh;                      // log2(tile/2), log2(w/2) when powers of two, else -1
  uint32_t xo_thr, mut_thr;
  uint64_t seed;
  int64_t npairs;
  int64_t row;                                 // padded genes per row (multiple of 16)
  const int32_t *cut;                          // pending cells before row-major position p
  const int8_t *xp; const int16_t *yp; const int64_t *fp;   // previous generation
  int8_t *xn; int16_t *yn;                     // next generation
};

// a6 for both cells of the pair at once: lane 16s + k, k < 5, holds
// candidate k of cell s (s = 0: (row, col), s = 1: (row, col + 1)) in the
// order self, N, S, E, W (torus inside the island, R17); a 3-step xor tree
// inside each 8-lane group keeps the largest fitness, ties -> smaller k (R18)
// (lanes k = 5..7 hold -1: every fitness is >= 0).
__device__ __forceinline__ void select_pair(int lane, const int64_t *fitI, int row, int col, int w, int h, int &wa,
                                            int &wb) {
  const int k = lane & 15, c = col + (lane >> 4);
  int nb = row * w + c;
  if (k == 1) nb = (row == 0 ? h - 1 : row - 1) * w + c;
  else if (k == 2) nb = (row + 1 == h ? 0 : row + 1) * w + c;
  else if (k == 3) nb = row * w + (c + 1 == w ? 0 : c + 1);
  else if (k == 4) nb = row * w + (c == 0 ? w - 1 : c - 1);
  long long f = k < 5 ? (long long)fitI[nb] : -1;
  int kk = k;
#pragma unroll
  for (int d = 4; d > 0; d >>= 1) {
    const long long f2 = __shfl_xor_sync(FULL, f, d);
    const int k2 = __shfl_xor_sync(FULL, kk, d);
    if (f2 > f || (f2 == f && k2 < kk)) { f = f2; kk = k2; }
  }
  const int ka = __shfl_sync(FULL, kk, 0), kb = __shfl_sync(FULL, kk, 16);
  wa = __shfl_sync(FULL, nb, ka);
  wb = __shfl_sync(FULL, nb, 16 + kb);
}

// bit masks of the genes before the cut inside one 16-B chunk (n = cut -
// first gene of the chunk): the low s bits of word k, by a clamping funnel
// shift (s >= 32: all ones)
__device__ __forceinline__ uint32_t mask_x(int n, int k) {   // word k of 16 int8 genes
  return __funnelshift_lc(0xFFFFFFFFu, 0u, (uint32_t)max(8 * (n - 4 * k), 0));
}
__device__ __forceinline__ uint32_t mask_y(int n, int k) {   // word k of 8 int16 genes
  return __funnelshift_lc(0xFFFFFFFFu, 0u, (uint32_t)max(16 * (n - 2 * k), 0));
}
__device__ __forceinline__ uint32_t wsel(uint4 v, int k) { return k == 0 ? v.x : k == 1 ? v.y : k == 2 ? v.z : v.w; }
__device__ __forceinline__ void wset(uint4 &v, int k, uint32_t w) {
  if (k == 0) v.x = w; else if (k == 1) v.y = w; else if (k == 2) v.z = w; else v.w = w;
}

// a8 on 16 machines: x <- (x + 1 + floor(r (o-1) / 2^32)) mod o, one Philox
// block per 4 genes (R15)
__device__ __forceinline__ uint4 mutate16(uint4 v, int g0, uint32_t cell, uint32_t kg, uint32_t I, uint32_t k0,
                                          uint32_t k1, int O, int o1) {
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const u32x4 r = philox((RNG_MUT_X << 24) | (uint32_t)((g0 >> 2) + b), cell, kg, I, k0, k1);
    uint32_t w = wsel(v, b), out = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int xv = (int)((w >> (8 * j)) & 0xFFu) + 1 + (int)bounded(word_of(r, j), (uint32_t)o1);
      if (xv >= O) xv -= O;
      out |= (uint32_t)xv << (8 * j);
    }
    wset(v, b, out);
  }
  return v;
}

// 32 byte-map entries (0 or 1, 16-B aligned) -> one word, entry b at bit b:
// (w * 0x01020408) >> 24 gathers the four bytes' low bits of w in order (no
// carries: the partial products land on distinct bits)
__device__ __forceinline__ uint32_t pack32(const uint8_t *m) {
  const uint4 lo = ((const uint4 *)m)[0], hi = ((const uint4 *)m)[1];
  const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) r |= ((w[k] * 0x01020408u) >> 24) << (4 * k);
  return r;
}

__global__ void __launch_bounds__(256, 4) generation_kernel(GenArgs a) {
  extern __shared__ __align__(16) unsigned char gsm[];
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.K, nwd = (K + 32) >> 5;   // 32-value words of the maps (values 0..K)
  const int fmb = nwd * 32;                 // byte maps indexed by value 0..K (slot 0: padding genes)
  const size_t per_warp = (size_t)2 * ((K * 2 + 15) & ~15) + (size_t)2 * fmb;
  uint16_t *LA = (uint16_t *)(gsm + warp * per_warp);
  uint16_t *LB = LA + ((K * 2 + 15) & ~15) / 2;
  uint8_t *FA = (uint8_t *)(LB + ((K * 2 + 15) & ~15) / 2);   // FA[v] = 1 iff v is in A's prefix
  uint8_t *FB = FA + fmb;
  const uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint32_t half = (uint32_t)a.tile >> 1, wh = (uint32_t)a.w >> 1;
  const int64_t row = a.row;
  const int nxv = (int)(row >> 4), nyv = (int)(row >> 3);   // 16-B words of a row
  const uint32_t npairs = (uint32_t)a.npairs;               // < 2^30 (count < 2^31)
  for (uint32_t pi = blockIdx.x * (blockDim.x >> 5) + warp; pi < npairs; pi += nw) {
    const uint32_t li = a.half_sh >= 0 ? pi >> a.half_sh : pi / half, pr = pi - li * half;
    const uint32_t prow = a.wh_sh >= 0 ? pr >> a.wh_sh : pr / wh;
    const int pcol = 2 * (int)(pr - prow * wh);
    const int ca = (int)prow * a.w + pcol, cb = ca + 1;
    const uint32_t I = (uint32_t)a.island0 + li, kg = (uint32_t)a.k;
    const int64_t base = (int64_t)li * a.tile;
    // a6: asteroid selection on the previous generation's fitness
    int wa, wb;
    select_pair(lane, a.fp + base, (int)prow, pcol, a.w, a.h, wa, wb);
    const uint4 *XA = (const uint4 *)(a.xp + (base + wa) * row), *XB = (const uint4 *)(a.xp + (base + wb) * row);
    const uint4 *YA = (const uint4 *)(a.yp + (base + wa) * row), *YB = (const uint4 *)(a.yp + (base + wb) * row);
    uint4 *xa = (uint4 *)(a.xn + (base + ca) * row), *xb = (uint4 *)(a.xn + (base + cb) * row);
    uint4 *ya = (uint4 *)(a.yn + (base + ca) * row), *yb = (uint4 *)(a.yn + (base + cb) * row);
    // the parents' rows into L2 now (HBM latency under the RNG and repair maps)
    {
      const int nxl = (int)((row + 127) >> 7), nyl = (int)((2 * row + 127) >> 7);
      for (int l = lane; l < 2 * (nxl + nyl); l += 32) {
        const int p = l >= nxl + nyl, q = l - p * (nxl + nyl);
        const char *src = q < nxl ? (const char *)(p ? XB : XA) + 128 * q : (const char *)(p ? YB : YA) + 128 * (q - nxl);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
      }
    }
    // the pair's three Philox blocks, one per lane 0..2, then broadcast:
    // lane 0 = crossover (a7), lanes 1, 2 = mutation of children a, b (a8)
    const u32x4 rl = philox(lane == 0 ? (RNG_XO << 24) : (RNG_MUT << 24), (uint32_t)(lane == 2 ? cb : ca), kg, I,
                            k0, k1);
    const uint32_t xo0 = __shfl_sync(FULL, rl.x, 0), xo1 = __shfl_sync(FULL, rl.y, 0);
    u32x4 rma, rmb;
    rma.x = __shfl_sync(FULL, rl.x, 1); rma.y = __shfl_sync(FULL, rl.y, 1); rma.z = __shfl_sync(FULL, rl.z, 1);
    rmb.x = __shfl_sync(FULL, rl.x, 2); rmb.y = __shfl_sync(FULL, rl.y, 2); rmb.z = __shfl_sync(FULL, rl.z, 2);
    rma.w = rmb.w = 0u;
    // a7: crossover fires with p_c; one row-major cut shared by X and Y (R13)
    int kc = K;
    if (xo0 < a.xo_thr) {
      int p = 1 + (int)bounded(xo1, (uint32_t)(a.cells - 1));
      kc = a.cut[p];
    }
    const bool ma = rma.x < a.mut_thr, mb = rmb.x < a.mut_thr;
    const bool repair = kc > 0 && kc < K;
    // the membership maps cover the shorter side of the cut: the parents'
    // prefix values (inv = false) or, when the suffix is shorter, their suffix
    // values (inv = true: "in the prefix" = "not in the suffix" for a value
    // in [1, K])
    const bool inv = 2 * kc > K;
    if (repair) {
      // correction (R14): duplicates of child a are the suffix genes of B
      // whose value occurs in A's prefix; missing values = in B's prefix, not
      // in A's prefix; assigned in ascending order to duplicates in gene order.
      for (int i = lane; i < (fmb >> 4); i += 32) {
        ((uint4 *)FA)[i] = make_uint4(0, 0, 0, 0);
        ((uint4 *)FB)[i] = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
      const int g_lo = inv ? kc : 0, g_hi = inv ? K : kc;
      for (int i = (g_lo >> 3) + lane; i < ((g_hi + 7) >> 3); i += 32) {
        const uint4 va = YA[i], vb = YB[i];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int g = 8 * i + j;
          if (g >= g_lo && g < g_hi) {   // values in [1, K]
            const int sh = 16 * (j & 1);
            const int va1 = (int)((wsel(va, j >> 1) >> sh) & 0xFFFFu), vb1 = (int)((wsel(vb, j >> 1) >> sh) & 0xFFFFu);
            FA[va1] = 1;
            FB[vb1] = 1;
          }
        }
      }
      __syncwarp();
      int offa = 0, offb = 0;
      for (int i0 = 0; i0 < nwd; i0 += 32) {
        int i = i0 + lane;
        // the maps' value bits (bit b of word i: value 32 i + b), packed in registers
        const uint32_t pa_ = i < nwd ? pack32(FA + 32 * i) : 0u, pb_ = i < nwd ? pack32(FB + 32 * i) : 0u;
        // missing of child a: in B's prefix and not in A's (= in A's suffix and not in B's)
        uint32_t wa_ = inv ? pa_ & ~pb_ : pb_ & ~pa_;
        uint32_t wb_ = inv ? pb_ & ~pa_ : pa_ & ~pb_;
        int na = __popc(wa_), nb = __popc(wb_);
        int ia = na | (nb << 16);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          int t1 = __shfl_up_sync(FULL, ia, d);
          if (lane >= d) ia += t1;
        }
        int pa = offa + (ia & 0xFFFF) - na, pb = offb + (ia >> 16) - nb;
        while (wa_) { int bit = __ffs(wa_) - 1; wa_ &= wa_ - 1; LA[pa++] = (uint16_t)(i * 32 + bit); }
        while (wb_) { int bit = __ffs(wb_) - 1; wb_ &= wb_ - 1; LB[pb++] = (uint16_t)(i * 32 + bit); }
        const int tot = __shfl_sync(FULL, ia, 31);
        offa += tot & 0xFFFF;
        offb += tot >> 16;
      }
      __syncwarp();
    }
    // children X, 16 genes per lane-word: prefix from own parent, suffix from
    // the other; a8 resamples every machine of a mutated child
    const int o1 = a.O - 1;
    for (int i = lane; i < nxv; i += 32) {
      const uint4 va = XA[i], vb = XB[i];
      uint4 za, zb;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t m = mask_x(kc - 16 * i, k), wa_ = wsel(va, k), wb_ = wsel(vb, k);
        wset(za, k, (wa_ & m) | (wb_ & ~m));
        wset(zb, k, (wb_ & m) | (wa_ & ~m));
      }
      if (ma && o1 >= 1) za = mutate16(za, 16 * i, (uint32_t)ca, kg, I, k0, k1, a.O, o1);
      if (mb && o1 >= 1) zb = mutate16(zb, 16 * i, (uint32_t)cb, kg, I, k0, k1, a.O, o1);
      xa[i] = za;
      xb[i] = zb;
    }
    // children Y, 8 genes per lane-word; suffix duplicates take the missing
    // values in gene order (lane order inside a step, steps ascending)
    int da = 0, db = 0;
    for (int i0 = 0; i0 < nyv; i0 += 32) {
      const int i = i0 + lane;
      uint4 va = make_uint4(0, 0, 0, 0), vb = va;
      if (i < nyv) { va = YA[i]; vb = YB[i]; }
      uint4 za, zb;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t m = mask_y(kc - 8 * i, k), wa_ = wsel(va, k), wb_ = wsel(vb, k);
        wset(za, k, (wa_ & m) | (wb_ & ~m));
        wset(zb, k, (wb_ & m) | (wa_ & ~m));
      }
      if (repair && 8 * (i0 + 32) > kc) {   // warp-uniform: some lane's word reaches the suffix
        // duplicates: suffix genes (kc <= g < K) whose value is in the own
        // parent's prefix -- one byte-map load per gene, no bit arithmetic
        // (padding genes hold value 0, slot 0 of the maps)
        const int lo = min(max(kc - 8 * i, 0), 8), hi = min(max(K - 8 * i, 0), 8);
        const uint32_t sfx = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
        uint32_t fa = 0, fb = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int sh = 16 * (j & 1);
          const uint32_t ta = (wsel(za, j >> 1) >> sh) & 0xFFFFu, tb = (wsel(zb, j >> 1) >> sh) & 0xFFFFu;
          fa += (uint32_t)FA[ta] << j;
          fb += (uint32_t)FB[tb] << j;
        }
        if (inv) {   // the maps hold the suffix values: "not in it" = "in the prefix"
          fa = ~fa;
          fb = ~fb;
        }
        fa &= sfx;
        fb &= sfx;
        const int na = __popc(fa), nb = __popc(fb);
        int ia = na | (nb << 16);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int t1 = __shfl_up_sync(FULL, ia, d);
          if (lane >= d) ia += t1;
        }
        int ra = da + (ia & 0xFFFF) - na, rb = db + (ia >> 16) - nb;
        const int tot = __shfl_sync(FULL, ia, 31);
        da += tot & 0xFFFF;
        db += tot >> 16;
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // half j&1 of word j/2 <- next missing value (byte permute)
          const uint32_t sel = (j & 1) ? 0x5410u : 0x3254u;
          if ((fa >> j) & 1u) wset(za, j >> 1, __byte_perm(wsel(za, j >> 1), (uint32_t)LA[ra++], sel));
          if ((fb >> j) & 1u) wset(zb, j >> 1, __byte_perm(wsel(zb, j >> 1), (uint32_t)LB[rb++], sel));
        }
      }
      if (i < nyv) {
        ya[i] = za;
        yb[i] = zb;
      }
    }
    __syncwarp();
    // a8: swap two priorities
    if (K >= 2 && lane < 2) {
      const uint32_t r1 = lane == 0 ? rma.y : rmb.y, r2 = lane == 0 ? rma.z : rmb.z;
      const bool fire = lane == 0 ? ma : mb;
      int16_t *yy = (int16_t *)(lane == 0 ? ya : yb);
      if (fire) {
        int g1 = (int)bounded(r1, (uint32_t)K);
        int g2 = (int)bounded(r2, (uint32_t)(K - 1));
        g2 += g2 >= g1;
        int16_t t = yy[g1];
        yy[g1] = yy[g2];
        yy[g2] = t;
      }
    }
    __syncwarp();
  }
}

size_t gen_smem_per_warp(int K) {
  const int nwd = (K + 32) >> 5;
  return (size_t)2 * ((K * 2 + 15) & ~15) + (size_t)2 * nwd * 32;
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static ffs_status evaluate_population(Run &r, int buf, bool with_fitness) {
  EvalArgs a{};
  a.image = r.st->image_dev;
  a.count = r.nloc;
  a.x = r.x[buf];
  a.y = r.y[buf];
  a.obj = r.obj[buf];
  a.row = r.row;
  a.fstart = r.st->fstart_dev;
  if (with_fitness) {
    a.emax = r.scal;
    a.fit = r.fit[buf];
  }
  r.evaluations += r.nloc;
  return launch_evaluate(*r.st, a, r.scr, r.s, &r.launches);
}

static ffs_status ga_init(Run &r) {
  const State &st = *r.st;
  int NP = 64;
  while (NP < r.K) NP <<= 1;
  const int warps = (int)std::min<size_t>(8, (size_t)kSmemLimit / ((size_t)NP * 8));
  if (warps < 1) return fail(FFS_ERR_INVALID_ARG, "K too large for initialisation");
  size_t smem = (size_t)warps * NP * 8;
  FFS_CUDA(cudaFuncSetAttribute(init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t grid = std::min<int64_t>((r.nloc + warps - 1) / warps, (int64_t)st.num_sms * 8);
  init_kernel<<<(unsigned)grid, warps * 32, smem, r.s>>>(r.K, NP, r.row, st.inst->o, r.nloc, r.tile,
                                                         r.cfg.island_begin, r.cfg.seed, r.x[0], r.y[0]);
  FFS_CUDA(cudaGetLastError());
  r.launches++;
  ffs_status e = evaluate_population(r, 0, false);
  if (e != FFS_OK) return e;
  max_kernel<<<1, 1024, 0, r.s>>>(r.obj[0], r.nloc, r.scal + 1);
  FFS_CUDA(cudaGetLastError());
  r.launches++;
  if (r.cfg.allreduce_max_i64 && r.cfg.world > 1) {
    // E_max over the global initial population (R23)
    if (r.cfg.allreduce_max_i64(r.cfg.user, r.scal + 1, (void *)r.s) != 0)
      return fail(FFS_ERR_COMM, "allreduce_max_i64 hook failed");
  }
  emax_fitness_kernel<<<(unsigned)std::min<int64_t>((r.nloc + 255) / 256, 1024), 256, 0, r.s>>>(
      r.scal, r.obj[0], r.fit[0], r.nloc, st.real_wt);
  FFS_CUDA(cudaGetLastError());
  history_init_kernel<<<r.nisl, 256, 0, r.s>>>(r.row, r.tile, r.x[0], r.y[0], r.obj[0], r.fit[0], r.hx, r.hy,
                                               r.hobj, r.hfit);
  FFS_CUDA(cudaGetLastError());
  trace0_kernel<<<r.nisl, 256, 0, r.s>>>(r.obj[0], r.tile, st.real_wt, r.nisl, r.parts, r.tcounter, r.tmin, r.tsum);
  FFS_CUDA(cudaGetLastError());
  r.launches += 3;
  r.cur = 0;
  r.gen = 0;
  return FFS_OK;
}

static ffs_status ga_generation(Run &r) {
  const State &st = *r.st;
  const int k = r.gen + 1;
  const int nb = 1 - r.cur;
  GenArgs g{};
  g.K = r.K; g.O = st.inst->o; g.cells = st.cells; g.w = r.cfg.island_w; g.h = r.cfg.island_h;
  g.tile = r.tile; g.island0 = r.cfg.island_begin; g.k = k;
  auto log2_or = [](int v) { return (v > 0 && (v & (v - 1)) == 0) ? __builtin_ctz((unsigned)v) : -1; };
  g.half_sh = log2_or(r.tile / 2);
  g.wh_sh = log2_or(r.cfg.island_w / 2);
  g.xo_thr = r.cfg.xo_threshold; g.mut_thr = r.cfg.mut_threshold; g.seed = r.cfg.seed;
  g.npairs = r.nloc / 2;
  g.cut = st.cut_dev;
  g.row = r.row;
  g.xp = r.x[r.cur]; g.yp = r.y[r.cur]; g.fp = r.fit[r.cur];
  g.xn = r.x[nb]; g.yn = r.y[nb];
  const int warps = 8;
  size_t smem = (size_t)warps * gen_smem_per_warp(r.K);
  if (smem > 48 * 1024) {
    ffs_status ea = ensure_smem_attr((const void *)generation_kernel, smem);
    if (ea != FFS_OK) return ea;
  }
  // 4 waves of 4 CTAs per SM: finer balancing of the pairs' uneven costs
  // than 2 waves (0.509 -> 0.505 ms per GA step), less launch work than 7
  int64_t grid = std::min<int64_t>((g.npairs + warps - 1) / warps, (int64_t)st.num_sms * 16);
  FFS_CUDA(launch_pdl(generation_kernel, dim3((unsigned)grid), dim3(warps * 32), smem, r.s, g));
  r.launches++;
  ffs_status e = evaluate_population(r, nb, true);
  if (e != FFS_OK) return e;
  const bool migrate = k % r.cfg.migration_interval == 0 && r.cfg.islands_total >= 2;
  TraceArgs tr{r.parts, r.tcounter, r.tmin, r.tsum, k, st.real_wt, r.nisl, migrate ? 0 : 1};
  FFS_CUDA(launch_pdl(replace_kernel, dim3(r.nisl), dim3(256), 0, r.s, r.row, r.tile, r.x[nb], r.y[nb], r.obj[nb],
                      r.fit[nb], r.hx, r.hy, r.hobj, r.hfit, tr));
  r.launches++;
  if (migrate) {
    FFS_CUDA(launch_pdl(donor_kernel, dim3(r.nisl), dim3(256), 0, r.s, r.K, r.row, r.tile, r.rec, r.x[nb], r.y[nb],
                        r.obj[nb], r.fit[nb], r.donor, r.worst_idx));
    r.launches++;
    const unsigned char *incoming = r.donor + (size_t)(r.nisl - 1) * r.rec;
    if (r.cfg.world > 1) {
      if (!r.cfg.allgather) return fail(FFS_ERR_INVALID_ARG, "world > 1 needs the allgather hook");
      if (r.cfg.allgather(r.cfg.user, r.donor + (size_t)(r.nisl - 1) * r.rec, r.recv, r.rec, (void *)r.s) != 0)
        return fail(FFS_ERR_COMM, "allgather hook failed");
      incoming = r.recv + (size_t)((r.cfg.rank + r.cfg.world - 1) % r.cfg.world) * r.rec;
    }
    if (r.cfg.world > 1) {
      // after the allgather hook (another library's stream work): plain
      // stream order, no programmatic overlap with anything before it
      import_kernel<<<r.nisl, 256, 0, r.s>>>(r.K, r.row, r.tile, r.rec, r.donor, incoming, r.worst_idx, r.x[nb],
                                             r.y[nb], r.obj[nb], r.fit[nb], tr);
      FFS_CUDA(cudaGetLastError());
    } else {
      FFS_CUDA(launch_pdl(import_kernel, dim3(r.nisl), dim3(256), 0, r.s, r.K, r.row, r.tile, r.rec,
                          (const unsigned char *)r.donor, incoming, (const int32_t *)r.worst_idx, r.x[nb], r.y[nb],
                          r.obj[nb], r.fit[nb], tr));
    }
    r.launches++;
  }
  r.cur = nb;
  r.gen = k;
  return FFS_OK;
}

}  // namespace edffs

struct ffs_run { edffs::Run v; };

using namespace edffs;

extern "C" {

ffs_status ffs_evolve_begin(ffs_state *sh, const ffs_ga_config *cfg, void *stream, ffs_run **out) {
  if (!sh || !cfg || !out) return fail(FFS_ERR_INVALID_ARG, "null argument");
  if (cfg->island_w < 2 || (cfg->island_w & 1) || cfg->island_h < 1)
    return fail(FFS_ERR_INVALID_ARG, "island_w must be even and >= 2, island_h >= 1");
  if ((int64_t)cfg->island_w * cfg->island_h > (1 << 20)) return fail(FFS_ERR_INVALID_ARG, "island tile > 2^20 cells");
  if (cfg->islands_total < 1 || cfg->island_begin < 0 || cfg->island_end > cfg->islands_total ||
      cfg->island_begin >= cfg->island_end)
    return fail(FFS_ERR_INVALID_ARG, "bad island shard");
  if (cfg->generations < 0 || cfg->migration_interval < 1) return fail(FFS_ERR_INVALID_ARG, "bad generations");
  if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return fail(FFS_ERR_INVALID_ARG, "bad rank/world");
  if (cfg->world > 1 && (!cfg->allgather || !cfg->allreduce_max_i64))
    return fail(FFS_ERR_INVALID_ARG, "world > 1 needs both collective hooks (allreduce_max_i64, allgather)");
  State &st = sh->v;
  cudaSetDevice(st.inst->dev);
  {
    // load every kernel a generation may launch now (CUDA's lazy loading
    // would otherwise load the migration kernels inside the 10th generation)
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, generation_kernel);
    cudaFuncGetAttributes(&fa, replace_kernel);
    cudaFuncGetAttributes(&fa, donor_kernel);
    cudaFuncGetAttributes(&fa, import_kernel);
    cudaFuncGetAttributes(&fa, trace0_kernel);
  }
  ffs_run *h = new ffs_run();
  Run &r = h->v;
  r.st = &st;
  r.cfg = *cfg;
  r.s = (cudaStream_t)stream;
  pool_keep(st.inst->dev);
  r.scr.pool = r.s;
  r.scr.pooled = true;
  r.tile = cfg->island_w * cfg->island_h;
  r.nisl = cfg->island_end - cfg->island_begin;
  r.nloc = (int64_t)r.nisl * r.tile;
  r.K = st.K;
  r.cells = st.cells;
  r.rec = ((size_t)3 * r.K + 16 + 15) & ~(size_t)15;
  r.row = ((int64_t)std::max(r.K, 1) + 15) & ~(int64_t)15;
  const size_t genes = (size_t)r.nloc * r.row;
  ffs_status e = FFS_OK;
  for (int b = 0; b < 2 && e == FFS_OK; ++b) {
    if (e == FFS_OK) e = r.alloc(&r.x[b], genes);
    if (e == FFS_OK) e = r.alloc(&r.y[b], genes);
    if (e == FFS_OK) e = r.alloc(&r.obj[b], (size_t)r.nloc);
    if (e == FFS_OK) e = r.alloc(&r.fit[b], (size_t)r.nloc);
  }
  if (e == FFS_OK) e = r.alloc(&r.hx, (size_t)r.nisl * r.row);
  if (e == FFS_OK) e = r.alloc(&r.hy, (size_t)r.nisl * r.row);
  // padding genes are never read as genes; zero them once for determinism
  for (int b = 0; b < 2 && e == FFS_OK; ++b) {
    cudaError_t ce = cudaMemsetAsync(r.x[b], 0, genes, r.s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(r.y[b], 0, genes * 2, r.s);
    if (ce != cudaSuccess) e = cuda_fail(ce, "population memset");
  }
  if (e == FFS_OK) e = r.alloc(&r.hobj, (size_t)r.nisl);
  if (e == FFS_OK) e = r.alloc(&r.hfit, (size_t)r.nisl);
  if (e == FFS_OK) e = r.alloc(&r.worst_idx, (size_t)r.nisl);
  if (e == FFS_OK) e = r.alloc(&r.donor, (size_t)r.nisl * r.rec);
  if (e == FFS_OK) e = r.alloc(&r.recv, (size_t)cfg->world * r.rec);
  if (e == FFS_OK) e = r.alloc(&r.scal, 2);
  if (e == FFS_OK) e = r.alloc(&r.tmin, (size_t)cfg->generations + 1);
  if (e == FFS_OK) e = r.alloc(&r.tsum, (size_t)cfg->generations + 1);
  if (e == FFS_OK) e = r.alloc(&r.parts, (size_t)2 * r.nisl);
  if (e == FFS_OK) e = r.alloc(&r.tcounter, 1);
  if (e == FFS_OK) e = r.alloc(&r.best_v, 2);
  if (e == FFS_OK) e = r.alloc(&r.best_s, (size_t)st.cells + 1);
  if (e == FFS_OK) {
    cudaError_t ce = cudaMemsetAsync(r.tcounter, 0, sizeof(unsigned), r.s);
    if (ce != cudaSuccess) e = cuda_fail(ce, "trace counter");
  }
  if (e == FFS_OK && r.K > 0) e = ga_init(r);
  if (e != FFS_OK) {
    delete h;
    return e;
  }
  *out = h;
  return FFS_OK;
}

ffs_status ffs_evolve_step(ffs_run *h, int32_t generations) {
  if (!h || generations < 0) return fail(FFS_ERR_INVALID_ARG, "bad arguments");
  Run &r = h->v;
  if (r.K == 0) return FFS_OK;
  if (r.gen + generations > r.cfg.generations)
    return fail(FFS_ERR_INVALID_ARG, "more generations than configured");
  cudaSetDevice(r.st->inst->dev);
  for (int i = 0; i < generations; ++i) {
    ffs_status e = ga_generation(r);
    if (e != FFS_OK) return e;
  }
  return FFS_OK;
}

ffs_status ffs_evolve(ffs_state *sh, const ffs_ga_config *cfg, void *stream, ffs_run **out) {
  ffs_run *h = nullptr;
  ffs_status e = ffs_evolve_begin(sh, cfg, stream, &h);
  if (e != FFS_OK) return e;
  e = ffs_evolve_step(h, cfg->generations);
  if (e == FFS_OK) {
    cudaError_t ce = cudaStreamSynchronize((cudaStream_t)stream);
    if (ce != cudaSuccess) e = cuda_fail(ce, "ffs_evolve sync");
  }
  if (e != FFS_OK) {
    ffs_run_destroy(h);
    return e;
  }
  *out = h;
  return FFS_OK;
}

ffs_status ffs_best(ffs_run *h, int8_t *x, int16_t *y, int32_t *assign, int32_t *start, int64_t *objective,
                    int64_t *total_tardiness, int32_t *makespan, int64_t *trace_min, int64_t *trace_sum) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null run");
  Run &r = h->v;
  State &st = *r.st;
  cudaSetDevice(st.inst->dev);
  FFS_CUDA(cudaStreamSynchronize(r.s));
  const int K = r.K;
  std::vector<int8_t> bx(std::max(K, 1), 0);
  std::vector<int16_t> by(std::max(K, 1), 1);
  int b = 0;
  if (K > 0) {
    std::vector<int64_t> hf(r.nisl);
    FFS_CUDA(cudaMemcpyAsync(hf.data(), r.hfit, (size_t)r.nisl * 8, cudaMemcpyDeviceToHost, r.s));
    FFS_CUDA(cudaStreamSynchronize(r.s));
    for (int i = 1; i < r.nisl; ++i)
      if (hf[i] > hf[b]) b = i;  // ties -> lowest island (R28)
  }
  // decode the elite once more, in place in the history row, to emit its
  // schedule (run-owned output buffers, everything ordered on the run's stream)
  EvalArgs a{};
  a.image = st.image_dev;
  a.count = 1;
  a.x = r.hx + (size_t)b * r.row;
  a.y = r.hy + (size_t)b * r.row;
  a.row = K > 0 ? r.row : 0;
  a.obj = r.best_v;
  a.tard = r.best_v + 1;
  a.cmax = r.best_s + st.cells;
  a.start_out = r.best_s;
  a.fstart = st.fstart_dev;
  ffs_status e = launch_evaluate(st, a, r.scr, r.s, nullptr);
  if (e != FFS_OK) return e;
  std::vector<int32_t> hs(st.cells + 1);
  int64_t hv[2] = {0, 0};
  FFS_CUDA(cudaMemcpyAsync(hs.data(), r.best_s, (size_t)(st.cells + 1) * 4, cudaMemcpyDeviceToHost, r.s));
  FFS_CUDA(cudaMemcpyAsync(hv, r.best_v, 16, cudaMemcpyDeviceToHost, r.s));
  if (K > 0) {
    FFS_CUDA(cudaMemcpyAsync(bx.data(), a.x, (size_t)K, cudaMemcpyDeviceToHost, r.s));
    FFS_CUDA(cudaMemcpyAsync(by.data(), a.y, (size_t)K * 2, cudaMemcpyDeviceToHost, r.s));
  }
  FFS_CUDA(cudaStreamSynchronize(r.s));
  if (x && K) std::memcpy(x, bx.data(), (size_t)K);
  if (y && K) std::memcpy(y, by.data(), (size_t)K * 2);
  if (start) std::memcpy(start, hs.data(), (size_t)st.cells * 4);
  if (assign) {
    for (int c = 0; c < st.cells; ++c) assign[c] = st.fassign[c];
    for (int k = 0; k < K; ++k) assign[st.gene_cell[k]] = bx[k];
  }
  if (objective) *objective = hv[0];
  if (total_tardiness) *total_tardiness = hv[1];
  if (makespan) *makespan = hs[st.cells];
  if (K > 0 && r.gen >= 0) {
    if (trace_min)
      FFS_CUDA(cudaMemcpyAsync(trace_min, r.tmin, (size_t)(r.gen + 1) * 8, cudaMemcpyDeviceToHost, r.s));
    if (trace_sum)
      FFS_CUDA(cudaMemcpyAsync(trace_sum, r.tsum, (size_t)(r.gen + 1) * 8, cudaMemcpyDeviceToHost, r.s));
    FFS_CUDA(cudaStreamSynchronize(r.s));
  }
  return FFS_OK;
}

ffs_status ffs_run_population(ffs_run *h, int8_t *x, int16_t *y, int64_t *objective, int64_t *fitness) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null run");
  Run &r = h->v;
  cudaSetDevice(r.st->inst->dev);
  FFS_CUDA(cudaStreamSynchronize(r.s));
  if (r.K == 0) return FFS_OK;
  if (x) FFS_CUDA(cudaMemcpy2D(x, (size_t)r.K, r.x[r.cur], (size_t)r.row, (size_t)r.K, (size_t)r.nloc,
                               cudaMemcpyDeviceToHost));
  if (y) FFS_CUDA(cudaMemcpy2D(y, (size_t)r.K * 2, r.y[r.cur], (size_t)r.row * 2, (size_t)r.K * 2, (size_t)r.nloc,
                               cudaMemcpyDeviceToHost));
  if (objective) FFS_CUDA(cudaMemcpy(objective, r.obj[r.cur], (size_t)r.nloc * 8, cudaMemcpyDeviceToHost));
  if (fitness) FFS_CUDA(cudaMemcpy(fitness, r.fit[r.cur], (size_t)r.nloc * 8, cudaMemcpyDeviceToHost));
  return FFS_OK;
}

ffs_status ffs_run_history(ffs_run *h, int8_t *x, int16_t *y, int64_t *objective, int64_t *fitness) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null run");
  Run &r = h->v;
  cudaSetDevice(r.st->inst->dev);
  FFS_CUDA(cudaStreamSynchronize(r.s));
  if (r.K == 0) return FFS_OK;
  if (x) FFS_CUDA(cudaMemcpy2D(x, (size_t)r.K, r.hx, (size_t)r.row, (size_t)r.K, (size_t)r.nisl,
                               cudaMemcpyDeviceToHost));
  if (y) FFS_CUDA(cudaMemcpy2D(y, (size_t)r.K * 2, r.hy, (size_t)r.row * 2, (size_t)r.K * 2, (size_t)r.nisl,
                               cudaMemcpyDeviceToHost));
  if (objective) FFS_CUDA(cudaMemcpy(objective, r.hobj, (size_t)r.nisl * 8, cudaMemcpyDeviceToHost));
  if (fitness) FFS_CUDA(cudaMemcpy(fitness, r.hfit, (size_t)r.nisl * 8, cudaMemcpyDeviceToHost));
  return FFS_OK;
}

ffs_status ffs_run_info(const ffs_run *h, int32_t *generation, int64_t *emax, int64_t *evaluations,
                        int32_t *kernel_launches) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null run");
  const Run &r = h->v;
  if (generation) *generation = r.gen;
  if (emax) {
    *emax = 0;
    if (r.K > 0) {
      cudaStreamSynchronize(r.s);
      FFS_CUDA(cudaMemcpy(emax, r.scal, 8, cudaMemcpyDeviceToHost));
    }
  }
  if (evaluations) *evaluations = r.evaluations;
  if (kernel_launches) *kernel_launches = r.launches;
  return FFS_OK;
}

ffs_status ffs_run_restore(ffs_run *h, int32_t generation, const int8_t *x, const int16_t *y,
                           const int64_t *objective, const int64_t *fitness, const int8_t *hx, const int16_t *hy,
                           const int64_t *hobj, const int64_t *hfit, int64_t emax, const int64_t *trace_min,
                           const int64_t *trace_sum) {
  if (!h) return fail(FFS_ERR_INVALID_ARG, "null run");
  Run &r = h->v;
  if (r.K == 0) {   // nothing evolves: the run has no generations to restore
    if (generation != r.gen) return fail(FFS_ERR_INVALID_ARG, "K = 0: the checkpoint generation must be the run's");
    return FFS_OK;
  }
  if (generation < 0 || generation > r.cfg.generations)
    return fail(FFS_ERR_INVALID_ARG, "checkpoint generation outside [0, generations]");
  if (!x || !y || !objective || !fitness || !hx || !hy || !hobj || !hfit || !trace_min || !trace_sum)
    return fail(FFS_ERR_INVALID_ARG, "null checkpoint array");
  cudaSetDevice(r.st->inst->dev);
  FFS_CUDA(cudaStreamSynchronize(r.s));
  const size_t K = (size_t)r.K;
  // rows padded to r.row genes: only the K genes are restored (the padding
  // stays the zeros written at creation)
  FFS_CUDA(cudaMemcpy2DAsync(r.x[r.cur], (size_t)r.row, x, K, K, (size_t)r.nloc, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpy2DAsync(r.y[r.cur], (size_t)r.row * 2, y, K * 2, K * 2, (size_t)r.nloc, cudaMemcpyHostToDevice,
                             r.s));
  FFS_CUDA(cudaMemcpyAsync(r.obj[r.cur], objective, (size_t)r.nloc * 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpyAsync(r.fit[r.cur], fitness, (size_t)r.nloc * 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpy2DAsync(r.hx, (size_t)r.row, hx, K, K, (size_t)r.nisl, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpy2DAsync(r.hy, (size_t)r.row * 2, hy, K * 2, K * 2, (size_t)r.nisl, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpyAsync(r.hobj, hobj, (size_t)r.nisl * 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpyAsync(r.hfit, hfit, (size_t)r.nisl * 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpyAsync(r.scal, &emax, 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpyAsync(r.tmin, trace_min, (size_t)(generation + 1) * 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaMemcpyAsync(r.tsum, trace_sum, (size_t)(generation + 1) * 8, cudaMemcpyHostToDevice, r.s));
  FFS_CUDA(cudaStreamSynchronize(r.s));   // the host arrays may go away after the call
  r.gen = generation;
  r.evaluations = (int64_t)(generation + 1) * r.nloc;
  return FFS_OK;
}

void ffs_run_destroy(ffs_run *h) {
  if (!h) return;
  cudaSetDevice(h->v.st->inst->dev);
  cudaStreamSynchronize(h->v.s);
  delete h;
}

}  // extern "C"
