// GPU brute-force enumerator ("enumeration
// count = o^K * K!/prod L_j!").  Ground truth for small K: every machine
// vector X in [0, o-1]^K times every linear extension of the job chains (the
// orders Algorithm 1 can produce), each decoded by the same
// Algorithm 2 kernels as the GA (ffs_evaluate's launch path).
//
// Enumeration index i = order_rank * o^K + x_rank.  x_rank is read as K base-o
// digits (gene g = digit g); order_rank is unranked into a linear extension by
// the multinomial number system (jobs in ascending index at every position).
// The order is turned into a priority vector y = K - position, whose greedy
// order (prefix-min of y along each job chain = y itself, since y falls along
// the chain) is exactly that linear extension.  The best objective word and the
// lowest index reaching it are kept on the device across chunks.
#include <climits>

#include "ffs_common.cuh"
#include "device_util.cuh"

namespace edffs {
namespace {

constexpr int kMaxBruteJobs = 64;
constexpr int kMaxBruteK = 64;

struct BruteArgs {
  int32_t K, O, nj;
  int32_t jfirst[kMaxBruteJobs];   // first gene of each job with pending genes
  int32_t jlen[kMaxBruteJobs];     // its number of pending genes (chain length L_j)
  uint64_t n_x;                    // o^K
  uint64_t n_orders;               // K! / prod L_j!
};

__global__ void __launch_bounds__(256) enumerate_kernel(BruteArgs b, uint64_t first, int64_t count, int8_t *x,
                                                        int16_t *y) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = first + (uint64_t)t;
    uint64_t xr = idx % b.n_x;
    uint64_t r = idx / b.n_x;
    int8_t *xo = x + t * b.K;
    int16_t *yo = y + t * b.K;
    for (int g = 0; g < b.K; ++g) {
      xo[g] = (int8_t)(xr % (uint64_t)b.O);
      xr /= (uint64_t)b.O;
    }
    int rem[kMaxBruteJobs];
    for (int j = 0; j < b.nj; ++j) rem[j] = b.jlen[j];
    uint64_t N = b.n_orders;   // linear extensions of the remaining chains
    int left = b.K;
    for (int p = 0; p < b.K; ++p) {
      int pick = -1;
      for (int j = 0; j < b.nj; ++j) {
        if (rem[j] == 0) continue;
        // extensions that start with job j: N * rem_j / left (exact)
        const uint64_t c = N / (uint64_t)left * (uint64_t)rem[j] + N % (uint64_t)left * (uint64_t)rem[j] / (uint64_t)left;
        if (r < c) {
          pick = j;
          N = c;
          break;
        }
        r -= c;
      }
      const int gene = b.jfirst[pick] + (b.jlen[pick] - rem[pick]);
      yo[gene] = (int16_t)(b.K - p);
      --rem[pick];
      --left;
    }
  }
}

// Running argmin over chunks: best[0] = objective word, best[1] = global index.
// One block; fixed order -> deterministic; ties -> lowest index.
__global__ void __launch_bounds__(1024) argmin_kernel(const int64_t *obj, int64_t count, uint64_t first,
                                                      int64_t *best) {
  __shared__ long long so[32];
  __shared__ unsigned long long si[32];
  long long bo = LLONG_MAX;
  unsigned long long bi = ULLONG_MAX;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const long long v = obj[i];
    if (v < bo) { bo = v; bi = first + (uint64_t)i; }   // strided: first hit is this thread's lowest index
  }
  for (int d = 16; d > 0; d >>= 1) {
    const long long o2 = __shfl_xor_sync(dev::FULL, bo, d);
    const unsigned long long i2 = __shfl_xor_sync(dev::FULL, bi, d);
    if (o2 < bo || (o2 == bo && i2 < bi)) { bo = o2; bi = i2; }
  }
  if ((threadIdx.x & 31) == 0) { so[threadIdx.x >> 5] = bo; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    bo = threadIdx.x < nw ? so[threadIdx.x] : LLONG_MAX;
    bi = threadIdx.x < nw ? si[threadIdx.x] : ULLONG_MAX;
    for (int d = 16; d > 0; d >>= 1) {
      const long long o2 = __shfl_xor_sync(dev::FULL, bo, d);
      const unsigned long long i2 = __shfl_xor_sync(dev::FULL, bi, d);
      if (o2 < bo || (o2 == bo && i2 < bi)) { bo = o2; bi = i2; }
    }
    if (threadIdx.x == 0 && (bo < best[0] || (bo == best[0] && (long long)bi < best[1]))) {
      best[0] = bo;
      best[1] = (long long)bi;
    }
  }
}

}  // namespace
}  // namespace edffs

using namespace edffs;

extern "C" {

ffs_status ffs_brute_force(const ffs_state *h, int64_t limit, int64_t *best_objective, int64_t *evaluated,
                           int8_t *best_x, int16_t *best_y, void *stream) {
  if (!h || limit <= 0) return fail(FFS_ERR_INVALID_ARG, "bad state or limit");
  State &st = const_cast<State &>(h->v);
  const int K = st.K, O = st.inst->o;
  if (K < 1) return fail(FFS_ERR_INVALID_ARG, "nothing to enumerate (K = 0)");
  if (K > kMaxBruteK) return fail(FFS_ERR_INVALID_ARG, "brute force needs K <= 64");
  BruteArgs b{};
  b.K = K;
  b.O = O;
  for (int k = 0; k < K; ++k) {
    if (k == 0 || st.gene_job[k] != st.gene_job[k - 1]) {
      if (b.nj == kMaxBruteJobs) return fail(FFS_ERR_INVALID_ARG, "brute force needs <= 64 jobs with pending ops");
      b.jfirst[b.nj] = k;
      b.jlen[b.nj] = 0;
      ++b.nj;
    }
    ++b.jlen[b.nj - 1];
  }
  // o^K and K!/prod L_j! with overflow checks against the limit
  const uint64_t lim = (uint64_t)limit;
  uint64_t nx = 1;
  for (int k = 0; k < K; ++k) {
    if (nx > lim / (uint64_t)O) return fail(FFS_ERR_INVALID_ARG, "o^K exceeds the enumeration limit");
    nx *= (uint64_t)O;
  }
  uint64_t no = 1;   // product of binomials C(prefix + L_j, L_j), each step exact
  int placed = 0;
  for (int j = 0; j < b.nj; ++j)
    for (int l = 1; l <= b.jlen[j]; ++l) {
      ++placed;
      // no * placed / l stays integral: no = C-products so far times C(placed, l)
      const unsigned __int128 v = (unsigned __int128)no * (uint64_t)placed / (uint64_t)l;
      if (v > lim) return fail(FFS_ERR_INVALID_ARG, "number of orders exceeds the enumeration limit");
      no = (uint64_t)v;
    }
  if (no > lim / nx) return fail(FFS_ERR_INVALID_ARG, "o^K * orders exceeds the enumeration limit");
  b.n_x = nx;
  b.n_orders = no;
  const uint64_t total = nx * no;

  cudaSetDevice(st.inst->dev);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t chunk = (int64_t)std::min<uint64_t>(total, (uint64_t)1 << 20);
  int8_t *dx = nullptr;
  int16_t *dy = nullptr;
  int64_t *dobj = nullptr, *dbest = nullptr;
  cudaError_t ce = cudaMallocAsync(&dx, (size_t)chunk * K, s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&dy, (size_t)chunk * K * 2, s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&dobj, (size_t)chunk * 8, s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(&dbest, 16, s);
  ffs_status e = FFS_OK;
  if (ce == cudaSuccess) {
    const int64_t init[2] = {LLONG_MAX, LLONG_MAX};
    ce = cudaMemcpyAsync(dbest, init, 16, cudaMemcpyHostToDevice, s);
  }
  if (ce != cudaSuccess) e = cuda_fail(ce, "brute force buffers");
  for (uint64_t first = 0; e == FFS_OK && first < total; first += (uint64_t)chunk) {
    const int64_t n = (int64_t)std::min<uint64_t>((uint64_t)chunk, total - first);
    const int64_t grid = std::min<int64_t>((n + 255) / 256, (int64_t)st.num_sms * 8);
    enumerate_kernel<<<(unsigned)grid, 256, 0, s>>>(b, first, n, dx, dy);
    ce = cudaGetLastError();
    if (ce != cudaSuccess) { e = cuda_fail(ce, "enumerate_kernel"); break; }
    EvalArgs a{};
    a.image = st.image_dev;
    a.count = n;
    a.x = dx;
    a.y = dy;
    a.obj = dobj;
    a.fstart = st.fstart_dev;
    e = launch_evaluate_shared(st, a, s);
    if (e != FFS_OK) break;
    argmin_kernel<<<1, 1024, 0, s>>>(dobj, n, first, dbest);
    ce = cudaGetLastError();
    if (ce != cudaSuccess) e = cuda_fail(ce, "argmin_kernel");
  }
  int64_t hb[2] = {0, 0};
  if (e == FFS_OK) {
    ce = cudaMemcpyAsync(hb, dbest, 16, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) e = cuda_fail(ce, "brute force result");
  }
  if (e == FFS_OK && (best_x || best_y)) {
    // regenerate the winning chromosome
    enumerate_kernel<<<1, 32, 0, s>>>(b, (uint64_t)hb[1], 1, dx, dy);
    std::vector<int8_t> bx(K);
    std::vector<int16_t> by(K);
    ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(bx.data(), dx, (size_t)K, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(by.data(), dy, (size_t)K * 2, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) e = cuda_fail(ce, "brute force best chromosome");
    if (e == FFS_OK) {
      if (best_x) std::copy(bx.begin(), bx.end(), best_x);
      if (best_y) std::copy(by.begin(), by.end(), best_y);
    }
  }
  cudaFreeAsync(dx, s);
  cudaFreeAsync(dy, s);
  cudaFreeAsync(dobj, s);
  cudaFreeAsync(dbest, s);
  if (e != FFS_OK) return e;
  if (best_objective) *best_objective = hb[0];
  if (evaluated) *evaluated = (int64_t)total;
  return FFS_OK;
}

}  // extern "C"
