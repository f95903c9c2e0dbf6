// ffs_common.cuh -- shared device/host definitions of the sm_100a library.
// Product code: independent of oracle/ (no shared code, tables or helpers).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/ffs.h"

namespace edffs {

// Programmatic dependent launch (sm_90+): kernels of the evaluate / GA chain
// are launched with launch_pdl, so a kernel's CTAs may start (launch, image
// staging, table building) while the previous kernel in the stream drains.
// Every kernel launched this way calls pdl_wait() -- in every CTA, before it
// touches anything an earlier kernel wrote -- and pdl_trigger() early, so its
// own successor can be scheduled.  Both are no-ops without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// launches on this thread that must NOT overlap what precedes them in their
// stream (e.g. the first kernel after a cross-stream event wait): launch_pdl
// uses plain stream order for that many launches
inline thread_local int t_plain_launches = 0;
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (t_plain_launches > 0) {
    --t_plain_launches;
    cfg.numAttrs = 0;
  }
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------------------
// Error plumbing (thread-local last error, status returns only)
// ---------------------------------------------------------------------------
void set_error(const std::string &msg);
ffs_status fail(ffs_status st, const std::string &msg);
ffs_status cuda_fail(cudaError_t e, const char *what);
#define FFS_CUDA(call)                                        \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return ::edffs::cuda_fail(_e, #call); \
  } while (0)

// ---------------------------------------------------------------------------
// Host-side objects behind the opaque handles
// ---------------------------------------------------------------------------
constexpr int kMaxWarpsPerCta = 32;
constexpr int kSmemLimit = 227 * 1024;

// The device state "image": one 16-byte aligned blob in global memory that
// every CTA stages into shared memory with cp.async.bulk (TMA) in its
// prologue.  Header followed by the arrays at the recorded offsets.
struct ImageHdr {
  int32_t K, NJ, G, O;
  int32_t rs, q_max;
  int32_t n_pjobs, lvl_words0;   // jobs with pending ops; 32-bit words of the initial profile
  int64_t wt;
  int64_t frozen_T;              // sum of T_j over jobs with no pending op (Eq. (2))
  int32_t frozen_cmax;           // max completion over those jobs (Eq. (3))
  int32_t cells;
  uint32_t off_pq;               // u32 [NJ*G*O]  p | q << 16
  uint32_t off_ginfo;            // u32 [K]       j | s << 16
  uint32_t off_head;             // u32 [ceil(K/32)] first pending gene of each job
  uint32_t off_ready0;           // i32 [NJ]      earliest start of the job's next op, rel. to RS
  uint32_t off_mfree0;           // i32 [G*O]     machine free time, rel. to RS
  uint32_t off_lvl0;             // u32 [lvl_words0] initial power profile (RUNNING ops), LVL-typed
  uint32_t off_pjob;             // i32 [n_pjobs] job index
  uint32_t off_pdue;             // i32 [n_pjobs] D_j - RS
  // lane-decode path (one lane per chromosome), see lane.cu
  uint32_t off_pqt;              // lane decoder's op table: mode 2 u32 [K*O] by gene (lane.cu), modes 0/1 u32 [NJ*G*O] p | q << 8 | j << 16
  uint32_t off_ready16;          // u32 [ceil(NJ/2)]  ready0 as u16 pairs
  uint32_t off_mfree16;          // u32 [ceil(G*O/2)] mfree0 as u16 pairs
  int32_t thr_min;               // Q_max - min Q: a slot is "blocked" for every op iff level > thr_min
  int32_t uniform_q;             // all Q_jsm equal
  uint32_t image_bytes;          // multiple of 16
  uint32_t lane_image_bytes;     // prefix staged by the lane-decode kernel
  int32_t lane_mode;             // 0 bytes/general q, 1 bytes/uniform q, 2 headroom planes (uniform Q = q, Q_max / q <= 15)
  int32_t lane_units;            // mode 2: Q_max / q, the number of ops that may run at once
  uint32_t off_hn0;              // u32 [hn_words0] initial headroom nibbles (mode 2)
  int32_t hn_words0;
  uint32_t off_bn0;              // u32 [bn_words0] initial blocked bits (mode 2)
  int32_t bn_words0;
  int32_t real_wt;               // 1: fractional WT (f3), objective/fitness are binary64 bit patterns
  int32_t pad_;
  double wt_f;                   // the real weight when real_wt
};

struct Instance {
  int dev = 0;
  int32_t n = 0, np = 0, g = 0, o = 0, NJ = 0;
  int32_t q_max = 0;
  int64_t wt = 0;
  std::vector<int32_t> P, Q, R, D;   // host copies [NJ*g*o], [NJ]
};

// Scratch of the overflow path (chromosomes whose schedule outgrows the
// in-SMEM profile are re-decoded with a global-memory profile).
struct OvfScratch {
  int32_t *list = nullptr;       // [1 + cap]: count, then chromosome ids
  int32_t *list2 = nullptr;      // [1 + cap]: what the LIST re-decode still overflows
  int64_t cap = 0;
  uint16_t *ordg = nullptr;      // lane path: rank-ordered ops, [tile][K][32]
  int64_t ordg_elems = 0;
  void *level = nullptr;         // [fallback warps * hfull * sizeof(LVL)]
  int64_t level_bytes = 0;
  // set (a GA run's scratch): allocations are stream-ordered from the
  // device's default memory pool on this stream (cheap re-allocation across
  // runs); unset: plain cudaMalloc
  cudaStream_t pool = nullptr;
  bool pooled = false;
  // cross-stream ordering of a state's shared scratch: `done` is recorded on
  // `last` after every call that used it; a call on another stream waits for it
  cudaEvent_t done = nullptr;
  cudaStream_t last = nullptr;
  bool used = false;
  ffs_status ensure(int64_t count, int64_t level_bytes_needed);
  ffs_status alloc(void **p, size_t bytes);
  void free_(void *p);
  void release();
};
// keep freed blocks of the default memory pool cached (no release to the
// driver at synchronisation points), once per device
void pool_keep(int dev);

// device staging of ffs_evaluate_host (grow-only)
struct HostStage {
  int8_t *x = nullptr;
  int16_t *y = nullptr;
  int64_t *obj = nullptr, *T = nullptr;
  int32_t *M = nullptr;
  int64_t cap = 0;
  size_t gene_cap = 0;
  cudaStream_t copy = nullptr, comp = nullptr;   // H2D stream, compute + D2H stream
  cudaEvent_t ev[9] = {};                         // [0..7] chunk uploaded, [8] entry / exit
  void release() {
    cudaFree(x); cudaFree(y); cudaFree(obj); cudaFree(T); cudaFree(M);
    x = nullptr; y = nullptr; obj = nullptr; T = nullptr; M = nullptr;
    cap = 0; gene_cap = 0;
  }
  void release_streams() {
    for (cudaEvent_t &e : ev)
      if (e) { cudaEventDestroy(e); e = nullptr; }
    if (copy) cudaStreamDestroy(copy);
    if (comp) cudaStreamDestroy(comp);
    copy = comp = nullptr;
  }
};

struct State {
  const Instance *inst = nullptr;
  int32_t rs = 0, K = 0, cells = 0;
  std::vector<int32_t> cell_state;   // 0 pending, 1 running, 2 completed, 3 kept (static policy)
  int32_t real_wt = 0;               // fractional WT (f3): binary64 objective words
  double wt_f = 0.0;
  std::vector<int32_t> fassign, fstart;
  std::vector<int32_t> gene_job, gene_stage, gene_cell;
  std::vector<int32_t> pend_before;  // [cells+1]
  int32_t h_bound = 0;               // slots needed for any schedule (rel. to RS)
  int32_t h_cap = 0;                 // slots of the in-SMEM profile
  int32_t h_cap_user = 0;
  int lvl_bytes = 1;                 // 1: u8 profile (Q_max <= 255), 2: u16
  std::vector<uint8_t> image_host;   // built for the current h_cap
  void *image_dev = nullptr;
  int32_t *fstart_dev = nullptr;     // [cells] frozen starts (abs), -1 pending
  int32_t *cut_dev = nullptr;        // [cells+1] pend_before on device
  uint32_t *gbase_dev = nullptr;     // [K] (j*G + s)*O of each gene
  // launch geometry of the evaluate kernel
  int warps_per_cta = 0, ctas_per_sm = 0, num_sms = 0;
  size_t smem_bytes = 0, per_warp_bytes = 0;
  size_t fb_smem_bytes = 0, fb_per_warp_bytes = 0;
  int fb_warps_per_cta = 4;
  bool fb_level_smem = false;        // fallback profile in shared memory (h_bound fits)
  bool fb_global_forced = false;     // FFS_FALLBACK_GLOBAL set: keep it in global memory
  int32_t relist_cap = -1;           // FFS_RELIST_CAP: cap of lane_hcap2 (0: no re-decode, <0: none)
  int32_t *ovf_seen_host = nullptr;  // mapped: nonzero once any lane decode of this state overflowed
  int32_t *ovf_seen_dev = nullptr;
  // lane-decode path geometry (valid when lane_ok)
  bool lane_ok = false;
  bool lane_disabled = false;        // FFS_DISABLE_LANE set: force the warp path
  bool ord_xs_disabled = false;      // FFS_ORDER_NO_XS set: order kernel without x staging
  int32_t lane_hcap = 0;             // profile slots per chromosome (multiple of 32)
  int32_t lane_wpt = 0;              // 32-bit state words per thread
  int lane_warps_per_cta = 0, lane_ctas_per_sm = 1;
  size_t lane_smem = 0;
  // mode 2's overflow re-decode (LIST launch): the same lane kernel over the
  // overflow list with a longer horizon and fewer warps per CTA (0: none)
  int32_t lane_hcap2 = 0, lane_wpt2 = 0;
  int lane_warps2 = 0;
  size_t lane_smem2 = 0;
  size_t ord_smem = 0, ord_hist_bytes = 0, ord_stride = 0, ord_xs_bytes = 0;
  bool ord_xs = false;   // order kernel stages x rows (ord_smem + ord_xs_bytes fits)
  // ^ order kernel (32 warps per CTA)
  int32_t max_pending = 0;                                   // most pending genes of one job
  int32_t ord_ubits = 1;                                     // order kernel: bits of u = K - pm (2^ubits >= K)
  int ord_ctas_per_sm = 1;
  OvfScratch scratch;
  HostStage stage;
  ffs_status build_image();
};

// Arguments of one evaluate launch (device pointers).
// Eq. (1) and Eq. (13) on the 64-bit objective/fitness words:
// integer WT (R25) -> exact int64; real WT (Table 11, f3) -> binary64 bit
// patterns of fl(fl(WT * sum T) + C_max) and max(E_max - obj, +0).  Every
// objective and fitness is >= 0, so the bit patterns order like the values
// and every GA comparison (selection, replacement, migration, E_max's
// max-reduction, trace min) works on the int64 words unchanged.
__device__ __forceinline__ int64_t objective_word(int real, int64_t wt, double wt_f, int64_t T, int32_t cm) {
  if (real) return __double_as_longlong(__dadd_rn(__dmul_rn(__ll2double_rn(T), wt_f), __int2double_rn(cm)));
  return wt * T + (int64_t)cm;
}
__device__ __forceinline__ int64_t fitness_word(int real, int64_t emax, int64_t obj) {
  if (real) {
    const double f = __dsub_rn(__longlong_as_double(emax), __longlong_as_double(obj));
    return f > 0.0 ? __double_as_longlong(f) : 0;
  }
  const int64_t f = emax - obj;
  return f > 0 ? f : 0;
}

struct EvalArgs {
  const void *image;
  int64_t count;
  const int8_t *x;
  const int16_t *y;
  int64_t *obj;
  int64_t *tard;
  int32_t *cmax;
  int32_t *start_out;            // optional full schedule
  const int32_t *fstart;         // frozen starts for start_out
  const int64_t *emax;           // optional: fitness = max(*emax - obj, 0)
  int64_t *fit;
  int32_t *ovf;                  // overflow list (count at [0])
  int32_t *ovf2;                 // LIST launch: its own overflows (count at [0])
  int32_t *ovf_seen;             // mapped host flag, set on any overflow (may be null)
  int32_t relist;                // lane path: launch the LIST re-decode (decided once per call)
  void *lvl_global;              // fallback: global profiles
  int32_t lvl_smem;              // fallback: profile in shared memory instead (h_cap fits)
  int32_t h_cap;                 // slots in the profile used by this launch
  int32_t per_warp_bytes;
  const uint16_t *ordg;          // lane path
  int64_t first;                 // lane path: first chromosome of this chunk
  int64_t row;                   // genes between consecutive chromosomes of x / y (0: K)
};

ffs_status launch_lane(const State &st, const EvalArgs &a, OvfScratch &scr, cudaStream_t s, int *launches);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) when `bytes` exceeds what
// was set before for this kernel on the current device (the attribute lives
// in the device context; the cache is keyed by kernel and device, thread-safe)
ffs_status ensure_smem_attr(const void *kernel, size_t bytes);

ffs_status launch_evaluate(const State &st, const EvalArgs &a, OvfScratch &scr, cudaStream_t s,
                           int *launches);
// launch_evaluate on the state's own scratch (every device-pointer call on a
// state: ffs_evaluate*, ffs_evaluate_host's chunks, ffs_brute_force): ordered
// after the previous such call when that one ran on another stream.
ffs_status launch_evaluate_shared(State &st, const EvalArgs &a, cudaStream_t s);
ffs_status launch_random_population(const State &st, int64_t count, uint64_t seed, int64_t first_id, int64_t row,
                                    int8_t *x, int16_t *y, cudaStream_t s);

// ---------------------------------------------------------------------------
// Philox4x32-10 (device), DESIGN.md "RNG"
// ---------------------------------------------------------------------------
struct u32x4 { uint32_t x, y, z, w; };
__host__ __device__ __forceinline__ u32x4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                  uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}
enum : uint32_t { RNG_INIT_X = 1, RNG_INIT_Y = 2, RNG_XO = 3, RNG_MUT = 4, RNG_MUT_X = 5 };
__host__ __device__ __forceinline__ uint32_t word_of(const u32x4 &v, int w) {
  return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
}
__host__ __device__ __forceinline__ uint32_t bounded(uint32_t u, uint32_t n) {
  return (uint32_t)(((uint64_t)u * n) >> 32);
}

#ifdef __CUDACC__
// The initialisation's priorities: y[g] = 1 + the rank of
// gene g's key, ascending by (key, gene index).  One warp sorts the composite
// keys key << 32 | g (distinct) with a bitonic network in shared memory
// (buf: NP u64, NP = a power of two >= max(K, 64); buf[0..K) filled by the
// caller) and scatters y.  O(K log^2 K) instead of O(K^2) comparisons.
__device__ __forceinline__ void rank_keys_warp(unsigned long long *buf, int K, int NP, int lane, int16_t *y) {
  for (int g = K + lane; g < NP; g += 32) buf[g] = ~0ull;
  __syncwarp();
  for (int k = 2; k <= NP; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < (NP >> 1); i += 32) {
        const int a = 2 * i - (i & (j - 1)), b = a + j;   // comparator i of this step: (a, a + j)
        const unsigned long long va = buf[a], vb = buf[b];
        if ((va > vb) == ((a & k) == 0)) {
          buf[a] = vb;
          buf[b] = va;
        }
      }
      __syncwarp();
    }
  }
  for (int p = lane; p < K; p += 32) y[(uint32_t)buf[p]] = (int16_t)(p + 1);
  __syncwarp();
}
#endif

}  // namespace edffs

struct ffs_instance { edffs::Instance v; };
struct ffs_state { edffs::State v; };
