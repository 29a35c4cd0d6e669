// Shared definitions for the B200-native anisotropic PQ library.
//
// Device data layout:
//   * dataset rows are stored "pair-tiled": rows grouped in tiles of 32, and
//     inside a tile each pair of dimensions (2p, 2p+1) is a contiguous block
//     of 32 float2 (one per row). A warp whose lanes own 32 consecutive rows
//     reads the sub-vector of one 2-D subspace as a single coalesced 256-byte
//     load; no shared-memory staging or transpose is needed in the encoders.
//   * norms are float64, computed on the device in the reference's order
//     (dataset.hpp:55-59: sequential sum of squares, then sqrt).
//   * codes are packed row-major: 4-bit (k <= 16, low nibble = even m) or
//     8-bit (k <= 256), row stride rounded up to 8 bytes.
//   * codebooks are kept in float64 (the reference's arithmetic) plus float32
//     staging tables used only as filters whose errors are bounded.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/anisoq_b200.h"

namespace aqd {

// ---- error plumbing -------------------------------------------------------
void set_error(int status, const char* fmt, ...);
int ref_error(int status, const char* detail);  // "<RefName>: detail"
const char* status_ref_name(int status);

#define AQ_CUDA(call)                                                     \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess) {                                              \
      ::aqd::set_error(AQ_E_CUDA, "CUDA error %s at %s:%d: %s",           \
                       cudaGetErrorName(e_), __FILE__, __LINE__,          \
                       cudaGetErrorString(e_));                           \
      return AQ_E_CUDA;                                                   \
    }                                                                     \
  } while (0)

#define AQ_TRY(expr)             \
  do {                           \
    int st_ = (expr);            \
    if (st_ != AQ_OK) return st_; \
  } while (0)

#define AQ_LAUNCHED(sess)                 \
  do {                                    \
    (sess)->launches++;                   \
    AQ_CUDA(cudaGetLastError());          \
  } while (0)

// Device-side error record: the smallest offending point index wins, which is
// the error the reference's sequential loops would raise first.
struct DevError {
  unsigned long long key;  // (index << 8) | status, ~0ull when clear
};

__device__ __forceinline__ void report_error(DevError* e, uint64_t index,
                                             int status) {
  atomicMin(&e->key, (unsigned long long)((index << 8) | (uint64_t)status));
}

// ---- scratch memory ---------------------------------------------------------
struct Scratch {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace aqd

// Optional per-kernel CUDA-event timers (bench.py's roofline evidence).
enum AqTimer { AQ_T_ENCODE = 0, AQ_T_ADC_SCORE = 1, AQ_T_ADC_MERGE = 2,
               AQ_T_RERANK = 3, AQ_T_LUT = 4, AQ_T_ASSEMBLE = 5, AQ_T_LLT = 6,
               AQ_T_KMEANS = 7, AQ_T_EXACT = 8, AQ_T_COUNT = 9 };

struct aq_session {
  int device = 0;
  bool timing = false;
  std::vector<cudaEvent_t> tev[AQ_T_COUNT];  // start/end pairs
  double tms[AQ_T_COUNT] = {0};
  uint64_t tcount[AQ_T_COUNT] = {0};
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;        // loss totals overlapped with the next update
  cudaEvent_t ev_main = nullptr, ev_side = nullptr;
  double* sum_host = nullptr;         // pinned, 64 slots
  uint64_t launches = 0;
  int num_sms = 148;
  aqd::DevError* err = nullptr;     // device
  aqd::DevError* err_host = nullptr;  // pinned mirror
  aqd::Scratch scratch[8];  // slot 6: scan tile sums (sort.cu), 7: ADC tensor-core work windows
  aqd::Scratch pinned[7];   // page-locked host staging (streamed host-pointer calls; 6: packed codes)
};

struct aq_dataset {
  aq_session* s = nullptr;
  size_t n = 0, d = 0;
  float* xt = nullptr;      // pair-tiled rows (encoders, search)
  float* xr = nullptr;      // row-major rows (normal equations, gathers)
  double* norms = nullptr;  // float64 norms
  // Datasets whose values are not all float32-exact (e.g. unit_normalize
  // output, dataset.hpp:229) keep float64 rows instead: f64 = 1, xt64 / xr64
  // set, xt / xr null. Every kernel that reads rows has a float64
  // instantiation; the float32-filter fast paths (sd = 2 encoders, k-means,
  // slot gathers, exact-search filter) are float32-only and are bypassed.
  int f64 = 0;
  double* xt64 = nullptr;
  double* xr64 = nullptr;
};

// Launch KERNEL<float>(ds->xr, ...) or KERNEL<double>(ds->xr64, ...) by the
// dataset's row type (row-major rows as the first kernel argument).
#define AQ_XR_LAUNCH(ds, KERNEL, grid, block, smem, stream, ...)                      \
  do {                                                                               \
    if ((ds)->f64)                                                                   \
      KERNEL<double><<<(grid), (block), (smem), (stream)>>>((ds)->xr64, __VA_ARGS__); \
    else                                                                             \
      KERNEL<float><<<(grid), (block), (smem), (stream)>>>((ds)->xr, __VA_ARGS__);   \
  } while (0)

struct aq_codebook {
  aq_session* s = nullptr;
  size_t M = 0, k = 0, sd = 0;
  double* d64 = nullptr;   // (m*k + j)*sd
  float4* f32 = nullptr;   // sd == 2: [M][16] {c0, c1, c0^2+c1^2, 0}
  float* rmax = nullptr;   // [M] max_j |c_mj| (float32 norm, rounded up)
};

struct aq_codes {
  aq_session* s = nullptr;
  size_t n = 0, M = 0, k = 0;
  size_t stride = 0;       // bytes per row
  int bits = 4;            // 4 or 8
  uint8_t* data = nullptr;
};

namespace aqd {

// Scratch buffers owned by the session, grown on demand (slot-indexed so that
// concurrently live temporaries never alias).
int scratch(aq_session* s, int slot, size_t bytes, void** out);
int check_session(aq_session* s);
int tile_rows_async(const float* xdev, size_t n, size_t d, float* xt, double* norms,
                    cudaStream_t stream);
int sync_and_check(aq_session* s, const char* what);  // reads DevError
int clear_dev_error(aq_session* s);

__host__ __device__ void timer_mark(aq_session* s, int slot);  // records an event if timing

__host__ __device__ inline size_t pairs_of(size_t d) { return (d + 1) / 2; }
inline size_t tiled_floats(size_t n, size_t d) {
  return ((n + 31) / 32) * pairs_of(d) * 64;
}
inline size_t code_stride(size_t M, int bits) {
  const size_t raw = bits == 4 ? (M + 1) / 2 : M;
  return (raw + 7) & ~size_t(7);
}

__host__ __device__ __forceinline__ size_t tiled_index(size_t i, size_t j,
                                                       size_t pairs) {
  return (((i >> 5) * pairs + (j >> 1)) * 32 + (i & 31)) * 2 + (j & 1);
}

__device__ __forceinline__ unsigned get_code(const uint8_t* row, int m,
                                             int bits) {
  if (bits == 4) return (row[m >> 1] >> ((m & 1) * 4)) & 15u;
  return row[m];
}

// Stable per-subspace bucket lists of points by code (update.cu): list[m][.]
// holds, for every code j, the points with code j at subspace m in ascending
// order starting at start[m][j], count[m][j] of them.
struct Buckets {
  uint32_t* list = nullptr;   // [M][n]
  uint32_t* start = nullptr;  // [M][K]
  uint32_t* count = nullptr;  // [M][K]
  int K = 0;
};
int build_buckets(aq_codes* c, int k, Buckets* B);
// exclusive scan of 32-bit counts in place (sort.cu)
int scan_device(aq_session* s, unsigned* hist, size_t total);

// Per-point anisotropic weights (update.cu): h_par, h_perp, coupling coefficient;
// flags[0] = some point anisotropic, flags[1] = first anisotropic |x| = 0 index + 1
// (~0 = none).
struct PointW {
  double* hp = nullptr;
  double* ho = nullptr;
  double* coef = nullptr;
  unsigned long long flags[2] = {0, 0};
};
int point_weights(aq_dataset* ds, const aq_weights* w, PointW* pw, void** owner);
int assemble_device(aq_dataset* ds, aq_codes* codes, const PointW& pw, const Buckets& B,
                    int k, bool full, double* A, double* rhs);
int llt_solve_device(aq_session* s, double* A, int n, double* x);
int trace_ridge_device(aq_session* s, double* A, size_t dim, double ridge);
// per-slot point-ordered sums (train.cu k_slot_sums): hp == null -> unit
// weights; dict != null -> means of non-empty slots, else num/den partials
int slot_sums_device(aq_session* s, const aq_dataset* ds, int M, int k, int sd,
                     const Buckets& B, const int* active, const double* hp, const double* ho,
                     double* dict, double* pnum, double* pden);

// ---- weights ------------------------------------------------------------------
// Resolved per point on the device from an aq_weights descriptor
// (geometry.hpp:119-145, eta_limit 395-402, CLI resolve_weights
// anisoq_main.cpp:108-142).
struct DevWeights {
  int mode;
  double hp, ho;          // UNIFORM
  const double* hp_arr;   // PER_POINT (device copies)
  const double* ho_arr;
  double threshold;       // THRESHOLD
  int policy;
  int d;
};

int make_dev_weights(aq_session* s, const aq_weights* w, size_t n, size_t d,
                     DevWeights* out);

__device__ __forceinline__ bool resolve_weights(const DevWeights& w,
                                                size_t i, double norm,
                                                double* hp, double* ho,
                                                int* status) {
  if (w.mode == AQ_WEIGHTS_UNIFORM) {
    *hp = w.hp;
    *ho = w.ho;
    return true;
  }
  if (w.mode == AQ_WEIGHTS_PER_POINT) {
    *hp = w.hp_arr[i];
    *ho = w.ho_arr[i];
    return true;
  }
  // eta_limit (geometry.hpp:395-402), op order kept.
  if (!(norm > 0.0)) {
    *status = AQ_E_INVALID_ARGUMENT;
    return false;
  }
  const double t = w.threshold;
  if (!(t >= 0.0) || t >= norm) {
    if (w.policy == AQ_THRESHOLD_PARALLEL_ONLY && t >= 0.0) {
      *hp = 1.0;  // eta = inf: parallel error only
      *ho = 0.0;
      return true;
    }
    *status = AQ_E_INVALID_THRESHOLD;
    return false;
  }
  const double r = __ddiv_rn(t, norm);
  const double rho = __dmul_rn(r, r);
  const double eta =
      __ddiv_rn(__dmul_rn((double)(w.d - 1), rho), __dsub_rn(1.0, rho));
  *hp = eta;
  *ho = 1.0;
  return true;
}

// ---- exact float64 primitives (no contraction; reference op order) ----------

// detail::residual_terms (geometry.hpp:182-192) for sd == 2.
__device__ __forceinline__ void residual2(double x0, double x1, double c0,
                                          double c1, double* d2, double* rd) {
  const double df0 = __dsub_rn(x0, c0);
  const double df1 = __dsub_rn(x1, c1);
  // 0.0 + df0^2 == df0^2 for every input (squares are >= +0 or NaN), so the
  // reference's first accumulation into zero is dropped for dist2; rdot keeps
  // it (0.0 + (-0.0) = +0.0)
  double a = __dmul_rn(df0, df0);
  a = __dadd_rn(a, __dmul_rn(df1, df1));
  double b = __dadd_rn(0.0, __dmul_rn(df0, x0));
  b = __dadd_rn(b, __dmul_rn(df1, x1));
  *d2 = a;
  *rd = b;
}

// detail::combined_loss (geometry.hpp:196-200).
__device__ __forceinline__ double combined_loss(double dist2, double rdot,
                                                double hp, double ho,
                                                double inv_norm2) {
  return __dadd_rn(
      __dmul_rn(ho, dist2),
      __dmul_rn(__dmul_rn(__dsub_rn(hp, ho), __dmul_rn(rdot, rdot)),
                inv_norm2));
}

// N-th largest key (.x, unsigned) over a query's candidate windows
// lists[r * cap + e], e < cnts[r], r < R, by a three-pass radix select
// (11 + 11 + 10 bits) with a shared-memory histogram `hist` (>= 2048 words).
// Equals the largest T with |{key >= T}| >= N (the result of a 32-step
// binary search) but reads the entries 3 times instead of 32. Requires
// total >= N >= 1; block-wide (every thread calls it), blockDim.x a
// multiple of 32 and <= 1024.
__device__ inline unsigned block_nth_largest(const uint2* lists, const int* cnts, int R,
                                             size_t cap, int N, unsigned* hist) {
  __shared__ unsigned s_wsum[32];
  __shared__ unsigned s_pick[2];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
  unsigned prefix = 0u, pmask = 0u;
  unsigned need = (unsigned)N;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
    const int nb = pass == 2 ? 1024 : 2048;
    for (int i = tid; i < nb; i += nt) hist[i] = 0u;
    __syncthreads();
    // warp per window: many windows' loads in flight at once
    for (int r = w; r < R; r += nt >> 5)
      for (int e = lane; e < cnts[r]; e += 32) {
        const unsigned key = lists[(size_t)r * cap + e].x;
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & (unsigned)(nb - 1)], 1u);
      }
    __syncthreads();
    // thread t owns `per` bins counted from the top; exclusive prefix from
    // the top finds the bin where the running count reaches `need`
    const int per = (nb + nt - 1) / nt;
    const int hi = nb - tid * per;  // bins [lo, hi), top first
    const int lo = max(0, hi - per);
    unsigned sum = 0u;
    for (int b = lo; b < hi; ++b) sum += hist[b];
    unsigned inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) s_wsum[w] = inc;
    __syncthreads();
    unsigned before = 0u;
    for (int t = 0; t < w; ++t) before += s_wsum[t];
    before += inc - sum;  // count in bins above this thread's range
    if (before < need && before + sum >= need) {
      unsigned run = before;
      for (int b = hi - 1; b >= lo; --b) {
        if (run + hist[b] >= need) {
          s_pick[0] = (unsigned)b;
          s_pick[1] = run;
          break;
        }
        run += hist[b];
      }
    }
    __syncthreads();
    prefix |= s_pick[0] << shift;
    pmask |= (unsigned)(nb - 1) << shift;
    need -= s_pick[1];
    __syncthreads();
  }
  return prefix;
}

// anisoq::Rng (rng.hpp:28-89) on the host: splitmix64, next_below by
// rejection; used for the trainers' seeded initial codewords.
struct HostRng {
  uint64_t state;
  uint64_t next_u64() {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  uint64_t next_below(uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
  // sample_distinct (rng.hpp:74-83): partial Fisher-Yates on iota(n); only the
  // touched positions are materialised, so it is O(k) instead of O(n).
  std::vector<size_t> sample_distinct(size_t n, size_t k) {
    std::unordered_map<size_t, size_t> moved;
    auto get = [&](size_t i) {
      auto it = moved.find(i);
      return it == moved.end() ? i : it->second;
    };
    std::vector<size_t> out;
    for (size_t i = 0; i < k && i < n; ++i) {
      const size_t j = i + (size_t)next_below(n - i);
      const size_t vi = get(i), vj = get(j);
      moved[i] = vj;
      moved[j] = vi;
      out.push_back(vj);
    }
    return out;
  }
};

}  // namespace aqd
