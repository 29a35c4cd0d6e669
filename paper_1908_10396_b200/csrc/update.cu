// Codebook update (pq_codebook_update, pq.hpp:356-464) on the device:
//   * stable per-subspace bucket lists of points by code (counting sort);
//   * the dense normal equations (assemble_selector_system, pq.hpp:290-343):
//     one warp per (row strip (m, j), 32 column subspaces); every entry is
//     accumulated by one lane over the strip's points in ascending point
//     order with the reference's operation order, so the matrix (and rhs) is
//     bit-identical to the reference's serial loop;
//   * ridge + blocked Cholesky + triangular solves mirroring the oracle's
//     pinned LLT (oracle/eigen_subset/Eigen/Dense): block 64, sequential inner
//     sums, products rounded before the add/sub;
//   * the isotropic weighted-mean path (pq.hpp:405-423);
//   * reseeding of unused codewords from the loss ranking (pq.hpp:443-462).
#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"

namespace aqd {

int sort_scores_desc(aq_session* s, const double* scores, uint32_t* idx, size_t n);
int run_encode(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes,
               int mode, int passes, int sweep_fixed, double* losses_dev,
               uint64_t* changed_out);
int stage_codebook(aq_codebook* cb);

constexpr int kBucketBlock = 1024;
constexpr int kLLT = 64;  // pinned block size (Eigen stand-in)

// ---- bucket lists -------------------------------------------------------------------

__global__ void k_bucket_hist(const uint8_t* __restrict__ codes, size_t n, int stride,
                              int bits, int K, unsigned* __restrict__ hist, size_t nb,
                              DevError* err, int k) {
  __shared__ unsigned h[256];
  const int m = blockIdx.y;
  for (int t = threadIdx.x; t < K; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * kBucketBlock;
  for (int t = threadIdx.x; t < kBucketBlock; t += blockDim.x) {
    const size_t i = base + t;
    if (i < n) {
      const unsigned c = get_code(codes + i * stride, m, bits);
      if ((int)c >= k) report_error(err, i, AQ_E_CODE_OUT_OF_RANGE);
      atomicAdd(&h[min(c, (unsigned)K - 1)], 1u);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < K; t += blockDim.x)
    hist[((size_t)m * K + t) * nb + blockIdx.x] = h[t];
}

// stable scatter (points keep ascending order inside every bucket)
__global__ void k_bucket_scatter(const uint8_t* __restrict__ codes, size_t n, int stride,
                                 int bits, int K, const unsigned* __restrict__ base,
                                 size_t nb, uint32_t* __restrict__ list) {
  __shared__ unsigned run[256];
  __shared__ unsigned wcnt[8][256];
  const int m = blockIdx.y;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < K; t += blockDim.x)
    run[t] = base[((size_t)m * K + t) * nb + blockIdx.x] - (unsigned)((size_t)m * n);
  const size_t b0 = (size_t)blockIdx.x * kBucketBlock;
  for (int round = 0; round < kBucketBlock / 256; ++round) {
    for (int t = threadIdx.x; t < 8 * 256; t += blockDim.x) (&wcnt[0][0])[t] = 0;
    __syncthreads();
    const size_t i = b0 + (size_t)round * 256 + threadIdx.x;
    const bool valid = i < n;
    const unsigned dg = valid ? min(get_code(codes + i * stride, m, bits), (unsigned)K - 1)
                              : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const unsigned rk = __popc(peers & ((1u << lane) - 1u));
    if (valid && rk == 0) wcnt[w][dg] = __popc(peers);
    __syncthreads();
    if (valid) {
      unsigned before = 0;
      for (int ww = 0; ww < w; ++ww) before += wcnt[ww][dg];
      list[(size_t)m * n + run[dg] + before + rk] = (uint32_t)i;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < K; t += blockDim.x) {
      unsigned s = 0;
      for (int ww = 0; ww < 8; ++ww) s += wcnt[ww][t];
      run[t] += s;
    }
    __syncthreads();
  }
}

// Row-staged variants (all subspaces per block): the block's 256-point code
// rows are copied to shared memory once (8-byte loads, coalesced) and every
// subspace reads its nibbles there, instead of one (block, subspace) CTA per
// pair re-reading each 32-byte sector for every subspace it holds (the
// per-subspace kernels above read the code matrix ~M/2 times through L2).
// Same histogram layout and the same stable order as the kernels above.
constexpr int kRowsRound = 256;

__device__ __forceinline__ void stage_code_rows(const uint8_t* codes, size_t n, int stride,
                                                size_t i0, uint8_t* rows) {
  const int words = stride >> 3;
  for (int t = threadIdx.x; t < kRowsRound * words; t += blockDim.x) {
    const int r = t / words, w = t % words;
    const size_t i = i0 + r;
    reinterpret_cast<uint2*>(rows)[t] =
        i < n ? reinterpret_cast<const uint2*>(codes + i * stride)[w] : make_uint2(0u, 0u);
  }
}

__global__ void __launch_bounds__(256) k_bucket_hist_rows(const uint8_t* __restrict__ codes,
                                                          size_t n, int stride, int bits, int M,
                                                          int K, unsigned* __restrict__ hist,
                                                          size_t nb, DevError* err, int k) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* h = reinterpret_cast<unsigned*>(sm);                // [M][K]
  uint8_t* rows = sm + (((size_t)M * K * 4 + 15) & ~(size_t)15);  // [256][stride]
  for (int t = threadIdx.x; t < M * K; t += blockDim.x) h[t] = 0;
  const size_t base = (size_t)blockIdx.x * kBucketBlock;
  for (int round = 0; round < kBucketBlock / kRowsRound; ++round) {
    const size_t i0 = base + (size_t)round * kRowsRound;
    if (i0 >= n) break;
    __syncthreads();
    stage_code_rows(codes, n, stride, i0, rows);
    __syncthreads();
    const size_t i = i0 + threadIdx.x;
    if (i < n) {
      const uint8_t* row = rows + (size_t)threadIdx.x * stride;
      for (int m = 0; m < M; ++m) {
        const unsigned c = get_code(row, m, bits);
        if ((int)c >= k) report_error(err, i, AQ_E_CODE_OUT_OF_RANGE);
        atomicAdd(&h[m * K + min(c, (unsigned)K - 1)], 1u);
      }
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < M * K; t += blockDim.x)
    hist[(size_t)t * nb + blockIdx.x] = h[t];
}

__global__ void __launch_bounds__(256) k_bucket_scatter_rows(const uint8_t* __restrict__ codes,
                                                             size_t n, int stride, int bits,
                                                             int M, int K,
                                                             const unsigned* __restrict__ base,
                                                             size_t nb,
                                                             uint32_t* __restrict__ list) {
  extern __shared__ __align__(16) unsigned char sm[];
  unsigned* run = reinterpret_cast<unsigned*>(sm);  // [M][K]
  unsigned* wcnt2 = run + (size_t)M * K;           // [2][8][K], alternating by m
  uint8_t* rows = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(wcnt2 + 16 * K) + 15) & ~(uintptr_t)15);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < M * K; t += blockDim.x)
    run[t] = base[(size_t)t * nb + blockIdx.x] - (unsigned)((size_t)(t / K) * n);
  const size_t b0 = (size_t)blockIdx.x * kBucketBlock;
  for (int round = 0; round < kBucketBlock / kRowsRound; ++round) {
    const size_t i0 = b0 + (size_t)round * kRowsRound;
    if (i0 >= n) break;
    __syncthreads();
    stage_code_rows(codes, n, stride, i0, rows);
    const size_t i = i0 + threadIdx.x;
    const bool valid = i < n;
    const uint8_t* row = rows + (size_t)threadIdx.x * stride;
    for (int m = 0; m < M; ++m) {
      // this buffer was last read two subspaces ago, three barriers back
      unsigned* wcnt = wcnt2 + (m & 1) * 8 * K;
      for (int t = threadIdx.x; t < 8 * K; t += blockDim.x) wcnt[t] = 0;
      __syncthreads();
      const unsigned dg = valid ? min(get_code(row, m, bits), (unsigned)K - 1) : 0xffffffffu;
      const unsigned peers = __match_any_sync(0xffffffffu, dg);
      const unsigned rk = __popc(peers & ((1u << lane) - 1u));
      if (valid && rk == 0) wcnt[w * K + dg] = __popc(peers);
      __syncthreads();
      if (valid) {
        unsigned before = 0;
        for (int ww = 0; ww < w; ++ww) before += wcnt[ww * K + dg];
        list[(size_t)m * n + run[m * K + dg] + before + rk] = (uint32_t)i;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < K; t += blockDim.x) {
        unsigned sacc = 0;
        for (int ww = 0; ww < 8; ++ww) sacc += wcnt[ww * K + t];
        run[m * K + t] += sacc;
      }
    }
  }
}

__global__ void k_bucket_offsets(const unsigned* __restrict__ base, size_t nb, int M, int K,
                                 size_t n, uint32_t* __restrict__ start,
                                 uint32_t* __restrict__ count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * K) return;
  const int m = t / K, j = t % K;
  const unsigned s0 = base[((size_t)m * K + j) * nb] - (unsigned)((size_t)m * n);
  const unsigned s1 = j + 1 < K ? base[((size_t)m * K + j + 1) * nb] - (unsigned)((size_t)m * n)
                                : (unsigned)n;
  start[t] = s0;
  count[t] = s1 - s0;
}


int build_buckets(aq_codes* c, int k, Buckets* B) {
  aq_session* s = c->s;
  const size_t n = c->n, M = c->M;
  // Offsets are scanned globally over [m][j][block] in 32-bit arithmetic; when
  // n M >= 2^32 they wrap, but every consumer subtracts m n in the same
  // modular arithmetic and the local offsets (< n) come out exact.
  const int K = k;
  const size_t nb = (n + kBucketBlock - 1) / kBucketBlock;
  void* p;
  AQ_TRY(scratch(s, 2, (M * n + 2 * M * K + M * K * nb) * sizeof(unsigned) + 256, &p));
  B->list = (uint32_t*)p;
  B->start = B->list + M * n;
  B->count = B->start + M * K;
  unsigned* hist = B->count + M * K;
  B->K = K;
  AQ_TRY(clear_dev_error(s));
  // row-staged kernels when the block's counters and 256 code rows fit
  const size_t hist_sm = (((size_t)M * K * 4 + 15) & ~(size_t)15) + (size_t)kRowsRound * c->stride;
  const size_t scat_sm = ((((size_t)M * K + 16 * K) * 4 + 15) & ~(size_t)15) +
                         (size_t)kRowsRound * c->stride;
  static const int rows_env = getenv("AQ_BUCKET_ROWS") ? atoi(getenv("AQ_BUCKET_ROWS")) : 1;
  const bool rows =
      rows_env && std::max(hist_sm, scat_sm) <= 160 * 1024 && (c->stride % 8) == 0;
  if (rows) {
    AQ_CUDA(cudaFuncSetAttribute(k_bucket_hist_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)hist_sm));
    k_bucket_hist_rows<<<(unsigned)nb, 256, hist_sm, s->stream>>>(
        c->data, n, (int)c->stride, c->bits, (int)M, K, hist, nb, s->err, k);
  } else {
    k_bucket_hist<<<dim3((unsigned)nb, (unsigned)M), 256, 0, s->stream>>>(
        c->data, n, (int)c->stride, c->bits, K, hist, nb, s->err, k);
  }
  AQ_LAUNCHED(s);
  AQ_TRY(sync_and_check(s, "codebook update: code out of range"));
  AQ_TRY(scan_device(s, hist, M * K * nb));
  if (rows) {
    AQ_CUDA(cudaFuncSetAttribute(k_bucket_scatter_rows,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scat_sm));
    k_bucket_scatter_rows<<<(unsigned)nb, 256, scat_sm, s->stream>>>(
        c->data, n, (int)c->stride, c->bits, (int)M, K, hist, nb, B->list);
  } else {
    k_bucket_scatter<<<dim3((unsigned)nb, (unsigned)M), 256, 0, s->stream>>>(
        c->data, n, (int)c->stride, c->bits, K, hist, nb, B->list);
  }
  AQ_LAUNCHED(s);
  k_bucket_offsets<<<(unsigned)((M * K + 255) / 256), 256, 0, s->stream>>>(
      hist, nb, (int)M, K, n, B->start, B->count);
  AQ_LAUNCHED(s);
  return AQ_OK;
}

// ---- per-point weights: h_par, h_perp, coupling coefficient -----------------------------
// coef = (h_par - h_perp) / |x|^2 exactly as pq.hpp:313-319; flags[0] = some
// point is anisotropic, flags[1] = smallest anisotropic zero-norm index + 1.
__global__ void k_point_weights(const double* __restrict__ norms, size_t n, DevWeights w,
                                double* __restrict__ hp, double* __restrict__ ho,
                                double* __restrict__ coef, unsigned long long* flags,
                                DevError* err) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a, b;
  int st = AQ_OK;
  if (!resolve_weights(w, i, norms[i], &a, &b, &st)) {
    report_error(err, i, st);
    a = b = 1.0;
  }
  hp[i] = a;
  ho[i] = b;
  double c = 0.0;
  bool zero = false;
  if (a != b) {
    const double n2 = __dmul_rn(norms[i], norms[i]);
    zero = n2 == 0.0;
    if (!zero) c = __ddiv_rn(__dsub_rn(a, b), n2);
  }
  coef[i] = c;
  // one atomic per warp (a per-point atomicOr on one word serialises n
  // updates: 6.5 ms at n = 1e7)
  const unsigned act = __activemask();
  const unsigned aniso = __ballot_sync(act, a != b);
  const int leader = __ffs(act) - 1;
  if (aniso && (int)(threadIdx.x & 31) == leader) atomicOr(&flags[0], 1ull);
  if (zero) atomicMin(&flags[1], (unsigned long long)i + 1ull);
}

// ---- dense normal equations ---------------------------------------------------------------

struct AsmArgs {
  const float* xr;  // float32 rows (every kernel), or null with xr64 set
  const double* xr64;  // float64 rows (k_assemble<double> only)
  size_t n;
  int d, M, k, sd;
  const uint8_t* codes;
  int stride, bits;
  const uint32_t* list;
  const uint32_t* start;
  const uint32_t* count;
  const double* hp;
  const double* ho;
  const double* coef;
  int full;        // 1: all column subspaces (API), 0: m2 <= m (lower, for LLT)
  double* A;       // dim x dim row-major
  double* rhs;     // dim
  int nchunk;      // column chunks of 32 subspaces per strip
  uint32_t lo, hi; // point-index block processed by this launch
  int resume;      // 1: accumulators continue from A / rhs (not the first block)
};

// first position in the ascending list L[0..cnt) with L[pos] >= v
__device__ __forceinline__ size_t lower_bound_u32(const uint32_t* L, size_t cnt, uint32_t v) {
  size_t lo = 0, hi = cnt;
  while (lo < hi) {
    const size_t mid = (lo + hi) >> 1;
    if (L[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One warp = (row strip (m, j), chunk of 32 column subspaces). Lane l owns
// column subspace m2 = 32 chunk + l; its accumulators for rows (m, j, a) x
// columns (m2, j2, b) sit in shared memory, lane-interleaved (no bank
// conflicts, no atomics). The strip's points are visited in ascending order,
// so each entry sees the reference's exact sequence of additions
// (pq.hpp:320-339): += h_perp on the diagonal first, then += (coef x_a) x_b.
// Points are staged 32 at a time (list entries, per-point scalars and every
// lane's column sub-vector / code) so the global gathers of a batch are
// independent and in flight together.
constexpr int kAsmSdMax = 4;
template <class TX>
__device__ __forceinline__ const TX* asm_rows(const AsmArgs& a);
template <>
__device__ __forceinline__ const float* asm_rows<float>(const AsmArgs& a) { return a.xr; }
template <>
__device__ __forceinline__ const double* asm_rows<double>(const AsmArgs& a) { return a.xr64; }

template <class TX>
__global__ void __launch_bounds__(32) k_assemble(const AsmArgs a) {
  extern __shared__ __align__(16) double acc[];  // [(aa*k + j2)*sd + b][32], rhs[sd]
  __shared__ double s_coef[32], s_ho[32], s_hp[32];
  __shared__ TX s_xm[32][kAsmSdMax];
  __shared__ TX s_xc[32][kAsmSdMax][33];  // [point][b][lane] (+1 pad)
  const TX* __restrict__ xr = asm_rows<TX>(a);
  __shared__ unsigned char s_j2[32][32];
  const int unit = blockIdx.x;
  const int chunk = unit % a.nchunk;
  const int strip = unit / a.nchunk;
  const int m = strip / a.k, j = strip % a.k;
  const int lane = threadIdx.x;
  const int sd = a.sd, k = a.k, d = a.d;
  const int m2 = chunk * 32 + lane;
  const int mcols = a.full ? a.M : m + 1;
  if (chunk * 32 >= mcols) return;
  const bool mine = m2 < mcols;
  const int nacc = sd * k * sd;
  double* racc = acc + (size_t)nacc * 32;
  for (int e = 0; e < nacc; ++e) acc[e * 32 + lane] = 0.0;
  if (lane < sd) racc[lane] = 0.0;
  const uint32_t* L = a.list + (size_t)m * a.n + a.start[m * k + j];
  const size_t cnt = a.count[m * k + j];
  const bool do_rhs = chunk == 0;
  for (size_t t0 = 0; t0 < cnt; t0 += 32) {
    const int nb = (int)min((size_t)32, cnt - t0);
    // stage: lane l fetches point t0 + l's scalars and strip sub-vector ...
    uint32_t pl = 0;
    if (lane < nb) {
      pl = L[t0 + lane];
      s_coef[lane] = a.coef[pl];
      s_ho[lane] = a.ho[pl];
      s_hp[lane] = a.hp[pl];
      for (int c = 0; c < sd; ++c) s_xm[lane][c] = xr[(size_t)pl * d + m * sd + c];
    }
    // ... and, for every point of the batch, its own column sub-vector and code
    if (mine) {
#pragma unroll 8
      for (int b = 0; b < nb; ++b) {
        const uint32_t p = __shfl_sync(0xffffffffu, pl, b);
        const TX* xp = xr + (size_t)p * d + m2 * sd;
        for (int c = 0; c < sd; ++c) s_xc[b][c][lane] = xp[c];
        s_j2[b][lane] = (unsigned char)get_code(a.codes + (size_t)p * a.stride, m2, a.bits);
      }
    } else {
      for (int b = 0; b < nb; ++b) __shfl_sync(0xffffffffu, pl, b);
    }
    __syncwarp();
    for (int b = 0; b < nb; ++b) {
      if (do_rhs && lane < sd)  // rhs += h_par * x (pq.hpp:326)
        racc[lane] = __dadd_rn(racc[lane], __dmul_rn(s_hp[b], (double)s_xm[b][lane]));
      if (!mine) continue;
      const unsigned j2 = s_j2[b][lane];
      if (m2 == m) {  // diagonal h_perp (pq.hpp:324-325), j2 == j here
        const double hop = s_ho[b];
        for (int aa = 0; aa < sd; ++aa) {
          double* e = acc + (size_t)((aa * k + j) * sd + aa) * 32 + lane;
          *e = __dadd_rn(*e, hop);
        }
      }
      const double cf = s_coef[b];
      if (cf == 0.0) continue;  // pq.hpp:328
      for (int aa = 0; aa < sd; ++aa) {
        const double xc = __dmul_rn(cf, (double)s_xm[b][aa]);
        for (int c2 = 0; c2 < sd; ++c2) {
          double* e = acc + (size_t)((aa * k + j2) * sd + c2) * 32 + lane;
          *e = __dadd_rn(*e, __dmul_rn(xc, (double)s_xc[b][c2][lane]));
        }
      }
    }
    __syncwarp();
  }
  const size_t dim = (size_t)k * d;
  if (mine) {
    for (int aa = 0; aa < sd; ++aa)
      for (int j2 = 0; j2 < k; ++j2)
        for (int b = 0; b < sd; ++b)
          a.A[((size_t)(m * k + j) * sd + aa) * dim + (size_t)(m2 * k + j2) * sd + b] =
              acc[(size_t)((aa * k + j2) * sd + b) * 32 + lane];
  }
  if (do_rhs && lane < sd) a.rhs[(size_t)(m * k + j) * sd + lane] = racc[lane];
}

// Specialisation for sub_dimension 2, k = 16, 4-bit codes, d % 4 == 0 (all
// BASELINE configs). Same per-entry operation order as k_assemble, cheaper
// per (point, lane):
//   * per point, once (staging lane): u_a = coef * x_m[a] and h_par * x_m[a]
//     in float64 (the reference's products, pq.hpp:326, 332);
//   * the batch's column rows (32 subspaces = 256 B per point) and code
//     words (16 B) are copied with 16-byte cp.async, two points per warp
//     instruction;
//   * the diagonal h_perp (pq.hpp:324-325) is added inside the same
//     read-modify-write, before the point's coupling product;
//   * no coef == 0 branch (pq.hpp:328): then u = 0 and every product is a
//     signed zero, and adding a signed zero never changes an accumulator
//     (accumulators start at +0 and are never -0), so the result is the same.
// Units (strip x column chunk) run largest strip first (`order`).
__global__ void __launch_bounds__(32) k_assemble_sd2(const AsmArgs a, const uint32_t* order) {
  // [aa*16 + j2][lane] of {b = 0, b = 1}: a point's 2x2 block is two 16-byte
  // accesses per lane (LDS.128 / STS.128)
  extern __shared__ __align__(16) double2 acc2[];
  __shared__ __align__(16) double2 s_u[32];      // coef * x_m
  __shared__ __align__(16) double2 s_r[32];      // h_par * x_m (rhs)
  __shared__ double s_ho[32];
  __shared__ __align__(16) float s_x[2][32][64];    // [buffer][point][column float]
  __shared__ __align__(16) uint32_t s_cw[2][32][4]; // [buffer][point][code word of lane >> 3]
  const int unit = order[blockIdx.x];
  const int chunk = unit % a.nchunk;
  const int strip = unit / a.nchunk;
  const int m = strip >> 4, j = strip & 15;
  const int lane = threadIdx.x;
  const int d = a.d;
  const int m2 = chunk * 32 + lane;
  const int mcols = a.full ? a.M : m + 1;
  const bool mine = m2 < mcols;
  const bool diag = m2 == m;
  const size_t dim = (size_t)16 * d;
  const bool do_rhs = chunk == 0 && lane == 0;
  const uint32_t* Lall = a.list + (size_t)m * a.n + a.start[m * 16 + j];
  const size_t call = a.count[m * 16 + j];
  const size_t t_lo = lower_bound_u32(Lall, call, a.lo);
  const size_t t_hi = lower_bound_u32(Lall, call, a.hi);
  if (t_lo == t_hi) return;  // accumulators already hold this block's state
  double r0 = 0.0, r1 = 0.0;
  if (a.resume) {
    if (mine) {
#pragma unroll 4
      for (int e = 0; e < 64; ++e) {
        const int aa = e >> 5, j2 = (e >> 1) & 15, b = e & 1;
        reinterpret_cast<double*>(acc2)[((e >> 1) * 32 + lane) * 2 + b] =
            a.A[((size_t)(m * 16 + j) * 2 + aa) * dim + (size_t)(m2 * 16 + j2) * 2 + b];
      }
    }
    if (do_rhs) {
      r0 = a.rhs[(size_t)(m * 16 + j) * 2];
      r1 = a.rhs[(size_t)(m * 16 + j) * 2 + 1];
    }
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e) acc2[e * 32 + lane] = make_double2(0.0, 0.0);
  }
  const uint32_t* L = Lall + t_lo;
  const size_t cnt = t_hi - t_lo;
  const int col0 = chunk * 64;                       // first float of the chunk's columns
  const int nf4 = min(16, (d - col0) >> 2);          // valid float4 per point row
  const int cb0 = chunk * 16;                        // first code byte of the chunk
  const int ncb = min(2, max(0, (a.stride - cb0) >> 3));  // valid 8-byte code slices
  const unsigned sx = (unsigned)__cvta_generic_to_shared(&s_x[0][0][0]);
  const unsigned sc = (unsigned)__cvta_generic_to_shared(&s_cw[0][0][0]);
  // batch t's rows and code words -> buffer t & 1 (cp.async, one group)
  auto issue_rows = [&](uint32_t pl, int nb, int buf) {
#pragma unroll 4
    for (int it = 0; it < 16; ++it) {
      const int idx = it * 32 + lane;
      const int b = idx >> 4, f = idx & 15;
      const uint32_t p = __shfl_sync(0xffffffffu, pl, b);
      if (b < nb && f < nf4) {
        const float* src = a.xr + (size_t)p * d + col0 + f * 4;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                         sx + (unsigned)((buf * 32 + b) * 64 + f * 4) * 4u),
                     "l"(src));
      }
    }
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int idx = it * 32 + lane;
      const int b = idx >> 1, h = idx & 1;
      const uint32_t p = __shfl_sync(0xffffffffu, pl, b);
      if (b < nb && h < ncb) {
        const uint8_t* src = a.codes + (size_t)p * a.stride + cb0 + h * 8;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                         sc + (unsigned)((buf * 32 + b) * 16 + h * 8)),
                     "l"(src));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // per-point scalars of a batch, into registers (lane = point)
  uint32_t pl = 0;
  double cf = 0.0, hp = 0.0, ho = 0.0;
  float2 xm = make_float2(0.f, 0.f);
  // h_par feeds only the rhs (chunk 0) and h_perp only the diagonal lane:
  // other units skip those gathers (each a 32-line access per warp, on the
  // L1 pipe the kernel is bound by)
  const bool need_hp = chunk == 0, need_ho = m >= chunk * 32 && m < chunk * 32 + 32;
  auto load_scalars = [&](size_t t0, int nb) {
    if (lane < nb) {
      pl = L[t0 + lane];
      cf = a.coef[pl];
      if (need_hp) hp = a.hp[pl];
      if (need_ho) ho = a.ho[pl];
      xm = *reinterpret_cast<const float2*>(a.xr + (size_t)pl * d + m * 2);
    }
  };
  int nb = (int)min((size_t)32, cnt);
  load_scalars(0, nb);
  issue_rows(pl, nb, 0);
  int buf = 0;
  for (size_t t0 = 0; t0 < cnt; t0 += 32) {
    // this batch's products into shared memory (lane = point)
    if (lane < nb) {
      s_u[lane] = make_double2(__dmul_rn(cf, (double)xm.x), __dmul_rn(cf, (double)xm.y));
      s_r[lane] = make_double2(__dmul_rn(hp, (double)xm.x), __dmul_rn(hp, (double)xm.y));
      s_ho[lane] = ho;
    }
    // next batch: scalars and rows in flight while this batch computes
    const size_t t1 = t0 + 32;
    const int nbn = t1 < cnt ? (int)min((size_t)32, cnt - t1) : 0;
    if (nbn) {
      load_scalars(t1, nbn);
      issue_rows(pl, nbn, buf ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncwarp();
    if (do_rhs)  // rhs += h_par * x (pq.hpp:326)
      for (int b = 0; b < nb; ++b) {
        const double2 r = s_r[b];
        r0 = __dadd_rn(r0, r.x);
        r1 = __dadd_rn(r1, r.y);
      }
    if (mine) {
      const int wsel = lane >> 3, sh = 4 * (lane & 7);
      // One point: h_perp on the diagonal first (pq.hpp:324-325; j2 == j
      // there), then the coupling products (pq.hpp:329-338).
      auto upd = [&](int b, double2& A0, double2& A1) {
        const double2 u = s_u[b];
        const float2 xc = *reinterpret_cast<const float2*>(&s_x[buf][b][lane * 2]);
        const double v0 = (double)xc.x, v1 = (double)xc.y;
        if (diag) {
          const double hop = s_ho[b];
          A0.x = __dadd_rn(A0.x, hop);
          A1.y = __dadd_rn(A1.y, hop);
        }
        A0.x = __dadd_rn(A0.x, __dmul_rn(u.x, v0));
        A0.y = __dadd_rn(A0.y, __dmul_rn(u.x, v1));
        A1.x = __dadd_rn(A1.x, __dmul_rn(u.y, v0));
        A1.y = __dadd_rn(A1.y, __dmul_rn(u.y, v1));
      };
      auto slot = [&](int b) { return (s_cw[buf][b][wsel] >> sh) & 15u; };
      // Points in pairs: both slots are loaded before either is stored; when
      // the pair shares a slot the second update continues from the first's
      // result, and the second store (program order) leaves the chained value.
      int b = 0;
      for (; b + 1 < nb; b += 2) {
        const unsigned ja = slot(b), jb = slot(b + 1);
        double2 A0 = acc2[ja * 32 + lane], A1 = acc2[(16 + ja) * 32 + lane];
        double2 B0 = acc2[jb * 32 + lane], B1 = acc2[(16 + jb) * 32 + lane];
        upd(b, A0, A1);
        if (ja == jb) {
          B0 = A0;
          B1 = A1;
        }
        upd(b + 1, B0, B1);
        acc2[ja * 32 + lane] = A0;
        acc2[(16 + ja) * 32 + lane] = A1;
        acc2[jb * 32 + lane] = B0;
        acc2[(16 + jb) * 32 + lane] = B1;
      }
      if (b < nb) {
        const unsigned ja = slot(b);
        double2 A0 = acc2[ja * 32 + lane], A1 = acc2[(16 + ja) * 32 + lane];
        upd(b, A0, A1);
        acc2[ja * 32 + lane] = A0;
        acc2[(16 + ja) * 32 + lane] = A1;
      }
    }
    __syncwarp();
    nb = nbn;
    buf ^= 1;
  }
  if (mine) {
#pragma unroll 4
    for (int e = 0; e < 64; ++e) {
      const int aa = e >> 5, j2 = (e >> 1) & 15, b = e & 1;
      a.A[((size_t)(m * 16 + j) * 2 + aa) * dim + (size_t)(m2 * 16 + j2) * 2 + b] =
          reinterpret_cast<const double*>(acc2)[((e >> 1) * 32 + lane) * 2 + b];
    }
  }
  if (do_rhs) {
    a.rhs[(size_t)(m * 16 + j) * 2] = r0;
    a.rhs[(size_t)(m * 16 + j) * 2 + 1] = r1;
  }
}

// Register-pipelined variant of k_assemble_sd2: no row staging in shared
// memory. Each lane loads its own column pair (float2) and code word for the
// point AH positions ahead straight from global memory (the warp reads the
// point's 256-byte column slice, coalesced) into a register ring, so a CTA
// holds only the 16 KB accumulator tile and twice as many warps fit per SM.
// Per-entry operation order is the same as k_assemble_sd2's.
template <int AH>
__global__ void __launch_bounds__(32, 12) k_assemble_sd2r(const AsmArgs a, const uint32_t* order) {
  static_assert(AH == 8 || AH == 16, "ring of 8 or 16 points");
  // [aa*16 + j2][lane] of {b = 0, b = 1}: a point's 2x2 block is two
  // 16-byte accesses per lane (LDS.128 / STS.128)
  extern __shared__ __align__(16) double2 acc2[];
  __shared__ __align__(16) double2 s_u[32];      // coef * x_m
  __shared__ __align__(16) double2 s_r[32];      // h_par * x_m (rhs)
  __shared__ double s_ho[32];
  const int unit = order[blockIdx.x];
  const int chunk = unit % a.nchunk;
  const int strip = unit / a.nchunk;
  const int m = strip >> 4, j = strip & 15;
  const int lane = threadIdx.x;
  const int d = a.d;
  const int m2 = chunk * 32 + lane;
  const int mcols = a.full ? a.M : m + 1;
  const bool mine = m2 < mcols;
  const bool diag = m2 == m;
  const size_t dim = (size_t)16 * d;
  const bool do_rhs = chunk == 0 && lane == 0;
  const uint32_t* Lall = a.list + (size_t)m * a.n + a.start[m * 16 + j];
  const size_t call = a.count[m * 16 + j];
  const size_t t_lo = lower_bound_u32(Lall, call, a.lo);
  const size_t t_hi = lower_bound_u32(Lall, call, a.hi);
  if (t_lo == t_hi) return;  // accumulators already hold this block's state
  double r0 = 0.0, r1 = 0.0;
  if (a.resume) {
    if (mine) {
#pragma unroll 4
      for (int e = 0; e < 64; ++e) {
        const int aa = e >> 5, j2 = (e >> 1) & 15, b = e & 1;
        reinterpret_cast<double*>(acc2)[((e >> 1) * 32 + lane) * 2 + b] =
            a.A[((size_t)(m * 16 + j) * 2 + aa) * dim + (size_t)(m2 * 16 + j2) * 2 + b];
      }
    }
    if (do_rhs) {
      r0 = a.rhs[(size_t)(m * 16 + j) * 2];
      r1 = a.rhs[(size_t)(m * 16 + j) * 2 + 1];
    }
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e) acc2[e * 32 + lane] = make_double2(0.0, 0.0);
  }
  const uint32_t* L = Lall + t_lo;
  const size_t cnt = t_hi - t_lo;
  const float* xcol = a.xr + chunk * 64 + 2 * lane;  // this lane's column pair
  const uint8_t* cwb = a.codes + chunk * 16 + (lane >> 3) * 4;
  const int sh = 4 * (lane & 7);
  // batch scalars, lane = point of the batch: current (c) and next (n)
  uint32_t plc = 0, pln = 0;
  double cfc = 0.0, hpc = 0.0, hoc = 0.0, cfn = 0.0, hpn = 0.0, hon = 0.0;
  float2 xmc = make_float2(0.f, 0.f), xmn = make_float2(0.f, 0.f);
  // h_par feeds only the rhs (chunk 0) and h_perp only the diagonal lane
  const bool need_hp = chunk == 0, need_ho = m >= chunk * 32 && m < chunk * 32 + 32;
  auto load_scalars = [&](size_t t0, uint32_t& pl, double& cf, double& hp, double& ho,
                          float2& xm) {
    if (t0 + lane < cnt) {
      pl = L[t0 + lane];
      cf = a.coef[pl];
      if (need_hp) hp = a.hp[pl];
      if (need_ho) ho = a.ho[pl];
      xm = *reinterpret_cast<const float2*>(a.xr + (size_t)pl * d + m * 2);
    }
  };
  float2 rx[AH];
  uint32_t rw[AH];
  auto fetch = [&](uint32_t p, float2& x, uint32_t& w) {
    if (mine) {
      x = __ldg(reinterpret_cast<const float2*>(xcol + (size_t)p * d));
      w = __ldg(reinterpret_cast<const uint32_t*>(cwb + (size_t)p * a.stride));
    }
  };
  load_scalars(0, plc, cfc, hpc, hoc, xmc);
  load_scalars(32, pln, cfn, hpn, hon, xmn);
#pragma unroll
  for (int v = 0; v < AH; ++v) {
    rx[v] = make_float2(0.f, 0.f);
    rw[v] = 0u;
    const uint32_t p = __shfl_sync(0xffffffffu, plc, v);
    if ((size_t)v < cnt) fetch(p, rx[v], rw[v]);
  }
  for (size_t t0 = 0; t0 < cnt; t0 += 32) {
    const int nb = (int)min((size_t)32, cnt - t0);
    if (lane < nb) {
      s_u[lane] = make_double2(__dmul_rn(cfc, (double)xmc.x), __dmul_rn(cfc, (double)xmc.y));
      s_r[lane] = make_double2(__dmul_rn(hpc, (double)xmc.x), __dmul_rn(hpc, (double)xmc.y));
      s_ho[lane] = hoc;
    }
    __syncwarp();
    if (do_rhs)
      for (int b = 0; b < nb; ++b) {  // rhs += h_par * x (pq.hpp:326)
        const double2 r = s_r[b];
        r0 = __dadd_rn(r0, r.x);
        r1 = __dadd_rn(r1, r.y);
      }
    // h_perp on the diagonal first (pq.hpp:324-325), then the coupling
    // products (pq.hpp:329-338)
    auto upd = [&](int b, float2 xc, double& e00, double& e01, double& e10, double& e11) {
      const double2 u = s_u[b];
      const double v0 = (double)xc.x, v1 = (double)xc.y;
      if (diag) {
        const double hop = s_ho[b];
        e00 = __dadd_rn(e00, hop);
        e11 = __dadd_rn(e11, hop);
      }
      e00 = __dadd_rn(e00, __dmul_rn(u.x, v0));
      e01 = __dadd_rn(e01, __dmul_rn(u.x, v1));
      e10 = __dadd_rn(e10, __dmul_rn(u.y, v0));
      e11 = __dadd_rn(e11, __dmul_rn(u.y, v1));
    };
#pragma unroll
    for (int g = 0; g < 32 / AH; ++g) {
      if (g * AH >= nb) break;
#pragma unroll
      for (int v = 0; v < AH; v += 2) {
        const int b = g * AH + v;
        if (mine && b < nb) {
          // pair (b, b + 1): both slots loaded before either is stored; a
          // shared slot chains the second update on the first's result
          const unsigned ja = (rw[v] >> sh) & 15u;
          double2* pa0 = acc2 + (size_t)ja * 32 + lane;
          double2* pa1 = acc2 + (size_t)(16 + ja) * 32 + lane;
          double2 A0 = *pa0, A1 = *pa1;
          if (b + 1 < nb) {
            const unsigned jb = (rw[v + 1] >> sh) & 15u;
            double2* pb0 = acc2 + (size_t)jb * 32 + lane;
            double2* pb1 = acc2 + (size_t)(16 + jb) * 32 + lane;
            double2 B0 = *pb0, B1 = *pb1;
            upd(b, rx[v], A0.x, A0.y, A1.x, A1.y);
            if (ja == jb) {
              B0 = A0;
              B1 = A1;
            }
            upd(b + 1, rx[v + 1], B0.x, B0.y, B1.x, B1.y);
            *pa0 = A0;
            *pa1 = A1;
            *pb0 = B0;
            *pb1 = B1;
          } else {
            upd(b, rx[v], A0.x, A0.y, A1.x, A1.y);
            *pa0 = A0;
            *pa1 = A1;
          }
        }
        // refill both slots with the points AH positions ahead
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int tn = b + q + AH;  // < 32: this batch, else the next
          const uint32_t p = __shfl_sync(0xffffffffu, tn < 32 ? plc : pln, tn & 31);
          if (t0 + tn < cnt) fetch(p, rx[v + q], rw[v + q]);
        }
      }
    }
    __syncwarp();
    plc = pln;
    cfc = cfn;
    hpc = hpn;
    hoc = hon;
    xmc = xmn;
    load_scalars(t0 + 64, pln, cfn, hpn, hon, xmn);
  }
  if (mine) {
#pragma unroll 4
    for (int e = 0; e < 64; ++e) {
      const int aa = e >> 5, j2 = (e >> 1) & 15, b = e & 1;
      a.A[((size_t)(m * 16 + j) * 2 + aa) * dim + (size_t)(m2 * 16 + j2) * 2 + b] =
          reinterpret_cast<const double*>(acc2)[((e >> 1) * 32 + lane) * 2 + b];
    }
  }
  if (do_rhs) {
    a.rhs[(size_t)(m * 16 + j) * 2] = r0;
    a.rhs[(size_t)(m * 16 + j) * 2 + 1] = r1;
  }
}

// trace (sequential, Eigen stand-in) and ridge = 1e-6 trace / dim (pq.hpp:431-435)
__global__ void k_trace_ridge(double* A, size_t dim, double ridge) {
  __shared__ double r;
  __shared__ double diag[4096];  // the diagonal gathered in parallel (dim <= 16384: chunks)
  double tr = 0.0;
  for (size_t c0 = 0; c0 < dim; c0 += 4096) {
    const size_t cn = min((size_t)4096, dim - c0);
    for (size_t i = threadIdx.x; i < cn; i += blockDim.x) diag[i] = A[(c0 + i) * dim + c0 + i];
    __syncthreads();
    if (threadIdx.x == 0)  // the sum itself stays sequential (index order)
      for (size_t i = 0; i < cn; ++i) tr = __dadd_rn(tr, diag[i]);
    __syncthreads();
  }
  if (threadIdx.x == 0) r = ridge < 0.0 ? __ddiv_rn(__dmul_rn(1e-6, tr), (double)dim) : ridge;
  __syncthreads();
  for (size_t i = threadIdx.x; i < dim; i += blockDim.x)
    A[i * dim + i] = __dadd_rn(A[i * dim + i], r);
}

int trace_ridge_device(aq_session* s, double* A, size_t dim, double ridge) {
  k_trace_ridge<<<1, 1024, 0, s->stream>>>(A, dim, ridge);
  AQ_LAUNCHED(s);
  return AQ_OK;
}

// ---- blocked Cholesky (lower, in place, row-major) --------------------------------------

// Panel of block [kb, be) (stand-in factor(), oracle/eigen_subset): every
// entry (i, j) of the block's columns takes its subtractions L(i,k) L(j,k) in
// ascending k, then the division by L(j,j) = sqrt(...). The same arithmetic is
// scheduled right-looking: once column k is final, each later entry of a row
// subtracts its term k, so the independent entries of a row advance together
// instead of one ordered chain per column. Every CTA factors the 64 x 64
// diagonal block (redundantly) while it solves its own rows below the block,
// column by column in lockstep: the square root, the divisions of column c,
// then every row's later entries (two threads per row). A fully unrolled
// register-resident variant (one thread per row, 160 registers) measured 2x
// slower: its ~160 KB of straight-line code thrashed the instruction cache.
// Global -> shared staging with eight loads in flight per thread: a plain
// element loop waits out a full memory round trip per element (the load
// feeds the store of the same iteration), which dominated these kernels.
// f(e) returns the value of element e (a global load or 0), g(e, v) stores it.
template <class F, class G>
__device__ __forceinline__ void stage8(int count, F f, G g) {
  for (int e0 = threadIdx.x; e0 < count; e0 += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      v[u] = e < count ? f(e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < count) g(e, v[u]);
    }
  }
}

// rows below the diagonal block per CTA: few, so that many CTAs share a
// panel (each also carries the 64 diagonal-block rows)
constexpr int kPanelRows = 16;
constexpr int kPanelThreads = 2 * (kLLT + kPanelRows);

// row[j] -= lic * D[j][c] for j = j0, j0 + step, ... < jend: the loads of a
// batch of 8 are issued before its stores (shared-memory stores would
// otherwise serialise against every later load: the rows may alias)
template <int STEP>
__device__ __forceinline__ void panel_axpy(double* row, const double (*D)[kLLT + 1], int c,
                                           double lic, int j0, int jend) {
  for (int j = j0; j < jend; j += 8 * STEP) {
    double rv[8], dv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int jj = j + u * STEP;
      rv[u] = jj < jend ? row[jj] : 0.0;
      dv[u] = jj < jend ? D[jj][c] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int jj = j + u * STEP;
      if (jj < jend) row[jj] = __dsub_rn(rv[u], __dmul_rn(lic, dv[u]));
    }
  }
}

__global__ void __launch_bounds__(kPanelThreads) k_llt_panel(double* A, int n, int kb, int* fail) {
  extern __shared__ __align__(16) double psm[];  // D[kLLT][kLLT + 1], R[kPanelRows][kLLT + 1]
  double(*D)[kLLT + 1] = reinterpret_cast<double(*)[kLLT + 1]>(psm);
  double(*R)[kLLT + 1] = reinterpret_cast<double(*)[kLLT + 1]>(psm + kLLT * (kLLT + 1));
  const int be = min(kb + kLLT, n), bs = be - kb;
  const int t = threadIdx.x;
  const int r0 = be + blockIdx.x * kPanelRows;
  const int nr = max(0, min(n, r0 + kPanelRows) - r0);
  stage8(
      bs * bs,
      [&](int e) {
        const int r = e / bs, c = e % bs;
        return c <= r ? A[(size_t)(kb + r) * n + kb + c] : 0.0;
      },
      [&](int e, double v) { D[e / bs][e % bs] = v; });
  stage8(
      nr * bs, [&](int e) { return A[(size_t)(r0 + e / bs) * n + kb + e % bs]; },
      [&](int e, double v) { R[e / bs][e % bs] = v; });
  __syncthreads();
  {
    // rows 0..bs-1: the diagonal block; bs..bs+nr-1: this CTA's panel rows;
    // two threads per row (thread q takes the columns j = q mod 2)
    const int r = t >> 1, q = t & 1;
    const int nrows = bs + nr;
    double* row = r < bs ? D[r] : R[min(r - bs, kPanelRows - 1)];
    const int jend = r < bs ? r + 1 : bs;  // diagonal rows stop at the diagonal
    // the square root of column c + 1 is taken by the thread that gives its
    // diagonal entry the last subtraction (column c's update), while the
    // other rows still update: two barriers per column
    auto pivot = [&](int c) {
      const double sv = D[c][c];
      if (sv <= 0.0) atomicExch(fail, 1);
      D[c][c] = __dsqrt_rn(sv);
    };
    if (t == 0 && bs > 0) pivot(0);
    __syncthreads();
    for (int c = 0; c < bs; ++c) {
      if (r > c && r < nrows && q == 0) row[c] = __ddiv_rn(row[c], D[c][c]);
      __syncthreads();
      if (r > c && r < nrows) panel_axpy<2>(row, D, c, row[c], c + 1 + ((q - c - 1) & 1), jend);
      if (r == c + 1 && r < bs && q == (r & 1)) pivot(r);
      __syncthreads();
    }
  }

  if (blockIdx.x == 0)
    for (int e = t; e < bs * bs; e += blockDim.x) {
      const int r = e / bs, c = e % bs;
      if (c <= r) A[(size_t)(kb + r) * n + kb + c] = D[r][c];
    }
  for (int e = t; e < nr * bs; e += blockDim.x) {
    const int r = e / bs, c = e % bs;
    A[(size_t)(r0 + r) * n + kb + c] = R[r][c];
  }
}

// Trailing update of the lower triangle: L[i][c] -= sum_{q in block} L[i][q] L[c][q]
// (sum sequential in q from 0.0, then one subtraction). 64 x 64 tiles.
// The panel slices are staged transposed with a row stride of 65 doubles:
// a warp's transposed stores (one row, 32 consecutive q) then fall in 16
// distinct bank pairs instead of one, and a full block (bs = 64) indexes by
// shifts instead of integer division.
constexpr int kTrailStride = kLLT + 1;
__global__ void __launch_bounds__(256) k_llt_trail(double* A, int n, int kb) {
  extern __shared__ __align__(16) double tsm[];
  // transposed panel slices: Pi[q][r] = L(i0 + r, kb + q), Pc[q][r] = L(c0 + r, kb + q)
  double(*Pi)[kTrailStride] = reinterpret_cast<double(*)[kTrailStride]>(tsm);
  double(*Pc)[kTrailStride] = reinterpret_cast<double(*)[kTrailStride]>(tsm + 64 * kTrailStride);
  const int be = min(kb + kLLT, n), bs = be - kb;
  // triangular tile index -> (ti, tc), tc <= ti
  const int tile = blockIdx.x;
  int ti = (int)((sqrt(8.0 * tile + 1.0) - 1.0) / 2.0);
  while ((ti + 1) * (ti + 2) / 2 <= tile) ++ti;
  while (ti * (ti + 1) / 2 > tile) --ti;
  const int tc = tile - ti * (ti + 1) / 2;
  const int i0 = be + ti * 64, c0 = be + tc * 64;
  const bool full = bs == kLLT;
  auto stage = [&](int r0, double(*P)[kTrailStride]) {
    stage8(
        64 * bs,
        [&](int e) {
          const int r = full ? e >> 6 : e / bs, q = full ? e & 63 : e % bs;
          return r0 + r < n ? A[(size_t)(r0 + r) * n + kb + q] : 0.0;
        },
        [&](int e, double v) {
          const int r = full ? e >> 6 : e / bs, q = full ? e & 63 : e % bs;
          P[q][r] = v;
        });
  };
  stage(i0, Pi);
  stage(c0, Pc);
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double s[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) s[u][v] = 0.0;
  for (int q = 0; q < bs; ++q) {
    double pi[4], pc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pi[u] = Pi[q][ty * 4 + u];
      pc[u] = Pc[q][tx * 4 + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) s[u][v] = __dadd_rn(s[u][v], __dmul_rn(pi[u], pc[v]));
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = i0 + ty * 4 + u, c = c0 + tx * 4 + v;
      if (i < n && c <= i) {
        double* e = A + (size_t)i * n + c;
        *e = __dsub_rn(*e, s[u][v]);
      }
    }
}

// LLT solve (forward L y = b, backward L^T x = y), blocked like the stand-in
// (oracle/eigen_subset/Eigen/Dense, solve), one launch per block and
// direction. Every CTA loads the block's diagonal triangle and redundantly
// solves it (warp 0), then updates its own rows outside the block:
//  forward  diagonal: y(i) = (y(i) - L(i,kb) y(kb) - ... - L(i,i-1) y(i-1)) /
//           L(i,i), subtractions in ascending k — scheduled right-looking
//           (lane i subtracts term c as soon as y(c) is final);
//           rows below: s = sum_k L(i,k) y(k) in k order from 0.0, y(i) -= s;
//  backward diagonal: x(i) = (x(i) - L(i+1,i) x(i+1) - ... ) / L(i,i) in
//           ascending k — one ordered chain (its first term needs x(i + 1),
//           the last value solved), lanes forming the rounded products;
//           rows above: s = sum_k L(k,i) x(k) in k order, x(i) -= s.
constexpr int kSolveRows = 256;  // rows outside the block per CTA (one per thread)
__global__ void __launch_bounds__(256) k_llt_fwd(const double* L, int n, int kb, double* x) {
  __shared__ double Ld[kLLT][kLLT + 1];
  __shared__ double yb[kLLT];
  const int be = min(kb + kLLT, n), bs = be - kb;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  stage8(
      bs * bs,
      [&](int e) {
        const int r = e / bs, c = e % bs;
        return c <= r ? __ldg(L + (size_t)(kb + r) * n + kb + c) : 0.0;
      },
      [&](int e, double v) { Ld[e / bs][e % bs] = v; });
  __syncthreads();
  if (w == 0) {
    double ti[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) ti[h] = lane + 32 * h < bs ? x[kb + lane + 32 * h] : 0.0;
    for (int c = 0; c < bs; ++c) {
      double yc = 0.0;
      if (lane == (c & 31)) {
        yc = __ddiv_rn(c < 32 ? ti[0] : ti[1], Ld[c][c]);
        yb[c] = yc;
      }
      yc = __shfl_sync(0xffffffffu, yc, c & 31);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        if (i > c && i < bs) ti[h] = __dsub_rn(ti[h], __dmul_rn(Ld[i][c], yc));
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && t < bs) x[kb + t] = yb[t];
  // rows below: one thread per row (its 512-byte row segment streams
  // through L1)
  const int i = be + blockIdx.x * kSolveRows + t;
  if (i < n) {
    const double* Li = L + (size_t)i * n + kb;
    double sum = 0.0;
    for (int q0 = 0; q0 < bs; q0 += 8) {  // a batch of loads in flight per step
      double lv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) lv[u] = q0 + u < bs ? __ldg(Li + q0 + u) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q0 + u < bs) sum = __dadd_rn(sum, __dmul_rn(lv[u], yb[q0 + u]));
    }
    x[i] = __dsub_rn(x[i], sum);
  }
}

__global__ void __launch_bounds__(256) k_llt_bwd(const double* L, int n, int kb, double* x) {
  __shared__ double Ld[kLLT][kLLT + 1];
  __shared__ double xb[kLLT];
  __shared__ double pr[kLLT];
  const int be = min(kb + kLLT, n), bs = be - kb;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  stage8(
      bs * bs,
      [&](int e) {
        const int r = e / bs, c = e % bs;
        return c <= r ? __ldg(L + (size_t)(kb + r) * n + kb + c) : 0.0;
      },
      [&](int e, double v) { Ld[e / bs][e % bs] = v; });
  if (t < bs) xb[t] = x[kb + t];
  __syncthreads();
  if (w == 0) {
    for (int r = bs - 1; r >= 0; --r) {
      for (int c = r + 1 + lane; c < bs; c += 32) pr[c] = __dmul_rn(Ld[c][r], xb[c]);
      __syncwarp();
      if (lane == 0) {
        double tv = xb[r];
        for (int c0 = r + 1; c0 < bs; c0 += 8) {  // loads off the subtraction chain
          double pv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) pv[u] = c0 + u < bs ? pr[c0 + u] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (c0 + u < bs) tv = __dsub_rn(tv, pv[u]);
        }
        xb[r] = __ddiv_rn(tv, Ld[r][r]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && t < bs) x[kb + t] = xb[t];
  const int i = blockIdx.x * kSolveRows + t;  // rows above the block
  if (i < kb) {
    double sum = 0.0;
    for (int q0 = 0; q0 < bs; q0 += 8) {  // a batch of loads in flight per step
      double lv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) lv[u] = q0 + u < bs ? __ldg(L + (size_t)(kb + q0 + u) * n + i) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (q0 + u < bs) sum = __dadd_rn(sum, __dmul_rn(lv[u], xb[q0 + u]));
    }
    x[i] = __dsub_rn(x[i], sum);
  }
}

// Whole forward / backward solve in one launch each: one CTA per 64-row
// block, taking its block index from a ticket (dispatch order), so a CTA only
// ever waits for blocks already running. A block applies the published
// blocks' updates in the stand-in's order (forward: blocks 0, 1, ..., r - 1;
// backward: nb - 1, ..., r + 1; each a from-zero ordered sum over the 64
// columns, then one subtraction), solves its diagonal triangle exactly as
// k_llt_fwd / k_llt_bwd, and publishes (x store, fence, release flag). The
// L tile of the next update is staged while the previous block is still
// solving, so the chain is one 64-term sum plus one triangle per block and
// there are no per-block launches.
__device__ __forceinline__ void flag_wait(const unsigned* f) {
  unsigned v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(f) : "memory");
    if (v) break;
    __nanosleep(20);
  }
}

template <bool FWD>
__global__ void __launch_bounds__(256) k_llt_flow(const double* L, int n, double* x, unsigned* sync) {
  extern __shared__ __align__(16) double fsm[];
  double(*Ld)[kLLT + 1] = reinterpret_cast<double(*)[kLLT + 1]>(fsm);
  double(*T)[kLLT + 1] = reinterpret_cast<double(*)[kLLT + 1]>(fsm + kLLT * (kLLT + 1));  // FWD: T[row][k]; BWD: T[k][row]
  __shared__ double xk[kLLT];
  __shared__ double xb[kLLT];
  __shared__ int s_r;
  const int nb = (n + kLLT - 1) / kLLT;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) s_r = (int)atomicAdd(sync, 1u);
  __syncthreads();
  const int bi = FWD ? s_r : nb - 1 - s_r;  // this CTA's block
  unsigned* ready = sync + 1;
  const int kb = bi * kLLT, be = min(kb + kLLT, n), bs = be - kb;
  stage8(
      bs * bs,
      [&](int e) {
        const int r = e / bs, c = e % bs;
        return c <= r ? __ldg(L + (size_t)(kb + r) * n + kb + c) : 0.0;
      },
      [&](int e, double v) { Ld[e / bs][e % bs] = v; });
  double xi = t < bs ? x[kb + t] : 0.0;
  // updates from the other blocks, in the stand-in's order
  for (int u = 0; u < (FWD ? bi : nb - 1 - bi); ++u) {
    const int ob = FWD ? u : nb - 1 - u;  // the published block
    const int ok = ob * kLLT, os = min(ok + kLLT, n) - ok;
    __syncthreads();  // T / xk of the previous update are consumed
    if (FWD)
      stage8(
          bs * os, [&](int e) { return __ldg(L + (size_t)(kb + e / os) * n + ok + e % os); },
          [&](int e, double v) { T[e / os][e % os] = v; });
    else
      stage8(
          os * bs, [&](int e) { return __ldg(L + (size_t)(ok + e / bs) * n + kb + e % bs); },
          [&](int e, double v) { T[e / bs][e % bs] = v; });
    if (t == 0) flag_wait(ready + ob);
    __syncthreads();
    if (t < os) xk[t] = __ldcg(x + ok + t);
    __syncthreads();
    if (t < bs) {
      double sum = 0.0;
      for (int q0 = 0; q0 < os; q0 += 8) {
        double lv[8], yv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          lv[q] = q0 + q < os ? (FWD ? T[t][q0 + q] : T[q0 + q][t]) : 0.0;
          yv[q] = q0 + q < os ? xk[q0 + q] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q0 + q < os) sum = __dadd_rn(sum, __dmul_rn(lv[q], yv[q]));
      }
      xi = __dsub_rn(xi, sum);
    }
  }
  if (t < bs) xb[t] = xi;
  __syncthreads();
  if (w == 0) {
    if (FWD) {
      double ti[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) ti[h] = lane + 32 * h < bs ? xb[lane + 32 * h] : 0.0;
      for (int c = 0; c < bs; ++c) {
        double yc = 0.0;
        if (lane == (c & 31)) {
          yc = __ddiv_rn(c < 32 ? ti[0] : ti[1], Ld[c][c]);
          xb[c] = yc;
        }
        yc = __shfl_sync(0xffffffffu, yc, c & 31);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = lane + 32 * h;
          if (i > c && i < bs) ti[h] = __dsub_rn(ti[h], __dmul_rn(Ld[i][c], yc));
        }
      }
    } else {
      // One ordered chain (the first term of row r needs x(r + 1), the value
      // just solved): lane 0 alone, the loads and products of each eight
      // terms issued ahead of their ascending subtractions (lanes 1..31
      // forming the next row's products in the other half of a divergent
      // branch only serialized with it: 86k -> ~70k cycles per block).
      if (lane == 0) {
        for (int r = bs - 1; r >= 0; --r) {
          double tv = xb[r];
          for (int c0 = r + 1; c0 < bs; c0 += 8) {
            double pv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              pv[u] = c0 + u < bs ? __dmul_rn(Ld[c0 + u][r], xb[c0 + u]) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (c0 + u < bs) tv = __dsub_rn(tv, pv[u]);
          }
          xb[r] = __ddiv_rn(tv, Ld[r][r]);
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (t < bs) x[kb + t] = xb[t];
  __threadfence();
  __syncthreads();
  if (t == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(ready + bi), "r"(1u) : "memory");
}

int llt_solve_device(aq_session* s, double* A, int n, double* x) {
  int* fail;
  void* p;
  const int nblk = (n + kLLT - 1) / kLLT;
  AQ_TRY(scratch(s, 4, 64 + 2 * (nblk + 1) * sizeof(unsigned), &p));
  fail = (int*)p;
  AQ_CUDA(cudaMemsetAsync(fail, 0, sizeof(int), s->stream));
  timer_mark(s, AQ_T_LLT);
  for (int kb = 0; kb < n; kb += kLLT) {
    const int be = std::min(kb + kLLT, n);
    const int below = n - be;
    const int ctas = std::max(1, (below + kPanelRows - 1) / kPanelRows);
    const int psmem = (kLLT + kPanelRows) * (kLLT + 1) * (int)sizeof(double);
    AQ_CUDA(cudaFuncSetAttribute(k_llt_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 psmem));
    k_llt_panel<<<ctas, kPanelThreads, psmem, s->stream>>>(A, n, kb, fail);
    AQ_LAUNCHED(s);
    if (below > 0) {
      const int T = (below + 63) / 64;
      const int tsmem = 2 * 64 * kTrailStride * (int)sizeof(double);
      AQ_CUDA(cudaFuncSetAttribute(k_llt_trail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   tsmem));
      k_llt_trail<<<T * (T + 1) / 2, 256, tsmem, s->stream>>>(A, n, kb);
      AQ_LAUNCHED(s);
    }
  }
  timer_mark(s, AQ_T_LLT);
  int hf = 0;
  AQ_CUDA(cudaMemcpyAsync(&hf, fail, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  if (hf) return ref_error(AQ_E_SINGULAR_SYSTEM, "joint codebook system is not positive definite");
  // AQ_LLT_SOLVE=1: one launch per block and direction (k_llt_fwd / k_llt_bwd)
  static const int solve_variant = getenv("AQ_LLT_SOLVE") ? atoi(getenv("AQ_LLT_SOLVE")) : 0;
  const int nb = (n + kLLT - 1) / kLLT;
  if (solve_variant == 0 && nb <= 4 * s->num_sms) {
    unsigned* sync = (unsigned*)((char*)p + 64);  // ticket + nb ready flags per direction
    AQ_CUDA(cudaMemsetAsync(sync, 0, 2 * (nb + 1) * sizeof(unsigned), s->stream));
    const int fsmem = 2 * kLLT * (kLLT + 1) * (int)sizeof(double);
    AQ_CUDA(cudaFuncSetAttribute(k_llt_flow<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem));
    AQ_CUDA(cudaFuncSetAttribute(k_llt_flow<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem));
    k_llt_flow<true><<<nb, 256, fsmem, s->stream>>>(A, n, x, sync);
    AQ_LAUNCHED(s);
    k_llt_flow<false><<<nb, 256, fsmem, s->stream>>>(A, n, x, sync + nb + 1);
    AQ_LAUNCHED(s);
    return AQ_OK;
  }
  for (int kb = 0; kb < n; kb += kLLT) {
    const int below = n - std::min(kb + kLLT, n);
    k_llt_fwd<<<std::max(1, (below + kSolveRows - 1) / kSolveRows), 256, 0, s->stream>>>(
        A, n, kb, x);
    AQ_LAUNCHED(s);
  }
  for (int kb = ((n - 1) / kLLT) * kLLT; kb >= 0; kb -= kLLT) {
    k_llt_bwd<<<std::max(1, (kb + kSolveRows - 1) / kSolveRows), 256, 0, s->stream>>>(
        A, n, kb, x);
    AQ_LAUNCHED(s);
  }
  return AQ_OK;
}

// ---- isotropic weighted means (pq.hpp:405-423) ------------------------------------------


// ---- M == 1: update_codeword per codeword (vq.hpp:139-192) -------------------------------
// One CTA per codeword j. Its members (points with code j, ascending) feed
// a d x d lower-triangle system: a(r, c) += (coef x_c) x_r (rankUpdate,
// column-wise), b += h_par x, diag = ridge + sum h_perp; every entry is a
// sequential chain over the members. Isotropic members only -> weighted mean.
// out: A[j] (d x d row-major, diagonal already += diag), rhs[j] (d), iso[j],
// mean path written straight to dict.
// coef[p] = (h_par - h_perp) / x.squaredNorm() (vq.hpp:178-181; the norm as a
// sequential sum of squares), NaN-free marker: n2 == 0 leaves coef = 0 and is
// reported by k_vq_systems.
template <class TX>
__global__ void k_vq_coef(const TX* __restrict__ xr, size_t n, int d,
                          const double* __restrict__ hp, const double* __restrict__ ho,
                          double* __restrict__ coef, double* __restrict__ n2out) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const TX* xp = xr + p * d;
  double n2 = 0.0;
  for (int q = 0; q < d; ++q) n2 = __dadd_rn(n2, __dmul_rn((double)xp[q], (double)xp[q]));
  n2out[p] = n2;
  coef[p] = n2 == 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(hp[p], ho[p]), n2);
}

template <class TX>
__global__ void k_vq_systems(const TX* __restrict__ xr, size_t n, int d, int k,
                             const uint32_t* __restrict__ list,
                             const uint32_t* __restrict__ start,
                             const uint32_t* __restrict__ count, const double* __restrict__ hp,
                             const double* __restrict__ ho, const double* __restrict__ coefs,
                             const double* __restrict__ n2s, double ridge, double* A,
                             double* rhs, int* mode, double* dict, DevError* err) {
  const int j = blockIdx.x;
  const size_t cnt = count[j];
  if (cnt == 0) return;
  const uint32_t* L = list + start[j];
  __shared__ int s_iso;
  __shared__ double s_diag;
  if (threadIdx.x == 0) {
    int iso = 1;
    for (size_t t = 0; t < cnt; ++t) iso &= hp[L[t]] == ho[L[t]];
    s_iso = iso;
    mode[j] = iso;
  }
  __syncthreads();
  if (s_iso) {  // weighted mean (vq.hpp:151-162)
    if (threadIdx.x == 0) {
      double den = 0.0;
      for (size_t t = 0; t < cnt; ++t) den = __dadd_rn(den, ho[L[t]]);
      s_diag = den;
      if (den <= 0.0) report_error(err, (uint64_t)j, AQ_E_SINGULAR_SYSTEM);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
      double s = 0.0;
      for (size_t t = 0; t < cnt; ++t)
        s = __dadd_rn(s, __dmul_rn(hp[L[t]], (double)xr[(size_t)L[t] * d + c]));
      if (s_diag > 0.0) dict[(size_t)j * d + c] = __ddiv_rn(s, s_diag);
    }
    return;
  }
  if (threadIdx.x == 0) {
    // mean_hperp, ridge_eff, diag (vq.hpp:165-186): sequential
    double mh = 0.0;
    for (size_t t = 0; t < cnt; ++t) mh = __dadd_rn(mh, ho[L[t]]);
    mh = __ddiv_rn(mh, (double)cnt);
    double diag = ridge < 0.0 ? __dmul_rn(1e-10, mh) : ridge;
    for (size_t t = 0; t < cnt; ++t) {
      if (n2s[L[t]] == 0.0) report_error(err, (uint64_t)L[t], AQ_E_ZERO_NORM_DATAPOINT);
      diag = __dadd_rn(diag, ho[L[t]]);
    }
    s_diag = diag;
  }
  __syncthreads();
  double* Aj = A + (size_t)j * d * d;
  const int ne = d * (d + 1) / 2;
  for (int e = threadIdx.x; e < ne + d; e += blockDim.x) {
    if (e < ne) {  // lower entry (r, c), r >= c
      int r = (int)((sqrt(8.0 * e + 1.0) - 1.0) / 2.0);
      while ((r + 1) * (r + 2) / 2 <= e) ++r;
      while (r * (r + 1) / 2 > e) --r;
      const int c = e - r * (r + 1) / 2;
      double v = 0.0;
      for (size_t t = 0; t < cnt; ++t) {
        const uint32_t p = L[t];
        const TX* xp = xr + (size_t)p * d;
        v = __dadd_rn(v, __dmul_rn(__dmul_rn(coefs[p], (double)xp[c]), (double)xp[r]));
      }
      if (r == c) v = __dadd_rn(v, s_diag);
      Aj[(size_t)r * d + c] = v;
    } else {  // rhs component
      const int c = e - ne;
      double v = 0.0;
      for (size_t t = 0; t < cnt; ++t)
        v = __dadd_rn(v, __dmul_rn(hp[L[t]], (double)xr[(size_t)L[t] * d + c]));
      rhs[(size_t)j * d + c] = v;
    }
  }
}

// unused-codeword reseeding: walk (m, j) lexicographically, consuming the
// loss ranking cyclically (pq.hpp:452-461)
template <class TX>
__global__ void k_reseed(const TX* xr, const uint32_t* count, int M, int k, int sd,
                         const uint32_t* order, size_t n, int d, double* dict) {
  size_t cursor = 0;
  for (int m = 0; m < M; ++m)
    for (int j = 0; j < k; ++j) {
      if (count[m * k + j] != 0) continue;
      const uint32_t p = order[cursor++ % n];
      for (int c = 0; c < sd; ++c)
        dict[((size_t)m * k + j) * sd + c] = (double)xr[(size_t)p * d + m * sd + c];
    }
}

__global__ void k_iota(uint32_t* v, size_t n) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) v[t] = (uint32_t)t;
}

int point_weights(aq_dataset* ds, const aq_weights* w, PointW* pw, void** owner) {
  aq_session* s = ds->s;
  const size_t n = ds->n;
  DevWeights dw;
  AQ_TRY(make_dev_weights(s, w, n, ds->d, &dw));
  double* buf;
  AQ_CUDA(cudaMallocAsync(&buf, (3 * n + 2) * sizeof(double), s->stream));
  *owner = buf;
  pw->hp = buf;
  pw->ho = buf + n;
  pw->coef = buf + 2 * n;
  unsigned long long* fl = (unsigned long long*)(buf + 3 * n);
  const unsigned long long init[2] = {0ull, ~0ull};
  AQ_CUDA(cudaMemcpyAsync(fl, init, sizeof init, cudaMemcpyHostToDevice, s->stream));
  AQ_TRY(clear_dev_error(s));
  if (n) {
    k_point_weights<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(
        ds->norms, n, dw, pw->hp, pw->ho, pw->coef, fl, s->err);
    AQ_LAUNCHED(s);
  }
  AQ_CUDA(cudaMemcpyAsync(pw->flags, fl, sizeof init, cudaMemcpyDeviceToHost, s->stream));
  AQ_TRY(sync_and_check(s, "weights"));
  return AQ_OK;
}

// Assembles the system into device buffers A (dim^2) and rhs (dim).
int assemble_device(aq_dataset* ds, aq_codes* codes, const PointW& pw, const Buckets& B,
                    int k, bool full, double* A, double* rhs) {
  aq_session* s = ds->s;
  const int M = (int)codes->M, d = (int)ds->d, sd = d / M;
  const size_t dim = (size_t)k * d;
  AQ_CUDA(cudaMemsetAsync(A, 0, dim * dim * sizeof(double), s->stream));
  AQ_CUDA(cudaMemsetAsync(rhs, 0, dim * sizeof(double), s->stream));
  const int nchunk = (M + 31) / 32;
  AsmArgs a{ds->xr, ds->xr64, ds->n, d, M, k, sd, codes->data, (int)codes->stride, codes->bits,
            B.list, B.start, B.count, pw.hp, pw.ho, pw.coef, full ? 1 : 0, A, rhs, nchunk,
            0u, (uint32_t)ds->n, 0};
  if (sd > kAsmSdMax)
    return ref_error(AQ_E_UNSUPPORTED, "device normal equations support sub_dimension <= 4");
  const size_t smem = ((size_t)sd * k * sd * 32 + 16) * sizeof(double);
  if (smem + (ds->f64 ? 40 : 20) * 1024 > 227 * 1024)
    return ref_error(AQ_E_UNSUPPORTED, "normal-equation strip exceeds shared memory");
  if (ds->f64)
    AQ_CUDA(cudaFuncSetAttribute(k_assemble<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  else
    AQ_CUDA(cudaFuncSetAttribute(k_assemble<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  const unsigned units = (unsigned)(M * k * nchunk);
  timer_mark(s, AQ_T_ASSEMBLE);
  if (sd == 2 && k == 16 && d % 4 == 0 && codes->bits == 4 && !ds->f64) {
    // 32 column subspaces per unit (a 16-column split with twice the units
    // measured slower: per-unit staging outweighs the extra warps)
    const int cols = 32, nch = nchunk;
    const unsigned units2 = (unsigned)(M * 16 * nch);
    // AQ_ASM_VARIANT=1: rows staged in shared memory (k_assemble_sd2), 3:
    // register ring (k_assemble_sd2r), 0 (default): the ring when a launch
    // has at least two waves of its 12-per-SM CTAs (config 5: 1136 vs 1207
    // ms per 3 iterations), else the staged kernel (config 2: 138 vs 200 ms)
    static const int asm_variant =
        getenv("AQ_ASM_VARIANT") ? atoi(getenv("AQ_ASM_VARIANT")) : 0;
    AQ_CUDA(cudaFuncSetAttribute(k_assemble_sd2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 64 * 32 * 8 + 14 * 1024));
    AQ_CUDA(cudaFuncSetAttribute(k_assemble_sd2r<16>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 32 * 8));

    // units with work, largest strip first (the longest point chains start
    // early instead of trailing the launch)
    std::vector<uint32_t> hc((size_t)M * 16);
    AQ_CUDA(cudaMemcpyAsync(hc.data(), B.count, hc.size() * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost, s->stream));
    AQ_CUDA(cudaStreamSynchronize(s->stream));
    std::vector<uint32_t> ord;
    ord.reserve(units2);
    for (uint32_t u = 0; u < units2; ++u) {
      const int ch = (int)(u % (unsigned)nch), st = (int)(u / (unsigned)nch);
      const int mcols = full ? M : st / 16 + 1;
      if (ch * cols < mcols && hc[st]) ord.push_back(u);
    }
    std::stable_sort(ord.begin(), ord.end(),
                     [&](uint32_t x, uint32_t y) { return hc[x / nch] > hc[y / nch]; });
    void* po;
    AQ_TRY(scratch(s, 5, ord.size() * sizeof(uint32_t) + 16, &po));
    uint32_t* dord = (uint32_t*)po;
    AQ_CUDA(cudaMemcpyAsync(dord, ord.data(), ord.size() * sizeof(uint32_t),
                            cudaMemcpyHostToDevice, s->stream));
    // point blocks whose rows (~48 MB) stay L2-resident while every unit
    // gathers from them; entries keep their point order across blocks
    const bool ring = asm_variant == 3 ||
                      (asm_variant == 0 && ord.size() >= (size_t)2 * 12 * s->num_sms);
    const size_t row_bytes = (size_t)d * sizeof(float);
    const size_t bsz = std::max<size_t>(4096, (48u << 20) / row_bytes);
    for (size_t lo = 0; lo < ds->n && !ord.empty(); lo += bsz) {
      a.lo = (uint32_t)lo;
      a.hi = (uint32_t)std::min(ds->n, lo + bsz);
      a.resume = lo > 0;
      // Up to 1.5 waves of 6 CTAs per SM (config 2: 1,088 units) the longest
      // strips' chains are the critical path: 14 KB of unused dynamic shared
      // memory caps the SM at 4 CTAs, so those chains share the shared-memory
      // pipe with fewer warps (config 2: 14.7 -> 14.2 ms; 5 per SM 14.4,
      // 3 per SM 17.6)
      const int pad = ord.size() <= (size_t)9 * s->num_sms ? 14 * 1024 : 0;
      if (!ring)
        k_assemble_sd2<<<(unsigned)ord.size(), 32, 64 * 32 * 8 + pad, s->stream>>>(a, dord);
      else
        k_assemble_sd2r<16><<<(unsigned)ord.size(), 32, 64 * 32 * 8, s->stream>>>(a, dord);
      AQ_LAUNCHED(s);
    }
  } else {
    a.lo = 0;
    a.hi = (uint32_t)ds->n;
    a.resume = 0;
    if (ds->f64)
      k_assemble<double><<<units, 32, smem, s->stream>>>(a);
    else
      k_assemble<float><<<units, 32, smem, s->stream>>>(a);
  }
  AQ_LAUNCHED(s);
  timer_mark(s, AQ_T_ASSEMBLE);
  return AQ_OK;
}

int check_update_args(aq_dataset* ds, aq_codes* codes, size_t M) {
  if (ds->n == 0) return ref_error(AQ_E_EMPTY_DATASET, "cannot update on an empty dataset");
  if (codes->n != ds->n || codes->M != M)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match dataset");
  if (M == 0 || ds->d % M != 0)
    return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  return AQ_OK;
}

}  // namespace aqd

using namespace aqd;

extern "C" {

// assemble_selector_system (pq.hpp:290-343): full matrix, host outputs.
int aq_dev_assemble_selector_system(aq_dataset* ds, aq_codes* codes, const aq_weights* w,
                                    double* A_out, double* rhs_out) {
  if (!ds || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  if (codes->n != ds->n || codes->M == 0)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match dataset");
  if (ds->d % codes->M != 0)
    return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  const int k = (int)codes->k, M = (int)codes->M;
  const size_t dim = (size_t)k * ds->d;
  void* owner = nullptr;
  PointW pw;
  {
    const int pst = point_weights(ds, w, &pw, &owner);
    if (pst != AQ_OK) {  // validation failures leave no allocation behind
      if (owner) cudaFreeAsync(owner, s->stream);
      return pst;
    }
  }
  int st = AQ_OK;
  if (pw.flags[1] != ~0ull) {
    char msg[128];
    snprintf(msg, sizeof msg, "anisotropic update undefined at |x| = 0 (point %llu)",
             pw.flags[1] - 1);
    st = ref_error(AQ_E_ZERO_NORM_DATAPOINT, msg);
  }
  Buckets B;
  double* A = nullptr;
  if (st == AQ_OK && ds->n) st = build_buckets(codes, k, &B);
  if (st == AQ_OK) {
    if (cudaMallocAsync(&A, (dim * dim + dim) * sizeof(double), s->stream) != cudaSuccess)
      st = ref_error(AQ_E_CUDA, "out of device memory for the normal equations");
  }
  if (st == AQ_OK && ds->n) st = assemble_device(ds, codes, pw, B, k, true, A, A + dim * dim);
  if (st == AQ_OK && !ds->n) {
    cudaMemsetAsync(A, 0, (dim * dim + dim) * sizeof(double), s->stream);
  }
  if (st == AQ_OK) {
    cudaMemcpyAsync(A_out, A, dim * dim * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
    cudaMemcpyAsync(rhs_out, A + dim * dim, dim * sizeof(double), cudaMemcpyDeviceToHost,
                    s->stream);
  }
  if (A) cudaFreeAsync(A, s->stream);
  cudaFreeAsync(owner, s->stream);
  cudaStreamSynchronize(s->stream);
  (void)M;
  return st;
}

// pq_codebook_update (pq.hpp:356-464): writes `out` (M x k x sd, allocated).
// rank_losses / keep_prev (train_avq, vq.hpp:276-292; both null for the
// reference pq_codebook_update): an unused codeword keeps keep_prev's value
// when keep_prev is set, else it takes the next point of the ranking of
// rank_losses (device, n values) when set, else of the point losses under
// the new codebook (pq.hpp:443-462).
static int codebook_update_impl(aq_dataset* ds, aq_codes* codes, const aq_weights* w,
                                double ridge, aq_codebook* out, const double* rank_losses,
                                const double* keep_prev) {
  if (!ds || !codes || !out) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t M = out->M, k = out->k;
  AQ_TRY(check_update_args(ds, codes, M));
  if (codes->k > k) return ref_error(AQ_E_CODE_OUT_OF_RANGE, "code out of range");
  const int sd = (int)(ds->d / M);
  if ((size_t)sd != out->sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "codebook sub-dimension does not match");
  if (sd > 16 && M != 1)
    return ref_error(AQ_E_UNSUPPORTED, "device update supports sub_dimension <= 16 (M > 1)");
  const size_t n = ds->n, dim = k * ds->d;
  Buckets B;
  AQ_TRY(build_buckets(codes, (int)k, &B));
  void* owner = nullptr;
  PointW pw;
  int st = point_weights(ds, w, &pw, &owner);
  double* A = nullptr;
  if (st == AQ_OK)
    st = cudaMemsetAsync(out->d64, 0, M * k * sd * sizeof(double), s->stream) == cudaSuccess
             ? AQ_OK
             : AQ_E_CUDA;
  const bool all_iso = pw.flags[0] == 0;
  if (st == AQ_OK && M == 1) {
    // per-codeword closed form (pq.hpp:387-404 -> vq.hpp:139-192)
    const size_t d = ds->d;
    double* As = nullptr;
    int* modes = nullptr;
    if (cudaMallocAsync(&As, (k * d * d + k * d + 2 * n) * sizeof(double), s->stream) !=
            cudaSuccess ||
        cudaMallocAsync(&modes, k * sizeof(int), s->stream) != cudaSuccess)
      st = ref_error(AQ_E_CUDA, "out of device memory");
    if (st == AQ_OK) st = clear_dev_error(s);  // falls through to the frees below
    if (st == AQ_OK) {
      cudaMemsetAsync(modes, 0xff, k * sizeof(int), s->stream);
      double* coefs = As + k * d * d + k * d;
      AQ_XR_LAUNCH(ds, k_vq_coef, (unsigned)((n + 255) / 256), 256, 0, s->stream, n, (int)d,
                   pw.hp, pw.ho, coefs, coefs + n);
      AQ_XR_LAUNCH(ds, k_vq_systems, (unsigned)k, 128, 0, s->stream, n, (int)d, (int)k, B.list,
                   B.start, B.count, pw.hp, pw.ho, coefs, coefs + n, ridge, As,
                   As + k * d * d, modes, out->d64, s->err);
      s->launches += 2;
      st = sync_and_check(s, "codeword update");
    }
    if (st == AQ_OK) {
      std::vector<int> hm(k);
      cudaMemcpyAsync(hm.data(), modes, k * sizeof(int), cudaMemcpyDeviceToHost, s->stream);
      cudaStreamSynchronize(s->stream);
      for (size_t j = 0; j < k && st == AQ_OK; ++j) {
        if (hm[j] != 0) continue;  // unused (-1) or mean path (1)
        st = llt_solve_device(s, As + j * d * d, (int)d, As + k * d * d + j * d);
        if (st == AQ_E_SINGULAR_SYSTEM)
          st = ref_error(AQ_E_SINGULAR_SYSTEM, "codeword system is not positive definite");
        if (st == AQ_OK)
          cudaMemcpyAsync(out->d64 + j * d, As + k * d * d + j * d, d * sizeof(double),
                          cudaMemcpyDeviceToDevice, s->stream);
      }
    }
    if (As) cudaFreeAsync(As, s->stream);
    if (modes) cudaFreeAsync(modes, s->stream);
  } else if (st == AQ_OK && all_iso) {
    AQ_TRY(clear_dev_error(s));
    st = slot_sums_device(s, ds, (int)M, (int)k, sd, B, nullptr, pw.hp, pw.ho, out->d64,
                          nullptr, nullptr);
    if (st == AQ_OK) st = sync_and_check(s, "zero total weight in block");
  } else if (st == AQ_OK) {
    if (dim > 16384) {
      st = ref_error(AQ_E_INVALID_ARGUMENT,
                     "stacked codebook system exceeds 16384 unknowns (pq.hpp:426-429)");
    } else if (pw.flags[1] != ~0ull) {
      char msg[128];
      snprintf(msg, sizeof msg, "anisotropic update undefined at |x| = 0 (point %llu)",
               pw.flags[1] - 1);
      st = ref_error(AQ_E_ZERO_NORM_DATAPOINT, msg);
    } else if (cudaMallocAsync(&A, (dim * dim + dim) * sizeof(double), s->stream) !=
               cudaSuccess) {
      st = ref_error(AQ_E_CUDA, "out of device memory for the normal equations");
    }
    if (st == AQ_OK) st = assemble_device(ds, codes, pw, B, (int)k, false, A, A + dim * dim);
    if (st == AQ_OK) {
      k_trace_ridge<<<1, 1024, 0, s->stream>>>(A, dim, ridge);
      s->launches++;
      st = llt_solve_device(s, A, (int)dim, A + dim * dim);
    }
    if (st == AQ_OK &&
        cudaMemcpyAsync(out->d64, A + dim * dim, dim * sizeof(double),
                        cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess)
      st = AQ_E_CUDA;
  }
  // reseed unused codewords from the loss ranking under the new codebook
  if (st == AQ_OK) {
    std::vector<uint32_t> hc(M * k);
    cudaMemcpyAsync(hc.data(), B.count, M * k * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                    s->stream);
    cudaStreamSynchronize(s->stream);
    bool any_unused = false;
    for (auto c : hc) any_unused |= c == 0;
    if (any_unused && keep_prev) {
      for (size_t t = 0; t < M * k && st == AQ_OK; ++t)
        if (hc[t] == 0 &&
            cudaMemcpyAsync(out->d64 + t * sd, keep_prev + t * sd, sd * sizeof(double),
                            cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess)
          st = AQ_E_CUDA;
    } else if (any_unused) {
      st = stage_codebook(out);
      double* losses = nullptr;
      uint32_t* idx = nullptr;
      uint32_t* cnt_copy = nullptr;
      if (st == AQ_OK) {
        cudaMallocAsync(&losses, n * sizeof(double), s->stream);
        cudaMallocAsync(&idx, n * sizeof(uint32_t), s->stream);
        cudaMallocAsync(&cnt_copy, M * k * sizeof(uint32_t), s->stream);
        cudaMemcpyAsync(cnt_copy, hc.data(), M * k * sizeof(uint32_t), cudaMemcpyHostToDevice,
                        s->stream);
        if (rank_losses)
          st = cudaMemcpyAsync(losses, rank_losses, n * sizeof(double), cudaMemcpyDeviceToDevice,
                               s->stream) == cudaSuccess
                   ? AQ_OK
                   : AQ_E_CUDA;
        else
          st = run_encode(ds, out, w, codes, 2, 0, 0, losses, nullptr);
      }
      if (st == AQ_OK) {
        k_iota<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(idx, n);
        s->launches++;
        st = sort_scores_desc(s, losses, idx, n);
      }
      if (st == AQ_OK) {
        AQ_XR_LAUNCH(ds, k_reseed, 1, 1, 0, s->stream, cnt_copy, (int)M, (int)k, sd, idx, n,
                     (int)ds->d, out->d64);
        s->launches++;
      }
      if (losses) cudaFreeAsync(losses, s->stream);
      if (idx) cudaFreeAsync(idx, s->stream);
      if (cnt_copy) cudaFreeAsync(cnt_copy, s->stream);
    }
  }
  if (st == AQ_OK) st = stage_codebook(out);
  if (A) cudaFreeAsync(A, s->stream);
  if (owner) cudaFreeAsync(owner, s->stream);
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (st == AQ_OK && e != cudaSuccess) {
    set_error(AQ_E_CUDA, "CUDA error %s", cudaGetErrorString(e));
    st = AQ_E_CUDA;
  }
  return st;
}

int aq_dev_pq_codebook_update(aq_dataset* ds, aq_codes* codes, const aq_weights* w,
                              double ridge, aq_codebook* out) {
  return codebook_update_impl(ds, codes, w, ridge, out, nullptr, nullptr);
}

// Host-pointer form of pq_codebook_update.
int aq_pq_codebook_update(aq_session* s, const float* x, size_t n, size_t d,
                          const uint32_t* codes, size_t M, size_t k, const aq_weights* w,
                          double ridge, double* dict_out) {
  AQ_TRY(check_session(s));
  if (n == 0) return ref_error(AQ_E_EMPTY_DATASET, "cannot update on an empty dataset");
  if (M == 0 || d % M != 0)
    return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  aq_dataset* ds = nullptr;
  aq_codes* cm = nullptr;
  aq_codebook* cb = nullptr;
  int st = aq_dataset_upload(s, x, n, d, &ds);
  if (st == AQ_OK) st = aq_codes_upload(s, codes, n, M, k, &cm);
  if (st == AQ_OK) st = aq_codebook_upload(s, nullptr, M, k, d / M, &cb);
  if (st == AQ_OK) st = aq_dev_pq_codebook_update(ds, cm, w, ridge, cb);
  if (st == AQ_OK) st = aq_codebook_download(cb, dict_out);
  aq_codebook_free(cb);
  aq_codes_free(cm);
  aq_dataset_free(ds);
  return st;
}

}  // extern "C"

namespace aqd {
// train_avq's codebook step (vq.hpp:276-307) for the device trainer.
int avq_codebook_update(aq_dataset* ds, aq_codes* codes, const aq_weights* w, double ridge,
                        aq_codebook* out, const double* rank_losses, const double* keep_prev) {
  return codebook_update_impl(ds, codes, w, ridge, out, rank_losses, keep_prev);
}
}  // namespace aqd
