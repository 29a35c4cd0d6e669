// Trainers on the device:
//   * train_l2_pq (pq.hpp:469-501): M independent isotropic k-means runs
//     (train_avq, vq.hpp:243-329, seed + m per subspace) advanced in lockstep,
//     each subspace stopping on its own criterion;
//   * train_apq (pq.hpp:513-575): warm or cold start, assignment pass
//     (encode.cu), joint codebook update (update.cu), loss history and the
//     reference's stopping rules.
// Loss totals are std::accumulate in index order (pq.hpp:553,562;
// vq.hpp:270,316): a single-thread float64 chain per subspace, so histories
// are bit-identical to the reference.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace aqd {

int sort_scores_desc(aq_session* s, const double* scores, uint32_t* idx, size_t n);
int run_encode(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes,
               int mode, int passes, int sweep_fixed, double* losses_dev,
               uint64_t* changed_out);
int stage_codebook(aq_codebook* cb);
int avq_codebook_update(aq_dataset* ds, aq_codes* codes, const aq_weights* w, double ridge,
                        aq_codebook* out, const double* rank_losses, const double* keep_prev);


// ---- Rng (rng.hpp:28-89), host side -----------------------------------------------------
// ---- kernels ------------------------------------------------------------------------------

// std::accumulate of `count` values (float64, index order), one warp per row.
// The chain of dependent adds is the bound (count x DADD latency), so the
// lanes keep it fed: block t + 1 (256 values, 8 per lane, coalesced) is in
// registers while lane 0 adds block t from shared memory in index order.
__global__ void k_seq_sums(const double* __restrict__ v, size_t ld, size_t count, int rows,
                           const int* __restrict__ active, double* __restrict__ out,
                           double init = 0.0) {
  __shared__ double buf[8][2][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + w;
  if (r >= rows || (active && !active[r])) return;
  const double* p = v + (size_t)r * ld;
  double s = init;
  double nxt[8];
  auto fetch = [&](size_t i0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const size_t i = i0 + u * 32 + lane;
      nxt[u] = i < count ? p[i] : 0.0;
    }
  };
  fetch(0);
  int cur = 0;
  for (size_t i0 = 0; i0 < count; i0 += 256) {
#pragma unroll
    for (int u = 0; u < 8; ++u) buf[w][cur][u * 32 + lane] = nxt[u];
    __syncwarp();
    if (i0 + 256 < count) fetch(i0 + 256);  // in flight during the chain below
    if (lane == 0) {
      const int nb = (int)min((size_t)256, count - i0);
      const double* b = buf[w][cur];
      if (nb == 256) {
#pragma unroll 16
        for (int t = 0; t < 256; ++t) s = __dadd_rn(s, b[t]);
      } else {
        for (int t = 0; t < nb; ++t) s = __dadd_rn(s, b[t]);
      }
    }
    cur ^= 1;
  }
  if (lane == 0) out[r] = s;
}

// ---- the same sums, chunk-parallel (non-negative rows) ------------------------------------
// std::accumulate over non-negative doubles is a monotone chain s_{i+1} =
// fl(s_i + v_i). While s stays inside one binade [2^E, 2^(E+1)) its ulp u is
// fixed and fl(s + v) = s + u * round(v / u) (to nearest; an exact half is a
// tie whose result depends on the parity of s / u). Over a chunk that keeps s
// inside the binade the chain is therefore a translation by u * K, K = the
// sum of the rounded v / u — an exact integer sum that threads may form in
// any order. The chain then steps over chunks instead of values: a chunk is
// applied as s += u K when the binade predicted for it (from approximate
// prefix sums) is the binade of s, it holds no tie, and s + u K <= 2^(E+1) -
// 2u (so every intermediate exact sum stays below 2^(E+1) - u / 2 and rounds
// to a multiple of u). Every other chunk — the few binade crossings, ties,
// s = 0 or tiny, a wrong prediction — is added value by value. Rows holding a
// negative or non-finite value run the plain chain. Bit-identical to
// k_seq_sums (tests/test_seq_sums_gpu.py).
constexpr int kSeqChunk = 2048;

__device__ __forceinline__ int dexp_field(double x) {
  return (int)((unsigned long long)__double_as_longlong(x) >> 52) & 0x7ff;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  T t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

// pass 1: approximate chunk sums (any order); rows with a negative or
// non-finite value are marked for the plain chain
__global__ void k_seqsum_approx(const double* __restrict__ v, size_t ld, size_t count, int nch,
                                const int* __restrict__ active, double* __restrict__ approx,
                                int* __restrict__ plain) {
  __shared__ double red[32];
  const int r = blockIdx.y, c = blockIdx.x;
  if (active && !active[r]) return;
  const double* p = v + (size_t)r * ld + (size_t)c * kSeqChunk;
  const int len = (int)min((size_t)kSeqChunk, count - (size_t)c * kSeqChunk);
  double s = 0.0;
  int bad = 0;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const double x = p[i];
    bad |= !(x >= 0.0 && x <= 1.7976931348623157e308);
    s += x;
  }
  s = block_sum(s, red);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    approx[(size_t)r * nch + c] = s;
    if (bad) plain[r] = 1;
  }
}

// pass 2: predicted chain value at every chunk start (init + approximate
// prefix), one block per row
__global__ void k_seqsum_predict(const double* __restrict__ approx, int nch, double init,
                                 const int* __restrict__ active, double* __restrict__ pred) {
  __shared__ double red[32];
  __shared__ double carry;
  const int r = blockIdx.x;
  if (active && !active[r]) return;
  if (threadIdx.x == 0) carry = init;
  __syncthreads();
  for (int base = 0; base < nch; base += blockDim.x) {
    const int c = base + threadIdx.x;
    const double a = c < nch ? approx[(size_t)r * nch + c] : 0.0;
    // inclusive warp scan, then warp offsets
    double inc = a;
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, inc, o);
      if ((threadIdx.x & 31) >= o) inc += t;
    }
    if ((threadIdx.x & 31) == 31) red[threadIdx.x >> 5] = inc;
    __syncthreads();
    double off = carry;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) off += red[w];
    if (c < nch) pred[(size_t)r * nch + c] = off + inc - a;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = off + inc;
    __syncthreads();
  }
}

// pass 3: per chunk, the ulp exponent predicted for it (-1: add value by
// value) and K = sum of round(v / u)
__global__ void k_seqsum_chunks(const double* __restrict__ v, size_t ld, size_t count, int nch,
                                const int* __restrict__ active, const double* __restrict__ pred,
                                const double* __restrict__ approx, int* __restrict__ efield,
                                unsigned long long* __restrict__ K) {
  __shared__ unsigned long long red[32];
  const int r = blockIdx.y, c = blockIdx.x;
  if (active && !active[r]) return;
  const double* p = v + (size_t)r * ld + (size_t)c * kSeqChunk;
  const int len = (int)min((size_t)kSeqChunk, count - (size_t)c * kSeqChunk);
  const double s0 = pred[(size_t)r * nch + c];
  const double s1 = s0 + approx[(size_t)r * nch + c];  // predicted chunk end
  const int e = dexp_field(s0);
  // tiny or zero start, or a predicted binade crossing: value by value
  bool seq = !(e >= 60 && e <= 2000) || dexp_field(s1) != e;
  unsigned long long k = 0ull;
  if (!seq) {
    const double inv_u = __longlong_as_double((long long)(1075 + 1023 - e) << 52);  // 2^(1075-e)
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const double q = __dmul_rn(p[i], inv_u);  // exact: a power-of-two scaling
      if (!(q < 4503599627370496.0)) {           // >= 2^52: cannot stay in the binade
        seq = true;
        break;
      }
      const double f = floor(q);
      const double fr = q - f;  // exact
      if (fr == 0.5) {          // a tie: rounding depends on the chain's parity
        seq = true;
        break;
      }
      k += (unsigned long long)f + (fr > 0.5 ? 1ull : 0ull);
    }
  }
  k = block_sum(k, red);
  seq = __syncthreads_or(seq);
  if (threadIdx.x == 0) {
    efield[(size_t)r * nch + c] = seq ? -1 : e;
    K[(size_t)r * nch + c] = k;
  }
}

// pass 4: the chain over chunks, one warp per row; value-by-value chunks are
// staged by the warp and added by lane 0 in index order
__global__ void k_seqsum_chain(const double* __restrict__ v, size_t ld, size_t count, int nch,
                               int rows, const int* __restrict__ active,
                               const int* __restrict__ plain, const int* __restrict__ efield,
                               const unsigned long long* __restrict__ K, double init,
                               double* __restrict__ out) {
  __shared__ double buf[4][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + w;
  if (r >= rows || (active && !active[r])) return;
  const double* row = v + (size_t)r * ld;
  const bool all_seq = plain[r] != 0;
  double s = init;
  auto chain = [&](size_t i0, size_t i1) {  // s += v[i] for i in [i0, i1), in order
    for (size_t b = i0; b < i1; b += 256) {
      const int nb = (int)min((size_t)256, i1 - b);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = u * 32 + lane;
        buf[w][t] = t < nb ? row[b + t] : 0.0;
      }
      __syncwarp();
      if (lane == 0)
        for (int t = 0; t < nb; ++t) s = __dadd_rn(s, buf[w][t]);
      __syncwarp();
    }
  };
  if (all_seq) {
    chain(0, count);
  } else {
    for (int c0 = 0; c0 < nch; c0 += 32) {
      const int c = c0 + lane;
      const int ef = c < nch ? efield[(size_t)r * nch + c] : -1;
      const unsigned long long kc = c < nch ? K[(size_t)r * nch + c] : 0ull;
      const int nc = min(32, nch - c0);
      for (int t = 0; t < nc; ++t) {
        const int e_t = __shfl_sync(0xffffffffu, ef, t);
        const unsigned long long k_t = __shfl_sync(0xffffffffu, kc, t);
        s = __shfl_sync(0xffffffffu, s, 0);
        bool fast = false;
        double nxt = 0.0;
        if (e_t >= 0 && dexp_field(s) == e_t && k_t < (1ull << 52)) {
          const double u = __longlong_as_double((long long)(e_t - 52) << 52);   // 2^(e-1075)
          const double top = __longlong_as_double((long long)(e_t + 1) << 52);  // 2^(e-1022)
          nxt = s + u * (double)k_t;  // exact: multiples of u inside the binade
          fast = nxt <= top - 2.0 * u;
        }
        if (fast) {
          s = nxt;
        } else {
          const size_t i0 = (size_t)(c0 + t) * kSeqChunk;
          chain(i0, min(count, i0 + kSeqChunk));
        }
      }
    }
  }
  if (lane == 0) out[r] = s;
}

// `rows` sequential sums (std::accumulate from init) of `count` values each
// (row r at v + r * ld), rows with active[r] == 0 skipped; out (device), on
// `st`. Long rows take the chunk-parallel passes (AQ_SEQSUM=0: the plain
// chain everywhere).
int seq_sums_on(aq_session* s, cudaStream_t st, const double* v, size_t ld, size_t count,
                int rows, const int* active_dev, double* out, double init) {
  static const int mode = getenv("AQ_SEQSUM") ? atoi(getenv("AQ_SEQSUM")) : 1;
  if (rows <= 0) return AQ_OK;
  if (mode == 0 || count < 65536) {
    k_seq_sums<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(v, ld, count, rows, active_dev, out,
                                                          init);
    AQ_LAUNCHED(s);
    return AQ_OK;
  }
  const int nch = (int)((count + kSeqChunk - 1) / kSeqChunk);
  const size_t cells = (size_t)rows * nch;
  void* buf = nullptr;
  const size_t bytes = cells * (2 * sizeof(double) + sizeof(unsigned long long) + sizeof(int)) +
                       rows * sizeof(int) + 64;
  AQ_CUDA(cudaMallocAsync(&buf, bytes, st));
  double* approx = (double*)buf;
  double* pred = approx + cells;
  unsigned long long* K = (unsigned long long*)(pred + cells);
  int* ef = (int*)(K + cells);
  int* plain = ef + cells;
  AQ_CUDA(cudaMemsetAsync(plain, 0, rows * sizeof(int), st));
  k_seqsum_approx<<<dim3((unsigned)nch, (unsigned)rows), 256, 0, st>>>(v, ld, count, nch,
                                                                      active_dev, approx, plain);
  AQ_LAUNCHED(s);
  k_seqsum_predict<<<(unsigned)rows, 1024, 0, st>>>(approx, nch, init, active_dev, pred);
  AQ_LAUNCHED(s);
  k_seqsum_chunks<<<dim3((unsigned)nch, (unsigned)rows), 256, 0, st>>>(v, ld, count, nch,
                                                                      active_dev, pred, approx,
                                                                      ef, K);
  AQ_LAUNCHED(s);
  k_seqsum_chain<<<(unsigned)((rows + 3) / 4), 128, 0, st>>>(v, ld, count, nch, rows, active_dev,
                                                             plain, ef, K, init, out);
  AQ_LAUNCHED(s);
  AQ_CUDA(cudaFreeAsync(buf, st));
  return AQ_OK;
}

int seq_sums_device(aq_session* s, const double* v, size_t ld, size_t count, int rows,
                    const int* active_dev, double* out) {
  return seq_sums_on(s, s->stream, v, ld, count, rows, active_dev, out, 0.0);
}

// std::accumulate(v, v + n, init) into *out (device), on the session stream
int seq_sum_device(aq_session* s, const double* v, size_t n, double init, double* out) {
  return seq_sums_on(s, s->stream, v, n, n, 1, nullptr, out, init);
}

// codewords from sampled rows: dict[m][j] = x[idx[m][j]][m-subvector]
template <class TX>
__global__ void k_init_codewords(const TX* __restrict__ xr, int d, int M, int k, int sd,
                                 const uint64_t* __restrict__ idx, double* __restrict__ dict) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M * k) return;
  const int m = t / k;
  const uint64_t p = idx[t];
  for (int c = 0; c < sd; ++c)
    dict[(size_t)t * sd + c] = (double)xr[p * d + (size_t)m * sd + c];
}

__device__ __forceinline__ void set_code(uint8_t* row, int m, int bits, unsigned c) {
  if (bits == 4) {
    const int sh = (m & 1) * 4;
    row[m >> 1] = (uint8_t)((row[m >> 1] & ~(15u << sh)) | (c << sh));
  } else {
    row[m] = (uint8_t)c;
  }
}

// vq_assign_pass with isotropic unit weights (vq.hpp:196-217, assign_scan
// 83-100): per subspace argmin of dist2 (first index wins), loss = 1.0 dist2.
// One thread per point walks the active subspaces (codes share bytes).
template <class TX>
__global__ void k_kmeans_assign(const TX* __restrict__ xr, size_t n, int d, int M, int k,
                                int sd, const double* __restrict__ dict,
                                const int* __restrict__ active, uint8_t* __restrict__ codes,
                                int stride, int bits, double* __restrict__ losses,
                                unsigned long long* __restrict__ changes) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t* row = codes + i * stride;
  const TX* xp = xr + i * d;
  for (int m = 0; m < M; ++m) {
    if (!active[m]) continue;
    const double* cm = dict + (size_t)m * k * sd;
    unsigned bj = 0;
    double bd = 0.0;
    for (int j = 0; j < k; ++j) {
      double d2 = 0.0;
      for (int c = 0; c < sd; ++c) {
        const double diff = __dsub_rn((double)xp[m * sd + c], cm[j * sd + c]);
        d2 = __dadd_rn(d2, __dmul_rn(diff, diff));
      }
      if (j == 0 || d2 < bd) {
        bd = d2;
        bj = (unsigned)j;
      }
    }
    const unsigned old = get_code(row, m, bits);
    if (old != bj) {
      set_code(row, m, bits, bj);
      atomicAdd(&changes[m], 1ull);
    }
    losses[(size_t)m * n + i] = __dmul_rn(1.0, bd);
  }
}

// Same pass for sub_dimension 2 with coalesced reads: the pair-tiled rows
// (32 points x one pair per 256-byte line), the codebook in shared memory,
// code words built in registers (written once per 8 subspaces), changed-code
// counts aggregated per warp and per CTA before one global atomic per
// subspace. Operation order per candidate as residual_terms (dist2 =
// df0^2 + df1^2; 0.0 + df0^2 == df0^2 exactly).
__global__ void __launch_bounds__(256) k_kmeans_assign_sd2(
    const float2* __restrict__ xt, size_t n, int pairs, int M, int k,
    const double* __restrict__ dict, const int* __restrict__ active, uint8_t* __restrict__ codes,
    int stride, double* __restrict__ losses, unsigned long long* __restrict__ changes) {
  extern __shared__ __align__(16) unsigned char ksm[];
  double2* cbs = reinterpret_cast<double2*>(ksm);            // [M][k]
  unsigned* chg = reinterpret_cast<unsigned*>(cbs + (size_t)M * k);  // [M]
  int* act = reinterpret_cast<int*>(chg + M);                 // [M]
  for (int t = threadIdx.x; t < M * k; t += blockDim.x)
    cbs[t] = reinterpret_cast<const double2*>(dict)[t];
  for (int t = threadIdx.x; t < M; t += blockDim.x) {
    chg[t] = 0u;
    act[t] = active[t];
  }
  __syncthreads();
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  const int lane = threadIdx.x & 31;
  const float2* xrow = xt + (i >> 5) * (size_t)pairs * 32 + (i & 31);
  uint32_t* crow = reinterpret_cast<uint32_t*>(codes + (valid ? i : 0) * (size_t)stride);
  uint32_t word = 0;
  for (int m = 0; m < M; ++m) {
    if ((m & 7) == 0 && valid) word = crow[m >> 3];
    if (act[m]) {
      unsigned bj = 0;
      bool ch = false;
      if (valid) {
        const float2 xv = xrow[(size_t)m * 32];
        const double x0 = xv.x, x1 = xv.y;
        const double2* cm = cbs + (size_t)m * k;
        double bd = 0.0;
        for (int j = 0; j < k; ++j) {
          const double2 c = cm[j];
          const double df0 = __dsub_rn(x0, c.x), df1 = __dsub_rn(x1, c.y);
          const double d2 = __dadd_rn(__dmul_rn(df0, df0), __dmul_rn(df1, df1));
          if (j == 0 || d2 < bd) {
            bd = d2;
            bj = (unsigned)j;
          }
        }
        const int sh = 4 * (m & 7);
        ch = ((word >> sh) & 15u) != bj;
        word = (word & ~(15u << sh)) | (bj << sh);
        losses[(size_t)m * n + i] = __dmul_rn(1.0, bd);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ch);
      if (lane == 0 && bal) atomicAdd(&chg[m], (unsigned)__popc(bal));
    }
    if (((m & 7) == 7 || m + 1 == M) && valid) crow[m >> 3] = word;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < M; t += blockDim.x)
    if (chg[t]) atomicAdd(&changes[t], (unsigned long long)chg[t]);
}

// update_codeword isotropic path (vq.hpp:151-162) with unit weights:
// mean = (sum 1.0 x) / (sum 1.0), members in ascending order. One warp per
// slot: the lanes gather 32 members' sub-vectors into shared memory (all in
// flight), lane 0 accumulates them in member order.
// Per-slot sums over the slot's members in ascending point order (the
// reference's loops): one warp per slot; rounds of 128 members — the lanes
// gather round r + 1 (rows and, weighted, h_par / h_perp) into registers while
// lane 0 adds round r in member order.
//   kWeighted = false: num += 1.0 x, den += 1.0 (k-means, vq.hpp:151-162)
//   kWeighted = true:  num += h_par x, den += h_perp (isotropic update,
//                      pq.hpp:405-417)
//   dict != null: dict = num / den for non-empty slots (weighted: den <= 0 is
//                 a singular block); else num / den are written as partials.
template <class TX, int SDC, bool kWeighted>
__global__ void k_slot_sums(const TX* __restrict__ xr, const float* __restrict__ xt, size_t n,
                            int d, int M, int k,
                            int sd_rt, const uint32_t* __restrict__ list,
                            const uint32_t* __restrict__ start,
                            const uint32_t* __restrict__ count, const int* __restrict__ active,
                            const double* __restrict__ hp, const double* __restrict__ ho,
                            double* __restrict__ dict, double* __restrict__ pnum,
                            double* __restrict__ pden, DevError* err) {
  constexpr int SDM = SDC > 0 ? SDC : 16;
  constexpr int G = SDC > 0 ? 4 : 1, R = 32 * G;
  const int sd = SDC > 0 ? SDC : sd_rt;
  // per member: the products a * x (float64, formed by the fetching lane)
  // and the weight o; lane 0 then runs only the dependent adds
  __shared__ double ps[4][2][R][SDM];
  __shared__ double ws[4][2][kWeighted ? R : 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * (blockDim.x >> 5) + w;
  if (slot >= M * k) return;
  const int m = slot / k;
  if (active && !active[m]) return;
  const size_t cnt = count[slot];
  const uint32_t* L = list + (size_t)m * n + start[slot];
  TX nx[G][SDM];
  double nh[G][2];
  auto fetch = [&](size_t r0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const size_t t = r0 + g * 32 + lane;
      if (t < cnt) {
        const uint32_t p = L[t];
        bool tiled = false;
        if constexpr (SDC == 2) {
          if (xt) {
            // pair-tiled rows: the 16 slots of subspace m read the same
            // 256-byte (32-point, pair m) blocks, so L2 serves most of them
            const float2 v = reinterpret_cast<const float2*>(
                xt)[(((size_t)(p >> 5) * (d >> 1)) + m) * 32 + (p & 31)];
            nx[g][0] = v.x;
            nx[g][1] = v.y;
            tiled = true;
          }
        }
        if (!tiled) {
          const TX* xp = xr + (size_t)p * d + m * sd;
#pragma unroll
          for (int c = 0; c < SDM; ++c)
            if (c < sd) nx[g][c] = xp[c];
        }
        if (kWeighted) {
          nh[g][0] = hp[p];
          nh[g][1] = ho[p];
        }
      }
    }
  };
  double num[SDM];
#pragma unroll
  for (int c = 0; c < SDM; ++c) num[c] = 0.0;
  double den = 0.0;
  if (cnt) fetch(0);
  int cur = 0;
  for (size_t r0 = 0; r0 < cnt; r0 += R) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const double a = kWeighted ? nh[g][0] : 1.0;
#pragma unroll
      for (int c = 0; c < SDM; ++c)
        if (c < sd) ps[w][cur][g * 32 + lane][c] = __dmul_rn(a, (double)nx[g][c]);
      if (kWeighted) ws[w][cur][g * 32 + lane] = nh[g][1];
    }
    __syncwarp();
    if (r0 + R < cnt) fetch(r0 + R);  // in flight during the chain below
    if (lane == 0) {
      const int nb = (int)min((size_t)R, cnt - r0);
      auto add = [&](int b) {
#pragma unroll
        for (int c = 0; c < SDM; ++c)
          if (c < sd) num[c] = __dadd_rn(num[c], ps[w][cur][b][c]);
        if (kWeighted) den = __dadd_rn(den, ws[w][cur][b]);
      };
      if (nb == R) {
        // unrolled: the loads and products of later members issue ahead, the
        // dependent adds are the only chain
#pragma unroll 16
        for (int b = 0; b < R; ++b) add(b);
      } else {
        for (int b = 0; b < nb; ++b) add(b);
      }
    }
    cur ^= 1;
  }
  if (lane != 0) return;
  // unit weights: den = 1 + 1 + ... in order, exact below 2^53
  if (!kWeighted) den = (double)cnt;
  if (dict) {
    if (cnt == 0) return;  // unused: reseeded (or kept) by the caller
    if (kWeighted && den <= 0.0) {
      report_error(err, (uint64_t)slot, AQ_E_SINGULAR_SYSTEM);
      return;
    }
#pragma unroll
    for (int c = 0; c < SDM; ++c)
      if (c < sd) dict[(size_t)slot * sd + c] = __ddiv_rn(num[c], den);
  } else {
#pragma unroll
    for (int c = 0; c < SDM; ++c)
      if (c < sd) pnum[(size_t)slot * sd + c] = num[c];
    pden[slot] = den;
  }
}

// Host wrapper of k_slot_sums (hp == null: unit weights).
int slot_sums_device(aq_session* s, const aq_dataset* ds, int M, int k, int sd,
                     const Buckets& B, const int* active, const double* hp, const double* ho,
                     double* dict, double* pnum, double* pden) {
  const unsigned grid = (unsigned)((M * k + 3) / 4);
  const size_t n = ds->n;
  const int d = (int)ds->d;
#define AQ_SLOTS(SDV, WV)                                                                     \
  do {                                                                                       \
    if (ds->f64)                                                                             \
      k_slot_sums<double, SDV, WV><<<grid, 128, 0, s->stream>>>(                             \
          ds->xr64, nullptr, n, d, M, k, sd, B.list, B.start, B.count, active, hp, ho, dict, \
          pnum, pden, s->err);                                                               \
    else                                                                                     \
      k_slot_sums<float, SDV, WV><<<grid, 128, 0, s->stream>>>(                              \
          ds->xr, ds->xt, n, d, M, k, sd, B.list, B.start, B.count, active, hp, ho, dict,    \
          pnum, pden, s->err);                                                               \
  } while (0)
  if (sd == 2) {
    if (hp) AQ_SLOTS(2, true);
    else AQ_SLOTS(2, false);
  } else {
    if (hp) AQ_SLOTS(0, true);
    else AQ_SLOTS(0, false);
  }
#undef AQ_SLOTS
  AQ_LAUNCHED(s);
  return AQ_OK;
}

// empty partitions (vq.hpp:284-292): j ascending, consuming the ranking
template <class TX>
__global__ void k_kmeans_reseed(const uint32_t* __restrict__ count, int m, int k, int sd,
                                const uint32_t* __restrict__ order, const TX* xr, int d,
                                double* dict) {
  size_t cursor = 0;
  for (int j = 0; j < k; ++j) {
    if (count[m * k + j] != 0) continue;
    const uint32_t p = order[cursor++];
    for (int c = 0; c < sd; ++c)
      dict[((size_t)m * k + j) * sd + c] = (double)xr[(size_t)p * d + m * sd + c];
  }
}

__global__ void k_iota2(uint32_t* v, size_t n) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) v[t] = (uint32_t)t;
}

// ---- train_l2_pq -----------------------------------------------------------------------------

int train_l2_pq_device(aq_dataset* ds, size_t M, size_t k, const aq_train_config* cfg,
                       aq_codebook** cb_out, aq_codes** codes_out) {
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  if (n == 0) return ref_error(AQ_E_EMPTY_DATASET, "cannot train on an empty dataset");
  if (M == 0 || d % M != 0) return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  if (k == 0 || k > n) return ref_error(AQ_E_INVALID_ARGUMENT, "need 1 <= k <= n");
  if (k > 256) return ref_error(AQ_E_UNSUPPORTED, "device trainers support k <= 256");
  const size_t sd = d / M;
  if (sd > 16) return ref_error(AQ_E_UNSUPPORTED, "device trainers support sub_dimension <= 16");
  aq_codebook* cb = nullptr;
  aq_codes* codes = nullptr;
  AQ_TRY(aq_codebook_upload(s, nullptr, M, k, sd, &cb));
  int st = aq_codes_alloc(s, n, M, k, &codes);
  // initial codewords: Rng(seed + m).sample_distinct(n, k) per subspace
  std::vector<uint64_t> hidx(M * k);
  for (size_t m = 0; m < M; ++m) {
    HostRng r{cfg->seed + m};
    const auto v = r.sample_distinct(n, k);
    for (size_t j = 0; j < k; ++j) hidx[m * k + j] = v[j];
  }
  double* losses = nullptr;
  double* totals = nullptr;
  unsigned long long* changes = nullptr;
  int* active = nullptr;
  uint64_t* didx = nullptr;
  uint32_t* order = nullptr;
  if (st == AQ_OK) {
    cudaMallocAsync(&losses, M * n * sizeof(double), s->stream);
    cudaMallocAsync(&totals, M * sizeof(double), s->stream);
    cudaMallocAsync(&changes, M * sizeof(unsigned long long), s->stream);
    cudaMallocAsync(&active, M * sizeof(int), s->stream);
    cudaMallocAsync(&didx, M * k * sizeof(uint64_t), s->stream);
    cudaMallocAsync(&order, n * sizeof(uint32_t), s->stream);
    cudaMemcpyAsync(didx, hidx.data(), M * k * sizeof(uint64_t), cudaMemcpyHostToDevice, s->stream);
    if (ds->f64)
      k_init_codewords<double><<<(unsigned)((M * k + 127) / 128), 128, 0, s->stream>>>(
          ds->xr64, (int)d, (int)M, (int)k, (int)sd, didx, cb->d64);
    else
      k_init_codewords<float><<<(unsigned)((M * k + 127) / 128), 128, 0, s->stream>>>(
          ds->xr, (int)d, (int)M, (int)k, (int)sd, didx, cb->d64);
    s->launches++;
  }
  std::vector<int> hact(M, 1);
  std::vector<double> htot(M), hprev(M);
  std::vector<unsigned long long> hchg(M);
  auto assign = [&]() -> int {
    AQ_CUDA(cudaMemcpyAsync(active, hact.data(), M * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    AQ_CUDA(cudaMemsetAsync(changes, 0, M * sizeof(unsigned long long), s->stream));
    if (sd == 2 && codes->bits == 4 && !ds->f64) {
      const size_t sm = (size_t)M * k * sizeof(double2) + 2 * M * sizeof(int);
      AQ_CUDA(cudaFuncSetAttribute(k_kmeans_assign_sd2,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_kmeans_assign_sd2<<<(unsigned)((n + 255) / 256), 256, sm, s->stream>>>(
          reinterpret_cast<const float2*>(ds->xt), n, (int)(d / 2), (int)M, (int)k, cb->d64,
          active, codes->data, (int)codes->stride, losses, changes);
    } else {
      AQ_XR_LAUNCH(ds, k_kmeans_assign, (unsigned)((n + 127) / 128), 128, 0, s->stream, n,
                   (int)d, (int)M, (int)k, (int)sd, cb->d64, active, codes->data,
                   (int)codes->stride, codes->bits, losses, changes);
    }
    AQ_LAUNCHED(s);
    // loss totals only feed the relative-tolerance test (vq.hpp:316-321)
    if (cfg->relative_tolerance > 0.0) {
      AQ_TRY(seq_sums_on(s, s->stream, losses, n, n, (int)M, active, totals, 0.0));
      AQ_CUDA(cudaMemcpyAsync(htot.data(), totals, M * sizeof(double), cudaMemcpyDeviceToHost,
                              s->stream));
    }
    AQ_CUDA(cudaMemcpyAsync(hchg.data(), changes, M * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s->stream));
    AQ_CUDA(cudaStreamSynchronize(s->stream));
    return AQ_OK;
  };
  if (st == AQ_OK) st = assign();
  for (int iter = 0; st == AQ_OK && iter < cfg->max_iterations; ++iter) {
    bool any = false;
    for (size_t m = 0; m < M; ++m) any |= hact[m] != 0;
    if (!any) break;
    Buckets B;
    st = build_buckets(codes, (int)k, &B);
    if (st != AQ_OK) break;
    AQ_CUDA(cudaMemcpyAsync(active, hact.data(), M * sizeof(int), cudaMemcpyHostToDevice, s->stream));
    AQ_TRY(slot_sums_device(s, ds, (int)M, (int)k, (int)sd, B, active, nullptr, nullptr,
                            cb->d64, nullptr, nullptr));
    s->launches++;
    if (cfg->empty_partition_policy == 0) {
      std::vector<uint32_t> hc(M * k);
      AQ_CUDA(cudaMemcpyAsync(hc.data(), B.count, M * k * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost, s->stream));
      AQ_CUDA(cudaStreamSynchronize(s->stream));
      for (size_t m = 0; m < M && st == AQ_OK; ++m) {
        if (!hact[m]) continue;
        bool empty = false;
        for (size_t j = 0; j < k; ++j) empty |= hc[m * k + j] == 0;
        if (!empty) continue;
        // loss_ranking of the last assignment pass (vq.hpp:221-229)
        uint32_t* cnt_copy = nullptr;
        cudaMallocAsync(&cnt_copy, M * k * sizeof(uint32_t), s->stream);
        cudaMemcpyAsync(cnt_copy, hc.data(), M * k * sizeof(uint32_t), cudaMemcpyHostToDevice,
                        s->stream);
        k_iota2<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(order, n);
        s->launches++;
        st = sort_scores_desc(s, losses + m * n, order, n);
        if (st == AQ_OK) {
          if (ds->f64)
            k_kmeans_reseed<double><<<1, 1, 0, s->stream>>>(cnt_copy, (int)m, (int)k, (int)sd,
                                                            order, ds->xr64, (int)d, cb->d64);
          else
            k_kmeans_reseed<float><<<1, 1, 0, s->stream>>>(cnt_copy, (int)m, (int)k, (int)sd,
                                                           order, ds->xr, (int)d, cb->d64);
          s->launches++;
        }
        cudaFreeAsync(cnt_copy, s->stream);
      }
    }
    if (st != AQ_OK) break;
    hprev = htot;
    st = assign();
    if (st != AQ_OK) break;
    for (size_t m = 0; m < M; ++m) {
      if (!hact[m]) continue;
      if (hchg[m] == 0) {
        hact[m] = 0;
        continue;
      }
      if (cfg->relative_tolerance > 0.0 &&
          (hprev[m] == 0.0 || hprev[m] - htot[m] <= cfg->relative_tolerance * hprev[m]))
        hact[m] = 0;
    }
  }
  cudaFreeAsync(losses, s->stream);
  cudaFreeAsync(totals, s->stream);
  cudaFreeAsync(changes, s->stream);
  cudaFreeAsync(active, s->stream);
  cudaFreeAsync(didx, s->stream);
  cudaFreeAsync(order, s->stream);
  if (st == AQ_OK) st = stage_codebook(cb);
  cudaStreamSynchronize(s->stream);
  if (st != AQ_OK) {
    aq_codebook_free(cb);
    aq_codes_free(codes);
    return st;
  }
  *cb_out = cb;
  *codes_out = codes;
  return AQ_OK;
}

}  // namespace aqd

using namespace aqd;

extern "C" {

int aq_dev_train_l2_pq(aq_dataset* ds, size_t M, size_t k, const aq_train_config* cfg,
                       aq_codebook** cb_out, aq_codes** codes_out) {
  if (!ds || !cfg || !cb_out || !codes_out) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  AQ_TRY(check_session(ds->s));
  return train_l2_pq_device(ds, M, k, cfg, cb_out, codes_out);
}

// train_apq (pq.hpp:513-575). history_out must hold max_iterations + 1 values.
int aq_dev_train_apq(aq_dataset* ds, size_t M, size_t k, const aq_weights* w,
                     const aq_train_config* cfg, int warm_start, aq_codebook** cb_out,
                     aq_codes** codes_out, double* history_out, size_t* history_len) {
  if (!ds || !cfg || !cb_out || !codes_out) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t n = ds->n, d = ds->d;
  if (n == 0) return ref_error(AQ_E_EMPTY_DATASET, "cannot train on an empty dataset");
  if (M == 0 || d % M != 0) return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  if (k == 0 || k > n) return ref_error(AQ_E_INVALID_ARGUMENT, "need 1 <= k <= n");
  if (history_len) *history_len = 0;
  const size_t sd = d / M;
  aq_codebook* cb = nullptr;
  aq_codes* codes = nullptr;
  if (warm_start) {
    timer_mark(s, AQ_T_KMEANS);
    AQ_TRY(train_l2_pq_device(ds, M, k, cfg, &cb, &codes));
    timer_mark(s, AQ_T_KMEANS);
  } else {
    // one generator, one sample_distinct per subspace (pq.hpp:533-542)
    HostRng r{cfg->seed};
    std::vector<uint64_t> hidx(M * k);
    for (size_t m = 0; m < M; ++m) {
      const auto v = r.sample_distinct(n, k);
      for (size_t j = 0; j < k; ++j) hidx[m * k + j] = v[j];
    }
    AQ_TRY(aq_codebook_upload(s, nullptr, M, k, sd, &cb));
    uint64_t* didx = nullptr;
    AQ_CUDA(cudaMallocAsync(&didx, M * k * sizeof(uint64_t), s->stream));
    AQ_CUDA(cudaMemcpyAsync(didx, hidx.data(), M * k * sizeof(uint64_t), cudaMemcpyHostToDevice,
                            s->stream));
    AQ_XR_LAUNCH(ds, k_init_codewords, (unsigned)((M * k + 127) / 128), 128, 0, s->stream,
                 (int)d, (int)M, (int)k, (int)sd, didx, cb->d64);
    s->launches++;
    cudaFreeAsync(didx, s->stream);
    int st = stage_codebook(cb);
    if (st == AQ_OK) st = aq_codes_alloc(s, n, M, k, &codes);
    // reconstruction_nearest_pass (pq.hpp:547): the encoder with 0 sweeps
    aq_weights iso{AQ_WEIGHTS_UNIFORM, 1.0, 1.0, nullptr, nullptr, 0.0, 0};
    if (st == AQ_OK) st = run_encode(ds, cb, &iso, codes, 0, 0, 0, nullptr, nullptr);
    if (st != AQ_OK) {
      aq_codebook_free(cb);
      aq_codes_free(codes);
      return st;
    }
  }
  double* losses = nullptr;
  double* total = nullptr;
  int st = AQ_OK;
  if (cudaMallocAsync(&losses, n * sizeof(double), s->stream) != cudaSuccess ||
      cudaMallocAsync(&total, sizeof(double), s->stream) != cudaSuccess)
    st = ref_error(AQ_E_CUDA, "out of device memory");
  // Assignment pass on the main stream; its loss total (a point-ordered
  // float64 chain, the slowest part of a pass) runs on the side stream so
  // the next codebook update can overlap it. The next pass waits for the sum
  // before it overwrites `losses`.
  auto pass_async = [&](uint64_t* changed) -> int {
    AQ_CUDA(cudaStreamWaitEvent(s->stream, s->ev_side, 0));
    AQ_TRY(run_encode(ds, cb, w, codes, 1, 0, cfg->sweep_to_fixed_point, losses, changed));
    AQ_CUDA(cudaEventRecord(s->ev_main, s->stream));
    AQ_CUDA(cudaStreamWaitEvent(s->side, s->ev_main, 0));
    AQ_TRY(seq_sums_on(s, s->side, losses, n, n, 1, nullptr, total, 0.0));
    AQ_CUDA(cudaMemcpyAsync(s->sum_host, total, sizeof(double), cudaMemcpyDeviceToHost, s->side));
    AQ_CUDA(cudaEventRecord(s->ev_side, s->side));
    return AQ_OK;
  };
  auto get_total = [&](double* tot_h) -> int {
    AQ_CUDA(cudaEventSynchronize(s->ev_side));
    *tot_h = s->sum_host[0];
    return AQ_OK;
  };
  double tot = 0.0;
  uint64_t changed = 0;
  size_t hl = 0;
  if (st == AQ_OK) st = pass_async(&changed);
  if (st == AQ_OK) st = get_total(&tot);
  if (st == AQ_OK && history_out) history_out[hl] = tot;
  if (st == AQ_OK) ++hl;
  aq_codebook* next = nullptr;
  if (st == AQ_OK) st = aq_codebook_upload(s, nullptr, M, k, sd, &next);
  bool have_next = false;  // `next` already holds the update of the current codes
  // AQ_TRACE=1: host wall time of each step of an iteration (stderr)
  static const bool trace = getenv("AQ_TRACE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  for (int iter = 0; st == AQ_OK && iter < cfg->max_iterations; ++iter) {
    const auto t0 = now();
    if (!have_next) st = aq_dev_pq_codebook_update(ds, codes, w, cfg->ridge, next);
    if (st != AQ_OK) break;
    const auto t1 = now();
    std::swap(cb, next);
    have_next = false;
    const double prev = tot;
    st = pass_async(&changed);
    if (st != AQ_OK) break;
    const auto t2 = now();
    // speculative next update (a pure function of the codes) while the
    // total is summed; discarded when the stopping rule fires below
    if (changed != 0 && iter + 1 < cfg->max_iterations) {
      st = aq_dev_pq_codebook_update(ds, codes, w, cfg->ridge, next);
      if (st != AQ_OK) break;
      have_next = true;
    }
    const auto t3 = now();
    st = get_total(&tot);
    if (st != AQ_OK) break;
    if (trace)
      fprintf(stderr, "[aq] iter %d: update %.1f ms, pass %.1f ms, spec update %.1f ms, total %.1f ms\n",
              iter, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, now()));
    if (history_out) history_out[hl] = tot;
    ++hl;
    if (changed == 0) break;
    if (cfg->relative_tolerance > 0.0 &&
        (prev == 0.0 || prev - tot <= cfg->relative_tolerance * prev))
      break;
  }
  cudaStreamSynchronize(s->side);
  if (history_len) *history_len = hl;
  aq_codebook_free(next);
  if (losses) cudaFreeAsync(losses, s->stream);
  if (total) cudaFreeAsync(total, s->stream);
  cudaStreamSynchronize(s->stream);
  if (st != AQ_OK) {
    aq_codebook_free(cb);
    aq_codes_free(codes);
    return st;
  }
  *cb_out = cb;
  *codes_out = codes;
  return AQ_OK;
}

// train_avq (vq.hpp:243-329): anisotropic vector quantization, i.e. one
// full-dimensional codebook (returned as M = 1). The assignment pass is the
// M = 1 encoder pass (pq_assign_pass with M = 1 is vq_assign_pass bit for
// bit: test_pq.cpp:79-95); the update is the per-codeword closed form with the
// VQ empty-partition policy: keep the codeword, or reseed from the ranking of
// the previous pass's losses (vq.hpp:276-292).
int aq_dev_train_avq(aq_dataset* ds, size_t k, const aq_weights* w, const aq_train_config* cfg,
                     aq_codebook** cb_out, aq_codes** codes_out, double* history_out,
                     size_t* history_len) {
  if (!ds || !cfg || !cb_out || !codes_out) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t n = ds->n, d = ds->d;
  if (history_len) *history_len = 0;
  if (n == 0) return ref_error(AQ_E_EMPTY_DATASET, "cannot train on an empty dataset");
  if (k == 0 || k > n)
    return ref_error(AQ_E_INVALID_ARGUMENT, "need 1 <= k <= n (codewords come from datapoints)");
  // codewords = rows Rng(seed).sample_distinct(n, k) (vq.hpp:257-264)
  HostRng r{cfg->seed};
  const auto v = r.sample_distinct(n, k);
  std::vector<uint64_t> hidx(v.begin(), v.end());
  aq_codebook* cb = nullptr;
  aq_codebook* next = nullptr;
  aq_codes* codes = nullptr;
  double* losses = nullptr;
  double* total = nullptr;
  uint64_t* didx = nullptr;
  int st = aq_codebook_upload(s, nullptr, 1, k, d, &cb);
  if (st == AQ_OK) st = aq_codebook_upload(s, nullptr, 1, k, d, &next);
  if (st == AQ_OK) st = aq_codes_alloc(s, n, 1, k, &codes);
  if (st == AQ_OK &&
      (cudaMallocAsync(&didx, k * sizeof(uint64_t), s->stream) != cudaSuccess ||
       cudaMallocAsync(&losses, n * sizeof(double), s->stream) != cudaSuccess ||
       cudaMallocAsync(&total, sizeof(double), s->stream) != cudaSuccess))
    st = ref_error(AQ_E_CUDA, "out of device memory");
  if (st == AQ_OK) {
    cudaMemcpyAsync(didx, hidx.data(), k * sizeof(uint64_t), cudaMemcpyHostToDevice, s->stream);
    AQ_XR_LAUNCH(ds, k_init_codewords, (unsigned)((k + 127) / 128), 128, 0, s->stream, (int)d,
                 1, (int)k, (int)d, didx, cb->d64);
    s->launches++;
    st = stage_codebook(cb);
  }
  const bool keep = cfg->empty_partition_policy == 1;
  size_t hl = 0;
  double tot = 0.0;
  uint64_t changed = 0;
  auto pass = [&]() -> int {
    AQ_TRY(run_encode(ds, cb, w, codes, 1, 0, 0, losses, &changed));
    AQ_TRY(seq_sum_device(s, losses, n, 0.0, total));
    AQ_CUDA(cudaMemcpyAsync(&tot, total, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    AQ_CUDA(cudaStreamSynchronize(s->stream));
    if (history_out) history_out[hl] = tot;
    ++hl;
    return AQ_OK;
  };
  if (st == AQ_OK) st = pass();
  for (int iter = 0; st == AQ_OK && iter < cfg->max_iterations; ++iter) {
    st = avq_codebook_update(ds, codes, w, cfg->ridge, next, keep ? nullptr : losses,
                             keep ? cb->d64 : nullptr);
    if (st != AQ_OK) break;
    std::swap(cb, next);
    const double prev = tot;
    st = pass();
    if (st != AQ_OK) break;
    if (changed == 0) break;
    if (cfg->relative_tolerance > 0.0 &&
        (prev == 0.0 || prev - tot <= cfg->relative_tolerance * prev))
      break;
  }
  if (history_len) *history_len = hl;
  aq_codebook_free(next);
  if (didx) cudaFreeAsync(didx, s->stream);
  if (losses) cudaFreeAsync(losses, s->stream);
  if (total) cudaFreeAsync(total, s->stream);
  cudaStreamSynchronize(s->stream);
  if (st != AQ_OK) {
    aq_codebook_free(cb);
    aq_codes_free(codes);
    return st;
  }
  *cb_out = cb;
  *codes_out = codes;
  return AQ_OK;
}

// One k-means assignment pass over this dataset's points for the active
// subspaces (sharded warm start): codes updated in place, losses (M x n,
// device) written for active subspaces, changes_out[m] = codes changed.
int aq_dev_kmeans_assign(aq_dataset* ds, aq_codebook* cb, aq_codes* codes,
                         const int* active_host, double* losses_dev, uint64_t* changes_out) {
  if (!ds || !cb || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t M = cb->M, n = ds->n;
  if (ds->d != M * cb->sd || codes->n != n || codes->M != M)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "shapes do not match");
  if (cb->sd > 16 || cb->k > 256)
    return ref_error(AQ_E_UNSUPPORTED, "device trainers support k <= 256, sub_dimension <= 16");
  int* act = nullptr;
  unsigned long long* chg = nullptr;
  AQ_CUDA(cudaMallocAsync(&act, M * sizeof(int), s->stream));
  AQ_CUDA(cudaMallocAsync(&chg, M * sizeof(unsigned long long), s->stream));
  AQ_CUDA(cudaMemcpyAsync(act, active_host, M * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  AQ_CUDA(cudaMemsetAsync(chg, 0, M * sizeof(unsigned long long), s->stream));
  if (n) {
    if (cb->sd == 2 && codes->bits == 4 && !ds->f64) {
      const size_t sm = (size_t)M * cb->k * sizeof(double2) + 2 * M * sizeof(int);
      AQ_CUDA(cudaFuncSetAttribute(k_kmeans_assign_sd2,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_kmeans_assign_sd2<<<(unsigned)((n + 255) / 256), 256, sm, s->stream>>>(
          reinterpret_cast<const float2*>(ds->xt), n, (int)(ds->d / 2), (int)M, (int)cb->k,
          cb->d64, act, codes->data, (int)codes->stride, losses_dev, chg);
    } else {
      AQ_XR_LAUNCH(ds, k_kmeans_assign, (unsigned)((n + 127) / 128), 128, 0, s->stream, n,
                   (int)ds->d, (int)M, (int)cb->k, (int)cb->sd, cb->d64, act, codes->data,
                   (int)codes->stride, codes->bits, losses_dev, chg);
    }
    s->launches++;
  }
  AQ_CUDA(cudaMemcpyAsync(changes_out, chg, M * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                          s->stream));
  cudaFreeAsync(act, s->stream);
  cudaFreeAsync(chg, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

}  // extern "C"

