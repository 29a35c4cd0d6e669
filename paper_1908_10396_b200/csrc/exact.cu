// Brute-force exact MIPS (exact_search / exact_ground_truth, index.hpp:137-162)
// and the single-point coordinate-descent API (pq_assign_point, pq.hpp:256-282).
//
// Exact search computes every score in float64 with detail::dot's order
// (geometry.hpp:170-174: s = 0, s += q_j x_j, j ascending, no contraction).
// Per (query block, point range) CTA, a per-query buffer keeps every point
// whose score is >= theta (the N-th largest score seen so far, ties kept);
// the merge kernel selects and sorts the union exactly (score desc, index
// asc). Scores are exact, so no window margin is needed.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace aqd {

int sort_scores_desc(aq_session* s, const double* scores, uint32_t* idx, size_t n);
int exact_filter_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                        double* scores, std::vector<int>& hflag, bool* ran);

constexpr int kXQ = 16;       // queries per CTA
constexpr int kXTile = 256;   // points per tile
constexpr int kXMaxN = 512;
constexpr int kXMergeCap = 2048;

struct XEntry {
  unsigned long long key;  // order-preserving image of the float64 score
  uint32_t idx;
  uint32_t pad;
};

__device__ __forceinline__ unsigned long long d2o(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double o2d(unsigned long long o) {
  return __longlong_as_double((long long)((o >> 63) ? (o & 0x7fffffffffffffffull) : ~o));
}

__device__ bool warp_nth_key(const XEntry* buf, int cnt, int N, unsigned long long* out) {
  if (cnt < N) return false;
  const int lane = threadIdx.x & 31;
  unsigned long long T = 0ull;
  for (int bit = 63; bit >= 0; --bit) {
    const unsigned long long cand = T | (1ull << bit);
    int c = 0;
    for (int e = lane; e < cnt; e += 32) c += buf[e].key >= cand;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= N) T = cand;
  }
  *out = T;
  return true;
}

__device__ int warp_keep_ge(XEntry* buf, int cnt, unsigned long long cut) {
  const int lane = threadIdx.x & 31;
  int kept = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int e = base + lane;
    XEntry v{};
    bool keep = false;
    if (e < cnt) {
      v = buf[e];
      keep = v.key >= cut;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) buf[kept + __popc(bal & ((1u << lane) - 1u))] = v;
    kept += __popc(bal);
    __syncwarp();
  }
  return kept;
}

struct XArgs {
  const void* xt;  // pair-tiled rows, float or double (TX)
  int pairs, d;
  size_t n;
  const double* Q;
  int nq, N, cap;
  size_t range_len;
  int R;
  XEntry* out_buf;  // [q][r][cap]
  int* out_cnt;
  int* out_flag;
};

template <class TX>
__global__ void __launch_bounds__(kXTile, 1) k_exact_score(const XArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* qs = reinterpret_cast<double*>(smem);  // [d][kXQ]
  unsigned long long* cut = reinterpret_cast<unsigned long long*>(qs + (size_t)a.d * kXQ);
  int* cnt = reinterpret_cast<int*>(cut + kXQ);
  int* flag = cnt + kXQ;
  XEntry* buf = reinterpret_cast<XEntry*>(flag + kXQ + 2);  // 16-byte aligned
  const int qb = blockIdx.y, r = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < a.d * kXQ; e += blockDim.x) {
    const int j = e / kXQ, q = e % kXQ;
    const int gq = qb * kXQ + q;
    qs[e] = gq < a.nq ? a.Q[(size_t)gq * a.d + j] : 0.0;
  }
  if (threadIdx.x < kXQ) {
    cut[threadIdx.x] = 0ull;
    cnt[threadIdx.x] = 0;
    flag[threadIdx.x] = 0;
  }
  __syncthreads();
  const size_t start = (size_t)r * a.range_len;
  const size_t end = min(a.n, start + a.range_len);
  for (size_t tb = start; tb < end; tb += kXTile) {
    const size_t p = tb + threadIdx.x;
    if (p < end) {
      double s[kXQ];
#pragma unroll
      for (int q = 0; q < kXQ; ++q) s[q] = 0.0;
      const TX* xrow =
          static_cast<const TX*>(a.xt) + ((p >> 5) * a.pairs * 32 + (p & 31)) * 2;
      for (int j = 0; j < a.d; ++j) {
        const double xv = (double)xrow[(size_t)(j >> 1) * 64 + (j & 1)];
        const double2* qj = reinterpret_cast<const double2*>(qs + (size_t)j * kXQ);
#pragma unroll
        for (int q = 0; q < kXQ / 2; ++q) {
          const double2 qq = qj[q];
          s[2 * q] = __dadd_rn(s[2 * q], __dmul_rn(qq.x, xv));
          s[2 * q + 1] = __dadd_rn(s[2 * q + 1], __dmul_rn(qq.y, xv));
        }
      }
#pragma unroll
      for (int q = 0; q < kXQ; ++q) {
        const unsigned long long key = d2o(s[q]);
        if (key >= cut[q]) {
          const int pos = atomicAdd(&cnt[q], 1);
          if (pos < a.cap)
            buf[q * a.cap + pos] = XEntry{key, (uint32_t)p, 0u};
          else
            flag[q] = 1;
        }
      }
    }
    __syncthreads();
    for (int q = warp; q < kXQ; q += kXTile / 32) {
      const int c = min(cnt[q], a.cap);
      unsigned long long th;
      if (c > a.cap - kXTile && !flag[q] && warp_nth_key(buf + q * a.cap, c, a.N, &th)) {
        const unsigned long long cq = max(cut[q], th);
        const int kept = warp_keep_ge(buf + q * a.cap, c, cq);
        if (lane == 0) {
          cut[q] = cq;
          cnt[q] = kept;
          if (kept > a.cap - kXTile) flag[q] = 1;
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  for (int q = warp; q < kXQ; q += kXTile / 32) {
    const int gq = qb * kXQ + q;
    int c = min(cnt[q], a.cap);
    unsigned long long th;
    if (warp_nth_key(buf + q * a.cap, c, a.N, &th))
      c = warp_keep_ge(buf + q * a.cap, c, max(cut[q], th));
    if (gq < a.nq) {
      XEntry* dst = a.out_buf + ((size_t)gq * a.R + r) * a.cap;
      for (int e = lane; e < c; e += 32) dst[e] = buf[q * a.cap + e];
      if (lane == 0) {
        a.out_cnt[(size_t)gq * a.R + r] = c;
        if (flag[q]) atomicOr(&a.out_flag[gq], 1);
      }
    }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256) k_exact_merge(const XEntry* buf, const int* cnt,
                                                      int* flag, int R, int cap, int N,
                                                      int topn_eff, uint32_t* ids,
                                                      double* scores) {
  __shared__ unsigned long long K[kXMergeCap];
  __shared__ uint32_t I[kXMergeCap];
  __shared__ int red[32];
  __shared__ int ncol;
  const int q = blockIdx.x;
  if (flag[q]) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const XEntry* lists = buf + (size_t)q * R * cap;
  const int* cn = cnt + (size_t)q * R;
  int total = 0;
  for (int r = 0; r < R; ++r) total += cn[r];
  unsigned long long T = 0ull;
  if (total >= N) {
    for (int bit = 63; bit >= 0; --bit) {
      const unsigned long long cand = T | (1ull << bit);
      int c = 0;
      for (int r = 0; r < R; ++r)
        for (int e = tid; e < cn[r]; e += blockDim.x) c += lists[(size_t)r * cap + e].key >= cand;
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0) red[w] = c;
      __syncthreads();
      int tot = 0;
      for (int t = 0; t < (int)(blockDim.x >> 5); ++t) tot += red[t];
      __syncthreads();
      if (tot >= N) T = cand;
    }
  }
  if (tid == 0) ncol = 0;
  __syncthreads();
  for (int r = 0; r < R; ++r)
    for (int e = tid; e < cn[r]; e += blockDim.x) {
      const XEntry v = lists[(size_t)r * cap + e];
      if (v.key >= T) {
        const int pos = atomicAdd(&ncol, 1);
        if (pos < kXMergeCap) {
          K[pos] = ~v.key;  // ascending == score descending
          I[pos] = v.idx;
        }
      }
    }
  __syncthreads();
  const int nc = ncol;
  if (nc > kXMergeCap) {
    if (tid == 0) flag[q] = 2;
    return;
  }
  int P = 1;
  while (P < nc) P <<= 1;
  for (int e = nc + tid; e < P; e += blockDim.x) {
    K[e] = ~0ull;
    I[e] = 0xffffffffu;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = tid; e < P; e += blockDim.x) {
        const int o = e ^ stride;
        if (o > e) {
          const bool up = (e & size) == 0;
          const unsigned long long ka = K[e], kb = K[o];
          const uint32_t ia = I[e], ib = I[o];
          const bool gt = ka > kb || (ka == kb && ia > ib);
          if (gt == up) {
            K[e] = kb;
            K[o] = ka;
            I[e] = ib;
            I[o] = ia;
          }
        }
      }
      __syncthreads();
    }
  for (int e = tid; e < topn_eff; e += blockDim.x) {
    ids[(size_t)q * topn_eff + e] = I[e];
    scores[(size_t)q * topn_eff + e] = o2d(~K[e]);
  }
}

template <class TX>
__global__ void k_exact_all(const TX* xt, int pairs, int d, size_t n, const double* q,
                            double* out, uint32_t* idx) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < d; ++j)
    s = __dadd_rn(s, __dmul_rn(q[j], (double)xt[tiled_index(i, (size_t)j, (size_t)pairs)]));
  out[i] = s;
  idx[i] = (uint32_t)i;
}

__global__ void k_take(const uint32_t* idx, const double* by_point, int te, uint32_t* ids,
                       double* sc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < te) {
    ids[e] = idx[e];
    sc[e] = by_point[idx[e]];
  }
}

int exact_search_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth,
                        uint32_t* ids, double* scores) {
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const size_t te = std::min(depth, n);
  const int pairs = (int)pairs_of(d);
  std::vector<int> hflag(nq, 1);
  // float32 filter + float64 window (exact_filter.cu); AQ_EXACT_FILTER=0
  // keeps the all-float64 scoring kernel below
  static const int use_filter = getenv("AQ_EXACT_FILTER") ? atoi(getenv("AQ_EXACT_FILTER")) : 1;
  bool ran = false;
  // (float32 datasets only: the filter reads float32 rows)
  if (use_filter && !ds->f64)
    AQ_TRY(exact_filter_device(ds, Qd, nq, depth, ids, scores, hflag, &ran));
  const bool fast = !ran && depth <= (size_t)kXMaxN;
  if (fast) {
    const size_t nqb = (nq + kXQ - 1) / kXQ;
    const int N = (int)te;
    const int cap = ((N + 31) & ~31) + kXTile + 32;
    const size_t tiles = (n + kXTile - 1) / kXTile;
    size_t R = std::max<size_t>(1, (2 * (size_t)s->num_sms + nqb - 1) / nqb);
    R = std::min(R, tiles);
    const size_t range_len = ((tiles + R - 1) / R) * kXTile;
    R = (n + range_len - 1) / range_len;
    void* p;
    AQ_TRY(scratch(s, 3, nq * R * cap * sizeof(XEntry) + nq * R * 4 + nq * 4 + 256, &p));
    XEntry* obuf = (XEntry*)p;
    int* ocnt = (int*)(obuf + nq * R * cap);
    int* oflag = ocnt + nq * R;
    AQ_CUDA(cudaMemsetAsync(oflag, 0, nq * sizeof(int), s->stream));
    const void* xt = ds->f64 ? (const void*)ds->xt64 : (const void*)ds->xt;
    XArgs a{xt, pairs, (int)d, n, Qd, (int)nq, N, cap, range_len, (int)R, obuf, ocnt, oflag};
    const size_t smem = d * kXQ * sizeof(double) + kXQ * 8 + 2 * kXQ * 4 + 8 +
                        (size_t)kXQ * cap * sizeof(XEntry);
    if (smem <= 227 * 1024) {
      const dim3 grid((unsigned)R, (unsigned)nqb);
      if (ds->f64) {
        AQ_CUDA(cudaFuncSetAttribute(k_exact_score<double>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_exact_score<double><<<grid, kXTile, smem, s->stream>>>(a);
      } else {
        AQ_CUDA(cudaFuncSetAttribute(k_exact_score<float>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_exact_score<float><<<grid, kXTile, smem, s->stream>>>(a);
      }
      AQ_LAUNCHED(s);
      k_exact_merge<<<(unsigned)nq, 256, 0, s->stream>>>(obuf, ocnt, oflag, (int)R, cap, N,
                                                         (int)te, ids, scores);
      AQ_LAUNCHED(s);
      AQ_CUDA(cudaMemcpyAsync(hflag.data(), oflag, nq * sizeof(int), cudaMemcpyDeviceToHost,
                              s->stream));
      AQ_CUDA(cudaStreamSynchronize(s->stream));
    }
  }
  bool any = false;
  for (auto f : hflag) any |= f != 0;
  if (any) {
    void* p3;
    AQ_TRY(scratch(s, 4, n * (sizeof(double) + sizeof(uint32_t)) + 64, &p3));
    double* all = (double*)p3;
    uint32_t* idx = (uint32_t*)(all + n);
    for (size_t q = 0; q < nq; ++q) {
      if (!hflag[q]) continue;
      if (ds->f64)
        k_exact_all<double><<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(
            ds->xt64, pairs, (int)d, n, Qd + q * d, all, idx);
      else
        k_exact_all<float><<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(
            ds->xt, pairs, (int)d, n, Qd + q * d, all, idx);
      AQ_LAUNCHED(s);
      AQ_TRY(sort_scores_desc(s, all, idx, n));
      k_take<<<(unsigned)((te + 255) / 256), 256, 0, s->stream>>>(idx, all, (int)te,
                                                                 ids + q * te, scores + q * te);
      AQ_LAUNCHED(s);
    }
  }
  return AQ_OK;
}

// ---- pq_assign_point (pq.hpp:256-282): one point, float64 input ---------------------------

// order: sweep_order (pq.hpp:273-276; subspaces may repeat), or null for
// default_sweep (0..M-1)
__global__ void k_assign_point(const double* x, int M, int k, int sd, const double* cb,
                               double hp, double ho, double inv, unsigned* codes,
                               const unsigned long long* order, int norder) {
  if (threadIdx.x || blockIdx.x) return;
  const bool iso = hp == ho;
  double s2 = 0.0, s1 = 0.0;
  auto resid = [&](int m, int j, double* d2, double* rd) {
    double a = 0.0, b = 0.0;
    for (int t = 0; t < sd; ++t) {
      const double xv = x[m * sd + t];
      const double df = __dsub_rn(xv, cb[((size_t)m * k + j) * sd + t]);
      a = __dadd_rn(a, __dmul_rn(df, df));
      b = __dadd_rn(b, __dmul_rn(df, xv));
    }
    *d2 = a;
    *rd = b;
  };
  for (int m = 0; m < M; ++m) {
    double t2, t1;
    resid(m, (int)codes[m], &t2, &t1);
    s2 = __dadd_rn(s2, t2);
    s1 = __dadd_rn(s1, t1);
  }
  for (int step = 0; step < norder; ++step) {
    const int m = order ? (int)order[step] : step;
    double t2, t1;
    resid(m, (int)codes[m], &t2, &t1);
    const double base2 = __dsub_rn(s2, t2), base1 = __dsub_rn(s1, t1);
    unsigned bj = 0;
    double bs = 0.0, b2 = 0.0, b1 = 0.0;
    for (int j = 0; j < k; ++j) {
      double c2, c1;
      resid(m, j, &c2, &c1);
      const double sc = iso ? c2
                            : combined_loss(__dadd_rn(base2, c2), __dadd_rn(base1, c1), hp, ho,
                                            inv);
      if (j == 0 || sc < bs) {
        bs = sc;
        bj = (unsigned)j;
        b2 = c2;
        b1 = c1;
      }
    }
    codes[m] = bj;
    s2 = __dadd_rn(base2, b2);
    s1 = __dadd_rn(base1, b1);
  }
}

}  // namespace aqd

using namespace aqd;

extern "C" {

int aq_dev_exact_search(aq_dataset* ds, const double* queries, size_t nq, size_t depth,
                        uint32_t* ids_out, double* scores_out) {
  if (!ds) return ref_error(AQ_E_INVALID_ARGUMENT, "null dataset");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  if (ds->n == 0) return ref_error(AQ_E_EMPTY_DATASET, "empty dataset");
  if (depth < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  const size_t te = std::min(depth, ds->n), d = ds->d;
  if (nq == 0) return AQ_OK;
  double* Qd;
  uint32_t* ids;
  double* sc;
  AQ_CUDA(cudaMallocAsync(&Qd, nq * d * sizeof(double), s->stream));
  AQ_CUDA(cudaMallocAsync(&ids, nq * te * sizeof(uint32_t), s->stream));
  AQ_CUDA(cudaMallocAsync(&sc, nq * te * sizeof(double), s->stream));
  AQ_CUDA(cudaMemcpyAsync(Qd, queries, nq * d * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  int st = exact_search_device(ds, Qd, nq, depth, ids, sc);
  if (st == AQ_OK) {
    cudaMemcpyAsync(ids_out, ids, nq * te * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream);
    cudaMemcpyAsync(scores_out, sc, nq * te * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  }
  cudaFreeAsync(Qd, s->stream);
  cudaFreeAsync(ids, s->stream);
  cudaFreeAsync(sc, s->stream);
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (st == AQ_OK && e != cudaSuccess) {
    set_error(AQ_E_CUDA, "CUDA error %s", cudaGetErrorString(e));
    st = AQ_E_CUDA;
  }
  return st;
}

// pq_assign_point (pq.hpp:256-282): validation order of the reference, then
// one coordinate-descent pass in the default order.
int aq_pq_assign_point_order(aq_session* s, const double* x, size_t d, const uint32_t* current,
                             const double* dict, size_t M, size_t k, size_t sd, double hp,
                             double ho, const size_t* order, size_t order_len,
                             uint32_t* codes_out) {
  AQ_TRY(check_session(s));
  if (d != M * sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "datapoint dimension does not match codebook");
  for (size_t m = 0; m < M; ++m)
    if (current[m] >= k) return ref_error(AQ_E_CODE_OUT_OF_RANGE, "current code out of range");
  if (!(hp >= 0.0) || !(ho >= 0.0) || !std::isfinite(hp) || !std::isfinite(ho))
    return ref_error(AQ_E_INVALID_ARGUMENT, "h coefficients must be finite and >= 0");
  // the reference indexes codes[m] unchecked (undefined behaviour for m >= M)
  for (size_t t = 0; t < order_len; ++t)
    if (order[t] >= M) return ref_error(AQ_E_INVALID_ARGUMENT, "sweep order entry out of range");
  double inv = 0.0;
  if (hp != ho) {
    double n2 = 0.0;  // detail::norm2 = dot(x, x), sequential (geometry.hpp:176)
    for (size_t j = 0; j < d; ++j) n2 += x[j] * x[j];
    if (n2 == 0.0)
      return ref_error(AQ_E_ZERO_NORM_DATAPOINT, "anisotropic assignment undefined at |x| = 0");
    inv = 1.0 / n2;
  }
  double *dx, *dcb;
  unsigned* dc;
  unsigned long long* dord = nullptr;
  AQ_CUDA(cudaMallocAsync(&dx, d * sizeof(double) + 8, s->stream));
  AQ_CUDA(cudaMallocAsync(&dcb, M * k * sd * sizeof(double) + 8, s->stream));
  AQ_CUDA(cudaMallocAsync(&dc, M * sizeof(unsigned) + 8, s->stream));
  AQ_CUDA(cudaMemcpyAsync(dx, x, d * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  AQ_CUDA(cudaMemcpyAsync(dcb, dict, M * k * sd * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  AQ_CUDA(cudaMemcpyAsync(dc, current, M * sizeof(unsigned), cudaMemcpyHostToDevice, s->stream));
  std::vector<unsigned long long> hord(order, order + order_len);
  if (order_len) {
    AQ_CUDA(cudaMallocAsync(&dord, order_len * sizeof(unsigned long long), s->stream));
    AQ_CUDA(cudaMemcpyAsync(dord, hord.data(), order_len * sizeof(unsigned long long),
                            cudaMemcpyHostToDevice, s->stream));
  }
  k_assign_point<<<1, 32, 0, s->stream>>>(dx, (int)M, (int)k, (int)sd, dcb, hp, ho, inv, dc,
                                          dord, order_len ? (int)order_len : (int)M);
  s->launches++;
  AQ_CUDA(cudaGetLastError());
  AQ_CUDA(cudaMemcpyAsync(codes_out, dc, M * sizeof(unsigned), cudaMemcpyDeviceToHost, s->stream));
  cudaFreeAsync(dx, s->stream);
  cudaFreeAsync(dcb, s->stream);
  cudaFreeAsync(dc, s->stream);
  if (dord) cudaFreeAsync(dord, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

int aq_pq_assign_point(aq_session* s, const double* x, size_t d, const uint32_t* current,
                       const double* dict, size_t M, size_t k, size_t sd, double hp,
                       double ho, uint32_t* codes_out) {
  return aq_pq_assign_point_order(s, x, d, current, dict, M, k, sd, hp, ho, nullptr, 0,
                                  codes_out);
}

}  // extern "C"
