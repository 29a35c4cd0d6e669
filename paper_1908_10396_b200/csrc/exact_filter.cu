// Exact MIPS through a bounded float32 filter (exact_search / exact_ground_truth,
// index.hpp:137-162). Same contract as exact.cu — float64 scores in
// detail::dot's order (geometry.hpp:170-174), hits ordered by (score desc,
// index asc) — at float32 FMA speed:
//
//   filter   f_p = fma chain of (float) q_j and x_j (x is float32-exact), per
//            (query block of 16, point slice) CTA; |f_p - s_p| <= B for every
//            point, B = 1.01 (d + 2) 2^-24 |q| max|x| + 1e-30 (query rounding,
//            d float32 roundings, the reference's own float64 roundings,
//            Cauchy-Schwarz on sum |q_j x_j|);
//   window   theta = the N-th largest f; every exact top-N point has
//            f >= theta - 2B (>= N points have s >= theta - B, so the N-th
//            exact score is >= theta - B, and f_p >= s_p - B). Each CTA keeps
//            f >= theta_cta - 2B (theta_cta <= theta), so the union holds
//            every candidate;
//   merge    per query: global theta, the window re-scored in float64 in the
//            reference's order, bitonic sort on (score desc, index asc).
//
// Windows that overflow (massive ties) fall back to the all-scores path.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace aqd {

#ifndef AQ_FQ
#define AQ_FQ 32
#endif
constexpr int kFQ = AQ_FQ;     // queries per CTA
constexpr int kFTile = 256;    // points per tile (= threads)
constexpr int kFPPT = 4;       // tiles between barriers
constexpr int kFMaxN = 4096;
constexpr int kFMergeCapMin = 2048, kFMergeCapMax = 8192;  // merge window (shared)

__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float funkey(uint32_t k) {
  return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}

// N-th largest key among buf[0..cnt) (warp-cooperative); false when cnt < N
__device__ bool warp_nth_key32(const uint2* buf, int cnt, int N, uint32_t* out) {
  if (cnt < N) return false;
  const int lane = threadIdx.x & 31;
  uint32_t T = 0u;
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t cand = T | (1u << bit);
    int c = 0;
    for (int e = lane; e < cnt; e += 32) c += buf[e].x >= cand;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= N) T = cand;
  }
  *out = T;
  return true;
}

__device__ int warp_keep_key32(uint2* buf, int cnt, uint32_t cut) {
  const int lane = threadIdx.x & 31;
  int kept = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int e = base + lane;
    uint2 v = make_uint2(0, 0);
    bool keep = false;
    if (e < cnt) {
      v = buf[e];
      keep = v.x >= cut;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) buf[kept + __popc(bal & ((1u << lane) - 1u))] = v;
    kept += __popc(bal);
    __syncwarp();
  }
  return kept;
}

// window cut for a local/global N-th filter score: key of (theta - 2B),
// rounded down so the window only grows
__device__ __forceinline__ uint32_t window_cut(uint32_t theta_key, float twoB) {
  const float th = funkey(theta_key);
  return fkey(__fsub_rd(th, twoB));
}

struct FArgs {
  const float* xt;       // pair-tiled rows
  int pairs, d;
  size_t n;
  const float* qf;       // [nqb][d][kFQ] float32 queries
  const float* twoB;     // [nq_pad] 2 B per query
  int nq, N, cap, R;
  size_t chunk;          // persistent slices of (query block, point) space
  int nqb;
  int mcap;              // merge window: power of two, kFMergeCapMin..kFMergeCapMax
  uint2* out_buf;        // [q][r][cap] {key, index}
  int* out_cnt;          // [q][r]
  int* out_flag;         // [q]
};

__global__ void __launch_bounds__(kFTile, 2) k_exact_filter(const FArgs a) {
  extern __shared__ __align__(16) unsigned char fsm[];
  float* qs = reinterpret_cast<float*>(fsm);  // [d][kFQ]
  uint32_t* cut = reinterpret_cast<uint32_t*>(qs + (size_t)a.d * kFQ);
  int* cnt = reinterpret_cast<int*>(cut + kFQ);
  int* flag = cnt + kFQ;
  float* tb2 = reinterpret_cast<float*>(flag + kFQ);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t total = (size_t)a.nqb * a.n;
  size_t Lpos = (size_t)blockIdx.x * a.chunk;
  const size_t Lend = min(total, Lpos + a.chunk);
  while (Lpos < Lend) {
    const int qb = (int)(Lpos / a.n);
    const size_t start = Lpos % a.n;
    const size_t end = min(a.n, start + (Lend - Lpos));
    const int r = (int)(blockIdx.x - ((size_t)qb * a.n) / a.chunk);
    Lpos += end - start;
    __syncthreads();
    {
      const float4* src = reinterpret_cast<const float4*>(a.qf + (size_t)qb * a.d * kFQ);
      float4* dst = reinterpret_cast<float4*>(qs);
      for (int t = threadIdx.x; t < a.d * kFQ / 4; t += blockDim.x) dst[t] = src[t];
    }
    if (threadIdx.x < kFQ) {
      cut[threadIdx.x] = 0u;
      cnt[threadIdx.x] = 0;
      flag[threadIdx.x] = 0;
      tb2[threadIdx.x] = a.twoB[qb * kFQ + threadIdx.x];
    }
    __syncthreads();
    uint2* const buf = a.out_buf + ((size_t)qb * kFQ * a.R + r) * a.cap;
    const size_t qstride = (size_t)a.R * a.cap;
    const int cap = a.cap;
    constexpr int SPAN = kFTile * kFPPT;
    for (size_t tb = start; tb < end;) {
      const int nu = tb == start ? 1 : kFPPT;
#pragma unroll 1
      for (int u = 0; u < nu; ++u) {
        const size_t p = tb + (size_t)u * kFTile + threadIdx.x;
        if (p < end) {
          // query pairs per packed FMA (FFMA2); the bound covers any rounding order
          float2 f2[kFQ / 2];
#pragma unroll
          for (int q = 0; q < kFQ / 2; ++q) f2[q] = make_float2(0.0f, 0.0f);
          const float2* xrow =
              reinterpret_cast<const float2*>(a.xt) + (p >> 5) * (size_t)a.pairs * 32 + (p & 31);
#pragma unroll 4
          for (int jp = 0; jp < a.pairs; ++jp) {
            const float2 xv = xrow[(size_t)jp * 32];
            const float4* q0 = reinterpret_cast<const float4*>(qs + (size_t)(2 * jp) * kFQ);
            const float2 xa = make_float2(xv.x, xv.x);
#pragma unroll
            for (int v = 0; v < kFQ / 4; ++v) {
              const float4 qq = q0[v];
              f2[2 * v] = __ffma2_rn(make_float2(qq.x, qq.y), xa, f2[2 * v]);
              f2[2 * v + 1] = __ffma2_rn(make_float2(qq.z, qq.w), xa, f2[2 * v + 1]);
            }
            if (2 * jp + 1 < a.d) {
              const float4* q1 = reinterpret_cast<const float4*>(qs + (size_t)(2 * jp + 1) * kFQ);
              const float2 xb = make_float2(xv.y, xv.y);
#pragma unroll
              for (int v = 0; v < kFQ / 4; ++v) {
                const float4 qq = q1[v];
                f2[2 * v] = __ffma2_rn(make_float2(qq.x, qq.y), xb, f2[2 * v]);
                f2[2 * v + 1] = __ffma2_rn(make_float2(qq.z, qq.w), xb, f2[2 * v + 1]);
              }
            }
          }
          float f[kFQ];
#pragma unroll
          for (int q = 0; q < kFQ / 2; ++q) {
            f[2 * q] = f2[q].x;
            f[2 * q + 1] = f2[q].y;
          }
#pragma unroll
          for (int q = 0; q < kFQ; ++q) {
            const uint32_t key = fkey(f[q]);
            if (key >= cut[q]) {
              const int pos = atomicAdd(&cnt[q], 1);
              if (pos < cap)
                buf[q * qstride + pos] = make_uint2(key, (unsigned)p);
              else
                flag[q] = 1;
            }
          }
        }
      }
      tb += (size_t)nu * kFTile;
      __syncthreads();
      for (int q = warp; q < kFQ; q += kFTile / 32) {
        const int c = min(cnt[q], cap);
        uint32_t th;
        if (c > cap - SPAN && !flag[q] && warp_nth_key32(buf + q * qstride, c, a.N, &th)) {
          const uint32_t cq = max(cut[q], window_cut(th, tb2[q]));
          const int kept = warp_keep_key32(buf + q * qstride, c, cq);
          if (lane == 0) {
            cut[q] = cq;
            cnt[q] = kept;
            if (kept > cap - SPAN) flag[q] = 1;  // window too large: ties
          }
        }
        __syncwarp();
      }
      __syncthreads();
    }
    for (int q = warp; q < kFQ; q += kFTile / 32) {
      const int gq = qb * kFQ + q;
      int c = min(cnt[q], cap);
      uint32_t th;
      if (warp_nth_key32(buf + q * qstride, c, a.N, &th))
        c = warp_keep_key32(buf + q * qstride, c, max(cut[q], window_cut(th, tb2[q])));
      if (gq < a.nq && lane == 0) {
        a.out_cnt[(size_t)gq * a.R + r] = c;
        if (flag[q]) atomicOr(&a.out_flag[gq], 1);
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ unsigned long long d2o64(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Per query: global window, float64 re-scoring (detail::dot order), exact sort.
__global__ void __launch_bounds__(1024) k_exact_fmerge(const FArgs a, const float* xr,
                                                       const double* Q, int topn_eff,
                                                       uint32_t* ids, double* scores) {
  extern __shared__ __align__(16) unsigned char msm[];
  unsigned long long* K = reinterpret_cast<unsigned long long*>(msm);
  uint32_t* I = reinterpret_cast<uint32_t*>(K + a.mcap);
  __shared__ int ncol;
  const int q = blockIdx.x;
  if (a.out_flag[q]) return;
  const int tid = threadIdx.x;
  const uint2* lists = a.out_buf + (size_t)q * a.R * a.cap;
  const int* cn = a.out_cnt + (size_t)q * a.R;
  int total = 0;
  for (int r = tid & 31; r < a.R; r += 32) total += cn[r];  // each warp, redundantly
  total = __reduce_add_sync(0xffffffffu, total);
  uint32_t cutk = 0u;
  if (total >= a.N)  // radix select; the histogram borrows the sort-key space
    cutk = window_cut(block_nth_largest(lists, cn, a.R, a.cap, a.N,
                                        reinterpret_cast<unsigned*>(K)),
                      a.twoB[q]);
  if (tid == 0) ncol = 0;
  __syncthreads();
  for (int r = tid >> 5; r < a.R; r += blockDim.x >> 5)  // warp per window
    for (int e = tid & 31; e < cn[r]; e += 32) {
      const uint2 v = lists[(size_t)r * a.cap + e];
      if (v.x >= cutk) {
        const int pos = atomicAdd(&ncol, 1);
        if (pos < a.mcap) I[pos] = v.y;
      }
    }
  __syncthreads();
  const int nc = ncol;
  if (nc > a.mcap) {
    if (tid == 0) a.out_flag[q] = 2;
    return;
  }
  const double* qv = Q + (size_t)q * a.d;
  for (int e = tid; e < nc; e += blockDim.x) {
    const float* x = xr + (size_t)I[e] * a.d;
    double s = 0.0;  // detail::dot (geometry.hpp:170-174)
    for (int j = 0; j < a.d; ++j) s = __dadd_rn(s, __dmul_rn(qv[j], (double)x[j]));
    K[e] = ~d2o64(s);  // ascending == score descending
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
    unsigned long long b = ~K[e];
    b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    ids[(size_t)q * topn_eff + e] = I[e];
    scores[(size_t)q * topn_eff + e] = __longlong_as_double((long long)b);
  }
}

// float32 query blocks [nqb][d][16] and 2 B per query; returns 0 for a query
// whose entries do not fit float32 (then the caller keeps the exact path)
__global__ void k_filter_queries(const double* Q, int nq, int d, double xmax, float* qf,
                                 float* twoB, int* flag) {
  const int q = blockIdx.x;  // padded query index
  const int qb = q / kFQ, qi = q % kFQ;
  __shared__ double red[32];
  double ss = 0.0;
  bool ok = true;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const double v = q < nq ? Q[(size_t)q * d + j] : 0.0;
    ok &= fabs(v) < 1e30;
    qf[((size_t)qb * d + j) * kFQ + qi] = (float)v;
    ss += v * v;
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const unsigned okb = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = okb == 0xffffffffu ? ss : -1.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    bool all = true;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (red[w] < 0.0) all = false;
      t += red[w] < 0.0 ? 0.0 : red[w];
    }
    // 1.01 (d + 2) 2^-24 |q| max|x|, |q| rounded up generously
    const double B = 1.01 * (d + 2) * 5.9604644775390625e-08 * sqrt(t) * 1.0000001 * xmax + 1e-30;
    twoB[q] = (float)(2.0 * B * (1.0 + 1e-6));
    if (!all && q < nq) flag[q] = 4;
  }
}

int exact_filter_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                        double* scores, std::vector<int>& hflag, bool* ran) {
  *ran = false;
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const size_t te = std::min(depth, n);
  const int N = (int)te;
  const size_t nqb = (nq + kFQ - 1) / kFQ, nq_pad = nqb * kFQ;
  // max |x| over the rows (norms are the reference's float64 norms)
  std::vector<double> hn(n);
  AQ_CUDA(cudaMemcpyAsync(hn.data(), ds->norms, n * sizeof(double), cudaMemcpyDeviceToHost,
                          s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  double xmax = 0.0;
  for (double v : hn) xmax = std::max(xmax, v);
  xmax *= 1.0000001;
  if (!(xmax < 1e30) || depth > (size_t)kFMaxN) return AQ_OK;  // caller's exact path
  // window: N, one span of appends, tie room growing with N (search.cu)
  const int cap = ((N + 31) & ~31) + kFTile * kFPPT + 32 + (N > 128 ? N : 0);
  const size_t G0 = (size_t)s->num_sms * 2;
  const size_t total = nqb * n;
  const size_t chunk = std::max<size_t>((total + G0 - 1) / G0, 16 * (size_t)kFTile);
  const size_t G = (total + chunk - 1) / chunk;
  size_t R = 1;
  for (size_t qb = 0; qb < nqb; ++qb)
    R = std::max(R, ((qb + 1) * n - 1) / chunk - qb * n / chunk + 1);
  const size_t qf_b = nqb * d * kFQ * sizeof(float), tb_b = nq_pad * sizeof(float);
  const size_t buf_b = nq_pad * R * cap * sizeof(uint2);
  void* p;
  // the filter kernel stages its query tile with 16-byte loads
  const size_t qf_off = (buf_b + 255) & ~(size_t)255;
  AQ_TRY(scratch(s, 3, qf_off + qf_b + tb_b + nq * R * sizeof(int) + nq * sizeof(int) + 256, &p));
  uint2* obuf = (uint2*)p;
  float* qf = (float*)((char*)p + qf_off);
  float* twoB = qf + nqb * d * kFQ;
  int* ocnt = (int*)(twoB + nq_pad);
  int* oflag = ocnt + nq * R;
  AQ_CUDA(cudaMemsetAsync(oflag, 0, nq * sizeof(int), s->stream));
  AQ_CUDA(cudaMemsetAsync(ocnt, 0, nq * R * sizeof(int), s->stream));
  k_filter_queries<<<(unsigned)nq_pad, 128, 0, s->stream>>>(Qd, (int)nq, (int)d, xmax, qf, twoB,
                                                            oflag);
  AQ_LAUNCHED(s);
  int mcap = kFMergeCapMin;
  while (mcap < N + N / 2 + 1024 && mcap < kFMergeCapMax) mcap <<= 1;
  FArgs a{ds->xt, (int)pairs_of(d), (int)d, n, qf, twoB, (int)nq, N, cap, (int)R,
          chunk, (int)nqb, mcap, obuf, ocnt, oflag};
  const size_t msmem = (size_t)mcap * (sizeof(unsigned long long) + sizeof(uint32_t));
  const size_t smem = (size_t)d * kFQ * sizeof(float) + kFQ * 16 + 64;
  if (smem > 200 * 1024) return AQ_OK;
  AQ_CUDA(cudaFuncSetAttribute(k_exact_filter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  timer_mark(s, AQ_T_EXACT);
  k_exact_filter<<<(unsigned)G, kFTile, smem, s->stream>>>(a);
  AQ_LAUNCHED(s);
  AQ_CUDA(cudaFuncSetAttribute(k_exact_fmerge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)msmem));
  k_exact_fmerge<<<(unsigned)nq, R >= 32 ? 1024 : 256, msmem, s->stream>>>(a, ds->xr, Qd, (int)te,
                                                                         ids, scores);
  AQ_LAUNCHED(s);
  timer_mark(s, AQ_T_EXACT);
  AQ_CUDA(cudaMemcpyAsync(hflag.data(), oflag, nq * sizeof(int), cudaMemcpyDeviceToHost,
                          s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  *ran = true;
  return AQ_OK;
}

}  // namespace aqd
