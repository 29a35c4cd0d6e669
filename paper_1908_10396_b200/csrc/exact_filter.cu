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
#include <cstring>
#include <vector>

#include <cuda_bf16.h>

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
      // padding queries of the last block never append
      cut[threadIdx.x] = qb * kFQ + (int)threadIdx.x < a.nq ? 0u : 0xFFFFFFFFu;
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

// ---- tensor-core filter (tcgen05) ------------------------------------------------
//
// The same filter / window / merge contract with the filter scores formed on
// the 5th-generation tensor cores: q.x ~ qh.xh + qh.xl + ql.xh with bf16 hi/lo
// splits of the float64 query and the float32 row (each product exact in
// float32, accumulated in float32 in TMEM), one 128-point x 128-query tile per
// 3 x Kp/16 tcgen05.mma (kind::f16, M = 128, N = 128, K = 16). Per element
//   |q x - (qh xh + qh xl + ql xh)| <= |ql xl| + |eq| |xh + xl| + |qh + ql| |ex|
//                                    <= 3.02 2^-18 |q_j x_j|
// (bf16 keeps 8 significant bits: |ql| <= 2^-9 |q|, the split residuals
// |eq| <= 2^-18 |q|, |ex| <= 2^-18 |x|), and each float32 accumulation adds
// at most one unit in the last place (any order, any rounding), so
//   |f - s| <= B = 1.01 [3.02 2^-18 + (1.01 Kp + 2) 2^-23] |q| max|x|
// (qh.xh accumulates in one TMEM accumulator, the two cross terms — 2^8
// smaller — in a second one, and the reader adds the two),
// and the windows keep f >= theta - 2B exactly as the float32 filter does.
// Operands sit in shared memory in the K-major SWIZZLE_NONE canonical layout
// (8-row x 16-byte core matrices; LBO = 128 B along K, SBO = Kp/8 x 128 B
// along M/N); point tiles are pre-laid-out in global memory so one
// cp.async.bulk per tile (mbarrier completion) stages them, double-buffered.
constexpr int kTM = 128;  // points per tile (UMMA M, TMEM lanes)
constexpr int kTQ = 128;  // queries per CTA (UMMA N, TMEM columns)
constexpr int kTKpMax = 128;
constexpr int kTPPT = 16;  // tiles between window shrinks

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}
// kind::f16: bf16 x bf16 -> f32, A and B K-major, M = 128, N = kTQ
constexpr uint32_t kTIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTQ >> 3) << 17) |
                             ((uint32_t)(kTM >> 4) << 24);

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
}
// one mbarrier transaction, issued as 8 bulk copies so the copy engine keeps
// several requests in flight (bytes a multiple of 128)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
  const uint32_t piece = bytes / 8;
#pragma unroll
  for (int u = 0; u < 8; ++u)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
            "r"(dst + u * piece), "l"(static_cast<const char*>(src) + u * piece), "r"(piece),
        "r"(bar)
        : "memory");
}

// canonical K-major index of element (r, k) in a 128-row tile with KC = Kp / 8
__device__ __forceinline__ int canon(int r, int k, int KC) {
  return ((r >> 3) * KC + (k >> 3)) * 64 + (r & 7) * 8 + (k & 7);
}

// rows -> per-128-point blocks of [hi tile | lo tile] bf16 (padding zero)
__global__ void k_tc_points(const float* __restrict__ xr, size_t n, int d, int Kp,
                            __nv_bfloat16* __restrict__ out) {
  const size_t blk = blockIdx.x;
  const int KC = Kp / 8;
  __nv_bfloat16* hi = out + blk * 2 * kTM * Kp;
  __nv_bfloat16* lo = hi + kTM * Kp;
  for (int e = threadIdx.x; e < kTM * Kp; e += blockDim.x) {
    const int r = e / Kp, k = e % Kp;
    const size_t p = blk * kTM + r;
    const float v = (p < n && k < d) ? xr[p * d + k] : 0.0f;
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    hi[canon(r, k, KC)] = h;
    lo[canon(r, k, KC)] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

// queries -> per-128-query blocks of [hi | lo] tiles and 2 B per query;
// non-finite or out-of-range queries flag 4 (the caller's exact path)
__global__ void k_tc_queries(const double* Q, int nq, int d, int Kp, double xmax,
                             __nv_bfloat16* __restrict__ out, float* twoB, int* flag) {
  const int q = blockIdx.x;  // padded query index
  const int qb = q / kTQ, r = q % kTQ, KC = Kp / 8;
  __nv_bfloat16* hi = out + (size_t)qb * 2 * kTQ * Kp;
  __nv_bfloat16* lo = hi + kTQ * Kp;
  __shared__ double red[32];
  double ss = 0.0;
  bool ok = true;
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    const double v = (q < nq && k < d) ? Q[(size_t)q * d + k] : 0.0;
    ok &= fabs(v) < 1e30;
    const __nv_bfloat16 h = __double2bfloat16(v);
    hi[canon(r, k, KC)] = h;
    lo[canon(r, k, KC)] = __double2bfloat16(v - (double)__bfloat162float(h));
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
    // split terms + the float32 accumulations: qh.xh in one accumulator
    // (Kp additions of terms <= |q_j x_j|), the two cross terms in another
    // (2 Kp additions of terms <= 2^-8 |q_j x_j|), one final add
    const double c = 3.02 * 3.814697265625e-06 + (1.01 * Kp + 2.0) * 1.1920928955078125e-07;
    const double B = 1.01 * c * sqrt(t) * 1.0000001 * xmax + 1e-30;
    twoB[q] = (float)(2.0 * B * (1.0 + 1e-6));
    // bf16 keeps float32's exponent range: values that would overflow or
    // lose the relative bound (subnormal parts) take the float32 filter
    if ((!all || sqrt(t) * xmax > 1e30) && q < nq) flag[q] = 4;
  }
}

struct TArgs {
  const __nv_bfloat16* xtile;  // [n / 128][hi | lo][128 x Kp]
  const __nv_bfloat16* qtile;  // [nqb][hi | lo][128 x Kp]
  const float* twoB;           // [nq_pad]
  size_t n;
  int Kp, nq, N, cap, R, nqb;
  size_t chunk;
  uint2* out_buf;  // [q][r][cap]
  int* out_cnt;    // [q][r]
  int* out_flag;   // [q]
};

// Warp-specialised: warp 16 is the producer (one lane stages the tiles with
// cp.async.bulk and issues the MMAs), warps 0..15 read the accumulators. Two
// TMEM accumulators and two point-tile buffers, handed over by mbarriers:
// full[acc] (the MMAs' tcgen05.commit), empty[acc] (one arrival per reading
// warp), A[buf] (bulk-copy bytes). Reading warp w takes TMEM lanes
// 32 (w mod 4) .. + 31 (its points) and columns 32 (w / 4) .. + 31 (its
// queries), one tcgen05.ld per tile; it keeps its 32 window cuts in
// registers (refreshed after each shrink) and builds a bit mask of the
// queries a point passes, so the rare appends are the only branches.
#ifdef AQ_TC_PROFILE
__device__ unsigned long long g_tcprof[8];
__device__ unsigned long long g_tccta[2048];
#endif
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

constexpr int kTReaders = 16;
constexpr int kTThreads = (kTReaders + 1) * 32;

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void readers_sync() {  // named barrier 1: the reading warps
  asm volatile("bar.sync 1, %0;\n" ::"n"(kTReaders * 32) : "memory");
}

__global__ void __launch_bounds__(kTThreads, 1) k_exact_tc(const TArgs a) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  const int Kp = a.Kp, KC = Kp / 8;
  const uint32_t tile_b = (uint32_t)(2 * kTM * Kp * 2);  // bytes of [hi | lo]
  unsigned char* sB = tsm + 2 * tile_b;  // point tiles: tsm + buffer * tile_b
  uint32_t* cut = reinterpret_cast<uint32_t*>(sB + tile_b);
  int* cnt = reinterpret_cast<int*>(cut + kTQ);
  int* flag = cnt + kTQ;
  float* tb2 = reinterpret_cast<float*>(flag + kTQ);
  uint64_t* bars = reinterpret_cast<uint64_t*>(tb2 + kTQ);  // A0 A1 B F0 F1 E0 E1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const bool producer = warp == kTReaders;
  // barrier addresses by index (no per-thread arrays: they would live in
  // local memory when indexed by the tile parity)
  const uint32_t bar0 = smem_addr(bars);
  const uint32_t barB = bar0 + 16;
  auto barA = [&](int b) { return bar0 + 8u * (uint32_t)b; };
  auto barF = [&](int b) { return bar0 + 24u + 8u * (uint32_t)b; };
  auto barE = [&](int b) { return bar0 + 40u + 8u * (uint32_t)b; };
  const uint32_t sA0 = smem_addr(tsm);
  if (t == 0) {
    for (int b = 0; b < 5; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(&bars[b])));
    for (int b = 5; b < 7; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&bars[b])),
                   "n"(kTReaders));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(4 * kTQ));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
#ifdef AQ_TC_PROFILE
  const long long kstart = clock64();
#endif
  // phases (bit b = parity of barrier b): producer and readers each track
  // the barriers they wait on
  uint32_t phA = 0u, phB = 0u, phF = 0u, phE = 0u;
  const size_t total = (size_t)a.nqb * a.n;
  size_t Lpos = (size_t)blockIdx.x * a.chunk;
  const size_t Lend = min(total, Lpos + a.chunk);
  const int cap = a.cap;
  const int lq = warp & 3, cq = warp >> 2;
  while (Lpos < Lend) {
    const int qb = (int)(Lpos / a.n);
    const size_t start = Lpos % a.n;
    const size_t end = min(a.n, start + (Lend - Lpos));
    const int r = (int)(blockIdx.x - ((size_t)qb * a.n) / a.chunk);
    Lpos += end - start;
    const size_t b0 = start / kTM, b1 = (end + kTM - 1) / kTM;  // point blocks of the segment
    const int nt = (int)(b1 - b0);
    __syncthreads();  // every warp is done with the previous segment's windows
    if (t < kTQ) {
      // padding queries of the last block (scores 0 everywhere) start with an
      // unreachable cut and never append
      cut[t] = qb * kTQ + t < a.nq ? 0u : 0xFFFFFFFFu;
      cnt[t] = 0;
      flag[t] = 0;
      tb2[t] = a.twoB[qb * kTQ + t];
    }
    __syncthreads();
    if (producer) {
      if (lane == 0) {
        bulk_load(smem_addr(sB), a.qtile + (size_t)qb * 2 * kTQ * Kp, tile_b, barB);
        bulk_load(sA0, a.xtile + b0 * 2 * kTM * Kp, tile_b, barA(0));
        if (nt > 1) bulk_load(sA0 + tile_b, a.xtile + (b0 + 1) * 2 * kTM * Kp, tile_b, barA(1));
        mbar_wait(barB, phB);
        phB ^= 1u;
        const uint32_t half = (uint32_t)(kTM * Kp * 2), lbo = 128, sbo = (uint32_t)KC * 128;
        for (int i = 0; i < nt; ++i) {
          const int acc = i & 1;
#ifdef AQ_TC_PROFILE
          long long c0 = clock64();
#endif
          if (i >= 2) {  // the readers are done with accumulator acc (tile i - 2)
            mbar_wait(barE(acc), (phE >> acc) & 1u);
            phE ^= 1u << acc;
          }
#ifdef AQ_TC_PROFILE
          long long c1 = clock64();
#endif
          mbar_wait(barA(acc), (phA >> acc) & 1u);
          phA ^= 1u << acc;
#ifdef AQ_TC_PROFILE
          long long c2 = clock64();
          if (blockIdx.x == 0) { atomicAdd(&g_tcprof[0], (unsigned long long)(c1 - c0)); atomicAdd(&g_tcprof[1], (unsigned long long)(c2 - c1)); atomicAdd(&g_tcprof[3], 1ull); }
#endif
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t aBase = sA0 + (uint32_t)acc * tile_b, bBase = smem_addr(sB);
          for (int term = 0; term < 3; ++term) {  // qh.xh -> D1; qh.xl, ql.xh -> D2
            const uint32_t aOff = term == 1 ? half : 0u, bOff = term == 2 ? half : 0u;
            const uint32_t dst = tmem + (uint32_t)(acc * 2 * kTQ + (term ? kTQ : 0));
            // K step ks: the start-address field advances by 256 B (16 units)
            uint64_t da = umma_sdesc(aBase + aOff, lbo, sbo);
            uint64_t db = umma_sdesc(bBase + bOff, lbo, sbo);
            uint32_t accum = term == 2 ? 1u : 0u;
            for (int ks = 0; ks < Kp / 16; ++ks, da += 16, db += 16) {
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dst),
                  "l"(da), "l"(db), "r"(kTIdesc), "r"(accum));
              accum = 1u;
            }
          }
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                  barF(acc))
              : "memory");
#ifdef AQ_TC_PROFILE
          if (blockIdx.x == 0) atomicAdd(&g_tcprof[4], (unsigned long long)(clock64() - c2));
#endif
          // tile i + 1 goes into the buffer of tile i - 1 once that tile's MMAs
          // are done (tiles 0 and 1 were loaded up front), while MMA(i) runs
          if (i >= 1 && i + 1 < nt) {
            const int pb = acc ^ 1;
#ifdef AQ_TC_PROFILE
            long long c3 = clock64();
#endif
            mbar_wait(barF(pb), (phF >> pb) & 1u);
            phF ^= 1u << pb;
#ifdef AQ_TC_PROFILE
            if (blockIdx.x == 0) atomicAdd(&g_tcprof[2], (unsigned long long)(clock64() - c3));
#endif
            bulk_load(sA0 + (uint32_t)pb * tile_b, a.xtile + (b0 + i + 1) * 2 * kTM * Kp, tile_b,
                      barA(pb));
          }
        }
        // consume the trailing phases so producer and readers stay in step:
        // the readers' arrivals for the last (up to) two tiles
        for (int i = (nt >= 2 ? nt - 2 : 0); i < nt; ++i) {
          const int acc = i & 1;
          mbar_wait(barE(acc), (phE >> acc) & 1u);
          phE ^= 1u << acc;
        }
        // MMA completions the producer did not wait on: tile nt - 1, and tile
        // 0 when nt == 1 (the loop waited on tiles 0 .. nt - 3 at i = 1 .. nt - 2)
        if (nt >= 2) {
          phF ^= 1u << ((nt - 2) & 1);
          phF ^= 1u << ((nt - 1) & 1);
        } else {
          phF ^= 1u;
        }
      }
      __syncwarp();
    } else {
      uint2* const buf = a.out_buf + ((size_t)qb * kTQ * a.R + r) * cap;
      const size_t qstride = (size_t)a.R * cap;
      constexpr int SPAN = kTM * kTPPT;
        float cr[32];  // this warp's 32 window cuts (filter-score floor)
#pragma unroll
      for (int j = 0; j < 32; ++j) cr[j] = -INFINITY;
      for (int i = 0; i < nt; ++i) {
        const int acc = i & 1;
        mbar_wait(barF(acc), (phF >> acc) & 1u);
        phF ^= 1u << acc;
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        uint32_t v[32], w2[32];
        const uint32_t taddr =
            tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(acc * 2 * kTQ + cq * 32);
        tmem_ld32(taddr, v);
        tmem_ld32(taddr + kTQ, w2);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __fadd_rn(__uint_as_float(v[j]), __uint_as_float(w2[j]));
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(barE(acc));  // accumulator acc may be overwritten
        if ((i % kTPPT) == 0) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const uint32_t ck = cut[cq * 32 + j];
            cr[j] = ck ? funkey(ck) : -INFINITY;  // key >= cut  <=>  f >= funkey(cut)
          }
        }
        const size_t p = (b0 + i) * kTM + lq * 32 + lane;
        if (p >= start && p < end) {
          uint32_t pass = 0u;
#pragma unroll
          for (int j = 0; j < 32; ++j) pass |= (uint32_t)(f[j] >= cr[j]) << j;
          while (pass) {
            const int j = __ffs(pass) - 1;
            pass &= pass - 1;
            const int q = cq * 32 + j;
            float fj = 0.0f;  // f[j] without dynamic register indexing (appends are rare)
#pragma unroll
            for (int u = 0; u < 32; ++u) fj = u == j ? f[u] : fj;
            const int pos = atomicAdd(&cnt[q], 1);
            if (pos < cap)
              buf[q * qstride + pos] = make_uint2(fkey(fj), (unsigned)p);
            else
              flag[q] = 1;
          }
        }
        if ((i % kTPPT) == kTPPT - 1 || i + 1 == nt) {
          readers_sync();  // appends of the last tiles visible
          for (int q = warp; q < kTQ; q += kTReaders) {
            const int c = min(cnt[q], cap);
            uint32_t th;
            if (c > cap - SPAN && !flag[q] && warp_nth_key32(buf + q * qstride, c, a.N, &th)) {
              const uint32_t cqv = max(cut[q], window_cut(th, tb2[q]));
              const int kept = warp_keep_key32(buf + q * qstride, c, cqv);
              if (lane == 0) {
                cut[q] = cqv;
                cnt[q] = kept;
                if (kept > cap - SPAN) flag[q] = 1;
              }
            }
            __syncwarp();
          }
          readers_sync();
        }
      }
      for (int q = warp; q < kTQ; q += kTReaders) {
        const int gq = qb * kTQ + q;
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
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
#ifdef AQ_TC_PROFILE
  if (t == 0 && blockIdx.x < 2048) g_tccta[blockIdx.x] = (unsigned long long)(clock64() - kstart);
#endif
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(4 * kTQ));
}

// Tensor-core filter + the float64 merge; *ran = false leaves the query set
// to the float32 filter (d > 128, non-finite values, windows too large).
int exact_tc_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                    double* scores, std::vector<int>& hflag, double xmax, bool* ran) {
  *ran = false;
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const int Kp = (int)((d + 15) / 16 * 16);
  if (Kp > kTKpMax || ds->f64 || !ds->xr) return AQ_OK;
  const size_t te = std::min(depth, n);
  const int N = (int)te;
  const size_t nqb = (nq + kTQ - 1) / kTQ, nq_pad = nqb * kTQ;
  const size_t nblk = (n + kTM - 1) / kTM;
  const int cap = ((N + 31) & ~31) + kTM * kTPPT + 32 + (N > 128 ? N : 0);
  const size_t G0 = (size_t)s->num_sms;
  const size_t total = nqb * n;
  size_t chunk = std::max<size_t>((total + G0 - 1) / G0, 16 * (size_t)kTM);
  const size_t G = (total + chunk - 1) / chunk;
  size_t R = 1;
  for (size_t qb = 0; qb < nqb; ++qb)
    R = std::max(R, ((qb + 1) * n - 1) / chunk - qb * n / chunk + 1);
  const size_t xt_b = nblk * 2 * kTM * Kp * sizeof(__nv_bfloat16);
  const size_t qt_b = nqb * 2 * kTQ * Kp * sizeof(__nv_bfloat16);
  const size_t buf_b = nq_pad * R * cap * sizeof(uint2);
  char* mem = nullptr;
  const size_t off_q = (xt_b + 1023) & ~(size_t)1023, off_b = (off_q + qt_b + 1023) & ~(size_t)1023;
  const size_t off_t = off_b + buf_b, off_c = off_t + nq_pad * sizeof(float);
  const size_t bytes = off_c + nq * R * sizeof(int) + nq * sizeof(int) + 256;
  AQ_CUDA(cudaMallocAsync((void**)&mem, bytes, s->stream));
  __nv_bfloat16* xtile = (__nv_bfloat16*)mem;
  __nv_bfloat16* qtile = (__nv_bfloat16*)(mem + off_q);
  uint2* obuf = (uint2*)(mem + off_b);
  float* twoB = (float*)(mem + off_t);
  int* ocnt = (int*)(mem + off_c);
  int* oflag = ocnt + nq * R;
  int st = AQ_OK;
  if (cudaMemsetAsync(oflag, 0, nq * sizeof(int), s->stream) != cudaSuccess ||
      cudaMemsetAsync(ocnt, 0, nq * R * sizeof(int), s->stream) != cudaSuccess)
    st = ref_error(AQ_E_CUDA, "memset failed");
  if (st == AQ_OK) {
    timer_mark(s, AQ_T_EXACT);
    k_tc_points<<<(unsigned)nblk, 256, 0, s->stream>>>(ds->xr, n, (int)d, Kp, xtile);
    k_tc_queries<<<(unsigned)nq_pad, 128, 0, s->stream>>>(Qd, (int)nq, (int)d, Kp, xmax, qtile,
                                                          twoB, oflag);
    s->launches += 2;
    TArgs a{xtile, qtile, twoB, n, Kp, (int)nq, N, cap, (int)R, (int)nqb, chunk, obuf, ocnt, oflag};
    const size_t smem = 3 * (size_t)(2 * kTM * Kp * 2) + kTQ * 16 + 7 * 8 + 16 + 1024;
    if (cudaFuncSetAttribute(k_exact_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      st = ref_error(AQ_E_CUDA, "shared memory attribute");
    if (st == AQ_OK) {
      k_exact_tc<<<(unsigned)G, kTThreads, smem, s->stream>>>(a);
      s->launches++;
#ifdef AQ_TC_PROFILE
      {
        unsigned long long h[8];
        cudaStreamSynchronize(s->stream);
        cudaMemcpyFromSymbol(h, g_tcprof, sizeof h);
        fprintf(stderr, "tc prof CTA0: tiles %llu, wait E %.0f, wait A %.0f, wait F %.0f, MMA issue %.0f cycles/tile\n",
                h[3], (double)h[0] / h[3], (double)h[1] / h[3], (double)h[2] / h[3], (double)h[4] / h[3]);
        std::vector<unsigned long long> cc(2048);
        cudaMemcpyFromSymbol(cc.data(), g_tccta, 2048 * 8);
        unsigned long long mn = ~0ull, mx = 0, sum = 0;
        for (size_t b = 0; b < G && b < 2048; ++b) { mn = std::min(mn, cc[b]); mx = std::max(mx, cc[b]); sum += cc[b]; }
        fprintf(stderr, "CTA cycles: G %zu min %llu avg %llu max %llu\n", G, mn, sum / G, mx);
      }
#endif
      int mcap = kFMergeCapMin;
      while (mcap < N + N / 2 + 1024 && mcap < kFMergeCapMax) mcap <<= 1;
      FArgs fa{nullptr, 0, (int)d, n, nullptr, twoB, (int)nq, N, cap, (int)R,
               chunk, (int)nqb, mcap, obuf, ocnt, oflag};
      const size_t msmem = (size_t)mcap * (sizeof(unsigned long long) + sizeof(uint32_t));
      cudaFuncSetAttribute(k_exact_fmerge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)msmem);
      k_exact_fmerge<<<(unsigned)nq, R >= 32 ? 1024 : 256, msmem, s->stream>>>(
          fa, ds->xr, Qd, (int)te, ids, scores);
      s->launches++;
      timer_mark(s, AQ_T_EXACT);
      if (cudaGetLastError() != cudaSuccess ||
          cudaMemcpyAsync(hflag.data(), oflag, nq * sizeof(int), cudaMemcpyDeviceToHost,
                          s->stream) != cudaSuccess ||
          cudaStreamSynchronize(s->stream) != cudaSuccess)
        st = ref_error(AQ_E_CUDA, "tensor-core exact filter failed");
    }
  }
  cudaFreeAsync(mem, s->stream);
  if (st == AQ_OK) *ran = true;
  return st;
}

// max of non-negative (or NaN) doubles by bit pattern: NaN norms compare
// above every finite value, so a non-finite row disables the filters
__global__ void k_max_norm(const double* __restrict__ v, size_t n, unsigned long long* out) {
  unsigned long long m = 0ull;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v[i]));
    m = b > m ? b : m;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

int exact_filter_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                        double* scores, std::vector<int>& hflag, bool* ran) {
  *ran = false;
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const size_t te = std::min(depth, n);
  const int N = (int)te;
  const size_t nqb = (nq + kFQ - 1) / kFQ, nq_pad = nqb * kFQ;
  // max |x| over the rows (norms are the reference's float64 norms), reduced
  // on the device: non-negative doubles order like their bit patterns
  void* pm;
  AQ_TRY(scratch(s, 6, 64, &pm));
  unsigned long long* dmax = (unsigned long long*)pm;
  AQ_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), s->stream));
  k_max_norm<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, s->stream>>>(ds->norms,
                                                                                      n, dmax);
  AQ_LAUNCHED(s);
  unsigned long long hbits = 0;
  AQ_CUDA(cudaMemcpyAsync(&hbits, dmax, sizeof hbits, cudaMemcpyDeviceToHost, s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  double xmax;
  std::memcpy(&xmax, &hbits, sizeof xmax);
  xmax *= 1.0000001;
  if (!(xmax < 1e30) || depth > (size_t)kFMaxN) return AQ_OK;  // caller's exact path
  // tensor-core filter first ($AQ_EXACT_TC=0 keeps the float32 FFMA filter);
  // flagged queries (non-finite values, overflowing windows) go on below
  static const int use_tc = getenv("AQ_EXACT_TC") ? atoi(getenv("AQ_EXACT_TC")) : 1;
  if (use_tc) {
    bool tc_ran = false;
    AQ_TRY(exact_tc_device(ds, Qd, nq, depth, ids, scores, hflag, xmax, &tc_ran));
    if (tc_ran) {
      *ran = true;
      return AQ_OK;
    }
  }
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
