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
// the 5th-generation tensor cores (kind::f16: bf16 operands, products exact
// in float32, float32 accumulation in TMEM), one 128-point x NQ-query tile
// per TERMS x Kp/16 tcgen05.mma (M = 128, N = NQ, K = 16). bf16 keeps 8
// significant bits, so rounding to it moves a value by at most 2^-8 of
// itself. Two precisions:
//
//  TERMS = 1   f = qh.xh, qh = bf16(q), xh = bf16(x). Per element
//              |q x - qh xh| = |qh (x - xh) + (q - qh) x| <= 2^-7 (1 + 2^-9) |q_j x_j|;
//  TERMS = 3   f = qh.xh + ql.xh + qh.xl with ql = bf16(q - qh), xl = bf16(x - xh),
//              whose residuals eq, ex are <= 2^-16 of |q|, |x|. Per element
//              |q x - f_j| = |qh ex + ql xl + ql ex + eq x| <= 3.02 2^-16 |q_j x_j|.
//
// The accumulator takes TERMS x Kp products whose absolute sum is <= 1.02
// sum |q_j x_j|; each step (a product joining the K = 16 reduction, or the
// reduction joining the accumulator: at most 1.07 TERMS Kp + 4 steps) is
// charged two units of the last float32 place, 2^-22 of that absolute sum,
// whatever the hardware's alignment and rounding. With E_T the per-element
// factor above,
//   |f - s| <= B = 1.01 [E_T + 1.02 (1.07 TERMS Kp + 4) 2^-22] |q| max|x|
// (Cauchy-Schwarz on sum |q_j x_j|; 1.01 covers the reference's own float64
// roundings), and the windows keep f >= theta - 2B exactly as the float32
// filter does. The one-term filter is three times cheaper on the tensor
// cores with a window about 60 x wider (config 2, depth 10: ~140 candidates
// per query, re-scored in float64 by the merge); queries whose windows
// overflow are re-run with TERMS = 3, then on the float32 filter.
//
// Layout and schedule (B200-first):
//  * operands in shared memory in the K-major SWIZZLE_NONE canonical layout
//    (8-row x 16-byte core matrices; LBO = 128 B along K, SBO = Kp/8 x 128 B
//    along M/N); point tiles are pre-laid-out in global memory as
//    [block][hi | lo][128 x Kp], so one cp.async.bulk stages a half tile;
//  * warp 16 loads (a ring of NS half-tile stages plus the query tile), warp
//    17 issues the MMAs (one elected lane), warps 0..15 read the two TMEM
//    accumulators (2 x NQ columns) and keep the windows;
//  * the point blocks are cut into S segments and the work items (segment,
//    query block) are dealt segment-major, item b + k G to CTA b: at any time
//    the grid streams two or three segments, so a point tile fetched from HBM
//    by one CTA serves the other query blocks from L2;
//  * one window per (query, segment); every window's cut is also published
//    to a per-query cut in global memory (atomicMax on the order-preserving
//    key) that later items start from. Any window's N-th filter score is <=
//    the global one, so every published cut stays <= theta - 2B.
constexpr int kTM = 128;   // points per tile (UMMA M, TMEM lanes)
constexpr int kTKpMax = 128;
constexpr int kTPPT = 8;   // tiles between window shrinks
constexpr int kTReaders = 16;
constexpr int kTThreads = (kTReaders + 2) * 32;  // + the loader and MMA warps
constexpr int kTMaxStages = 8;
constexpr int kTSmemMax = 232448;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}
// kind::f16: bf16 x bf16 -> f32, A and B K-major, M = 128, N = NQ
template <int NQ>
constexpr uint32_t kTIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NQ >> 3) << 17) |
                             ((uint32_t)(kTM >> 4) << 24);

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "n"(1000000)  // suspend up to 1 ms (woken by the phase)
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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
      : "memory");
}
// D (+)= A B over nks K = 16 steps (the start-address field advances 256 B per step)
__device__ __forceinline__ void umma_chain(uint32_t dst, uint64_t da, uint64_t db, int nks,
                                           uint32_t idesc, uint32_t acc0) {
#pragma unroll
  for (int ks = 0; ks < kTKpMax / 16; ++ks)
    if (ks < nks)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dst),
          "l"(da + 16u * ks), "l"(db + 16u * ks), "r"(idesc), "r"(ks ? 1u : acc0));
}
__device__ __forceinline__ void readers_sync() {  // named barrier 1: the reading warps
  asm volatile("bar.sync 1, %0;\n" ::"n"(kTReaders * 32) : "memory");
}
// N-th largest key among buf[0..cnt) (warp-cooperative; false when cnt < N):
// windows of up to 128 entries select in registers (32 bit passes, no
// memory traffic), larger ones in four 8-bit passes over a 256-bin shared
// histogram of this warp
__device__ bool warp_nth_key_tc(const uint2* buf, int cnt, int N, uint32_t* hist,
                                uint32_t* out) {
  if (cnt < N) return false;
  const int lane = threadIdx.x & 31;
  if (cnt <= 128) {
    uint32_t k[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = lane + 32 * u < cnt ? buf[lane + 32 * u].x : 0u;
    uint32_t T = 0u;
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t cand = T | (1u << bit);
      const int c = __reduce_add_sync(0xffffffffu, (int)(k[0] >= cand) + (int)(k[1] >= cand) +
                                                       (int)(k[2] >= cand) + (int)(k[3] >= cand));
      if (c >= N) T = cand;
    }
    *out = T;
    return true;
  }
  uint32_t prefix = 0u, mask = 0u;
  int need = N;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0u;
    __syncwarp();
    for (int e = lane; e < cnt; e += 32) {
      const uint32_t key = buf[e].x;
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    // lane l owns digits 255 - 8 l .. 248 - 8 l (descending)
    int c8[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c8[j] = (int)hist[255 - 8 * lane - j];
      sum += c8[j];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int digit = -1, above = 0;
    if (incl - sum < need && need <= incl) {
      int acc = incl - sum;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (digit < 0 && acc + c8[j] >= need) {
          digit = 255 - 8 * lane - j;
          above = acc;
        }
        acc += c8[j];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, digit >= 0)) - 1;
    digit = __shfl_sync(0xffffffffu, digit, src);
    above = __shfl_sync(0xffffffffu, above, src);
    prefix |= (uint32_t)digit << shift;
    mask |= 255u << shift;
    need -= above;
    __syncwarp();
  }
  *out = prefix;
  return true;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
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

// canonical K-major index of element (r, k) in a tile with KC = Kp / 8
__device__ __forceinline__ int canon(int r, int k, int KC) {
  return ((r >> 3) * KC + (k >> 3)) * 64 + (r & 7) * 8 + (k & 7);
}

// rows -> per-128-point blocks of [hi tile | lo tile] bf16 (padding zero)
__global__ void k_tc_points(const float* __restrict__ xr, size_t n, int d, int Kp, int terms,
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
    if (terms == 3) lo[canon(r, k, KC)] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

// queries -> per-NQ-query blocks of [hi | lo] tiles and 2 B per query;
// non-finite or out-of-range queries flag 4 (the caller's exact path)
__global__ void k_tc_queries(const double* Q, int nq, int d, int Kp, int NQ, int terms, double xmax,
                             __nv_bfloat16* __restrict__ out, float* twoB, int* flag) {
  const int q = blockIdx.x;  // padded query index
  const int qb = q / NQ, r = q % NQ, KC = Kp / 8;
  __nv_bfloat16* hi = out + (size_t)qb * 2 * NQ * Kp;
  __nv_bfloat16* lo = hi + (size_t)NQ * Kp;
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
    // split terms + the float32 accumulation steps (header comment)
    const double et = terms == 3 ? 3.02 * 1.52587890625e-05 : 7.8125e-03 * (1.0 + 1.953125e-03);
    const double c = et + 1.02 * (1.07 * terms * Kp + 4.0) * 2.384185791015625e-07;
    const double B = 1.01 * c * sqrt(t) * 1.0000001 * xmax + 1e-30;
    twoB[q] = (float)(2.0 * B * (1.0 + 1e-6));
    // bf16 keeps float32's exponent range: values that would overflow or
    // lose the relative bound (subnormal parts) take the float32 filter
    if ((!all || sqrt(t) * xmax > 1e30) && q < nq) flag[q] = 4;
  }
}

struct TArgs {
  const __nv_bfloat16* xtile;  // [nblk][hi | lo][128 x Kp]
  const __nv_bfloat16* qtile;  // [nqb][hi | lo][NQ x Kp] (this batch)
  const float* twoB;           // [nqb * NQ]
  uint32_t* gcut;              // [nq] published window cut per query (key)
  size_t n;
  int Kp, nq, N, cap, nqb;     // nq, nqb: this batch
  int S, T, nblk, NS, items;   // segments of T point blocks (last shorter); items = S nqb
  uint2* out_buf;  // [q][S][cap]
  int* out_cnt;    // [q][S]
  int* out_flag;   // [q]
};

template <int NQ, int TERMS>
__global__ void __launch_bounds__(kTThreads, 1) k_exact_tc(const TArgs a) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  constexpr int CPW = NQ / 4;  // accumulator columns per reading warp
  constexpr uint32_t kIdesc = kTIdesc<NQ>;
  const int Kp = a.Kp, KC = Kp / 8, NS = a.NS, cap = a.cap;
  const uint32_t half_b = (uint32_t)(kTM * Kp * 2), qhalf_b = (uint32_t)(NQ * Kp * 2);
  // [query hi | query lo (TERMS = 3)][NS point half tiles][cutf][cut][cnt][flag][tb2][hist][barriers][tmem slot]
  constexpr int HALVES = TERMS == 3 ? 2 : 1;  // point half tiles (hi, lo) per tile
  unsigned char* ring = tsm + HALVES * qhalf_b;
  float* cutf = reinterpret_cast<float*>(ring + (size_t)NS * half_b);
  uint32_t* cut = reinterpret_cast<uint32_t*>(cutf + NQ);
  int* cnt = reinterpret_cast<int*>(cut + NQ);
  int* flag = cnt + NQ;
  float* tb2 = reinterpret_cast<float*>(flag + NQ);
  uint32_t* hist = reinterpret_cast<uint32_t*>(tb2 + NQ) + (threadIdx.x >> 5) * 256;  // per reader warp
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint32_t*>(tb2 + NQ) + kTReaders * 256);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kTMaxStages + 6);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // barrier addresses by index: full[st], empty[st], F[acc], E[acc], Qfull, Qempty
  const uint32_t bar0 = smem_addr(bars);
  auto bFull = [&](int st) { return bar0 + 8u * (uint32_t)st; };
  auto bEmpty = [&](int st) { return bar0 + 8u * (uint32_t)(kTMaxStages + st); };
  auto bF = [&](int acc) { return bar0 + 8u * (uint32_t)(2 * kTMaxStages + acc); };
  auto bE = [&](int acc) { return bar0 + 8u * (uint32_t)(2 * kTMaxStages + 2 + acc); };
  const uint32_t bQf = bar0 + 8u * (2 * kTMaxStages + 4), bQe = bQf + 8u;
  if (t == 0) {
    for (int b = 0; b < 2 * kTMaxStages + 6; ++b) {
      const bool e = b == 2 * kTMaxStages + 2 || b == 2 * kTMaxStages + 3;
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar0 + 8u * b),
                   "r"(e ? kTReaders : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(2 * NQ));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int G = gridDim.x;

  if (warp == kTReaders) {  // ---- loader
    if (lane == 0) {
      int st = 0;            // ring stage of the next half tile
      uint32_t ph = 0u;      // its use count's parity
      uint32_t issued = 0u;  // half tiles issued
      int k = 0;
      for (int it = blockIdx.x; it < a.items; it += G, ++k) {
        const int s = it / a.nqb, qb = it % a.nqb;
        const int tb0 = s * a.T, tb1 = min(a.nblk, tb0 + a.T);
        if (k > 0) mbar_wait(bQe, (uint32_t)(k - 1) & 1u);  // the last item's MMAs are done
        bulk_load(smem_addr(tsm), a.qtile + (size_t)qb * 2 * NQ * Kp, HALVES * qhalf_b, bQf);
        const __nv_bfloat16* src = a.xtile + (size_t)tb0 * 2 * kTM * Kp;
        // TERMS = 1 reads the hi half of each [hi | lo] block only
        for (int hh = 0; hh < HALVES * (tb1 - tb0);
             ++hh, ++issued, src += (TERMS == 3 ? 1 : 2) * kTM * Kp) {
          if (issued >= (uint32_t)NS) mbar_wait(bEmpty(st), ph ^ 1u);
          bulk_load(smem_addr(ring) + (uint32_t)st * half_b, src, half_b, bFull(st));
          if (++st == NS) {
            st = 0;
            ph ^= 1u;
          }
        }
      }
      // every commit has landed before the CTA exits: the last use of each
      // stage and the last item's query tile
      for (int e = 0; e < NS && (uint32_t)e < issued; ++e) {
        if (st == 0) ph ^= 1u;
        st = st == 0 ? NS - 1 : st - 1;
        mbar_wait(bEmpty(st), ph);
      }
      if (k > 0) mbar_wait(bQe, (uint32_t)(k - 1) & 1u);
    }
    __syncwarp();
  } else if (warp == kTReaders + 1) {  // ---- MMA issue
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0u, c = 0u;
      int k = 0;
      const int nks = Kp / 16;
      const uint32_t lbo = 128, sbo = (uint32_t)KC * 128;
      // descriptors: the query hi / lo tiles, ring stage 0 (stage st adds
      // st x half_b >> 4 to the start-address field)
      const uint64_t dqh = umma_sdesc(smem_addr(tsm), lbo, sbo);
      const uint64_t dql = umma_sdesc(smem_addr(tsm) + qhalf_b, lbo, sbo);
      const uint64_t dx0 = umma_sdesc(smem_addr(ring), lbo, sbo);
      const uint32_t dstep = half_b >> 4;
      for (int it = blockIdx.x; it < a.items; it += G, ++k) {
        const int s = it / a.nqb;
        const int ntile = min(a.nblk, (s + 1) * a.T) - s * a.T;
        mbar_wait(bQf, (uint32_t)k & 1u);
        for (int i = 0; i < ntile; ++i, ++c) {
          const int acc = (int)(c & 1u);
          if (c >= 2) mbar_wait(bE(acc), ((c >> 1) - 1) & 1u);  // readers done with acc
          const int sh = st;
          const uint32_t phh = ph;
          if (++st == NS) {
            st = 0;
            ph ^= 1u;
          }
          const uint32_t dst = tmem + (uint32_t)(acc * NQ);
          if constexpr (TERMS == 1) {
            mbar_wait(bFull(sh), phh);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            umma_chain(dst, dx0 + (uint64_t)(sh * dstep), dqh, nks, kIdesc, 0u);
            umma_commit(bEmpty(sh));
          } else {
            const int sl = st;
            const uint32_t phl = ph;
            if (++st == NS) {
              st = 0;
              ph ^= 1u;
            }
            mbar_wait(bFull(sh), phh);
            mbar_wait(bFull(sl), phl);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint64_t dxh = dx0 + (uint64_t)(sh * dstep), dxl = dx0 + (uint64_t)(sl * dstep);
            // qh.xh, ql.xh (the hi stage), then qh.xl (the lo stage)
            umma_chain(dst, dxh, dqh, nks, kIdesc, 0u);
            umma_chain(dst, dxh, dql, nks, kIdesc, 1u);
            umma_commit(bEmpty(sh));
            umma_chain(dst, dxl, dqh, nks, kIdesc, 1u);
            umma_commit(bEmpty(sl));
          }
          umma_commit(bF(acc));
        }
        umma_commit(bQe);
      }
    }
    __syncwarp();
  } else {  // ---- readers: warp w takes TMEM lanes 32 (w mod 4).. and columns CPW (w / 4)..
    const int lq = warp & 3, cg = warp >> 2;
    constexpr int SPAN = kTM * kTPPT;
    constexpr int QPW = NQ / kTReaders;  // queries per warp in the window passes
    uint32_t c = 0;
    for (int it = blockIdx.x; it < a.items; it += G) {
      const int s = it / a.nqb, qb = it % a.nqb;
      const int tb0 = s * a.T, ntile = min(a.nblk, tb0 + a.T) - tb0;
      readers_sync();  // the previous item's windows are finished
      for (int q = t; q < NQ; q += kTReaders * 32) {
        const int gq = qb * NQ + q;
        // padding queries (scores 0 everywhere) get an unreachable cut
        const uint32_t c0 = gq < a.nq ? *(volatile const uint32_t*)(a.gcut + gq) : 0xFFFFFFFFu;
        cut[q] = c0;
        cutf[q] = c0 ? funkey(c0) : -INFINITY;  // key >= cut  <=>  f >= funkey(cut)
        cnt[q] = 0;
        flag[q] = 0;
        tb2[q] = a.twoB[gq];
      }
      readers_sync();
      uint2* const buf = a.out_buf + ((size_t)qb * NQ * a.S + s) * cap;
      const size_t qstride = (size_t)a.S * cap;
      for (int i = 0; i < ntile; ++i, ++c) {
        const int acc = (int)(c & 1u);
        mbar_wait(bF(acc), (c >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t taddr = tmem + ((uint32_t)(lq * 32) << 16) + (uint32_t)(acc * NQ + cg * CPW);
        const size_t p = (size_t)(tb0 + i) * kTM + lq * 32 + lane;
        // 32 columns at a time (registers); the accumulator is released
        // after the last chunk's load
#pragma unroll
        for (int h = 0; h < CPW / 32; ++h) {
          uint32_t v[32];
          __syncwarp();  // converged after the previous chunk's appends (.sync.aligned)
          tmem_ld32(taddr + 32 * h, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
          if (h == CPW / 32 - 1) {
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(bE(acc));  // accumulator acc may be overwritten
          }
          const float4* cf = reinterpret_cast<const float4*>(cutf + cg * CPW + 32 * h);
          // one predicate-OR compare per column; the pass mask only when a
          // query passes (rare once the cuts have settled)
          bool any = false;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 cc = cf[j4];
            any |= __uint_as_float(v[4 * j4]) >= cc.x;
            any |= __uint_as_float(v[4 * j4 + 1]) >= cc.y;
            any |= __uint_as_float(v[4 * j4 + 2]) >= cc.z;
            any |= __uint_as_float(v[4 * j4 + 3]) >= cc.w;
          }
          if (any && p < a.n) {
            uint32_t pass = 0u;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              pass |= (uint32_t)(__uint_as_float(v[j]) >= cutf[cg * CPW + 32 * h + j]) << j;
            while (pass) {
              const int j = __ffs(pass) - 1;
              pass &= pass - 1;
              const int q = cg * CPW + 32 * h + j;
              uint32_t vj = 0u;  // v[j] without dynamic register indexing
#pragma unroll
              for (int u = 0; u < 32; ++u) vj = u == j ? v[u] : vj;
              const int pos = atomicAdd(&cnt[q], 1);
              if (pos < cap)
                buf[q * qstride + pos] = make_uint2(fkey(__uint_as_float(vj)), (unsigned)p);
              else
                flag[q] = 1;
            }
          }
        }
        const bool last = i + 1 == ntile;
        if ((i % kTPPT) == kTPPT - 1 || last) {
          readers_sync();  // appends of the last tiles visible
          // lane j < QPW owns query warp + 16 j: its published cut, count and
          // whether its window shrinks now (the next span could overflow, or
          // the item ends); the warp then shrinks those windows one by one
          const int qj = warp + kTReaders * lane, gqj = qb * NQ + qj;
          uint32_t oldc = 0u, cqj = 0u;
          int c2j = 0;
          bool need = false;
          if (lane < QPW) {
            oldc = cut[qj];
            cqj = max(oldc, gqj < a.nq ? *(volatile const uint32_t*)(a.gcut + gqj) : 0u);
            c2j = min(cnt[qj], cap);
            need = (last || c2j > cap - SPAN) && !flag[qj] && c2j >= a.N;
            // an overflowed window (the query goes to the next tier) stops
            // appending: unreachable cut, not published
            if (flag[qj]) cqj = 0xFFFFFFFFu;
          }
          unsigned todo = __ballot_sync(0xffffffffu, need);
          while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int q = warp + kTReaders * j;
            const int cj = __shfl_sync(0xffffffffu, c2j, j);
            uint32_t cq = __shfl_sync(0xffffffffu, cqj, j), th = 0u;
            warp_nth_key_tc(buf + q * qstride, cj, a.N, hist, &th);
            cq = max(cq, window_cut(th, tb2[q]));
            const int kept = warp_keep_key32(buf + q * qstride, cj, cq);
            if (lane == j) {
              cqj = cq;
              c2j = kept;
            }
          }
          if (lane < QPW) {
            if (need) {
              cnt[qj] = c2j;
              if (gqj < a.nq && cqj > oldc) atomicMax(a.gcut + gqj, cqj);
            }
            if (cqj != oldc) {
              cut[qj] = cqj;
              cutf[qj] = funkey(cqj);  // 0xFFFFFFFF: NaN, nothing passes
            }
            if (last && gqj < a.nq) {
              a.out_cnt[(size_t)gqj * a.S + s] = c2j;
              if (flag[qj]) atomicOr(&a.out_flag[gqj], 1);
            }
          }
          readers_sync();
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(2 * NQ));
}

namespace {
// shared memory of k_exact_tc<NQ, terms> with NS ring stages
size_t tc_smem(int NQ, int Kp, int NS, int terms) {
  return (terms == 3 ? 2 : 1) * (size_t)NQ * Kp * 2 + (size_t)NS * kTM * Kp * 2 + (size_t)NQ * 20 +
         (size_t)kTReaders * 256 * 4 + 8 * (2 * kTMaxStages + 6) + 16 + 1024;
}
}  // namespace

// Tensor-core filter (TERMS = terms) + the float64 merge; *ran = false leaves
// the query set to the next tier (d > 128, float64 data).
int exact_tc_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                    double* scores, std::vector<int>& hflag, double xmax, int terms, bool* ran) {
  *ran = false;
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const int Kp = (int)((d + 15) / 16 * 16);
  if (Kp > kTKpMax || ds->f64 || !ds->xr) return AQ_OK;
  const size_t te = std::min(depth, n);
  const int N = (int)te;
  // 256 queries per CTA when the query tile and three ring stages fit
  // (three-term: one ring stage is a hi or lo half tile, two per tile)
  int NQ = 256, NS = 0;
  auto stages = [&](int nqv) {
    const size_t fixed = tc_smem(nqv, Kp, 0, terms);
    return fixed > (size_t)kTSmemMax
               ? 0
               : (int)std::min<size_t>(kTMaxStages, (kTSmemMax - fixed) / ((size_t)kTM * Kp * 2));
  };
  NS = stages(256);
  if (NS < (terms == 3 ? 3 : 2) || nq <= 128) {
    NQ = 128;
    NS = stages(128);
  }
  const size_t nqb = (nq + NQ - 1) / NQ, nq_pad = nqb * NQ;
  const int nblk = (int)((n + kTM - 1) / kTM);
  // window: N, one span of appends, room for the filter's near-ties
  // (the one-term window is wide), tie room growing with N
  const int cap = ((N + 31) & ~31) + kTM * kTPPT + (terms == 1 ? 256 : 32) + (N > 128 ? N : 0);
  const int G0 = s->num_sms;
  const size_t tile_b = 2 * (size_t)kTM * Kp * 2;
  // query batches whose windows (nq x S x cap entries) stay within ~4 GB
  const size_t win_budget = (size_t)4 << 30;
  const int Smax_seg = std::max(1, std::min(64, nblk));
  // segments: at most ~24 MB of point tiles each (two or three are live in
  // L2 at a time); among those, the count whose item deal loads the CTAs
  // most evenly
  auto choose_S = [&](size_t nqb_b, int Scap) {
    const int Smin = (int)std::min<size_t>(
        (size_t)Scap, std::max<size_t>(1, (nblk * tile_b + (24u << 20) - 1) / (24u << 20)));
    int bestS = Smin;
    double best = 1e300;
    for (int S = Smin; S <= Scap; ++S) {
      const int T = (nblk + S - 1) / S, Se = (nblk + T - 1) / T;
      const size_t items = (size_t)Se * nqb_b, G = std::min<size_t>(G0, items);
      double worst = 0.0;
      for (size_t b = 0; b < G; ++b) {
        double w = 0.0;
        for (size_t it = b; it < items; it += G) {
          const int sg = (int)(it / nqb_b);
          w += std::min(nblk, (sg + 1) * T) - sg * T + 6;  // + item overhead (tiles)
        }
        worst = std::max(worst, w);
      }
      const double cost = worst * (1.0 + 0.002 * Se);
      if (cost < best * 0.999) {
        best = cost;
        bestS = Se;
      }
    }
    return bestS;
  };
  // one launch for all query blocks unless their windows (nq x S x cap
  // entries) exceed the budget; then batches of query blocks
  size_t qb_batch = nqb;
  int Scap_mem = Smax_seg;
  {
    const size_t per_qb = (size_t)NQ * cap * sizeof(uint2);  // one segment's windows
    const int S_all = choose_S(nqb, Smax_seg);
    if (nqb * S_all * per_qb > win_budget) {
      qb_batch = std::max<size_t>(1, win_budget / (S_all * per_qb));
      Scap_mem = (int)std::max<size_t>(1, std::min<size_t>(Smax_seg, win_budget / (qb_batch * per_qb)));
    } else {
      Scap_mem = S_all;
    }
  }
  const size_t xt_b = (size_t)nblk * tile_b;
  const size_t qt_b = nqb * 2 * (size_t)NQ * Kp * sizeof(__nv_bfloat16);
  const size_t buf_b = qb_batch * NQ * (size_t)Scap_mem * cap * sizeof(uint2);
  auto up = [](size_t v) { return (v + 1023) & ~(size_t)1023; };
  const size_t off_q = up(xt_b), off_b = up(off_q + qt_b), off_t = up(off_b + buf_b);
  const size_t off_g = up(off_t + nq_pad * sizeof(float));
  const size_t off_c = up(off_g + nq * sizeof(uint32_t));
  const size_t bytes = off_c + nq * (size_t)Scap_mem * sizeof(int) + nq * sizeof(int) + 256;
  char* mem = nullptr;
  AQ_CUDA(cudaMallocAsync((void**)&mem, bytes, s->stream));
  __nv_bfloat16* xtile = (__nv_bfloat16*)mem;
  __nv_bfloat16* qtile = (__nv_bfloat16*)(mem + off_q);
  uint2* obuf = (uint2*)(mem + off_b);
  float* twoB = (float*)(mem + off_t);
  uint32_t* gcut = (uint32_t*)(mem + off_g);
  int* ocnt = (int*)(mem + off_c);
  int* oflag = ocnt + nq * (size_t)Scap_mem;
  int st = AQ_OK;
  if (cudaMemsetAsync(oflag, 0, nq * sizeof(int), s->stream) != cudaSuccess ||
      cudaMemsetAsync(gcut, 0, nq * sizeof(uint32_t), s->stream) != cudaSuccess)
    st = ref_error(AQ_E_CUDA, "memset failed");
  auto kern = NQ == 256 ? (terms == 3 ? k_exact_tc<256, 3> : k_exact_tc<256, 1>)
                        : (terms == 3 ? k_exact_tc<128, 3> : k_exact_tc<128, 1>);
  const size_t smem = tc_smem(NQ, Kp, NS, terms);
  if (st == AQ_OK &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
          cudaSuccess)
    st = ref_error(AQ_E_CUDA, "shared memory attribute");
  int mcap = kFMergeCapMin;
  while (mcap < N + N / 2 + 1024 && mcap < kFMergeCapMax) mcap <<= 1;
  const size_t msmem = (size_t)mcap * (sizeof(unsigned long long) + sizeof(uint32_t));
  if (st == AQ_OK)
    cudaFuncSetAttribute(k_exact_fmerge, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem);
  if (st == AQ_OK) {
    timer_mark(s, AQ_T_EXACT);
    k_tc_points<<<(unsigned)nblk, 256, 0, s->stream>>>(ds->xr, n, (int)d, Kp, terms, xtile);
    k_tc_queries<<<(unsigned)nq_pad, 128, 0, s->stream>>>(Qd, (int)nq, (int)d, Kp, NQ, terms,
                                                          xmax, qtile, twoB, oflag);
    s->launches += 2;
    for (size_t qb0 = 0; qb0 < nqb && st == AQ_OK; qb0 += qb_batch) {
      const size_t nqb_b = std::min(qb_batch, nqb - qb0);
      const size_t q0 = qb0 * NQ, nq_b = std::min(nq, (qb0 + nqb_b) * NQ) - q0;
      const int S = choose_S(nqb_b, Scap_mem);
      const int T = (nblk + S - 1) / S;
      const size_t items = (size_t)S * nqb_b;
      TArgs a{xtile, qtile + qb0 * 2 * (size_t)NQ * Kp, twoB + q0, gcut + q0, n, Kp, (int)nq_b,
              N, cap, (int)nqb_b, S, T, nblk, NS, (int)items, obuf, ocnt + q0 * S, oflag + q0};
      kern<<<(unsigned)std::min<size_t>(G0, items), kTThreads, smem, s->stream>>>(a);
      FArgs fa{nullptr, 0, (int)d, n, nullptr, twoB + q0, (int)nq_b, N, cap, S,
               0, (int)nqb_b, mcap, obuf, ocnt + q0 * S, oflag + q0};
      k_exact_fmerge<<<(unsigned)nq_b, S >= 32 ? 1024 : 256, msmem, s->stream>>>(
          fa, ds->xr, Qd + q0 * d, (int)te, ids + q0 * te, scores + q0 * te);
      s->launches += 2;
      if (cudaGetLastError() != cudaSuccess) st = ref_error(AQ_E_CUDA, "tensor-core exact filter failed");
    }
    timer_mark(s, AQ_T_EXACT);
    if (st == AQ_OK &&
        (cudaMemcpyAsync(hflag.data(), oflag, nq * sizeof(int), cudaMemcpyDeviceToHost,
                         s->stream) != cudaSuccess ||
         cudaStreamSynchronize(s->stream) != cudaSuccess))
      st = ref_error(AQ_E_CUDA, "tensor-core exact filter failed");
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

namespace {
// float32 FFMA filter + the float64 merge (the tier after the tensor cores)
int ffma_filter_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                       double* scores, std::vector<int>& hflag, double xmax, bool* ran) {
  *ran = false;
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const size_t te = std::min(depth, n);
  const int N = (int)te;
  const size_t nqb = (nq + kFQ - 1) / kFQ, nq_pad = nqb * kFQ;
  const size_t smem = (size_t)d * kFQ * sizeof(float) + kFQ * 16 + 64;
  if (smem > 200 * 1024) return AQ_OK;
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

__global__ void k_gather_queries(const double* Q, const uint32_t* idx, int d, double* out) {
  const double* src = Q + (size_t)idx[blockIdx.x] * d;
  for (int j = threadIdx.x; j < d; j += blockDim.x) out[(size_t)blockIdx.x * d + j] = src[j];
}
__global__ void k_scatter_hits(const uint32_t* ids_sub, const double* sc_sub, const uint32_t* idx,
                               int te, uint32_t* ids, double* scores) {
  const size_t q = idx[blockIdx.x];
  for (int e = threadIdx.x; e < te; e += blockDim.x) {
    ids[q * te + e] = ids_sub[(size_t)blockIdx.x * te + e];
    scores[q * te + e] = sc_sub[(size_t)blockIdx.x * te + e];
  }
}

// Runs one filter tier on the queries still flagged (hflag != 0): all of
// them in place, or a gathered subset whose hits and flags are scattered back.
template <class Tier>
int run_tier(aq_session* s, const double* Qd, size_t nq, size_t d, size_t te, uint32_t* ids,
             double* scores, std::vector<int>& hflag, bool* any_ran, Tier&& tier) {
  std::vector<uint32_t> idx;
  for (size_t q = 0; q < nq; ++q)
    if (hflag[q]) idx.push_back((uint32_t)q);
  if (idx.empty()) return AQ_OK;
  bool ran = false;
  if (idx.size() == nq) {
    std::vector<int> hf(nq, 1);
    AQ_TRY(tier(Qd, nq, ids, scores, hf, &ran));
    if (ran) hflag.swap(hf);
  } else {
    const size_t m = idx.size();
    char* mem = nullptr;
    const size_t b_idx = (m * 4 + 255) & ~(size_t)255, b_q = m * d * 8, b_ids = (m * te * 4 + 255) & ~(size_t)255;
    AQ_CUDA(cudaMallocAsync((void**)&mem, b_idx + b_q + b_ids + m * te * 8, s->stream));
    uint32_t* didx = (uint32_t*)mem;
    double* qsub = (double*)(mem + b_idx);
    uint32_t* ids_sub = (uint32_t*)(mem + b_idx + b_q);
    double* sc_sub = (double*)(mem + b_idx + b_q + b_ids);
    int st = AQ_OK;
    if (cudaMemcpyAsync(didx, idx.data(), m * 4, cudaMemcpyHostToDevice, s->stream) != cudaSuccess)
      st = ref_error(AQ_E_CUDA, "query gather failed");
    if (st == AQ_OK) {
      k_gather_queries<<<(unsigned)m, 128, 0, s->stream>>>(Qd, didx, (int)d, qsub);
      s->launches++;
      std::vector<int> hf(m, 1);
      st = tier(qsub, m, ids_sub, sc_sub, hf, &ran);
      if (st == AQ_OK && ran) {
        k_scatter_hits<<<(unsigned)m, 128, 0, s->stream>>>(ids_sub, sc_sub, didx, (int)te, ids,
                                                            scores);
        s->launches++;
        for (size_t i = 0; i < m; ++i) hflag[idx[i]] = hf[i];
      }
    }
    cudaFreeAsync(mem, s->stream);
    if (st == AQ_OK && cudaStreamSynchronize(s->stream) != cudaSuccess)
      st = ref_error(AQ_E_CUDA, "query scatter failed");
    AQ_TRY(st);
  }
  *any_ran |= ran;
  return AQ_OK;
}
}  // namespace

// Exact MIPS through the filter tiers: three-term tensor cores, then float32
// FFMA; each tier takes the queries the previous one flagged (non-finite
// values, overflowing windows) and the caller's float64 path the rest.
// $AQ_EXACT_TC: 1 (default) as above, 13 the one-term tensor-core tier first
// (three times fewer MMAs, but its wide window appends more than it saves
// while the window cuts come from single segments: DESIGN.md 4.3), 0 the
// float32 filter alone.
int exact_filter_device(aq_dataset* ds, const double* Qd, size_t nq, size_t depth, uint32_t* ids,
                        double* scores, std::vector<int>& hflag, bool* ran) {
  *ran = false;
  aq_session* s = ds->s;
  const size_t n = ds->n, d = ds->d;
  const size_t te = std::min(depth, n);
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
  static const int use_tc = getenv("AQ_EXACT_TC") ? atoi(getenv("AQ_EXACT_TC")) : 1;
  std::fill(hflag.begin(), hflag.end(), 1);
  for (int terms : {1, 3}) {
    if (!use_tc || (terms == 1 && use_tc != 13)) continue;
    AQ_TRY(run_tier(s, Qd, nq, d, te, ids, scores, hflag, ran,
                    [&](const double* Q, size_t m, uint32_t* I, double* S, std::vector<int>& hf,
                        bool* r) { return exact_tc_device(ds, Q, m, depth, I, S, hf, xmax, terms, r); }));
  }
  AQ_TRY(run_tier(s, Qd, nq, d, te, ids, scores, hflag, ran,
                  [&](const double* Q, size_t m, uint32_t* I, double* S, std::vector<int>& hf,
                      bool* r) { return ffma_filter_device(ds, Q, m, depth, I, S, hf, xmax, r); }));
  return AQ_OK;
}

}  // namespace aqd
