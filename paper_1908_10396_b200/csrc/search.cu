// Query path: LUT build (build_lut, index.hpp:56-70), 4-bit ADC scoring with
// top-N selection (adc_search / select_top, index.hpp:88-134), exact-dot
// rerank (north_star; restated from exact_search, index.hpp:137-147) and
// brute-force exact MIPS (exact_ground_truth, index.hpp:150-162).
//
// Exactness. The reference scores a point by summing M
// float64 LUT entries in subspace order and orders hits by (score desc,
// index asc). The scoring kernel sums 13-bit integer images of the entries
// (v = rint(lut / s), s = max|lut| / 4095; the integer sum S is exact and
// |s S - score| <= M s / 2) and keeps, per query, every point with
// S >= theta - M - 1, theta being an integer score that at least N points
// reach. The merge kernel re-scores that window in float64 in the
// reference's order and sorts exactly, so ids AND scores equal the
// reference's. Inputs whose windows do not fit (massive ties, N > 512) take
// an exact full-sort fallback.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace aqd {

int sort_scores_desc(aq_session* s, const double* scores, uint32_t* idx,
                     size_t n);
bool adc_tc_supported(int M, int bits, int k);
int adc_tc_queries();
int adc_tc_plan(aq_session* s, size_t nq, size_t n, int M, size_t* R, size_t* chunk, size_t* G);
int adc_tc_launch(aq_session* s, const uint8_t* codes, size_t n, int stride, const uint8_t* lutA,
                  int M, size_t nq, int N, int cap, size_t R, size_t chunk, size_t G, uint2* obuf,
                  int* ocnt, int* oflag);

// Scoring CTA shapes: query pairs per CTA, points per tile (= threads),
// min CTAs per SM. Selected per launch (AQ_ADC_VARIANT overrides).
struct AdcShape {
  int qp, tile, minb;
  bool gbuf;  // candidate windows in global memory (L2) instead of shared
};
// 1 (default): windows in global memory, 4 CTAs/SM; 0: shared-memory windows
// (the first design, kept as a reference point); 2: 2 query pairs, 6 CTAs/SM.
// The others measured in this round (6 or 12 query pairs, 3 CTAs/SM, 8-bit
// entries) were slower on config 2 and were dropped.
constexpr AdcShape kShapes[] = {{8, 256, 2, false}, {8, 256, 4, true}, {4, 256, 6, true}};
constexpr int kGbPointsPerThread = 4;  // points per thread between barriers (GB)
constexpr int kNumShapes = sizeof(kShapes) / sizeof(kShapes[0]);
constexpr int kLutQP = 16;  // lut kernel of the single-query host entry
constexpr int kMaxTopN = 4096;   // fast path limit
constexpr int kMergeCapMin = 2048, kMergeCapMax = 8192;  // merge window (shared)
constexpr int kQMax = 4095;      // |v| <= 4095: 13-bit fields, 8 adds per 16-bit lane

// ---- LUT ---------------------------------------------------------------------
// One CTA per query: lut64[q][m][j] exactly as build_lut computes it, and the
// integer filter table: v = rint(lut / s) + 4096 with s = max|lut| / 4095, so
// |s v' - lut| <= s / 2 per entry and a sum of M entries is within M s / 2 of
// the exact score. Two queries share a 32-bit word (low = even query) and
// two such pairs an 8-byte slot: layout [qblock][pair/2][M][16] x uint2, so
// one LDS.64 per (subspace, code) serves four queries. (8-bit entries would
// halve shared-memory traffic, but trained LUTs have a few large entries and
// 127 levels widen the candidate windows past any fixed capacity.)
__global__ void k_build_lut(const double* __restrict__ Q, int nq, int d,
                            const double* __restrict__ cb, int M, int k,
                            int sd, double* __restrict__ lut64,
                            uint16_t* __restrict__ lutq, int QP,
                            uint8_t* __restrict__ lutA) {
  __shared__ double red[32];
  const int q = blockIdx.x;
  const double* qv = Q + (size_t)q * d;
  double* L = lut64 + (size_t)q * M * k;
  double mx = 0.0;
  for (int e = threadIdx.x; e < M * k; e += blockDim.x) {
    const int m = e / k;
    const double* c = cb + (size_t)e * sd;
    double v = 0.0;  // detail::dot (geometry.hpp:170-174)
    for (int t = 0; t < sd; ++t) v = __dadd_rn(v, __dmul_rn(qv[m * sd + t], c[t]));
    L[e] = v;
    mx = fmax(mx, fabs(v));
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int t = 0; t < (int)(blockDim.x >> 5); ++t) mx = fmax(mx, red[t]);
  const double sc = mx > 0.0 ? mx / kQMax : 1.0;
  const int qb = q / (2 * QP), qi = q % (2 * QP);
  const int pp = qi / 2;  // query pair within the block
  uint16_t* T = lutq + ((((size_t)qb * (QP / 2) + pp / 2) * M * 16) * 2 + (pp & 1)) * 2 + (qi & 1);
  for (int e = threadIdx.x; e < M * 16; e += blockDim.x) {
    const int m = e / 16, j = e % 16;
    int v = 0;
    if (j < k) {
      v = (int)rint(L[m * k + j] / sc);
      v = max(-kQMax, min(kQMax, v));
    }
    T[(size_t)e * 4] = (uint16_t)(v + kQMax + 1);
    if (lutA) {  // tensor-core filter bytes: u = 64 hi + lo (adc_tc.cu)
      const unsigned u = (unsigned)(v + kQMax + 1);
      uint8_t* Aq = lutA + ((size_t)q * M + m) * 32;
      Aq[j] = (uint8_t)(u >> 6);
      Aq[16 + j] = (uint8_t)(u & 63u);
    }
  }
}

// ---- scoring with a per-CTA candidate window ------------------------------------

struct ScoreArgs {
  const uint8_t* codes;
  size_t n;
  int stride;      // bytes per code row
  const uint32_t* lutq;
  int M;
  int nq;
  int N;           // top-N
  int cap;         // candidate buffer per query
  size_t range_len;
  int R;           // number of point ranges (window slots per query)
  size_t chunk;    // > 0: persistent slices of chunk (query block, point) pairs
  int nqb;         // query blocks
  uint2* out_buf;  // [q][r][cap] {integer score, index}
  int* out_cnt;    // [q][r]
  int* out_flag;   // [q]
};

// Warp-cooperative: the N-th largest integer score among buf[0..cnt);
// false when cnt < N.
// top: highest bit any key can have (keys <= M * 8191, 13-bit LUT entries).
__device__ bool warp_nth_largest(const uint2* buf, int cnt, int N, unsigned* out, int top) {
  if (cnt < N) return false;
  const int lane = threadIdx.x & 31;
  unsigned T = 0u;
  for (int bit = top; bit >= 0; --bit) {
    const unsigned cand = T | (1u << bit);
    int c = 0;
    for (int e = lane; e < cnt; e += 32) c += buf[e].x >= cand;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= N) T = cand;
  }
  *out = T;
  return true;
}

// Keep only entries >= cut (warp-cooperative, in place); returns new count.
__device__ int warp_compact(uint2* buf, int cnt, int cut) {
  const int lane = threadIdx.x & 31;
  int kept = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int e = base + lane;
    uint2 v = make_uint2(0, 0);
    bool keep = false;
    if (e < cnt) {
      v = buf[e];
      keep = (int)v.x >= cut;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) buf[kept + __popc(bal & ((1u << lane) - 1u))] = v;
    kept += __popc(bal);
    __syncwarp();
  }
  return kept;
}

// Integer-LUT ADC over one (query block, point range). Each lane owns a point;
// per 8 subspaces and query pair, 8 LDS.32 words (two 16-bit entries each)
// are summed with IADD3 into packed 16-bit lanes, then split into 32-bit
// accumulators. Shared-memory delivery is the bound: 64 lookups per
// wavefront. MP > 0 fixes M at compile time (immediate LDS offsets).
// GB: the per-query candidate windows live in this CTA's slice of out_buf
// (global, L2-resident; appends are rare once the cut has risen) instead of
// shared memory, so shared memory holds only the LUT and more CTAs fit.
template <int MP, int QP, int TILE, int MINB, bool GB>
__global__ void __launch_bounds__(TILE, MINB) k_adc_score(const ScoreArgs a) {
  static_assert(QP % 2 == 0, "LUT slots hold two query pairs");
  constexpr int QB = 2 * QP;
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = MP > 0 ? MP : a.M;
  uint32_t* T = reinterpret_cast<uint32_t*>(smem);  // [QP][M][16]
  int* cut = reinterpret_cast<int*>(T + QP * M * 16);
  int* cnt = cut + QB;
  int* flag = cnt + QB;
  const size_t total = (size_t)a.nqb * a.n;
  // Segments: one (query block, point range) per CTA (grid mode), or a
  // persistent slice [c chunk, (c + 1) chunk) of the linearised (query block,
  // point) space split at query-block edges; the segment's window slot is
  // its index among the CTAs covering that query block.
  size_t Lpos = a.chunk ? (size_t)blockIdx.x * a.chunk : 0;
  const size_t Lend = a.chunk ? min(total, Lpos + a.chunk) : 1;
  while (Lpos < Lend) {
  int qb, r;
  size_t start, end;
  if (a.chunk) {
    qb = (int)(Lpos / a.n);
    start = Lpos % a.n;
    end = min(a.n, start + (Lend - Lpos));
    r = (int)(blockIdx.x - ((size_t)qb * a.n) / a.chunk);
    Lpos += end - start;
  } else {
    qb = blockIdx.y;
    r = blockIdx.x;
    start = (size_t)r * a.range_len;
    end = min(a.n, start + a.range_len);
    Lpos = Lend;
  }
  __syncthreads();  // the previous segment is done with the LUT and counters
  // window of query q: shared [QB][cap], or out_buf[(qb QB + q) R + r][cap]
  uint2* const buf = GB ? a.out_buf + ((size_t)qb * QB * a.R + r) * a.cap
                        : reinterpret_cast<uint2*>(flag + QB);
  const size_t qstride = GB ? (size_t)a.R * a.cap : (size_t)a.cap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.lutq + (size_t)qb * QP * M * 16);
    uint4* dst = reinterpret_cast<uint4*>(T);
    for (int t = threadIdx.x; t < QP * M * 4; t += blockDim.x) dst[t] = src[t];
  }
  if (threadIdx.x < QB) {
    // padding slots of the last query block never append
    cut[threadIdx.x] = qb * QB + (int)threadIdx.x < a.nq ? INT_MIN : INT_MAX;
    cnt[threadIdx.x] = 0;
    flag[threadIdx.x] = 0;
  }
  __syncthreads();
  const int cap = a.cap;
  const int margin = M + 1;  // 2 * (M s / 2) / s, plus one unit for float64
  const int top = 31 - __clz(max(M * 8191, 1));
  // points scored between two barriers (windows in global memory are cheap
  // to size for it; shared windows keep one point per thread)
  constexpr int PPT = GB ? kGbPointsPerThread : 1;
  constexpr int SPAN = TILE * PPT;
  // the first span is one tile: its appends (cut still INT_MIN) set the cut
  for (size_t tb = start; tb < end;) {
    const int nu = tb == start ? 1 : PPT;
#pragma unroll 1
   for (int u = 0; u < nu; ++u) {
    const size_t p = tb + (size_t)u * TILE + threadIdx.x;
    if (p < end) {
      uint32_t acc[QB];
#pragma unroll
      for (int q = 0; q < QB; ++q) acc[q] = 0u;
      const uint32_t* crow = reinterpret_cast<const uint32_t*>(a.codes + p * a.stride);
      // MP > 0: the row's code words in registers up front, in 16- (or 8-)
      // byte loads: a warp's narrow loads at a 32-byte row stride each touch
      // eight 128-byte lines, so seven 4-byte loads cost the L1 pipe 56
      // wavefronts per 32 points against 16 for two 16-byte loads; the
      // chunk loop then shifts the next word down (static indices)
      constexpr int kNW = MP > 0 ? (MP + 7) / 8 : 1;
      constexpr int kStride = (((MP > 0 ? MP : 2) + 1) / 2 + 7) & ~7;  // code_stride(MP, 4)
      uint32_t cw[kNW];
      if constexpr (MP > 0) {
        if constexpr (kStride % 16 == 0) {
          const uint4* r4 = reinterpret_cast<const uint4*>(crow);
#pragma unroll
          for (int i = 0; i < (kNW + 3) / 4; ++i) {
            const uint4 v = __ldg(r4 + i);
            if (4 * i < kNW) cw[4 * i] = v.x;
            if (4 * i + 1 < kNW) cw[4 * i + 1] = v.y;
            if (4 * i + 2 < kNW) cw[4 * i + 2] = v.z;
            if (4 * i + 3 < kNW) cw[4 * i + 3] = v.w;
          }
        } else {
          const uint2* r2 = reinterpret_cast<const uint2*>(crow);
#pragma unroll
          for (int i = 0; i < (kNW + 1) / 2; ++i) {
            const uint2 v = __ldg(r2 + i);
            if (2 * i < kNW) cw[2 * i] = v.x;
            if (2 * i + 1 < kNW) cw[2 * i + 1] = v.y;
          }
        }
      }
      // full chunks of 8 subspaces, then the tail (compile-time when MP > 0)
      const int nfull = M >> 3, tail = M & 7;
#pragma unroll 1
      for (int ch = 0; ch < nfull; ++ch) {
        uint32_t w;
        if constexpr (MP > 0) {
          w = cw[0];
#pragma unroll
          for (int i = 0; i + 1 < kNW; ++i) cw[i] = cw[i + 1];
        } else {
          w = __ldg(crow + ch);
        }
        int off[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) off[t] = (ch * 8 + t) * 16 + ((w >> (4 * t)) & 15u);
#pragma unroll
        for (int qq = 0; qq < QP / 2; ++qq) {
          const uint2* Tq = reinterpret_cast<const uint2*>(T) + qq * M * 16;
          const uint2 v0 = Tq[off[0]], v1 = Tq[off[1]], v2 = Tq[off[2]], v3 = Tq[off[3]];
          const uint2 v4 = Tq[off[4]], v5 = Tq[off[5]], v6 = Tq[off[6]], v7 = Tq[off[7]];
          const uint32_t pa = (v0.x + v1.x + v2.x) + (v3.x + v4.x + v5.x) + (v6.x + v7.x);
          const uint32_t pb = (v0.y + v1.y + v2.y) + (v3.y + v4.y + v5.y) + (v6.y + v7.y);
          acc[4 * qq] += pa & 0xffffu;
          acc[4 * qq + 1] += pa >> 16;
          acc[4 * qq + 2] += pb & 0xffffu;
          acc[4 * qq + 3] += pb >> 16;
        }
      }
      if (tail) {
        uint32_t w;
        if constexpr (MP > 0)
          w = cw[0];
        else
          w = __ldg(crow + nfull);
        int off[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) off[t] = (nfull * 8 + t) * 16 + ((w >> (4 * t)) & 15u);
#pragma unroll
        for (int qq = 0; qq < QP / 2; ++qq) {
          const uint2* Tq = reinterpret_cast<const uint2*>(T) + qq * M * 16;
          uint32_t pa = 0u, pb = 0u;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < tail) {
              const uint2 v = Tq[off[t]];
              pa += v.x;
              pb += v.y;
            }
          acc[4 * qq] += pa & 0xffffu;
          acc[4 * qq + 1] += pa >> 16;
          acc[4 * qq + 2] += pb & 0xffffu;
          acc[4 * qq + 3] += pb >> 16;
        }
      }
#pragma unroll
      for (int q4 = 0; q4 < QB; q4 += 4) {  // cuts four at a time (one broadcast LDS.128)
        const int4 c4 = *reinterpret_cast<const int4*>(cut + q4);
        const int cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q4 + u;
          if ((int)acc[q] >= cv[u]) {
            const int pos = atomicAdd(&cnt[q], 1);
            if (pos < cap)
              buf[q * qstride + pos] = make_uint2(acc[q], (unsigned)p);
            else
              flag[q] = 1;
          }
        }
      }
    }
   }
    tb += (size_t)nu * TILE;
    __syncthreads();
    // shrink buffers that could overflow during the next span
    for (int q = warp; q < QB; q += TILE / 32) {
      const int c = min(cnt[q], cap);
      unsigned th;
      if (c > cap - SPAN && !flag[q] && warp_nth_largest(buf + q * qstride, c, a.N, &th, top)) {
        const int cq = max(cut[q], (int)th - margin);
        const int kept = warp_compact(buf + q * qstride, c, cq);
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
  // final shrink + write-out
  for (int q = warp; q < QB; q += TILE / 32) {
    const int gq = qb * QB + q;
    int c = min(cnt[q], cap);
    unsigned th;
    if (warp_nth_largest(buf + q * qstride, c, a.N, &th, top))
      c = warp_compact(buf + q * qstride, c, max(cut[q], (int)th - margin));
    if (gq < a.nq) {
      if (!GB) {
        uint2* dst = a.out_buf + ((size_t)gq * a.R + r) * cap;
        for (int e = lane; e < c; e += 32) dst[e] = buf[q * qstride + e];
      }
      if (lane == 0) {
        a.out_cnt[(size_t)gq * a.R + r] = c;
        if (flag[q]) atomicOr(&a.out_flag[gq], 1);
      }
    }
    __syncwarp();
  }
  }  // segments
}

// ---- merge: global window, float64 re-scoring, exact order --------------------

struct MergeArgs {
  const uint2* buf;
  const int* cnt;
  int* flag;
  int R, cap, N, topn_eff;
  int mcap;  // merge window capacity: power of two, kMergeCapMin..kMergeCapMax
  const double* lut64;
  const uint8_t* codes;
  int stride, bits, M, k;
  uint32_t* ids;    // [q][topn_eff]
  double* scores;
};

__global__ void __launch_bounds__(1024) k_adc_merge(const MergeArgs a) {
  extern __shared__ __align__(16) unsigned char msm[];
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(msm);  // sort keys
  double* ssc = reinterpret_cast<double*>(skey + a.mcap);
  uint32_t* sid = reinterpret_cast<uint32_t*>(ssc + a.mcap);
  __shared__ int ncol;
  const int q = blockIdx.x;
  if (a.flag[q]) return;  // handled by the exact fallback
  const int tid = threadIdx.x;
  // total entries
  const uint2* lists = a.buf + (size_t)q * a.R * a.cap;
  const int* cnts = a.cnt + (size_t)q * a.R;
  // global N-th largest integer score over the union (radix select; the
  // histogram borrows the sort-key space, filled only later)
  unsigned T = 0u;
  int total = 0;
  for (int r = tid & 31; r < a.R; r += 32) total += cnts[r];  // each warp, redundantly
  total = __reduce_add_sync(0xffffffffu, total);
  const bool have = total >= a.N;
  if (have) T = block_nth_largest(lists, cnts, a.R, a.cap, a.N, reinterpret_cast<unsigned*>(skey));
  const int cutv = have ? (int)T - (a.M + 1) : INT_MIN;
  if (tid == 0) ncol = 0;
  __syncthreads();
  for (int r = tid >> 5; r < a.R; r += blockDim.x >> 5)  // warp per window
    for (int e = tid & 31; e < cnts[r]; e += 32) {
      const uint2 v = lists[(size_t)r * a.cap + e];
      if ((int)v.x >= cutv) {
        const int pos = atomicAdd(&ncol, 1);
        if (pos < a.mcap) sid[pos] = v.y;
      }
    }
  __syncthreads();
  const int nc = ncol;
  if (nc > a.mcap) {
    if (tid == 0) a.flag[q] = 2;
    return;
  }
  // float64 re-scoring in the reference's order (index.hpp:127-133)
  const double* lq = a.lut64 + (size_t)q * a.M * a.k;
  for (int e = tid; e < nc; e += blockDim.x) {
    const uint8_t* row = a.codes + (size_t)sid[e] * a.stride;
    double s = 0.0;
    for (int m = 0; m < a.M; ++m) s = __dadd_rn(s, lq[m * a.k + get_code(row, m, a.bits)]);
    ssc[e] = s;
  }
  // bitonic sort of (score desc, index asc) over the next power of two
  int P = 1;
  while (P < nc) P <<= 1;
  for (int e = tid; e < P; e += blockDim.x) {
    if (e < nc) {
      unsigned long long b = (unsigned long long)__double_as_longlong(ssc[e]);
      b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
      skey[e] = ~b;  // ascending == score descending
    } else {
      skey[e] = ~0ull;
      sid[e] = 0xffffffffu;
    }
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = tid; e < P; e += blockDim.x) {
        const int o = e ^ stride;
        if (o > e) {
          const bool up = (e & size) == 0;
          const unsigned long long ka = skey[e], kb = skey[o];
          const uint32_t ia = sid[e], ib = sid[o];
          const bool gt = ka > kb || (ka == kb && ia > ib);
          if (gt == up) {
            skey[e] = kb;
            skey[o] = ka;
            sid[e] = ib;
            sid[o] = ia;
          }
        }
      }
      __syncthreads();
    }
  for (int e = tid; e < a.topn_eff; e += blockDim.x) {
    unsigned long long b = ~skey[e];
    b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    a.ids[(size_t)q * a.topn_eff + e] = sid[e];
    a.scores[(size_t)q * a.topn_eff + e] = __longlong_as_double((long long)b);
  }
}

// ---- exact fallback: all float64 scores + stable radix sort ---------------------

__global__ void k_adc_all_scores(const uint8_t* __restrict__ codes, size_t n,
                                 int stride, int bits, int M, int k,
                                 const double* __restrict__ lq,
                                 double* __restrict__ out,
                                 uint32_t* __restrict__ idx) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* row = codes + i * stride;
  double s = 0.0;
  for (int m = 0; m < M; ++m) s = __dadd_rn(s, lq[m * k + get_code(row, m, bits)]);
  out[i] = s;
  idx[i] = (uint32_t)i;
}

__global__ void k_gather_top(const uint32_t* __restrict__ idx,
                             const double* __restrict__ scores_by_point,
                             int topn_eff, uint32_t* ids, double* sc) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= topn_eff) return;
  ids[e] = idx[e];
  sc[e] = scores_by_point[idx[e]];
}

// Device-pointer core. Q (float64, nq x d), ids/scores device (nq x topn_eff).
int adc_search_device(aq_codes* codes, aq_codebook* cb, const double* Qd,
                      size_t nq, size_t topn, uint32_t* ids, double* scores) {
  aq_session* s = codes->s;
  AQ_TRY(check_session(s));
  if (codes->n == 0) return ref_error(AQ_E_EMPTY_INDEX, "no quantized datapoints");
  if (topn < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  if (codes->M != cb->M || codes->k > cb->k)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match codebook");
  if (cb->k > 256 || (codes->bits == 4 && cb->k > 16 && codes->k > 16))
    return ref_error(AQ_E_UNSUPPORTED, "device search supports k <= 256");
  if (cb->M > 1024) return ref_error(AQ_E_UNSUPPORTED, "device search supports M <= 1024");
  if (nq == 0) return AQ_OK;
  const int M = (int)cb->M, k = (int)cb->k;
  const size_t n = codes->n;
  const size_t topn_eff = std::min(topn, n);
  const size_t d = cb->M * cb->sd;
  int variant = 1;
  if (const char* v = getenv("AQ_ADC_VARIANT")) variant = std::min(std::max(atoi(v), 0), kNumShapes - 1);
  if (!kShapes[variant].gbuf && topn > 512) variant = 1;  // shared windows hold N <= 512
  const AdcShape shp = kShapes[variant];
  const int QB = 2 * shp.qp, TILE = shp.tile;
  const size_t nqb = (nq + QB - 1) / QB;
  // Tensor-core filter (adc_tc.cu) for long per-SM slices: each slice pays
  // a window warm-up (appends and shrinks until its cut rises) that the
  // scalar kernel amortises better on short ones. Measured (bench.py, one
  // B200): config 4 (1e8 x 4,096, 2.8e6 points per SM slice) 1217 -> 842 ms,
  // config 2 (1.18e6 x 10,000, 6.3e5 per slice) 41.0 -> 48.3 ms, so the
  // default takes it from 1.5e6 points per slice. AQ_ADC_TC=1 / 0 forces it
  // on / off. M > 50 and 8-bit codes always take the scalar kernel.
  static const int tc_env = getenv("AQ_ADC_TC") ? atoi(getenv("AQ_ADC_TC")) : -1;
  const size_t per_sm = ((nq + 127) / 128) * n / (size_t)s->num_sms;
  const bool use_tc = adc_tc_supported(M, codes->bits, k) && topn <= (size_t)kMaxTopN &&
                      (tc_env == 1 || (tc_env < 0 && per_sm >= 1500000));
  // workspace
  const size_t lut64_b = nq * M * k * sizeof(double);
  const size_t lutq_b = nqb * shp.qp * (size_t)M * 16 * sizeof(uint32_t);
  const size_t luta_b = use_tc ? nq * (size_t)M * 32 : 0;
  void* p;
  // the score kernel stages the filter table with 16-byte loads: its offset
  // is rounded up (nq M k doubles can be an odd multiple of 8 bytes)
  const size_t lutq_off = (lut64_b + 255) & ~(size_t)255;
  const size_t luta_off = (lutq_off + lutq_b + 255) & ~(size_t)255;
  AQ_TRY(scratch(s, 1, luta_off + luta_b + 256, &p));
  double* lut64 = (double*)p;
  uint32_t* lutq = (uint32_t*)((char*)p + lutq_off);
  uint8_t* luta = use_tc ? (uint8_t*)p + luta_off : nullptr;
  AQ_CUDA(cudaMemsetAsync(lutq, 0, lutq_b, s->stream));
  timer_mark(s, AQ_T_LUT);
  k_build_lut<<<(unsigned)nq, 256, 0, s->stream>>>(Qd, (int)nq, (int)d, cb->d64, M, k,
                                                  (int)cb->sd, lut64, (uint16_t*)lutq,
                                                  shp.qp, luta);
  AQ_LAUNCHED(s);
  timer_mark(s, AQ_T_LUT);

  const bool fast = codes->bits == 4 && topn <= (size_t)kMaxTopN && M <= 256;
  std::vector<int> hflag(nq, fast ? 0 : 1);
  // windows -> global theta, float64 re-scoring, exact order (both filters);
  // the per-query overflow flags come back to the host for the fallback
  auto merge = [&](const uint2* obuf, const int* ocnt, int* oflag, size_t R, int cap) -> int {
    const int N = (int)topn_eff;
    // merge window: N plus room for near-threshold ties, a power of two
    int mcap = kMergeCapMin;
    while (mcap < N + N / 2 + 1024 && mcap < kMergeCapMax) mcap <<= 1;
    MergeArgs ma{obuf, ocnt, oflag, (int)R, cap, N, (int)topn_eff, mcap, lut64,
                 codes->data, (int)codes->stride, codes->bits, M, k, ids, scores};
    const size_t msmem = (size_t)mcap * (2 * sizeof(double) + sizeof(uint32_t));
    AQ_CUDA(cudaFuncSetAttribute(k_adc_merge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)msmem));
    timer_mark(s, AQ_T_ADC_MERGE);
    // many windows per query (small batches): more warps walk them at once
    k_adc_merge<<<(unsigned)nq, R >= 32 ? 1024 : 256, msmem, s->stream>>>(ma);
    AQ_LAUNCHED(s);
    timer_mark(s, AQ_T_ADC_MERGE);
    AQ_CUDA(cudaMemcpyAsync(hflag.data(), oflag, nq * sizeof(int), cudaMemcpyDeviceToHost,
                            s->stream));
    AQ_CUDA(cudaStreamSynchronize(s->stream));
    return AQ_OK;
  };
  if (fast) {
    const int N = (int)topn_eff;
    // window: N, one span of appends, and room for near-threshold ties
    // (their count grows with the depth of the N-th score)
    const int cap = ((N + 31) & ~31) + TILE * (shp.gbuf ? kGbPointsPerThread : 1) + 32 +
                    (N > 128 ? N : 0);
    if (use_tc) {
      const int TQ = adc_tc_queries();
      // per-(query, slice) list handed to the merge: N plus room for
      // near-threshold ties, as the scalar kernel's (the work windows inside
      // the kernel are larger)
      const int cap = ((N + 31) & ~31) + 1024 + 32 + (N > 128 ? N : 0);
      size_t R, chunk, G;
      AQ_TRY(adc_tc_plan(s, nq, n, M, &R, &chunk, &G));
      const size_t nq_pad = (nq + TQ - 1) / TQ * TQ;
      const size_t buf_b = nq_pad * R * cap * sizeof(uint2);
      void* p2;
      AQ_TRY(scratch(s, 3, buf_b + nq * R * sizeof(int) + nq * sizeof(int) + 256, &p2));
      uint2* obuf = (uint2*)p2;
      int* ocnt = (int*)(obuf + nq_pad * R * cap);
      int* oflag = ocnt + nq * R;
      AQ_CUDA(cudaMemsetAsync(oflag, 0, nq * sizeof(int), s->stream));
      AQ_CUDA(cudaMemsetAsync(ocnt, 0, nq * R * sizeof(int), s->stream));
      timer_mark(s, AQ_T_ADC_SCORE);
      AQ_TRY(adc_tc_launch(s, codes->data, n, (int)codes->stride, luta, M, nq, N, cap, R, chunk,
                           G, obuf, ocnt, oflag));
      timer_mark(s, AQ_T_ADC_SCORE);
      AQ_TRY(merge(obuf, ocnt, oflag, R, cap));
    } else {
    // point ranges: enough CTAs for ~2 waves, ranges of whole tiles
    const size_t tiles = (n + TILE - 1) / TILE;
    // Windows in global memory: one persistent CTA per resident slot, each
    // an equal slice of the (query block, point) space — no partial last
    // wave, long ranges. Shared windows (variant 0): ~4 waves of (query
    // block x point range) CTAs.
    static const int persist_env = getenv("AQ_ADC_PERSIST") ? atoi(getenv("AQ_ADC_PERSIST")) : 1;
    const bool persist = shp.gbuf && persist_env;
    size_t R, range_len = 0, chunk = 0, G = 0;
    if (persist) {
      G = (size_t)s->num_sms * shp.minb;
      const size_t total = nqb * n;
      static const size_t min_tiles =
          getenv("AQ_ADC_MINCHUNK") ? (size_t)atoi(getenv("AQ_ADC_MINCHUNK")) : 16;
      chunk = std::max<size_t>((total + G - 1) / G, min_tiles * (size_t)TILE);
      G = (total + chunk - 1) / chunk;
      R = 1;
      for (size_t qb = 0; qb < nqb; ++qb) {
        const size_t c0 = qb * n / chunk, c1 = ((qb + 1) * n - 1) / chunk;
        R = std::max(R, c1 - c0 + 1);
      }
    } else {
      static const int waves = getenv("AQ_ADC_WAVES") ? atoi(getenv("AQ_ADC_WAVES")) : 4;
      R = std::max<size_t>(1, (waves * (size_t)s->num_sms * shp.minb + nqb - 1) / nqb);
      R = std::min(R, tiles);
      range_len = ((tiles + R - 1) / R) * TILE;
      R = (n + range_len - 1) / range_len;
    }
    const size_t nq_pad = nqb * QB;  // GB windows exist for padding queries too
    const size_t buf_b = nq_pad * R * cap * sizeof(uint2);
    void* p2;
    AQ_TRY(scratch(s, 3, buf_b + nq * R * sizeof(int) + nq * sizeof(int) + 256, &p2));
    uint2* obuf = (uint2*)p2;
    int* ocnt = (int*)(obuf + nq_pad * R * cap);
    int* oflag = ocnt + nq * R;
    AQ_CUDA(cudaMemsetAsync(oflag, 0, nq * sizeof(int), s->stream));
    if (persist)  // query blocks covered by fewer slices leave slots empty
      AQ_CUDA(cudaMemsetAsync(ocnt, 0, nq * R * sizeof(int), s->stream));
    ScoreArgs sa{codes->data, n, (int)codes->stride, lutq, M, (int)nq, N, cap,
                 range_len, (int)R, chunk, (int)nqb, obuf, ocnt, oflag};
    const size_t smem = (size_t)shp.qp * M * 16 * sizeof(uint32_t) + 3 * QB * sizeof(int) +
                        (shp.gbuf ? 0 : (size_t)QB * cap * sizeof(uint2));
    if (smem > 227 * 1024)
      return ref_error(AQ_E_UNSUPPORTED, "ADC working set exceeds shared memory");
    const dim3 grid = persist ? dim3((unsigned)G, 1) : dim3((unsigned)R, (unsigned)nqb);
    timer_mark(s, AQ_T_ADC_SCORE);
#define AQ_SCORE_LAUNCH(MM, QPv, TL, MB, G)                                           \
  do {                                                                              \
    AQ_CUDA(cudaFuncSetAttribute(k_adc_score<MM, QPv, TL, MB, G>,                    \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_adc_score<MM, QPv, TL, MB, G><<<grid, TL, smem, s->stream>>>(sa);             \
  } while (0)
#define AQ_SCORE_V(MM)                                                  \
  switch (variant) {                                                   \
    case 0: AQ_SCORE_LAUNCH(MM, 8, 256, 2, false); break;              \
    case 2: AQ_SCORE_LAUNCH(MM, 4, 256, 6, true); break;               \
    default: AQ_SCORE_LAUNCH(MM, 8, 256, 4, true); break;              \
  }
#define AQ_SCORE_M(MM) \
  case MM:             \
    AQ_SCORE_V(MM)     \
    break;
    switch (M) {
      AQ_SCORE_M(16)
      AQ_SCORE_M(32)
      AQ_SCORE_M(48)
      AQ_SCORE_M(50)
      AQ_SCORE_M(64)
      AQ_SCORE_M(128)
      default:
        AQ_SCORE_V(0)
    }
#undef AQ_SCORE_M
#undef AQ_SCORE_LAUNCH
    AQ_LAUNCHED(s);
    timer_mark(s, AQ_T_ADC_SCORE);
    AQ_TRY(merge(obuf, ocnt, oflag, R, cap));
    }  // scalar filter
  }
  // exact fallback for flagged queries
  bool any = false;
  for (size_t q = 0; q < nq; ++q) any |= hflag[q] != 0;
  if (any) {
    void* p3;
    AQ_TRY(scratch(s, 4, n * (sizeof(double) + sizeof(uint32_t)) + 64, &p3));
    double* all = (double*)p3;
    uint32_t* idx = (uint32_t*)(all + n);
    for (size_t q = 0; q < nq; ++q) {
      if (!hflag[q]) continue;
      k_adc_all_scores<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(
          codes->data, n, (int)codes->stride, codes->bits, M, k, lut64 + q * M * k, all, idx);
      AQ_LAUNCHED(s);
      AQ_TRY(sort_scores_desc(s, all, idx, n));
      k_gather_top<<<(unsigned)((topn_eff + 255) / 256), 256, 0, s->stream>>>(
          idx, all, (int)topn_eff, ids + q * topn_eff, scores + q * topn_eff);
      AQ_LAUNCHED(s);
    }
  }
  return AQ_OK;
}

// ---- rerank (exact float64 dot, sequential order) -------------------------------

// One warp per query: candidates rescored with detail::dot against the row
// (float32-exact values) and the best `keep` returned in select_top order.
template <class TX>
__global__ void k_rerank(const TX* __restrict__ xr, int d,
                         const double* __restrict__ Q, int nq,
                         const uint32_t* __restrict__ cand, int ncand, int keep,
                         uint32_t* __restrict__ ids, double* __restrict__ sc,
                         size_t n, DevError* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wpb = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x * wpb + w;
  const int P = 1 << (32 - __clz(max(ncand, 2) - 1));  // next pow2
  unsigned long long* K = reinterpret_cast<unsigned long long*>(smem) + (size_t)w * P;
  uint32_t* I = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned long long*>(smem) + (size_t)wpb * P) + (size_t)w * P;
  if (q >= nq) return;
  const double* qv = Q + (size_t)q * d;
  for (int e = lane; e < P; e += 32) {
    if (e < ncand) {
      const uint32_t id = cand[(size_t)q * ncand + e];
      double s = 0.0;
      if (id < n) {
        const TX* row = xr + (size_t)id * d;  // row-major: contiguous gather
        for (int j = 0; j < d; ++j) s = __dadd_rn(s, __dmul_rn(qv[j], (double)row[j]));
      } else {
        report_error(err, (uint64_t)q, AQ_E_INVALID_ARGUMENT);
      }
      unsigned long long b = (unsigned long long)__double_as_longlong(s);
      b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
      K[e] = ~b;
      I[e] = id;
    } else {
      K[e] = ~0ull;
      I[e] = 0xffffffffu;
    }
  }
  __syncwarp();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = lane; e < P; e += 32) {
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
      __syncwarp();
    }
  for (int e = lane; e < keep; e += 32) {
    unsigned long long b = ~K[e];
    b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    ids[(size_t)q * keep + e] = I[e];
    sc[(size_t)q * keep + e] = __longlong_as_double((long long)b);
  }
}

// Exact float64 dots for candidate ids, in the given order (no selection):
// the per-shard half of the multi-GPU rerank.
template <class TX>
__global__ void k_exact_dots(const TX* __restrict__ xr, int d,
                             const double* __restrict__ Q, size_t nq,
                             const uint32_t* __restrict__ cand, size_t ncand, size_t n,
                             double* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nq * ncand) return;
  const size_t q = t / ncand;
  const uint32_t id = cand[t];
  double s = 0.0;
  if (id < n)
    for (int j = 0; j < d; ++j)
      s = __dadd_rn(s, __dmul_rn(Q[q * d + j], (double)xr[(size_t)id * d + j]));
  out[t] = id < n ? s : -INFINITY;
}

// Long candidate lists (> 4096, beyond one warp's shared-memory sort): per
// query, float64 dots of every candidate (k_exact_dots), then two stable radix
// sorts — candidate id ascending, then exact score descending — which is the
// (score desc, index asc) order of k_rerank.
__global__ void k_rerank_prep(const uint32_t* __restrict__ cand, size_t ncand, size_t n,
                              double* __restrict__ negid, uint32_t* __restrict__ pos,
                              DevError* err) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ncand) return;
  if (cand[e] >= n) report_error(err, e, AQ_E_INVALID_ARGUMENT);
  negid[e] = -(double)cand[e];  // exact: ids < 2^32
  pos[e] = (uint32_t)e;
}
__global__ void k_rerank_regather(const uint32_t* __restrict__ pos,
                                  const uint32_t* __restrict__ cand,
                                  const double* __restrict__ dots, size_t ncand,
                                  uint32_t* __restrict__ ids2, double* __restrict__ sc2,
                                  uint32_t* __restrict__ pos2) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ncand) return;
  ids2[e] = cand[pos[e]];
  sc2[e] = dots[pos[e]];
  pos2[e] = (uint32_t)e;
}
__global__ void k_rerank_take(const uint32_t* __restrict__ pos2,
                              const uint32_t* __restrict__ ids2,
                              const double* __restrict__ sc2, size_t keep,
                              uint32_t* __restrict__ ids, double* __restrict__ sc) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= keep) return;
  ids[e] = ids2[pos2[e]];
  sc[e] = sc2[pos2[e]];
}

static int rerank_long(aq_dataset* ds, const double* Qd, size_t nq, const uint32_t* cand,
                       size_t ncand, size_t keep_eff, uint32_t* ids, double* sc) {
  aq_session* s = ds->s;
  char* buf = nullptr;
  const size_t bytes = ncand * (3 * sizeof(double) + 3 * sizeof(uint32_t)) + 256;
  AQ_CUDA(cudaMallocAsync((void**)&buf, bytes, s->stream));
  double* dots = (double*)buf;
  double* negid = dots + ncand;
  double* sc2 = negid + ncand;
  uint32_t* pos = (uint32_t*)(sc2 + ncand);
  uint32_t* ids2 = pos + ncand;
  uint32_t* pos2 = ids2 + ncand;
  const unsigned g = (unsigned)((ncand + 255) / 256);
  int st = clear_dev_error(s);
  for (size_t q = 0; q < nq && st == AQ_OK; ++q) {
    const uint32_t* c = cand + q * ncand;
    k_rerank_prep<<<g, 256, 0, s->stream>>>(c, ncand, ds->n, negid, pos, s->err);
    AQ_XR_LAUNCH(ds, k_exact_dots, g, 256, 0, s->stream, (int)ds->d, Qd + q * ds->d, 1, c,
                 ncand, ds->n, dots);
    s->launches += 2;
    st = sort_scores_desc(s, negid, pos, ncand);  // id ascending
    if (st != AQ_OK) break;
    k_rerank_regather<<<g, 256, 0, s->stream>>>(pos, c, dots, ncand, ids2, sc2, pos2);
    s->launches++;
    st = sort_scores_desc(s, sc2, pos2, ncand);  // score descending, stable
    if (st != AQ_OK) break;
    k_rerank_take<<<(unsigned)((keep_eff + 255) / 256), 256, 0, s->stream>>>(
        pos2, ids2, sc2, keep_eff, ids + q * keep_eff, sc + q * keep_eff);
    s->launches++;
  }
  cudaFreeAsync(buf, s->stream);
  if (st != AQ_OK) return st;
  return sync_and_check(s, "rerank");
}

int rerank_device(aq_dataset* ds, const double* Qd, size_t nq,
                  const uint32_t* cand, size_t ncand, size_t keep, uint32_t* ids,
                  double* sc) {
  aq_session* s = ds->s;
  if (ncand == 0 || nq == 0) return AQ_OK;
  const size_t keep_eff = std::min(keep, ncand);
  if (ncand > 4096) return rerank_long(ds, Qd, nq, cand, ncand, keep_eff, ids, sc);
  int P = 1;
  while (P < (int)ncand) P <<= 1;
  const int wpb = std::max(1, std::min(8, (int)(40 * 1024 / (P * 12))));
  const size_t smem = (size_t)wpb * P * 12;
  AQ_TRY(clear_dev_error(s));
  timer_mark(s, AQ_T_RERANK);
  AQ_XR_LAUNCH(ds, k_rerank, (unsigned)((nq + wpb - 1) / wpb), wpb * 32, smem, s->stream,
               (int)ds->d, Qd, (int)nq, cand, (int)ncand, (int)keep_eff, ids, sc, ds->n,
               s->err);
  AQ_LAUNCHED(s);
  timer_mark(s, AQ_T_RERANK);
  return AQ_OK;
}

}  // namespace aqd

using namespace aqd;

namespace {

int upload_queries(aq_session* s, const double* Q, size_t nq, size_t d, int slot,
                   double** out) {
  void* p;
  AQ_TRY(scratch(s, slot, nq * d * sizeof(double) + 16, &p));
  if (nq * d)
    AQ_CUDA(cudaMemcpyAsync(p, Q, nq * d * sizeof(double), cudaMemcpyHostToDevice,
                            s->stream));
  *out = (double*)p;
  return AQ_OK;
}

}  // namespace

extern "C" {

int aq_dev_adc_search_d(aq_codes* codes, aq_codebook* cb, const double* q_dev,
                        size_t nq, size_t topn, uint32_t* ids_dev, double* scores_dev) {
  if (!codes || !cb) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  return adc_search_device(codes, cb, q_dev, nq, topn, ids_dev, scores_dev);
}

int aq_dev_adc_search(aq_codes* codes, aq_codebook* cb, const double* queries,
                      size_t nq, size_t topn, uint32_t* ids_out, double* scores_out) {
  if (!codes || !cb) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = codes->s;
  AQ_TRY(check_session(s));
  if (codes->n == 0) return ref_error(AQ_E_EMPTY_INDEX, "no quantized datapoints");
  if (topn < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  const size_t d = cb->M * cb->sd;
  const size_t te = std::min(topn, codes->n);
  double* Qd;
  AQ_TRY(upload_queries(s, queries, nq, d, 0, &Qd));
  uint32_t* ids;
  double* sc;
  AQ_CUDA(cudaMallocAsync(&ids, nq * te * sizeof(uint32_t) + 8, s->stream));
  AQ_CUDA(cudaMallocAsync(&sc, nq * te * sizeof(double) + 8, s->stream));
  int st = adc_search_device(codes, cb, Qd, nq, topn, ids, sc);
  if (st == AQ_OK && nq) {
    cudaMemcpyAsync(ids_out, ids, nq * te * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream);
    cudaMemcpyAsync(scores_out, sc, nq * te * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  }
  cudaFreeAsync(ids, s->stream);
  cudaFreeAsync(sc, s->stream);
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (st == AQ_OK && e != cudaSuccess) {
    set_error(AQ_E_CUDA, "CUDA error %s", cudaGetErrorString(e));
    return AQ_E_CUDA;
  }
  return st;
}

// adc_search (index.hpp:118-134) with host arrays: one query.
int aq_adc_search(aq_session* s, const double* q, size_t d, const uint32_t* codes,
                  size_t n, size_t M, size_t codes_k, const double* dict, size_t cbM,
                  size_t k, size_t sd, size_t topn, uint32_t* ids_out,
                  double* scores_out, size_t* count_out) {
  AQ_TRY(check_session(s));
  if (n == 0) return ref_error(AQ_E_EMPTY_INDEX, "no quantized datapoints");
  if (topn < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  if (M != cbM || codes_k > k)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match codebook");
  if (d != cbM * sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "query dimension does not match codebook");
  aq_codebook* cb = nullptr;
  aq_codes* cm = nullptr;
  // the reference does not range-check codes here (index.hpp:121-124); the
  // device packs them with the codebook's k as bound
  AQ_TRY(aq_codebook_upload(s, dict, cbM, k, sd, &cb));
  int st = aq_codes_upload(s, codes, n, M, std::max<size_t>(codes_k, 1), &cm);
  if (st == AQ_OK) st = aq_dev_adc_search(cm, cb, q, 1, topn, ids_out, scores_out);
  if (count_out) *count_out = std::min(topn, n);
  aq_codes_free(cm);
  aq_codebook_free(cb);
  return st;
}

int aq_build_lut(aq_session* s, const double* q, size_t d, const double* dict,
                 size_t M, size_t k, size_t sd, double* lut_out) {
  AQ_TRY(check_session(s));
  if (d != M * sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "query dimension does not match codebook");
  aq_codebook* cb = nullptr;
  AQ_TRY(aq_codebook_upload(s, dict, M, k, sd, &cb));
  double* Qd;
  int st = upload_queries(s, q, 1, d, 0, &Qd);
  void* p = nullptr;
  const size_t lq = (size_t)kLutQP * M * 16 * sizeof(uint32_t);
  if (st == AQ_OK) st = scratch(s, 1, M * k * sizeof(double) + lq + 64, &p);
  if (st == AQ_OK) {
    double* l64 = (double*)p;
    uint16_t* lutq = (uint16_t*)(l64 + M * k);
    k_build_lut<<<1, 256, 0, s->stream>>>(Qd, 1, (int)d, cb->d64, (int)M, (int)k, (int)sd,
                                          l64, lutq, kLutQP, nullptr);
    s->launches++;
    cudaMemcpyAsync(lut_out, l64, M * k * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
    if (cudaStreamSynchronize(s->stream) != cudaSuccess) st = AQ_E_CUDA;
  }
  aq_codebook_free(cb);
  return st;
}

// Exact-dot rerank of host candidate lists.
int aq_dev_rerank(aq_dataset* ds, const double* queries, size_t nq,
                  const uint32_t* cand_ids, size_t ncand, size_t keep,
                  uint32_t* ids_out, double* scores_out) {
  if (!ds) return ref_error(AQ_E_INVALID_ARGUMENT, "null dataset");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t ke = std::min(keep, ncand);
  double* Qd;
  AQ_TRY(upload_queries(s, queries, nq, ds->d, 0, &Qd));
  uint32_t *cand, *ids;
  double* sc;
  AQ_CUDA(cudaMallocAsync(&cand, nq * ncand * sizeof(uint32_t) + 8, s->stream));
  AQ_CUDA(cudaMallocAsync(&ids, nq * ke * sizeof(uint32_t) + 8, s->stream));
  AQ_CUDA(cudaMallocAsync(&sc, nq * ke * sizeof(double) + 8, s->stream));
  AQ_CUDA(cudaMemcpyAsync(cand, cand_ids, nq * ncand * sizeof(uint32_t),
                          cudaMemcpyHostToDevice, s->stream));
  int st = rerank_device(ds, Qd, nq, cand, ncand, keep, ids, sc);
  if (st == AQ_OK) st = sync_and_check(s, "rerank: candidate id out of range");
  if (st == AQ_OK && nq * ke) {
    cudaMemcpyAsync(ids_out, ids, nq * ke * sizeof(uint32_t), cudaMemcpyDeviceToHost, s->stream);
    cudaMemcpyAsync(scores_out, sc, nq * ke * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
  }
  cudaFreeAsync(cand, s->stream);
  cudaFreeAsync(ids, s->stream);
  cudaFreeAsync(sc, s->stream);
  cudaStreamSynchronize(s->stream);
  return st;
}

// Exact dots of candidate ids (device pointers), aligned with the input.
int aq_dev_exact_dots_d(aq_dataset* ds, const double* q_dev, size_t nq,
                        const uint32_t* cand_dev, size_t ncand, double* out_dev) {
  if (!ds) return ref_error(AQ_E_INVALID_ARGUMENT, "null dataset");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t total = nq * ncand;
  if (total == 0) return AQ_OK;
  AQ_XR_LAUNCH(ds, k_exact_dots, (unsigned)((total + 255) / 256), 256, 0, s->stream,
               (int)ds->d, q_dev, nq, cand_dev, ncand, ds->n, out_dev);
  AQ_LAUNCHED(s);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

// Device-pointer pipeline (queries and all outputs on the device).
int aq_dev_search_rerank_d(aq_dataset* ds, aq_codes* codes, aq_codebook* cb,
                           const double* q_dev, size_t nq, size_t topn, size_t keep,
                           uint32_t* adc_ids_dev, double* adc_scores_dev,
                           uint32_t* ids_dev, double* scores_dev) {
  if (!ds || !codes || !cb) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = codes->s;
  AQ_TRY(check_session(s));
  if (ds->n != codes->n)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match dataset");
  const size_t te = std::min(topn, codes->n), ke = std::min(keep, te);
  AQ_TRY(adc_search_device(codes, cb, q_dev, nq, topn, adc_ids_dev, adc_scores_dev));
  AQ_TRY(rerank_device(ds, q_dev, nq, adc_ids_dev, te, ke, ids_dev, scores_dev));
  return sync_and_check(s, "search");
}

// Fused query pipeline: ADC top-`topn` then exact rerank to `keep`, device
// resident index and dataset, host queries in / host results out.
int aq_dev_search_rerank(aq_dataset* ds, aq_codes* codes, aq_codebook* cb,
                         const double* queries, size_t nq, size_t topn, size_t keep,
                         uint32_t* adc_ids_out, double* adc_scores_out,
                         uint32_t* ids_out, double* scores_out) {
  if (!ds || !codes || !cb) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = codes->s;
  AQ_TRY(check_session(s));
  if (codes->n == 0) return ref_error(AQ_E_EMPTY_INDEX, "no quantized datapoints");
  if (topn < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  if (ds->n != codes->n)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match dataset");
  const size_t te = std::min(topn, codes->n), ke = std::min(keep, te);
  double* Qd;
  AQ_TRY(upload_queries(s, queries, nq, ds->d, 0, &Qd));
  void* p;
  AQ_TRY(scratch(s, 5, nq * (te * 12 + ke * 12) + 64, &p));
  uint32_t* aid = (uint32_t*)p;
  double* asc = (double*)(((uintptr_t)(aid + nq * te) + 15) & ~(uintptr_t)15);
  uint32_t* rid = (uint32_t*)(asc + nq * te);
  double* rsc = (double*)(((uintptr_t)(rid + nq * ke) + 15) & ~(uintptr_t)15);
  AQ_TRY(adc_search_device(codes, cb, Qd, nq, topn, aid, asc));
  AQ_TRY(rerank_device(ds, Qd, nq, aid, te, ke, rid, rsc));
  if (adc_ids_out)
    AQ_CUDA(cudaMemcpyAsync(adc_ids_out, aid, nq * te * 4, cudaMemcpyDeviceToHost, s->stream));
  if (adc_scores_out)
    AQ_CUDA(cudaMemcpyAsync(adc_scores_out, asc, nq * te * 8, cudaMemcpyDeviceToHost, s->stream));
  if (ids_out)
    AQ_CUDA(cudaMemcpyAsync(ids_out, rid, nq * ke * 4, cudaMemcpyDeviceToHost, s->stream));
  if (scores_out)
    AQ_CUDA(cudaMemcpyAsync(scores_out, rsc, nq * ke * 8, cudaMemcpyDeviceToHost, s->stream));
  return sync_and_check(s, "search");
}

}  // extern "C"
