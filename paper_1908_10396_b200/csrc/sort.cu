// Stable LSD radix sort of (float64 score, uint32 index) pairs into the
// reference's result order: score descending, index ascending
// (select_top, index.hpp:88-112; loss_ranking, vq.hpp:221-229). Used by the
// exact fallback of ADC search (ties / large top-N) and by codebook reseeding.
// Deterministic: no floating-point arithmetic, stable scatter.
#include "common.cuh"

namespace aqd {

constexpr int kSortBlock = 1024;  // items per block
constexpr int kSortThreads = 256;

// ascending order of the returned key == descending float64 order
__device__ __forceinline__ unsigned long long desc_key(double s) {
  unsigned long long b = (unsigned long long)__double_as_longlong(s);
  b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending transform
  return ~b;
}

__global__ void k_make_keys(const double* __restrict__ s, size_t n,
                            unsigned long long* __restrict__ keys) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) keys[t] = desc_key(s[t]);
}

__global__ void k_radix_hist(const unsigned long long* __restrict__ keys,
                             size_t n, int shift, unsigned* __restrict__ hist,
                             size_t nblocks) {
  __shared__ unsigned h[256];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) h[t] = 0;
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * kSortBlock;
  for (int t = threadIdx.x; t < kSortBlock; t += blockDim.x) {
    const size_t i = base + t;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    hist[(size_t)t * nblocks + blockIdx.x] = h[t];
}

// exclusive scan of hist (digit-major), single CTA
// In-place exclusive scan of hist[lo, hi) starting from `carry0`, by one CTA
// (chunks of blockDim in order, carried across chunks).
__device__ void cta_exclusive_scan(unsigned* __restrict__ hist, size_t lo, size_t hi,
                                   unsigned long long carry0) {
  __shared__ unsigned long long carry;
  __shared__ unsigned warp_sums[32];
  if (threadIdx.x == 0) carry = carry0;
  __syncthreads();
  for (size_t base = lo; base < hi; base += blockDim.x) {
    const size_t i = base + threadIdx.x;
    const unsigned v = i < hi ? hist[i] : 0u;
    // block inclusive scan
    unsigned x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned ws = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      warp_sums[lane] = ws;
    }
    __syncthreads();
    const unsigned prefix = w ? warp_sums[w - 1] : 0u;
    const unsigned long long c = carry;
    if (i < hi) hist[i] = (unsigned)(c + prefix + x - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c + prefix + x;
    __syncthreads();
  }
}

__global__ void k_radix_scan(unsigned* __restrict__ hist, size_t total) {
  cta_exclusive_scan(hist, 0, total, 0ull);
}

// multi-CTA scan: tile sums -> scan of the sums -> per-tile rescan
constexpr size_t kScanTile = 16384;
__global__ void k_scan_tile_sums(const unsigned* __restrict__ hist, size_t total,
                                 unsigned* __restrict__ sums) {
  const size_t lo = (size_t)blockIdx.x * kScanTile, hi = min(total, lo + kScanTile);
  unsigned long long acc = 0;
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += hist[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ unsigned long long ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    sums[blockIdx.x] = (unsigned)t;
  }
}
__global__ void k_scan_tiles(unsigned* __restrict__ hist, size_t total,
                             const unsigned* __restrict__ offs) {
  const size_t lo = (size_t)blockIdx.x * kScanTile, hi = min(total, lo + kScanTile);
  cta_exclusive_scan(hist, lo, hi, offs[blockIdx.x]);
}

// stable scatter: items of a block are ranked in order
__global__ void k_radix_scatter(const unsigned long long* __restrict__ kin,
                                const uint32_t* __restrict__ vin, size_t n,
                                int shift, const unsigned* __restrict__ hist,
                                size_t nblocks,
                                unsigned long long* __restrict__ kout,
                                uint32_t* __restrict__ vout) {
  __shared__ unsigned run[256];      // running count per digit in this block
  __shared__ unsigned wcnt[8][256];  // per-warp digit counts of a round
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    run[t] = hist[(size_t)t * nblocks + blockIdx.x];
  const size_t base = (size_t)blockIdx.x * kSortBlock;
  for (int round = 0; round < kSortBlock / kSortThreads; ++round) {
    for (int t = threadIdx.x; t < 8 * 256; t += blockDim.x)
      (&wcnt[0][0])[t] = 0;
    __syncthreads();
    const size_t i = base + (size_t)round * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    const unsigned long long key = valid ? kin[i] : 0ull;
    const unsigned dg = valid ? (unsigned)((key >> shift) & 255) : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const unsigned rank_in_warp = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank_in_warp == 0) wcnt[w][dg] = __popc(peers);
    __syncthreads();
    if (valid) {
      unsigned before = 0;
      for (int ww = 0; ww < w; ++ww) before += wcnt[ww][dg];
      const unsigned pos = run[dg] + before + rank_in_warp;
      kout[pos] = key;
      vout[pos] = vin[i];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 256; t += blockDim.x) {
      unsigned s = 0;
      for (int ww = 0; ww < 8; ++ww) s += wcnt[ww][t];
      run[t] += s;
    }
    __syncthreads();
  }
}

// Sorts idx (initially any order) by (score desc, index asc). scores is
// indexed by position i (scores[i] belongs to idx[i]). Caller must have idx in
// ascending index order for the index tie-break (stable sort).
// Exclusive scan of `total` counts in place (sums fit in 32 bits).
int scan_device(aq_session* s, unsigned* hist, size_t total) {
  if (total <= 4 * kScanTile) {
    k_radix_scan<<<1, 1024, 0, s->stream>>>(hist, total);
    AQ_LAUNCHED(s);
    return AQ_OK;
  }
  const size_t tiles = (total + kScanTile - 1) / kScanTile;
  void* p;
  AQ_TRY(scratch(s, 6, tiles * sizeof(unsigned) + 64, &p));
  unsigned* sums = (unsigned*)p;
  k_scan_tile_sums<<<(unsigned)tiles, 512, 0, s->stream>>>(hist, total, sums);
  AQ_LAUNCHED(s);
  k_radix_scan<<<1, 1024, 0, s->stream>>>(sums, tiles);
  AQ_LAUNCHED(s);
  k_scan_tiles<<<(unsigned)tiles, 512, 0, s->stream>>>(hist, total, sums);
  AQ_LAUNCHED(s);
  return AQ_OK;
}

int sort_scores_desc(aq_session* s, const double* scores, uint32_t* idx,
                     size_t n) {
  if (n <= 1) return AQ_OK;
  const size_t nb = (n + kSortBlock - 1) / kSortBlock;
  void* p;
  const size_t kbytes = n * sizeof(unsigned long long);
  AQ_TRY(scratch(s, 2, 2 * kbytes + n * sizeof(uint32_t) + 256 * nb * sizeof(unsigned) + 64, &p));
  unsigned long long* k0 = (unsigned long long*)p;
  unsigned long long* k1 = k0 + n;
  uint32_t* v1 = (uint32_t*)(k1 + n);
  unsigned* hist = (unsigned*)(v1 + n);
  k_make_keys<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(scores, n, k0);
  AQ_LAUNCHED(s);
  unsigned long long* kin = k0;
  unsigned long long* kout = k1;
  uint32_t* vin = idx;
  uint32_t* vout = v1;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = pass * 8;
    k_radix_hist<<<(unsigned)nb, kSortThreads, 0, s->stream>>>(kin, n, shift, hist, nb);
    AQ_LAUNCHED(s);
    AQ_TRY(scan_device(s, hist, 256 * nb));
    k_radix_scatter<<<(unsigned)nb, kSortThreads, 0, s->stream>>>(
        kin, vin, n, shift, hist, nb, kout, vout);
    AQ_LAUNCHED(s);
    std::swap(kin, kout);
    std::swap(vin, vout);
  }
  // 8 passes: results are back in k0 / idx
  return AQ_OK;
}

}  // namespace aqd
