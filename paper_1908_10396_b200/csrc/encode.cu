// Anisotropic encode: reconstruction-nearest init + coordinate-descent sweeps
// (pq_quantize, pq.hpp:581-612) and the training assignment pass
// (detail::pq_assign_pass, pq.hpp:202-221), one thread per datapoint.
//
// Bit-exactness strategy. The reference decides every
// code by comparing float64 losses (cd_sweep, pq.hpp:151-185). Evaluating all
// M*k candidates in float64 would run on the half-rate FP64 pipe, so the
// fast kernel (sub_dimension 2, k <= 16) ranks the 16 candidates of a
// subspace with a float32 proxy whose error against the reference's float64
// value is bounded by `delta`:
//     K_j = a_j * (g' a_j - beta') + C_j + off,   a_j = <x_m, c_j>,
//     C_j = |c_j|^2,  g' = (h_par - h_perp) / (h_perp |x|^2),
//     beta' = 2 (g' (base1 + |x_m|^2) + 1),
// which equals (loss_j - const) / h_perp with every constant that is common
// to the 16 candidates dropped. If the runner-up is more than 2*delta above
// the winner the float32 argmin IS the float64 argmin; otherwise every
// candidate inside the window is re-scored in float64 with the reference's
// exact operation order and the lowest index wins ties (pq.hpp:168). Per-point
// state (s2, s1, t2[m], t1[m]) is kept in float64 with the reference's
// operation order, so the resulting codes are bit-identical.
#include "common.cuh"

namespace aqd {

struct EncodeArgs {
  const float2* xt;  // pair-tiled rows
  const double* norms;
  size_t n;
  int d, M, k, pairs;
  const double* cb64;
  const float4* cb32;
  const float* rmax;
  DevWeights w;
  uint8_t* codes;
  size_t stride;
  int bits;
  int mode;         // 0 = pq_quantize, 1 = assign pass, 2 = point losses only
  int passes;       // mode 0
  int sweep_fixed;  // mode 1
  double* losses;   // mode 1/2
  unsigned long long* changed;  // mode 1
  DevError* err;
  size_t base;  // index of point 0 in the caller's numbering (error reports)
};


// Exact float64 scoring of one candidate with the reference's formula.
__device__ __forceinline__ double exact_score2(double x0, double x1, double c0,
                                               double c1, bool iso,
                                               double base2, double base1,
                                               double hp, double ho,
                                               double inv, double* c2,
                                               double* c1o) {
  residual2(x0, x1, c0, c1, c2, c1o);
  return iso ? *c2
             : combined_loss(__dadd_rn(base2, *c2), __dadd_rn(base1, *c1o),
                             hp, ho, inv);
}

// Rare path: re-score in float64 the candidates in `mask` (the float32
// window), ascending j, strict < (pq.hpp:163-174 / 236-243). `nearest`
// selects the reconstruction-nearest score (dist2 only). Out of line so the
// hot loop stays small; returns the winner only.
// pw: this thread's {h_par, h_perp, 1/|x|^2} in shared memory at stride ps
// (kept out of registers across the sweep loop); unused when `nearest`.
__device__ __noinline__ unsigned exact_window(
    float xf0, float xf1, const double2* __restrict__ cbm, unsigned mask,
    bool nearest, double base2, double base1, const double* pw, int ps,
    unsigned long long* stats) {
  if (stats) atomicAdd(stats, 1ull);
  double hp = 0.0, ho = 0.0, inv = 0.0;
  if (!nearest) {
    hp = pw[0];
    ho = pw[ps];
    inv = pw[2 * ps];
  }
  const bool iso = hp == ho;
  const double x0 = xf0, x1 = xf1;
  unsigned jb = 0;
  double bs = 0.0;
  bool first = true;
  while (mask) {
    const int j = __ffs(mask) - 1;
    mask &= mask - 1;
    const double2 cj = cbm[j];
    double c2, c1, sc;
    if (nearest) {
      residual2(x0, x1, cj.x, cj.y, &c2, &c1);
      sc = c2;
    } else {
      sc = exact_score2(x0, x1, cj.x, cj.y, iso, base2, base1, hp, ho, inv,
                        &c2, &c1);
    }
    if (first || sc < bs) {
      first = false;
      bs = sc;
      jb = (unsigned)j;
    }
  }
  return jb;
}

// Staged float32 codebook per subspace: 8 float4 {c0_j, c0_j+1, c1_j, c1_j+1}
// (candidate pairs for the packed f32x2 FMAs), then 4 float4 of C_j = |c_j|^2
// (slots j >= k hold 1e30 so they never enter a window), then 4 float4 of C
// for h_perp == 0 points (0, or 1e30 padding).
constexpr int kCbStride = 16;  // float4 per subspace

// Float32 proxy over the 16 candidates: exact float32 minimum (FMNMX3 tree),
// then the bitmask of candidates within best + 2 delta. A single-bit mask
// proves the float64 argmin; otherwise the mask lists
// every candidate the exact path must re-score.
template <bool kNearest>
__device__ __forceinline__ unsigned proxy_mask(float xf0, float xf1,
                                               const float4* __restrict__ sc,
                                               int coff, float gp, float beta,
                                               float delta) {
  // two candidates per packed FMA (FFMA2): a = x . c, K = a (g' a - beta) + C
  // (kNearest: K = C - 2a); the bound of DESIGN.md §4.1 allows fused products
  float K[16];
  const float2 X0 = make_float2(xf0, xf0), X1 = make_float2(xf1, xf1);
  const float2 GP = make_float2(gp, gp), NB = make_float2(-beta, -beta);
  const float2 M2 = make_float2(-2.0f, -2.0f);
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const float4 c = sc[t];
    const float4 C4 = sc[coff + (t >> 1)];
    const float2 Cp = (t & 1) ? make_float2(C4.z, C4.w) : make_float2(C4.x, C4.y);
    const float2 A = __ffma2_rn(X1, make_float2(c.z, c.w), __fmul2_rn(X0, make_float2(c.x, c.y)));
    float2 Kp;
    if (kNearest) {
      Kp = __ffma2_rn(M2, A, Cp);
    } else {
      Kp = __ffma2_rn(A, __ffma2_rn(GP, A, NB), Cp);
    }
    K[2 * t] = Kp.x;
    K[2 * t + 1] = Kp.y;
  }
  float m6[6];
#pragma unroll
  for (int t = 0; t < 5; ++t)
    m6[t] = fminf(fminf(K[3 * t], K[3 * t + 1]), K[3 * t + 2]);
  m6[5] = K[15];
  const float best = fminf(fminf(fminf(m6[0], m6[1]), m6[2]),
                           fminf(fminf(m6[3], m6[4]), m6[5]));
  const float thr = best + 2.0f * delta + fabsf(best) * 2.384185791015625e-07f;
  if (!(thr < 1e30f) || !(best > -1e30f)) return 0u;  // out of envelope
  // FSETP + predicated OR per candidate, four independent chains (a single
  // chain is 16 dependent adds deep)
  unsigned mk[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 0; j < 16; ++j)
    asm("{\n\t.reg .pred p;\n\tsetp.le.f32 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
        : "+r"(mk[j & 3])
        : "f"(K[j]), "f"(thr), "r"(1u << j));
  return (mk[0] | mk[1]) | (mk[2] | mk[3]);
}

// Fast kernel: sub_dimension == 2, k <= 16, 4-bit codes.
// stats (debug, may be null): [0] exact windows, [1 + s] points that ran s
// sweeps (s = 0..7, mode 0).
template <int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB)
    k_encode_sd2(const EncodeArgs a, unsigned long long* stats) {
  constexpr int kEncThreads = TPB;
  extern __shared__ __align__(16) unsigned char smem[];
  float4* scb = reinterpret_cast<float4*>(smem);                          // [M+1][16]
  double2* cb2 = reinterpret_cast<double2*>(scb + (a.M + 1) * kCbStride);  // [M+1][16]
  float* srm = reinterpret_cast<float*>(cb2 + (a.M + 1) * 16);
  uint32_t* scode = reinterpret_cast<uint32_t*>(srm + a.M);
  // per-thread {h_par, h_perp, inv} for the exact path, [3][TPB] doubles
  double* swt = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(scode + ((a.M + 7) / 8 + 1) * kEncThreads) + 7) &
      ~(uintptr_t)7);
  {
    const double2* g2 = reinterpret_cast<const double2*>(a.cb64);
    for (int t = threadIdx.x; t < a.M * 16; t += blockDim.x) {
      const int m = t >> 4, j = t & 15;
      const float4 v = a.cb32[t];  // {c0, c1, C, 0}; C = 1e30 pads j >= k
      float* row = reinterpret_cast<float*>(scb + m * kCbStride);
      row[(j >> 1) * 4 + (j & 1)] = v.x;
      row[(j >> 1) * 4 + 2 + (j & 1)] = v.y;
      row[32 + j] = v.z;
      row[48 + j] = j < a.k ? 0.0f : 1e30f;
      cb2[t] = j < a.k ? g2[(size_t)m * a.k + j] : make_double2(0.0, 0.0);
    }
  }
  for (int t = threadIdx.x; t < a.M; t += blockDim.x) srm[t] = a.rmax[t];
  for (int t = threadIdx.x; t < 16; t += blockDim.x) cb2[a.M * 16 + t] = make_double2(0.0, 0.0);
  __syncthreads();

  const size_t i = (size_t)blockIdx.x * kEncThreads + threadIdx.x;
  if (i >= a.n) return;
  const int M = a.M;
  const int W = (M + 7) >> 3;
  const unsigned all_mask = (1u << a.k) - 1u;
  uint32_t* mycode = scode + threadIdx.x;  // word w at mycode[w * kEncThreads]
  const float2* xrow = a.xt + (i >> 5) * (size_t)a.pairs * 32 + (i & 31);
  uint8_t* crow = a.codes + i * a.stride;

  double hp, ho;
  int st = AQ_OK;
  if (!resolve_weights(a.w, i, a.norms[i], &hp, &ho, &st)) {
    report_error(a.err, a.base + i, st);
    return;
  }
  const bool iso = hp == ho;
  double inv = 0.0;
  const bool need_inv = a.mode != 0 || a.passes > 0;
  if (!iso) {
    const double n2 = __dmul_rn(a.norms[i], a.norms[i]);
    if (n2 == 0.0) {
      if (need_inv) {
        report_error(a.err, a.base + i, AQ_E_ZERO_NORM_DATAPOINT);
        return;
      }
    } else {
      inv = __ddiv_rn(1.0, n2);
    }
  }
  // proxy constants: loss / h_perp when h_perp > 0; the h_perp == 0 policy
  // points (eta = inf) use loss itself with the |r|^2 term absent (cC = 0)
  const bool zeroC = !iso && !(ho > 0.0);
  float gp = 0.0f;
  if (!iso) {
    const double g = __dmul_rn(__dsub_rn(hp, ho), inv);
    gp = (float)(zeroC ? g : g / ho);
  }
  const float cC = zeroC ? 0.0f : 1.0f;
  const int coff = zeroC ? 12 : 8;
  const bool fast = fabsf(gp) < 1e30f;

  double s2 = 0.0, s1 = 0.0;
  // per-point magnitudes for the error budget (float, over all subspaces):
  // |base1| <= sum_m (X_m + ax_m) = B1, base2 <= sum_m (l1_m + rm_m)^2 = B2
  float B1 = 0.0f, B2 = 0.0f, Amax = 0.0f, Xmax = 0.0f;
  if (a.mode == 0) {
    // reconstruction_nearest_pass + pq_point_state (pq.hpp:594, 603)
    uint32_t cw = 0;
    float2 xv = xrow[0];
    for (int m = 0; m < M; ++m) {
      const float2 xn = xrow[(size_t)(m + 1) * 32];  // padded
      const float rm = srm[m];
      const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
      const float l1 = fabsf(xv.x) + fabsf(xv.y);
      const float ax = l1 * rm;
      B1 += X + ax;
      B2 += (l1 + rm) * (l1 + rm);
      Amax = fmaxf(Amax, ax);
      Xmax = fmaxf(Xmax, X);
      // error budget: < 12u (2 ax + rm^2); 2^-18 = 64u
      const float Wn = 2.0f * ax + rm * rm + X * 9.094947e-13f;
      const float delta = Wn * 3.814697265625e-06f + 1e-30f;
      unsigned mask = Wn < 1e30f ? proxy_mask<true>(xv.x, xv.y, scb + m * kCbStride,
                                                   8, 0.0f, 0.0f, delta)
                                 : 0u;
      unsigned jb;
      if (mask != 0u && (mask & (mask - 1u)) == 0u) {
        jb = (unsigned)(__ffs(mask) - 1);
      } else {
        jb = exact_window(xv.x, xv.y, cb2 + m * 16, mask ? mask : all_mask,
                          true, 0.0, 0.0, nullptr, 0, stats);
      }
      const double2 cj = cb2[m * 16 + jb];
      double t2, t1;
      residual2(xv.x, xv.y, cj.x, cj.y, &t2, &t1);
      s2 = __dadd_rn(s2, t2);
      s1 = __dadd_rn(s1, t1);
      cw |= jb << (4 * (m & 7));
      if ((m & 7) == 7 || m + 1 == M) {
        mycode[(m >> 3) * kEncThreads] = cw;
        cw = 0;
      }
      xv = xn;
    }
  } else {
    const uint32_t* r4 = reinterpret_cast<const uint32_t*>(crow);
    for (int w = 0; w < W; ++w) mycode[w * kEncThreads] = r4[w];
    if (a.mode == 1) {
      // pq_point_state from the current codes (pq.hpp:213)
#pragma unroll 4
      for (int m = 0; m < M; ++m) {
        const float2 xv = xrow[(size_t)m * 32];
        const unsigned c = (mycode[(m >> 3) * kEncThreads] >> (4 * (m & 7))) & 15u;
        const double2 cj = cb2[m * 16 + c];
        double t2, t1;
        residual2(xv.x, xv.y, cj.x, cj.y, &t2, &t1);
        s2 = __dadd_rn(s2, t2);
        s1 = __dadd_rn(s1, t1);
        const float rm = srm[m];
        const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
        const float l1 = fabsf(xv.x) + fabsf(xv.y);
        B1 += X + l1 * rm;
        B2 += (l1 + rm) * (l1 + rm);
        Amax = fmaxf(Amax, l1 * rm);
        Xmax = fmaxf(Xmax, X);
      }
    }
  }

  // Error-budget constants. Per step the proxy's float32
  // error is < 12u W2, W2 = |g'| ax^2 + beta^ ax + cC rm^2 with
  // beta^ = 2(|g'|(|base1| + X) + cC), i.e. W2 = ax (|g'| (ax + 2(|base1| +
  // X)) + 2 cC) + cC rm^2 (computed per step). The reference's own float64
  // rounding is covered by 2^-40 of a per-point magnitude bound (|base1| <=
  // B1 and base2 <= B2 over all steps), hoisted here.
  B1 *= 1.0009765625f;  // slack for the float32 accumulation of the bounds
  B2 *= 1.0009765625f;
  const float agp = fabsf(gp);
  const float AB = Amax + B1 + Xmax;
  const float W2max = Amax * (agp * (Amax + 2.0f * (B1 + Xmax)) + 2.0f) + 4.0f * B2;
  const float dabs = (B2 + Xmax + W2max + agp * AB * AB) * 9.094947e-13f + 1e-30f;
  const bool bounds_ok = dabs < 1e25f;
  const bool fastpt = fast && bounds_ok;
  swt[threadIdx.x] = hp;
  swt[kEncThreads + threadIdx.x] = ho;
  swt[2 * kEncThreads + threadIdx.x] = inv;

  // coordinate-descent sweeps (cd_sweep, pq.hpp:151-185)
  const int max_sweeps = a.mode == 0 ? a.passes : (a.mode == 1 ? 64 : 0);
  int sweeps_run = 0;
  for (int p = 0; p < max_sweeps; ++p) {
    ++sweeps_run;
    bool changed = false;
    uint32_t cw = mycode[0];
    float2 xv = xrow[0];
    unsigned cur = cw & 15u;
    double2 cc = cb2[cur];
    // software pipeline one subspace ahead; the prefetch of subspace M reads
    // padding (row tile, smem codebook and code words are over-allocated)
#pragma unroll 2
    for (int m = 0; m < M; ++m) {
      const int mn = m + 1;
      const uint32_t wnext = ((mn & 7) == 0) ? mycode[(mn >> 3) * kEncThreads] : cw;
      const unsigned curn = (wnext >> (4 * (mn & 7))) & 15u;
      const float2 xn = xrow[(size_t)mn * 32];
      const double2 cn = cb2[mn * 16 + curn];
      double t2, t1;
      residual2(xv.x, xv.y, cc.x, cc.y, &t2, &t1);
      const double base2 = __dsub_rn(s2, t2);
      const double base1 = __dsub_rn(s1, t1);
      const float rm = srm[m];
      const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
      const float ax = (fabsf(xv.x) + fabsf(xv.y)) * rm;
      // isotropic points have gp = agp = 0, cC = 1: beta = 2, W2 = 2 ax + rm^2
      const float b1f = (float)base1;
      const float beta = 2.0f * __fmaf_rn(gp, b1f + X, cC);
      const float W2 = __fmaf_rn(ax, __fmaf_rn(agp, __fmaf_rn(2.0f, fabsf(b1f) + X, ax), 2.0f * cC),
                                 cC * rm * rm);
      const float delta = __fmaf_rn(W2, 3.814697265625e-06f, dabs);  // 2^-18 W2 + abs
      // proxy_mask returns 0 (exact path) for non-finite windows
      const unsigned mask =
          fastpt ? proxy_mask<false>(xv.x, xv.y, scb + m * kCbStride, coff, gp, beta, delta)
                 : 0u;
      unsigned jb;
      if (mask != 0u && (mask & (mask - 1u)) == 0u) {
        jb = (unsigned)(__ffs(mask) - 1);
      } else {
        jb = exact_window(xv.x, xv.y, cb2 + m * 16, mask ? mask : all_mask,
                          false, base2, base1, swt + threadIdx.x, kEncThreads, stats);
      }
      double b2 = t2, b1 = t1;
      if (jb != cur) {
        const double2 cj = cb2[m * 16 + jb];
        residual2(xv.x, xv.y, cj.x, cj.y, &b2, &b1);
        changed = true;
        cw = (cw & ~(15u << (4 * (m & 7)))) | (jb << (4 * (m & 7)));
      }
      s2 = __dadd_rn(base2, b2);
      s1 = __dadd_rn(base1, b1);
      if ((mn & 7) == 0) {
        mycode[(m >> 3) * kEncThreads] = cw;
        cw = wnext;
      }
      xv = xn;
      cc = cn;
      cur = curn;
    }
    if (M & 7) mycode[((M - 1) >> 3) * kEncThreads] = cw;
    if (a.mode == 0) {
      if (!changed) break;  // pq.hpp:605-606
    } else {
      // pq.hpp:215-216: repeat only when sweeping to a fixed point
      if (!(changed && a.sweep_fixed && p + 1 < 64)) break;
    }
  }
  if (stats && a.mode == 0) atomicAdd(stats + 1 + min(sweeps_run, 7), 1ull);

  if (a.mode >= 1) {
    const volatile double* vw = swt + threadIdx.x;
    const double hp = vw[0], ho = vw[kEncThreads], inv = vw[2 * kEncThreads];
    const bool iso = hp == ho;
    // pq_point_loss (pq.hpp:137-146): state recomputed from scratch
    double r2 = 0.0, r1 = 0.0;
    unsigned long long nchg = 0;
    for (int w = 0; w < W; ++w) {
      const uint32_t cw = mycode[w * kEncThreads];
      const uint32_t old = reinterpret_cast<const uint32_t*>(crow)[w];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int m = w * 8 + q;
        if (m < M) {
          const float2 xv = xrow[(size_t)m * 32];
          const unsigned c = (cw >> (4 * q)) & 15u;
          nchg += c != ((old >> (4 * q)) & 15u);
          const double2 cj = cb2[m * 16 + c];
          double t2, t1;
          residual2(xv.x, xv.y, cj.x, cj.y, &t2, &t1);
          r2 = __dadd_rn(r2, t2);
          r1 = __dadd_rn(r1, t1);
        }
      }
    }
    double loss;
    if (iso) {
      loss = __dmul_rn(ho, r2);
    } else {
      loss = combined_loss(r2, r1, hp, ho, inv);
      loss = loss > 0.0 ? loss : 0.0;
    }
    if (a.losses) a.losses[i] = loss;
    if (a.changed) {  // one atomic per warp
      const unsigned act = __activemask();
      const unsigned tot = __reduce_add_sync(act, (unsigned)nchg);
      if (tot && (int)(threadIdx.x & 31) == __ffs(act) - 1)
        atomicAdd(a.changed, (unsigned long long)tot);
    }
  }
  if (a.mode <= 1) {
    // rows are 8-byte aligned with stride a multiple of 8 (code_stride)
    uint2* r8 = reinterpret_cast<uint2*>(crow);
    for (int w = 0; w < (int)(a.stride >> 3); ++w) {
      const uint32_t lo = 2 * w < W ? mycode[(2 * w) * kEncThreads] : 0u;
      const uint32_t hi = 2 * w + 1 < W ? mycode[(2 * w + 1) * kEncThreads] : 0u;
      r8[w] = make_uint2(lo, hi);
    }
  }
}

// ---- word-unrolled fast kernel ---------------------------------------------
//
// Same decisions as k_encode_sd2 (float32 proxy, window, float64 re-score of
// windows with more than one candidate), fewer instructions per subspace:
//  * window mask: the 16 differences K_j - thr are formed two per FADD2 and
//    each sign bit is shifted into one of four chains by a funnel shift (one
//    SHF per candidate instead of FSETP + predicated add);
//  * error budget: h_perp = 0 points use the cC = 1 budget (an upper bound),
//    one expression for every point;
//  * the subspace loop is unrolled over the 8 codes of a packed word: code
//    extraction and insertion (funnel shift right) have constant shifts;
//  * point rows are prefetched two subspaces ahead (the tile buffer carries
//    four pair tiles of padding).

// Proxy keys K_j = a_j (g' a_j - beta') + C_j (kNearest: C_j - 2 a_j), two
// candidates per packed FMA; nbeta = -beta'.
template <bool kNearest>
__device__ __forceinline__ void proxy_keys(float xf0, float xf1,
                                           const float4* __restrict__ sc,
                                           int coff, float gp, float nbeta,
                                           float (&K)[16]) {
  const float2 X0 = make_float2(xf0, xf0), X1 = make_float2(xf1, xf1);
  const float2 GP = make_float2(gp, gp), NB = make_float2(nbeta, nbeta);
  const float2 M2 = make_float2(-2.0f, -2.0f);
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const float4 c = sc[t];
    const float4 C4 = sc[coff + (t >> 1)];
    const float2 Cp = (t & 1) ? make_float2(C4.z, C4.w) : make_float2(C4.x, C4.y);
    const float2 A = __ffma2_rn(X1, make_float2(c.z, c.w), __fmul2_rn(X0, make_float2(c.x, c.y)));
    const float2 Kp = kNearest ? __ffma2_rn(M2, A, Cp)
                               : __ffma2_rn(A, __ffma2_rn(GP, A, NB), Cp);
    K[2 * t] = Kp.x;
    K[2 * t + 1] = Kp.y;
  }
}

// Window of K: thr = best + |best| 2^-22 + dpad (dpad = 2 delta); bit 15 - j of
// the result is set iff K_j < thr (the sign bit of K_j - thr). NaN dpad gives
// a NaN thr, which fails the caller's envelope test.
__device__ __forceinline__ unsigned window_mask(const float (&K)[16], float dpad,
                                                float* best_out, float* thr_out) {
  float m6[6];
#pragma unroll
  for (int t = 0; t < 5; ++t)
    m6[t] = fminf(fminf(K[3 * t], K[3 * t + 1]), K[3 * t + 2]);
  m6[5] = K[15];
  const float best = fminf(fminf(fminf(m6[0], m6[1]), m6[2]),
                           fminf(fminf(m6[3], m6[4]), m6[5]));
  const float thr = __fadd_rn(__fmaf_rn(fabsf(best), 2.384185791015625e-07f, best), dpad);
  const float2 NT = make_float2(-thr, -thr);
  unsigned c[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const float2 D = __fadd2_rn(make_float2(K[2 * t], K[2 * t + 1]), NT);
    c[t >> 1] = __funnelshift_l(__float_as_uint(D.x), c[t >> 1], 1);
    c[t >> 1] = __funnelshift_l(__float_as_uint(D.y), c[t >> 1], 1);
  }
  *best_out = best;
  *thr_out = thr;
  return (((c[0] << 4) | c[1]) << 8) | ((c[2] << 4) | c[3]);
}

// Decision from a window: the single candidate, else the float64 re-score of
// the window (or of all candidates when the proxies left the envelope).
__device__ __forceinline__ unsigned decide(unsigned mask, float best, float thr,
                                           float xf0, float xf1,
                                           const double2* __restrict__ cbm,
                                           unsigned all_mask, bool nearest,
                                           double base2, double base1,
                                           const double* pw, int ps,
                                           unsigned long long* stats) {
  const bool env = thr < 1e30f && best > -1e30f;
  if (env && __popc(mask) == 1) return (unsigned)(__clz(mask) - 16);
  const unsigned wm = (env && mask) ? (__brev(mask) >> 16) : all_mask;
  return exact_window(xf0, xf1, cbm, wm, nearest, base2, base1, pw, ps, stats);
}

struct SweepPoint {
  float gp, ngp2, ncC2, agp, dabs2;
  int coff;
};

// One coordinate-descent step at subspace m (cd_sweep body, pq.hpp:157-183).
template <int TPB>
__device__ __forceinline__ unsigned cd_step(const float2 xv, const unsigned cur, const int m,
                                            const float4* __restrict__ scb,
                                            const double2* __restrict__ cb2,
                                            const float2* __restrict__ srm,
                                            const SweepPoint& P, double& s2,
                                            double& s1, const double* pw,
                                            unsigned all_mask,
                                            unsigned long long* stats) {
  const double2 cc = cb2[m * 16 + cur];
  double t2, t1;
  residual2(xv.x, xv.y, cc.x, cc.y, &t2, &t1);
  const double base2 = __dsub_rn(s2, t2);
  const double base1 = __dsub_rn(s1, t1);
  const float2 rr = srm[m];
  const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
  const float ax = (fabsf(xv.x) + fabsf(xv.y)) * rr.x;
  // W2 >= |g'| ax^2 + beta^ ax + cC rm^2 (budget note in k_encode_sd2)
  const float b1f = (float)base1;
  const float W2 = __fmaf_rn(ax, __fmaf_rn(P.agp, __fmaf_rn(2.0f, fabsf(b1f) + X, ax), 2.0f), rr.y);
  const float dpad = __fmaf_rn(W2, 7.62939453125e-06f, P.dabs2);  // 2 (2^-18 W2 + abs)
  const float nbeta = __fmaf_rn(P.ngp2, b1f + X, P.ncC2);
  float K[16];
  proxy_keys<false>(xv.x, xv.y, scb + m * kCbStride, P.coff, P.gp, nbeta, K);
  float best, thr;
  const unsigned mask = window_mask(K, dpad, &best, &thr);
  const unsigned jb = decide(mask, best, thr, xv.x, xv.y, cb2 + m * 16, all_mask,
                             false, base2, base1, pw, TPB, stats);
  double b2 = t2, b1 = t1;
  if (jb != cur) {
    const double2 cj = cb2[m * 16 + jb];
    residual2(xv.x, xv.y, cj.x, cj.y, &b2, &b1);
  }
  s2 = __dadd_rn(base2, b2);
  s1 = __dadd_rn(base1, b1);
  return jb;
}

// reconstruction_nearest_pass step (pq.hpp:236-243) + pq_point_state terms.
__device__ __forceinline__ unsigned nearest_step(const float2 xv, const int m,
                                                 const float4* __restrict__ scb,
                                                 const double2* __restrict__ cb2,
                                                 const float2 rr, unsigned all_mask,
                                                 double& s2, double& s1,
                                                 unsigned long long* stats) {
  const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
  const float ax = (fabsf(xv.x) + fabsf(xv.y)) * rr.x;
  // error budget: < 12u (2 ax + rm^2); 2^-18 = 64u
  const float Wn = 2.0f * ax + rr.y + X * 9.094947e-13f;
  const float dpad = Wn < 1e30f ? __fmaf_rn(Wn, 7.62939453125e-06f, 2e-30f) : __int_as_float(0x7fffffff);
  float K[16];
  proxy_keys<true>(xv.x, xv.y, scb + m * kCbStride, 8, 0.0f, 0.0f, K);
  float best, thr;
  const unsigned mask = window_mask(K, dpad, &best, &thr);
  const unsigned jb = decide(mask, best, thr, xv.x, xv.y, cb2 + m * 16, all_mask,
                             true, 0.0, 0.0, nullptr, 0, stats);
  const double2 cj = cb2[m * 16 + jb];
  double t2, t1;
  residual2(xv.x, xv.y, cj.x, cj.y, &t2, &t1);
  s2 = __dadd_rn(s2, t2);
  s1 = __dadd_rn(s1, t1);
  return jb;
}

#ifndef AQ_SWEEP_UNROLL
#define AQ_SWEEP_UNROLL 4  // measured: 1 6.99, 2 6.67, 3 7.09, 4 6.55, 8 6.66 ms (4e6 config-3 points)
#endif
constexpr int kSweepUnroll = AQ_SWEEP_UNROLL;  // subspace steps per loop body
#ifndef AQ_NEAREST_UNROLL
#define AQ_NEAREST_UNROLL 2
#endif
constexpr int kNearestUnroll = AQ_NEAREST_UNROLL;
// MT > 0: M known at compile time (every shared-memory offset is a constant);
// MT = 0: any M.
template <int TPB, int MINB, int MT>
__global__ void __launch_bounds__(TPB, MINB)
    k_encode_sd2w(const EncodeArgs a, unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = MT > 0 ? MT : a.M;
  float4* scb = reinterpret_cast<float4*>(smem);                        // [M+1][16]
  double2* cb2 = reinterpret_cast<double2*>(scb + (M + 1) * kCbStride);  // [M+1][16]
  float2* srm = reinterpret_cast<float2*>(cb2 + (M + 1) * 16);          // [M+1] {rm, rm^2}
  uint32_t* scode = reinterpret_cast<uint32_t*>(srm + M + 1);
  double* swt = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(scode + ((M + 7) / 8 + 1) * TPB) + 7) & ~(uintptr_t)7);
  {
    const double2* g2 = reinterpret_cast<const double2*>(a.cb64);
    for (int t = threadIdx.x; t < M * 16; t += blockDim.x) {
      const int m = t >> 4, j = t & 15;
      const float4 v = a.cb32[t];  // {c0, c1, C, 0}; C = 1e30 pads j >= k
      float* row = reinterpret_cast<float*>(scb + m * kCbStride);
      row[(j >> 1) * 4 + (j & 1)] = v.x;
      row[(j >> 1) * 4 + 2 + (j & 1)] = v.y;
      row[32 + j] = v.z;
      row[48 + j] = j < a.k ? 0.0f : 1e30f;
      cb2[t] = j < a.k ? g2[(size_t)m * a.k + j] : make_double2(0.0, 0.0);
    }
  }
  for (int t = threadIdx.x; t <= M; t += blockDim.x) {
    const float r = t < M ? a.rmax[t] : 0.0f;
    srm[t] = make_float2(r, r * r);
  }
  for (int t = threadIdx.x; t < 16; t += blockDim.x) cb2[M * 16 + t] = make_double2(0.0, 0.0);
  __syncthreads();

  const size_t i = (size_t)blockIdx.x * TPB + threadIdx.x;
  if (i >= a.n) return;
  const int W = (M + 7) >> 3;
  const int Wf = M >> 3, Mr = M & 7;
  const unsigned all_mask = (1u << a.k) - 1u;
  uint32_t* mycode = scode + threadIdx.x;  // word w at mycode[w * TPB]
  const float2* xrow = a.xt + (i >> 5) * (size_t)a.pairs * 32 + (i & 31);
  uint8_t* crow = a.codes + i * a.stride;

  double hp, ho;
  int st = AQ_OK;
  if (!resolve_weights(a.w, i, a.norms[i], &hp, &ho, &st)) {
    report_error(a.err, a.base + i, st);
    return;
  }
  const bool iso = hp == ho;
  double inv = 0.0;
  const bool need_inv = a.mode != 0 || a.passes > 0;
  if (!iso) {
    const double n2 = __dmul_rn(a.norms[i], a.norms[i]);
    if (n2 == 0.0) {
      if (need_inv) {
        report_error(a.err, a.base + i, AQ_E_ZERO_NORM_DATAPOINT);
        return;
      }
    } else {
      inv = __ddiv_rn(1.0, n2);
    }
  }
  const bool zeroC = !iso && !(ho > 0.0);
  float gp = 0.0f;
  if (!iso) {
    const double g = __dmul_rn(__dsub_rn(hp, ho), inv);
    gp = (float)(zeroC ? g : g / ho);
  }
  const float cC = zeroC ? 0.0f : 1.0f;
  const bool fast = fabsf(gp) < 1e30f;

  double s2 = 0.0, s1 = 0.0;
  float B1 = 0.0f, B2 = 0.0f, Amax = 0.0f, Xmax = 0.0f;
  if (a.mode == 0) {
    // reconstruction_nearest_pass + pq_point_state (pq.hpp:594, 603)
    float2 xa = xrow[0], xb = xrow[32];
    uint32_t nw = 0;
#pragma unroll kNearestUnroll
    for (int m = 0; m < M; ++m) {
      const float2 xv = xa;
      xa = xb;
      xb = xrow[(size_t)(m + 2) * 32];  // padded
      const float2 rr = srm[m];
      const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
      const float l1 = fabsf(xv.x) + fabsf(xv.y);
      const float ax = l1 * rr.x;
      B1 += X + ax;
      B2 += (l1 + rr.x) * (l1 + rr.x);
      Amax = fmaxf(Amax, ax);
      Xmax = fmaxf(Xmax, X);
      const unsigned jb = nearest_step(xv, m, scb, cb2, rr, all_mask, s2, s1, stats);
      nw = __funnelshift_r(nw, jb, 4);
      if ((m & 7) == 7) mycode[(m >> 3) * TPB] = nw;
    }
    if (Mr) mycode[Wf * TPB] = nw >> ((32 - 4 * Mr) & 31);
  } else {
    const uint32_t* r4 = reinterpret_cast<const uint32_t*>(crow);
    for (int w = 0; w < W; ++w) mycode[w * TPB] = r4[w];
    if (a.mode == 1) {
      // pq_point_state from the current codes (pq.hpp:213)
#pragma unroll 4
      for (int m = 0; m < M; ++m) {
        const float2 xv = xrow[(size_t)m * 32];
        const unsigned c = (mycode[(m >> 3) * TPB] >> (4 * (m & 7))) & 15u;
        const double2 cj = cb2[m * 16 + c];
        double t2, t1;
        residual2(xv.x, xv.y, cj.x, cj.y, &t2, &t1);
        s2 = __dadd_rn(s2, t2);
        s1 = __dadd_rn(s1, t1);
        const float rm = srm[m].x;
        const float X = __fmaf_rn(xv.y, xv.y, xv.x * xv.x);
        const float l1 = fabsf(xv.x) + fabsf(xv.y);
        B1 += X + l1 * rm;
        B2 += (l1 + rm) * (l1 + rm);
        Amax = fmaxf(Amax, l1 * rm);
        Xmax = fmaxf(Xmax, X);
      }
    }
  }

  // error-budget constants (as k_encode_sd2)
  B1 *= 1.0009765625f;
  B2 *= 1.0009765625f;
  const float agp = fabsf(gp);
  const float AB = Amax + B1 + Xmax;
  const float W2max = Amax * (agp * (Amax + 2.0f * (B1 + Xmax)) + 2.0f) + 4.0f * B2;
  const float dabs = (B2 + Xmax + W2max + agp * AB * AB) * 9.094947e-13f + 1e-30f;
  const bool fastpt = fast && dabs < 1e25f;
  SweepPoint P;
  P.gp = gp;
  P.ngp2 = -2.0f * gp;
  P.ncC2 = -2.0f * cC;
  P.agp = agp;
  P.dabs2 = fastpt ? 2.0f * dabs : __int_as_float(0x7fffffff);  // NaN: exact path
  P.coff = zeroC ? 12 : 8;
  swt[threadIdx.x] = hp;
  swt[TPB + threadIdx.x] = ho;
  swt[2 * TPB + threadIdx.x] = inv;
  const double* pw = swt + threadIdx.x;

  // coordinate-descent sweeps (cd_sweep, pq.hpp:151-185)
  const int max_sweeps = a.mode == 0 ? a.passes : (a.mode == 1 ? 64 : 0);
  int sweeps_run = 0;
  for (int p = 0; p < max_sweeps; ++p) {
    ++sweeps_run;
    unsigned chg = 0;
    float2 xa = xrow[0], xb = xrow[32];
    uint32_t cw = mycode[0], nw = 0;
#pragma unroll kSweepUnroll
    for (int m = 0; m < M; ++m) {
      const float2 xv = xa;
      xa = xb;
      xb = xrow[(size_t)(m + 2) * 32];  // padded
      const unsigned cur = cw & 15u;
      cw >>= 4;
      const unsigned jb = cd_step<TPB>(xv, cur, m, scb, cb2, srm, P, s2, s1, pw,
                                       all_mask, stats);
      chg |= jb ^ cur;
      nw = __funnelshift_r(nw, jb, 4);
      if ((m & 7) == 7) {
        mycode[(m >> 3) * TPB] = nw;
        cw = mycode[((m >> 3) + 1) * TPB];  // padded word
      }
    }
    if (Mr) mycode[Wf * TPB] = nw >> ((32 - 4 * Mr) & 31);
    const bool changed = chg != 0;
    if (a.mode == 0) {
      if (!changed) break;  // pq.hpp:605-606
    } else {
      // pq.hpp:215-216: repeat only when sweeping to a fixed point
      if (!(changed && a.sweep_fixed && p + 1 < 64)) break;
    }
  }
  if (stats && a.mode == 0) atomicAdd(stats + 1 + min(sweeps_run, 7), 1ull);

  if (a.mode >= 1) {
    // weights re-read from shared memory (not kept live across the sweeps)
    const volatile double* vw = swt + threadIdx.x;
    const double hp = vw[0], ho = vw[TPB], inv = vw[2 * TPB];
    const bool iso = hp == ho;
    // pq_point_loss (pq.hpp:137-146): state recomputed from scratch
    double r2 = 0.0, r1 = 0.0;
    unsigned long long nchg = 0;
    for (int w = 0; w < W; ++w) {
      const uint32_t cw = mycode[w * TPB];
      const uint32_t old = reinterpret_cast<const uint32_t*>(crow)[w];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int m = w * 8 + q;
        if (m < M) {
          const float2 xv = xrow[(size_t)m * 32];
          const unsigned c = (cw >> (4 * q)) & 15u;
          nchg += c != ((old >> (4 * q)) & 15u);
          const double2 cj = cb2[m * 16 + c];
          double t2, t1;
          residual2(xv.x, xv.y, cj.x, cj.y, &t2, &t1);
          r2 = __dadd_rn(r2, t2);
          r1 = __dadd_rn(r1, t1);
        }
      }
    }
    double loss;
    if (iso) {
      loss = __dmul_rn(ho, r2);
    } else {
      loss = combined_loss(r2, r1, hp, ho, inv);
      loss = loss > 0.0 ? loss : 0.0;
    }
    if (a.losses) a.losses[i] = loss;
    if (a.changed) {  // one atomic per warp
      const unsigned act = __activemask();
      const unsigned tot = __reduce_add_sync(act, (unsigned)nchg);
      if (tot && (int)(threadIdx.x & 31) == __ffs(act) - 1)
        atomicAdd(a.changed, (unsigned long long)tot);
    }
  }
  if (a.mode <= 1) {
    uint2* r8 = reinterpret_cast<uint2*>(crow);
    for (int w = 0; w < (int)(a.stride >> 3); ++w) {
      const uint32_t lo = 2 * w < W ? mycode[(2 * w) * TPB] : 0u;
      const uint32_t hi = 2 * w + 1 < W ? mycode[(2 * w + 1) * TPB] : 0u;
      r8[w] = make_uint2(lo, hi);
    }
  }
}

// ---- generic exact kernel (any sub_dimension, k <= 256) ---------------------

template <class TX>
__device__ __forceinline__ double xval(const TX* __restrict__ xt, size_t i, int j, int pairs) {
  return (double)xt[tiled_index(i, (size_t)j, (size_t)pairs)];
}

// detail::residual_terms for general sd (geometry.hpp:182-192)
template <class TX>
__device__ __forceinline__ void residual_g(const TX* __restrict__ xt,
                                           size_t i, int pairs, int off,
                                           const double* c, int sd,
                                           double* d2, double* rd) {
  double a = 0.0, b = 0.0;
  for (int t = 0; t < sd; ++t) {
    const double xv = xval(xt, i, off + t, pairs);
    const double df = __dsub_rn(xv, c[t]);
    a = __dadd_rn(a, __dmul_rn(df, df));
    b = __dadd_rn(b, __dmul_rn(df, xv));
  }
  *d2 = a;
  *rd = b;
}

__device__ __forceinline__ unsigned gcode(const uint8_t* row, int m, int bits) {
  return get_code(row, m, bits);
}
__device__ __forceinline__ void scode(uint8_t* row, int m, int bits,
                                      unsigned c) {
  if (bits == 4) {
    const int sh = (m & 1) * 4;
    row[m >> 1] = (uint8_t)((row[m >> 1] & ~(15u << sh)) | (c << sh));
  } else {
    row[m] = (uint8_t)c;
  }
}

// Exact float64 mirror of the reference loops; codes are edited in place in
// a per-thread scratch row (global memory) so any M works.
template <class TX>
__global__ void k_encode_generic(const EncodeArgs a, const TX* xt,
                                 int sd, uint8_t* work) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  double hp, ho;
  int st = AQ_OK;
  if (!resolve_weights(a.w, i, a.norms[i], &hp, &ho, &st)) {
    report_error(a.err, a.base + i, st);
    return;
  }
  const bool iso = hp == ho;
  double inv = 0.0;
  const bool need_inv = a.mode != 0 || a.passes > 0;
  if (!iso) {
    const double n2 = __dmul_rn(a.norms[i], a.norms[i]);
    if (n2 == 0.0) {
      if (need_inv) {
        report_error(a.err, a.base + i, AQ_E_ZERO_NORM_DATAPOINT);
        return;
      }
    } else {
      inv = __ddiv_rn(1.0, n2);
    }
  }
  uint8_t* row = work + i * a.stride;
  const uint8_t* orig = a.codes + i * a.stride;
  for (size_t b = 0; b < a.stride; ++b) row[b] = orig[b];
  const int M = a.M, k = a.k, bits = a.bits;
  double s2 = 0.0, s1 = 0.0;
  if (a.mode == 0) {
    for (int m = 0; m < M; ++m) {
      unsigned bj = 0;
      double bd = 0.0;
      for (int j = 0; j < k; ++j) {
        double c2, c1;
        residual_g(xt, i, a.pairs, m * sd, a.cb64 + ((size_t)m * k + j) * sd,
                   sd, &c2, &c1);
        if (j == 0 || c2 < bd) {
          bd = c2;
          bj = (unsigned)j;
        }
      }
      scode(row, m, bits, bj);
    }
  }
  if (a.mode <= 1) {
    for (int m = 0; m < M; ++m) {
      double t2, t1;
      residual_g(xt, i, a.pairs, m * sd,
                 a.cb64 + ((size_t)m * k + gcode(row, m, bits)) * sd, sd, &t2,
                 &t1);
      s2 = __dadd_rn(s2, t2);
      s1 = __dadd_rn(s1, t1);
    }
    const int max_sweeps = a.mode == 0 ? a.passes : 64;
    for (int p = 0; p < max_sweeps; ++p) {
      bool changed = false;
      for (int m = 0; m < M; ++m) {
        const unsigned cur = gcode(row, m, bits);
        double t2, t1;
        residual_g(xt, i, a.pairs, m * sd, a.cb64 + ((size_t)m * k + cur) * sd,
                   sd, &t2, &t1);
        const double base2 = __dsub_rn(s2, t2);
        const double base1 = __dsub_rn(s1, t1);
        unsigned bj = 0;
        double bs = 0.0, b2 = 0.0, b1 = 0.0;
        for (int j = 0; j < k; ++j) {
          double c2, c1;
          residual_g(xt, i, a.pairs, m * sd,
                     a.cb64 + ((size_t)m * k + j) * sd, sd, &c2, &c1);
          const double sc =
              iso ? c2
                  : combined_loss(__dadd_rn(base2, c2), __dadd_rn(base1, c1),
                                  hp, ho, inv);
          if (j == 0 || sc < bs) {
            bs = sc;
            bj = (unsigned)j;
            b2 = c2;
            b1 = c1;
          }
        }
        if (bj != cur) {
          scode(row, m, bits, bj);
          changed = true;
        }
        s2 = __dadd_rn(base2, b2);
        s1 = __dadd_rn(base1, b1);
      }
      if (a.mode == 0) {
        if (!changed) break;
      } else if (!(changed && a.sweep_fixed && p + 1 < 64)) {
        break;
      }
    }
  }
  if (a.mode >= 1) {
    double r2 = 0.0, r1 = 0.0;
    unsigned long long nchg = 0;
    for (int m = 0; m < M; ++m) {
      const unsigned c = gcode(row, m, bits);
      nchg += c != gcode(orig, m, bits);
      double t2, t1;
      residual_g(xt, i, a.pairs, m * sd, a.cb64 + ((size_t)m * k + c) * sd, sd,
                 &t2, &t1);
      r2 = __dadd_rn(r2, t2);
      r1 = __dadd_rn(r1, t1);
    }
    double loss;
    if (iso) {
      loss = __dmul_rn(ho, r2);
    } else {
      loss = combined_loss(r2, r1, hp, ho, inv);
      loss = loss > 0.0 ? loss : 0.0;
    }
    if (a.losses) a.losses[i] = loss;
    if (a.changed) {  // one atomic per warp
      const unsigned act = __activemask();
      const unsigned tot = __reduce_add_sync(act, (unsigned)nchg);
      if (tot && (int)(threadIdx.x & 31) == __ffs(act) - 1)
        atomicAdd(a.changed, (unsigned long long)tot);
    }
  }
}

__global__ void k_copy_rows(const uint8_t* src, uint8_t* dst, size_t bytes) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < bytes) dst[t] = src[t];
}

// Runs one encode flavour over a dataset. codes: in/out (modes 0, 1) or in (2).
unsigned long long* g_stats = nullptr;  // debug: exact-window count

static int run_encode_impl(aq_dataset* ds, aq_codebook* cb, const aq_weights* w,
                           aq_codes* codes, int mode, int passes, int sweep_fixed,
                           double* losses_dev, uint64_t* changed_out, size_t base,
                           bool async) {
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  if (ds->d != cb->M * cb->sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH,
                     "dataset dimension does not match codebook");
  if (passes < 0) return ref_error(AQ_E_INVALID_ARGUMENT, "passes must be >= 0");
  if (codes->n != ds->n || codes->M != cb->M)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match dataset");
  if (cb->k > 256) return ref_error(AQ_E_UNSUPPORTED, "device encode supports k <= 256");
  if (cb->k == 0) return ref_error(AQ_E_INVALID_ARGUMENT, "empty codebook");
  if (ds->n == 0) {
    if (changed_out) *changed_out = 0;
    return AQ_OK;
  }
  EncodeArgs a{};
  a.xt = reinterpret_cast<const float2*>(ds->xt);
  a.norms = ds->norms;
  a.n = ds->n;
  a.d = (int)ds->d;
  a.M = (int)cb->M;
  a.k = (int)cb->k;
  a.pairs = (int)pairs_of(ds->d);
  a.cb64 = cb->d64;
  a.cb32 = cb->f32;
  a.rmax = cb->rmax;
  AQ_TRY(make_dev_weights(s, w, ds->n, ds->d, &a.w));
  a.codes = codes->data;
  a.stride = codes->stride;
  a.bits = codes->bits;
  a.mode = mode;
  a.passes = passes;
  a.sweep_fixed = sweep_fixed;
  a.losses = losses_dev;
  a.err = s->err;
  a.base = base;
  unsigned long long* dchg = nullptr;
  if (mode == 1) {
    void* p;
    AQ_TRY(scratch(s, 4, 64, &p));
    dchg = (unsigned long long*)p;
    AQ_CUDA(cudaMemsetAsync(dchg, 0, 8, s->stream));
  }
  a.changed = dchg;
  if (!async) AQ_TRY(clear_dev_error(s));
  const bool fast = cb->sd == 2 && cb->k <= 16 && codes->bits == 4 && !ds->f64;
  if (fast) {
    const int W = (a.M + 7) / 8;
    // 256 threads, 3 CTAs/SM (24 warps at 80 registers), measured best for
    // both kernels; AQ_ENC_VARIANT=1 forces the previous kernel for every M
    int variant = 11;
    if (const char* v = getenv("AQ_ENC_VARIANT")) variant = atoi(v);
    const int tpb = 256;
    const size_t smv = (size_t)(a.M + 1) * (kCbStride * sizeof(float4) + 16 * sizeof(double2)) +
                       (a.M + 1) * sizeof(float2) + (size_t)(W + 1) * tpb * sizeof(uint32_t) + 16 +
                       3 * tpb * sizeof(double) + 8;
    const unsigned grid = (unsigned)((ds->n + tpb - 1) / tpb);
    if (smv > 200 * 1024) return ref_error(AQ_E_UNSUPPORTED, "M too large for the fast encoder");
    timer_mark(s, AQ_T_ENCODE);
#define AQ_ENC_LAUNCH(T, B)                                                              \
  do {                                                                                  \
    AQ_CUDA(cudaFuncSetAttribute(k_encode_sd2<T, B>,                                    \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
    k_encode_sd2<T, B><<<grid, T, smv, s->stream>>>(a, g_stats);                        \
  } while (0)
#define AQ_ENCW_LAUNCH(T, B, MT)                                                         \
  do {                                                                                  \
    AQ_CUDA(cudaFuncSetAttribute(k_encode_sd2w<T, B, MT>,                               \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
    k_encode_sd2w<T, B, MT><<<grid, T, smv, s->stream>>>(a, g_stats);                   \
  } while (0)
    if (variant == 11) {
      // M-specialised instances for the common shapes; other M run the
      // previous kernel (faster than the runtime-M instance of this one)
      switch (a.M) {
        case 16: AQ_ENCW_LAUNCH(256, 3, 16); break;
        case 32: AQ_ENCW_LAUNCH(256, 3, 32); break;
        case 48: AQ_ENCW_LAUNCH(256, 3, 48); break;
        case 50: AQ_ENCW_LAUNCH(256, 3, 50); break;
        case 64: AQ_ENCW_LAUNCH(256, 3, 64); break;
        case 96: AQ_ENCW_LAUNCH(256, 3, 96); break;
        case 128: AQ_ENCW_LAUNCH(256, 3, 128); break;
        default: AQ_ENC_LAUNCH(256, 3); break;
      }
    } else {
      AQ_ENC_LAUNCH(256, 3);
    }
#undef AQ_ENC_LAUNCH
#undef AQ_ENCW_LAUNCH
    AQ_LAUNCHED(s);
    timer_mark(s, AQ_T_ENCODE);
  } else {
    void* work;
    AQ_TRY(scratch(s, 3, ds->n * codes->stride + 16, &work));
    const unsigned grid = (unsigned)((ds->n + 127) / 128);
    if (ds->f64)
      k_encode_generic<double><<<grid, 128, 0, s->stream>>>(a, ds->xt64, (int)cb->sd,
                                                            (uint8_t*)work);
    else
      k_encode_generic<float><<<grid, 128, 0, s->stream>>>(a, ds->xt, (int)cb->sd,
                                                           (uint8_t*)work);
    AQ_LAUNCHED(s);
    if (mode <= 1) {
      const size_t bytes = ds->n * codes->stride;
      k_copy_rows<<<(unsigned)((bytes + 255) / 256), 256, 0, s->stream>>>(
          (const uint8_t*)work, codes->data, bytes);
      AQ_LAUNCHED(s);
    }
  }
  if (changed_out && dchg) {
    unsigned long long h = 0;
    AQ_CUDA(cudaMemcpyAsync(&h, dchg, 8, cudaMemcpyDeviceToHost, s->stream));
    AQ_TRY(sync_and_check(s, "encode"));
    *changed_out = h;
    return AQ_OK;
  }
  return async ? AQ_OK : sync_and_check(s, "encode");
}

int run_encode(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes, int mode,
               int passes, int sweep_fixed, double* losses_dev, uint64_t* changed_out) {
  return run_encode_impl(ds, cb, w, codes, mode, passes, sweep_fixed, losses_dev, changed_out, 0,
                         false);
}

// pq_quantize of one chunk of a larger host dataset (aq_pq_quantize's
// streamed path): no error reset, no synchronisation; device errors carry
// base + i and are checked once after the last chunk.
int run_encode_chunk(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes,
                     int passes, size_t base) {
  return run_encode_impl(ds, cb, w, codes, 0, passes, 0, nullptr, nullptr, base, true);
}

}  // namespace aqd

using namespace aqd;

extern "C" {

int aq_dev_pq_quantize(aq_dataset* ds, aq_codebook* cb, const aq_weights* w,
                       int passes, aq_codes* out) {
  if (!ds || !cb || !out) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  return run_encode(ds, cb, w, out, 0, passes, 0, nullptr, nullptr);
}

int aq_dev_pq_assign_pass(aq_dataset* ds, aq_codebook* cb, const aq_weights* w,
                          int sweep_to_fixed_point, aq_codes* codes,
                          double* losses_dev, uint64_t* changed) {
  if (!ds || !cb || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  return run_encode(ds, cb, w, codes, 1, 0, sweep_to_fixed_point, losses_dev,
                    changed);
}

}  // extern "C"

extern "C" {
// Debug/evidence hook: counts exact-window re-scorings in the fast encoder
// (how often the float32 filter could not decide alone). enable=1 allocates
// and zeroes the counters, enable=0 reads them back (count[0] = exact
// windows, count[1+s] = points that ran s sweeps) and disables counting.
int aq_debug_exact_window_count(aq_session* s, int enable, uint64_t* count) {
  AQ_TRY(check_session(s));
  if (enable) {
    if (!g_stats) AQ_CUDA(cudaMalloc(&g_stats, 9 * 8));
    AQ_CUDA(cudaMemsetAsync(g_stats, 0, 9 * 8, s->stream));
    AQ_CUDA(cudaStreamSynchronize(s->stream));
    return AQ_OK;
  }
  unsigned long long h[9] = {0};
  if (g_stats) {
    AQ_CUDA(cudaMemcpyAsync(h, g_stats, 9 * 8, cudaMemcpyDeviceToHost, s->stream));
    AQ_CUDA(cudaStreamSynchronize(s->stream));
    cudaFree(g_stats);
    g_stats = nullptr;
  }
  if (count)
    for (int t = 0; t < 9; ++t) count[t] = h[t];
  return AQ_OK;
}
}
