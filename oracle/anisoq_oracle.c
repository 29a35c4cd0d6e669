/* oracle/anisoq_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * Plain-C, float64, single-threaded restatement of the reference hot path
 * (/root/reference/proj/include/anisoq). Every function cites the reference
 * lines it follows; operation order is kept literally (compiled with
 * -ffp-contract=off, like proj/CMakeLists.txt:11-13) so results are
 * bit-identical to the reference, which tests/test_oracle.py checks against
 * oracle/_ref (the reference compiled in place) and the reference tests'
 * worked examples.
 *
 * Never linked into, loaded by, or called from the product path.
 */
#include "anisoq_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/anisoq_b200.h"

static __thread char g_err[512];

const char* orc_last_error(void) { return g_err; }

static int fail(int code, const char* name, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s: %s", name, msg);
  return code;
}
#define E_INVALID(m) fail(AQ_E_INVALID_ARGUMENT, "InvalidArgument", m)
#define E_ZERONORM(m) fail(AQ_E_ZERO_NORM_DATAPOINT, "ZeroNormDatapoint", m)
#define E_THRESH(m) fail(AQ_E_INVALID_THRESHOLD, "InvalidThreshold", m)
#define E_EMPTY(m) fail(AQ_E_EMPTY_DATASET, "EmptyDataset", m)
#define E_EMPTYIDX(m) fail(AQ_E_EMPTY_INDEX, "EmptyIndex", m)
#define E_DIM(m) fail(AQ_E_DIMENSION_MISMATCH, "DimensionMismatch", m)
#define E_DIV(m) fail(AQ_E_DIMENSION_NOT_DIVISIBLE, "DimensionNotDivisible", m)
#define E_CODE(m) fail(AQ_E_CODE_OUT_OF_RANGE, "CodeOutOfRange", m)
#define E_SING(m) fail(AQ_E_SINGULAR_SYSTEM, "SingularSystem", m)

/* ---- geometry.hpp -------------------------------------------------------- */

/* detail::residual_terms, geometry.hpp:182-192 */
static void residual_terms(const double* x, const double* c, size_t sd,
                           double* dist2, double* rdot) {
  double d2 = 0.0, rd = 0.0;
  for (size_t j = 0; j < sd; ++j) {
    const double diff = x[j] - c[j];
    d2 += diff * diff;
    rd += diff * x[j];
  }
  *dist2 = d2;
  *rdot = rd;
}

/* detail::combined_loss, geometry.hpp:196-200 */
static double combined_loss(double dist2, double rdot, double hp, double ho,
                            double inv_norm2) {
  return ho * dist2 + (hp - ho) * (rdot * rdot) * inv_norm2;
}

/* detail::dot, geometry.hpp:170-174 */
static double dot(const double* a, const double* b, size_t n) {
  double s = 0.0;
  for (size_t j = 0; j < n; ++j) s += a[j] * b[j];
  return s;
}

/* detail::row_norm, dataset.hpp:55-59 */
void orc_row_norms(const double* x, size_t n, size_t d, double* norms) {
  for (size_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < d; ++j) s += x[i * d + j] * x[i * d + j];
    norms[i] = sqrt(s);
  }
}

/* eta_limit, geometry.hpp:395-402 */
int orc_eta_limit(double t, double norm, int d, double* out) {
  if (!(norm > 0.0)) return E_INVALID("norm must be positive");
  if (!(t >= 0.0) || t >= norm) return E_THRESH("need 0 <= T < norm");
  if (d < 2) return E_INVALID("eta_limit needs d >= 2");
  const double rho = (t / norm) * (t / norm);
  *out = (double)(d - 1) * rho / (1.0 - rho);
  return AQ_OK;
}

/* resolve_weights (anisoq_main.cpp:127-133): h_par = eta, h_perp = 1
 * (AnisotropicWeights::from_eta, geometry.hpp:139-142). */
int orc_threshold_weights(const double* norms, size_t n, size_t d, double t,
                          int policy, double* hp, double* ho) {
  for (size_t i = 0; i < n; ++i) {
    if (policy == AQ_THRESHOLD_PARALLEL_ONLY && norms[i] > 0.0 &&
        t >= norms[i] && t >= 0.0) {
      hp[i] = 1.0; /* eta = inf: parallel error only */
      ho[i] = 0.0;
      continue;
    }
    double eta;
    const int st = orc_eta_limit(t, norms[i], (int)d, &eta);
    if (st) return st;
    hp[i] = eta;
    ho[i] = 1.0;
  }
  return AQ_OK;
}

static int is_iso(double hp, double ho) { return hp == ho; } /* geometry.hpp:124 */

/* ---- pq.hpp: encode -------------------------------------------------------- */

typedef struct {
  double* t2;
  double* t1;
  double s2, s1;
} pq_state;

/* detail::pq_point_state, pq.hpp:122-135 */
static void pq_point_state(const double* x, const uint32_t* row,
                           const double* dict, size_t M, size_t k, size_t sd,
                           pq_state* st) {
  st->s2 = 0.0;
  st->s1 = 0.0;
  for (size_t m = 0; m < M; ++m) {
    residual_terms(x + m * sd, dict + (m * k + row[m]) * sd, sd, &st->t2[m],
                   &st->t1[m]);
    st->s2 += st->t2[m];
    st->s1 += st->t1[m];
  }
}

/* detail::pq_point_loss, pq.hpp:137-146 */
static double pq_point_loss(const double* x, const uint32_t* row,
                            const double* dict, size_t M, size_t k, size_t sd,
                            double hp, double ho, double inv_norm2,
                            pq_state* st) {
  pq_point_state(x, row, dict, M, k, sd, st);
  if (is_iso(hp, ho)) return ho * st->s2;
  const double loss = combined_loss(st->s2, st->s1, hp, ho, inv_norm2);
  return loss > 0.0 ? loss : 0.0;
}

/* detail::cd_sweep, pq.hpp:151-185 (default sweep order 0..M-1, 196-200) */
static int cd_sweep(const double* x, uint32_t* codes, const double* dict,
                    size_t M, size_t k, size_t sd, double hp, double ho,
                    double inv_norm2, pq_state* st) {
  const int iso = is_iso(hp, ho);
  int changed = 0;
  for (size_t m = 0; m < M; ++m) {
    const double* xs = x + m * sd;
    const double base2 = st->s2 - st->t2[m];
    const double base1 = st->s1 - st->t1[m];
    size_t best_j = 0;
    double best_score = 0.0, best2 = 0.0, best1 = 0.0;
    for (size_t j = 0; j < k; ++j) {
      double c2, c1;
      residual_terms(xs, dict + (m * k + j) * sd, sd, &c2, &c1);
      const double score =
          iso ? c2 : combined_loss(base2 + c2, base1 + c1, hp, ho, inv_norm2);
      if (j == 0 || score < best_score) {
        best_score = score;
        best_j = j;
        best2 = c2;
        best1 = c1;
      }
    }
    if (best_j != codes[m]) {
      codes[m] = (uint32_t)best_j;
      changed = 1;
    }
    st->t2[m] = best2;
    st->t1[m] = best1;
    st->s2 = base2 + best2;
    st->s1 = base1 + best1;
  }
  return changed;
}

/* detail::point_inv_norm2, pq.hpp:187-194 */
static int point_inv_norm2(double norm, double hp, double ho, double* out) {
  if (is_iso(hp, ho)) {
    *out = 0.0;
    return AQ_OK;
  }
  const double n2 = norm * norm;
  if (n2 == 0.0) return E_ZERONORM("anisotropic loss undefined at |x| = 0");
  *out = 1.0 / n2;
  return AQ_OK;
}

/* detail::reconstruction_nearest_pass, pq.hpp:225-248 */
static void reconstruction_nearest(const double* x, size_t n, size_t d,
                                   const double* dict, size_t M, size_t k,
                                   size_t sd, uint32_t* codes) {
  for (size_t i = 0; i < n; ++i) {
    for (size_t m = 0; m < M; ++m) {
      size_t best_j = 0;
      double best = 0.0;
      for (size_t j = 0; j < k; ++j) {
        double c2, c1;
        residual_terms(x + i * d + m * sd, dict + (m * k + j) * sd, sd, &c2,
                       &c1);
        if (j == 0 || c2 < best) {
          best = c2;
          best_j = j;
        }
      }
      codes[i * M + m] = (uint32_t)best_j;
    }
  }
}

/* pq_quantize, pq.hpp:581-612 */
int orc_pq_quantize(const double* x, size_t n, size_t d, const double* dict,
                    size_t M, size_t k, size_t sd, const double* hp,
                    const double* ho, int passes, uint32_t* codes) {
  if (d != M * sd) return E_DIM("dataset dimension does not match codebook");
  if (passes < 0) return E_INVALID("passes must be >= 0");
  reconstruction_nearest(x, n, d, dict, M, k, sd, codes);
  if (passes == 0) return AQ_OK;
  double* norms = malloc(sizeof(double) * (n ? n : 1));
  double* buf = malloc(sizeof(double) * 2 * (M ? M : 1));
  pq_state st = {buf, buf + M, 0.0, 0.0};
  orc_row_norms(x, n, d, norms);
  int status = AQ_OK;
  for (size_t i = 0; i < n && !status; ++i) {
    double inv;
    status = point_inv_norm2(norms[i], hp[i], ho[i], &inv);
    if (status) break;
    pq_point_state(x + i * d, codes + i * M, dict, M, k, sd, &st);
    for (int p = 0; p < passes; ++p)
      if (!cd_sweep(x + i * d, codes + i * M, dict, M, k, sd, hp[i], ho[i],
                    inv, &st))
        break;
  }
  free(buf);
  free(norms);
  return status;
}

/* detail::pq_assign_pass, pq.hpp:202-221 */
int orc_pq_assign_pass(const double* x, size_t n, size_t d,
                       const double* dict, size_t M, size_t k, size_t sd,
                       const double* hp, const double* ho, int sweep_fixed,
                       uint32_t* codes, double* losses) {
  double* norms = malloc(sizeof(double) * (n ? n : 1));
  double* buf = malloc(sizeof(double) * 2 * (M ? M : 1));
  pq_state st = {buf, buf + M, 0.0, 0.0};
  orc_row_norms(x, n, d, norms);
  int status = AQ_OK;
  for (size_t i = 0; i < n; ++i) {
    double inv;
    status = point_inv_norm2(norms[i], hp[i], ho[i], &inv);
    if (status) break;
    uint32_t* row = codes + i * M;
    pq_point_state(x + i * d, row, dict, M, k, sd, &st);
    int sweeps = 0;
    while (cd_sweep(x + i * d, row, dict, M, k, sd, hp[i], ho[i], inv, &st) &&
           sweep_fixed && ++sweeps < 64) {
    }
    losses[i] = pq_point_loss(x + i * d, row, dict, M, k, sd, hp[i], ho[i],
                              inv, &st);
  }
  free(buf);
  free(norms);
  return status;
}

/* per-point pq_point_loss (as used by reseeding, pq.hpp:446-450) */
int orc_pq_point_losses(const double* x, size_t n, size_t d,
                        const double* dict, size_t M, size_t k, size_t sd,
                        const double* hp, const double* ho,
                        const uint32_t* codes, double* losses) {
  double* norms = malloc(sizeof(double) * (n ? n : 1));
  double* buf = malloc(sizeof(double) * 2 * (M ? M : 1));
  pq_state st = {buf, buf + M, 0.0, 0.0};
  orc_row_norms(x, n, d, norms);
  int status = AQ_OK;
  for (size_t i = 0; i < n; ++i) {
    double inv;
    status = point_inv_norm2(norms[i], hp[i], ho[i], &inv);
    if (status) break;
    losses[i] = pq_point_loss(x + i * d, codes + i * M, dict, M, k, sd, hp[i],
                              ho[i], inv, &st);
  }
  free(buf);
  free(norms);
  return status;
}

/* ---- pq.hpp: codebook update ---------------------------------------------- */

/* assemble_selector_system, pq.hpp:290-343. A row-major (dim x dim). */
int orc_assemble_selector_system(const double* x, size_t n, size_t d,
                                 const uint32_t* codes, const double* hp,
                                 const double* ho, size_t M, size_t k,
                                 double* A, double* rhs) {
  if (M == 0 || d % M != 0) return E_DIV("dimension not divisible by M");
  const size_t sd = d / M;
  const size_t dim = k * d;
  memset(A, 0, sizeof(double) * dim * dim);
  memset(rhs, 0, sizeof(double) * dim);
  double* norms = malloc(sizeof(double) * (n ? n : 1));
  orc_row_norms(x, n, d, norms);
  int status = AQ_OK;
  for (size_t i = 0; i < n && !status; ++i) {
    const double* xi = x + i * d;
    const uint32_t* row = codes + i * M;
    double coef = 0.0;
    if (hp[i] != ho[i]) {
      const double n2 = norms[i] * norms[i];
      if (n2 == 0.0) {
        status = E_ZERONORM("anisotropic update undefined at |x| = 0");
        break;
      }
      coef = (hp[i] - ho[i]) / n2;
    }
    for (size_t m = 0; m < M; ++m) {
      if (row[m] >= k) {
        status = E_CODE("code out of range");
        break;
      }
      const size_t rb = (m * k + row[m]) * sd;
      for (size_t c = 0; c < sd; ++c) {
        A[(rb + c) * dim + rb + c] += ho[i];
        rhs[rb + c] += hp[i] * xi[m * sd + c];
      }
      if (coef == 0.0) continue;
      for (size_t m2 = 0; m2 < M; ++m2) {
        const size_t cbk = (m2 * k + row[m2]) * sd;
        for (size_t c1 = 0; c1 < sd; ++c1) {
          const double xc = coef * xi[m * sd + c1];
          for (size_t c2 = 0; c2 < sd; ++c2)
            A[(rb + c1) * dim + cbk + c2] += xc * xi[m2 * sd + c2];
        }
      }
    }
  }
  free(norms);
  return status;
}

/* Eigen::LLT<MatrixXd>(A).solve(b) as pinned by the stand-in
 * (oracle/eigen_subset/Eigen/Dense): blocked, BS = 64, sequential inner
 * sums, no FMA. A is read on its lower triangle. */
#define LLT_BS 64
int orc_llt_solve(const double* A, size_t n, const double* b, double* xout) {
  double* L = malloc(sizeof(double) * (n * n ? n * n : 1));
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j <= i; ++j) L[i * n + j] = A[i * n + j];
  for (size_t kb = 0; kb < n; kb += LLT_BS) {
    const size_t be = kb + LLT_BS < n ? kb + LLT_BS : n;
    for (size_t j = kb; j < be; ++j) {
      double s = L[j * n + j];
      for (size_t q = kb; q < j; ++q) s = s - L[j * n + q] * L[j * n + q];
      if (s <= 0.0) {
        free(L);
        return E_SING("joint codebook system is not positive definite");
      }
      const double dg = sqrt(s);
      L[j * n + j] = dg;
      for (size_t i = j + 1; i < n; ++i) {
        double t = L[i * n + j];
        for (size_t q = kb; q < j; ++q) t = t - L[i * n + q] * L[j * n + q];
        L[i * n + j] = t / dg;
      }
    }
    for (size_t i = be; i < n; ++i)
      for (size_t j = be; j <= i; ++j) {
        double s = 0.0;
        for (size_t q = kb; q < be; ++q) s = s + L[i * n + q] * L[j * n + q];
        L[i * n + j] = L[i * n + j] - s;
      }
  }
  double* y = malloc(sizeof(double) * (n ? n : 1));
  memcpy(y, b, sizeof(double) * n);
  for (size_t kb = 0; kb < n; kb += LLT_BS) {
    const size_t be = kb + LLT_BS < n ? kb + LLT_BS : n;
    for (size_t i = kb; i < be; ++i) {
      double t = y[i];
      for (size_t q = kb; q < i; ++q) t = t - L[i * n + q] * y[q];
      y[i] = t / L[i * n + i];
    }
    for (size_t i = be; i < n; ++i) {
      double s = 0.0;
      for (size_t q = kb; q < be; ++q) s = s + L[i * n + q] * y[q];
      y[i] = y[i] - s;
    }
  }
  memcpy(xout, y, sizeof(double) * n);
  const size_t nb = (n + LLT_BS - 1) / LLT_BS;
  for (size_t bi = nb; bi-- > 0;) {
    const size_t kb = bi * LLT_BS;
    const size_t be = kb + LLT_BS < n ? kb + LLT_BS : n;
    for (size_t i = be; i-- > kb;) {
      double t = xout[i];
      for (size_t q = i + 1; q < be; ++q) t = t - L[q * n + i] * xout[q];
      xout[i] = t / L[i * n + i];
    }
    for (size_t i = 0; i < kb; ++i) {
      double s = 0.0;
      for (size_t q = kb; q < be; ++q) s = s + L[q * n + i] * xout[q];
      xout[i] = xout[i] - s;
    }
  }
  free(y);
  free(L);
  return AQ_OK;
}

/* update_codeword, vq.hpp:139-192 (members row-major, m x d) */
static int update_codeword(size_t d, const double* pts, size_t m,
                           const double* hp, const double* ho, double ridge,
                           double* out) {
  int all_iso = 1;
  for (size_t i = 0; i < m; ++i) all_iso &= is_iso(hp[i], ho[i]);
  if (all_iso) {
    double den = 0.0;
    for (size_t j = 0; j < d; ++j) out[j] = 0.0;
    for (size_t i = 0; i < m; ++i) {
      for (size_t j = 0; j < d; ++j) out[j] += hp[i] * pts[i * d + j];
      den += ho[i];
    }
    if (den <= 0.0) return E_SING("all h_perp weights are zero");
    for (size_t j = 0; j < d; ++j) out[j] /= den;
    return AQ_OK;
  }
  double mean_hperp = 0.0;
  for (size_t i = 0; i < m; ++i) mean_hperp += ho[i];
  mean_hperp /= (double)m;
  const double ridge_eff = ridge < 0.0 ? 1e-10 * mean_hperp : ridge;
  double* a = calloc(d * d, sizeof(double));
  double* b = calloc(d, sizeof(double));
  double diag = ridge_eff;
  for (size_t i = 0; i < m; ++i) {
    const double* xi = pts + i * d;
    double n2 = 0.0;
    for (size_t j = 0; j < d; ++j) n2 += xi[j] * xi[j];
    if (n2 == 0.0) {
      free(a);
      free(b);
      return E_ZERONORM("anisotropic update undefined at |x| = 0");
    }
    const double coef = (hp[i] - ho[i]) / n2;
    for (size_t c = 0; c < d; ++c) { /* lower rank-1 update, column c */
      const double ac = coef * xi[c];
      for (size_t r = c; r < d; ++r) a[r * d + c] += ac * xi[r];
    }
    for (size_t j = 0; j < d; ++j) b[j] += hp[i] * xi[j];
    diag += ho[i];
  }
  for (size_t j = 0; j < d; ++j) a[j * d + j] += diag;
  const int st = orc_llt_solve(a, d, b, out);
  free(a);
  free(b);
  if (st) return E_SING("codeword system is not positive definite");
  return AQ_OK;
}

/* stable ranking by loss descending, index ascending (vq.hpp:221-229) */
static const double* g_rank_losses;
static int rank_cmp(const void* pa, const void* pb) {
  const size_t a = *(const size_t*)pa, b = *(const size_t*)pb;
  const double la = g_rank_losses[a], lb = g_rank_losses[b];
  if (la > lb) return -1;
  if (lb > la) return 1;
  return a < b ? -1 : (a > b);
}
static void loss_ranking(const double* losses, size_t n, size_t* order) {
  for (size_t i = 0; i < n; ++i) order[i] = i;
  g_rank_losses = losses;
  qsort(order, n, sizeof(size_t), rank_cmp);
}

/* pq_codebook_update, pq.hpp:356-464 */
int orc_pq_codebook_update(const double* x, size_t n, size_t d,
                           const uint32_t* codes, const double* hp,
                           const double* ho, size_t M, size_t k, double ridge,
                           double* dict) {
  if (n == 0) return E_EMPTY("cannot update on an empty dataset");
  if (M == 0 || d % M != 0) return E_DIV("dimension not divisible by M");
  const size_t sd = d / M;
  memset(dict, 0, sizeof(double) * M * k * sd);
  uint32_t* usage = calloc(M * k, sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i)
    for (size_t m = 0; m < M; ++m) {
      if (codes[i * M + m] >= k) {
        free(usage);
        return E_CODE("code out of range");
      }
      ++usage[m * k + codes[i * M + m]];
    }
  int all_iso = 1;
  for (size_t i = 0; i < n; ++i) all_iso &= is_iso(hp[i], ho[i]);
  int status = AQ_OK;
  if (M == 1) {
    double* buf = malloc(sizeof(double) * n * d);
    double* whp = malloc(sizeof(double) * n);
    double* who = malloc(sizeof(double) * n);
    for (size_t j = 0; j < k && !status; ++j) {
      if (usage[j] == 0) continue;
      size_t cnt = 0;
      for (size_t i = 0; i < n; ++i) {
        if (codes[i] != j) continue;
        memcpy(buf + cnt * d, x + i * d, sizeof(double) * d);
        whp[cnt] = hp[i];
        who[cnt] = ho[i];
        ++cnt;
      }
      status = update_codeword(d, buf, cnt, whp, who, ridge, dict + j * d);
    }
    free(buf);
    free(whp);
    free(who);
  } else if (all_iso) {
    double* num = calloc(M * k * sd, sizeof(double));
    double* den = calloc(M * k, sizeof(double));
    for (size_t i = 0; i < n; ++i)
      for (size_t m = 0; m < M; ++m) {
        const size_t slot = m * k + codes[i * M + m];
        for (size_t c = 0; c < sd; ++c)
          num[slot * sd + c] += hp[i] * x[i * d + m * sd + c];
        den[slot] += ho[i];
      }
    for (size_t slot = 0; slot < M * k && !status; ++slot) {
      if (usage[slot] == 0) continue;
      if (den[slot] <= 0.0) {
        status = E_SING("zero total weight in block");
        break;
      }
      for (size_t c = 0; c < sd; ++c)
        dict[slot * sd + c] = num[slot * sd + c] / den[slot];
    }
    free(num);
    free(den);
  } else {
    const size_t dim = k * d;
    if (dim > 16384) {
      free(usage);
      return E_INVALID("stacked codebook system too large");
    }
    double* A = malloc(sizeof(double) * dim * dim);
    double* rhs = malloc(sizeof(double) * dim);
    status = orc_assemble_selector_system(x, n, d, codes, hp, ho, M, k, A, rhs);
    if (!status) {
      double tr = 0.0;
      for (size_t i = 0; i < dim; ++i) tr += A[i * dim + i];
      const double ridge_eff = ridge < 0.0 ? 1e-6 * tr / (double)dim : ridge;
      for (size_t i = 0; i < dim; ++i) A[i * dim + i] += ridge_eff;
      status = orc_llt_solve(A, dim, rhs, dict);
    }
    free(A);
    free(rhs);
  }
  if (!status) {
    int any_unused = 0;
    for (size_t s = 0; s < M * k; ++s) any_unused |= usage[s] == 0;
    if (any_unused) {
      double* losses = malloc(sizeof(double) * n);
      status = orc_pq_point_losses(x, n, d, dict, M, k, sd, hp, ho, codes,
                                   losses);
      if (!status) {
        size_t* order = malloc(sizeof(size_t) * n);
        loss_ranking(losses, n, order);
        size_t cursor = 0;
        for (size_t m = 0; m < M; ++m)
          for (size_t j = 0; j < k; ++j) {
            if (usage[m * k + j] != 0) continue;
            const size_t p = order[cursor++ % n];
            memcpy(dict + (m * k + j) * sd, x + p * d + m * sd,
                   sizeof(double) * sd);
          }
        free(order);
      }
      free(losses);
    }
  }
  free(usage);
  return status;
}

/* ---- rng.hpp ---------------------------------------------------------------- */

/* Rng::next_u64 (splitmix64), rng.hpp:32-38 */
uint64_t orc_rng_next_u64(uint64_t* s) {
  *s += 0x9E3779B97F4A7C15ull;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Rng::next_below, rng.hpp:46-52 */
static uint64_t next_below(uint64_t* s, uint64_t n) {
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const uint64_t r = orc_rng_next_u64(s);
    if (r >= threshold) return r % n;
  }
}

/* Rng::sample_distinct, rng.hpp:74-83, continuing a generator state */
static void sample_distinct_state(uint64_t* s, size_t n, size_t k,
                                  size_t* out) {
  size_t* idx = malloc(sizeof(size_t) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) idx[i] = i;
  for (size_t i = 0; i < k && i < n; ++i) {
    const size_t j = i + (size_t)next_below(s, n - i);
    const size_t t = idx[i];
    idx[i] = idx[j];
    idx[j] = t;
  }
  for (size_t i = 0; i < k && i < n; ++i) out[i] = idx[i];
  free(idx);
}

void orc_sample_distinct(uint64_t seed, size_t n, size_t k, size_t* out) {
  uint64_t s = seed;
  sample_distinct_state(&s, n, k, out);
}

/* ---- vq.hpp: isotropic k-means (warm start engine) --------------------------- */

/* train_avq with isotropic unit weights, vq.hpp:243-329; data n x d. */
static int train_avq_iso(const double* x, size_t n, size_t d, size_t k,
                         int max_it, double tol, uint64_t seed, double* cb,
                         uint32_t* assign) {
  if (n == 0) return E_EMPTY("cannot train on an empty dataset");
  if (k == 0 || k > n) return E_INVALID("need 1 <= k <= n");
  size_t* idx = malloc(sizeof(size_t) * k);
  orc_sample_distinct(seed, n, k, idx);
  for (size_t j = 0; j < k; ++j) memcpy(cb + j * d, x + idx[j] * d, sizeof(double) * d);
  free(idx);
  double* losses = malloc(sizeof(double) * n);
  uint32_t* prev = malloc(sizeof(uint32_t) * n);
  size_t* order = malloc(sizeof(size_t) * n);
  double* mean = malloc(sizeof(double) * d);
  /* vq_assign_pass, vq.hpp:196-217 (iso: score = dist2, loss = 1.0 * dist2) */
#define ASSIGN_PASS()                                                      \
  for (size_t i = 0; i < n; ++i) {                                         \
    size_t bj = 0;                                                         \
    double bd = 0.0;                                                       \
    for (size_t j = 0; j < k; ++j) {                                       \
      double d2, rd;                                                       \
      residual_terms(x + i * d, cb + j * d, d, &d2, &rd);                  \
      if (j == 0 || d2 < bd) {                                             \
        bd = d2;                                                           \
        bj = j;                                                            \
      }                                                                    \
    }                                                                      \
    assign[i] = (uint32_t)bj;                                              \
    losses[i] = 1.0 * bd;                                                  \
  }
  ASSIGN_PASS();
  double total = 0.0;
  for (size_t i = 0; i < n; ++i) total += losses[i];
  for (int iter = 0; iter < max_it; ++iter) {
    int have_order = 0;
    size_t cursor = 0;
    for (size_t j = 0; j < k; ++j) {
      size_t cnt = 0;
      double den = 0.0;
      for (size_t t = 0; t < d; ++t) mean[t] = 0.0;
      for (size_t i = 0; i < n; ++i) {
        if (assign[i] != j) continue;
        for (size_t t = 0; t < d; ++t) mean[t] += 1.0 * x[i * d + t];
        den += 1.0;
        ++cnt;
      }
      if (cnt == 0) { /* reseed_highest_loss, vq.hpp:284-292 */
        if (!have_order) {
          loss_ranking(losses, n, order);
          have_order = 1;
        }
        const size_t p = order[cursor++];
        memcpy(cb + j * d, x + p * d, sizeof(double) * d);
        continue;
      }
      for (size_t t = 0; t < d; ++t) cb[j * d + t] = mean[t] / den;
    }
    memcpy(prev, assign, sizeof(uint32_t) * n);
    ASSIGN_PASS();
    const double prev_total = total;
    total = 0.0;
    for (size_t i = 0; i < n; ++i) total += losses[i];
    size_t changes = 0;
    for (size_t i = 0; i < n; ++i) changes += assign[i] != prev[i];
    if (changes == 0) break;
    if (tol > 0.0 && (prev_total == 0.0 || prev_total - total <= tol * prev_total))
      break;
  }
#undef ASSIGN_PASS
  free(losses);
  free(prev);
  free(order);
  free(mean);
  return AQ_OK;
}

/* train_l2_pq, pq.hpp:469-501 */
int orc_train_l2_pq(const double* x, size_t n, size_t d, size_t M, size_t k,
                    int max_it, double tol, uint64_t seed, double* dict,
                    uint32_t* codes) {
  if (n == 0) return E_EMPTY("cannot train on an empty dataset");
  if (M == 0 || d % M != 0) return E_DIV("dimension not divisible by M");
  if (k == 0 || k > n) return E_INVALID("need 1 <= k <= n");
  const size_t sd = d / M;
  double* sub = malloc(sizeof(double) * n * sd);
  uint32_t* a = malloc(sizeof(uint32_t) * n);
  int st = AQ_OK;
  for (size_t m = 0; m < M && !st; ++m) {
    for (size_t i = 0; i < n; ++i)
      memcpy(sub + i * sd, x + i * d + m * sd, sizeof(double) * sd);
    st = train_avq_iso(sub, n, sd, k, max_it, tol, seed + m, dict + m * k * sd, a);
    for (size_t i = 0; i < n; ++i) codes[i * M + m] = a[i];
  }
  free(sub);
  free(a);
  return st;
}

/* train_apq, pq.hpp:513-575 */
int orc_train_apq(const double* x, size_t n, size_t d, size_t M, size_t k,
                  const double* hp, const double* ho, int max_it, double tol,
                  uint64_t seed, double ridge, int sweep_fixed, int warm_start,
                  double* dict, uint32_t* codes, double* history,
                  size_t* history_len) {
  if (n == 0) return E_EMPTY("cannot train on an empty dataset");
  if (M == 0 || d % M != 0) return E_DIV("dimension not divisible by M");
  if (k == 0 || k > n) return E_INVALID("need 1 <= k <= n");
  const size_t sd = d / M;
  int st;
  *history_len = 0;
  if (warm_start) {
    st = orc_train_l2_pq(x, n, d, M, k, max_it, tol, seed, dict, codes);
    if (st) return st;
  } else {
    uint64_t s = seed;
    size_t* idx = malloc(sizeof(size_t) * k);
    for (size_t m = 0; m < M; ++m) {
      sample_distinct_state(&s, n, k, idx);
      for (size_t j = 0; j < k; ++j)
        memcpy(dict + (m * k + j) * sd, x + idx[j] * d + m * sd,
               sizeof(double) * sd);
    }
    free(idx);
    reconstruction_nearest(x, n, d, dict, M, k, sd, codes);
  }
  double* losses = malloc(sizeof(double) * n);
  uint32_t* prev = malloc(sizeof(uint32_t) * n * M);
  st = orc_pq_assign_pass(x, n, d, dict, M, k, sd, hp, ho, sweep_fixed, codes,
                          losses);
  double total = 0.0;
  if (!st) {
    for (size_t i = 0; i < n; ++i) total += losses[i];
    history[(*history_len)++] = total;
  }
  for (int iter = 0; iter < max_it && !st; ++iter) {
    st = orc_pq_codebook_update(x, n, d, codes, hp, ho, M, k, ridge, dict);
    if (st) break;
    memcpy(prev, codes, sizeof(uint32_t) * n * M);
    st = orc_pq_assign_pass(x, n, d, dict, M, k, sd, hp, ho, sweep_fixed,
                            codes, losses);
    if (st) break;
    const double prev_total = total;
    total = 0.0;
    for (size_t i = 0; i < n; ++i) total += losses[i];
    history[(*history_len)++] = total;
    size_t changes = 0;
    for (size_t i = 0; i < n * M; ++i) changes += codes[i] != prev[i];
    if (changes == 0) break;
    if (tol > 0.0 && (prev_total == 0.0 || prev_total - total <= tol * prev_total))
      break;
  }
  free(losses);
  free(prev);
  return st;
}

/* detail::vq_assign_pass, vq.hpp:196-217 (assign_scan 83-100, recorded_loss
   102-105): per point the lowest-index argmin of the full-vector loss. */
static int vq_assign_pass(const double* x, size_t n, size_t d, const double* cw,
                          size_t k, const double* norms, const double* hp,
                          const double* ho, uint32_t* assign, double* losses) {
  for (size_t i = 0; i < n; ++i) {
    const int iso = is_iso(hp[i], ho[i]);
    double inv = 0.0;
    if (!iso) {
      const double n2 = norms[i] * norms[i];
      if (n2 == 0.0) return E_ZERONORM("anisotropic assignment undefined at |x|=0");
      inv = 1.0 / n2;
    }
    size_t best_j = 0;
    double bs = 0.0, b2 = 0.0;
    for (size_t j = 0; j < k; ++j) {
      double c2, c1;
      residual_terms(x + i * d, cw + j * d, d, &c2, &c1);
      const double score = iso ? c2 : combined_loss(c2, c1, hp[i], ho[i], inv);
      if (j == 0 || score < bs) {
        bs = score;
        b2 = c2;
        best_j = j;
      }
    }
    assign[i] = (uint32_t)best_j;
    losses[i] = iso ? ho[i] * b2 : (bs > 0.0 ? bs : 0.0);
  }
  return AQ_OK;
}

/* vq_quantize, vq.hpp:332-343 */
int orc_vq_quantize(const double* x, size_t n, size_t d, const double* cw, size_t k,
                    const double* hp, const double* ho, uint32_t* assign) {
  double* norms = malloc(sizeof(double) * (n ? n : 1));
  double* losses = malloc(sizeof(double) * (n ? n : 1));
  orc_row_norms(x, n, d, norms);
  const int st = vq_assign_pass(x, n, d, cw, k, norms, hp, ho, assign, losses);
  free(norms);
  free(losses);
  return st;
}

/* assign_point, vq.hpp:112-132 */
int orc_assign_point(const double* x, size_t d, const double* cw, size_t k, double hp,
                     double ho, uint32_t* out) {
  if (k == 0) return E_INVALID("empty codebook");
  double norm;
  orc_row_norms(x, 1, d, &norm);
  if (!is_iso(hp, ho) && norm * norm == 0.0)
    return E_ZERONORM("anisotropic assignment undefined at |x| = 0");
  double losses;
  return vq_assign_pass(x, 1, d, cw, k, &norm, &hp, &ho, out, &losses);
}

/* update_codeword, vq.hpp:139-192 */
int orc_update_codeword(size_t d, const double* pts, size_t m, const double* hp,
                        const double* ho, double ridge, double* out) {
  if (d == 0 || m == 0) return E_INVALID("points must be a non-empty multiple of d");
  return update_codeword(d, pts, m, hp, ho, ridge, out);
}

/* train_avq, vq.hpp:243-329: codewords = rows Rng(seed).sample_distinct(n, k);
   assignment pass -> history[0]; then per iteration the per-partition
   update_codeword (members in ascending order; an empty partition keeps its
   codeword or takes the next point of the loss ranking of the PREVIOUS pass),
   assignment pass, stopping rules as train_apq. */
int orc_train_avq(const double* x, size_t n, size_t d, size_t k, const double* hp,
                  const double* ho, int max_it, double tol, uint64_t seed, double ridge,
                  int keep_previous, double* cw, uint32_t* assign, double* history,
                  size_t* history_len) {
  *history_len = 0;
  if (n == 0) return E_EMPTY("cannot train on an empty dataset");
  if (k == 0 || k > n) return E_INVALID("need 1 <= k <= n (codewords come from datapoints)");
  {
    uint64_t s = seed;
    size_t* idx = malloc(sizeof(size_t) * k);
    sample_distinct_state(&s, n, k, idx);
    for (size_t j = 0; j < k; ++j) memcpy(cw + j * d, x + idx[j] * d, sizeof(double) * d);
    free(idx);
  }
  double* norms = malloc(sizeof(double) * n);
  double* losses = malloc(sizeof(double) * n);
  uint32_t* prev = malloc(sizeof(uint32_t) * n);
  uint32_t* counts = malloc(sizeof(uint32_t) * k);
  double* buf = malloc(sizeof(double) * n * d);
  double* whp = malloc(sizeof(double) * n);
  double* who = malloc(sizeof(double) * n);
  size_t* order = malloc(sizeof(size_t) * n);
  orc_row_norms(x, n, d, norms);
  int st = vq_assign_pass(x, n, d, cw, k, norms, hp, ho, assign, losses);
  double total = 0.0;
  if (!st) {
    for (size_t i = 0; i < n; ++i) total += losses[i];
    history[(*history_len)++] = total;
  }
  for (int iter = 0; iter < max_it && !st; ++iter) {
    memset(counts, 0, sizeof(uint32_t) * k);
    for (size_t i = 0; i < n; ++i) ++counts[assign[i]];
    int ranked = 0;
    size_t cursor = 0;
    for (size_t j = 0; j < k && !st; ++j) {
      if (counts[j] == 0) {
        if (keep_previous) continue;
        if (!ranked) {
          loss_ranking(losses, n, order);
          ranked = 1;
        }
        memcpy(cw + j * d, x + order[cursor++] * d, sizeof(double) * d);
        continue;
      }
      size_t cnt = 0;
      for (size_t i = 0; i < n; ++i) {
        if (assign[i] != j) continue;
        memcpy(buf + cnt * d, x + i * d, sizeof(double) * d);
        whp[cnt] = hp[i];
        who[cnt] = ho[i];
        ++cnt;
      }
      st = update_codeword(d, buf, cnt, whp, who, ridge, cw + j * d);
    }
    if (st) break;
    memcpy(prev, assign, sizeof(uint32_t) * n);
    st = vq_assign_pass(x, n, d, cw, k, norms, hp, ho, assign, losses);
    if (st) break;
    const double prev_total = total;
    total = 0.0;
    for (size_t i = 0; i < n; ++i) total += losses[i];
    history[(*history_len)++] = total;
    size_t changes = 0;
    for (size_t i = 0; i < n; ++i) changes += assign[i] != prev[i];
    if (changes == 0) break;
    if (tol > 0.0 && (prev_total == 0.0 || prev_total - total <= tol * prev_total)) break;
  }
  free(norms);
  free(losses);
  free(prev);
  free(counts);
  free(buf);
  free(whp);
  free(who);
  free(order);
  return st;
}

/* ---- index.hpp ----------------------------------------------------------------- */

/* build_lut, index.hpp:56-70 */
int orc_build_lut(const double* q, size_t d, const double* dict, size_t M,
                  size_t k, size_t sd, double* lut) {
  if (d != M * sd) return E_DIM("query dimension does not match codebook");
  for (size_t m = 0; m < M; ++m)
    for (size_t j = 0; j < k; ++j)
      lut[m * k + j] = dot(q + m * sd, dict + (m * k + j) * sd, sd);
  return AQ_OK;
}

typedef struct {
  uint32_t index;
  double score;
} hit;

/* select_top order: score descending, index ascending (index.hpp:88-112) */
static int hit_cmp(const void* pa, const void* pb) {
  const hit* a = pa;
  const hit* b = pb;
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  return a->index < b->index ? -1 : (a->index > b->index);
}

/* adc_search, index.hpp:118-134, for each query of a batch */
int orc_adc_search_batch(const double* Q, size_t nq, size_t d,
                         const uint32_t* codes, size_t n, size_t M,
                         size_t codes_k, const double* dict, size_t cbM,
                         size_t k, size_t sd, size_t topn, uint32_t* ids,
                         double* scores) {
  if (n == 0) return E_EMPTYIDX("no quantized datapoints");
  if (topn < 1) return E_INVALID("topn must be >= 1");
  if (M != cbM || codes_k > k) return E_DIM("code matrix does not match codebook");
  const size_t te = topn < n ? topn : n;
  double* lut = malloc(sizeof(double) * M * k);
  hit* all = malloc(sizeof(hit) * n);
  int st = AQ_OK;
  for (size_t qi = 0; qi < nq && !st; ++qi) {
    st = orc_build_lut(Q + qi * d, d, dict, M, k, sd, lut);
    if (st) break;
    for (size_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (size_t m = 0; m < M; ++m) s += lut[m * k + codes[i * M + m]];
      all[i].index = (uint32_t)i;
      all[i].score = s;
    }
    qsort(all, n, sizeof(hit), hit_cmp);
    for (size_t t = 0; t < te; ++t) {
      ids[qi * te + t] = all[t].index;
      scores[qi * te + t] = all[t].score;
    }
  }
  free(lut);
  free(all);
  return st;
}

/* Exact-dot rerank (north_star A22; restated from exact_search, index.hpp:137-147) */
int orc_rerank(const double* Q, size_t nq, const double* x, size_t n,
               size_t d, const uint32_t* cand, size_t ncand, size_t keep,
               uint32_t* ids, double* scores) {
  const size_t ke = keep < ncand ? keep : ncand;
  hit* h = malloc(sizeof(hit) * (ncand ? ncand : 1));
  for (size_t qi = 0; qi < nq; ++qi) {
    for (size_t c = 0; c < ncand; ++c) {
      const uint32_t id = cand[qi * ncand + c];
      if (id >= n) {
        free(h);
        return E_INVALID("candidate id out of range");
      }
      h[c].index = id;
      h[c].score = dot(Q + qi * d, x + (size_t)id * d, d);
    }
    qsort(h, ncand, sizeof(hit), hit_cmp);
    for (size_t t = 0; t < ke; ++t) {
      ids[qi * ke + t] = h[t].index;
      scores[qi * ke + t] = h[t].score;
    }
  }
  free(h);
  return AQ_OK;
}

/* exact_search / exact_ground_truth, index.hpp:137-162 */
int orc_exact_search_batch(const double* Q, size_t nq, const double* x,
                           size_t n, size_t d, size_t depth, uint32_t* ids,
                           double* scores) {
  if (n == 0) return E_EMPTY("empty dataset");
  if (depth < 1) return E_INVALID("topn must be >= 1");
  const size_t te = depth < n ? depth : n;
  hit* all = malloc(sizeof(hit) * n);
  for (size_t qi = 0; qi < nq; ++qi) {
    for (size_t i = 0; i < n; ++i) {
      all[i].index = (uint32_t)i;
      all[i].score = dot(Q + qi * d, x + i * d, d);
    }
    qsort(all, n, sizeof(hit), hit_cmp);
    for (size_t t = 0; t < te; ++t) {
      ids[qi * te + t] = all[t].index;
      scores[qi * te + t] = all[t].score;
    }
  }
  free(all);
  return AQ_OK;
}
