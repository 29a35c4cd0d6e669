/* oracle/anisoq_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (anisoq, arXiv 1908.10396),
 * used as the parity checker for the CUDA path. Pinned against the reference
 * itself (oracle/_ref, built from /root/reference by oracle/Makefile) and the
 * reference tests' worked examples / golden bytes (tests/test_oracle.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. Status codes are those of include/anisoq_b200.h.
 */
#ifndef ANISOQ_ORACLE_H_
#define ANISOQ_ORACLE_H_
#include <stddef.h>
#include <stdint.h>

const char* orc_last_error(void);

void orc_row_norms(const double* x, size_t n, size_t d, double* norms);
int orc_eta_limit(double t, double norm, int d, double* out);
/* CLI resolve_weights (anisoq_main.cpp:108-142) with the |x| <= T policy:
 * policy 0 -> error, 1 -> (h_par, h_perp) = (1, 0). */
int orc_threshold_weights(const double* norms, size_t n, size_t d, double t,
                          int policy, double* hp, double* ho);

int orc_pq_quantize(const double* x, size_t n, size_t d, const double* dict,
                    size_t M, size_t k, size_t sd, const double* hp,
                    const double* ho, int passes, uint32_t* codes);
int orc_pq_assign_pass(const double* x, size_t n, size_t d,
                       const double* dict, size_t M, size_t k, size_t sd,
                       const double* hp, const double* ho, int sweep_fixed,
                       uint32_t* codes, double* losses);
int orc_pq_point_losses(const double* x, size_t n, size_t d,
                        const double* dict, size_t M, size_t k, size_t sd,
                        const double* hp, const double* ho,
                        const uint32_t* codes, double* losses);

int orc_assemble_selector_system(const double* x, size_t n, size_t d,
                                 const uint32_t* codes, const double* hp,
                                 const double* ho, size_t M, size_t k,
                                 double* A /* row-major dim^2 */,
                                 double* rhs);
int orc_llt_solve(const double* A /* row-major, lower used */, size_t dim,
                  const double* b, double* x);
int orc_pq_codebook_update(const double* x, size_t n, size_t d,
                           const uint32_t* codes, const double* hp,
                           const double* ho, size_t M, size_t k, double ridge,
                           double* dict);

int orc_train_l2_pq(const double* x, size_t n, size_t d, size_t M, size_t k,
                    int max_it, double tol, uint64_t seed, double* dict,
                    uint32_t* codes);
int orc_train_apq(const double* x, size_t n, size_t d, size_t M, size_t k,
                  const double* hp, const double* ho, int max_it, double tol,
                  uint64_t seed, double ridge, int sweep_fixed, int warm_start,
                  double* dict, uint32_t* codes, double* history,
                  size_t* history_len);

int orc_vq_quantize(const double* x, size_t n, size_t d, const double* cw, size_t k,
                    const double* hp, const double* ho, uint32_t* assign);
int orc_assign_point(const double* x, size_t d, const double* cw, size_t k, double hp,
                     double ho, uint32_t* out);
int orc_update_codeword(size_t d, const double* pts, size_t m, const double* hp,
                        const double* ho, double ridge, double* out);
int orc_train_avq(const double* x, size_t n, size_t d, size_t k, const double* hp,
                  const double* ho, int max_it, double tol, uint64_t seed, double ridge,
                  int keep_previous, double* codewords, uint32_t* assignments,
                  double* history, size_t* history_len);
int orc_build_lut(const double* q, size_t d, const double* dict, size_t M,
                  size_t k, size_t sd, double* lut);
int orc_adc_search_batch(const double* Q, size_t nq, size_t d,
                         const uint32_t* codes, size_t n, size_t M,
                         size_t codes_k, const double* dict, size_t cbM,
                         size_t k, size_t sd, size_t topn, uint32_t* ids,
                         double* scores);
int orc_rerank(const double* Q, size_t nq, const double* x, size_t n,
               size_t d, const uint32_t* cand, size_t ncand, size_t keep,
               uint32_t* ids, double* scores);
int orc_exact_search_batch(const double* Q, size_t nq, const double* x,
                           size_t n, size_t d, size_t depth, uint32_t* ids,
                           double* scores);

/* rng.hpp:28-89 */
uint64_t orc_rng_next_u64(uint64_t* state);
void orc_sample_distinct(uint64_t seed, size_t n, size_t k, size_t* out);

#endif
