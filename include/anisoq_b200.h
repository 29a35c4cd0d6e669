/* anisoq_b200.h — C ABI of the B200-native anisotropic PQ hot path.
 *
 * Drop-in boundary for the reference `anisoq` C++ library
 * (/root/reference/proj/include/anisoq, header-only C++20). The reference has
 * no FFI of its own; its public surface is the set of C++ functions below,
 * and every `aq_*` entry point here is the plain-pointer form of one of them
 * (same argument meaning, same validation order, same error classes). The
 * C++ headers under include/anisoq/ and the Python module
 * paper_1908_10396_b200/anisoq.py rebuild the reference signatures on top.
 *
 *   aq_pq_quantize            <- anisoq::pq_quantize            pq.hpp:581-612
 *   aq_pq_assign_pass         <- anisoq::detail::pq_assign_pass pq.hpp:202-221
 *   aq_pq_assign_point        <- anisoq::pq_assign_point        pq.hpp:256-282
 *   aq_assemble_selector_system <- anisoq::assemble_selector_system pq.hpp:290-343
 *   aq_pq_codebook_update     <- anisoq::pq_codebook_update     pq.hpp:356-464
 *   aq_train_l2_pq            <- anisoq::train_l2_pq            pq.hpp:469-501
 *   aq_train_apq              <- anisoq::train_apq              pq.hpp:513-575
 *   aq_train_avq              <- anisoq::train_avq              vq.hpp:243-329
 *   aq_build_lut              <- anisoq::build_lut              index.hpp:56-70
 *   aq_adc_search             <- anisoq::adc_search             index.hpp:118-134
 *   aq_adc_search_batch       <- adc_search over a query batch (evaluate, index.hpp:251-259)
 *   aq_rerank                 <- exact-dot rerank (north_star; restated from
 *                                exact_search index.hpp:137-147, dot geometry.hpp:170-174)
 *   aq_exact_search_batch     <- anisoq::exact_ground_truth     index.hpp:150-162
 *
 * Conventions
 *   - Every function returns an aq_status. 0 = success. Codes 1..13 are the
 *     reference exception types of error.hpp:43-55 in declaration order;
 *     aq_error_class() gives their ErrorClass (error.hpp:25). The message of
 *     the last failure on the calling thread is aq_last_error(), formatted as
 *     the reference's `what()` ("<TypeName>: <detail>").
 *   - Host arrays are row-major, little-endian. Datasets are float32 values
 *     (the reference holds doubles that are float32-exact: dataset.hpp:146-151,
 *     288); norms are recomputed on the device in float64 exactly as
 *     dataset.hpp:55-59 does.
 *   - Codebooks are float64, entry (m, j) at (m*k + j)*sub_dimension
 *     (pq.hpp:36-52). Codes are uint32 n x M row-major on the host
 *     (pq.hpp:54-67) and packed 4-bit (k <= 16; low nibble = even m) or
 *     8-bit (k <= 256) on the device.
 *   - Per-point weights (geometry.hpp:119-145) are given by aq_weights.
 *   - All calls are synchronous with respect to the host, like the reference.
 *     Device-resident variants (aq_dev_*) operate on session-owned buffers
 *     and are stream-ordered on the session stream.
 *   - Threads: a session (its stream, scratch buffers and the objects created
 *     from it) must be used by one thread at a time; concurrent callers use
 *     one session each (several sessions may share a device). The last-error
 *     message is per thread.
 */
#ifndef ANISOQ_B200_H_
#define ANISOQ_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum aq_status {
  AQ_OK = 0,
  AQ_E_INVALID_ARGUMENT = 1,
  AQ_E_ZERO_NORM_DATAPOINT = 2,
  AQ_E_INVALID_THRESHOLD = 3,
  AQ_E_EMPTY_DATASET = 4,
  AQ_E_EMPTY_INDEX = 5,
  AQ_E_DIMENSION_MISMATCH = 6,
  AQ_E_DIMENSION_NOT_DIVISIBLE = 7,
  AQ_E_CODE_OUT_OF_RANGE = 8,
  AQ_E_MALFORMED_FILE = 9,
  AQ_E_INSUFFICIENT_DATA = 10,
  AQ_E_GROUND_TRUTH_MISMATCH = 11,
  AQ_E_QUADRATURE_FAILURE = 12,
  AQ_E_SINGULAR_SYSTEM = 13,
  AQ_E_CUDA = 100,        /* device / driver failure (runtime class) */
  AQ_E_UNSUPPORTED = 101  /* shape outside the device kernels' envelope */
} aq_status;

/* ErrorClass (error.hpp:25): 0 = validation, 1 = runtime. */
int aq_error_class(int status);
const char* aq_last_error(void);
const char* aq_status_name(int status);

/* ---- weights (geometry.hpp:119-145; CLI resolve_weights anisoq_main.cpp:108-142) */
typedef enum aq_weight_mode {
  AQ_WEIGHTS_UNIFORM = 0,   /* every point uses (h_parallel, h_perpendicular) */
  AQ_WEIGHTS_PER_POINT = 1, /* h_parallel[i], h_perpendicular[i] host arrays */
  AQ_WEIGHTS_THRESHOLD = 2  /* h_par = eta_limit(T, |x_i|, d), h_perp = 1;
                               |x_i| <= T -> policy below */
} aq_weight_mode;

typedef enum aq_threshold_policy {
  AQ_THRESHOLD_THROW = 0,         /* reference: InvalidThreshold (geometry.hpp:397) */
  AQ_THRESHOLD_PARALLEL_ONLY = 1  /* eta = inf: h_par = 1, h_perp = 0 */
} aq_threshold_policy;

typedef struct aq_weights {
  int mode;                       /* aq_weight_mode */
  double h_parallel;              /* UNIFORM */
  double h_perpendicular;         /* UNIFORM */
  const double* h_parallel_arr;   /* PER_POINT, length n */
  const double* h_perpendicular_arr;
  double threshold;               /* THRESHOLD */
  int threshold_policy;           /* aq_threshold_policy */
} aq_weights;

/* ---- session ----------------------------------------------------------- */
typedef struct aq_session aq_session;

int aq_session_create(int device, aq_session** out);
int aq_session_destroy(aq_session* s);
/* cudaStream_t of the session, for callers that time or order work on it. */
void* aq_session_stream(aq_session* s);
int aq_session_sync(aq_session* s);
/* Kernel launches issued by this session so far (evidence counter). */
uint64_t aq_session_launches(aq_session* s);

/* Per-kernel CUDA-event timers on the session stream (evidence for the
 * roofline in bench.py). Slots: 0 encode, 1 adc_score, 2 adc_merge,
 * 3 rerank, 4 lut, 5 normal-equation assembly, 6 Cholesky, 7 k-means warm
 * start, 8 exact search (filter + merge). */
int aq_session_timing(aq_session* s, int enable);
int aq_session_timer_read(aq_session* s, int slot, double* ms, uint64_t* count,
                          int reset);

/* ---- device-resident objects ------------------------------------------- */
typedef struct aq_dataset aq_dataset;   /* x (fp32 n x d) + norms (fp64) */
typedef struct aq_codebook aq_codebook; /* fp64 dictionaries + fp32 staging */
typedef struct aq_codes aq_codes;       /* packed codes n x M */

/* Upload float32 rows; norms are computed on the device (dataset.hpp:55-59). */
int aq_dataset_upload(aq_session* s, const float* x, size_t n, size_t d,
                      aq_dataset** out);
/* Upload float64 rows (the reference's Dataset values, dataset.hpp:41-51).
   Stored as float32 when every value is float32-exact (fvecs files, the
   reference generator: dataset.hpp:146-151, 288), else as float64 — e.g.
   unit_normalize output (dataset.hpp:229). Results equal the reference's
   either way; the float64 storage runs the generic kernels. */
int aq_dataset_upload_f64(aq_session* s, const double* x, size_t n, size_t d,
                          aq_dataset** out);
/* 1 when the dataset holds float64 rows. */
int aq_dataset_is_f64(const aq_dataset* ds);
/* Wrap rows already on this session's device (not copied, not freed). */
int aq_dataset_wrap_device(aq_session* s, const float* x_dev, size_t n,
                           size_t d, aq_dataset** out);
int aq_dataset_free(aq_dataset* ds);
int aq_dataset_norms(aq_dataset* ds, double* norms_out /* n */);

int aq_codebook_upload(aq_session* s, const double* dictionaries, size_t M,
                       size_t k, size_t sub_dimension, aq_codebook** out);
int aq_codebook_download(aq_codebook* cb, double* dictionaries_out);
int aq_codebook_free(aq_codebook* cb);

int aq_codes_alloc(aq_session* s, size_t n, size_t M, size_t k,
                   aq_codes** out);
int aq_codes_upload(aq_session* s, const uint32_t* codes, size_t n, size_t M,
                    size_t k, aq_codes** out);
/* Upload codes already packed in the device layout (rows of M/2 bytes for
 * k <= 16, M bytes otherwise). */
int aq_codes_upload_packed(aq_session* s, const uint8_t* packed, size_t n,
                           size_t M, size_t k, aq_codes** out);
int aq_codes_download(aq_codes* c, uint32_t* codes_out /* n*M */);
int aq_codes_download_packed(aq_codes* c, uint8_t* packed_out);
size_t aq_codes_row_bytes(aq_codes* c);
int aq_codes_free(aq_codes* c);

/* ---- encode (pq.hpp:581-612, 202-221) ------------------------------------ */
/* Re-quantize `ds` against `cb`: reconstruction-nearest init then `passes`
 * coordinate-descent sweeps with per-point early exit. Writes `out`. */
int aq_dev_pq_quantize(aq_dataset* ds, aq_codebook* cb, const aq_weights* w,
                       int passes, aq_codes* out);
/* One assignment pass (training): state from current codes, one sweep (or up
 * to 64 when sweep_to_fixed_point), per-point loss into losses_dev (device
 * fp64, length n) if non-NULL; number of changed codes into *changed. */
int aq_dev_pq_assign_pass(aq_dataset* ds, aq_codebook* cb,
                          const aq_weights* w, int sweep_to_fixed_point,
                          aq_codes* codes, double* losses_dev,
                          uint64_t* changed);

/* Host-pointer forms (reference by-value semantics). */
int aq_pq_quantize(aq_session* s, const float* x, size_t n, size_t d,
                   const double* dictionaries, size_t M, size_t k,
                   size_t sub_dimension, const aq_weights* w, int passes,
                   uint32_t* codes_out);
int aq_pq_assign_pass(aq_session* s, const float* x, size_t n, size_t d,
                      const double* dictionaries, size_t M, size_t k,
                      size_t sub_dimension, const aq_weights* w,
                      int sweep_to_fixed_point, uint32_t* codes_inout,
                      double* losses_out);
int aq_pq_assign_point(aq_session* s, const double* x, size_t d,
                       const uint32_t* current_codes,
                       const double* dictionaries, size_t M, size_t k,
                       size_t sub_dimension, double h_parallel,
                       double h_perpendicular, uint32_t* codes_out);
/* pq_assign_point with an explicit sweep_order (pq.hpp:256-282): the
 * subspaces visited in order (repeats allowed); order_len 0 = default_sweep.
 * Entries >= M are rejected (AQ_E_INVALID_ARGUMENT; undefined in the
 * reference). */
int aq_pq_assign_point_order(aq_session* s, const double* x, size_t d,
                             const uint32_t* current, const double* dictionaries,
                             size_t M, size_t k, size_t sub_dimension,
                             double h_parallel, double h_perpendicular,
                             const size_t* sweep_order, size_t order_len,
                             uint32_t* codes_out);

/* ---- search (index.hpp:56-134) ------------------------------------------ */
int aq_build_lut(aq_session* s, const double* q, size_t d,
                 const double* dictionaries, size_t M, size_t k,
                 size_t sub_dimension, double* lut_out /* M*k */);
/* Batched ADC top-N: for each query the exact reference ordering
 * (score desc, index asc) of sum_m lut[m][code]; scores bit-identical to the
 * reference's float64 sequential sum. ids_out/scores_out are nq x topn_eff,
 * topn_eff = min(topn, n). */
int aq_dev_adc_search(aq_codes* codes, aq_codebook* cb, const double* queries,
                      size_t nq, size_t topn, uint32_t* ids_out,
                      double* scores_out);
/* Same with device pointers (q_dev float64 nq x d; outputs on the device). */
int aq_dev_adc_search_d(aq_codes* codes, aq_codebook* cb, const double* q_dev,
                        size_t nq, size_t topn, uint32_t* ids_dev,
                        double* scores_dev);
/* Fused query pipeline: ADC top-`topn` then exact-dot rerank to `keep`
 * (host queries in, host results out; index and dataset resident). Any of
 * the four outputs may be NULL. */
int aq_dev_search_rerank(aq_dataset* ds, aq_codes* codes, aq_codebook* cb,
                         const double* queries, size_t nq, size_t topn,
                         size_t keep, uint32_t* adc_ids_out,
                         double* adc_scores_out, uint32_t* ids_out,
                         double* scores_out);
int aq_dev_search_rerank_d(aq_dataset* ds, aq_codes* codes, aq_codebook* cb,
                           const double* q_dev, size_t nq, size_t topn,
                           size_t keep, uint32_t* adc_ids_dev,
                           double* adc_scores_dev, uint32_t* ids_dev,
                           double* scores_dev);
/* Exact float64 dots dot(q, x[id]) for candidate ids, aligned with the
 * input (device pointers): the per-shard half of the multi-GPU rerank. */
int aq_dev_exact_dots_d(aq_dataset* ds, const double* q_dev, size_t nq,
                        const uint32_t* cand_dev, size_t ncand, double* out_dev);
int aq_adc_search(aq_session* s, const double* q, size_t d,
                  const uint32_t* codes, size_t n, size_t M, size_t codes_k,
                  const double* dictionaries, size_t cb_M, size_t k,
                  size_t sub_dimension, size_t topn, uint32_t* ids_out,
                  double* scores_out, size_t* count_out);
/* Exact-dot rerank of candidate ids: score = dot(q, x[id]) in float64
 * sequential order; keep the best `keep` by (score desc, index asc). */
int aq_dev_rerank(aq_dataset* ds, const double* queries, size_t nq,
                  const uint32_t* cand_ids, size_t ncand, size_t keep,
                  uint32_t* ids_out, double* scores_out);
/* Brute-force exact MIPS top-`depth` (exact_ground_truth). */
int aq_dev_exact_search(aq_dataset* ds, const double* queries, size_t nq,
                        size_t depth, uint32_t* ids_out, double* scores_out);

/* ---- codebook update (pq.hpp:290-464) ------------------------------------ */
int aq_dev_assemble_selector_system(aq_dataset* ds, aq_codes* codes,
                                    const aq_weights* w, double* A_out,
                                    double* rhs_out);
int aq_dev_pq_codebook_update(aq_dataset* ds, aq_codes* codes,
                              const aq_weights* w, double ridge,
                              aq_codebook* out);

int aq_pq_codebook_update(aq_session* s, const float* x, size_t n, size_t d,
                          const uint32_t* codes, size_t M, size_t k,
                          const aq_weights* w, double ridge, double* dict_out);

/* ---- trainers (pq.hpp:469-575) ------------------------------------------- */
typedef struct aq_train_config {  /* vq.hpp:55-69 */
  int max_iterations;
  double relative_tolerance;
  uint64_t seed;
  int empty_partition_policy;     /* 0 reseed_highest_loss, 1 keep_previous */
  double ridge;
  int threads;                    /* host knob; results never depend on it */
  int sweep_to_fixed_point;
} aq_train_config;

int aq_dev_train_l2_pq(aq_dataset* ds, size_t M, size_t k,
                       const aq_train_config* cfg, aq_codebook** cb_out,
                       aq_codes** codes_out);
int aq_dev_train_apq(aq_dataset* ds, size_t M, size_t k, const aq_weights* w,
                     const aq_train_config* cfg, int warm_start,
                     aq_codebook** cb_out, aq_codes** codes_out,
                     double* loss_history_out, size_t* history_len);
/* train_avq (vq.hpp:243-329): one k x d codebook, returned as M = 1;
 * cfg->empty_partition_policy 0 reseeds an empty partition from the previous
 * pass's loss ranking, 1 keeps its codeword. */
int aq_dev_train_avq(aq_dataset* ds, size_t k, const aq_weights* w,
                     const aq_train_config* cfg, aq_codebook** cb_out,
                     aq_codes** codes_out, double* loss_history_out,
                     size_t* history_len);

/* ---- host-pointer forms (the reference's by-value semantics) ------------- */
/* adc_search over nq queries: ids/scores nq x min(topn, n) */
int aq_adc_search_batch(aq_session* s, const double* queries, size_t nq, size_t d,
                        const uint32_t* codes, size_t n, size_t M, size_t codes_k,
                        const double* dictionaries, size_t cb_M, size_t k,
                        size_t sub_dimension, size_t topn, uint32_t* ids_out,
                        double* scores_out);
/* exact-dot rerank of ncand candidates per query, keep min(keep, ncand) */
int aq_rerank(aq_session* s, const double* queries, size_t nq, const float* x,
              size_t n, size_t d, const uint32_t* cand_ids, size_t ncand,
              size_t keep, uint32_t* ids_out, double* scores_out);
/* exact_ground_truth: exact top-min(depth, n) per query */
int aq_exact_search_batch(aq_session* s, const double* queries, size_t nq,
                          const float* x, size_t n, size_t d, size_t depth,
                          uint32_t* ids_out, double* scores_out);
/* assemble_selector_system: A_out (k d)^2 row-major, rhs_out k d */
int aq_assemble_selector_system(aq_session* s, const float* x, size_t n, size_t d,
                                const uint32_t* codes, size_t M, size_t k,
                                const aq_weights* w, double* A_out, double* rhs_out);
/* train_l2_pq / train_apq: dictionaries M k (d / M) float64, codes n x M */
int aq_train_l2_pq(aq_session* s, const float* x, size_t n, size_t d, size_t M,
                   size_t k, const aq_train_config* cfg, double* dictionaries_out,
                   uint32_t* codes_out);
int aq_train_apq(aq_session* s, const float* x, size_t n, size_t d, size_t M, size_t k,
                 const aq_weights* w, const aq_train_config* cfg, int warm_start,
                 double* dictionaries_out, uint32_t* codes_out,
                 double* loss_history_out, size_t* history_len);
/* train_avq: codewords_out k x d, assignments_out n, history <= max_iterations + 1 */
int aq_train_avq(aq_session* s, const float* x, size_t n, size_t d, size_t k,
                 const aq_weights* w, const aq_train_config* cfg, double* codewords_out,
                 uint32_t* assignments_out, double* loss_history_out, size_t* history_len);

/* ---- row-sharded training building blocks (multi-GPU) -----
 * The reference trains in one process (pq.hpp:513-575); a sharded trainer
 * splits its sums by rows: every rank computes the partial quantities below
 * on its own shard, the host combines them across ranks in rank order
 * (paper_1908_10396_b200/distributed.py) and every rank solves the same
 * system. Buffers ending in _dev are device pointers on the session's GPU. */

/* flags of this shard's weights: flags_out[0] = some point anisotropic (the
 * dense path, pq.hpp:383-386), flags_out[1] = first anisotropic |x| = 0 point
 * + 1 (0 = none) */
int aq_dev_weight_flags(aq_dataset* ds, const aq_weights* w, uint64_t* flags_out);
/* pq.hpp:290-343 on this shard: lower triangle of A (k d x k d) and rhs,
 * usage[m][j] = points with code j at subspace m. flags_out[0] = some point is
 * anisotropic; flags_out[1] = first anisotropic |x| = 0 point + 1 (0 = none). */
int aq_dev_normal_equations_partial(aq_dataset* ds, aq_codes* codes,
                                    const aq_weights* w, size_t k, double* A_dev,
                                    double* rhs_dev, uint32_t* usage_dev,
                                    uint64_t* flags_out);
/* pq.hpp:405-417 on this shard: num[m][j][c] = sum h_par x_c, den[m][j] =
 * sum h_perp over the members in ascending order. */
int aq_dev_iso_partials(aq_dataset* ds, aq_codes* codes, const aq_weights* w,
                        size_t k, double* num_dev, double* den_dev,
                        uint32_t* usage_dev);
/* pq.hpp:430-443: ridge (ridge < 0 -> 1e-6 trace / dim), Cholesky, solve, in
 * place (A -> L, rhs -> solution). AQ_E_SINGULAR_SYSTEM when not SPD. */
int aq_dev_solve_normal_equations(aq_session* s, double* A_dev, double* rhs_dev,
                                  size_t dim, double ridge);
/* replace a codebook's dictionaries from device memory */
int aq_codebook_set_device(aq_codebook* cb, const double* dict_dev);
/* pq_point_loss (pq.hpp:137-146) of every point of this shard */
int aq_dev_point_losses(aq_dataset* ds, aq_codebook* cb, const aq_weights* w,
                        aq_codes* codes, double* losses_dev);
/* loss_ranking order (vq.hpp:221-229): idx_dev (ascending on entry) sorted
 * by (score desc, idx asc) */
int aq_dev_sort_desc(aq_session* s, const double* scores_dev, uint32_t* idx_dev,
                     size_t n);
/* std::accumulate(v, v + n, init) in index order */
int aq_dev_seq_sum(aq_session* s, const double* v_dev, size_t n, double init,
                   double* out);
/* `rows` such sums in one launch (row r at v_dev + r * ld, `count` values);
 * rows with active_host[r] == 0 (active_host may be NULL) give 0 */
int aq_dev_seq_sums(aq_session* s, const double* v_dev, size_t ld, size_t count,
                    size_t rows, const int* active_host, double* out_host);
/* vq_assign_pass (vq.hpp:196-217) with unit weights for the active subspaces
 * of this shard: codes in place, losses_dev (M x n), changes_out[M] */
int aq_dev_kmeans_assign(aq_dataset* ds, aq_codebook* cb, aq_codes* codes,
                         const int* active_host, double* losses_dev,
                         uint64_t* changes_out);
/* update_codeword unit-weight sums (vq.hpp:151-162) on this shard for the
 * active subspaces: num (M k sd), den (M k), count (M k) */
int aq_dev_kmeans_partials(aq_dataset* ds, aq_codes* codes, size_t k,
                           const int* active_host, double* num_dev, double* den_dev,
                           uint32_t* count_dev);

/* ---- multi-device session (one process, the GPUs of one box) ----------
 * The database shards by contiguous rows over `count` sessions, one per
 * entry of `devices` (a device may appear more than once: several shards on
 * one GPU). Exchanges are device-to-device copies over NVLink, summed in shard
 * order. Results depend only on the shard count:
 *   aq_multi_pq_quantize, aq_multi_adc_search: equal to the single-device
 *     calls (pq_quantize pq.hpp:581-612, adc_search index.hpp:118-134);
 *   aq_multi_train_apq (pq.hpp:513-575): one shard = the single-device
 *     trainer bit for bit; W shards re-associate the float64 partial sums at
 *     W - 1 shard boundaries. M == 1 and sub_dimension > 16 run on shard 0. */
typedef struct aq_multi aq_multi;
/* number of visible CUDA devices */
int aq_device_count(int* count);
int aq_multi_create(const int* devices, int count, aq_multi** out);
int aq_multi_destroy(aq_multi* m);
int aq_multi_shards(const aq_multi* m);
aq_session* aq_multi_session(aq_multi* m, int shard);
int aq_multi_pq_quantize(aq_multi* m, const float* x, size_t n, size_t d,
                         const double* dictionaries, size_t M, size_t k,
                         size_t sub_dimension, const aq_weights* w, int passes,
                         uint32_t* codes_out);
/* ids_out / scores_out: nq x min(topn, n), (score desc, index asc) */
int aq_multi_adc_search(aq_multi* m, const double* queries, size_t nq, size_t d,
                        const uint32_t* codes, size_t n, size_t codes_M,
                        size_t codes_k, const double* dictionaries, size_t cb_M,
                        size_t k, size_t sub_dimension, size_t topn,
                        uint32_t* ids_out, double* scores_out);
int aq_multi_train_apq(aq_multi* m, const float* x, size_t n, size_t d, size_t M,
                       size_t k, const aq_weights* w, const aq_train_config* cfg,
                       int warm_start, double* dictionaries_out, uint32_t* codes_out,
                       double* loss_history_out, size_t* history_len);

#ifdef __cplusplus
}
#endif
#endif /* ANISOQ_B200_H_ */
