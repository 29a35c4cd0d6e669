// Host-pointer entry points: the reference's by-value semantics (inputs in,
// owning outputs back) built from the device-resident API. Validation order
// follows the reference function each one replaces.
#include <algorithm>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "common.cuh"

namespace aqd {
int run_encode_chunk(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes,
                     int passes, size_t base);
int codes_unpack_async(aq_codes* c, uint32_t* dev_out);
int pinned_buffer(aq_session* s, int slot, size_t bytes, void** out);
int clear_dev_error(aq_session* s);
int sync_and_check(aq_session* s, const char* what);
}  // namespace aqd

using namespace aqd;

namespace {

// memcpy split over up to 8 host threads (pageable <-> page-locked staging)
void parallel_copy(void* dst, const void* src, size_t bytes) {
  constexpr size_t kPiece = size_t(16) << 20;
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>({8, hw, (bytes + kPiece - 1) / kPiece});
  if (nt <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes + nt - 1) / nt;
  std::vector<std::thread> th;
  for (size_t t = 1; t < nt; ++t) {
    const size_t b = t * per;
    if (b >= bytes) break;
    const size_t e = std::min(bytes, b + per);
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
    });
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

// pq_quantize over host rows in chunks: the host copies chunk i + 1 into
// page-locked staging (and chunk i - 1's codes out of it) while the device
// uploads, tiles, encodes and unpacks chunk i. Points are independent
// (pq.hpp:581-612), so the codes equal the single-shot call's; device errors
// carry global point indices and are checked once at the end.
int pq_quantize_streamed(aq_session* s, const float* x, size_t n, size_t d, aq_codebook* cb,
                         const aq_weights* w, int passes, uint32_t* codes_out, size_t chunk) {
  const size_t M = cb->M;
  void* hin[2];
  void* hout[2];
  for (int b = 0; b < 2; ++b) {
    AQ_TRY(pinned_buffer(s, b, chunk * d * sizeof(float), &hin[b]));
    AQ_TRY(pinned_buffer(s, 2 + b, chunk * M * sizeof(uint32_t), &hout[b]));
  }
  float* dx[2] = {nullptr, nullptr};
  uint32_t* dcodes[2] = {nullptr, nullptr};
  cudaEvent_t h2d[2] = {nullptr, nullptr}, d2h[2] = {nullptr, nullptr};
  int st = AQ_OK;
  for (int b = 0; b < 2 && st == AQ_OK; ++b) {
    if (cudaMallocAsync(&dx[b], chunk * d * sizeof(float), s->stream) != cudaSuccess ||
        cudaMallocAsync(&dcodes[b], chunk * M * sizeof(uint32_t), s->stream) != cudaSuccess ||
        cudaEventCreateWithFlags(&h2d[b], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d2h[b], cudaEventDisableTiming) != cudaSuccess)
      st = ref_error(AQ_E_CUDA, "out of device memory for the streamed encode");
  }
  if (st == AQ_OK) st = clear_dev_error(s);
  const size_t nch = (n + chunk - 1) / chunk;
  for (size_t i = 0; i <= nch && st == AQ_OK; ++i) {
    if (i < nch) {
      const int b = (int)(i & 1);
      const size_t off = i * chunk, cn = std::min(chunk, n - off);
      if (i >= 2) cudaEventSynchronize(h2d[b]);  // staging slot b is free again
      parallel_copy(hin[b], x + off * d, cn * d * sizeof(float));
      if (cudaMemcpyAsync(dx[b], hin[b], cn * d * sizeof(float), cudaMemcpyHostToDevice,
                          s->stream) != cudaSuccess ||
          cudaEventRecord(h2d[b], s->stream) != cudaSuccess) {
        st = AQ_E_CUDA;
        break;
      }
      aq_dataset* ds = nullptr;
      aq_codes* cc = nullptr;
      st = aq_dataset_wrap_device(s, dx[b], cn, d, &ds);
      if (st == AQ_OK) st = aq_codes_alloc(s, cn, M, cb->k, &cc);
      if (st == AQ_OK) st = run_encode_chunk(ds, cb, w, cc, passes, off);
      if (st == AQ_OK) st = codes_unpack_async(cc, dcodes[b]);
      if (st == AQ_OK &&
          (cudaMemcpyAsync(hout[b], dcodes[b], cn * M * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
           cudaEventRecord(d2h[b], s->stream) != cudaSuccess))
        st = AQ_E_CUDA;
      aq_codes_free(cc);
      aq_dataset_free(ds);
      if (st != AQ_OK) break;
    }
    if (i >= 1) {  // chunk i - 1's codes, while the device works on chunk i
      const size_t j = i - 1, off = j * chunk, cn = std::min(chunk, n - off);
      const int b = (int)(j & 1);
      cudaEventSynchronize(d2h[b]);
      parallel_copy(codes_out + off * M, hout[b], cn * M * sizeof(uint32_t));
    }
  }
  const int fin = sync_and_check(s, "encode");
  if (st == AQ_OK) st = fin;
  for (int b = 0; b < 2; ++b) {
    if (dx[b]) cudaFreeAsync(dx[b], s->stream);
    if (dcodes[b]) cudaFreeAsync(dcodes[b], s->stream);
    if (h2d[b]) cudaEventDestroy(h2d[b]);
    if (d2h[b]) cudaEventDestroy(d2h[b]);
  }
  return st;
}

struct DsGuard {
  aq_dataset* p = nullptr;
  ~DsGuard() { aq_dataset_free(p); }
};
struct CbGuard {
  aq_codebook* p = nullptr;
  ~CbGuard() { aq_codebook_free(p); }
};
struct CodesGuard {
  aq_codes* p = nullptr;
  ~CodesGuard() { aq_codes_free(p); }
};

}  // namespace

extern "C" {

// pq_quantize (pq.hpp:581-612)
int aq_pq_quantize(aq_session* s, const float* x, size_t n, size_t d,
                   const double* dict, size_t M, size_t k, size_t sd,
                   const aq_weights* w, int passes, uint32_t* codes_out) {
  AQ_TRY(check_session(s));
  if (d != M * sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH,
                     "dataset dimension does not match codebook");
  if (passes < 0) return ref_error(AQ_E_INVALID_ARGUMENT, "passes must be >= 0");
  DsGuard ds;
  CbGuard cb;
  CodesGuard codes;
  // large host datasets: chunked, copies overlapped with the device work
  // (uniform / threshold weights; per-point arrays take the single-shot path)
  size_t chunk = std::max<size_t>(1024, (size_t(128) << 20) / (d * sizeof(float)));
  if (const char* e = getenv("AQ_STREAM_CHUNK")) chunk = std::max<size_t>(1, strtoull(e, nullptr, 10));
  if (w && w->mode != AQ_WEIGHTS_PER_POINT && n >= 4 * chunk && k <= 256 && k > 0) {
    AQ_TRY(aq_codebook_upload(s, dict, M, k, sd, &cb.p));
    return pq_quantize_streamed(s, x, n, d, cb.p, w, passes, codes_out, chunk);
  }
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  AQ_TRY(aq_codebook_upload(s, dict, M, k, sd, &cb.p));
  AQ_TRY(aq_codes_alloc(s, n, M, k, &codes.p));
  AQ_TRY(aq_dev_pq_quantize(ds.p, cb.p, w, passes, codes.p));
  return aq_codes_download(codes.p, codes_out);
}

// detail::pq_assign_pass (pq.hpp:202-221)
int aq_pq_assign_pass(aq_session* s, const float* x, size_t n, size_t d,
                      const double* dict, size_t M, size_t k, size_t sd,
                      const aq_weights* w, int sweep_to_fixed_point,
                      uint32_t* codes_inout, double* losses_out) {
  AQ_TRY(check_session(s));
  if (d != M * sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH,
                     "dataset dimension does not match codebook");
  DsGuard ds;
  CbGuard cb;
  CodesGuard codes;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  AQ_TRY(aq_codebook_upload(s, dict, M, k, sd, &cb.p));
  AQ_TRY(aq_codes_upload(s, codes_inout, n, M, k, &codes.p));
  double* losses = nullptr;
  if (n) AQ_CUDA(cudaMallocAsync(&losses, n * sizeof(double), s->stream));
  uint64_t changed = 0;
  int st = aq_dev_pq_assign_pass(ds.p, cb.p, w, sweep_to_fixed_point, codes.p,
                                 losses, &changed);
  if (st == AQ_OK && n) {
    if (losses_out) {
      cudaError_t e = cudaMemcpyAsync(losses_out, losses, n * sizeof(double),
                                      cudaMemcpyDeviceToHost, s->stream);
      if (e != cudaSuccess) st = AQ_E_CUDA;
    }
    if (st == AQ_OK) st = aq_codes_download(codes.p, codes_inout);
  }
  if (losses) cudaFreeAsync(losses, s->stream);
  cudaStreamSynchronize(s->stream);
  return st;
}

// adc_search over a query batch (index.hpp:118-134 per query; evaluate runs
// it per query, index.hpp:251-259): ids/scores nq x min(topn, n).
int aq_adc_search_batch(aq_session* s, const double* queries, size_t nq, size_t d,
                        const uint32_t* codes, size_t n, size_t M, size_t codes_k,
                        const double* dict, size_t cb_M, size_t k, size_t sd, size_t topn,
                        uint32_t* ids_out, double* scores_out) {
  AQ_TRY(check_session(s));
  if (n == 0) return ref_error(AQ_E_EMPTY_INDEX, "no quantized datapoints");
  if (topn < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  if (M != cb_M || codes_k > k)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match codebook");
  if (d != cb_M * sd)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "query dimension does not match codebook");
  CbGuard cb;
  CodesGuard cm;
  AQ_TRY(aq_codebook_upload(s, dict, cb_M, k, sd, &cb.p));
  AQ_TRY(aq_codes_upload(s, codes, n, M, std::max<size_t>(codes_k, 1), &cm.p));
  return aq_dev_adc_search(cm.p, cb.p, queries, nq, topn, ids_out, scores_out);
}

// exact-dot rerank of candidate lists (north_star), host pointers.
int aq_rerank(aq_session* s, const double* queries, size_t nq, const float* x, size_t n,
              size_t d, const uint32_t* cand_ids, size_t ncand, size_t keep,
              uint32_t* ids_out, double* scores_out) {
  AQ_TRY(check_session(s));
  DsGuard ds;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  return aq_dev_rerank(ds.p, queries, nq, cand_ids, ncand, keep, ids_out, scores_out);
}

// exact_ground_truth (index.hpp:150-162): exact top-`depth` per query.
int aq_exact_search_batch(aq_session* s, const double* queries, size_t nq, const float* x,
                          size_t n, size_t d, size_t depth, uint32_t* ids_out,
                          double* scores_out) {
  AQ_TRY(check_session(s));
  DsGuard ds;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  return aq_dev_exact_search(ds.p, queries, nq, depth, ids_out, scores_out);
}

// assemble_selector_system (pq.hpp:290-343): full (k d)^2 matrix row-major.
int aq_assemble_selector_system(aq_session* s, const float* x, size_t n, size_t d,
                                const uint32_t* codes, size_t M, size_t k,
                                const aq_weights* w, double* A_out, double* rhs_out) {
  AQ_TRY(check_session(s));
  if (M == 0 || d % M != 0)
    return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  DsGuard ds;
  CodesGuard cm;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  AQ_TRY(aq_codes_upload(s, codes, n, M, k, &cm.p));
  return aq_dev_assemble_selector_system(ds.p, cm.p, w, A_out, rhs_out);
}

// train_l2_pq (pq.hpp:469-501): dictionaries M k (d / M), codes n x M.
int aq_train_l2_pq(aq_session* s, const float* x, size_t n, size_t d, size_t M, size_t k,
                   const aq_train_config* cfg, double* dict_out, uint32_t* codes_out) {
  AQ_TRY(check_session(s));
  DsGuard ds;
  CbGuard cb;
  CodesGuard cm;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  AQ_TRY(aq_dev_train_l2_pq(ds.p, M, k, cfg, &cb.p, &cm.p));
  AQ_TRY(aq_codebook_download(cb.p, dict_out));
  return aq_codes_download(cm.p, codes_out);
}

// train_apq (pq.hpp:513-575); history_out holds max_iterations + 1 values.
int aq_train_apq(aq_session* s, const float* x, size_t n, size_t d, size_t M, size_t k,
                 const aq_weights* w, const aq_train_config* cfg, int warm_start,
                 double* dict_out, uint32_t* codes_out, double* history_out,
                 size_t* history_len) {
  AQ_TRY(check_session(s));
  DsGuard ds;
  CbGuard cb;
  CodesGuard cm;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  AQ_TRY(aq_dev_train_apq(ds.p, M, k, w, cfg, warm_start, &cb.p, &cm.p, history_out,
                          history_len));
  AQ_TRY(aq_codebook_download(cb.p, dict_out));
  return aq_codes_download(cm.p, codes_out);
}

int aq_train_avq(aq_session* s, const float* x, size_t n, size_t d, size_t k,
                 const aq_weights* w, const aq_train_config* cfg, double* cw_out,
                 uint32_t* assign_out, double* history_out, size_t* history_len) {
  AQ_TRY(check_session(s));
  DsGuard ds;
  CbGuard cb;
  CodesGuard cm;
  AQ_TRY(aq_dataset_upload(s, x, n, d, &ds.p));
  AQ_TRY(aq_dev_train_avq(ds.p, k, w, cfg, &cb.p, &cm.p, history_out, history_len));
  AQ_TRY(aq_codebook_download(cb.p, cw_out));
  return aq_codes_download(cm.p, assign_out);
}

}  // extern "C"
