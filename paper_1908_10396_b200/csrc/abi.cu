// Host-pointer entry points: the reference's by-value semantics (inputs in,
// owning outputs back) built from the device-resident API. Validation order
// follows the reference function each one replaces.
#include <memory>
#include <vector>

#include "common.cuh"

using namespace aqd;

namespace {

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

}  // extern "C"
