// Host-pointer entry points: the reference's by-value semantics (inputs in,
// owning outputs back) built from the device-resident API. Validation order
// follows the reference function each one replaces.
#include <algorithm>
#include <cstring>
#include <emmintrin.h>
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

// memcpy-bound host loop split over up to `nt` threads: f(begin, end)
template <class F>
void parallel_rows(size_t rows, size_t nt, F f) {
  nt = std::max<size_t>(1, std::min(nt, rows / 1024 + 1));
  if (nt <= 1) {
    f(0, rows);
    return;
  }
  const size_t per = (rows + nt - 1) / nt;
  std::vector<std::thread> th;
  for (size_t t = 1; t < nt; ++t) {
    const size_t b = t * per;
    if (b >= rows) break;
    th.emplace_back([=] { f(b, std::min(rows, b + per)); });
  }
  f(0, std::min(per, rows));
  for (auto& t : th) t.join();
}

// pq_quantize over host rows in chunks, three stages in flight:
//   host     copies chunk i's rows into page-locked staging (every host
//            thread) while a second thread group unpacks chunk i - 2's 4-bit
//            codes from staging into codes_out;
//   up       H2D of chunk i on its own stream;
//   compute  tiles and encodes chunk i - 1, then its packed codes (M/2 bytes
//            per row, 8x fewer than uint32) go D2H on a third stream.
// Buffers (page-locked, device rows, tiled datasets, packed codes) are a ring
// of three, allocated once per call. Page-locked caller buffers skip the host
// side: rows go H2D straight from `x`, and the codes are widened to uint32 on
// the device and go D2H straight into `codes_out` (the copy engines then
// carry both directions at once and no host thread touches the data).
// Points are independent
// (pq.hpp:581-612), so the codes equal the single-shot call's; device errors
// carry global point indices and are checked once at the end.
int pq_quantize_streamed(aq_session* s, const float* x, size_t n, size_t d, aq_codebook* cb,
                         const aq_weights* w, int passes, uint32_t* codes_out, size_t chunk) {
  constexpr int NB = 3;
  const size_t M = cb->M;
  const int bits = cb->k <= 16 ? 4 : 8;
  const size_t stride = code_stride(M, bits);
  const size_t nt = std::max(1u, std::thread::hardware_concurrency());
  auto page_locked = [](const void* p) {
    cudaPointerAttributes at;
    const bool pl = cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();  // a pageable pointer may leave an error behind on older drivers
    return pl;
  };
  const bool pin_in = page_locked(x) && page_locked(x + n * d - 1);
  const bool pin_out = page_locked(codes_out) && page_locked(codes_out + n * M - 1);
  void* hin[NB] = {};
  void* hout[NB] = {};
  uint32_t* du[NB] = {};  // device uint32 codes (page-locked codes_out only)
  for (int b = 0; b < NB; ++b) {
    if (!pin_in) AQ_TRY(pinned_buffer(s, b, chunk * d * sizeof(float), &hin[b]));
    if (!pin_out) AQ_TRY(pinned_buffer(s, NB + b, chunk * stride, &hout[b]));
  }
  cudaStream_t up = nullptr, down = nullptr;
  float* dx[NB] = {};
  aq_dataset ds[NB];
  aq_codes* cc[NB] = {};
  cudaEvent_t ev_up[NB] = {}, ev_enc[NB] = {}, ev_down[NB] = {};
  int st = AQ_OK;
  if (cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking) != cudaSuccess)
    st = ref_error(AQ_E_CUDA, "stream creation failed");
  for (int b = 0; b < NB && st == AQ_OK; ++b) {
    ds[b].s = s;
    ds[b].d = d;
    if (cudaMalloc(&dx[b], chunk * d * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&ds[b].xt, (tiled_floats(chunk, d) + 256) * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&ds[b].norms, chunk * sizeof(double)) != cudaSuccess ||
        cudaMemset(ds[b].xt + tiled_floats(chunk, d), 0, 256 * sizeof(float)) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_up[b], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_enc[b], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_down[b], cudaEventDisableTiming) != cudaSuccess ||
        (pin_out && cudaMalloc(&du[b], chunk * M * sizeof(uint32_t)) != cudaSuccess))
      st = ref_error(AQ_E_CUDA, "out of device memory for the streamed encode");
    if (st == AQ_OK) st = aq_codes_alloc(s, chunk, M, cb->k, &cc[b]);
  }
  if (st == AQ_OK) st = clear_dev_error(s);
  const size_t nch = (n + chunk - 1) / chunk;
  auto rows_of = [&](size_t i) { return std::min(chunk, n - i * chunk); };
  auto unpack = [&](size_t k) {  // chunk k: staging (packed) -> codes_out (uint32)
    const int b = (int)(k % NB);
    const size_t cn = rows_of(k);
    const uint8_t* src = static_cast<const uint8_t*>(hout[b]);
    uint32_t* dst = codes_out + k * chunk * M;
    parallel_rows(cn, std::max<size_t>(1, nt / 2), [&](size_t r0, size_t r1) {
      // 4-bit codes, M % 16 == 0, 16-byte aligned rows: sixteen codes per step
      // (SSE2 nibble split + widening) with non-temporal stores (the 4-byte
      // output is never read back here, so no read-for-ownership traffic)
      const bool vec = bits == 4 && M % 16 == 0 &&
                       ((reinterpret_cast<uintptr_t>(dst) | (M * 4)) & 15) == 0;
      const __m128i nib = _mm_set1_epi8(0x0F), z = _mm_setzero_si128();
      for (size_t r = r0; r < r1; ++r) {
        const uint8_t* row = src + r * stride;
        uint32_t* o = dst + r * M;
        if (vec) {
          for (size_t m = 0; m < M; m += 16) {
            const __m128i b = _mm_loadl_epi64(reinterpret_cast<const __m128i*>(row + m / 2));
            const __m128i lo = _mm_and_si128(b, nib);
            const __m128i hi = _mm_and_si128(_mm_srli_epi16(b, 4), nib);
            const __m128i c8 = _mm_unpacklo_epi8(lo, hi);  // codes m .. m + 15 as bytes
            const __m128i w0 = _mm_unpacklo_epi8(c8, z), w1 = _mm_unpackhi_epi8(c8, z);
            __m128i* out = reinterpret_cast<__m128i*>(o + m);
            _mm_stream_si128(out, _mm_unpacklo_epi16(w0, z));
            _mm_stream_si128(out + 1, _mm_unpackhi_epi16(w0, z));
            _mm_stream_si128(out + 2, _mm_unpacklo_epi16(w1, z));
            _mm_stream_si128(out + 3, _mm_unpackhi_epi16(w1, z));
          }
        } else if (bits == 4) {
          for (size_t m = 0; m < M; ++m) o[m] = (row[m >> 1] >> ((m & 1) * 4)) & 15u;
        } else {
          for (size_t m = 0; m < M; ++m) o[m] = row[m];
        }
      }
      _mm_sfence();
    });
  };
  for (size_t i = 0; i < nch + 2 && st == AQ_OK; ++i) {
    std::thread unpacker;
    if (i >= 2 && !pin_out) {  // chunk i - 2's codes, concurrently with chunk i's copy-in
      const size_t k = i - 2;
      if (cudaEventSynchronize(ev_down[k % NB]) != cudaSuccess) {
        st = ref_error(AQ_E_CUDA, "streamed encode failed");
        break;
      }
      unpacker = std::thread(unpack, k);
    }
    if (i < nch) {  // chunk i: host staging, then H2D on `up`
      const int b = (int)(i % NB);
      const size_t cn = rows_of(i);
      const float* src = x + i * chunk * d;
      if (!pin_in) {
        if (i >= NB) cudaEventSynchronize(ev_up[b]);  // staging slot b is free again
        float* dst = static_cast<float*>(hin[b]);
        parallel_rows(cn, std::max<size_t>(1, i >= 2 ? nt / 2 : nt), [&](size_t r0, size_t r1) {
          std::memcpy(dst + r0 * d, src + r0 * d, (r1 - r0) * d * sizeof(float));
        });
      }
      if (i >= NB) cudaStreamWaitEvent(up, ev_enc[b], 0);  // dx[b] read by chunk i - 3
      if (cudaMemcpyAsync(dx[b], pin_in ? src : hin[b], cn * d * sizeof(float),
                          cudaMemcpyHostToDevice, up) !=
              cudaSuccess ||
          cudaEventRecord(ev_up[b], up) != cudaSuccess)
        st = ref_error(AQ_E_CUDA, "streamed encode upload failed");
    }
    if (st == AQ_OK && i >= 1 && i - 1 < nch) {  // chunk i - 1: tile + encode, then D2H
      const size_t j = i - 1;
      const int b = (int)(j % NB);
      const size_t cn = rows_of(j);
      cudaStreamWaitEvent(s->stream, ev_up[b], 0);
      if (j >= NB) cudaStreamWaitEvent(s->stream, ev_down[b], 0);  // cc[b] downloaded
      ds[b].n = cn;
      ds[b].xr = dx[b];
      cc[b]->n = cn;
      st = tile_rows_async(dx[b], cn, d, ds[b].xt, ds[b].norms, s->stream);
      if (st == AQ_OK) st = run_encode_chunk(&ds[b], cb, w, cc[b], passes, j * chunk);
      if (st == AQ_OK && pin_out) st = codes_unpack_async(cc[b], du[b]);
      if (st == AQ_OK && (cudaEventRecord(ev_enc[b], s->stream) != cudaSuccess ||
                          cudaStreamWaitEvent(down, ev_enc[b], 0) != cudaSuccess ||
                          (pin_out ? cudaMemcpyAsync(codes_out + j * chunk * M, du[b],
                                                     cn * M * sizeof(uint32_t),
                                                     cudaMemcpyDeviceToHost, down)
                                   : cudaMemcpyAsync(hout[b], cc[b]->data, cn * stride,
                                                     cudaMemcpyDeviceToHost, down)) != cudaSuccess ||
                          cudaEventRecord(ev_down[b], down) != cudaSuccess))
        st = ref_error(AQ_E_CUDA, "streamed encode download failed");
    }
    if (unpacker.joinable()) unpacker.join();
  }
  const int fin = sync_and_check(s, "encode");
  if (st == AQ_OK) st = fin;
  if (up) cudaStreamSynchronize(up);
  if (down) cudaStreamSynchronize(down);
  for (int b = 0; b < NB; ++b) {
    if (cc[b]) {
      cc[b]->n = chunk;
      aq_codes_free(cc[b]);
    }
    cudaFree(dx[b]);
    cudaFree(du[b]);
    cudaFree(ds[b].xt);
    cudaFree(ds[b].norms);
    ds[b].xt = nullptr;
    ds[b].norms = nullptr;
    ds[b].xr = nullptr;
    if (ev_up[b]) cudaEventDestroy(ev_up[b]);
    if (ev_enc[b]) cudaEventDestroy(ev_enc[b]);
    if (ev_down[b]) cudaEventDestroy(ev_down[b]);
  }
  if (up) cudaStreamDestroy(up);
  if (down) cudaStreamDestroy(down);
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
