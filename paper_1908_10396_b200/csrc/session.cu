// Sessions, device-resident objects, layouts, weights and error plumbing.
#include <algorithm>
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace aqd {

static thread_local char g_msg[1024];

static const char* kRefNames[] = {
    "Ok",               "InvalidArgument",   "ZeroNormDatapoint",
    "InvalidThreshold", "EmptyDataset",      "EmptyIndex",
    "DimensionMismatch", "DimensionNotDivisible", "CodeOutOfRange",
    "MalformedFile",    "InsufficientData",  "GroundTruthMismatch",
    "QuadratureFailure", "SingularSystem"};

const char* status_ref_name(int status) {
  if (status >= 0 && status <= 13) return kRefNames[status];
  if (status == AQ_E_CUDA) return "CudaError";
  if (status == AQ_E_UNSUPPORTED) return "Unsupported";
  return "Unknown";
}

void set_error(int status, const char* fmt, ...) {
  (void)status;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_msg, sizeof g_msg, fmt, ap);
  va_end(ap);
}

int ref_error(int status, const char* detail) {
  set_error(status, "%s: %s", status_ref_name(status), detail);
  return status;
}

int check_session(aq_session* s) {
  if (!s) return ref_error(AQ_E_INVALID_ARGUMENT, "null session");
  AQ_CUDA(cudaSetDevice(s->device));
  return AQ_OK;
}

int scratch(aq_session* s, int slot, size_t bytes, void** out) {
  Scratch& sc = s->scratch[slot];
  if (sc.bytes < bytes) {
    if (sc.p) AQ_CUDA(cudaFreeAsync(sc.p, s->stream));
    size_t want = bytes + bytes / 4 + 256;
    AQ_CUDA(cudaMallocAsync(&sc.p, want, s->stream));
    sc.bytes = want;
  }
  *out = sc.p;
  return AQ_OK;
}

// Page-locked host buffer `slot`, grown on demand and kept for the session.
int pinned_buffer(aq_session* s, int slot, size_t bytes, void** out) {
  Scratch& sc = s->pinned[slot];
  if (sc.bytes < bytes) {
    if (sc.p) {
      AQ_CUDA(cudaStreamSynchronize(s->stream));
      AQ_CUDA(cudaFreeHost(sc.p));
      sc.p = nullptr;
      sc.bytes = 0;
    }
    AQ_CUDA(cudaHostAlloc(&sc.p, bytes, cudaHostAllocDefault));
    sc.bytes = bytes;
  }
  *out = sc.p;
  return AQ_OK;
}

void timer_mark(aq_session* s, int slot) {
  if (!s->timing) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, s->stream);
  s->tev[slot].push_back(e);
}

int clear_dev_error(aq_session* s) {
  AQ_CUDA(cudaMemsetAsync(s->err, 0xff, sizeof(DevError), s->stream));
  return AQ_OK;
}

static const char* kDevErrDetail[] = {
    "", "invalid argument", "anisotropic loss undefined at |x| = 0",
    "need 0 <= T < norm", "", "", "", "", "code out of range", "", "", "",
    "", "system is not positive definite"};

int sync_and_check(aq_session* s, const char* what) {
  AQ_CUDA(cudaMemcpyAsync(s->err_host, s->err, sizeof(DevError),
                          cudaMemcpyDeviceToHost, s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  const unsigned long long key = s->err_host->key;
  if (key != ~0ull) {
    const int st = (int)(key & 0xff);
    const unsigned long long idx = key >> 8;
    char buf[256];
    snprintf(buf, sizeof buf, "%s (%s, point %llu)",
             st < 14 ? kDevErrDetail[st] : "device error", what, idx);
    return ref_error(st, buf);
  }
  return AQ_OK;
}

// ---- kernels ------------------------------------------------------------------

// Row-major fp32 -> pair-tiled layout, and float64 norms in the reference's
// order (dataset.hpp:55-59). One thread per row for the norm; the tiled write
// of a 32-row tile is coalesced because lanes own consecutive rows.
template <class T>
__global__ void k_tile_rows(const T* __restrict__ x, size_t n, size_t d,
                            T* __restrict__ xt, double* __restrict__ norms) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t pairs = pairs_of(d);
  const size_t ntile = ((n + 31) / 32) * 32;
  if (i >= ntile) return;
  double s = 0.0;
  for (size_t j = 0; j < 2 * pairs; ++j) {
    T v = 0;
    if (i < n && j < d) v = x[i * d + j];
    xt[tiled_index(i, j, pairs)] = v;
    if (j < d) s = __dadd_rn(s, __dmul_rn((double)v, (double)v));
  }
  if (i < n) norms[i] = __dsqrt_rn(s);
}

// Pair-tiles n float32 rows (device) into an existing dataset's xt / norms on
// `stream` (the streamed host-pointer encode reuses one dataset per buffer).
int tile_rows_async(const float* xdev, size_t n, size_t d, float* xt, double* norms,
                    cudaStream_t stream) {
  const size_t ntile = ((n + 31) / 32) * 32;
  if (ntile)
    k_tile_rows<float><<<(unsigned)((ntile + 127) / 128), 128, 0, stream>>>(xdev, n, d, xt, norms);
  AQ_CUDA(cudaGetLastError());
  return AQ_OK;
}

// float32 staging of an sd == 2 codebook for the filter kernels:
// {c0, c1, c0^2 + c1^2} per (m, j); slots j >= k are padded with a huge C so
// they never win and never look like a near tie. rmax[m] bounds |c_mj| from
// above (rounded up) for the error budgets.
__global__ void k_stage_codebook2(const double* __restrict__ cb, int M, int k,
                                  float4* __restrict__ f32,
                                  float* __restrict__ rmax) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  float r = 0.0f;
  for (int j = 0; j < 16; ++j) {
    float4 v;
    if (j < k) {
      const float c0 = (float)cb[(m * k + j) * 2];
      const float c1 = (float)cb[(m * k + j) * 2 + 1];
      v = make_float4(c0, c1, __fmaf_rn(c1, c1, c0 * c0), 0.0f);
      const double nn = sqrt(cb[(m * k + j) * 2] * cb[(m * k + j) * 2] +
                             cb[(m * k + j) * 2 + 1] * cb[(m * k + j) * 2 + 1]);
      r = fmaxf(r, __double2float_ru(nn * (1.0 + 1e-12)));
    } else {
      v = make_float4(0.0f, 0.0f, 1e30f, 0.0f);
    }
    f32[m * 16 + j] = v;
  }
  rmax[m] = r;
}

__global__ void k_pack_codes(const uint32_t* __restrict__ in, size_t n,
                             size_t M, int bits, size_t stride,
                             uint8_t* __restrict__ out,
                             DevError* err, uint32_t k) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t* row = out + i * stride;
  for (size_t b = 0; b < stride; ++b) row[b] = 0;
  for (size_t m = 0; m < M; ++m) {
    const uint32_t c = in[i * M + m];
    if (c >= k) report_error(err, i * M + m, AQ_E_CODE_OUT_OF_RANGE);
    if (bits == 4)
      row[m >> 1] |= (uint8_t)((c & 15u) << ((m & 1) * 4));
    else
      row[m] = (uint8_t)c;
  }
}

__global__ void k_unpack_codes(const uint8_t* __restrict__ in, size_t n,
                               size_t M, int bits, size_t stride,
                               uint32_t* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * M) return;
  const size_t i = t / M, m = t % M;
  out[t] = get_code(in + i * stride, (int)m, bits);
}

__global__ void k_check_weights(const double* hp, const double* ho, size_t n,
                                DevError* err) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = hp[i], b = ho[i];
  // AnisotropicWeights::from_h validation (geometry.hpp:127-129)
  if (!(a >= 0.0) || !(b >= 0.0) || !isfinite(a) || !isfinite(b))
    report_error(err, i, AQ_E_INVALID_ARGUMENT);
}

int make_dev_weights(aq_session* s, const aq_weights* w, size_t n, size_t d,
                     DevWeights* out) {
  if (!w) return ref_error(AQ_E_INVALID_ARGUMENT, "null weights");
  DevWeights dw{};
  dw.mode = w->mode;
  dw.d = (int)d;
  switch (w->mode) {
    case AQ_WEIGHTS_UNIFORM:
      if (!(w->h_parallel >= 0.0) || !(w->h_perpendicular >= 0.0) ||
          !std::isfinite(w->h_parallel) || !std::isfinite(w->h_perpendicular))
        return ref_error(AQ_E_INVALID_ARGUMENT,
                         "h coefficients must be finite and >= 0");
      dw.hp = w->h_parallel;
      dw.ho = w->h_perpendicular;
      break;
    case AQ_WEIGHTS_PER_POINT: {
      if (!w->h_parallel_arr || !w->h_perpendicular_arr)
        return ref_error(AQ_E_INVALID_ARGUMENT,
                         "need one AnisotropicWeights per datapoint");
      void* p;
      AQ_TRY(scratch(s, 5, 2 * n * sizeof(double) + 16, &p));
      double* hp = (double*)p;
      double* ho = hp + n;
      if (n) {
        AQ_CUDA(cudaMemcpyAsync(hp, w->h_parallel_arr, n * sizeof(double),
                                cudaMemcpyHostToDevice, s->stream));
        AQ_CUDA(cudaMemcpyAsync(ho, w->h_perpendicular_arr,
                                n * sizeof(double), cudaMemcpyHostToDevice,
                                s->stream));
        AQ_TRY(clear_dev_error(s));
        k_check_weights<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(
            hp, ho, n, s->err);
        AQ_LAUNCHED(s);
        AQ_TRY(sync_and_check(s, "weights"));
      }
      dw.hp_arr = hp;
      dw.ho_arr = ho;
      break;
    }
    case AQ_WEIGHTS_THRESHOLD:
      if (d < 2) return ref_error(AQ_E_INVALID_ARGUMENT, "eta_limit needs d >= 2");
      dw.threshold = w->threshold;
      dw.policy = w->threshold_policy;
      break;
    default:
      return ref_error(AQ_E_INVALID_ARGUMENT, "unknown weight mode");
  }
  *out = dw;
  return AQ_OK;
}

int stage_codebook(aq_codebook* cb) {
  aq_session* s = cb->s;
  if (cb->sd != 2 || cb->k > 16) return AQ_OK;
  if (!cb->f32) {
    AQ_CUDA(cudaMallocAsync(&cb->f32, cb->M * 16 * sizeof(float4), s->stream));
    AQ_CUDA(cudaMallocAsync(&cb->rmax, cb->M * sizeof(float), s->stream));
  }
  k_stage_codebook2<<<(unsigned)((cb->M + 127) / 128), 128, 0, s->stream>>>(
      cb->d64, (int)cb->M, (int)cb->k, cb->f32, cb->rmax);
  AQ_LAUNCHED(s);
  return AQ_OK;
}

}  // namespace aqd

using namespace aqd;

extern "C" {

int aq_error_class(int status) {
  // ErrorClass (error.hpp:25): QuadratureFailure / SingularSystem are runtime,
  // device failures are runtime, everything else validation.
  return (status == AQ_E_QUADRATURE_FAILURE || status == AQ_E_SINGULAR_SYSTEM ||
          status == AQ_E_CUDA)
             ? 1
             : 0;
}

const char* aq_last_error(void) { return g_msg; }
const char* aq_status_name(int status) { return status_ref_name(status); }

int aq_session_create(int device, aq_session** out) {
  if (!out) return ref_error(AQ_E_INVALID_ARGUMENT, "null out");
  int count = 0;
  AQ_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count)
    return ref_error(AQ_E_INVALID_ARGUMENT, "device index out of range");
  AQ_CUDA(cudaSetDevice(device));
  aq_session* s = new aq_session();
  s->device = device;
  cudaDeviceProp prop;
  AQ_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    delete s;
    set_error(AQ_E_CUDA, "this library is built for sm_100a (B200); device is sm_%d%d",
              prop.major, prop.minor);
    return AQ_E_CUDA;
  }
  s->num_sms = prop.multiProcessorCount;
  // Keep stream-ordered allocations in the device's pool across
  // synchronisations (the default threshold 0 returns freed memory at every
  // sync, so the next cudaMallocAsync of a multi-GB training buffer maps it
  // again); $AQ_POOL_KEEP=0 restores the default.
  {
    const char* keep = getenv("AQ_POOL_KEEP");
    cudaMemPool_t pool;
    if ((!keep || atoi(keep) != 0) && cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  // a failure part-way releases what was created (aq_session_destroy skips nulls)
  const cudaError_t e[] = {
      cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking),
      cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking),
      cudaEventCreateWithFlags(&s->ev_main, cudaEventDisableTiming),
      cudaEventCreateWithFlags(&s->ev_side, cudaEventDisableTiming),
      cudaMallocHost(&s->sum_host, 64 * sizeof(double)),
      cudaMalloc(&s->err, sizeof(DevError)),
      cudaMallocHost(&s->err_host, sizeof(DevError))};
  for (cudaError_t x : e)
    if (x != cudaSuccess) {
      aq_session_destroy(s);
      set_error(AQ_E_CUDA, "session setup failed: %s", cudaGetErrorString(x));
      return AQ_E_CUDA;
    }
  *out = s;
  return AQ_OK;
}

int aq_session_destroy(aq_session* s) {
  if (!s) return AQ_OK;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (auto& sc : s->scratch)
    if (sc.p) cudaFree(sc.p);
  for (auto& sc : s->pinned)
    if (sc.p) cudaFreeHost(sc.p);
  if (s->err) cudaFree(s->err);
  if (s->err_host) cudaFreeHost(s->err_host);
  if (s->side) cudaStreamSynchronize(s->side);
  if (s->sum_host) cudaFreeHost(s->sum_host);
  if (s->ev_main) cudaEventDestroy(s->ev_main);
  if (s->ev_side) cudaEventDestroy(s->ev_side);
  if (s->side) cudaStreamDestroy(s->side);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return AQ_OK;
}

void* aq_session_stream(aq_session* s) { return s ? (void*)s->stream : nullptr; }

int aq_session_sync(aq_session* s) {
  AQ_TRY(check_session(s));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

uint64_t aq_session_launches(aq_session* s) { return s ? s->launches : 0; }

// Kernel timers: enable=1 starts recording CUDA events around the timed
// kernels (encode, adc_score, adc_merge, rerank, lut) on the session stream;
// aq_session_timer_read syncs, folds the recorded pairs into totals and
// returns total milliseconds and launch count for a slot.
int aq_session_timing(aq_session* s, int enable) {
  AQ_TRY(check_session(s));
  s->timing = enable != 0;
  return AQ_OK;
}

int aq_session_timer_read(aq_session* s, int slot, double* ms, uint64_t* count,
                          int reset) {
  AQ_TRY(check_session(s));
  if (slot < 0 || slot >= AQ_T_COUNT) return ref_error(AQ_E_INVALID_ARGUMENT, "bad timer slot");
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  for (int t = 0; t < AQ_T_COUNT; ++t) {
    auto& v = s->tev[t];
    for (size_t e = 0; e + 1 < v.size(); e += 2) {
      float x = 0.0f;
      AQ_CUDA(cudaEventElapsedTime(&x, v[e], v[e + 1]));
      s->tms[t] += x;
      s->tcount[t] += 1;
    }
    for (auto ev : v) cudaEventDestroy(ev);
    v.clear();
  }
  if (ms) *ms = s->tms[slot];
  if (count) *count = s->tcount[slot];
  if (reset) {
    s->tms[slot] = 0;
    s->tcount[slot] = 0;
  }
  return AQ_OK;
}

static int dataset_from_device_rows(aq_session* s, const float* xdev, size_t n,
                                    size_t d, aq_dataset** out) {
  aq_dataset* ds = new aq_dataset();
  ds->s = s;
  ds->n = n;
  ds->d = d;
  const size_t tf = tiled_floats(n, d);
  // +64 floats: the encoder prefetches one dimension pair past a row's end
  // four pair tiles of padding: the encoders prefetch up to two pairs past a row
  AQ_CUDA(cudaMallocAsync(&ds->xt, (tf + 256) * sizeof(float), s->stream));
  AQ_CUDA(cudaMemsetAsync(ds->xt + tf, 0, 256 * sizeof(float), s->stream));
  AQ_CUDA(cudaMallocAsync(&ds->norms, (n ? n : 1) * sizeof(double), s->stream));
  AQ_CUDA(cudaMallocAsync(&ds->xr, (n * d ? n * d : 1) * sizeof(float), s->stream));
  if (n * d)
    AQ_CUDA(cudaMemcpyAsync(ds->xr, xdev, n * d * sizeof(float), cudaMemcpyDeviceToDevice,
                            s->stream));
  const size_t ntile = ((n + 31) / 32) * 32;
  if (ntile) {
    k_tile_rows<float><<<(unsigned)((ntile + 127) / 128), 128, 0, s->stream>>>(
        xdev, n, d, ds->xt, ds->norms);
    AQ_LAUNCHED(s);
  }
  *out = ds;
  return AQ_OK;
}

// float64 rows (values that are not float32-exact): row-major + pair-tiled
// float64 copies, norms in the reference's order.
static int dataset_from_device_rows64(aq_session* s, const double* xdev, size_t n, size_t d,
                                      aq_dataset** out) {
  aq_dataset* ds = new aq_dataset();
  ds->s = s;
  ds->n = n;
  ds->d = d;
  ds->f64 = 1;
  const size_t tf = tiled_floats(n, d);
  int st = AQ_OK;
  if (cudaMallocAsync(&ds->xt64, (tf + 256) * sizeof(double), s->stream) != cudaSuccess ||
      cudaMallocAsync(&ds->norms, (n ? n : 1) * sizeof(double), s->stream) != cudaSuccess ||
      cudaMallocAsync(&ds->xr64, (n * d ? n * d : 1) * sizeof(double), s->stream) !=
          cudaSuccess)
    st = ref_error(AQ_E_CUDA, "out of device memory for the dataset");
  if (st == AQ_OK) {
    cudaMemsetAsync(ds->xt64 + tf, 0, 256 * sizeof(double), s->stream);
    if (n * d)
      cudaMemcpyAsync(ds->xr64, xdev, n * d * sizeof(double), cudaMemcpyDeviceToDevice,
                      s->stream);
    const size_t ntile = ((n + 31) / 32) * 32;
    if (ntile) {
      k_tile_rows<double><<<(unsigned)((ntile + 127) / 128), 128, 0, s->stream>>>(
          xdev, n, d, ds->xt64, ds->norms);
      AQ_LAUNCHED(s);
    }
  }
  if (st != AQ_OK) {
    aq_dataset_free(ds);
    return st;
  }
  *out = ds;
  return AQ_OK;
}

// float64 host rows: float32 storage when every value is float32-exact
// (the fast kernels), float64 storage otherwise.
int aq_dataset_upload_f64(aq_session* s, const double* x, size_t n, size_t d,
                          aq_dataset** out) {
  AQ_TRY(check_session(s));
  if (d == 0) return ref_error(AQ_E_INVALID_ARGUMENT, "dimension must be positive");
  bool exact32 = true;
  for (size_t e = 0; e < n * d && exact32; ++e)
    exact32 = (double)(float)x[e] == x[e] || x[e] != x[e];
  if (exact32) {
    std::vector<float> f(n * d);
    for (size_t e = 0; e < n * d; ++e) f[e] = (float)x[e];
    return aq_dataset_upload(s, f.data(), n, d, out);
  }
  void* stage = nullptr;
  AQ_TRY(scratch(s, 0, n * d * sizeof(double) + 16, &stage));
  AQ_CUDA(cudaMemcpyAsync(stage, x, n * d * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  AQ_TRY(dataset_from_device_rows64(s, (const double*)stage, n, d, out));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

int aq_dataset_is_f64(const aq_dataset* ds) { return ds ? ds->f64 : 0; }

int aq_dataset_upload(aq_session* s, const float* x, size_t n, size_t d,
                      aq_dataset** out) {
  AQ_TRY(check_session(s));
  if (d == 0) return ref_error(AQ_E_INVALID_ARGUMENT, "dimension must be positive");
  void* stage = nullptr;
  AQ_TRY(scratch(s, 0, n * d * sizeof(float) + 16, &stage));
  if (n) AQ_CUDA(cudaMemcpyAsync(stage, x, n * d * sizeof(float),
                                 cudaMemcpyHostToDevice, s->stream));
  AQ_TRY(dataset_from_device_rows(s, (const float*)stage, n, d, out));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

int aq_dataset_wrap_device(aq_session* s, const float* x_dev, size_t n,
                           size_t d, aq_dataset** out) {
  AQ_TRY(check_session(s));
  if (d == 0) return ref_error(AQ_E_INVALID_ARGUMENT, "dimension must be positive");
  return dataset_from_device_rows(s, x_dev, n, d, out);
}

int aq_dataset_free(aq_dataset* ds) {
  if (!ds) return AQ_OK;
  cudaSetDevice(ds->s->device);
  cudaFreeAsync(ds->xt, ds->s->stream);
  cudaFreeAsync(ds->xr, ds->s->stream);
  cudaFreeAsync(ds->xt64, ds->s->stream);
  cudaFreeAsync(ds->xr64, ds->s->stream);
  cudaFreeAsync(ds->norms, ds->s->stream);
  delete ds;
  return AQ_OK;
}

int aq_dataset_norms(aq_dataset* ds, double* norms_out) {
  AQ_TRY(check_session(ds->s));
  if (ds->n)
    AQ_CUDA(cudaMemcpyAsync(norms_out, ds->norms, ds->n * sizeof(double),
                            cudaMemcpyDeviceToHost, ds->s->stream));
  AQ_CUDA(cudaStreamSynchronize(ds->s->stream));
  return AQ_OK;
}

int aq_codebook_upload(aq_session* s, const double* dict, size_t M, size_t k,
                       size_t sd, aq_codebook** out) {
  AQ_TRY(check_session(s));
  if (M == 0 || sd == 0)
    return ref_error(AQ_E_INVALID_ARGUMENT, "codebook needs M >= 1 and sub_dimension >= 1");
  aq_codebook* cb = new aq_codebook();
  cb->s = s;
  cb->M = M;
  cb->k = k;
  cb->sd = sd;
  const size_t cnt = M * k * sd;
  AQ_CUDA(cudaMallocAsync(&cb->d64, (cnt ? cnt : 1) * sizeof(double), s->stream));
  if (cnt && dict)
    AQ_CUDA(cudaMemcpyAsync(cb->d64, dict, cnt * sizeof(double),
                            cudaMemcpyHostToDevice, s->stream));
  else if (cnt)  // an output codebook: defined contents until written
    AQ_CUDA(cudaMemsetAsync(cb->d64, 0, cnt * sizeof(double), s->stream));
  AQ_TRY(stage_codebook(cb));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  *out = cb;
  return AQ_OK;
}

int aq_codebook_download(aq_codebook* cb, double* out) {
  AQ_TRY(check_session(cb->s));
  const size_t cnt = cb->M * cb->k * cb->sd;
  if (cnt)
    AQ_CUDA(cudaMemcpyAsync(out, cb->d64, cnt * sizeof(double),
                            cudaMemcpyDeviceToHost, cb->s->stream));
  AQ_CUDA(cudaStreamSynchronize(cb->s->stream));
  return AQ_OK;
}

int aq_codebook_free(aq_codebook* cb) {
  if (!cb) return AQ_OK;
  cudaSetDevice(cb->s->device);
  cudaFreeAsync(cb->d64, cb->s->stream);
  if (cb->f32) cudaFreeAsync(cb->f32, cb->s->stream);
  if (cb->rmax) cudaFreeAsync(cb->rmax, cb->s->stream);
  delete cb;
  return AQ_OK;
}

int aq_codes_alloc(aq_session* s, size_t n, size_t M, size_t k,
                   aq_codes** out) {
  AQ_TRY(check_session(s));
  if (M == 0) return ref_error(AQ_E_INVALID_ARGUMENT, "M must be positive");
  if (k > 256)
    return ref_error(AQ_E_UNSUPPORTED, "device codes support k <= 256");
  aq_codes* c = new aq_codes();
  c->s = s;
  c->n = n;
  c->M = M;
  c->k = k;
  c->bits = k <= 16 ? 4 : 8;
  c->stride = code_stride(M, c->bits);
  AQ_CUDA(cudaMallocAsync(&c->data, (n * c->stride) ? n * c->stride : 8, s->stream));
  if (n) AQ_CUDA(cudaMemsetAsync(c->data, 0, n * c->stride, s->stream));
  *out = c;
  return AQ_OK;
}

int aq_codes_upload(aq_session* s, const uint32_t* codes, size_t n, size_t M,
                    size_t k, aq_codes** out) {
  AQ_TRY(aq_codes_alloc(s, n, M, k, out));
  aq_codes* c = *out;
  if (n == 0) return AQ_OK;
  if (n * M >= ((size_t)1 << 22)) {
    // Large code matrices (the reference-signature calls pass them by value,
    // 4 bytes per code): packed on the host by every core straight into
    // page-locked memory, then one copy of the packed rows (M / 2 bytes
    // per row for 4-bit codes) instead of a pageable copy of n M words.
    // Same bytes and the same error as k_pack_codes: the lowest flat index
    // of a code >= k.
    void* pin;
    int st = aqd::pinned_buffer(s, 6, n * c->stride, &pin);
    if (st != AQ_OK) {
      aq_codes_free(c);
      *out = nullptr;
      return st;
    }
    uint8_t* dst = static_cast<uint8_t*>(pin);
    const uint32_t kk = (uint32_t)(k ? k : 1);
    const size_t nt = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(),
                                                            n / 4096 + 1));
    std::vector<size_t> bad(nt, SIZE_MAX);
    auto pack = [&](size_t t) {
      const size_t r0 = n * t / nt, r1 = n * (t + 1) / nt;
      for (size_t i = r0; i < r1; ++i) {
        uint8_t* row = dst + i * c->stride;
        std::memset(row, 0, c->stride);
        const uint32_t* in = codes + i * M;
        for (size_t m = 0; m < M; ++m) {
          const uint32_t v = in[m];
          if (v >= kk && bad[t] == SIZE_MAX) bad[t] = i * M + m;
          if (c->bits == 4)
            row[m >> 1] |= (uint8_t)((v & 15u) << ((m & 1) * 4));
          else
            row[m] = (uint8_t)v;
        }
      }
    };
    std::vector<std::thread> th;
    for (size_t t = 1; t < nt; ++t) th.emplace_back(pack, t);
    pack(0);
    for (auto& x : th) x.join();
    const size_t first = *std::min_element(bad.begin(), bad.end());
    if (first != SIZE_MAX) {
      char buf[256];
      snprintf(buf, sizeof buf, "%s (%s, point %llu)", kDevErrDetail[AQ_E_CODE_OUT_OF_RANGE],
               "codes upload", (unsigned long long)first);
      aq_codes_free(c);
      *out = nullptr;
      return ref_error(AQ_E_CODE_OUT_OF_RANGE, buf);
    }
    st = cudaMemcpyAsync(c->data, dst, n * c->stride, cudaMemcpyHostToDevice, s->stream) ==
                 cudaSuccess &&
                 cudaStreamSynchronize(s->stream) == cudaSuccess
             ? AQ_OK
             : ref_error(AQ_E_CUDA, "codes upload copy failed");
    if (st) {
      aq_codes_free(c);
      *out = nullptr;
    }
    return st;
  }
  void* stage;
  AQ_TRY(scratch(s, 0, n * M * sizeof(uint32_t), &stage));
  AQ_CUDA(cudaMemcpyAsync(stage, codes, n * M * sizeof(uint32_t),
                          cudaMemcpyHostToDevice, s->stream));
  AQ_TRY(clear_dev_error(s));
  k_pack_codes<<<(unsigned)((n + 255) / 256), 256, 0, s->stream>>>(
      (const uint32_t*)stage, n, M, c->bits, c->stride, c->data, s->err,
      (uint32_t)(k ? k : 1));
  AQ_LAUNCHED(s);
  const int st = sync_and_check(s, "codes upload");
  if (st) {
    aq_codes_free(c);
    *out = nullptr;
  }
  return st;
}

int aq_codes_upload_packed(aq_session* s, const uint8_t* packed, size_t n,
                           size_t M, size_t k, aq_codes** out) {
  AQ_TRY(aq_codes_alloc(s, n, M, k, out));
  aq_codes* c = *out;
  if (n) AQ_CUDA(cudaMemcpyAsync(c->data, packed, n * c->stride,
                                 cudaMemcpyHostToDevice, s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

}  // extern "C"

namespace aqd {
// codes -> uint32 per code on the device (async, session stream)
int codes_unpack_async(aq_codes* c, uint32_t* dev_out) {
  const size_t total = c->n * c->M;
  if (!total) return AQ_OK;
  k_unpack_codes<<<(unsigned)((total + 255) / 256), 256, 0, c->s->stream>>>(
      c->data, c->n, c->M, c->bits, c->stride, dev_out);
  AQ_LAUNCHED(c->s);
  return AQ_OK;
}
}  // namespace aqd

extern "C" {

int aq_codes_download(aq_codes* c, uint32_t* out) {
  aq_session* s = c->s;
  AQ_TRY(check_session(s));
  if (c->n == 0) return AQ_OK;
  void* stage;
  AQ_TRY(scratch(s, 0, c->n * c->M * sizeof(uint32_t), &stage));
  const size_t total = c->n * c->M;
  k_unpack_codes<<<(unsigned)((total + 255) / 256), 256, 0, s->stream>>>(
      c->data, c->n, c->M, c->bits, c->stride, (uint32_t*)stage);
  AQ_LAUNCHED(s);
  AQ_CUDA(cudaMemcpyAsync(out, stage, total * sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, s->stream));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

int aq_codes_download_packed(aq_codes* c, uint8_t* out) {
  AQ_TRY(check_session(c->s));
  if (c->n)
    AQ_CUDA(cudaMemcpyAsync(out, c->data, c->n * c->stride,
                            cudaMemcpyDeviceToHost, c->s->stream));
  AQ_CUDA(cudaStreamSynchronize(c->s->stream));
  return AQ_OK;
}

size_t aq_codes_row_bytes(aq_codes* c) { return c ? c->stride : 0; }

int aq_codes_free(aq_codes* c) {
  if (!c) return AQ_OK;
  cudaSetDevice(c->s->device);
  cudaFreeAsync(c->data, c->s->stream);
  delete c;
  return AQ_OK;
}

}  // extern "C"
