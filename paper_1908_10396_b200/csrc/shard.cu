// Building blocks of the row-sharded (multi-GPU) trainer, exported over the C
// ABI so the host orchestration (paper_1908_10396_b200/distributed.py) can
// combine per-shard partials with NCCL:
//   * local normal equations (lower triangle) / isotropic partial sums and the
//     usage histogram of this shard -> all-reduce(sum) -> replicated solve;
//   * local k-means assignment and per-slot partial sums -> all-reduce;
//   * exact sequential float64 sums of this shard's losses (chained in rank
//     order by the host) and the stable loss ranking for reseeding.
// With one shard every result equals the single-GPU trainer's bit for bit.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace aqd {

int run_encode(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes, int mode,
               int passes, int sweep_fixed, double* losses_dev, uint64_t* changed_out);
int sort_scores_desc(aq_session* s, const double* scores, uint32_t* idx, size_t n);
int stage_codebook(aq_codebook* cb);
int seq_sum_device(aq_session* s, const double* v, size_t n, double init, double* out);
int seq_sums_device(aq_session* s, const double* v, size_t ld, size_t count, int rows,
                    const int* active_dev, double* out);

// per-slot partial sums for the isotropic path (pq.hpp:405-417), members in


__global__ void k_copy_counts(const uint32_t* count, size_t total, uint32_t* out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < total) out[t] = count[t];
}

}  // namespace aqd

using namespace aqd;

extern "C" {

// Weight flags of this shard (which update path pq.hpp:383-386 takes):
// flags_out[0] = some point anisotropic, flags_out[1] = first anisotropic
// zero-norm point + 1 (0 = none).
int aq_dev_weight_flags(aq_dataset* ds, const aq_weights* w, uint64_t* flags_out) {
  if (!ds || !flags_out) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  void* owner = nullptr;
  PointW pw;
  int st = point_weights(ds, w, &pw, &owner);
  if (st == AQ_OK) {
    flags_out[0] = pw.flags[0];
    flags_out[1] = pw.flags[1] == ~0ull ? 0ull : pw.flags[1];
  }
  if (owner) cudaFreeAsync(owner, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return st;
}

// Local (this shard's) normal equations, lower triangle, into caller buffers
// (device): A (dim x dim, dim = k d), rhs (dim), usage (M x k uint32).
// flags_out[0] = 1 if any point is anisotropic; flags_out[1] = first
// anisotropic zero-norm point + 1 (0 = none).
int aq_dev_normal_equations_partial(aq_dataset* ds, aq_codes* codes, const aq_weights* w,
                                    size_t k, double* A_dev, double* rhs_dev,
                                    uint32_t* usage_dev, uint64_t* flags_out) {
  if (!ds || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t M = codes->M, dim = k * ds->d;
  void* owner = nullptr;
  PointW pw;
  {
    const int pst = point_weights(ds, w, &pw, &owner);
    if (pst != AQ_OK) {  // validation failures leave no allocation behind
      if (owner) cudaFreeAsync(owner, s->stream);
      return pst;
    }
  }
  Buckets B;
  int st = AQ_OK;
  if (ds->n) st = build_buckets(codes, (int)k, &B);
  if (st == AQ_OK && ds->n) st = assemble_device(ds, codes, pw, B, (int)k, false, A_dev, rhs_dev);
  if (st == AQ_OK && !ds->n) {
    cudaMemsetAsync(A_dev, 0, dim * dim * sizeof(double), s->stream);
    cudaMemsetAsync(rhs_dev, 0, dim * sizeof(double), s->stream);
  }
  if (st == AQ_OK && usage_dev) {
    if (ds->n) {
      k_copy_counts<<<(unsigned)((M * k + 255) / 256), 256, 0, s->stream>>>(B.count, M * k,
                                                                            usage_dev);
      s->launches++;
    } else {
      cudaMemsetAsync(usage_dev, 0, M * k * sizeof(uint32_t), s->stream);
    }
  }
  if (flags_out) {
    flags_out[0] = pw.flags[0];
    flags_out[1] = pw.flags[1] == ~0ull ? 0ull : pw.flags[1];
  }
  cudaFreeAsync(owner, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return st;
}

// Local isotropic partial sums per slot: num (M k sd), den (M k), usage.
int aq_dev_iso_partials(aq_dataset* ds, aq_codes* codes, const aq_weights* w, size_t k,
                        double* num_dev, double* den_dev, uint32_t* usage_dev) {
  if (!ds || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t M = codes->M, sd = ds->d / M;
  void* owner = nullptr;
  PointW pw;
  {
    const int pst = point_weights(ds, w, &pw, &owner);
    if (pst != AQ_OK) {  // validation failures leave no allocation behind
      if (owner) cudaFreeAsync(owner, s->stream);
      return pst;
    }
  }
  Buckets B;
  int st = AQ_OK;
  if (ds->n) {
    st = build_buckets(codes, (int)k, &B);
    if (st == AQ_OK) {
      st = slot_sums_device(s, ds, (int)M, (int)k, (int)sd, B, nullptr, pw.hp, pw.ho, nullptr,
                            num_dev, den_dev);
      if (usage_dev) {
        k_copy_counts<<<(unsigned)((M * k + 255) / 256), 256, 0, s->stream>>>(B.count, M * k,
                                                                              usage_dev);
        s->launches++;
      }
    }
  } else {
    cudaMemsetAsync(num_dev, 0, M * k * sd * sizeof(double), s->stream);
    cudaMemsetAsync(den_dev, 0, M * k * sizeof(double), s->stream);
    if (usage_dev) cudaMemsetAsync(usage_dev, 0, M * k * sizeof(uint32_t), s->stream);
  }
  cudaFreeAsync(owner, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return st;
}

// Ridge (1e-6 trace / dim when ridge < 0) + blocked Cholesky + solve, in
// place on device buffers: A is overwritten by L, rhs by the solution.
int aq_dev_solve_normal_equations(aq_session* s, double* A_dev, double* rhs_dev, size_t dim,
                                  double ridge) {
  AQ_TRY(check_session(s));
  AQ_TRY(trace_ridge_device(s, A_dev, dim, ridge));
  AQ_TRY(llt_solve_device(s, A_dev, (int)dim, rhs_dev));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

// Overwrite a codebook's dictionaries from device memory (and restage).
int aq_codebook_set_device(aq_codebook* cb, const double* dict_dev) {
  if (!cb) return ref_error(AQ_E_INVALID_ARGUMENT, "null codebook");
  AQ_TRY(check_session(cb->s));
  AQ_CUDA(cudaMemcpyAsync(cb->d64, dict_dev, cb->M * cb->k * cb->sd * sizeof(double),
                          cudaMemcpyDeviceToDevice, cb->s->stream));
  AQ_TRY(stage_codebook(cb));
  AQ_CUDA(cudaStreamSynchronize(cb->s->stream));
  return AQ_OK;
}

// pq_point_loss for every local point (pq.hpp:137-146) into losses_dev.
int aq_dev_point_losses(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes,
                        double* losses_dev) {
  if (!ds || !cb || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  return run_encode(ds, cb, w, codes, 2, 0, 0, losses_dev, nullptr);
}

// Stable ranking: idx (ascending on entry) reordered by (score desc, idx asc).
int aq_dev_sort_desc(aq_session* s, const double* scores_dev, uint32_t* idx_dev, size_t n) {
  AQ_TRY(check_session(s));
  AQ_TRY(sort_scores_desc(s, scores_dev, idx_dev, n));
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

// Sequential float64 sum continuing from `init` (std::accumulate order).
int aq_dev_seq_sum(aq_session* s, const double* v_dev, size_t n, double init, double* out) {
  AQ_TRY(check_session(s));
  double* d;
  AQ_CUDA(cudaMallocAsync(&d, sizeof(double), s->stream));
  AQ_TRY(seq_sum_device(s, v_dev, n, init, d));
  AQ_CUDA(cudaMemcpyAsync(out, d, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  cudaFreeAsync(d, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

// Sequential float64 sums of `rows` rows of `count` values (row r at
// v_dev + r * ld), one launch; rows with active_host[r] == 0 give 0.
int aq_dev_seq_sums(aq_session* s, const double* v_dev, size_t ld, size_t count, size_t rows,
                    const int* active_host, double* out_host) {
  AQ_TRY(check_session(s));
  if (rows == 0) return AQ_OK;
  int* act = nullptr;
  double* d;
  AQ_CUDA(cudaMallocAsync(&d, rows * sizeof(double), s->stream));
  AQ_CUDA(cudaMemsetAsync(d, 0, rows * sizeof(double), s->stream));
  if (active_host) {
    AQ_CUDA(cudaMallocAsync(&act, rows * sizeof(int), s->stream));
    AQ_CUDA(cudaMemcpyAsync(act, active_host, rows * sizeof(int), cudaMemcpyHostToDevice,
                            s->stream));
  }
  AQ_TRY(seq_sums_device(s, v_dev, ld, count, (int)rows, act, d));
  AQ_CUDA(cudaMemcpyAsync(out_host, d, rows * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  cudaFreeAsync(d, s->stream);
  if (act) cudaFreeAsync(act, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return AQ_OK;
}

// Local k-means partial sums per slot (unit weights) for active subspaces.
int aq_dev_kmeans_partials(aq_dataset* ds, aq_codes* codes, size_t k, const int* active_host,
                           double* num_dev, double* den_dev, uint32_t* count_dev) {
  if (!ds || !codes) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  aq_session* s = ds->s;
  AQ_TRY(check_session(s));
  const size_t M = codes->M, sd = ds->d / M;
  int* act;
  AQ_CUDA(cudaMallocAsync(&act, M * sizeof(int), s->stream));
  AQ_CUDA(cudaMemcpyAsync(act, active_host, M * sizeof(int), cudaMemcpyHostToDevice, s->stream));
  AQ_CUDA(cudaMemsetAsync(num_dev, 0, M * k * sd * sizeof(double), s->stream));
  AQ_CUDA(cudaMemsetAsync(den_dev, 0, M * k * sizeof(double), s->stream));
  int st = AQ_OK;
  if (ds->n) {
    Buckets B;
    st = build_buckets(codes, (int)k, &B);
    if (st == AQ_OK) {
      st = slot_sums_device(s, ds, (int)M, (int)k, (int)sd, B, act, nullptr, nullptr, nullptr,
                            num_dev, den_dev);
      k_copy_counts<<<(unsigned)((M * k + 255) / 256), 256, 0, s->stream>>>(B.count, M * k,
                                                                            count_dev);
      s->launches++;
    }
  } else {
    cudaMemsetAsync(count_dev, 0, M * k * sizeof(uint32_t), s->stream);
  }
  cudaFreeAsync(act, s->stream);
  AQ_CUDA(cudaStreamSynchronize(s->stream));
  return st;
}

}  // extern "C"
