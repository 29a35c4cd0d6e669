// Multi-device session: the database sharded by contiguous rows over the
// GPUs of one box, driven from one host process (the C++ drop-in's model:
// one call uses every GPU). One aq_session per shard; a device may carry
// several shards (tests run W shards on one B200), and results depend only on
// the shard count:
//   * pq_quantize: points are independent (pq.hpp:581-612) — no exchange;
//     codes equal the single-device call's;
//   * adc_search: per-shard exact top-N, then the lists (global ids) are
//     copied peer-to-peer to shard 0 and merged in the reference's order
//     (score desc, index asc; index.hpp:88-112) — equal to the single-device
//     result;
//   * train_apq / train_l2_pq: the row-sharded trainer of DESIGN.md §7
//     (paper_1908_10396_b200/distributed.py restated over peer memory): per
//     shard partial sums (normal equations, isotropic / k-means sums, loss
//     totals), summed in shard order along a chain of device-to-device
//     copies (the normal equations as their lower triangle, chunk-pipelined
//     across the shards' streams), solved once on the last shard and the
//     solution broadcast. One shard = the single-device trainer bit for bit;
//     W shards re-associate each float64 sum at W - 1 boundaries.
// Every exchange is a cudaMemcpyPeerAsync over NVLink between the shards'
// devices (a plain device copy when two shards share a device); the sums are
// ordered by shard, which an NCCL all-reduce cannot guarantee.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"

namespace aqd {
int adc_search_device(aq_codes* codes, aq_codebook* cb, const double* Qd, size_t nq,
                      size_t topn, uint32_t* ids, double* scores);
int run_encode_chunk(aq_dataset* ds, aq_codebook* cb, const aq_weights* w, aq_codes* codes,
                     int passes, size_t base);
int sync_and_check(aq_session* s, const char* what);
int clear_dev_error(aq_session* s);
int stage_codebook(aq_codebook* cb);
}  // namespace aqd

using namespace aqd;

struct aq_multi {
  std::vector<aq_session*> s;  // one per shard
};

namespace {

void shard_bounds(size_t n, size_t W, size_t r, size_t* lo, size_t* hi) {
  const size_t base = n / W, extra = n % W;
  *lo = r * base + std::min(r, extra);
  *hi = *lo + base + (r < extra ? 1 : 0);
}

// One host thread per shard (every per-shard call is host-synchronous); the
// first failing shard's status and message are re-raised on the caller's
// thread (messages are thread-local).
template <class F>
int run_shards(aq_multi* m, F f) {
  const size_t W = m->s.size();
  std::vector<int> st(W, AQ_OK);
  std::vector<std::string> msg(W);
  std::vector<std::thread> th;
  for (size_t r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      cudaSetDevice(m->s[r]->device);
      st[r] = f(r);
      if (st[r] != AQ_OK) msg[r] = aq_last_error();
    });
  for (auto& t : th) t.join();
  for (size_t r = 0; r < W; ++r)
    if (st[r] != AQ_OK) {
      set_error(st[r], "%s", msg[r].c_str());
      return st[r];
    }
  return AQ_OK;
}

aq_weights shard_weights(const aq_weights* w, size_t lo) {
  aq_weights o = *w;
  if (w->mode == AQ_WEIGHTS_PER_POINT) {
    o.h_parallel_arr = w->h_parallel_arr + lo;
    o.h_perpendicular_arr = w->h_perpendicular_arr + lo;
  }
  return o;
}

__global__ void k_add_into(double* acc, const double* own, size_t cnt) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) acc[t] = __dadd_rn(acc[t], own[t]);  // running sum of lower shards + own
}

__global__ void k_pack_lower(const double* A, size_t dim, double* out) {
  const size_t i = blockIdx.x;
  for (size_t j = threadIdx.x; j <= i; j += blockDim.x) out[i * (i + 1) / 2 + j] = A[i * dim + j];
}
__global__ void k_unpack_lower(const double* in, size_t dim, double* A) {
  const size_t i = blockIdx.x;
  for (size_t j = threadIdx.x; j < dim; j += blockDim.x)
    A[i * dim + j] = j <= i ? in[i * (i + 1) / 2 + j] : 0.0;
}

__global__ void k_offset_ids(const uint32_t* in, size_t cnt, uint64_t off, uint64_t* out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < cnt) out[t] = in[t] + off;
}

// Merge of per-shard top-N lists: one CTA per query, the W x te candidates
// bitonic-sorted on (score desc, global id asc), the first topn kept.
__global__ void k_merge_lists(const uint64_t* ids, const double* sc, int W, int te, int topn,
                              size_t nq, uint32_t* ids_out, double* sc_out) {
  extern __shared__ __align__(16) unsigned char msm[];
  const int q = blockIdx.x;
  const int tot = W * te;
  int P = 1;
  while (P < tot) P <<= 1;
  unsigned long long* K = reinterpret_cast<unsigned long long*>(msm);
  uint64_t* I = reinterpret_cast<uint64_t*>(K + P);
  for (int e = threadIdx.x; e < P; e += blockDim.x) {
    if (e < tot) {
      const int r = e / te, c = e % te;
      const size_t at = ((size_t)r * nq + q) * te + c;  // shard-major blocks
      unsigned long long b = (unsigned long long)__double_as_longlong(sc[at]);
      b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
      K[e] = ~b;  // ascending == score descending
      I[e] = ids[at];
    } else {
      K[e] = ~0ull;
      I[e] = ~0ull;
    }
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int e = threadIdx.x; e < P; e += blockDim.x) {
        const int o = e ^ stride;
        if (o > e) {
          const bool up = (e & size) == 0;
          const unsigned long long ka = K[e], kb = K[o];
          const uint64_t ia = I[e], ib = I[o];
          const bool gt = ka > kb || (ka == kb && ia > ib);
          if (gt == up) {
            K[e] = kb;
            K[o] = ka;
            I[e] = ib;
            I[o] = ia;
          }
        }
      }
      __syncthreads();
    }
  for (int e = threadIdx.x; e < topn; e += blockDim.x) {
    unsigned long long b = ~K[e];
    b = (b >> 63) ? (b & 0x7fffffffffffffffull) : ~b;
    ids_out[(size_t)q * topn + e] = (uint32_t)I[e];
    sc_out[(size_t)q * topn + e] = __longlong_as_double((long long)b);
  }
}

// ---- the sharded trainer --------------------------------------------------------------

struct Shard {
  aq_session* s = nullptr;
  size_t lo = 0, hi = 0;
  aq_dataset* ds = nullptr;
  aq_codebook* cb = nullptr;
  aq_codes* codes = nullptr;
  aq_weights w{};
  double* buf = nullptr;  // per-shard device scratch (losses, partials)
  size_t buf_cnt = 0;
  double* xbuf = nullptr;  // exchange buffer (a lower shard's running sum)
  size_t xbuf_cnt = 0;
  size_t n() const { return hi - lo; }
};

int ensure(aq_session* s, double** p, size_t* have, size_t cnt) {
  if (*have >= cnt) return AQ_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *have = 0;
  AQ_CUDA(cudaMalloc(p, std::max<size_t>(cnt, 1) * sizeof(double)));
  *have = cnt;
  return AQ_OK;
}

class Trainer {
 public:
  Trainer(aq_multi* m, const float* x, size_t n, size_t d, const aq_weights* w)
      : m_(m), x_(x), n_(n), d_(d), W_(m->s.size()), sh_(W_) {
    for (size_t r = 0; r < W_; ++r) {
      sh_[r].s = m->s[r];
      shard_bounds(n, W_, r, &sh_[r].lo, &sh_[r].hi);
      sh_[r].w = shard_weights(w, sh_[r].lo);
    }
  }
  ~Trainer() {
    for (auto& h : sh_) {
      cudaSetDevice(h.s->device);
      aq_dataset_free(h.ds);
      aq_codebook_free(h.cb);
      aq_codes_free(h.codes);
      if (h.buf) cudaFree(h.buf);
      if (h.xbuf) cudaFree(h.xbuf);
    }
  }

  int upload() {
    return run_shards(m_, [&](size_t r) -> int {
      Shard& h = sh_[r];
      return aq_dataset_upload(h.s, x_ + h.lo * d_, h.n(), d_, &h.ds);
    });
  }

  // replicated codebook on every shard (host values)
  int set_codebook(const std::vector<double>& dict, size_t M, size_t k, size_t sd) {
    return run_shards(m_, [&](size_t r) -> int {
      Shard& h = sh_[r];
      if (!h.cb || h.cb->M != M || h.cb->k != k || h.cb->sd != sd) {
        aq_codebook_free(h.cb);
        h.cb = nullptr;
        AQ_TRY(aq_codebook_upload(h.s, dict.data(), M, k, sd, &h.cb));
      } else {
        AQ_CUDA(cudaMemcpyAsync(h.cb->d64, dict.data(), dict.size() * sizeof(double),
                                cudaMemcpyHostToDevice, h.s->stream));
        AQ_TRY(stage_codebook(h.cb));
        AQ_CUDA(cudaStreamSynchronize(h.s->stream));
      }
      if (!h.codes || h.codes->M != M || h.codes->k != k) {
        aq_codes_free(h.codes);
        h.codes = nullptr;
        AQ_TRY(aq_codes_alloc(h.s, h.n(), M, k, &h.codes));
      }
      return AQ_OK;
    });
  }

  // rows of global ids (float32 values, exact in float64) from the host copy
  std::vector<double> init_rows(const std::vector<size_t>& gid, size_t M, size_t k, size_t sd) {
    std::vector<double> dict(M * k * sd);
    for (size_t t = 0; t < M * k; ++t) {
      const size_t m = t / k;
      for (size_t c = 0; c < sd; ++c) dict[t * sd + c] = x_[gid[t] * d_ + m * sd + c];
    }
    return dict;
  }

  // rank-ordered sum of per-shard device vectors (shard r's at part[r]) along
  // the chain r = 0 .. W-1, pipelined in chunks; the total lands in part[W-1]
  int chain_sum(std::vector<double*>& part, size_t cnt) {
    if (W_ == 1 || cnt == 0) return AQ_OK;
    const size_t chunk = size_t(1) << 21;  // 16 MB of doubles
    const size_t nch = (cnt + chunk - 1) / chunk;
    std::vector<std::vector<cudaEvent_t>> ev(W_, std::vector<cudaEvent_t>(nch));
    for (size_t r = 0; r < W_; ++r) {
      cudaSetDevice(sh_[r].s->device);
      for (auto& e : ev[r]) AQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      if (r > 0) AQ_TRY(ensure(sh_[r].s, &sh_[r].xbuf, &sh_[r].xbuf_cnt, cnt));
    }
    for (size_t c = 0; c < nch; ++c) {
      const size_t b = c * chunk, e = std::min(cnt, b + chunk);
      cudaSetDevice(sh_[0].s->device);
      AQ_CUDA(cudaEventRecord(ev[0][c], sh_[0].s->stream));
      for (size_t r = 1; r < W_; ++r) {
        aq_session* s = sh_[r].s;
        cudaSetDevice(s->device);
        AQ_CUDA(cudaStreamWaitEvent(s->stream, ev[r - 1][c], 0));
        AQ_CUDA(cudaMemcpyPeerAsync(sh_[r].xbuf + b, s->device, part[r - 1] + b,
                                    sh_[r - 1].s->device, (e - b) * sizeof(double), s->stream));
        // part[r] = (running sum of shards < r) + own
        k_add_into<<<(unsigned)((e - b + 255) / 256), 256, 0, s->stream>>>(sh_[r].xbuf + b,
                                                                            part[r] + b, e - b);
        AQ_LAUNCHED(s);
        AQ_CUDA(cudaMemcpyAsync(part[r] + b, sh_[r].xbuf + b, (e - b) * sizeof(double),
                                cudaMemcpyDeviceToDevice, s->stream));
        AQ_CUDA(cudaEventRecord(ev[r][c], s->stream));
      }
    }
    for (size_t r = 0; r < W_; ++r) {
      cudaSetDevice(sh_[r].s->device);
      AQ_CUDA(cudaStreamSynchronize(sh_[r].s->stream));
      for (auto& e : ev[r]) cudaEventDestroy(e);
    }
    return AQ_OK;
  }

  // rank-ordered sum of per-shard host values
  static double ordered(const std::vector<double>& v) {
    double a = v[0];
    for (size_t r = 1; r < v.size(); ++r) a = a + v[r];
    return a;
  }

  // first `take` global ids of loss_ranking (vq.hpp:221-229) over all shards:
  // per-shard stable ranking, merged by (loss desc, id asc); losses[r] are
  // shard r's device losses (count n_r, stride `ld` rows apart by `row`)
  int global_ranking(const std::vector<const double*>& losses, size_t take,
                     std::vector<size_t>* out) {
    take = std::min(take, n_);
    std::vector<std::vector<double>> v(W_);
    std::vector<std::vector<uint32_t>> id(W_);
    AQ_TRY(run_shards(m_, [&](size_t r) -> int {
      Shard& h = sh_[r];
      const size_t nr = h.n(), t = std::min(take, nr);
      if (!nr) return AQ_OK;
      uint32_t* idx = nullptr;
      AQ_CUDA(cudaMalloc(&idx, nr * sizeof(uint32_t)));
      std::vector<uint32_t> iota(nr);
      for (size_t i = 0; i < nr; ++i) iota[i] = (uint32_t)i;
      cudaMemcpy(idx, iota.data(), nr * sizeof(uint32_t), cudaMemcpyHostToDevice);
      int st = aq_dev_sort_desc(h.s, losses[r], idx, nr);
      if (st == AQ_OK) {
        id[r].resize(t);
        v[r].resize(t);
        cudaMemcpy(id[r].data(), idx, t * sizeof(uint32_t), cudaMemcpyDeviceToHost);
        std::vector<double> all(nr);
        cudaMemcpy(all.data(), losses[r], nr * sizeof(double), cudaMemcpyDeviceToHost);
        for (size_t i = 0; i < t; ++i) v[r][i] = all[id[r][i]];
      }
      cudaFree(idx);
      return st;
    }));
    std::vector<std::pair<double, size_t>> c;
    for (size_t r = 0; r < W_; ++r)
      for (size_t i = 0; i < v[r].size(); ++i) c.push_back({v[r][i], sh_[r].lo + id[r][i]});
    std::stable_sort(c.begin(), c.end(), [](const auto& a, const auto& b) {
      return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    out->clear();
    for (size_t i = 0; i < take && i < c.size(); ++i) out->push_back(c[i].second);
    return AQ_OK;
  }

  // ---- train_l2_pq (pq.hpp:469-501): per-subspace k-means in lockstep ----------------
  int train_l2_pq(size_t M, size_t k, const aq_train_config* cfg, std::vector<double>* dict_out) {
    const size_t sd = d_ / M;
    std::vector<size_t> hidx;
    for (size_t m = 0; m < M; ++m) {
      HostRng rng{cfg->seed + m};
      const auto v = rng.sample_distinct(n_, k);
      hidx.insert(hidx.end(), v.begin(), v.end());
    }
    std::vector<double> dict = init_rows(hidx, M, k, sd);
    AQ_TRY(set_codebook(dict, M, k, sd));
    std::vector<int> active(M, 1);
    std::vector<unsigned long long> chg(M);
    std::vector<double> tot(M, 0.0), prev(M);
    auto assign = [&]() -> int {
      std::vector<std::vector<uint64_t>> ch(W_, std::vector<uint64_t>(M, 0));
      std::vector<std::vector<double>> loc(W_, std::vector<double>(M, 0.0));
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        Shard& h = sh_[r];
        AQ_TRY(ensure(h.s, &h.buf, &h.buf_cnt, M * std::max<size_t>(h.n(), 1)));
        AQ_TRY(aq_dev_kmeans_assign(h.ds, h.cb, h.codes, active.data(), h.buf, ch[r].data()));
        if (cfg->relative_tolerance > 0.0)
          AQ_TRY(aq_dev_seq_sums(h.s, h.buf, h.n(), h.n(), M, active.data(), loc[r].data()));
        return AQ_OK;
      }));
      for (size_t mm = 0; mm < M; ++mm) {
        chg[mm] = 0;
        std::vector<double> parts(W_);
        for (size_t r = 0; r < W_; ++r) {
          chg[mm] += ch[r][mm];
          parts[r] = loc[r][mm];
        }
        tot[mm] = cfg->relative_tolerance > 0.0 ? ordered(parts) : 0.0;
      }
      return AQ_OK;
    };
    AQ_TRY(assign());
    for (int it = 0; it < cfg->max_iterations; ++it) {
      bool any = false;
      for (int a : active) any |= a != 0;
      if (!any) break;
      // per-shard k-means sums, summed in shard order
      std::vector<double*> num(W_), den(W_);
      std::vector<std::vector<uint32_t>> cnt(W_, std::vector<uint32_t>(M * k));
      std::vector<double*> bufs(W_);
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        Shard& h = sh_[r];
        double* p = nullptr;
        AQ_CUDA(cudaMalloc(&p, (M * k * sd + M * k) * sizeof(double) + M * k * 4 + 64));
        bufs[r] = p;
        num[r] = p;
        den[r] = p + M * k * sd;
        uint32_t* c = reinterpret_cast<uint32_t*>(p + M * k * sd + M * k);
        AQ_TRY(aq_dev_kmeans_partials(h.ds, h.codes, k, active.data(), num[r], den[r], c));
        cudaMemcpy(cnt[r].data(), c, M * k * 4, cudaMemcpyDeviceToHost);
        return AQ_OK;
      }));
      int st = chain_sum(num, M * k * sd + M * k);  // num and den are contiguous
      std::vector<double> hn(M * k * sd), hd(M * k);
      if (st == AQ_OK) {
        cudaSetDevice(sh_[W_ - 1].s->device);
        cudaMemcpy(hn.data(), num[W_ - 1], hn.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hd.data(), den[W_ - 1], hd.size() * 8, cudaMemcpyDeviceToHost);
      }
      for (size_t r = 0; r < W_; ++r) {
        cudaSetDevice(sh_[r].s->device);
        cudaFree(bufs[r]);
      }
      AQ_TRY(st);
      std::vector<uint64_t> c(M * k, 0);
      for (size_t r = 0; r < W_; ++r)
        for (size_t t = 0; t < M * k; ++t) c[t] += cnt[r][t];
      for (size_t t = 0; t < M * k; ++t)
        if (active[t / k] && c[t] > 0)
          for (size_t q = 0; q < sd; ++q) dict[t * sd + q] = hn[t * sd + q] / hd[t];
      if (cfg->empty_partition_policy == 0) {  // reseed_highest_loss (vq.hpp:284-292)
        for (size_t mm = 0; mm < M; ++mm) {
          if (!active[mm]) continue;
          std::vector<size_t> empty;
          for (size_t j = 0; j < k; ++j)
            if (c[mm * k + j] == 0) empty.push_back(j);
          if (empty.empty()) continue;
          std::vector<const double*> ls(W_);
          for (size_t r = 0; r < W_; ++r) ls[r] = sh_[r].buf + mm * sh_[r].n();
          std::vector<size_t> order;
          AQ_TRY(global_ranking(ls, empty.size(), &order));
          for (size_t e = 0; e < empty.size(); ++e)
            for (size_t q = 0; q < sd; ++q)
              dict[(mm * k + empty[e]) * sd + q] = x_[order[e] * d_ + mm * sd + q];
        }
      }
      AQ_TRY(set_codebook(dict, M, k, sd));
      prev = tot;
      AQ_TRY(assign());
      for (size_t mm = 0; mm < M; ++mm) {
        if (!active[mm]) continue;
        if (chg[mm] == 0) {
          active[mm] = 0;
          continue;
        }
        if (cfg->relative_tolerance > 0.0 &&
            (prev[mm] == 0.0 || prev[mm] - tot[mm] <= cfg->relative_tolerance * prev[mm]))
          active[mm] = 0;
      }
    }
    *dict_out = dict;
    return AQ_OK;
  }

  // ---- pq_codebook_update (pq.hpp:356-464), M > 1 ---------------------------------
  int codebook_update(size_t M, size_t k, double ridge, std::vector<double>* x_out) {
    const size_t sd = d_ / M, dim = k * d_;
    // which path: any anisotropic point; first anisotropic |x| = 0 (global)
    std::vector<uint64_t> fl(2 * W_, 0);
    AQ_TRY(run_shards(m_, [&](size_t r) -> int {
      return aq_dev_weight_flags(sh_[r].ds, &sh_[r].w, fl.data() + 2 * r);
    }));
    bool aniso = false;
    uint64_t zmin = ~0ull;
    for (size_t r = 0; r < W_; ++r) {
      aniso |= fl[2 * r] != 0;
      if (fl[2 * r + 1]) zmin = std::min<uint64_t>(zmin, sh_[r].lo + fl[2 * r + 1] - 1);
    }
    std::vector<double> x(M * k * sd, 0.0);
    std::vector<uint64_t> usage(M * k, 0);
    std::vector<std::vector<uint32_t>> us(W_, std::vector<uint32_t>(M * k));
    if (!aniso) {
      std::vector<double*> part(W_);
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        Shard& h = sh_[r];
        AQ_TRY(ensure(h.s, &h.buf, &h.buf_cnt, M * k * sd + M * k + M * k));
        part[r] = h.buf;
        uint32_t* u = reinterpret_cast<uint32_t*>(h.buf + M * k * sd + M * k);
        AQ_TRY(aq_dev_iso_partials(h.ds, h.codes, &h.w, k, h.buf, h.buf + M * k * sd, u));
        cudaMemcpy(us[r].data(), u, M * k * 4, cudaMemcpyDeviceToHost);
        return AQ_OK;
      }));
      AQ_TRY(chain_sum(part, M * k * sd + M * k));
      std::vector<double> hn(M * k * sd), hd(M * k);
      cudaSetDevice(sh_[W_ - 1].s->device);
      cudaMemcpy(hn.data(), part[W_ - 1], hn.size() * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(hd.data(), part[W_ - 1] + M * k * sd, hd.size() * 8, cudaMemcpyDeviceToHost);
      for (size_t r = 0; r < W_; ++r)
        for (size_t t = 0; t < M * k; ++t) usage[t] += us[r][t];
      for (size_t t = 0; t < M * k; ++t)
        if (usage[t] > 0 && hd[t] <= 0.0)
          return ref_error(AQ_E_SINGULAR_SYSTEM, "zero total weight in block");
      for (size_t t = 0; t < M * k; ++t)
        if (usage[t] > 0)
          for (size_t q = 0; q < sd; ++q) x[t * sd + q] = hn[t * sd + q] / hd[t];
    } else {
      if (dim > 16384)
        return ref_error(AQ_E_INVALID_ARGUMENT,
                         "stacked codebook system exceeds 16384 unknowns (pq.hpp:426-429)");
      if (zmin != ~0ull) {
        char msg[128];
        snprintf(msg, sizeof msg, "anisotropic update undefined at |x| = 0 (point %llu)",
                 (unsigned long long)zmin);
        return ref_error(AQ_E_ZERO_NORM_DATAPOINT, msg);
      }
      const size_t low = dim * (dim + 1) / 2;
      std::vector<double*> packed(W_);
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        Shard& h = sh_[r];
        AQ_TRY(ensure(h.s, &h.buf, &h.buf_cnt, dim * dim + dim + (M * k + 1) / 2 + low + dim));
        double* A = h.buf;
        double* rhs = A + dim * dim;
        uint32_t* u = reinterpret_cast<uint32_t*>(rhs + dim);
        double* pk = h.buf + dim * dim + dim + (M * k + 1) / 2;  // [lower | rhs]
        uint64_t f2[2];
        AQ_TRY(aq_dev_normal_equations_partial(h.ds, h.codes, &h.w, k, A, rhs, u, f2));
        k_pack_lower<<<(unsigned)dim, 256, 0, h.s->stream>>>(A, dim, pk);
        AQ_LAUNCHED(h.s);
        AQ_CUDA(cudaMemcpyAsync(pk + low, rhs, dim * sizeof(double), cudaMemcpyDeviceToDevice,
                                h.s->stream));
        cudaMemcpyAsync(us[r].data(), u, M * k * 4, cudaMemcpyDeviceToHost, h.s->stream);
        AQ_CUDA(cudaStreamSynchronize(h.s->stream));
        packed[r] = pk;
        return AQ_OK;
      }));
      for (size_t r = 0; r < W_; ++r)
        for (size_t t = 0; t < M * k; ++t) usage[t] += us[r][t];
      AQ_TRY(chain_sum(packed, low + dim));
      // solve once, on the last shard
      Shard& L = sh_[W_ - 1];
      cudaSetDevice(L.s->device);
      double* A = L.buf;
      double* rhs = A + dim * dim;
      k_unpack_lower<<<(unsigned)dim, 256, 0, L.s->stream>>>(packed[W_ - 1], dim, A);
      AQ_LAUNCHED(L.s);
      AQ_CUDA(cudaMemcpyAsync(rhs, packed[W_ - 1] + low, dim * sizeof(double),
                              cudaMemcpyDeviceToDevice, L.s->stream));
      AQ_TRY(aq_dev_solve_normal_equations(L.s, A, rhs, dim, ridge));
      AQ_CUDA(cudaMemcpy(x.data(), rhs, dim * sizeof(double), cudaMemcpyDeviceToHost));
    }
    std::vector<size_t> unused;
    for (size_t t = 0; t < M * k; ++t)
      if (usage[t] == 0) unused.push_back(t);
    if (!unused.empty()) {
      // reseed from the loss ranking under the new codebook (pq.hpp:446-462)
      AQ_TRY(set_codebook(x, M, k, sd));
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        Shard& h = sh_[r];
        AQ_TRY(ensure(h.s, &h.buf, &h.buf_cnt, std::max<size_t>(h.n(), 1)));
        return aq_dev_point_losses(h.ds, h.cb, &h.w, h.codes, h.buf);
      }));
      std::vector<const double*> ls(W_);
      for (size_t r = 0; r < W_; ++r) ls[r] = sh_[r].buf;
      std::vector<size_t> order;
      AQ_TRY(global_ranking(ls, unused.size(), &order));
      for (size_t c = 0; c < unused.size(); ++c) {
        const size_t t = unused[c], mm = t / k, g = order[c % order.size()];
        for (size_t q = 0; q < sd; ++q) x[t * sd + q] = x_[g * d_ + mm * sd + q];
      }
    }
    AQ_TRY(set_codebook(x, M, k, sd));
    *x_out = x;
    return AQ_OK;
  }

  // ---- train_apq (pq.hpp:513-575) ------------------------------------------------------
  int train_apq(size_t M, size_t k, const aq_train_config* cfg, int warm_start,
                std::vector<double>* dict_out, std::vector<double>* hist) {
    const size_t sd = d_ / M;
    std::vector<double> dict;
    if (warm_start) {
      AQ_TRY(train_l2_pq(M, k, cfg, &dict));
    } else {
      HostRng rng{cfg->seed};  // one generator for all subspaces (pq.hpp:533-542)
      std::vector<size_t> hidx;
      for (size_t m = 0; m < M; ++m) {
        const auto v = rng.sample_distinct(n_, k);
        hidx.insert(hidx.end(), v.begin(), v.end());
      }
      dict = init_rows(hidx, M, k, sd);
      AQ_TRY(set_codebook(dict, M, k, sd));
      aq_weights iso{AQ_WEIGHTS_UNIFORM, 1.0, 1.0, nullptr, nullptr, 0.0, 0};
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        return aq_dev_pq_quantize(sh_[r].ds, sh_[r].cb, &iso, 0, sh_[r].codes);
      }));
    }
    auto apass = [&](double* tot, uint64_t* changed) -> int {
      std::vector<double> loc(W_, 0.0);
      std::vector<uint64_t> ch(W_, 0);
      AQ_TRY(run_shards(m_, [&](size_t r) -> int {
        Shard& h = sh_[r];
        AQ_TRY(ensure(h.s, &h.buf, &h.buf_cnt, std::max<size_t>(h.n(), 1)));
        AQ_TRY(aq_dev_pq_assign_pass(h.ds, h.cb, &h.w, cfg->sweep_to_fixed_point, h.codes,
                                     h.n() ? h.buf : nullptr, &ch[r]));
        return aq_dev_seq_sum(h.s, h.buf, h.n(), 0.0, &loc[r]);
      }));
      *tot = ordered(loc);
      *changed = 0;
      for (uint64_t c : ch) *changed += c;
      return AQ_OK;
    };
    double tot;
    uint64_t changed;
    AQ_TRY(apass(&tot, &changed));
    hist->assign(1, tot);
    for (int it = 0; it < cfg->max_iterations; ++it) {
      AQ_TRY(codebook_update(M, k, cfg->ridge, &dict));
      const double prev = tot;
      AQ_TRY(apass(&tot, &changed));
      hist->push_back(tot);
      if (changed == 0) break;
      if (cfg->relative_tolerance > 0.0 &&
          (prev == 0.0 || prev - tot <= cfg->relative_tolerance * prev))
        break;
    }
    *dict_out = dict;
    return AQ_OK;
  }

  int download_codes(uint32_t* codes_out, size_t M) {
    return run_shards(m_, [&](size_t r) -> int {
      return sh_[r].n() ? aq_codes_download(sh_[r].codes, codes_out + sh_[r].lo * M) : AQ_OK;
    });
  }

 private:
  aq_multi* m_;
  const float* x_;
  size_t n_, d_, W_;
  std::vector<Shard> sh_;
};

}  // namespace

extern "C" {

int aq_device_count(int* count) {
  if (!count) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  AQ_CUDA(cudaGetDeviceCount(count));
  return AQ_OK;
}

int aq_multi_create(const int* devices, int count, aq_multi** out) {
  if (!out || !devices || count < 1)
    return ref_error(AQ_E_INVALID_ARGUMENT, "need at least one device");
  aq_multi* m = new aq_multi();
  for (int r = 0; r < count; ++r) {
    aq_session* s = nullptr;
    const int st = aq_session_create(devices[r], &s);
    if (st != AQ_OK) {
      aq_multi_destroy(m);
      return st;
    }
    m->s.push_back(s);
  }
  // peer access between distinct devices (NVLink / NVSwitch)
  for (int a = 0; a < count; ++a)
    for (int b = 0; b < count; ++b) {
      const int da = devices[a], db = devices[b];
      if (da == db) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, da, db);
      if (ok) {
        cudaSetDevice(da);
        if (cudaDeviceEnablePeerAccess(db, 0) != cudaSuccess) cudaGetLastError();
      }
    }
  *out = m;
  return AQ_OK;
}

int aq_multi_destroy(aq_multi* m) {
  if (!m) return AQ_OK;
  for (aq_session* s : m->s) aq_session_destroy(s);
  delete m;
  return AQ_OK;
}

int aq_multi_shards(const aq_multi* m) { return m ? (int)m->s.size() : 0; }

aq_session* aq_multi_session(aq_multi* m, int shard) {
  return m && shard >= 0 && shard < (int)m->s.size() ? m->s[shard] : nullptr;
}

// pq_quantize (pq.hpp:581-612) over row shards, one per session.
int aq_multi_pq_quantize(aq_multi* m, const float* x, size_t n, size_t d,
                         const double* dictionaries, size_t M, size_t k, size_t sub_dimension,
                         const aq_weights* w, int passes, uint32_t* codes_out) {
  if (!m || !w) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  if (d != M * sub_dimension)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "dataset dimension does not match codebook");
  if (passes < 0) return ref_error(AQ_E_INVALID_ARGUMENT, "passes must be >= 0");
  const size_t W = m->s.size();
  return run_shards(m, [&](size_t r) -> int {
    size_t lo, hi;
    shard_bounds(n, W, r, &lo, &hi);
    if (hi == lo) return AQ_OK;
    const aq_weights wr = shard_weights(w, lo);
    aq_session* s = m->s[r];
    aq_dataset* ds = nullptr;
    aq_codebook* cb = nullptr;
    aq_codes* codes = nullptr;
    int st = aq_dataset_upload(s, x + lo * d, hi - lo, d, &ds);
    if (st == AQ_OK) st = aq_codebook_upload(s, dictionaries, M, k, sub_dimension, &cb);
    if (st == AQ_OK) st = aq_codes_alloc(s, hi - lo, M, k, &codes);
    if (st == AQ_OK) st = clear_dev_error(s);
    // device errors carry global point indices (base = lo)
    if (st == AQ_OK) st = run_encode_chunk(ds, cb, &wr, codes, passes, lo);
    if (st == AQ_OK) st = sync_and_check(s, "encode");
    if (st == AQ_OK) st = aq_codes_download(codes, codes_out + lo * M);
    aq_codes_free(codes);
    aq_codebook_free(cb);
    aq_dataset_free(ds);
    return st;
  });
}

// Batched adc_search (index.hpp:118-134) over row shards of host codes:
// per-shard exact top-N, merged on shard 0 in (score desc, index asc) order.
int aq_multi_adc_search(aq_multi* m, const double* queries, size_t nq, size_t d,
                        const uint32_t* codes, size_t n, size_t codes_M, size_t codes_k,
                        const double* dictionaries, size_t cb_M, size_t k, size_t sub_dimension,
                        size_t topn, uint32_t* ids_out, double* scores_out) {
  if (!m) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  if (n == 0) return ref_error(AQ_E_EMPTY_INDEX, "no quantized datapoints");
  if (topn < 1) return ref_error(AQ_E_INVALID_ARGUMENT, "topn must be >= 1");
  if (codes_M != cb_M || codes_k > k)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "code matrix does not match codebook");
  if (d != cb_M * sub_dimension)
    return ref_error(AQ_E_DIMENSION_MISMATCH, "query dimension does not match codebook");
  if (nq == 0) return AQ_OK;
  for (size_t e = 0; e < n * codes_M; ++e)
    if (codes[e] >= k) return ref_error(AQ_E_CODE_OUT_OF_RANGE, "code exceeds codebook size");
  const size_t W = m->s.size();
  const size_t topn_eff = std::min(topn, n);
  size_t te_max = 0;
  for (size_t r = 0; r < W; ++r) {
    size_t lo, hi;
    shard_bounds(n, W, r, &lo, &hi);
    te_max = std::max(te_max, std::min(topn, hi - lo));
  }
  // shard 0 holds the merge buffers: [r][q][te_max] global ids and scores
  aq_session* s0 = m->s[0];
  cudaSetDevice(s0->device);
  uint64_t* gid = nullptr;
  double* gsc = nullptr;
  uint32_t* oid = nullptr;
  double* osc = nullptr;
  AQ_CUDA(cudaMalloc(&gid, W * nq * te_max * sizeof(uint64_t)));
  AQ_CUDA(cudaMalloc(&gsc, W * nq * te_max * sizeof(double)));
  AQ_CUDA(cudaMalloc(&oid, nq * topn_eff * sizeof(uint32_t)));
  AQ_CUDA(cudaMalloc(&osc, nq * topn_eff * sizeof(double)));
  // padding: score -inf, id ~0 (sorts after every real candidate)
  {
    std::vector<double> ninf(W * nq * te_max, -INFINITY);
    cudaMemcpy(gsc, ninf.data(), ninf.size() * 8, cudaMemcpyHostToDevice);
    cudaMemset(gid, 0xff, W * nq * te_max * sizeof(uint64_t));
  }
  int st = run_shards(m, [&](size_t r) -> int {
    size_t lo, hi;
    shard_bounds(n, W, r, &lo, &hi);
    if (hi == lo) return AQ_OK;
    aq_session* s = m->s[r];
    const size_t te = std::min(topn, hi - lo);
    aq_codes* cm = nullptr;
    aq_codebook* cb = nullptr;
    double* Qd = nullptr;
    uint32_t* ids = nullptr;
    uint64_t* g64 = nullptr;
    double* sc = nullptr;
    int st = aq_codes_upload(s, codes + lo * codes_M, hi - lo, codes_M, codes_k, &cm);
    if (st == AQ_OK) st = aq_codebook_upload(s, dictionaries, cb_M, k, sub_dimension, &cb);
    if (st == AQ_OK && (cudaMalloc(&Qd, nq * d * 8) != cudaSuccess ||
                        cudaMalloc(&ids, nq * te * 4) != cudaSuccess ||
                        cudaMalloc(&g64, nq * te * 8) != cudaSuccess ||
                        cudaMalloc(&sc, nq * te * 8) != cudaSuccess))
      st = ref_error(AQ_E_CUDA, "out of device memory");
    if (st == AQ_OK)
      st = cudaMemcpy(Qd, queries, nq * d * 8, cudaMemcpyHostToDevice) == cudaSuccess
               ? AQ_OK
               : ref_error(AQ_E_CUDA, "query upload failed");
    if (st == AQ_OK) st = adc_search_device(cm, cb, Qd, nq, topn, ids, sc);
    if (st == AQ_OK) {
      k_offset_ids<<<(unsigned)((nq * te + 255) / 256), 256, 0, s->stream>>>(ids, nq * te, lo,
                                                                            g64);
      // rows of te entries into the [r][q][te_max] blocks on shard 0
      for (size_t q = 0; q < nq && st == AQ_OK; ++q) {
        const size_t at = (r * nq + q) * te_max;
        if (cudaMemcpyPeerAsync(gid + at, s0->device, g64 + q * te, s->device, te * 8,
                                s->stream) != cudaSuccess ||
            cudaMemcpyPeerAsync(gsc + at, s0->device, sc + q * te, s->device, te * 8,
                                s->stream) != cudaSuccess)
          st = ref_error(AQ_E_CUDA, "peer copy failed");
      }
      if (cudaStreamSynchronize(s->stream) != cudaSuccess)
        st = ref_error(AQ_E_CUDA, "shard search failed");
    }
    cudaFree(Qd);
    cudaFree(ids);
    cudaFree(g64);
    cudaFree(sc);
    aq_codebook_free(cb);
    aq_codes_free(cm);
    return st;
  });
  if (st == AQ_OK) {
    cudaSetDevice(s0->device);
    int P = 1;
    while ((size_t)P < W * te_max) P <<= 1;
    const size_t smem = (size_t)P * 16;
    if (smem > 227 * 1024) {
      st = ref_error(AQ_E_UNSUPPORTED, "multi-device merge window exceeds shared memory");
    } else {
      cudaFuncSetAttribute(k_merge_lists, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      k_merge_lists<<<(unsigned)nq, 512, smem, s0->stream>>>(gid, gsc, (int)W, (int)te_max,
                                                             (int)topn_eff, nq, oid, osc);
      s0->launches++;
      if (cudaMemcpyAsync(ids_out, oid, nq * topn_eff * 4, cudaMemcpyDeviceToHost,
                          s0->stream) != cudaSuccess ||
          cudaMemcpyAsync(scores_out, osc, nq * topn_eff * 8, cudaMemcpyDeviceToHost,
                          s0->stream) != cudaSuccess ||
          cudaStreamSynchronize(s0->stream) != cudaSuccess)
        st = ref_error(AQ_E_CUDA, "merge failed");
    }
  }
  cudaSetDevice(s0->device);
  cudaFree(gid);
  cudaFree(gsc);
  cudaFree(oid);
  cudaFree(osc);
  return st;
}

// train_apq (pq.hpp:513-575) over row shards; history_out holds
// max_iterations + 1 values.
int aq_multi_train_apq(aq_multi* m, const float* x, size_t n, size_t d, size_t M, size_t k,
                       const aq_weights* w, const aq_train_config* cfg, int warm_start,
                       double* dict_out, uint32_t* codes_out, double* history_out,
                       size_t* history_len) {
  if (!m || !w || !cfg) return ref_error(AQ_E_INVALID_ARGUMENT, "null argument");
  if (n == 0) return ref_error(AQ_E_EMPTY_DATASET, "cannot train on an empty dataset");
  if (M == 0 || d % M != 0)
    return ref_error(AQ_E_DIMENSION_NOT_DIVISIBLE, "dimension not divisible by M");
  if (k == 0 || k > n) return ref_error(AQ_E_INVALID_ARGUMENT, "need 1 <= k <= n");
  if (m->s.size() == 1 || M == 1 || d / M > 16)  // one shard / the VQ update: one device
    return aq_train_apq(m->s[0], x, n, d, M, k, w, cfg, warm_start, dict_out, codes_out,
                        history_out, history_len);
  Trainer t(m, x, n, d, w);
  AQ_TRY(t.upload());
  std::vector<double> dict, hist;
  AQ_TRY(t.train_apq(M, k, cfg, warm_start, &dict, &hist));
  std::memcpy(dict_out, dict.data(), dict.size() * sizeof(double));
  std::memcpy(history_out, hist.data(), hist.size() * sizeof(double));
  if (history_len) *history_len = hist.size();
  return t.download_codes(codes_out, M);
}

}  // extern "C"
