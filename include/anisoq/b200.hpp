// anisoq drop-in (B200): process-wide device session and argument marshalling
// shared by the drop-in headers. Everything here is plumbing over the C ABI in
// include/anisoq_b200.h; the computation happens in libanisoq_b200.so.
#pragma once

#include <cstdlib>
#include <mutex>
#include <string>
#include <span>
#include <vector>

#include "error.hpp"
#include "geometry.hpp"

namespace anisoq::b200 {

// One session per process, on $ANISOQ_DEVICE (default 0), created lazily.
inline aq_session* session() {
  static aq_session* s = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* dev = std::getenv("ANISOQ_DEVICE");
    check(aq_session_create(dev ? std::atoi(dev) : 0, &s));
  });
  return s;
}

// $ANISOQ_DEVICES = "0,1,..." or "all": with two or more entries, a
// multi-device session over those GPUs (contiguous row shards, one session
// per entry); pq_quantize, adc_search and train_apq then use all of them
// (include/anisoq_b200.h, aq_multi_*). Unset or one device: nullptr.
inline aq_multi* multi() {
  static aq_multi* m = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("ANISOQ_DEVICES");
    if (!env) return;
    std::vector<int> devs;
    if (std::string(env) == "all") {
      int cnt = 0;
      check(aq_device_count(&cnt));
      for (int i = 0; i < cnt; ++i) devs.push_back(i);
    } else {
      for (const char* p = env; *p;) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) throw InvalidArgument("ANISOQ_DEVICES: expected a list of device ids");
        devs.push_back(static_cast<int>(v));
        p = *end == ',' ? end + 1 : end;
      }
    }
    if (devs.size() >= 2) check(aq_multi_create(devs.data(), (int)devs.size(), &m));
  });
  return m;
}

// aq_weights for a span of per-point weights: uniform spans (the common case,
// e.g. std::vector(n, from_eta(...))) are passed as one pair, otherwise as
// arrays that `hold` keeps alive for the call.
struct WeightArgs {
  aq_weights w{};
  std::vector<double> hp, ho;
};

inline void make_weights(std::span<const AnisotropicWeights> ws, WeightArgs& out) {
  out.w = aq_weights{};
  bool uniform = true;
  for (const auto& w : ws)
    uniform &= w.h_parallel == ws[0].h_parallel && w.h_perpendicular == ws[0].h_perpendicular;
  if (uniform && !ws.empty()) {
    out.w.mode = AQ_WEIGHTS_UNIFORM;
    out.w.h_parallel = ws[0].h_parallel;
    out.w.h_perpendicular = ws[0].h_perpendicular;
    return;
  }
  out.hp.resize(ws.size());
  out.ho.resize(ws.size());
  for (size_t i = 0; i < ws.size(); ++i) {
    out.hp[i] = ws[i].h_parallel;
    out.ho[i] = ws[i].h_perpendicular;
  }
  out.w.mode = AQ_WEIGHTS_PER_POINT;
  out.w.h_parallel_arr = out.hp.data();
  out.w.h_perpendicular_arr = out.ho.data();
}

template <class Handle, int (*Free)(Handle*)>
struct Owned {
  Handle* p = nullptr;
  Owned() = default;
  Owned(const Owned&) = delete;
  Owned& operator=(const Owned&) = delete;
  ~Owned() { Free(p); }
};
using OwnedDataset = Owned<aq_dataset, aq_dataset_free>;
using OwnedCodebook = Owned<aq_codebook, aq_codebook_free>;
using OwnedCodes = Owned<aq_codes, aq_codes_free>;

}  // namespace anisoq::b200
