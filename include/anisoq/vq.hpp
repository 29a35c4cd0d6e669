// anisoq drop-in (B200): trainer configuration (reference vq.hpp:55-69).
#pragma once

#include <cstdint>

namespace anisoq {

enum class EmptyPartitionPolicy { reseed_highest_loss, keep_previous };

struct TrainConfig {
  int max_iterations = 100;
  double relative_tolerance = 1e-6;
  std::uint64_t seed = 0;
  EmptyPartitionPolicy empty_partition_policy = EmptyPartitionPolicy::reseed_highest_loss;
  double ridge = -1.0;
  int threads = 1;  // host knob of the reference; results never depend on it
  bool sweep_to_fixed_point = false;
};

}  // namespace anisoq
