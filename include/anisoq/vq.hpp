// anisoq drop-in (B200): trainer configuration (reference vq.hpp:55-69).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

namespace anisoq {

// A single (M = 1) codebook (reference vq.hpp:32-43): k codewords of dimension d.
struct Codebook {
  std::size_t k = 0;
  std::size_t d = 0;
  std::vector<double> codewords;  // row-major k*d

  std::span<const double> row(std::size_t j) const { return {codewords.data() + j * d, d}; }
  std::span<double> mutable_row(std::size_t j) { return {codewords.data() + j * d, d}; }
};

// Result of train_avq (reference vq.hpp:45-50).
struct VqAssignment {
  std::vector<std::uint32_t> assignments;  // one codeword index per datapoint
  std::vector<double> loss_history;        // total loss after each assignment pass
};

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
