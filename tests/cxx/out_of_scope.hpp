// Declarations the reference's unit-test files mention but the B200 hot path
// does not provide (baseline compressors, the
// generic error-feedback wrapper, compute-time split, JSON I/O).  TEST
// INFRASTRUCTURE ONLY: force-included when compiling the reference's test
// sources so they build; the definitions (out_of_scope.cpp) throw, and the
// test cases that use them are skipped by name (tests/test_cxx_dropin.py).
#pragma once
#include <nlohmann/json_fwd.hpp>

#include "covap/b200_api.hpp"

namespace covap {

struct SparseSelection {
  std::vector<std::size_t> indices;
  std::vector<double> values;
};
SparseSelection topk_compress(std::span<const double> x, double k_fraction);
SparseSelection randomk_compress(std::span<const double> x, double k_fraction, std::uint64_t seed);
TensorVec fp16_roundtrip(std::span<const double> x, std::uint64_t* saturation_count = nullptr);
std::uint16_t half_bits_from_float(float value, bool* saturated = nullptr);
float float_from_half_bits(std::uint16_t bits);

class GradientFilter {
 public:
  virtual ~GradientFilter() = default;
  virtual GradientSet keep(const GradientSet& gradients, std::uint64_t step) const = 0;
  virtual std::uint64_t transmitted_elements(const GradientSet& gradients, std::uint64_t step) const = 0;
};
class CovapFilter final : public GradientFilter {
 public:
  CovapFilter(std::uint32_t, SelectionRule = SelectionRule::kMatchStep) {}
  GradientSet keep(const GradientSet&, std::uint64_t) const override;
  std::uint64_t transmitted_elements(const GradientSet&, std::uint64_t) const override;
};
class TopkFilter final : public GradientFilter {
 public:
  explicit TopkFilter(double) {}
  GradientSet keep(const GradientSet&, std::uint64_t) const override;
  std::uint64_t transmitted_elements(const GradientSet&, std::uint64_t) const override;
};
class RandomkFilter final : public GradientFilter {
 public:
  RandomkFilter(double, std::uint64_t) {}
  GradientSet keep(const GradientSet&, std::uint64_t) const override;
  std::uint64_t transmitted_elements(const GradientSet&, std::uint64_t) const override;
};
class ErrorFeedback {
 public:
  ErrorFeedback(const std::vector<std::uint64_t>&, EfSchedule) {}
  GradientSet step(const GradientSet&, const GradientFilter&);
  const GradientSet& residuals() const { return r_; }

 private:
  GradientSet r_;
};

std::vector<double> split_compute_times(const ModelSpec&, const BucketPlan&, double);
ModelSpec model_from_json(const nlohmann::json&);
nlohmann::json model_to_json(const ModelSpec&);
nlohmann::json plan_to_json(const BucketPlan&);

}  // namespace covap
