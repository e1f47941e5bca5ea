// Stubs for tests/cxx/out_of_scope.hpp — TEST INFRASTRUCTURE ONLY.
#include "out_of_scope.hpp"

#include <nlohmann/json.hpp>

namespace covap {
namespace {
[[noreturn]] void oos(const char* what) {
  throw Error(std::string("out of scope for the B200 hot path: ") + what);
}
}  // namespace
SparseSelection topk_compress(std::span<const double>, double) { oos("topk_compress"); }
SparseSelection randomk_compress(std::span<const double>, double, std::uint64_t) { oos("randomk_compress"); }
TensorVec fp16_roundtrip(std::span<const double>, std::uint64_t*) { oos("fp16_roundtrip"); }
std::uint16_t half_bits_from_float(float, bool*) { oos("half_bits_from_float"); }
float float_from_half_bits(std::uint16_t) { oos("float_from_half_bits"); }
GradientSet CovapFilter::keep(const GradientSet&, std::uint64_t) const { oos("CovapFilter"); }
std::uint64_t CovapFilter::transmitted_elements(const GradientSet&, std::uint64_t) const { oos("CovapFilter"); }
GradientSet TopkFilter::keep(const GradientSet&, std::uint64_t) const { oos("TopkFilter"); }
std::uint64_t TopkFilter::transmitted_elements(const GradientSet&, std::uint64_t) const { oos("TopkFilter"); }
GradientSet RandomkFilter::keep(const GradientSet&, std::uint64_t) const { oos("RandomkFilter"); }
std::uint64_t RandomkFilter::transmitted_elements(const GradientSet&, std::uint64_t) const { oos("RandomkFilter"); }
GradientSet ErrorFeedback::step(const GradientSet&, const GradientFilter&) { oos("ErrorFeedback"); }
std::vector<double> split_compute_times(const ModelSpec&, const BucketPlan&, double) { oos("split_compute_times"); }
ModelSpec model_from_json(const nlohmann::json&) { oos("model_from_json"); }
nlohmann::json model_to_json(const ModelSpec&) { oos("model_to_json"); }
nlohmann::json plan_to_json(const BucketPlan&) { oos("plan_to_json"); }
}  // namespace covap
