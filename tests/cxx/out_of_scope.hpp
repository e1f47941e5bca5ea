// Declarations the reference's unit-test files mention but the B200 hot path
// does not provide (compute-time split, JSON I/O).  TEST
// INFRASTRUCTURE ONLY: force-included when compiling the reference's test
// sources so they build; the definitions (out_of_scope.cpp) throw, and the
// test cases that use them are skipped by name (tests/test_cxx_dropin.py).
// The baseline compressors and the error-feedback wrapper are NOT stubbed:
// they come from include/covap/b200_api.hpp (device kernels, §8(f4)).
#pragma once
#include <nlohmann/json_fwd.hpp>

#include "covap/b200_api.hpp"

namespace covap {

std::vector<double> split_compute_times(const ModelSpec&, const BucketPlan&, double);
ModelSpec model_from_json(const nlohmann::json&);
nlohmann::json model_to_json(const ModelSpec&);
nlohmann::json plan_to_json(const BucketPlan&);

}  // namespace covap
