// covap_plan.hpp — host planner of the B200 COVAP path (internal).
//
// Integer-exact restatement of the reference planner and selection rule,
// compiled into the device-facing send layout:
//   buckets          allocate_buckets   (model.cpp:36-60)
//   twice_median     median_numel       (model.cpp:66-82)
//   tensors          shard_plan + effective_tensors (model.cpp:95-137)
//   phases[p]        select_tensors at step ≡ p (mod K) (compress.cpp:13-28),
//                    as runs of consecutive selected tensors + send offsets
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "covap_internal.h"

namespace covapb {

struct PlanBucket {
  uint64_t numel = 0;
  uint64_t begin = 0;   // flat element offset
  uint64_t dbegin = 0;  // device offset (== begin unless the plan is padded)
  uint64_t bytes = 0;
  uint64_t first_layer = 0;
  uint64_t n_layers = 0;
};

struct PlanTensor {
  uint64_t bucket = 0;
  uint64_t begin = 0;  // flat
  uint64_t end = 0;
  uint64_t dbegin = 0;  // device
  uint64_t dend = 0;
};

struct BucketSel {
  uint64_t sel_begin = 0, sel_end = 0;  // device coordinates; empty when equal
  uint64_t send_offset = 0;
};

struct Phase {
  std::vector<uint8_t> keep;          // per effective tensor
  std::vector<Run> runs;              // maximal runs of selected tensors (device coords)
  std::vector<BucketSel> per_bucket;  // at most one selected range per bucket
  uint64_t send_elems = 0;            // send-buffer length incl. alignment gaps
  uint64_t payload_elems = 0;         // sum of selected numels
};

struct Plan {
  uint64_t n_layers = 0;
  std::vector<PlanBucket> buckets;
  std::vector<PlanTensor> tensors;
  uint64_t twice_median = 0;
  uint64_t total = 0;   // N
  uint64_t dtotal = 0;  // device arena length (N plus bucket padding)
  bool padded = false;
  uint32_t interval = 1;
  int rule = 0;
  bool sharded = false;
  std::vector<Phase> phases;  // K entries
  uint64_t max_send = 0;
};

// Throws covap::InvalidInput exactly where the reference does.
Plan build_plan(const uint64_t* layer_numel, const uint32_t* bytes_per_param, size_t n_layers,
                uint64_t cap_bytes, uint32_t interval, int rule, int shard, bool pad = false);

uint64_t median_twice(std::vector<uint64_t> sizes);                       // model.cpp:66-82
std::vector<uint8_t> select(uint64_t step, uint32_t interval, size_t count, int rule);
double ef_coefficient(uint64_t step, int enabled, double init, uint64_t ascend, double range);
double ccr(double comm_ms, double comp_ms);                                // perf.cpp:40-47
uint32_t choose_interval(double ccr_value);                                // perf.cpp:49-53

struct Schedule {  // OverlapSchedule (perf.hpp:40-58)
  double total = 0.0, stream_end = 0.0, unoverlapped = 0.0;
  std::vector<double> comm_start, comm_end;
  std::vector<int64_t> comm_tensor;
  std::vector<std::pair<int64_t, double>> bubbles;  // (after tensor, duration)
};
Schedule overlap_schedule(double before_ms, const double* comp_ms, const double* compress_ms,
                          const double* comm_ms, const uint8_t* communicated, size_t n);

}  // namespace covapb
