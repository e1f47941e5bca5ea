#pragma once
// The C++ face of the B200 COVAP path: the hot-path subset of the reference
// library's public API (proj/include/covap/{compress,model,perf,sim,trainer,
// rng}.hpp), re-implemented over the C-ABI of libcovap_b200.so
// (include/covap_c.h).  Same names, argument meaning, value semantics and
// exception classes, so reference callers — and the reference's own unit
// tests — compile against it unchanged; the arithmetic runs in the sm_100a
// kernels (fp64 instantiation, bit-exact with the reference's double code).
//
// The value-semantics functions copy host data to the device per call; the
// device-resident classes at the end (covap::b200::Plan/State/Comm/Sync) are
// the production interface.  Built into libcovap_cxx.so
// (paper_2311_04499_b200/csrc/covap_cxx.cpp).

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "covap/errors.hpp"
#include "covap_c.h"

namespace covap {

// ------------------------------------------------------------------ rng
// splitmix64 stream (the reference's generator, rng.hpp:12-66 — same
// algorithm, so seeds give the same streams).
class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : s_(seed) {}
  std::uint64_t next();
  double next_unit();                        // [0, 1), 53 random bits
  std::uint64_t next_below(std::uint64_t n); // unbiased, rejection sampling
  double next_normal();                      // Box-Muller, pairs cached

 private:
  std::uint64_t s_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag);

// ------------------------------------------------------------------ model
struct LayerSpec {
  std::string name;
  std::uint64_t param_count = 0;
  std::uint32_t bytes_per_param = 4;
  double backward_ms = 0.0;
  std::uint64_t bytes() const { return param_count * bytes_per_param; }
};

struct ModelSpec {
  static constexpr std::uint64_t kDefaultBucketCapBytes = 25ULL << 20;
  std::vector<LayerSpec> layers;  // backward completion order
  std::uint64_t bucket_cap_bytes = kDefaultBucketCapBytes;
  std::uint64_t total_params() const;
  double total_backward_ms() const;
  void validate() const;  // InvalidInput
};

struct Bucket {
  std::size_t index = 0;
  std::vector<std::size_t> layer_refs;
  std::uint64_t numel = 0;
  std::uint64_t bytes = 0;
};

struct Shard {
  std::size_t parent_bucket = 0;
  std::uint64_t begin_elem = 0, end_elem = 0;
  std::uint64_t numel() const { return end_elem - begin_elem; }
};

struct MedianNumel {
  std::uint64_t twice = 0;  // exact: twice the median is an integer
  double value() const { return static_cast<double>(twice) / 2.0; }
  std::uint64_t floor_ratio(std::uint64_t numel) const { return (2 * numel) / twice; }
};

struct BucketPlan {
  std::vector<Bucket> buckets;
  std::uint64_t cap_bytes = ModelSpec::kDefaultBucketCapBytes;
  std::vector<Shard> shards;
  bool bucket_is_sharded(std::size_t bucket_index) const;
  std::uint64_t total_numel() const;
};

struct EffectiveTensor {
  std::size_t bucket = 0;
  std::uint64_t begin = 0, end = 0;  // global flat offsets
  std::uint64_t numel() const { return end - begin; }
};

BucketPlan allocate_buckets(const ModelSpec& model, std::uint64_t cap_bytes);
BucketPlan allocate_buckets(const ModelSpec& model);
MedianNumel median_numel(const BucketPlan& plan);
BucketPlan shard_plan(const BucketPlan& plan, std::uint32_t interval);
std::vector<EffectiveTensor> effective_tensors(const BucketPlan& plan);
std::vector<std::uint64_t> effective_numels(const BucketPlan& plan);

// ------------------------------------------------------------------ compress
using TensorVec = std::vector<double>;
using GradientSet = std::vector<TensorVec>;  // one vector per effective tensor

enum class SelectionRule { kMatchStep, kPlusStep };

std::vector<std::size_t> select_tensors(std::uint64_t num_steps, std::uint32_t interval,
                                        std::size_t tensor_count,
                                        SelectionRule rule = SelectionRule::kMatchStep);

struct EfSchedule {
  bool enabled = true;
  double init_value = 0.3;
  std::uint64_t ascend_steps = 100;
  double ascend_range = 0.1;
};
double ef_coefficient(std::uint64_t num_steps, const EfSchedule& schedule);

struct CovapConfig {
  std::uint32_t interval = 1;
  SelectionRule rule = SelectionRule::kMatchStep;
  EfSchedule ef;
};

struct CompressorState {
  GradientSet residuals;
  std::uint64_t num_steps = 0;
  static CompressorState zeros(const std::vector<std::uint64_t>& numels);
};

struct CompressedUpdate {
  std::vector<std::size_t> selected;  // ascending
  GradientSet payload;                // payload[i] <-> selected[i]
  std::uint64_t step = 0;
  std::uint64_t payload_elements() const;
};

// K1 on the GPU (fp64): fold scheduled residuals in, pack the selected
// tensors, write the rest back as residuals, advance the step.
CompressedUpdate covap_compress(const GradientSet& gradients, CompressorState& state,
                                const CovapConfig& config);
// K2 on the GPU (fp64): payload at its tensor slots, zeros elsewhere.
GradientSet covap_decompress(const CompressedUpdate& update,
                             const std::vector<std::uint64_t>& numels);

// ------------------------------------------------------------------ baseline compressors
// (compress.hpp:66-164), on the GPU (covap_feedback.cu).

struct SparseSelection {
  std::vector<std::size_t> indices;
  std::vector<double> values;  // aligned with indices
};

// ceil(k_fraction * d) entries of largest magnitude; ties keep the lower index.
SparseSelection topk_compress(std::span<const double> x, double k_fraction);
// ceil(k_fraction * d) indices sampled uniformly without replacement from
// SplitMix64(seed), ascending.
SparseSelection randomk_compress(std::span<const double> x, double k_fraction, std::uint64_t seed);
// Nearest half-precision value, widened back; clamps to +-65504 and counts.
TensorVec fp16_roundtrip(std::span<const double> x, std::uint64_t* saturation_count = nullptr);
std::uint16_t half_bits_from_float(float value, bool* saturated = nullptr);
float float_from_half_bits(std::uint16_t bits);

// A dense view of a compressor (compress.hpp:95-102).  The built-in filters
// below run on the device; descriptor() names the kernel.  A user-defined
// subclass may override keep() / transmitted_elements() for direct calls;
// ErrorFeedback runs only the built-in filters (InvalidInput otherwise).
class GradientFilter {
 public:
  virtual ~GradientFilter() = default;
  virtual GradientSet keep(const GradientSet& gradients, std::uint64_t step) const;
  virtual std::uint64_t transmitted_elements(const GradientSet& gradients,
                                             std::uint64_t step) const;
  // kind < 0: not a built-in filter.
  virtual covap_filter descriptor() const { return covap_filter{-1, 1, 0, 0.0, 0}; }
};

class IdentityFilter final : public GradientFilter {
 public:
  covap_filter descriptor() const override { return covap_filter{COVAP_FILTER_IDENTITY, 1, 0, 0.0, 0}; }
};

class CovapFilter final : public GradientFilter {
 public:
  CovapFilter(std::uint32_t interval, SelectionRule rule = SelectionRule::kMatchStep)
      : interval_(interval), rule_(rule) {}
  covap_filter descriptor() const override {
    return covap_filter{COVAP_FILTER_COVAP, interval_, rule_ == SelectionRule::kPlusStep ? 1 : 0,
                        0.0, 0};
  }

 private:
  std::uint32_t interval_;
  SelectionRule rule_;
};

class TopkFilter final : public GradientFilter {
 public:
  explicit TopkFilter(double k_fraction) : k_fraction_(k_fraction) {}
  covap_filter descriptor() const override { return covap_filter{COVAP_FILTER_TOPK, 1, 0, k_fraction_, 0}; }

 private:
  double k_fraction_;
};

class RandomkFilter final : public GradientFilter {
 public:
  RandomkFilter(double k_fraction, std::uint64_t seed) : k_fraction_(k_fraction), seed_(seed) {}
  covap_filter descriptor() const override {
    return covap_filter{COVAP_FILTER_RANDOMK, 1, 0, k_fraction_, seed_};
  }

 private:
  double k_fraction_;
  std::uint64_t seed_;
};

class Fp16Filter final : public GradientFilter {
 public:
  covap_filter descriptor() const override { return covap_filter{COVAP_FILTER_FP16, 1, 0, 0.0, 0}; }
};

// Residual accumulation around any built-in filter (compress.hpp:151-164):
// G += coeff * residuals before filtering, residuals = G - kept afterwards.
// Value semantics as in the reference (residuals live on the host between
// steps); the step itself runs in the device kernels.
class ErrorFeedback {
 public:
  ErrorFeedback(const std::vector<std::uint64_t>& numels, EfSchedule schedule);
  ~ErrorFeedback();
  ErrorFeedback(const ErrorFeedback&) = delete;
  ErrorFeedback& operator=(const ErrorFeedback&) = delete;

  GradientSet step(const GradientSet& gradients, const GradientFilter& filter);

  const GradientSet& residuals() const { return residuals_; }
  std::uint64_t num_steps() const { return num_steps_; }

 private:
  struct Device;
  std::vector<std::uint64_t> numels_;
  GradientSet residuals_;
  EfSchedule schedule_;
  std::uint64_t num_steps_ = 0;
  std::unique_ptr<Device> dev_;
};

// ------------------------------------------------------------------ trainer
// (0 + v_0 + ... + v_{P-1}) * (1/P) in worker order, on the GPU.
std::vector<double> allreduce_mean(const std::vector<std::vector<double>>& per_worker);

// ------------------------------------------------------------------ perf / sim
double ccr(double comm_ms, double comp_ms);
std::uint32_t choose_interval(double ccr_value);

// overlap_schedule (perf.hpp:37-58, perf.cpp:63-103): the exact overlapped
// iteration of per-tensor compute / compression / communication times.
struct ScheduleBubble {
  std::int64_t after_tensor = 0;
  double duration_ms = 0.0;
};
struct OverlapSchedule {
  double total_ms = 0.0;
  double stream_end_ms = 0.0;
  double unoverlapped_comm_ms = 0.0;
  std::vector<double> comm_start_ms;  // communicated tensors only
  std::vector<double> comm_end_ms;
  std::vector<std::int64_t> comm_tensor;
  std::vector<ScheduleBubble> bubbles;
};
OverlapSchedule overlap_schedule(double before_ms, std::span<const double> comp_ms,
                                 std::span<const double> compress_ms,
                                 std::span<const double> comm_ms,
                                 const std::vector<bool>& communicated = {});

enum class EventKind { kComputeStart, kComputeEnd, kCompressStart, kCompressEnd, kCommStart, kCommEnd };
struct Event {
  EventKind kind;
  std::int64_t tensor;
  std::uint32_t worker;
  double time_ms;
};
// One worker's (or every worker's) trace of an iteration (sim.hpp:45-52).
struct IterationTimeline {
  std::vector<Event> events;
  double t_total_ms = 0.0;
  std::vector<ScheduleBubble> bubbles;
  double unoverlapped_comm_ms = 0.0;
  std::uint64_t transmitted_bytes = 0;
};
struct ProfileResult {
  double ccr = 0.0;
  double comp_ms = 0.0;
  double comm_aligned_ms = 0.0;
  std::vector<double> naive_comm_ms;
  std::uint32_t recommended_interval = 1;
};
ProfileResult profile_ccr(std::span<const IterationTimeline> per_worker,
                          std::uint32_t expected_workers);

// ------------------------------------------------------------------ settings (a17)
// The "covap" section of an experiment document (config.cpp:133-157),
// parsed natively (covap_settings_from_json): ConfigError with the field
// path on a bad value; the document's other sections are not read.
struct CovapSettings {
  std::uint32_t interval = 1;
  bool auto_interval = false;  // "auto": K = choose_interval(measured CCR)
  SelectionRule rule = SelectionRule::kMatchStep;
  EfSchedule ef;
  CovapConfig config(std::uint32_t k) const { return CovapConfig{k, rule, ef}; }
};
CovapSettings covap_settings_from_json(const std::string& document);
// resolve_interval (config.cpp:238-241)
std::uint32_t resolve_interval(const CovapSettings& settings, double ccr_value);

// ------------------------------------------------------------------ device-resident API
namespace b200 {

namespace detail {
[[noreturn]] void raise(covap_status st);
inline void check(covap_status st) {
  if (st != COVAP_OK) raise(st);
}
}  // namespace detail

class Comm;

// BucketPlan + effective tensors + per-phase send layout for one K.
class Plan {
 public:
  Plan(const ModelSpec& model, std::uint32_t interval,
       SelectionRule rule = SelectionRule::kMatchStep, int shard = -1);
  const covap_plan* get() const { return p_.get(); }
  covap_plan_info info() const;

 private:
  std::shared_ptr<covap_plan> p_;
};

// CompressorState resident on one GPU (fp32 or fp64 arena).
class State {
 public:
  State(const Plan& plan, int dtype, int device, const EfSchedule& ef);
  covap_state* get() const { return s_.get(); }
  std::uint64_t num_steps() const;

 private:
  std::shared_ptr<covap_state> s_;
};

class Comm {
 public:
  static std::vector<std::uint8_t> unique_id();
  Comm(const std::vector<std::uint8_t>& id, int nranks, int rank, int device);
  covap_comm* get() const { return c_.get(); }
  const std::shared_ptr<covap_comm>& shared() const { return c_; }

 private:
  std::shared_ptr<covap_comm> c_;
};

// One rank's gradient synchronisation (trainer.cpp:365-386 per rank).
class Sync {
 public:
  Sync(const Plan& plan, const Comm* comm, int dtype, int device, const EfSchedule& ef);
  void step(const void* grad, void* out, void* stream);                   // covap_sync_step
  void bucket_ready(std::size_t bucket, const void* grad, void* out, void* stream);
  void dense_bucket_ready(std::size_t bucket, void* grad, void* out, void* stream);
  void finish(void* stream);
  // Per bucket: this rank's arrival -> completion time of its last
  // collective, ms (-1: none ran).  Blocks on the side stream.
  std::vector<double> last_comm_ms();
  State& state() { return state_; }

 private:
  State state_;
  covap_comm* comm_;
  std::size_t n_buckets_;
};

// One rank's synchronisation with C1 as the NVLink peer collective
// (covap_peer_*) on `state`: the send buffers in an NCCL symmetric window on
// comm (collective over its ranks), reduced in rank order — bit-identical to
// allreduce_mean for any P — or, with multimem, in the NVSwitch (the NCCL
// tolerance).  mode: 0 all-gather then unpack, 1 the unpack fused into the
// collective kernel (default), 2 the whole step as one kernel.
class PeerSync {
 public:
  PeerSync(State& state, const Comm& comm, bool multimem = false, int mode = 1);
  void step(const void* grad, void* out, void* stream);  // covap_peer_sync_step
  bool multimem() const;
  void check_timeouts() const;                          // covap_peer_check

 private:
  covap_state* state_;
  std::shared_ptr<covap_comm> comm_;  // outlives the peer
  std::shared_ptr<covap_peer> p_;
};

// The CCR-driven choice of K on a live job (PAPER §IV-B, sim.cpp:164-216,
// perf.cpp:40-53): profile one dense iteration through Sync with the
// dense_bucket_ready schedule, then decide() with this rank's per-bucket
// durations and backward time — rank-min exchange over the communicator,
// rank 0's compute time; every rank gets the same result.
class CcrController {
 public:
  explicit CcrController(const Comm* comm) : comm_(comm ? comm->get() : nullptr) {}
  ProfileResult decide(const std::vector<double>& own_comm_ms, double own_comp_ms) const;
  // "auto" -> the decided K, else the configured one (config.cpp:238-241).
  std::uint32_t interval(const CovapSettings& settings, const std::vector<double>& own_comm_ms,
                         double own_comp_ms) const;

 private:
  covap_comm* comm_;
};

}  // namespace b200
}  // namespace covap
