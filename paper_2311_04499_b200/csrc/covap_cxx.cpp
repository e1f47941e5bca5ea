// covap_cxx.cpp — the reference-compatible C++ API (include/covap/b200_api.hpp)
// implemented over the C-ABI (include/covap_c.h).  Host code only: every
// compute call goes to libcovap_b200.so's kernels; this file never touches
// CUDA directly.  Built into libcovap_cxx.so.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <tuple>

#include "covap/b200_api.hpp"

namespace covap {
namespace b200 {
namespace detail {

[[noreturn]] void raise(covap_status st) {
  const std::string msg = covap_last_error();
  switch (st) {
    case COVAP_ERR_INVALID_INPUT: throw InvalidInput(msg);
    case COVAP_ERR_INVALID_STATE: throw InvalidState(msg);
    case COVAP_ERR_UNDEFINED_RATIO: throw UndefinedRatio(msg);
    case COVAP_ERR_INCOMPLETE_PROFILE: throw IncompleteProfile(msg);
    case COVAP_ERR_CONFIG: throw ConfigError(msg);
    default: throw Error(msg);
  }
}

}  // namespace detail

using detail::check;

namespace {

covap_ef ef_of(const EfSchedule& e) {
  return covap_ef{e.enabled ? 1 : 0, e.init_value, e.ascend_steps, e.ascend_range};
}

int rule_of(SelectionRule r) { return r == SelectionRule::kPlusStep ? 1 : 0; }

// A device buffer owned by the C++ layer.
struct DevBuf {
  void* p = nullptr;
  uint64_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(uint64_t b) : bytes(b) { check(covap_device_alloc(0, b, &p)); }
  ~DevBuf() {
    if (p) covap_device_free(0, p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// One layer per effective tensor and a 1-byte cap give one bucket per
// tensor, unsharded: the plan's tensors are exactly the GradientSet's.
struct FlatContext {
  std::vector<uint64_t> numels;
  std::vector<uint64_t> offsets;
  uint64_t total = 0;
  Plan plan;
  State state;
  std::unique_ptr<DevBuf> grad;

  FlatContext(const std::vector<uint64_t>& nv, const CovapConfig& cfg)
      : numels(nv),
        plan(model_of(nv), cfg.interval, cfg.rule, 0),
        state(plan, COVAP_F64, 0, cfg.ef) {
    offsets.resize(nv.size());
    for (size_t t = 0; t < nv.size(); ++t) {
      offsets[t] = total;
      total += nv[t];
    }
    grad = std::make_unique<DevBuf>(std::max<uint64_t>(total, 1) * sizeof(double));
  }

  static ModelSpec model_of(const std::vector<uint64_t>& nv) {
    ModelSpec m;
    for (size_t t = 0; t < nv.size(); ++t) m.layers.push_back({"t" + std::to_string(t), nv[t], 4, 0.0});
    m.bucket_cap_bytes = 1;  // every tensor alone in its bucket
    return m;
  }
};

using ContextKey = std::tuple<std::vector<uint64_t>, uint32_t, int, int, double, uint64_t, double>;

FlatContext& context_for(const std::vector<uint64_t>& numels, const CovapConfig& cfg) {
  thread_local std::map<ContextKey, std::unique_ptr<FlatContext>> cache;
  ContextKey key{numels, cfg.interval, rule_of(cfg.rule), cfg.ef.enabled ? 1 : 0,
                 cfg.ef.init_value, cfg.ef.ascend_steps, cfg.ef.ascend_range};
  auto it = cache.find(key);
  if (it == cache.end()) {
    if (cache.size() > 16) cache.clear();
    it = cache.emplace(key, std::make_unique<FlatContext>(numels, cfg)).first;
  }
  return *it->second;
}

}  // namespace

// ------------------------------------------------------------------ Plan / State / Comm / Sync

Plan::Plan(const ModelSpec& model, std::uint32_t interval, SelectionRule rule, int shard) {
  std::vector<uint64_t> numel;
  std::vector<uint32_t> bpp;
  for (const auto& l : model.layers) {
    numel.push_back(l.param_count);
    bpp.push_back(l.bytes_per_param);
  }
  covap_plan* p = nullptr;
  check(covap_plan_create(numel.data(), bpp.data(), numel.size(), model.bucket_cap_bytes, interval,
                          rule_of(rule), shard, &p));
  p_.reset(p, covap_plan_destroy);
}

covap_plan_info Plan::info() const {
  covap_plan_info i;
  check(covap_plan_get_info(p_.get(), &i));
  return i;
}

State::State(const Plan& plan, int dtype, int device, const EfSchedule& ef) {
  covap_state* s = nullptr;
  const covap_ef e = ef_of(ef);
  check(covap_state_create(plan.get(), dtype, device, &e, &s));
  s_.reset(s, covap_state_destroy);
}

std::uint64_t State::num_steps() const {
  uint64_t n = 0;
  check(covap_state_get_step(s_.get(), &n));
  return n;
}

std::vector<std::uint8_t> Comm::unique_id() {
  std::vector<std::uint8_t> id(128);
  check(covap_comm_unique_id(id.data()));
  return id;
}

Comm::Comm(const std::vector<std::uint8_t>& id, int nranks, int rank, int device) {
  if (id.size() != 128) throw InvalidInput("NCCL unique id must be 128 bytes");
  covap_comm* c = nullptr;
  check(covap_comm_create(id.data(), nranks, rank, device, &c));
  c_.reset(c, covap_comm_destroy);
}

PeerSync::PeerSync(State& state, const Comm& comm, bool multimem, int mode)
    : state_(state.get()), comm_(comm.shared()) {
  covap_peer* p = nullptr;
  check(covap_peer_create_nccl(state_, comm_.get(), multimem ? 1 : 0, &p));
  p_.reset(p, covap_peer_destroy);
  check(covap_peer_set_fused(p, mode));
}

void PeerSync::step(const void* grad, void* out, void* stream) {
  check(covap_peer_sync_step(state_, p_.get(), grad, out, stream));
}

bool PeerSync::multimem() const {
  int on = 0;
  check(covap_peer_multimem(p_.get(), &on));
  return on != 0;
}

void PeerSync::check_timeouts() const { check(covap_peer_check(p_.get())); }

Sync::Sync(const Plan& plan, const Comm* comm, int dtype, int device, const EfSchedule& ef)
    : state_(plan, dtype, device, ef), comm_(comm ? comm->get() : nullptr),
      n_buckets_(plan.info().n_buckets) {}

void Sync::step(const void* grad, void* out, void* stream) {
  check(covap_sync_step(state_.get(), comm_, grad, out, stream));
}

void Sync::bucket_ready(std::size_t bucket, const void* grad, void* out, void* stream) {
  check(covap_bucket_ready(state_.get(), comm_, bucket, grad, out, stream));
}

void Sync::dense_bucket_ready(std::size_t bucket, void* grad, void* out, void* stream) {
  check(covap_dense_bucket_ready(state_.get(), comm_, bucket, grad, out, stream));
}

void Sync::finish(void* stream) { check(covap_step_finish(state_.get(), stream)); }

std::vector<double> Sync::last_comm_ms() {
  std::vector<double> d(n_buckets_);
  if (!d.empty()) check(covap_state_last_comm_ms(state_.get(), d.data(), d.size()));
  return d;
}

ProfileResult CcrController::decide(const std::vector<double>& own_comm_ms,
                                    double own_comp_ms) const {
  covap_ccr_result r{};
  check(covap_ccr_decide(comm_, own_comm_ms.data(), own_comm_ms.size(), own_comp_ms, &r));
  ProfileResult out;
  out.ccr = r.ccr;
  out.comp_ms = r.comp_ms;
  out.comm_aligned_ms = r.comm_aligned_ms;
  out.recommended_interval = r.recommended_interval;
  for (double x : own_comm_ms) out.naive_comm_ms.push_back(x > 0.0 ? x : 0.0);
  return out;
}

std::uint32_t CcrController::interval(const CovapSettings& settings,
                                      const std::vector<double>& own_comm_ms,
                                      double own_comp_ms) const {
  if (!settings.auto_interval) return resolve_interval(settings, 0.0);
  return resolve_interval(settings, decide(own_comm_ms, own_comp_ms).ccr);
}

}  // namespace b200

using b200::detail::check;

// ------------------------------------------------------------------ rng

std::uint64_t SplitMix64::next() {
  std::uint64_t z = (s_ += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double SplitMix64::next_unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

std::uint64_t SplitMix64::next_below(std::uint64_t n) {
  if (n == 0) return 0;
  const std::uint64_t floor = (0 - n) % n;  // reject the biased low range
  while (true) {
    const std::uint64_t x = next();
    if (x >= floor) return x % n;
  }
}

double SplitMix64::next_normal() {
  if (spare_ok_) {
    spare_ok_ = false;
    return spare_;
  }
  double u = next_unit();
  const double v = next_unit();
  while (u <= 0.0) u = next_unit();
  const double rad = std::sqrt(-2.0 * std::log(u));
  const double ang = 6.283185307179586476925286766559 * v;
  spare_ = rad * std::sin(ang);
  spare_ok_ = true;
  return rad * std::cos(ang);
}

std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t tag) {
  return SplitMix64(seed ^ (0x632be59bd9b4e019ULL + tag * 0x9e3779b97f4a7c15ULL)).next();
}

// ------------------------------------------------------------------ model

std::uint64_t ModelSpec::total_params() const {
  std::uint64_t n = 0;
  for (const auto& l : layers) n += l.param_count;
  return n;
}

double ModelSpec::total_backward_ms() const {
  double t = 0.0;
  for (const auto& l : layers) t += l.backward_ms;
  return t;
}

void ModelSpec::validate() const {
  if (layers.empty()) throw InvalidInput("model has no layers");
  for (const auto& l : layers) {
    if (l.param_count < 1) throw InvalidInput("layer '" + l.name + "' has param_count < 1");
    if (l.bytes_per_param != 2 && l.bytes_per_param != 4)
      throw InvalidInput("layer '" + l.name + "' has bytes_per_param outside {2, 4}");
    if (l.backward_ms < 0.0) throw InvalidInput("layer '" + l.name + "' has negative backward_ms");
  }
}

bool BucketPlan::bucket_is_sharded(std::size_t b) const {
  return std::any_of(shards.begin(), shards.end(),
                     [b](const Shard& s) { return s.parent_bucket == b; });
}

std::uint64_t BucketPlan::total_numel() const {
  std::uint64_t n = 0;
  for (const auto& b : buckets) n += b.numel;
  return n;
}

namespace {

// Buckets (and, when sharded, shards) of a native plan.
BucketPlan from_native(const ModelSpec& model, const b200::Plan& p, bool sharded) {
  const covap_plan_info info = p.info();
  std::vector<uint64_t> numel(info.n_buckets), begin(info.n_buckets), first(info.n_buckets),
      count(info.n_buckets);
  check(covap_plan_buckets(p.get(), numel.data(), begin.data(), first.data(), count.data()));
  BucketPlan out;
  out.cap_bytes = model.bucket_cap_bytes;
  for (size_t b = 0; b < info.n_buckets; ++b) {
    Bucket bk;
    bk.index = b;
    bk.numel = numel[b];
    for (uint64_t l = first[b]; l < first[b] + count[b]; ++l) {
      bk.layer_refs.push_back(l);
      bk.bytes += model.layers[l].bytes();
    }
    out.buckets.push_back(bk);
  }
  if (sharded) {
    std::vector<uint64_t> tb(info.n_tensors), t0(info.n_tensors), t1(info.n_tensors);
    check(covap_plan_tensors(p.get(), tb.data(), t0.data(), t1.data()));
    std::vector<size_t> per(info.n_buckets, 0);
    for (size_t t = 0; t < info.n_tensors; ++t) ++per[tb[t]];
    for (size_t t = 0; t < info.n_tensors; ++t)
      if (per[tb[t]] > 1)
        out.shards.push_back(Shard{tb[t], t0[t] - begin[tb[t]], t1[t] - begin[tb[t]]});
  }
  return out;
}

ModelSpec model_of_plan(const BucketPlan& plan) {
  // One synthetic layer per bucket and a cap no bucket exceeds alone but any
  // two do: re-bucketing reproduces the same buckets (bytes at 4 B/elem).
  ModelSpec m;
  for (const auto& b : plan.buckets) m.layers.push_back({"b" + std::to_string(b.index), b.numel, 4, 0.0});
  m.bucket_cap_bytes = 1;
  return m;
}

}  // namespace

BucketPlan allocate_buckets(const ModelSpec& model, std::uint64_t cap_bytes) {
  model.validate();
  ModelSpec m = model;
  m.bucket_cap_bytes = cap_bytes;
  b200::Plan p(m, 1, SelectionRule::kMatchStep, 0);
  BucketPlan out = from_native(model, p, false);
  out.cap_bytes = cap_bytes;
  return out;
}

BucketPlan allocate_buckets(const ModelSpec& model) {
  return allocate_buckets(model, model.bucket_cap_bytes);
}

MedianNumel median_numel(const BucketPlan& plan) {
  std::vector<uint64_t> sizes;
  for (const auto& b : plan.buckets) sizes.push_back(b.numel);
  uint64_t twice = 0;
  check(covap_median_twice(sizes.data(), sizes.size(), &twice));
  return MedianNumel{twice};
}

BucketPlan shard_plan(const BucketPlan& plan, std::uint32_t interval) {
  if (interval < 1) throw InvalidInput("shard interval must be >= 1");
  if (plan.buckets.empty()) throw InvalidInput("median_numel needs at least one bucket");
  b200::Plan p(model_of_plan(plan), interval, SelectionRule::kMatchStep, 1);
  const covap_plan_info info = p.info();
  std::vector<uint64_t> tb(info.n_tensors), t0(info.n_tensors), t1(info.n_tensors);
  check(covap_plan_tensors(p.get(), tb.data(), t0.data(), t1.data()));
  std::vector<uint64_t> base(plan.buckets.size(), 0);
  for (size_t b = 1; b < plan.buckets.size(); ++b) base[b] = base[b - 1] + plan.buckets[b - 1].numel;
  // A bucket is sharded when floor(numel / median) >= 2 (model.cpp:102-103),
  // even if the interval caps it at one part.
  const MedianNumel median{info.twice_median};
  BucketPlan out = plan;
  out.shards.clear();
  for (size_t t = 0; t < info.n_tensors; ++t)
    if (median.floor_ratio(plan.buckets[tb[t]].numel) >= 2)
      out.shards.push_back(Shard{tb[t], t0[t] - base[tb[t]], t1[t] - base[tb[t]]});
  return out;
}

std::vector<EffectiveTensor> effective_tensors(const BucketPlan& plan) {
  std::vector<EffectiveTensor> out;
  uint64_t base = 0;
  for (const auto& b : plan.buckets) {
    bool any = false;
    for (const auto& s : plan.shards) {
      if (s.parent_bucket != b.index) continue;
      out.push_back(EffectiveTensor{b.index, base + s.begin_elem, base + s.end_elem});
      any = true;
    }
    if (!any) out.push_back(EffectiveTensor{b.index, base, base + b.numel});
    base += b.numel;
  }
  return out;
}

std::vector<std::uint64_t> effective_numels(const BucketPlan& plan) {
  std::vector<std::uint64_t> out;
  for (const auto& t : effective_tensors(plan)) out.push_back(t.numel());
  return out;
}

// ------------------------------------------------------------------ compress

std::vector<std::size_t> select_tensors(std::uint64_t num_steps, std::uint32_t interval,
                                        std::size_t count, SelectionRule rule) {
  std::vector<uint8_t> keep(std::max<size_t>(count, 1));
  check(covap_select_tensors(num_steps, interval, count, b200::rule_of(rule), keep.data()));
  std::vector<std::size_t> out;
  for (size_t t = 0; t < count; ++t)
    if (keep[t]) out.push_back(t);
  return out;
}

double ef_coefficient(std::uint64_t num_steps, const EfSchedule& schedule) {
  const covap_ef e = b200::ef_of(schedule);
  double c = 0.0;
  check(covap_ef_coefficient(num_steps, &e, &c));
  return c;
}

CompressorState CompressorState::zeros(const std::vector<std::uint64_t>& numels) {
  CompressorState s;
  for (auto n : numels) s.residuals.emplace_back(n, 0.0);
  return s;
}

std::uint64_t CompressedUpdate::payload_elements() const {
  std::uint64_t n = 0;
  for (const auto& p : payload) n += p.size();
  return n;
}

CompressedUpdate covap_compress(const GradientSet& gradients, CompressorState& state,
                                const CovapConfig& config) {
  if (gradients.size() != state.residuals.size())
    throw InvalidState("gradient tensor count does not match compressor state");
  std::vector<uint64_t> numels;
  for (size_t t = 0; t < gradients.size(); ++t) {
    if (gradients[t].size() != state.residuals[t].size())
      throw InvalidState("gradient shape does not match residual shape at tensor " +
                         std::to_string(t));
    numels.push_back(gradients[t].size());
  }
  if (config.interval < 1) throw InvalidInput("selection interval must be >= 1");
  if (numels.empty()) throw InvalidInput("selection needs at least one tensor");
  if (config.ef.enabled && config.ef.ascend_steps < 1)
    throw InvalidInput("ascend_steps must be >= 1");
  for (auto n : numels)
    if (n == 0) throw InvalidInput("the device path needs non-empty tensors");

  b200::FlatContext& ctx = b200::context_for(numels, config);
  covap_state* st = ctx.state.get();
  void* res = nullptr;
  void* send = nullptr;
  uint64_t rn = 0, cap = 0;
  check(covap_state_residual(st, &res, &rn));
  check(covap_state_send(st, &send, &cap));
  // Upload gradient and residual store; run K1 at the state's step.
  std::vector<double> flat(ctx.total);
  for (size_t t = 0; t < gradients.size(); ++t)
    std::copy(gradients[t].begin(), gradients[t].end(), flat.begin() + ctx.offsets[t]);
  check(covap_memcpy(ctx.grad->p, flat.data(), ctx.total * 8, 0, nullptr));
  for (size_t t = 0; t < gradients.size(); ++t)
    std::copy(state.residuals[t].begin(), state.residuals[t].end(), flat.begin() + ctx.offsets[t]);
  check(covap_memcpy(res, flat.data(), ctx.total * 8, 0, nullptr));
  check(covap_state_set_step(st, state.num_steps));
  check(covap_filter_pack(st, ctx.grad->p, nullptr, 0, gradients.size(), nullptr));
  // Read back: residuals, and the selected tensors out of the send buffer.
  check(covap_memcpy(flat.data(), res, ctx.total * 8, 1, nullptr));
  std::vector<double> sendh(cap);
  check(covap_memcpy(sendh.data(), send, cap * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  for (size_t t = 0; t < gradients.size(); ++t)
    std::copy(flat.begin() + ctx.offsets[t], flat.begin() + ctx.offsets[t] + numels[t],
              state.residuals[t].begin());

  CompressedUpdate u;
  u.step = state.num_steps;
  std::vector<uint8_t> keep(numels.size());
  check(covap_plan_selection(ctx.plan.get(), state.num_steps, keep.data()));
  for (size_t t = 0; t < numels.size(); ++t) {
    if (!keep[t]) continue;
    covap_bucket_range br;
    check(covap_plan_bucket_range(ctx.plan.get(), state.num_steps, t, &br));
    u.selected.push_back(t);
    u.payload.emplace_back(sendh.begin() + br.send_offset,
                           sendh.begin() + br.send_offset + numels[t]);
  }
  ++state.num_steps;
  return u;
}

GradientSet covap_decompress(const CompressedUpdate& update,
                             const std::vector<std::uint64_t>& numels) {
  if (update.selected.size() != update.payload.size())
    throw InvalidInput("payload count does not match selected tensor count");
  std::vector<uint64_t> off(numels.size(), 0);
  uint64_t total = 0;
  for (size_t t = 0; t < numels.size(); ++t) {
    off[t] = total;
    total += numels[t];
  }
  std::vector<uint64_t> b, e, po;
  std::vector<double> packed;
  for (size_t i = 0; i < update.selected.size(); ++i) {
    const size_t t = update.selected[i];
    if (t >= numels.size()) throw InvalidInput("selected tensor index out of range");
    if (update.payload[i].size() != numels[t])
      throw InvalidInput("payload shape mismatch at tensor " + std::to_string(t));
    b.push_back(off[t]);
    e.push_back(off[t] + numels[t]);
    po.push_back(packed.size());
    packed.insert(packed.end(), update.payload[i].begin(), update.payload[i].end());
  }
  // Ascending ranges for the device run table (selection may be unsorted).
  std::vector<size_t> order(b.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return b[x] < b[y]; });
  std::vector<uint64_t> sb, se, so;
  for (size_t k : order) {
    if (!sb.empty() && b[k] < se.back()) throw InvalidInput("selected tensor appears twice");
    sb.push_back(b[k]);
    se.push_back(e[k]);
    so.push_back(po[k]);
  }
  GradientSet out;
  for (auto n : numels) out.emplace_back(n, 0.0);
  if (total == 0) return out;
  b200::DevBuf dpay(std::max<uint64_t>(packed.size(), 1) * 8), dout(total * 8);
  if (!packed.empty()) check(covap_memcpy(dpay.p, packed.data(), packed.size() * 8, 0, nullptr));
  check(covap_embed(0, COVAP_F64, dpay.p, dout.p, total, sb.data(), se.data(), so.data(), sb.size(),
                    1.0, 0, nullptr));
  std::vector<double> flat(total);
  check(covap_memcpy(flat.data(), dout.p, total * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  for (size_t t = 0; t < numels.size(); ++t)
    std::copy(flat.begin() + off[t], flat.begin() + off[t] + numels[t], out[t].begin());
  return out;
}

// ------------------------------------------------------------------ trainer / perf / sim

std::vector<double> allreduce_mean(const std::vector<std::vector<double>>& per_worker) {
  if (per_worker.empty()) throw InvalidInput("allreduce needs at least one worker vector");
  const size_t n = per_worker[0].size();
  for (const auto& v : per_worker)
    if (v.size() != n) throw InvalidInput("allreduce vectors differ in length");
  std::vector<double> out(n, 0.0);
  if (n == 0) return out;
  const size_t P = per_worker.size();
  std::vector<double> rows(P * n);
  for (size_t w = 0; w < P; ++w) std::copy(per_worker[w].begin(), per_worker[w].end(), rows.begin() + w * n);
  b200::DevBuf drows(rows.size() * 8), dout(n * 8);
  check(covap_memcpy(drows.p, rows.data(), rows.size() * 8, 0, nullptr));
  check(covap_mean_rows(0, COVAP_F64, drows.p, dout.p, P, n, nullptr));
  check(covap_memcpy(out.data(), dout.p, n * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  return out;
}

// ------------------------------------------------------------------ baseline compressors (§8(f4))

namespace {

std::vector<uint64_t> numels_of(const GradientSet& g) {
  std::vector<uint64_t> n;
  for (const auto& t : g) n.push_back(t.size());
  return n;
}

std::vector<double> flatten(const GradientSet& g, uint64_t total) {
  std::vector<double> flat;
  flat.reserve(total);
  for (const auto& t : g) flat.insert(flat.end(), t.begin(), t.end());
  return flat;
}

GradientSet unflatten(const std::vector<double>& flat, const std::vector<uint64_t>& numels) {
  GradientSet out;
  uint64_t off = 0;
  for (uint64_t n : numels) {
    out.emplace_back(flat.begin() + off, flat.begin() + off + n);
    off += n;
  }
  return out;
}

struct FeedbackHandle {
  covap_feedback* f = nullptr;
  ~FeedbackHandle() {
    if (f) covap_feedback_destroy(f);
  }
};

SparseSelection sparse_select(std::span<const double> x, double k_fraction, bool topk,
                              std::uint64_t seed) {
  uint64_t k = 0;
  check(covap_sparsifier_k(x.size(), k_fraction, &k));
  b200::DevBuf dx(x.size() * 8), di(x.size() * 8), dv(x.size() * 8);
  check(covap_memcpy(dx.p, x.data(), x.size() * 8, 0, nullptr));
  uint64_t got = 0;
  if (topk)
    check(covap_topk_compress(0, COVAP_F64, dx.p, x.size(), k_fraction, static_cast<uint64_t*>(di.p),
                              dv.p, &got, nullptr));
  else
    check(covap_randomk_compress(0, COVAP_F64, dx.p, x.size(), k_fraction, seed,
                                 static_cast<uint64_t*>(di.p), dv.p, &got, nullptr));
  std::vector<uint64_t> idx(got);
  SparseSelection out;
  out.values.resize(got);
  check(covap_memcpy(idx.data(), di.p, got * 8, 1, nullptr));
  check(covap_memcpy(out.values.data(), dv.p, got * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  out.indices.assign(idx.begin(), idx.end());
  return out;
}

}  // namespace

SparseSelection topk_compress(std::span<const double> x, double k_fraction) {
  return sparse_select(x, k_fraction, true, 0);
}

SparseSelection randomk_compress(std::span<const double> x, double k_fraction,
                                 std::uint64_t seed) {
  return sparse_select(x, k_fraction, false, seed);
}

TensorVec fp16_roundtrip(std::span<const double> x, std::uint64_t* saturation_count) {
  TensorVec out(x.size());
  if (x.empty()) return out;
  b200::DevBuf dx(x.size() * 8), dy(x.size() * 8);
  check(covap_memcpy(dx.p, x.data(), x.size() * 8, 0, nullptr));
  uint64_t sat = 0;
  check(covap_fp16_roundtrip(0, COVAP_F64, dx.p, x.size(), dy.p, &sat, nullptr));
  check(covap_memcpy(out.data(), dy.p, x.size() * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  if (saturation_count) *saturation_count += sat;
  return out;
}

std::uint16_t half_bits_from_float(float value, bool* saturated) {
  b200::DevBuf dx(4), dh(2);
  check(covap_memcpy(dx.p, &value, 4, 0, nullptr));
  uint64_t sat = 0;
  check(covap_fp16_encode(0, COVAP_F32, dx.p, 1, static_cast<uint16_t*>(dh.p), &sat, nullptr));
  std::uint16_t h = 0;
  check(covap_memcpy(&h, dh.p, 2, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  if (sat && saturated) *saturated = true;
  return h;
}

float float_from_half_bits(std::uint16_t bits) {
  b200::DevBuf dh(2), dx(4);
  check(covap_memcpy(dh.p, &bits, 2, 0, nullptr));
  check(covap_fp16_decode(0, static_cast<const uint16_t*>(dh.p), 1, static_cast<float*>(dx.p),
                          nullptr));
  float v = 0.0f;
  check(covap_memcpy(&v, dx.p, 4, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  return v;
}

// GradientFilter::keep for the built-in filters: one error-feedback step
// with compensation off (c = g), at `step`, on the device.
GradientSet GradientFilter::keep(const GradientSet& g, std::uint64_t step) const {
  const covap_filter d = descriptor();
  if (d.kind < 0) throw InvalidInput("keep() is not implemented by this filter");
  const auto numels = numels_of(g);
  if (numels.empty()) return {};
  uint64_t total = 0;
  for (auto n : numels) total += n;
  const covap_ef off{0, 0.0, 1, 0.0};
  FeedbackHandle h;
  check(covap_feedback_create(numels.data(), numels.size(), COVAP_F64, &off, &d, 0, &h.f));
  check(covap_feedback_set_step(h.f, step));
  b200::DevBuf dg(total * 8), dk(total * 8);
  const auto flat = flatten(g, total);
  check(covap_memcpy(dg.p, flat.data(), total * 8, 0, nullptr));
  check(covap_feedback_step(h.f, dg.p, dk.p, nullptr));
  std::vector<double> kept(total);
  check(covap_memcpy(kept.data(), dk.p, total * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  return unflatten(kept, numels);
}

std::uint64_t GradientFilter::transmitted_elements(const GradientSet& g,
                                                   std::uint64_t step) const {
  const covap_filter d = descriptor();
  if (d.kind < 0) throw InvalidInput("transmitted_elements() is not implemented by this filter");
  const auto numels = numels_of(g);
  if (numels.empty()) return 0;
  const covap_ef off{0, 0.0, 1, 0.0};
  FeedbackHandle h;
  check(covap_feedback_create(numels.data(), numels.size(), COVAP_F64, &off, &d, 0, &h.f));
  uint64_t e = 0;
  check(covap_feedback_transmitted(h.f, step, &e, nullptr));
  return e;
}

// The device state behind one ErrorFeedback, rebuilt when the filter changes.
struct ErrorFeedback::Device {
  covap_filter filter{};
  FeedbackHandle h;
  std::unique_ptr<b200::DevBuf> grad, kept;
};

ErrorFeedback::ErrorFeedback(const std::vector<std::uint64_t>& numels, EfSchedule schedule)
    : numels_(numels), schedule_(schedule) {
  residuals_.reserve(numels.size());
  for (std::uint64_t n : numels) residuals_.emplace_back(n, 0.0);
}

ErrorFeedback::~ErrorFeedback() = default;

GradientSet ErrorFeedback::step(const GradientSet& gradients, const GradientFilter& filter) {
  if (gradients.size() != residuals_.size())
    throw InvalidState("gradient tensor count does not match error-feedback state");
  for (size_t t = 0; t < gradients.size(); ++t)
    if (gradients[t].size() != residuals_[t].size())
      throw InvalidState("gradient shape mismatch at tensor " + std::to_string(t));
  const covap_filter d = filter.descriptor();
  if (d.kind < 0) throw InvalidInput("ErrorFeedback on the device runs the built-in filters");
  if (numels_.empty()) {
    ++num_steps_;
    return {};
  }
  uint64_t total = 0;
  for (auto n : numels_) total += n;
  const bool same = dev_ && dev_->filter.kind == d.kind && dev_->filter.interval == d.interval &&
                    dev_->filter.rule == d.rule && dev_->filter.k_fraction == d.k_fraction &&
                    dev_->filter.seed == d.seed;
  if (!same) {
    auto dv = std::make_unique<Device>();
    dv->filter = d;
    const covap_ef ef = b200::ef_of(schedule_);
    check(covap_feedback_create(numels_.data(), numels_.size(), COVAP_F64, &ef, &d, 0, &dv->h.f));
    dv->grad = std::make_unique<b200::DevBuf>(total * 8);
    dv->kept = std::make_unique<b200::DevBuf>(total * 8);
    dev_ = std::move(dv);
  }
  covap_feedback* f = dev_->h.f;
  void* res = nullptr;
  check(covap_feedback_residual(f, &res, nullptr));
  const auto g = flatten(gradients, total);
  const auto r = flatten(residuals_, total);
  check(covap_memcpy(dev_->grad->p, g.data(), total * 8, 0, nullptr));
  check(covap_memcpy(res, r.data(), total * 8, 0, nullptr));
  check(covap_feedback_set_step(f, num_steps_));
  check(covap_feedback_step(f, dev_->grad->p, dev_->kept->p, nullptr));
  std::vector<double> kept(total), rnew(total);
  check(covap_memcpy(kept.data(), dev_->kept->p, total * 8, 1, nullptr));
  check(covap_memcpy(rnew.data(), res, total * 8, 1, nullptr));
  check(covap_stream_synchronize(nullptr));
  residuals_ = unflatten(rnew, numels_);
  ++num_steps_;
  return unflatten(kept, numels_);
}

OverlapSchedule overlap_schedule(double before_ms, std::span<const double> comp_ms,
                                 std::span<const double> compress_ms,
                                 std::span<const double> comm_ms,
                                 const std::vector<bool>& communicated) {
  const size_t n = comp_ms.size();
  if (comm_ms.size() != n || (!compress_ms.empty() && compress_ms.size() != n) ||
      (!communicated.empty() && communicated.size() != n))
    throw InvalidInput("per-tensor lists have inconsistent lengths");
  std::vector<std::uint8_t> sent(communicated.begin(), communicated.end());
  OverlapSchedule o;
  o.comm_start_ms.resize(n);
  o.comm_end_ms.resize(n);
  o.comm_tensor.resize(n);
  std::vector<std::int64_t> after(n);
  std::vector<double> bubble(n);
  size_t nc = 0, nb = 0;
  check(covap_overlap_schedule(before_ms, comp_ms.data(),
                               compress_ms.empty() ? nullptr : compress_ms.data(), comm_ms.data(),
                               sent.empty() ? nullptr : sent.data(), n, &o.total_ms,
                               &o.stream_end_ms, &o.unoverlapped_comm_ms, o.comm_start_ms.data(),
                               o.comm_end_ms.data(), o.comm_tensor.data(), &nc, after.data(),
                               bubble.data(), &nb));
  o.comm_start_ms.resize(nc);
  o.comm_end_ms.resize(nc);
  o.comm_tensor.resize(nc);
  for (size_t i = 0; i < nb; ++i) o.bubbles.push_back(ScheduleBubble{after[i], bubble[i]});
  return o;
}

CovapSettings covap_settings_from_json(const std::string& document) {
  covap_settings c{};
  check(::covap_settings_from_json(document.c_str(), &c));
  CovapSettings s;
  s.interval = c.interval;
  s.auto_interval = c.auto_interval != 0;
  s.rule = c.rule == 1 ? SelectionRule::kPlusStep : SelectionRule::kMatchStep;
  s.ef = EfSchedule{c.ef.enabled != 0, c.ef.init_value, c.ef.ascend_steps, c.ef.ascend_range};
  return s;
}

std::uint32_t resolve_interval(const CovapSettings& settings, double ccr_value) {
  covap_settings c{};
  c.interval = settings.interval;
  c.auto_interval = settings.auto_interval ? 1 : 0;
  c.rule = settings.rule == SelectionRule::kPlusStep ? 1 : 0;
  c.ef = covap_ef{settings.ef.enabled ? 1 : 0, settings.ef.init_value, settings.ef.ascend_steps,
                  settings.ef.ascend_range};
  std::uint32_t k = 0;
  check(covap_resolve_interval(&c, ccr_value, &k));
  return k;
}

double ccr(double comm_ms, double comp_ms) {
  double c = 0.0;
  check(covap_ccr(comm_ms, comp_ms, &c));
  return c;
}

std::uint32_t choose_interval(double ccr_value) {
  uint32_t k = 0;
  check(covap_choose_interval(ccr_value, &k));
  return k;
}

ProfileResult profile_ccr(std::span<const IterationTimeline> per_worker,
                          std::uint32_t expected_workers) {
  if (per_worker.size() != expected_workers || expected_workers == 0)
    throw IncompleteProfile("expected " + std::to_string(expected_workers) +
                            " worker traces, got " + std::to_string(per_worker.size()));
  for (const auto& v : per_worker)
    if (v.events.empty()) throw IncompleteProfile("a worker trace is empty");
  // Gather arrivals per collective and the shared completions (sim.cpp:172-201).
  std::map<std::int64_t, std::pair<std::vector<double>, std::pair<double, size_t>>> coll;
  const size_t W = per_worker.size();
  for (size_t w = 0; w < W; ++w)
    for (const auto& e : per_worker[w].events) {
      if (e.kind == EventKind::kCommStart) {
        auto& c = coll[e.tensor];
        c.first.resize(W, NAN);
        c.first[w] = e.time_ms;
      } else if (e.kind == EventKind::kCommEnd) {
        auto& c = coll[e.tensor];
        c.first.resize(W, NAN);
        c.second.first = e.time_ms;
        ++c.second.second;
      }
    }
  std::vector<double> starts(W * coll.size()), ends(coll.size());
  size_t c = 0;
  for (const auto& [tensor, v] : coll) {
    for (size_t w = 0; w < W; ++w) {
      if (std::isnan(v.first[w]) || v.second.second != W)
        throw IncompleteProfile("collective for tensor " + std::to_string(tensor) +
                                " is missing worker arrivals");
      starts[w * coll.size() + c] = v.first[w];
    }
    ends[c++] = v.second.first;
  }
  double comp = 0.0;  // worker 0's compute time (sim.cpp:208-211)
  for (const auto& e : per_worker[0].events) {
    if (e.kind == EventKind::kComputeStart) comp -= e.time_ms;
    if (e.kind == EventKind::kComputeEnd) comp += e.time_ms;
  }
  ProfileResult r;
  r.naive_comm_ms.assign(W, 0.0);
  r.comp_ms = comp;
  check(covap_profile_ccr(starts.data(), ends.data(), W, expected_workers, coll.size(), comp,
                          &r.comm_aligned_ms, r.naive_comm_ms.data(), &r.ccr,
                          &r.recommended_interval));
  return r;
}

}  // namespace covap
