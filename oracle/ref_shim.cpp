// ref_shim.cpp — extern "C" probe over the REFERENCE library's own C++ API.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libcovap_ref.so.  Nothing here re-implements the algorithm: each
// entry point converts flat arrays to the reference's value types and calls
// the reference function named in its comment, so tests and bench.py's
// reference arm run the unmodified reference code path.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <vector>

#include "covap/compress.hpp"
#include "covap/errors.hpp"
#include "covap/model.hpp"
#include "covap/perf.hpp"
#include "covap/sim.hpp"
#include "covap/trainer.hpp"

using namespace covap;

namespace {

int code_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const InvalidInput&) {
    return 1;
  } catch (const InvalidState&) {
    return 2;
  } catch (const UndefinedRatio&) {
    return 3;
  } catch (const IncompleteProfile&) {
    return 4;
  } catch (const ConfigError&) {
    return 5;
  } catch (const Error&) {
    return 6;
  } catch (...) {
    return 7;
  }
}

#define GUARD(...)                          \
  try {                                     \
    __VA_ARGS__;                            \
    return 0;                               \
  } catch (...) {                           \
    return code_of(std::current_exception()); \
  }

ModelSpec model_of(const std::uint64_t* numel, const std::uint32_t* bpp, std::size_t n) {
  ModelSpec m;
  for (std::size_t i = 0; i < n; ++i)
    m.layers.push_back({"l" + std::to_string(i), numel[i], bpp ? bpp[i] : 4u, 0.0});
  return m;
}

GradientSet split(const double* flat, const std::vector<std::uint64_t>& numels) {
  GradientSet g;
  g.reserve(numels.size());
  std::uint64_t off = 0;
  for (auto n : numels) {
    g.emplace_back(flat + off, flat + off + n);
    off += n;
  }
  return g;
}

}  // namespace

extern "C" {

// allocate_buckets (model.cpp:36) [+ shard_plan (model.cpp:95) when shard] +
// median_numel (model.cpp:66) + effective_tensors (model.cpp:117).
int ref_plan(const std::uint64_t* layer_numel, const std::uint32_t* bpp, std::size_t n_layers,
             std::uint64_t cap_bytes, std::uint32_t interval, int shard,
             std::uint64_t* bucket_numel, std::size_t cap_buckets, std::size_t* n_buckets,
             std::uint64_t* twice_median, std::uint64_t* t_bucket, std::uint64_t* t_begin,
             std::uint64_t* t_end, std::size_t cap_tensors, std::size_t* n_tensors) {
  GUARD({
    BucketPlan plan = allocate_buckets(model_of(layer_numel, bpp, n_layers), cap_bytes);
    if (plan.buckets.size() > cap_buckets) return 9;
    *n_buckets = plan.buckets.size();
    for (std::size_t b = 0; b < plan.buckets.size(); ++b) bucket_numel[b] = plan.buckets[b].numel;
    *twice_median = median_numel(plan).twice;
    if (shard) plan = shard_plan(plan, interval);
    const auto ts = effective_tensors(plan);
    if (ts.size() > cap_tensors) return 9;
    *n_tensors = ts.size();
    for (std::size_t t = 0; t < ts.size(); ++t) {
      t_bucket[t] = ts[t].bucket;
      t_begin[t] = ts[t].begin;
      t_end[t] = ts[t].end;
    }
  })
}

// select_tensors (compress.cpp:13).
int ref_select(std::uint64_t step, std::uint32_t interval, std::size_t count, int rule,
               std::uint64_t* out, std::size_t* n_out) {
  GUARD({
    const auto s = select_tensors(step, interval, count,
                                  rule ? SelectionRule::kPlusStep : SelectionRule::kMatchStep);
    *n_out = s.size();
    for (std::size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  })
}

// ef_coefficient (compress.cpp:30).
int ref_ef_coefficient(std::uint64_t step, int enabled, double init, std::uint64_t ascend,
                       double range, double* out) {
  GUARD({ *out = ef_coefficient(step, EfSchedule{enabled != 0, init, ascend, range}); })
}

// covap_compress (compress.cpp:50) on one worker.  residual (flat) and
// *num_steps are the CompressorState, read and written back.
int ref_compress(const double* g, const std::uint64_t* numels, std::size_t n_tensors,
                 double* residual, std::uint64_t* num_steps, std::uint32_t interval, int rule,
                 int ef_enabled, double init, std::uint64_t ascend, double range,
                 double* payload, std::uint64_t* selected, std::size_t* n_selected) {
  GUARD({
    std::vector<std::uint64_t> nv(numels, numels + n_tensors);
    CompressorState state;
    state.residuals = split(residual, nv);
    state.num_steps = *num_steps;
    CovapConfig cfg;
    cfg.interval = interval;
    cfg.rule = rule ? SelectionRule::kPlusStep : SelectionRule::kMatchStep;
    cfg.ef = EfSchedule{ef_enabled != 0, init, ascend, range};
    const auto u = covap_compress(split(g, nv), state, cfg);
    std::uint64_t off = 0;
    for (const auto& r : state.residuals) {
      std::memcpy(residual + off, r.data(), r.size() * sizeof(double));
      off += r.size();
    }
    *num_steps = state.num_steps;
    off = 0;
    for (const auto& p : u.payload) {
      std::memcpy(payload + off, p.data(), p.size() * sizeof(double));
      off += p.size();
    }
    *n_selected = u.selected.size();
    for (std::size_t i = 0; i < u.selected.size(); ++i) selected[i] = u.selected[i];
  })
}

// covap_decompress (compress.cpp:87).
int ref_decompress(const double* payload, const std::uint64_t* selected, std::size_t n_selected,
                   const std::uint64_t* numels, std::size_t n_tensors, double* out) {
  GUARD({
    std::vector<std::uint64_t> nv(numels, numels + n_tensors);
    CompressedUpdate u;
    std::uint64_t off = 0;
    for (std::size_t i = 0; i < n_selected; ++i) {
      u.selected.push_back(selected[i]);
      const std::uint64_t n = selected[i] < n_tensors ? numels[selected[i]] : 0;
      u.payload.emplace_back(payload + off, payload + off + n);
      off += n;
    }
    const auto full = covap_decompress(u, nv);
    off = 0;
    for (const auto& t : full) {
      std::memcpy(out + off, t.data(), t.size() * sizeof(double));
      off += t.size();
    }
  })
}

// allreduce_mean (trainer.cpp:35).
int ref_allreduce_mean(const double* per_worker, std::size_t P, std::size_t n, double* out) {
  GUARD({
    std::vector<std::vector<double>> v;
    for (std::size_t w = 0; w < P; ++w) v.emplace_back(per_worker + w * n, per_worker + (w + 1) * n);
    const auto m = allreduce_mean(v);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  })
}

// ccr / choose_interval (perf.cpp:40-53).
int ref_ccr(double comm, double comp, double* out) { GUARD({ *out = ccr(comm, comp); }) }
int ref_choose_interval(double c, std::uint32_t* out) { GUARD({ *out = choose_interval(c); }) }

// profile_ccr (sim.cpp:164) over per-worker timelines built from dense arrays.
// n_workers_given < expected exercises the IncompleteProfile path.
int ref_profile_ccr(const double* comm_start, const double* comm_end, std::size_t n_workers_given,
                    std::uint32_t expected, std::size_t n_coll, double comp_ms, double* aligned,
                    double* naive, double* ccr_out, std::uint32_t* interval_out) {
  GUARD({
    std::vector<IterationTimeline> views(n_workers_given);
    for (std::size_t w = 0; w < n_workers_given; ++w) {
      auto& ev = views[w].events;
      ev.push_back({EventKind::kComputeStart, 0, (std::uint32_t)w, 0.0});
      ev.push_back({EventKind::kComputeEnd, 0, (std::uint32_t)w, comp_ms});
      for (std::size_t c = 0; c < n_coll; ++c) {
        ev.push_back({EventKind::kCommStart, (std::int64_t)c, (std::uint32_t)w,
                      comm_start[w * n_coll + c]});
        ev.push_back({EventKind::kCommEnd, (std::int64_t)c, (std::uint32_t)w, comm_end[c]});
      }
    }
    const auto r = profile_ccr(views, expected);
    *aligned = r.comm_aligned_ms;
    for (std::size_t w = 0; w < r.naive_comm_ms.size(); ++w) naive[w] = r.naive_comm_ms[w];
    *ccr_out = r.ccr;
    *interval_out = r.recommended_interval;
  })
}

// ---------------------------------------------------------------------------
// The reference's COVAP sync sequence, trainer.cpp:365-386, minus the toy
// model: per worker split_by_tensors + covap_compress, one allreduce_mean per
// selected tensor, covap_decompress, add_flat into the update vector.  Used
// for parity of whole steps and as bench.py's reference (CPU) arm.

struct RefSession {
  std::vector<std::uint64_t> numels;
  std::vector<CompressorState> states;
  CovapConfig cfg;
};

void* ref_session_create(const std::uint64_t* numels, std::size_t n_tensors, std::uint32_t P,
                         std::uint32_t interval, int rule, int ef_enabled, double init,
                         std::uint64_t ascend, double range) {
  auto* s = new RefSession;
  s->numels.assign(numels, numels + n_tensors);
  s->states.assign(P, CompressorState::zeros(s->numels));
  s->cfg.interval = interval;
  s->cfg.rule = rule ? SelectionRule::kPlusStep : SelectionRule::kMatchStep;
  s->cfg.ef = EfSchedule{ef_enabled != 0, init, ascend, range};
  return s;
}

void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

// grads: P rows of d doubles (worker-major).  update: d doubles (the mean of
// the transmitted tensors, zeros elsewhere).  residual_w0 (optional): worker
// 0's residual store after the step.  *seconds: wall time of the sequence.
int ref_session_step(void* h, const double* grads, double* update, double* residual_w0,
                     double* seconds) {
  auto* s = static_cast<RefSession*>(h);
  GUARD({
    const auto t0 = std::chrono::steady_clock::now();
    const std::size_t P = s->states.size();
    std::uint64_t d = 0;
    for (auto n : s->numels) d += n;
    std::vector<CompressedUpdate> updates;
    updates.reserve(P);
    for (std::size_t w = 0; w < P; ++w)
      updates.push_back(covap_compress(split(grads + w * d, s->numels), s->states[w], s->cfg));
    CompressedUpdate mean = updates[0];
    for (std::size_t t = 0; t < mean.payload.size(); ++t) {
      std::vector<std::vector<double>> per_worker;
      per_worker.reserve(P);
      for (std::size_t w = 0; w < P; ++w) per_worker.push_back(updates[w].payload[t]);
      mean.payload[t] = allreduce_mean(per_worker);
    }
    const GradientSet dense = covap_decompress(mean, s->numels);
    std::uint64_t off = 0;
    for (const auto& t : dense) {
      for (std::size_t i = 0; i < t.size(); ++i) update[off + i] = 0.0 + 1.0 * t[i];  // add_flat
      off += t.size();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (residual_w0) {
      off = 0;
      for (const auto& r : s->states[0].residuals) {
        std::memcpy(residual_w0 + off, r.data(), r.size() * sizeof(double));
        off += r.size();
      }
    }
  })
}

}  // extern "C"

extern "C" {

// overlap_schedule (perf.cpp:63-103).
int ref_overlap_schedule(double before, const double* comp, const double* compress,
                         const double* comm, const uint8_t* communicated, std::size_t n,
                         double* total, double* stream_end, double* unoverlapped,
                         double* comm_start, double* comm_end, std::int64_t* comm_tensor,
                         std::size_t* n_comm, std::int64_t* bubble_after, double* bubble_ms,
                         std::size_t* n_bubbles) {
  GUARD({
    std::vector<bool> sent;
    if (communicated)
      for (std::size_t i = 0; i < n; ++i) sent.push_back(communicated[i] != 0);
    const auto sc = overlap_schedule(before, std::span<const double>(comp, n),
                                     compress ? std::span<const double>(compress, n)
                                              : std::span<const double>(),
                                     std::span<const double>(comm, n), sent);
    *total = sc.total_ms;
    *stream_end = sc.stream_end_ms;
    *unoverlapped = sc.unoverlapped_comm_ms;
    *n_comm = sc.comm_tensor.size();
    for (std::size_t i = 0; i < sc.comm_tensor.size(); ++i) {
      comm_start[i] = sc.comm_start_ms[i];
      comm_end[i] = sc.comm_end_ms[i];
      comm_tensor[i] = sc.comm_tensor[i];
    }
    *n_bubbles = sc.bubbles.size();
    for (std::size_t i = 0; i < sc.bubbles.size(); ++i) {
      bubble_after[i] = sc.bubbles[i].after_tensor;
      bubble_ms[i] = sc.bubbles[i].duration_ms;
    }
  })
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Baseline compressors and the generic error-feedback wrapper.
extern "C" {

// topk_compress (compress.cpp:119-133): indices in the reference's order
// (largest magnitude first, ties to the lower index) and their values.
int ref_topk(const double* x, std::size_t d, double k_fraction, std::uint64_t* indices,
             double* values, std::size_t* k) {
  GUARD({
    const auto s = topk_compress(std::span<const double>(x, d), k_fraction);
    *k = s.indices.size();
    for (std::size_t i = 0; i < s.indices.size(); ++i) {
      indices[i] = s.indices[i];
      values[i] = s.values[i];
    }
  })
}

// randomk_compress (compress.cpp:135-143): ascending indices.
int ref_randomk(const double* x, std::size_t d, double k_fraction, std::uint64_t seed,
                std::uint64_t* indices, double* values, std::size_t* k) {
  GUARD({
    const auto s = randomk_compress(std::span<const double>(x, d), k_fraction, seed);
    *k = s.indices.size();
    for (std::size_t i = 0; i < s.indices.size(); ++i) {
      indices[i] = s.indices[i];
      values[i] = s.values[i];
    }
  })
}

// fp16_roundtrip (compress.cpp:226-236) and half_bits_from_float (157-205).
int ref_fp16_roundtrip(const double* x, std::size_t n, double* out, std::uint64_t* saturated) {
  GUARD({
    std::uint64_t sat = 0;
    const auto y = fp16_roundtrip(std::span<const double>(x, n), &sat);
    for (std::size_t i = 0; i < n; ++i) out[i] = y[i];
    if (saturated) *saturated = sat;
  })
}

std::uint16_t ref_half_bits(float v, int* saturated) {
  bool s = false;
  const std::uint16_t h = half_bits_from_float(v, &s);
  if (saturated) *saturated = s ? 1 : 0;
  return h;
}

float ref_float_from_half(std::uint16_t h) { return float_from_half_bits(h); }

// ErrorFeedback (compress.cpp:316-344) around one GradientFilter
// (compress.cpp:241-314).  kind: 0 identity, 1 covap, 2 topk, 3 randomk, 4 fp16.
struct RefFeedback {
  std::vector<std::uint64_t> numels;
  std::unique_ptr<GradientFilter> filter;
  std::unique_ptr<ErrorFeedback> ef;
};

void* ref_feedback_create(const std::uint64_t* numels, std::size_t n, int kind,
                          std::uint32_t interval, int rule, double k_fraction,
                          std::uint64_t seed, int ef_enabled, double init, std::uint64_t ascend,
                          double range) {
  auto* s = new RefFeedback;
  s->numels.assign(numels, numels + n);
  switch (kind) {
    case 0: s->filter = std::make_unique<IdentityFilter>(); break;
    case 1:
      s->filter = std::make_unique<CovapFilter>(
          interval, rule ? SelectionRule::kPlusStep : SelectionRule::kMatchStep);
      break;
    case 2: s->filter = std::make_unique<TopkFilter>(k_fraction); break;
    case 3: s->filter = std::make_unique<RandomkFilter>(k_fraction, seed); break;
    default: s->filter = std::make_unique<Fp16Filter>(); break;
  }
  s->ef = std::make_unique<ErrorFeedback>(s->numels,
                                          EfSchedule{ef_enabled != 0, init, ascend, range});
  return s;
}

void ref_feedback_destroy(void* h) { delete static_cast<RefFeedback*>(h); }

// One ErrorFeedback::step on a flat gradient; kept and the residual come back
// flat.  *transmitted = filter.transmitted_elements(g, step) (trainer.cpp:397).
int ref_feedback_step(void* h, const double* g, double* kept, double* residual,
                      std::uint64_t* transmitted, double* seconds) {
  auto* s = static_cast<RefFeedback*>(h);
  GUARD({
    const GradientSet gs = split(g, s->numels);
    const std::uint64_t step = s->ef->num_steps();
    const auto t0 = std::chrono::steady_clock::now();
    const GradientSet k = s->ef->step(gs, *s->filter);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (transmitted) *transmitted = s->filter->transmitted_elements(gs, step);
    std::uint64_t off = 0;
    for (std::size_t t = 0; t < k.size(); ++t) {
      std::memcpy(kept + off, k[t].data(), k[t].size() * sizeof(double));
      if (residual)
        std::memcpy(residual + off, s->ef->residuals()[t].data(), k[t].size() * sizeof(double));
      off += k[t].size();
    }
  })
}

}  // extern "C"
