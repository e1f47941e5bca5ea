// covap_plan.cpp — host planner (see covap_plan.hpp for the reference map).
#include "covap_plan.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <string>

#include "covap/errors.hpp"

namespace covapb {

uint64_t median_twice(std::vector<uint64_t> sizes) {
  if (sizes.empty()) throw covap::InvalidInput("median_numel needs at least one bucket");
  std::sort(sizes.begin(), sizes.end(), std::greater<>());
  const size_t n = sizes.size(), mid = n / 2;
  if (n % 2 == 1) return 2 * sizes[mid];
  if (n == 2) return sizes[0] + sizes[1];
  // Even n > 2: the reference averages the pair one rank below the
  // conventional middle of the descending order (model.cpp:77-81).
  return sizes[mid] + sizes[mid + 1];
}

std::vector<uint8_t> select(uint64_t step, uint32_t interval, size_t count, int rule) {
  if (interval < 1) throw covap::InvalidInput("selection interval must be >= 1");
  if (count < 1) throw covap::InvalidInput("selection needs at least one tensor");
  const uint64_t phase = step % interval;
  std::vector<uint8_t> keep(count);
  for (size_t t = 0; t < count; ++t) {
    const uint64_t r = t % interval;
    keep[t] = rule == 0 ? (r == phase) : ((r + phase) % interval == 0);
  }
  return keep;
}

double ef_coefficient(uint64_t step, int /*enabled*/, double init, uint64_t ascend,
                      double range) {
  if (ascend < 1) throw covap::InvalidInput("ascend_steps must be >= 1");
  const double raised = init + static_cast<double>(step / ascend) * range;
  return std::min(raised, 1.0);
}

double ccr(double comm_ms, double comp_ms) {
  if (comm_ms < 0.0 || comp_ms < 0.0) throw covap::InvalidInput("phase times must be non-negative");
  if (comp_ms == 0.0) {
    if (comm_ms == 0.0) return 0.0;
    throw covap::UndefinedRatio("CCR is undefined for zero computation time");
  }
  return comm_ms / comp_ms;
}

uint32_t choose_interval(double ccr_value) {
  if (ccr_value < 0.0) throw covap::InvalidInput("CCR must be non-negative");
  const double up = std::ceil(ccr_value);
  return up < 1.0 ? 1u : static_cast<uint32_t>(up);
}

Plan build_plan(const uint64_t* layer_numel, const uint32_t* bpp, size_t n_layers,
                uint64_t cap_bytes, uint32_t interval, int rule, int shard, bool pad) {
  // ModelSpec::validate (model.cpp:24-34).
  if (n_layers == 0) throw covap::InvalidInput("model has no layers");
  for (size_t i = 0; i < n_layers; ++i) {
    const std::string name = "l" + std::to_string(i);
    if (layer_numel[i] < 1) throw covap::InvalidInput("layer '" + name + "' has param_count < 1");
    const uint32_t w = bpp ? bpp[i] : 4u;
    if (w != 2 && w != 4)
      throw covap::InvalidInput("layer '" + name + "' has bytes_per_param outside {2, 4}");
  }
  if (cap_bytes < 1) throw covap::InvalidInput("bucket capacity must be at least one byte");
  if (interval < 1) throw covap::InvalidInput("shard interval must be >= 1");
  if (rule != 0 && rule != 1) throw covap::InvalidInput("unknown selection rule");

  Plan plan;
  plan.n_layers = n_layers;
  plan.interval = interval;
  plan.rule = rule;

  // Greedy bucketing: a layer joins the open bucket unless that bucket is
  // non-empty and would exceed the cap (model.cpp:53); an oversized layer
  // therefore sits alone, unsplit.
  PlanBucket cur;
  bool open = false;
  uint64_t flat = 0;
  for (size_t i = 0; i < n_layers; ++i) {
    const uint64_t bytes = layer_numel[i] * (bpp ? bpp[i] : 4u);
    if (open && cur.bytes + bytes > cap_bytes) {
      plan.buckets.push_back(cur);
      cur = PlanBucket{};
      open = false;
    }
    if (!open) {
      cur.first_layer = i;
      cur.begin = flat;
      open = true;
    }
    cur.numel += layer_numel[i];
    cur.bytes += bytes;
    cur.n_layers += 1;
    flat += layer_numel[i];
  }
  plan.buckets.push_back(cur);
  plan.total = flat;

  // Device coordinates: the flat layout, or with every bucket starting on a
  // kSendAlign-element boundary (padded), so a bucket's own 16-byte-aligned
  // buffer (a DDP GradBucket) can stand for its slice of the arena.
  plan.padded = pad;
  uint64_t dev = 0;
  for (auto& b : plan.buckets) {
    b.dbegin = dev;
    dev += b.numel;
    if (pad) dev = (dev + kSendAlign - 1) / kSendAlign * kSendAlign;
  }
  plan.dtotal = plan.buckets.back().dbegin + plan.buckets.back().numel;

  std::vector<uint64_t> sizes;
  for (const auto& b : plan.buckets) sizes.push_back(b.numel);
  plan.twice_median = median_twice(sizes);

  // shard_plan runs only when K > 1 in train() (trainer.cpp:269-271).
  plan.sharded = shard < 0 ? interval > 1 : shard != 0;
  for (size_t b = 0; b < plan.buckets.size(); ++b) {
    const auto& bk = plan.buckets[b];
    uint64_t parts = 1;
    if (plan.sharded) {
      const uint64_t ratio = (2 * bk.numel) / plan.twice_median;  // model.hpp:56
      if (ratio >= 2) parts = std::min<uint64_t>(ratio, interval);  // model.cpp:103-104
    }
    const uint64_t base = bk.numel / parts, extra = bk.numel % parts;
    uint64_t off = 0;
    for (uint64_t p = 0; p < parts; ++p) {
      const uint64_t size = base + (p < extra ? 1 : 0);  // first numel%parts get +1
      plan.tensors.push_back(PlanTensor{b, bk.begin + off, bk.begin + off + size, bk.dbegin + off,
                                        bk.dbegin + off + size});
      off += size;
    }
  }

  // Per-phase send layout.  Selection depends only on (step mod K, K,
  // count), so K phase tables describe every step (compress.cpp:18-24).
  plan.phases.resize(interval);
  for (uint32_t p = 0; p < interval; ++p) {
    Phase& ph = plan.phases[p];
    ph.keep = select(p, interval, plan.tensors.size(), rule);
    ph.per_bucket.assign(plan.buckets.size(), BucketSel{});
    uint64_t cursor = 0;
    for (size_t t = 0; t < plan.tensors.size(); ++t) {
      if (!ph.keep[t]) continue;
      const PlanTensor& ts = plan.tensors[t];  // runs live in device coordinates
      if (!ph.runs.empty() && ph.runs.back().end == ts.dbegin && t > 0 && ph.keep[t - 1]) {
        ph.runs.back().end = ts.dend;  // extend the run: contiguous in the arena and in send
      } else {
        const uint64_t dst = cursor + ((ts.dbegin + kSendAlign - cursor % kSendAlign) % kSendAlign);
        ph.runs.push_back(Run{ts.dbegin, ts.dend, dst});
      }
      cursor = ph.runs.back().dst + (ph.runs.back().end - ph.runs.back().begin);
      ph.payload_elems += ts.end - ts.begin;
      BucketSel& bs = ph.per_bucket[ts.bucket];
      const uint64_t off = ph.runs.back().dst + (ts.dbegin - ph.runs.back().begin);
      if (bs.sel_end == bs.sel_begin) {
        bs.sel_begin = ts.dbegin;
        bs.sel_end = ts.dend;
        bs.send_offset = off;
      } else {
        // Shards of one bucket are <= K consecutive indices, so at most one
        // is selected per phase; a second one would break the per-bucket
        // single-range invariant the overlapped schedule relies on.
        throw covap::Error("internal: two selected shards in one bucket");
      }
    }
    ph.send_elems = cursor;
    plan.max_send = std::max(plan.max_send, cursor);
  }
  return plan;
}

}  // namespace covapb

namespace covapb {

// perf.cpp:63-103: the exact overlapped schedule over per-tensor times.
// Tensor i leaves the compute stream at the start of its block; its transfer
// starts when the channel is free and the tensor is available; a gap between
// transfers is a bubble; total = max(stream end, last transfer end).
Schedule overlap_schedule(double before_ms, const double* comp_ms, const double* compress_ms,
                          const double* comm_ms, const uint8_t* communicated, size_t n) {
  Schedule sc;
  double stream = before_ms;
  double channel = 0.0;
  bool channel_used = false;
  int64_t prev = -1;
  for (size_t i = 0; i < n; ++i) {
    const double available = stream;
    stream += comp_ms[i];
    if (compress_ms) stream += compress_ms[i];
    const bool sends = communicated == nullptr || communicated[i] != 0;
    if (!sends) continue;
    const double start = channel_used ? std::max(channel, available) : available;
    if (channel_used && start > channel) sc.bubbles.push_back({prev, start - channel});
    const double end = start + comm_ms[i];
    sc.comm_tensor.push_back(static_cast<int64_t>(i));
    sc.comm_start.push_back(start);
    sc.comm_end.push_back(end);
    channel = end;
    channel_used = true;
    prev = static_cast<int64_t>(i);
  }
  sc.stream_end = stream;
  sc.total = channel_used ? std::max(stream, channel) : stream;
  sc.unoverlapped = std::max(0.0, sc.total - sc.stream_end);
  return sc;
}

}  // namespace covapb
