// covap_capi.cpp — the C-ABI (include/covap_c.h): planner handles, device
// state, NCCL communicator and the per-step stream schedule.
//
// Reference map (paths under /root/reference/proj):
//   covap_plan_*          model.cpp:36-143, compress.cpp:13-28
//   covap_state_create    CompressorState::zeros, compress.cpp:37-42
//   covap_filter_pack     covap_compress, compress.cpp:50-85 (K1)
//   covap_unpack          covap_decompress + allreduce_mean's scale, compress.cpp:87-103,
//                         trainer.cpp:41-45 (K2)
//   covap_sync_step       the COVAP branch of train(), trainer.cpp:365-386
//   covap_allreduce       allreduce_mean's sum, trainer.cpp:41-43 (C1, NCCL)
//   covap_ccr / covap_choose_interval / covap_profile_ccr   perf.cpp:40-53, sim.cpp:164-216
#include "covap_c.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "covap/errors.hpp"
#include "covap_internal.h"
#include "covap_plan.hpp"
#include "covap_capi_common.hpp"

struct covap_plan {
  covapb::Plan p;
};


struct covap_state {
  covapb::Plan plan;
  int dtype = COVAP_F32;
  size_t esize = 4;
  int device = 0;
  covap_ef ef{1, 0.3, 100, 0.1};
  uint64_t num_steps = 0;
  void* residual = nullptr;
  void* send = nullptr;
  uint64_t send_cap = 0;
  covapb::Run* d_runs = nullptr;  // all phases back to back, then one full run
  std::vector<uint64_t> phase_off;
  covapb::Run* d_full = nullptr;  // {[0, N), dst 0}: the dense (uncompressed) mean
  cudaStream_t comm_stream = nullptr;
  int free_sms = 0;  // SMs K1 / K2 leave to the collective in the overlapped schedules
  cudaStream_t h2d_stream = nullptr;  // host-buffer pipeline (covap_sync_step_host)
  cudaStream_t d2h_stream = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_k, ev_out;  // per-chunk event pools (reused cyclically)
  // The previous covap_sync_step_host call's chunking, stream and device
  // buffers: a call with the same ones chains onto it chunk by chunk.
  std::vector<uint64_t> host_cuts;
  cudaStream_t host_stream = nullptr;
  const void* host_dev_grad = nullptr;
  const void* host_dev_out = nullptr;
  cudaEvent_t done = nullptr;
  std::vector<cudaEvent_t> ready, arrive, end;  // per bucket
  std::vector<cudaEvent_t> k1s, k2e;            // timeline: K1 start, K2 end, per bucket
  bool timeline = false;                        // record k1s / k2e in the overlapped schedule
  std::vector<uint8_t> tl_mode;                 // per bucket: 0 fused, 1 covap, 2 dense
  std::vector<uint8_t> timed;                   // bucket had a collective in the last step
  bool fuse_single_rank = true;                 // P = 1: run K1F instead of K1 -> C1 -> K2
  uint64_t ramp_min = 1u << 20;                 // host pipeline: smallest ramp chunk (elements)
  int pipeline = 1;                             // P > 1 sync step: bucket groups (1 = serial)
  // send buffer from ncclMemAlloc, registered as a symmetric NCCL window on
  // win_comm (covap_state_use_symmetric); NULL: plain cudaMalloc
  ncclWindow_t win = nullptr;
  covap_comm* win_comm = nullptr;
  bool send_nccl_mem = false;
};

namespace covapb {
thread_local std::string g_last_error;
}  // namespace covapb

namespace {
// Communicators alive right now: a state holding a window on a communicator
// that is already gone must not deregister it (the communicator did).
std::mutex g_comms_mu;
std::set<covap_comm*> g_live_comms;

void drop_window(covap_state* s) {
  if (!s->win) return;
  std::lock_guard<std::mutex> lock(g_comms_mu);
  if (s->win_comm && g_live_comms.count(s->win_comm)) {
    auto& w = s->win_comm->windows;
    const auto it = std::find(w.begin(), w.end(), s->win);
    if (it != w.end()) {
      ncclCommWindowDeregister(s->win_comm->nccl, s->win);
      w.erase(it);
    }
  }
  s->win = nullptr;
  s->win_comm = nullptr;
}
}  // namespace

namespace {

constexpr int kChunkEvents = 64;


const covapb::Phase& phase_of(const covapb::Plan& p, uint64_t step) {
  return p.phases[step % p.interval];
}

double coeff_of(const covap_state* s) {
  return s->ef.enabled ? covapb::ef_coefficient(s->num_steps, 1, s->ef.init_value,
                                                s->ef.ascend_steps, s->ef.ascend_range)
                       : 0.0;
}


// K1 over [a, b).  out != NULL: K1 also writes the zero fill of the
// unselected slots (compress.cpp:91) so that the unpack after the allreduce
// (k2sel_range) touches only the selected ones.
void k1_range(covap_state* s, const void* grad, void* send, uint64_t a, uint64_t b,
              cudaStream_t st, void* out = nullptr) {
  const size_t ph = s->num_steps % s->plan.interval;
  const int nr = static_cast<int>(s->plan.phases[ph].runs.size());
  CK(covapb::launch_filter_pack(s->dtype, grad, s->residual, send ? send : s->send,
                                s->d_runs + s->phase_off[ph], nr, a, b, coeff_of(s),
                                s->ef.enabled, st, out));
}

// K2 over the selected slots of [a, b) only (after k1_range with out): no
// launch at all when nothing in [a, b) is selected.
void k2sel_range(covap_state* s, const void* recv, void* out, double inv, uint64_t a, uint64_t b,
                 cudaStream_t st) {
  const size_t ph = s->num_steps % s->plan.interval;
  const auto& runs = s->plan.phases[ph].runs;
  CK(covapb::launch_unpack(s->dtype, recv ? recv : s->send, out, s->d_runs + s->phase_off[ph],
                           static_cast<int>(runs.size()), a, b, inv, 1, st, 0, runs.data()));
}

void k1f_range(covap_state* s, const void* grad, void* out, double inv, uint64_t a, uint64_t b,
               cudaStream_t st) {
  const size_t ph = s->num_steps % s->plan.interval;
  const int nr = static_cast<int>(s->plan.phases[ph].runs.size());
  CK(covapb::launch_filter_unpack(s->dtype, grad, s->residual, out, s->d_runs + s->phase_off[ph],
                                  nr, a, b, coeff_of(s), s->ef.enabled, inv, st));
}

void k2_range(covap_state* s, const void* recv, void* out, double inv, int mean, uint64_t a,
              uint64_t b, cudaStream_t st) {
  const size_t ph = s->num_steps % s->plan.interval;
  const int nr = static_cast<int>(s->plan.phases[ph].runs.size());
  CK(covapb::launch_unpack(s->dtype, recv ? recv : s->send, out, s->d_runs + s->phase_off[ph], nr,
                           a, b, inv, mean, st));
}

}  // namespace

extern "C" {

const char* covap_last_error(void) { return g_last_error.c_str(); }

int covap_version(void) { return 10000; }

covap_status covap_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n == 0) throw CudaError{cudaErrorNoDevice, "cudaGetDeviceCount"};
    *count = n;
  });
}

// ---------------------------------------------------------------- planner

covap_status covap_plan_create(const uint64_t* layer_numel, const uint32_t* bytes_per_param,
                               size_t n_layers, uint64_t cap_bytes, uint32_t interval, int rule,
                               int shard, covap_plan** out) {
  return covap_plan_create_ex(layer_numel, bytes_per_param, n_layers, cap_bytes, interval, rule,
                              shard, 0, out);
}

covap_status covap_plan_create_ex(const uint64_t* layer_numel, const uint32_t* bytes_per_param,
                                  size_t n_layers, uint64_t cap_bytes, uint32_t interval,
                                  int rule, int shard, int flags, covap_plan** out) {
  return guarded([&] {
    need(out != nullptr, "out must not be NULL");
    need(n_layers == 0 || layer_numel != nullptr, "layer_numel must not be NULL");
    need((flags & ~COVAP_PLAN_PAD_BUCKETS) == 0, "unknown plan flag");
    auto* p = new covap_plan;
    try {
      p->p = covapb::build_plan(layer_numel, bytes_per_param, n_layers, cap_bytes, interval, rule,
                                shard, (flags & COVAP_PLAN_PAD_BUCKETS) != 0);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

void covap_plan_destroy(covap_plan* plan) { delete plan; }

covap_status covap_plan_get_info(const covap_plan* plan, covap_plan_info* info) {
  return guarded([&] {
    need(plan && info, "NULL argument");
    const auto& p = plan->p;
    info->n_layers = p.n_layers;
    info->n_buckets = p.buckets.size();
    info->n_tensors = p.tensors.size();
    info->total_numel = p.total;
    info->twice_median = p.twice_median;
    info->interval = p.interval;
    info->rule = p.rule;
    info->sharded = p.sharded ? 1 : 0;
    info->align = static_cast<int32_t>(covapb::kSendAlign);
    info->max_send_elems = p.max_send;
    info->device_numel = p.dtotal;
    info->padded = p.padded ? 1 : 0;
  });
}

covap_status covap_plan_buckets(const covap_plan* plan, uint64_t* numel, uint64_t* begin,
                                uint64_t* first_layer, uint64_t* n_layers) {
  return guarded([&] {
    need(plan != nullptr, "NULL plan");
    const auto& bs = plan->p.buckets;
    for (size_t b = 0; b < bs.size(); ++b) {
      if (numel) numel[b] = bs[b].numel;
      if (begin) begin[b] = bs[b].begin;
      if (first_layer) first_layer[b] = bs[b].first_layer;
      if (n_layers) n_layers[b] = bs[b].n_layers;
    }
  });
}

covap_status covap_plan_tensors(const covap_plan* plan, uint64_t* bucket, uint64_t* begin,
                                uint64_t* end) {
  return guarded([&] {
    need(plan != nullptr, "NULL plan");
    const auto& ts = plan->p.tensors;
    for (size_t t = 0; t < ts.size(); ++t) {
      if (bucket) bucket[t] = ts[t].bucket;
      if (begin) begin[t] = ts[t].begin;
      if (end) end[t] = ts[t].end;
    }
  });
}

covap_status covap_plan_selection(const covap_plan* plan, uint64_t num_steps, uint8_t* keep) {
  return guarded([&] {
    need(plan && keep, "NULL argument");
    const auto& k = phase_of(plan->p, num_steps).keep;
    std::memcpy(keep, k.data(), k.size());
  });
}

covap_status covap_plan_bucket_range(const covap_plan* plan, uint64_t num_steps, size_t bucket,
                                     covap_bucket_range* out) {
  return guarded([&] {
    need(plan && out, "NULL argument");
    need(bucket < plan->p.buckets.size(), "bucket index out of range");
    const auto& bk = plan->p.buckets[bucket];
    const auto& sel = phase_of(plan->p, num_steps).per_bucket[bucket];
    out->bucket_begin = bk.begin;
    out->bucket_end = bk.begin + bk.numel;
    // the selected range in flat coordinates (the planner keeps device ones)
    out->sel_begin = sel.sel_end > sel.sel_begin ? sel.sel_begin - bk.dbegin + bk.begin : bk.begin;
    out->sel_end = sel.sel_end > sel.sel_begin ? sel.sel_end - bk.dbegin + bk.begin : bk.begin;
    out->send_offset = sel.send_offset;
    out->device_begin = bk.dbegin;
  });
}

covap_status covap_plan_send_elems(const covap_plan* plan, uint64_t num_steps,
                                   uint64_t* send_elems, uint64_t* payload_elems) {
  return guarded([&] {
    need(plan != nullptr, "NULL plan");
    const auto& ph = phase_of(plan->p, num_steps);
    if (send_elems) *send_elems = ph.send_elems;
    if (payload_elems) *payload_elems = ph.payload_elems;
  });
}

covap_status covap_median_twice(const uint64_t* bucket_numel, size_t n, uint64_t* twice) {
  return guarded([&] {
    need(twice != nullptr, "NULL argument");
    *twice = covapb::median_twice(std::vector<uint64_t>(bucket_numel, bucket_numel + n));
  });
}

covap_status covap_select_tensors(uint64_t num_steps, uint32_t interval, size_t count, int rule,
                                  uint8_t* keep) {
  return guarded([&] {
    const auto k = covapb::select(num_steps, interval, count, rule);
    std::memcpy(keep, k.data(), k.size());
  });
}

covap_status covap_ef_coefficient(uint64_t num_steps, const covap_ef* ef, double* coeff) {
  return guarded([&] {
    need(ef && coeff, "NULL argument");
    *coeff = covapb::ef_coefficient(num_steps, ef->enabled, ef->init_value, ef->ascend_steps,
                                    ef->ascend_range);
  });
}

covap_status covap_ccr(double comm_ms, double comp_ms, double* out) {
  return guarded([&] { *out = covapb::ccr(comm_ms, comp_ms); });
}

covap_status covap_choose_interval(double ccr_value, uint32_t* out) {
  return guarded([&] { *out = covapb::choose_interval(ccr_value); });
}

covap_status covap_profile_ccr(const double* comm_start, const double* comm_end, size_t workers,
                               size_t expected, size_t n_coll, double comp_ms,
                               double* aligned_ms, double* naive_ms, double* ccr_out,
                               uint32_t* interval_out) {
  return guarded([&] {
    // sim.cpp:166-201: every expected worker must be present.
    if (workers != expected || expected == 0)
      throw covap::IncompleteProfile("expected " + std::to_string(expected) +
                                     " worker traces, got " + std::to_string(workers));
    double aligned = 0.0;
    for (size_t w = 0; w < workers; ++w) naive_ms[w] = 0.0;
    for (size_t c = 0; c < n_coll; ++c) {
      double last = comm_start[c];
      for (size_t w = 1; w < workers; ++w) last = std::max(last, comm_start[w * n_coll + c]);
      aligned += comm_end[c] - last;  // sim.cpp:202-203
      for (size_t w = 0; w < workers; ++w) naive_ms[w] += comm_end[c] - comm_start[w * n_coll + c];
    }
    *aligned_ms = aligned;
    *ccr_out = covapb::ccr(aligned, comp_ms);
    *interval_out = covapb::choose_interval(*ccr_out);
  });
}

covap_status covap_overlap_schedule(double before_ms, const double* comp_ms,
                                    const double* compress_ms, const double* comm_ms,
                                    const uint8_t* communicated, size_t n, double* total_ms,
                                    double* stream_end_ms, double* unoverlapped_ms,
                                    double* comm_start_ms, double* comm_end_ms,
                                    int64_t* comm_tensor, size_t* n_comm, int64_t* bubble_after,
                                    double* bubble_ms, size_t* n_bubbles) {
  return guarded([&] {
    need(n == 0 || (comp_ms && comm_ms), "NULL per-tensor list");
    const covapb::Schedule sc =
        covapb::overlap_schedule(before_ms, comp_ms, compress_ms, comm_ms, communicated, n);
    if (total_ms) *total_ms = sc.total;
    if (stream_end_ms) *stream_end_ms = sc.stream_end;
    if (unoverlapped_ms) *unoverlapped_ms = sc.unoverlapped;
    if (n_comm) *n_comm = sc.comm_tensor.size();
    for (size_t i = 0; i < sc.comm_tensor.size(); ++i) {
      if (comm_start_ms) comm_start_ms[i] = sc.comm_start[i];
      if (comm_end_ms) comm_end_ms[i] = sc.comm_end[i];
      if (comm_tensor) comm_tensor[i] = sc.comm_tensor[i];
    }
    if (n_bubbles) *n_bubbles = sc.bubbles.size();
    for (size_t i = 0; i < sc.bubbles.size(); ++i) {
      if (bubble_after) bubble_after[i] = sc.bubbles[i].first;
      if (bubble_ms) bubble_ms[i] = sc.bubbles[i].second;
    }
  });
}

// ---------------------------------------------------------------- state

void covap_state_destroy(covap_state* s) {
  if (!s) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(s->device);
  if (s->comm_stream) cudaStreamSynchronize(s->comm_stream);
  cudaDeviceSynchronize();
  drop_window(s);
  cudaFree(s->residual);
  if (s->send_nccl_mem)
    ncclMemFree(s->send);
  else
    cudaFree(s->send);
  cudaFree(s->d_runs);
  for (auto e : s->ready) cudaEventDestroy(e);
  for (auto e : s->k1s) cudaEventDestroy(e);
  for (auto e : s->k2e) cudaEventDestroy(e);
  for (auto e : s->arrive) cudaEventDestroy(e);
  for (auto e : s->end) cudaEventDestroy(e);
  if (s->done) cudaEventDestroy(s->done);
  for (auto e : s->ev_in) cudaEventDestroy(e);
  for (auto e : s->ev_k) cudaEventDestroy(e);
  for (auto e : s->ev_out) cudaEventDestroy(e);
  if (s->h2d_stream) cudaStreamDestroy(s->h2d_stream);
  if (s->d2h_stream) cudaStreamDestroy(s->d2h_stream);
  if (s->comm_stream) cudaStreamDestroy(s->comm_stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete s;
}

covap_status covap_state_create(const covap_plan* plan, int dtype, int device,
                                const covap_ef* ef, covap_state** out) {
  covap_state* s = nullptr;
  const covap_status st = guarded([&] {
    need(plan && out, "NULL argument");
    need(dtype == COVAP_F32 || dtype == COVAP_F64, "dtype must be COVAP_F32 or COVAP_F64");
    if (ef && ef->enabled && ef->ascend_steps < 1)
      throw covap::InvalidInput("ascend_steps must be >= 1");
    DeviceGuard dg(device);
    s = new covap_state;
    s->plan = plan->p;
    s->dtype = dtype;
    s->esize = dtype == COVAP_F64 ? 8 : 4;
    s->device = device;
    if (ef) s->ef = *ef;
    const uint64_t n = s->plan.dtotal;
    CK(cudaMalloc(&s->residual, std::max<uint64_t>(n, 1) * s->esize));
    CK(cudaMemset(s->residual, 0, std::max<uint64_t>(n, 1) * s->esize));
    s->send_cap = std::max<uint64_t>(s->plan.max_send, 1);
    CK(cudaMalloc(&s->send, s->send_cap * s->esize));
    CK(cudaMemset(s->send, 0, s->send_cap * s->esize));  // alignment gaps stay zero forever
    std::vector<covapb::Run> all;
    for (const auto& ph : s->plan.phases) {
      s->phase_off.push_back(all.size());
      all.insert(all.end(), ph.runs.begin(), ph.runs.end());
    }
    const size_t full_off = all.size();
    all.push_back(covapb::Run{0, n, 0});
    CK(cudaMalloc(&s->d_runs, all.size() * sizeof(covapb::Run)));
    CK(cudaMemcpy(s->d_runs, all.data(), all.size() * sizeof(covapb::Run),
                  cudaMemcpyHostToDevice));
    s->d_full = s->d_runs + full_off;
    CK(cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->h2d_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->d2h_stream, cudaStreamNonBlocking));
    s->ev_in.resize(kChunkEvents);
    s->ev_k.resize(kChunkEvents);
    s->ev_out.resize(kChunkEvents);
    for (int i = 0; i < kChunkEvents; ++i) {
      CK(cudaEventCreateWithFlags(&s->ev_in[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_k[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_out[i], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming));
    const size_t nb = s->plan.buckets.size();
    s->ready.resize(nb);
    s->arrive.resize(nb);
    s->end.resize(nb);
    s->timed.assign(nb, 0);
    s->k1s.resize(nb);
    s->k2e.resize(nb);
    s->tl_mode.assign(nb, 0);
    for (size_t b = 0; b < nb; ++b) {
      CK(cudaEventCreate(&s->k1s[b]));
      CK(cudaEventCreate(&s->k2e[b]));
    }
    for (size_t b = 0; b < nb; ++b) {
      CK(cudaEventCreate(&s->ready[b]));  // timed: the K1-end mark of the timeline
      CK(cudaEventCreate(&s->arrive[b]));
      CK(cudaEventCreate(&s->end[b]));
    }
    *out = s;
  });
  if (st != COVAP_OK && s) {
    covap_state_destroy(s);
  }
  return st;
}

covap_status covap_state_residual(covap_state* s, void** dev_ptr, uint64_t* n) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    if (dev_ptr) *dev_ptr = s->residual;
    if (n) *n = s->plan.dtotal;
  });
}

covap_status covap_state_send(covap_state* s, void** dev_ptr, uint64_t* capacity) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    if (dev_ptr) *dev_ptr = s->send;
    if (capacity) *capacity = s->send_cap;
  });
}

covap_status covap_state_get_step(const covap_state* s, uint64_t* num_steps) {
  return guarded([&] {
    need(s && num_steps, "NULL argument");
    *num_steps = s->num_steps;
  });
}

covap_status covap_state_set_step(covap_state* s, uint64_t num_steps) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    s->num_steps = num_steps;
  });
}

covap_status covap_state_set_fused(covap_state* s, int fuse_single_rank) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    s->fuse_single_rank = fuse_single_rank != 0;
  });
}

covap_status covap_state_set_free_sms(covap_state* s, int n) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    need(n >= 0, "free SMs must be >= 0");
    s->free_sms = n;
  });
}

covap_status covap_state_set_pipeline(covap_state* s, int groups) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    need(groups >= 1, "groups must be >= 1");
    s->pipeline = groups;
  });
}

covap_status covap_state_use_symmetric(covap_state* s, covap_comm* c) {
  return guarded([&] {
    need(s && c, "NULL argument");
    need(c->device == s->device, "communicator and state are on different devices");
    need(!s->win, "the send buffer is already a symmetric window");
    DeviceGuard dg(s->device);
    CK(cudaDeviceSynchronize());  // nothing may still use the old buffer
    const size_t bytes = (s->send_cap * s->esize + NCCL_WIN_REQUIRED_ALIGNMENT - 1) /
                         NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    void* buf = nullptr;
    NK(ncclMemAlloc(&buf, bytes));
    const cudaError_t me = cudaMemset(buf, 0, bytes);  // alignment gaps stay zero forever
    if (me != cudaSuccess) {
      ncclMemFree(buf);
      throw CudaError{me, "cudaMemset(symmetric send buffer)"};
    }
    ncclWindow_t win = nullptr;
    const ncclResult_t r = ncclCommWindowRegister(c->nccl, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
      ncclMemFree(buf);
      throw NcclError{r, "ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)"};
    }
    if (s->send_nccl_mem)
      ncclMemFree(s->send);
    else
      cudaFree(s->send);
    s->send = buf;
    s->send_nccl_mem = true;
    s->win = win;
    s->win_comm = c;
    std::lock_guard<std::mutex> lock(g_comms_mu);
    c->windows.push_back(win);
  });
}

covap_status covap_state_set_host_ramp(covap_state* s, uint64_t ramp_min_elems) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    s->ramp_min = std::max<uint64_t>(ramp_min_elems, 8192);
  });
}

covap_status covap_state_reset(covap_state* s, void* stream) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    DeviceGuard dg(s->device);
    CK(cudaMemsetAsync(s->residual, 0, std::max<uint64_t>(s->plan.dtotal, 1) * s->esize,
                       as_stream(stream)));
  });
}

// ---------------------------------------------------------------- K1 / K2

covap_status covap_filter_pack(covap_state* s, const void* grad, void* send, size_t b0, size_t b1,
                               void* stream) {
  return guarded([&] {
    need(s != nullptr && grad != nullptr, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(grad, "grad");
    if (send) need_aligned(send, "send");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    k1_range(s, grad, send, a, b, as_stream(stream));
  });
}

covap_status covap_unpack(covap_state* s, const void* recv, void* out, double scale, int mean,
                          size_t b0, size_t b1, void* stream) {
  return guarded([&] {
    need(s != nullptr && out != nullptr, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(out, "out");
    if (recv) need_aligned(recv, "recv");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    k2_range(s, recv, out, scale, mean, a, b, as_stream(stream));
  });
}

covap_status covap_filter_pack_zero(covap_state* s, const void* grad, void* send, void* out,
                                    size_t b0, size_t b1, void* stream) {
  return guarded([&] {
    need(s && grad && out, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    if (send) need_aligned(send, "send");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    k1_range(s, grad, send, a, b, as_stream(stream), out);
  });
}

covap_status covap_unpack_selected(covap_state* s, const void* recv, void* out, double scale,
                                   size_t b0, size_t b1, void* stream) {
  return guarded([&] {
    need(s != nullptr && out != nullptr, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(out, "out");
    if (recv) need_aligned(recv, "recv");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    k2sel_range(s, recv, out, scale, a, b, as_stream(stream));
  });
}

covap_status covap_filter_unpack(covap_state* s, const void* grad, void* out, double scale,
                                 size_t b0, size_t b1, void* stream) {
  return guarded([&] {
    need(s && grad && out, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    k1f_range(s, grad, out, scale, a, b, as_stream(stream));
  });
}

covap_status covap_filter_sgd(covap_state* s, const void* grad, void* params, double lr,
                              double scale, size_t b0, size_t b1, void* stream) {
  return guarded([&] {
    need(s && grad && params, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(grad, "grad");
    need_aligned(params, "params");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    const size_t ph = s->num_steps % s->plan.interval;
    CK(covapb::launch_filter_sgd(s->dtype, grad, s->residual, params, s->d_runs + s->phase_off[ph],
                                 static_cast<int>(s->plan.phases[ph].runs.size()), a, b,
                                 coeff_of(s), s->ef.enabled, scale, lr, as_stream(stream)));
  });
}

covap_status covap_unpack_sgd(covap_state* s, const void* recv, void* params, double lr,
                              double scale, int mean, size_t b0, size_t b1, void* stream) {
  return guarded([&] {
    need(s && params, "NULL argument");
    need(b0 <= b1 && b1 <= s->plan.buckets.size(), "bucket range out of bounds");
    need_aligned(params, "params");
    if (recv) need_aligned(recv, "recv");
    if (b0 == b1) return;
    DeviceGuard dg(s->device);
    const uint64_t a = s->plan.buckets[b0].dbegin;
    const uint64_t b = s->plan.buckets[b1 - 1].dbegin + s->plan.buckets[b1 - 1].numel;
    const size_t ph = s->num_steps % s->plan.interval;
    CK(covapb::launch_unpack_sgd(s->dtype, recv ? recv : s->send, params,
                                 s->d_runs + s->phase_off[ph],
                                 static_cast<int>(s->plan.phases[ph].runs.size()), a, b, scale,
                                 mean, lr, as_stream(stream)));
  });
}

covap_status covap_sync_step_sgd(covap_state* s, covap_comm* comm, const void* grad,
                                 void* params, double lr, void* stream) {
  return guarded([&] {
    need(s && grad && params, "NULL argument");
    need_aligned(grad, "grad");
    need_aligned(params, "params");
    if (comm) need(comm->device == s->device, "communicator and state are on different devices");
    DeviceGuard dg(s->device);
    cudaStream_t st = as_stream(stream);
    const uint64_t n = s->plan.dtotal;
    const auto& ph = phase_of(s->plan, s->num_steps);
    const int P = world(comm);
    const int nr = static_cast<int>(ph.runs.size());
    const covapb::Run* runs = s->d_runs + s->phase_off[s->num_steps % s->plan.interval];
    if (P == 1 && s->fuse_single_rank) {
      CK(covapb::launch_filter_sgd(s->dtype, grad, s->residual, params, runs, nr, 0, n, coeff_of(s),
                                   s->ef.enabled, 1.0, lr, st));
    } else {
      k1_range(s, grad, nullptr, 0, n, st);
      if (comm && ph.send_elems > 0)
        NK(ncclAllReduce(s->send, s->send, ph.send_elems, nccl_type(s->dtype), ncclSum,
                         comm->nccl, st));
      CK(covapb::launch_unpack_sgd(s->dtype, s->send, params, runs, nr, 0, n,
                                   1.0 / static_cast<double>(P), 1, lr, st));
    }
    ++s->num_steps;
  });
}

covap_status covap_step_end(covap_state* s) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    ++s->num_steps;
  });
}

covap_status covap_sync_step(covap_state* s, covap_comm* comm, const void* grad, void* out,
                             void* stream) {
  return guarded([&] {
    need(s && grad && out, "NULL argument");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    if (comm) need(comm->device == s->device, "communicator and state are on different devices");
    DeviceGuard dg(s->device);
    cudaStream_t st = as_stream(stream);
    const uint64_t n = s->plan.dtotal;
    const auto& ph = phase_of(s->plan, s->num_steps);
    const int P = world(comm);
    if (P == 1 && s->fuse_single_rank) {
      // One rank: the allreduce is the identity, so K1 and K2 fuse into one
      // pass (K1F) that writes (0 + c) * 1 straight to the selected slots.
      k1f_range(s, grad, out, 1.0, 0, n, st);
    } else if (s->pipeline > 1 && s->plan.buckets.size() > 1) {
      const covapb::ScopedFreeSms reserve(s->free_sms);  // SMs for the overlapped allreduces
      // Pipelined: consecutive bucket groups of about n / G elements; group
      // g's allreduce (comm stream) overlaps K1 of groups > g (compute
      // stream), and its K2 follows as soon as its allreduce is done.  Every
      // rank derives the same groups and envelopes from the plan.
      const auto& bs = s->plan.buckets;
      const size_t G = std::min<size_t>(static_cast<size_t>(s->pipeline), bs.size());
      std::vector<size_t> first{0};
      for (size_t b = 1; b < bs.size() && first.size() < G; ++b)
        if (bs[b].dbegin >= n * first.size() / G) first.push_back(b);
      const size_t ng = first.size();
      auto lo_of = [&](size_t g) { return g == 0 ? uint64_t(0) : bs[first[g]].dbegin; };
      auto hi_of = [&](size_t g) { return g + 1 < ng ? bs[first[g + 1]].dbegin : n; };
      CK(cudaEventRecord(s->done, st));
      CK(cudaStreamWaitEvent(s->comm_stream, s->done, 0));
      for (size_t g = 0; g < ng; ++g) {
        k1_range(s, grad, nullptr, lo_of(g), hi_of(g), st, out);
        uint64_t lo = UINT64_MAX, hi = 0;
        const size_t b1 = g + 1 < ng ? first[g + 1] : bs.size();
        for (size_t b = first[g]; b < b1; ++b) {
          const auto& sel = ph.per_bucket[b];
          if (sel.sel_end <= sel.sel_begin) continue;
          lo = std::min(lo, sel.send_offset);
          hi = std::max(hi, sel.send_offset + (sel.sel_end - sel.sel_begin));
        }
        CK(cudaEventRecord(s->ready[g], st));
        CK(cudaStreamWaitEvent(s->comm_stream, s->ready[g], 0));
        if (comm && hi > lo)
          NK(ncclAllReduce(static_cast<char*>(s->send) + lo * s->esize,
                           static_cast<char*>(s->send) + lo * s->esize, hi - lo,
                           nccl_type(s->dtype), ncclSum, comm->nccl, s->comm_stream));
        CK(cudaEventRecord(s->end[g], s->comm_stream));
      }
      for (size_t g = 0; g < ng; ++g) {
        CK(cudaStreamWaitEvent(st, s->end[g], 0));
        k2sel_range(s, nullptr, out, 1.0 / static_cast<double>(P), lo_of(g), hi_of(g), st);
      }
    } else {
      k1_range(s, grad, nullptr, 0, n, st, out);
      if (comm && ph.send_elems > 0)
        NK(ncclAllReduce(s->send, s->send, ph.send_elems, nccl_type(s->dtype), ncclSum,
                         comm->nccl, st));
      k2sel_range(s, nullptr, out, 1.0 / static_cast<double>(P), 0, n, st);
    }
    ++s->num_steps;
  });
}

covap_status covap_sync_step_host(covap_state* s, covap_comm* comm, const void* host_grad,
                                  void* host_out, void* dev_grad, void* dev_out,
                                  uint64_t chunk_elems, void* stream) {
  return guarded([&] {
    need(s && host_grad && host_out && dev_grad && dev_out, "NULL argument");
    need_aligned(dev_grad, "dev_grad");
    need_aligned(dev_out, "dev_out");
    if (comm) need(comm->device == s->device, "communicator and state are on different devices");
    DeviceGuard dg(s->device);
    cudaStream_t st = as_stream(stream);
    const uint64_t n = s->plan.dtotal;
    const size_t es = s->esize;
    // Chunk boundaries (multiples of 8192 elements): C-sized chunks in the
    // middle, ramping geometrically (C/2^k, ..., C/4, C/2, from ramp_min
    // elements) at both ends so the first H2D and the last D2H — the parts
    // no other copy overlaps — are short.
    // Default C = max(4 Mi, N / 32): measured best for ResNet-50 (4 Mi) and
    // BERT-large (~10 Mi) on B200 PCIe (profiles/r1_design_study.md).
    uint64_t chunk = std::max<uint64_t>(
        chunk_elems ? chunk_elems : std::max<uint64_t>(4u << 20, n / 32), 1u << 20);
    chunk = (chunk + 8191) / 8192 * 8192;
    std::vector<uint64_t> cuts{0};
    if (n >= 3 * chunk) {
      std::vector<uint64_t> ramp;  // C/2, C/4, ... down to ramp_min
      for (uint64_t c = chunk / 2; c >= s->ramp_min && c >= 8192; c /= 2) ramp.push_back(c / 8192 * 8192);
      if (ramp.empty()) ramp.push_back(chunk / 2 / 8192 * 8192);
      uint64_t head = 0;
      for (size_t i = ramp.size(); i-- > 0;) {
        head += ramp[i];
        cuts.push_back(head);
      }
      const uint64_t mid_end = n - head;
      const uint64_t m = (mid_end - head + chunk - 1) / chunk;
      for (uint64_t i = 1; i < m; ++i) cuts.push_back(head + ((mid_end - head) * i / m) / 8192 * 8192);
      uint64_t tail = mid_end;
      for (size_t i = 0; i < ramp.size(); ++i) {
        cuts.push_back(tail);
        tail += ramp[i];
      }
    } else {
      for (uint64_t a = chunk; a < n; a += chunk) cuts.push_back(a);
    }
    cuts.push_back(n);
    const int P = world(comm);
    const auto& ph = phase_of(s->plan, s->num_steps);
    const double inv = 1.0 / static_cast<double>(P);
    // Step boundary.  A call that repeats the previous one's chunking,
    // stream and device buffers chains onto it chunk by chunk: chunk c's H2D
    // waits only until the previous step's kernels are done with chunk c of
    // dev_grad, so this step's uploads overlap the previous step's downloads
    // (the kernels still follow the previous step's last download, through
    // the wait on `stream` at its end).  Otherwise the copy streams start
    // after everything already on `stream`.
    const bool chained = s->host_cuts == cuts && s->host_stream == st &&
                         s->host_dev_grad == dev_grad && s->host_dev_out == dev_out;
    if (!chained) {
      CK(cudaEventRecord(s->done, st));
      CK(cudaStreamWaitEvent(s->h2d_stream, s->done, 0));
    }
    for (size_t c = 0; c + 1 < cuts.size(); ++c) {
      const uint64_t a = cuts[c], b = cuts[c + 1];
      if (b <= a) continue;
      cudaEvent_t ein = s->ev_in[c % kChunkEvents], ek = s->ev_k[c % kChunkEvents];
      cudaEvent_t eout = s->ev_out[c % kChunkEvents];
      // (a pool event reused by a later chunk was recorded later on the same
      // stream: waiting on it over-synchronises, never under-)
      if (chained) {
        CK(cudaStreamWaitEvent(s->h2d_stream, ek, 0));  // kernels done with dev_grad chunk c
        if (dev_grad == dev_out)  // and, aliased, the download of its outputs
          CK(cudaStreamWaitEvent(s->h2d_stream, eout, 0));
      }
      CK(cudaMemcpyAsync(static_cast<char*>(dev_grad) + a * es,
                         static_cast<const char*>(host_grad) + a * es, (b - a) * es,
                         cudaMemcpyHostToDevice, s->h2d_stream));
      CK(cudaEventRecord(ein, s->h2d_stream));
      CK(cudaStreamWaitEvent(st, ein, 0));
      if (P == 1 && s->fuse_single_rank) {
        k1f_range(s, dev_grad, dev_out, 1.0, a, b, st);
      } else {
        k1_range(s, dev_grad, nullptr, a, b, st, dev_out);
        // The chunk's selected elements occupy one contiguous envelope of the
        // send buffer (runs map monotonically); every rank derives the same
        // envelopes from the plan, so the collectives match.
        uint64_t lo = UINT64_MAX, hi = 0;
        for (const auto& r : ph.runs) {
          const uint64_t x0 = std::max(a, r.begin), x1 = std::min(b, r.end);
          if (x0 >= x1) continue;
          lo = std::min(lo, r.dst + (x0 - r.begin));
          hi = std::max(hi, r.dst + (x1 - r.begin));
        }
        if (comm && hi > lo)
          NK(ncclAllReduce(static_cast<char*>(s->send) + lo * es,
                           static_cast<char*>(s->send) + lo * es, hi - lo, nccl_type(s->dtype),
                           ncclSum, comm->nccl, st));
        k2sel_range(s, nullptr, dev_out, inv, a, b, st);
      }
      CK(cudaEventRecord(ek, st));
      CK(cudaStreamWaitEvent(s->d2h_stream, ek, 0));
      CK(cudaMemcpyAsync(static_cast<char*>(host_out) + a * es,
                         static_cast<const char*>(dev_out) + a * es, (b - a) * es,
                         cudaMemcpyDeviceToHost, s->d2h_stream));
      CK(cudaEventRecord(eout, s->d2h_stream));
    }
    CK(cudaEventRecord(s->done, s->d2h_stream));
    CK(cudaStreamWaitEvent(st, s->done, 0));
    s->host_cuts = cuts;
    s->host_stream = st;
    s->host_dev_grad = dev_grad;
    s->host_dev_out = dev_out;
    ++s->num_steps;
  });
}

covap_status covap_bucket_ready(covap_state* s, covap_comm* comm, size_t bucket, const void* grad,
                                void* out, void* stream) {
  return guarded([&] {
    need(s && grad && out, "NULL argument");
    need(bucket < s->plan.buckets.size(), "bucket index out of range");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    DeviceGuard dg(s->device);
    cudaStream_t st = as_stream(stream);
    const auto& bk = s->plan.buckets[bucket];
    const auto& sel = phase_of(s->plan, s->num_steps).per_bucket[bucket];
    const uint64_t a = bk.dbegin, b = bk.dbegin + bk.numel;
    const int P = world(comm);
    if (s->timeline) CK(cudaEventRecord(s->k1s[bucket], st));
    if (P == 1 && s->fuse_single_rank) {  // no exchange: the fused pass on the producing stream
      k1f_range(s, grad, out, 1.0, a, b, st);
      if (s->timeline) CK(cudaEventRecord(s->ready[bucket], st));
      s->timed[bucket] = 0;
      s->tl_mode[bucket] = 0;
      return;
    }
    // K1 also zero-fills the bucket's unselected output, so the side stream
    // only carries the allreduce of the selected range and its unpack — and
    // nothing at all for a bucket with no selected shard this step.
    const covapb::ScopedFreeSms reserve(s->free_sms);  // SMs for the side stream's allreduce
    k1_range(s, grad, nullptr, a, b, st, out);
    CK(cudaEventRecord(s->ready[bucket], st));
    CK(cudaStreamWaitEvent(s->comm_stream, s->ready[bucket], 0));
    const uint64_t len = sel.sel_end - sel.sel_begin;
    s->timed[bucket] = len > 0 ? 1 : 0;
    s->tl_mode[bucket] = 1;
    CK(cudaEventRecord(s->arrive[bucket], s->comm_stream));
    if (comm && len > 0)
      NK(ncclAllReduce(static_cast<char*>(s->send) + sel.send_offset * s->esize,
                       static_cast<char*>(s->send) + sel.send_offset * s->esize, len,
                       nccl_type(s->dtype), ncclSum, comm->nccl, s->comm_stream));
    CK(cudaEventRecord(s->end[bucket], s->comm_stream));
    k2sel_range(s, nullptr, out, 1.0 / static_cast<double>(P), a, b, s->comm_stream);
    if (s->timeline) CK(cudaEventRecord(s->k2e[bucket], s->comm_stream));
  });
}

covap_status covap_state_side_stream(covap_state* s, void** stream) {
  return guarded([&] {
    need(s && stream, "NULL argument");
    *stream = s->comm_stream;
  });
}

covap_status covap_state_set_timeline(covap_state* s, int on) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    s->timeline = on != 0;
  });
}

covap_status covap_state_timeline(covap_state* s, double* rows, size_t n) {
  return guarded([&] {
    need(s && rows, "NULL argument");
    need(s->timeline, "timeline recording is off (covap_state_set_timeline)");
    need(n <= s->plan.buckets.size(), "n exceeds bucket count");
    DeviceGuard dg(s->device);
    CK(cudaStreamSynchronize(s->comm_stream));
    CK(cudaDeviceSynchronize());
    auto ms = [&](cudaEvent_t e) {
      float v = 0.f;
      CK(cudaEventElapsedTime(&v, s->k1s[0], e));
      return static_cast<double>(v);
    };
    for (size_t b = 0; b < n; ++b) {
      double* r = rows + 5 * b;
      r[0] = ms(s->k1s[b]);
      r[1] = s->tl_mode[b] == 2 ? r[0] : ms(s->ready[b]);
      r[2] = s->tl_mode[b] == 0 ? -1.0 : ms(s->arrive[b]);
      r[3] = s->tl_mode[b] == 0 ? -1.0 : ms(s->end[b]);
      r[4] = s->tl_mode[b] == 0 ? r[1] : ms(s->k2e[b]);
    }
  });
}

covap_status covap_dense_bucket_ready(covap_state* s, covap_comm* comm, size_t bucket, void* grad,
                                      void* out, void* stream) {
  return guarded([&] {
    need(s && grad && out, "NULL argument");
    need(bucket < s->plan.buckets.size(), "bucket index out of range");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    DeviceGuard dg(s->device);
    cudaStream_t st = as_stream(stream);
    const auto& bk = s->plan.buckets[bucket];
    const uint64_t a = bk.dbegin, b = bk.dbegin + bk.numel;
    if (s->timeline) CK(cudaEventRecord(s->k1s[bucket], st));
    CK(cudaEventRecord(s->ready[bucket], st));
    CK(cudaStreamWaitEvent(s->comm_stream, s->ready[bucket], 0));
    const int P = world(comm);
    s->timed[bucket] = 1;
    s->tl_mode[bucket] = 2;
    CK(cudaEventRecord(s->arrive[bucket], s->comm_stream));
    if (comm)
      NK(ncclAllReduce(static_cast<char*>(grad) + a * s->esize,
                       static_cast<char*>(grad) + a * s->esize, bk.numel, nccl_type(s->dtype),
                       ncclSum, comm->nccl, s->comm_stream));
    CK(cudaEventRecord(s->end[bucket], s->comm_stream));
    // allreduce_mean's "0 + sum, then x 1/P" (trainer.cpp:41-45) in place.
    CK(covapb::launch_unpack(s->dtype, grad, out, s->d_full, 1, a, b,
                             1.0 / static_cast<double>(P), 1, s->comm_stream));
    if (s->timeline) CK(cudaEventRecord(s->k2e[bucket], s->comm_stream));
  });
}

namespace {
// A bucket's own buffer stands for its slice [dbegin, dbegin + numel) of the
// arena: the kernels only touch that slice, so the arena base is the buffer
// address minus dbegin elements.  Needs a 16-byte-aligned dbegin (padded plan).
covap_status local_bases(covap_state* s, size_t bucket, const void* g, const void* o,
                         const char** gb, char** ob) {
  return guarded([&] {
    need(s && g && o, "NULL argument");
    need(bucket < s->plan.buckets.size(), "bucket index out of range");
    need_aligned(g, "bucket grad");
    need_aligned(o, "bucket out");
    const uint64_t off = s->plan.buckets[bucket].dbegin * s->esize;
    if (off % 16 != 0)
      throw covap::InvalidInput("bucket-local calls need a padded plan (COVAP_PLAN_PAD_BUCKETS)");
    *gb = static_cast<const char*>(g) - off;
    *ob = static_cast<char*>(const_cast<void*>(o)) - off;
  });
}
}  // namespace

covap_status covap_bucket_ready_local(covap_state* s, covap_comm* comm, size_t bucket,
                                      const void* bucket_grad, void* bucket_out, void* stream) {
  const char* g = nullptr;
  char* o = nullptr;
  const covap_status st = local_bases(s, bucket, bucket_grad, bucket_out, &g, &o);
  if (st != COVAP_OK) return st;
  return covap_bucket_ready(s, comm, bucket, g, o, stream);
}

covap_status covap_dense_bucket_ready_local(covap_state* s, covap_comm* comm, size_t bucket,
                                            void* bucket_grad, void* bucket_out, void* stream) {
  const char* g = nullptr;
  char* o = nullptr;
  const covap_status st = local_bases(s, bucket, bucket_grad, bucket_out, &g, &o);
  if (st != COVAP_OK) return st;
  return covap_dense_bucket_ready(s, comm, bucket, const_cast<char*>(g), o, stream);
}

covap_status covap_step_finish(covap_state* s, void* stream) {
  return guarded([&] {
    need(s != nullptr, "NULL state");
    DeviceGuard dg(s->device);
    CK(cudaEventRecord(s->done, s->comm_stream));
    CK(cudaStreamWaitEvent(as_stream(stream), s->done, 0));
    ++s->num_steps;
  });
}

covap_status covap_state_last_comm_ms(covap_state* s, double* dur, size_t n) {
  return guarded([&] {
    need(s && dur, "NULL argument");
    need(n <= s->plan.buckets.size(), "n exceeds bucket count");
    DeviceGuard dg(s->device);
    CK(cudaStreamSynchronize(s->comm_stream));
    for (size_t b = 0; b < n; ++b) {
      if (!s->timed[b]) {
        dur[b] = -1.0;
        continue;
      }
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, s->arrive[b], s->end[b]));
      dur[b] = ms;
    }
  });
}

// ---------------------------------------------------------------- comm

covap_status covap_comm_unique_id(uint8_t id[128]) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId uid;
    NK(ncclGetUniqueId(&uid));
    std::memcpy(id, &uid, 128);
  });
}

covap_status covap_comm_create(const uint8_t id[128], int nranks, int rank, int device,
                               covap_comm** out) {
  return guarded([&] {
    need(id && out, "NULL argument");
    need(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / world size");
    DeviceGuard dg(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    auto* c = new covap_comm;
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    const ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      throw NcclError{r, "ncclCommInitRank"};
    }
    {
      std::lock_guard<std::mutex> lock(g_comms_mu);
      g_live_comms.insert(c);
    }
    *out = c;
  });
}

void covap_comm_destroy(covap_comm* c) {
  if (!c) return;
  {
    std::lock_guard<std::mutex> lock(g_comms_mu);
    g_live_comms.erase(c);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (ncclWindow_t w : c->windows) ncclCommWindowDeregister(c->nccl, w);
    c->windows.clear();
    for (covapb::NcclPeerMem* m : c->peer_mems) covapb::nccl_peer_mem_release(c->nccl, m);
    c->peer_mems.clear();
    if (prev >= 0) cudaSetDevice(prev);
  }
  if (c->nccl) ncclCommDestroy(c->nccl);
  delete c;
}

covap_status covap_comm_size(const covap_comm* c, int* nranks, int* rank) {
  return guarded([&] {
    need(c != nullptr, "NULL comm");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
  });
}

covap_status covap_allreduce(covap_comm* c, void* buf, uint64_t count, int dtype, void* stream) {
  return guarded([&] {
    need(c && buf, "NULL argument");
    if (count == 0 || c->nranks == 1) return;
    DeviceGuard dg(c->device);
    NK(ncclAllReduce(buf, buf, count, nccl_type(dtype), ncclSum, c->nccl, as_stream(stream)));
  });
}

covap_status covap_comm_allreduce_mean(covap_comm* c, int dtype, void* buf, void* out,
                                       uint64_t count, void* stream) {
  return guarded([&] {
    need(dtype == COVAP_F32 || dtype == COVAP_F64, "bad dtype");
    if (count == 0) return;  // allreduce_mean of empty vectors is empty (trainer.cpp:40)
    need(buf && out, "NULL argument");
    need_aligned(buf, "buf");
    need_aligned(out, "out");
    const int P = world(c);
    int dev = 0;
    if (c) {
      dev = c->device;
    } else {
      CK(cudaGetDevice(&dev));
    }
    DeviceGuard dg(dev);
    cudaStream_t st = as_stream(stream);
    if (c && P > 1) NK(ncclAllReduce(buf, buf, count, nccl_type(dtype), ncclSum, c->nccl, st));
    // (0 + sum) * (1/P), trainer.cpp:41-45: one row, scale 1/P
    CK(covapb::launch_mean_rows(dtype, buf, out, 1, count, st, 1.0 / static_cast<double>(P)));
  });
}

covap_status covap_comm_profile_exchange(covap_comm* c, const double* dur, size_t n_coll,
                                         double comp_ms, double* aligned_ms, double* comp_out) {
  return guarded([&] {
    need(dur && aligned_ms && comp_out, "NULL argument");
    if (!c) {
      std::copy(dur, dur + n_coll, aligned_ms);
      *comp_out = comp_ms;
      return;
    }
    DeviceGuard dg(c->device);
    std::vector<double> host(n_coll + 1);
    std::copy(dur, dur + n_coll, host.begin());
    host[n_coll] = comp_ms;
    double* d = nullptr;
    cudaStream_t st = nullptr;
    CK(cudaMalloc(&d, host.size() * sizeof(double)));
    try {
      CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      CK(cudaMemcpyAsync(d, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, st));
      NK(ncclGroupStart());
      if (n_coll) NK(ncclAllReduce(d, d, n_coll, ncclFloat64, ncclMin, c->nccl, st));
      NK(ncclBroadcast(d + n_coll, d + n_coll, 1, ncclFloat64, 0, c->nccl, st));
      NK(ncclGroupEnd());
      CK(cudaMemcpyAsync(host.data(), d, host.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } catch (...) {
      if (st) cudaStreamDestroy(st);
      cudaFree(d);
      throw;
    }
    cudaStreamDestroy(st);
    cudaFree(d);
    std::copy(host.begin(), host.begin() + n_coll, aligned_ms);
    *comp_out = host[n_coll];
  });
}

// ---------------------------------------------------------------- memory / generic kernels

covap_status covap_device_alloc(int device, uint64_t bytes, void** out) {
  return guarded([&] {
    need(out != nullptr, "NULL out");
    DeviceGuard dg(device);
    *out = nullptr;
    CK(cudaMalloc(out, std::max<uint64_t>(bytes, 16)));
  });
}

covap_status covap_device_free(int device, void* p) {
  return guarded([&] {
    DeviceGuard dg(device);
    CK(cudaFree(p));
  });
}

covap_status covap_memcpy(void* dst, const void* src, uint64_t bytes, int kind, void* stream) {
  return guarded([&] {
    need(kind >= 0 && kind <= 2, "kind must be 0 (H2D), 1 (D2H) or 2 (D2D)");
    if (bytes == 0) return;
    need(dst && src, "NULL argument");
    const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                             : kind == 1 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    CK(cudaMemcpyAsync(dst, src, bytes, k, as_stream(stream)));
  });
}

covap_status covap_stream_synchronize(void* stream) {
  return guarded([&] { CK(cudaStreamSynchronize(as_stream(stream))); });
}

covap_status covap_embed(int device, int dtype, const void* payload, void* out, uint64_t total,
                         const uint64_t* sel_begin, const uint64_t* sel_end,
                         const uint64_t* payload_off, size_t nsel, double scale, int mean,
                         void* stream) {
  return guarded([&] {
    need(out != nullptr && (nsel == 0 || (payload && sel_begin && sel_end && payload_off)),
         "NULL argument");
    need(dtype == COVAP_F32 || dtype == COVAP_F64, "bad dtype");
    need_aligned(out, "out");
    std::vector<covapb::Run> runs(nsel);
    for (size_t i = 0; i < nsel; ++i) {
      need(sel_begin[i] <= sel_end[i] && sel_end[i] <= total, "selection range out of bounds");
      need(i == 0 || sel_begin[i] >= sel_end[i - 1], "selection ranges must ascend");
      runs[i] = covapb::Run{sel_begin[i], sel_end[i], payload_off[i]};
    }
    DeviceGuard dg(device);
    cudaStream_t st = as_stream(stream);
    covapb::Run* d_runs = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d_runs), std::max<size_t>(nsel, 1) * sizeof(covapb::Run), st));
    if (nsel)
      CK(cudaMemcpyAsync(d_runs, runs.data(), nsel * sizeof(covapb::Run), cudaMemcpyHostToDevice, st));
    const cudaError_t e = covapb::launch_unpack(dtype, payload, out, d_runs, static_cast<int>(nsel),
                                                0, total, scale, mean, st);
    cudaFreeAsync(d_runs, st);
    CK(e);
    CK(cudaStreamSynchronize(st));  // the host run table above is stack memory
  });
}

covap_status covap_mean_rows(int device, int dtype, const void* rows, void* out, uint64_t P,
                             uint64_t n, void* stream) {
  return guarded([&] {
    need(rows && out, "NULL argument");
    need(P >= 1, "allreduce needs at least one worker vector");
    DeviceGuard dg(device);
    CK(covapb::launch_mean_rows(dtype, rows, out, P, n, as_stream(stream)));
  });
}

// ---------------------------------------------------------------- harness

uint64_t covap_stream_key(uint64_t seed, uint64_t rank, uint64_t step) {
  return covapb::stream_key(seed, rank, step);
}

covap_status covap_generate(void* out, uint64_t n, int dtype, uint64_t key, int kind,
                            uint64_t begin, void* stream) {
  return guarded([&] {
    need(out != nullptr, "NULL out");
    need(dtype == COVAP_F32 || dtype == COVAP_F64, "bad dtype");
    need_aligned(out, "out");
    CK(covapb::launch_generate(dtype, out, n, key, kind, begin, as_stream(stream)));
  });
}

covap_status covap_spin(double us, int blocks, void* stream) {
  return guarded([&] { CK(covapb::launch_spin(us, blocks, as_stream(stream))); });
}

covap_status covap_busy(double us, double slice_us, void* stream) {
  return guarded([&] { CK(covapb::launch_busy(us, slice_us, as_stream(stream))); });
}

}  // extern "C"

// ---------------------------------------------------------------- peer collective
//
// C1 as one load/store kernel over NVLink peer memory (covap_peer.cu): the
// packed send buffers live in memory every rank can address — CUDA IPC
// between processes, plain device pointers within one process — and the
// allreduce sums them in rank order.

struct covap_peer {
  int device = 0;
  int P = 1, rank = 0;
  uint64_t cap = 0;                 // send-buffer capacity, elements
  size_t esize = 4;
  void* bufs[2] = {nullptr, nullptr};  // my send buffers (step parity)
  uint64_t* flags = nullptr;           // my flag block (covapb::peer_flag_words(cmax) words)
  uint64_t cmax = 0;                   // send chunks the flag block covers (whole-step mode)
  unsigned* counter = nullptr;
  unsigned* queue = nullptr;           // whole-step mode: work queue + finished CTAs
  int* err = nullptr;
  void* peer_bufs[2][covapb::kMaxPeers] = {};
  uint64_t* peer_flags[covapb::kMaxPeers] = {};
  std::vector<void*> opened;  // IPC mappings to close
  uint64_t epoch = 0;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;  // 20 s
  int max_ctas = 0;
  bool attached = false;
  // 0: K1, allreduce kernel (all-gather), K2; 1: K1, allreduce kernel with
  // the unpack fused (default); 2: the whole step in one kernel (peer_step_kernel)
  int mode = 1;
  uint64_t posted = 0;  // last epoch at which every rank published an arrival
  // Collective launches so far.  The send buffer is picked by its parity, not
  // by the step's: a step with an empty selection launches no collective (no
  // barrier), so two step-parity-equal steps around empty phases could have
  // no barrier between them, and K1 of the later one could rewrite a buffer
  // a slower peer is still reading.  Consecutive LAUNCHES alternate buffers,
  // and launch j + 2 is packed only after this rank passed launch j + 1's
  // arrival barrier, which every peer reaches only after finishing launch j.
  uint64_t launches = 0;
  // NCCL transport (covap_peer_create_nccl): the buffers and flag block live
  // in one NCCL symmetric window; mc[k] = buffer k's NVSwitch multicast
  // address when multimem was requested (NULL otherwise).
  covapb::NcclPeerMem* nmem = nullptr;
  covap_comm* ncomm = nullptr;
  void* mc[2] = {nullptr, nullptr};
};

extern "C" {

covap_status covap_peer_create(covap_state* s, int nranks, int rank, covap_peer** out) {
  covap_peer* p = nullptr;
  const covap_status st = guarded([&] {
    need(s && out, "NULL argument");
    need(nranks >= 1 && nranks <= covapb::kMaxPeers && rank >= 0 && rank < nranks,
         "peer collective supports 1..8 ranks");
    DeviceGuard dg(s->device);
    p = new covap_peer;
    p->device = s->device;
    p->P = nranks;
    p->rank = rank;
    p->esize = s->esize;
    p->cap = s->send_cap + 64;  // room for the last vector
    for (int k = 0; k < 2; ++k) {
      CK(cudaMalloc(&p->bufs[k], p->cap * p->esize));
      CK(cudaMemset(p->bufs[k], 0, p->cap * p->esize));  // alignment gaps stay zero
    }
    p->cmax = (p->cap + covapb::kPeerChunk - 1) / covapb::kPeerChunk;
    const size_t fbytes = covapb::peer_flag_words(p->cmax) * sizeof(uint64_t);
    CK(cudaMalloc(reinterpret_cast<void**>(&p->flags), fbytes));
    CK(cudaMemset(p->flags, 0, fbytes));
    CK(cudaMalloc(reinterpret_cast<void**>(&p->counter), sizeof(unsigned)));
    CK(cudaMemset(p->counter, 0, sizeof(unsigned)));
    CK(cudaMalloc(reinterpret_cast<void**>(&p->queue), 2 * sizeof(unsigned)));
    CK(cudaMemset(p->queue, 0, 2 * sizeof(unsigned)));
    CK(cudaMalloc(reinterpret_cast<void**>(&p->err), sizeof(int)));
    CK(cudaMemset(p->err, 0, sizeof(int)));
    for (int k = 0; k < 2; ++k) p->peer_bufs[k][rank] = p->bufs[k];
    p->peer_flags[rank] = p->flags;
    *out = p;
  });
  if (st != COVAP_OK && p) covap_peer_destroy(p);
  return st;
}

covap_status covap_peer_create_nccl(covap_state* s, covap_comm* c, int multimem,
                                    covap_peer** out) {
  covap_peer* p = nullptr;
  const covap_status st = guarded([&] {
    need(s && c && out, "NULL argument");
    need(c->device == s->device, "communicator and state are on different devices");
    need(c->nranks >= 1 && c->nranks <= covapb::kMaxPeers, "peer collective supports 1..8 ranks");
    DeviceGuard dg(s->device);
    p = new covap_peer;
    p->device = s->device;
    p->P = c->nranks;
    p->rank = c->rank;
    p->esize = s->esize;
    p->cap = s->send_cap + 64;  // room for the last vector
    p->cmax = (p->cap + covapb::kPeerChunk - 1) / covapb::kPeerChunk;
    // one window: [buffer 0 | buffer 1 | flag block], 4 KB-aligned parts
    const size_t a = 4096;
    const size_t bb = (p->cap * p->esize + a - 1) / a * a;
    const size_t fbytes = covapb::peer_flag_words(p->cmax) * sizeof(uint64_t);
    const size_t bytes = (2 * bb + fbytes + NCCL_WIN_REQUIRED_ALIGNMENT - 1) /
                         NCCL_WIN_REQUIRED_ALIGNMENT * NCCL_WIN_REQUIRED_ALIGNMENT;
    void* peers[covapb::kMaxPeers] = {};
    void* mc = nullptr;
    const char* what = "";
    if (covapb::nccl_peer_mem_create(c->nccl, p->P, bytes, multimem, &p->nmem, peers, &mc, &what))
      throw covap::Error(std::string("NCCL peer window: ") + what);
    p->ncomm = c;
    {
      std::lock_guard<std::mutex> lock(g_comms_mu);
      c->peer_mems.push_back(p->nmem);
    }
    for (int q = 0; q < p->P; ++q) {
      char* b = static_cast<char*>(peers[q]);
      p->peer_bufs[0][q] = b;
      p->peer_bufs[1][q] = b + bb;
      p->peer_flags[q] = reinterpret_cast<uint64_t*>(b + 2 * bb);
    }
    p->bufs[0] = p->peer_bufs[0][p->rank];
    p->bufs[1] = p->peer_bufs[1][p->rank];
    p->flags = p->peer_flags[p->rank];
    if (mc) {
      p->mc[0] = mc;
      p->mc[1] = static_cast<char*>(mc) + bb;
    }
    CK(cudaMalloc(reinterpret_cast<void**>(&p->counter), sizeof(unsigned)));
    CK(cudaMemset(p->counter, 0, sizeof(unsigned)));
    CK(cudaMalloc(reinterpret_cast<void**>(&p->queue), 2 * sizeof(unsigned)));
    CK(cudaMemset(p->queue, 0, 2 * sizeof(unsigned)));
    CK(cudaMalloc(reinterpret_cast<void**>(&p->err), sizeof(int)));
    CK(cudaMemset(p->err, 0, sizeof(int)));
    p->attached = true;
    *out = p;
  });
  if (st != COVAP_OK && p) covap_peer_destroy(p);
  return st;
}

covap_status covap_peer_multimem(const covap_peer* p, int* on) {
  return guarded([&] {
    need(p && on, "NULL argument");
    *on = p->mc[0] != nullptr;
  });
}

void covap_peer_destroy(covap_peer* p) {
  if (!p) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  for (void* q : p->opened) cudaIpcCloseMemHandle(q);
  if (p->nmem) {  // NCCL window: released here unless its communicator went first
    std::lock_guard<std::mutex> lock(g_comms_mu);
    ncclComm_t live = nullptr;
    if (g_live_comms.count(p->ncomm)) {
      live = p->ncomm->nccl;
      auto& v = p->ncomm->peer_mems;
      v.erase(std::remove(v.begin(), v.end(), p->nmem), v.end());
    }
    covapb::nccl_peer_mem_destroy(live, p->nmem);
  } else {
    cudaFree(p->bufs[0]);
    cudaFree(p->bufs[1]);
    cudaFree(p->flags);
  }
  cudaFree(p->queue);
  cudaFree(p->counter);
  cudaFree(p->err);
  if (prev >= 0) cudaSetDevice(prev);
  delete p;
}

covap_status covap_peer_export(covap_peer* p, uint8_t* blob, size_t cap, size_t* len) {
  return guarded([&] {
    need(p && len, "NULL argument");
    need(!p->nmem, "an NCCL-window peer is attached at creation (nothing to export)");
    constexpr size_t h = sizeof(cudaIpcMemHandle_t);
    *len = 3 * h;
    if (!blob) return;
    need(cap >= 3 * h, "blob too small");
    DeviceGuard dg(p->device);
    cudaIpcMemHandle_t hs[3];
    CK(cudaIpcGetMemHandle(&hs[0], p->bufs[0]));
    CK(cudaIpcGetMemHandle(&hs[1], p->bufs[1]));
    CK(cudaIpcGetMemHandle(&hs[2], p->flags));
    std::memcpy(blob, hs, 3 * h);
  });
}

covap_status covap_peer_import(covap_peer* p, const uint8_t* blobs, size_t len) {
  return guarded([&] {
    need(p && blobs, "NULL argument");
    constexpr size_t h = sizeof(cudaIpcMemHandle_t);
    need(len == 3 * h, "blob length mismatch");
    need(!p->nmem, "an NCCL-window peer is attached at creation (nothing to import)");
    DeviceGuard dg(p->device);
    for (int q = 0; q < p->P; ++q) {
      if (q == p->rank) continue;
      cudaIpcMemHandle_t hs[3];
      std::memcpy(hs, blobs + q * len, 3 * h);
      void* ptr[3];
      for (int k = 0; k < 3; ++k) {
        CK(cudaIpcOpenMemHandle(&ptr[k], hs[k], cudaIpcMemLazyEnablePeerAccess));
        p->opened.push_back(ptr[k]);
      }
      p->peer_bufs[0][q] = ptr[0];
      p->peer_bufs[1][q] = ptr[1];
      p->peer_flags[q] = static_cast<uint64_t*>(ptr[2]);
    }
    p->attached = true;
  });
}

covap_status covap_peer_attach_local(covap_peer** peers, int nranks) {
  return guarded([&] {
    need(peers != nullptr && nranks >= 1 && nranks <= covapb::kMaxPeers, "bad peer list");
    for (int i = 0; i < nranks; ++i) {
      need(peers[i] && peers[i]->P == nranks && peers[i]->rank == i, "peer i must be rank i");
      need(!peers[i]->nmem, "an NCCL-window peer is attached at creation");
    }
    for (int i = 0; i < nranks; ++i) {
      for (int q = 0; q < nranks; ++q) {
        peers[i]->peer_bufs[0][q] = peers[q]->bufs[0];
        peers[i]->peer_bufs[1][q] = peers[q]->bufs[1];
        peers[i]->peer_flags[q] = peers[q]->flags;
      }
      peers[i]->attached = true;
    }
  });
}

covap_status covap_peer_set_limits(covap_peer* p, int max_ctas, double timeout_s) {
  return guarded([&] {
    need(p != nullptr, "NULL peer");
    p->max_ctas = max_ctas;
    if (timeout_s > 0) p->timeout_ns = static_cast<uint64_t>(timeout_s * 1e9);
  });
}

covap_status covap_peer_set_fused(covap_peer* p, int mode) {
  return guarded([&] {
    need(p != nullptr, "NULL peer");
    need(mode >= 0 && mode <= 2, "peer mode must be 0, 1 or 2");
    p->mode = mode;
  });
}

covap_status covap_peer_check(covap_peer* p) {
  return guarded([&] {
    need(p != nullptr, "NULL peer");
    DeviceGuard dg(p->device);
    int err = 0;
    CK(cudaMemcpy(&err, p->err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) throw covap::Error("peer collective timed out waiting for a rank");
  });
}

covap_status covap_peer_sync_step(covap_state* s, covap_peer* p, const void* grad, void* out,
                                  void* stream) {
  return guarded([&] {
    need(s && p && grad && out, "NULL argument");
    need(p->attached || p->P == 1, "peer buffers are not attached (covap_peer_import)");
    need(p->device == s->device && p->esize == s->esize, "peer and state differ");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    DeviceGuard dg(s->device);
    cudaStream_t st = as_stream(stream);
    const uint64_t n = s->plan.dtotal;
    const auto& ph = phase_of(s->plan, s->num_steps);
    const int par = static_cast<int>(p->launches & 1);
    void* buf = p->bufs[par];
    if (p->mode == 2) {  // K1 + collective + unpack in one kernel
      need(!p->mc[0], "the whole-step kernel (mode 2) has no multimem variant: use mode 0 or 1");
      covapb::PeerStepArgs a{};
      for (int q = 0; q < p->P; ++q) {
        a.bufs[q] = p->peer_bufs[par][q];
        a.flags[q] = p->peer_flags[q];
      }
      a.queue = p->queue;
      a.err = p->err;
      a.epoch = ++p->epoch;
      a.wait_epoch = p->posted;
      a.len = ph.send_elems;
      a.cmax = p->cmax;
      a.timeout_ns = p->timeout_ns;
      a.P = p->P;
      a.rank = p->rank;
      a.g = grad;
      a.r = s->residual;
      a.out = out;
      a.runs = s->d_runs + s->phase_off[s->num_steps % s->plan.interval];
      a.nruns = static_cast<int>(ph.runs.size());
      a.n_out = n;
      a.coeff = coeff_of(s);
      a.ef = s->ef.enabled;
      a.inv = 1.0 / static_cast<double>(p->P);
      need(a.len <= p->cmax * covapb::kPeerChunk, "send length exceeds the peer flag capacity");
      CK(covapb::launch_peer_step(s->dtype, a, p->max_ctas, st));
      ++p->launches;
      p->posted = p->epoch;
      ++s->num_steps;
      return;
    }
    k1_range(s, grad, buf, 0, n, st, out);  // + zero fill of the unselected output
    ++p->epoch;
    if (ph.send_elems > 0) p->posted = p->epoch;
    if (ph.send_elems > 0) {
      covapb::PeerArgs a{};
      for (int q = 0; q < p->P; ++q) {
        a.bufs[q] = p->peer_bufs[par][q];
        a.flags[q] = p->peer_flags[q];
      }
      a.counter = p->counter;
      a.err = p->err;
      a.epoch = p->epoch;
      a.len = ph.send_elems;
      a.timeout_ns = p->timeout_ns;
      a.P = p->P;
      a.rank = p->rank;
      a.fused = p->mode == 1 ? 1 : 0;
      a.out = out;
      a.runs = s->d_runs + s->phase_off[s->num_steps % s->plan.interval];
      a.nruns = static_cast<int>(ph.runs.size());
      a.n_out = n;
      a.inv = 1.0 / static_cast<double>(p->P);
      a.zfill = 0;  // K1 zeroed the unselected output
      a.mc = p->mc[par];
      CK(covapb::launch_peer_allreduce(s->dtype, a, p->max_ctas, st));
      ++p->launches;
    }
    // fused: the collective already wrote the selected output (C1 + K2 in one kernel)
    if (p->mode != 1) k2sel_range(s, buf, out, 1.0 / static_cast<double>(p->P), 0, n, st);
    ++s->num_steps;
  });
}

}  // extern "C"
