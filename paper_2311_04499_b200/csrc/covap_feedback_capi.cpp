// covap_feedback_capi.cpp — C-ABI of the baseline compressors under the
// generic error-feedback wrapper (include/covap_c.h, covap_feedback_*;
// SURVEY.md §8(f4)).
//
// Reference map (paths under /root/reference/proj):
//   covap_feedback_create      ErrorFeedback::ErrorFeedback, compress.cpp:316-321
//   covap_feedback_step        ErrorFeedback::step, compress.cpp:323-344, with
//                              GradientFilter::keep, compress.cpp:241-309
//   covap_feedback_transmitted transmitted_elements, compress.cpp:246-314; bytes
//                              as train() counts them, trainer.cpp:396-400
//   covap_feedback_sync_step   the non-COVAP branch of train(), trainer.cpp:387-403
//   covap_topk_compress        topk_compress, compress.cpp:119-133
//   covap_randomk_compress     randomk_compress, compress.cpp:135-155
//   covap_fp16_roundtrip       fp16_roundtrip, compress.cpp:226-236
//   covap_sparsifier_k         sparsifier_k, compress.cpp:107-116
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "covap_capi_common.hpp"
#include "covap_feedback.h"
#include "covap_internal.h"
#include "covap_plan.hpp"

namespace fb = covapb::fb;

struct covap_feedback {
  int dtype = COVAP_F32;
  size_t esize = 4;
  int device = 0;
  int sms = 148;
  covap_ef ef{1, 0.3, 100, 0.1};
  covap_filter filter{};
  std::vector<uint64_t> numel, begin, k, list_off;
  uint64_t total = 0, k_total = 0;
  uint64_t num_steps = 0;
  void* residual = nullptr;
  fb::Chunk* chunks = nullptr;
  uint32_t nchunks = 0;
  uint64_t* d_begin = nullptr;
  uint64_t* d_numel = nullptr;
  uint64_t* d_list_off = nullptr;
  unsigned long long* d_sat = nullptr;
  // top-k
  uint32_t* hist = nullptr;
  uint32_t* d_k = nullptr;
  uint32_t* thr = nullptr;
  uint32_t* need = nullptr;
  uint32_t* sel_cnt = nullptr;
  uint32_t* cand_cnt = nullptr;
  void* cand_key = nullptr;
  uint32_t* cand_idx = nullptr;
  uint32_t* hist2 = nullptr;
  uint32_t* thr2 = nullptr;
  uint32_t* need2 = nullptr;
  uint32_t* cand2_cnt = nullptr;
  void* cand2_key = nullptr;
  uint32_t* cand2_idx = nullptr;
  void* acc = nullptr;  // rank-ordered scatter accumulator, zero between steps
  // random-k
  uint32_t* tensor_of = nullptr;
  uint32_t *j = nullptr, *prv = nullptr, *src = nullptr;
  uint32_t *key = nullptr, *draw_iota = nullptr, *key_sorted = nullptr, *draw_sorted = nullptr;
  void* sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  unsigned long long* table = nullptr;  // hash variant of the selection (tbits > 0)
  uint32_t tbits = 0;
  uint32_t *slot = nullptr, *nxt = nullptr;
  int* reject = nullptr;
  cudaStream_t side = nullptr;  // index sampling, concurrent with the compensation pass
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // Selections made ahead: pos[b] holds the flat sampled positions of step
  // pos_step[b] (b = step & 1) once ev_pos[b] completes; ev_used[b] marks
  // the gather that last read pos[b].
  uint32_t* pos[3] = {};
  uint32_t* bits[3] = {};  // sample bitmaps (n / 32 + 8 words), zero between uses
  uint32_t* toff[3] = {};  // list offset of every filter tile
  uint64_t rk_te = 0, rk_ntiles = 0;       // the fused pass's tile geometry
  int rk_free = 0;                         // SMs the pass leaves to the selection chain
  uint32_t* rk_cnt = nullptr;
  void* rk_tmp = nullptr;
  size_t rk_tmp_bytes = 0;
  uint64_t pos_step[3] = {~0ull, ~0ull, ~0ull};
  cudaEvent_t ev_pos[3] = {}, ev_used[3] = {};
  // wire
  uint32_t* list_idx = nullptr;
  void* list_val = nullptr;
  uint16_t* half = nullptr;
  // exchange scratch
  void* recv_a = nullptr;
  void* recv_b = nullptr;
  uint64_t cap_a = 0, cap_b = 0;
  std::vector<void*> owned;
};

namespace {

template <typename P>
P* dalloc(covap_feedback* f, uint64_t bytes) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<uint64_t>(bytes, 16)));
  f->owned.push_back(p);
  return static_cast<P*>(p);
}

void release(covap_feedback* f) {
  if (!f) return;
  DeviceGuard dg(f->device);
  cudaDeviceSynchronize();
  for (void* p : f->owned) cudaFree(p);
  if (f->ev_fork) cudaEventDestroy(f->ev_fork);
  if (f->ev_join) cudaEventDestroy(f->ev_join);
  for (int b = 0; b < 3; ++b) {
    if (f->ev_pos[b]) cudaEventDestroy(f->ev_pos[b]);
    if (f->ev_used[b]) cudaEventDestroy(f->ev_used[b]);
  }
  if (f->side) cudaStreamDestroy(f->side);
  if (f->recv_a) cudaFree(f->recv_a);
  if (f->recv_b) cudaFree(f->recv_b);
  delete f;
}

uint64_t sparsifier_k(uint64_t d, double kf) {  // compress.cpp:107-116
  if (d == 0) throw covap::InvalidInput("cannot sparsify an empty vector");
  if (!(kf > 0.0) || kf > 1.0) throw covap::InvalidInput("k_fraction must be in (0, 1]");
  const auto k = static_cast<uint64_t>(std::ceil(kf * static_cast<double>(d)));
  return std::min(std::max<uint64_t>(k, 1), d);
}

bool sparse(const covap_feedback* f) {
  return f->filter.kind == COVAP_FILTER_TOPK || f->filter.kind == COVAP_FILTER_RANDOMK;
}

double coeff_of(const covap_feedback* f) {
  return f->ef.enabled ? covapb::ef_coefficient(f->num_steps, 1, f->ef.init_value,
                                                f->ef.ascend_steps, f->ef.ascend_range)
                       : 0.0;
}

fb::RandomkArgs randomk_args(covap_feedback* f, uint64_t step, uint32_t* pos) {
  fb::RandomkArgs a{};
  a.pos = pos;
  a.t_begin = f->d_begin;
  a.t_numel = f->d_numel;
  a.list_off = f->d_list_off;
  a.tensor_of = f->tensor_of;
  a.ntensors = static_cast<uint32_t>(f->numel.size());
  a.total = f->k_total;
  a.seed = f->filter.seed;
  a.step = step;
  a.j = f->j;
  a.key = f->key;
  a.draw_iota = f->draw_iota;
  a.key_sorted = f->key_sorted;
  a.draw_sorted = f->draw_sorted;
  a.sort_tmp = f->sort_tmp;
  a.sort_tmp_bytes = f->sort_tmp_bytes;
  a.layout_n = f->total;
  a.prv = f->prv;
  a.src = f->src;
  a.table = f->table;
  a.tbits = f->tbits;
  a.slot = f->slot;
  a.nxt = f->nxt;
  a.reject = f->reject;
  return a;
}

#ifndef COVAP_RK_SORT_FREE_SMS  // random-k, sort variant: SMs left to the selection chain
#define COVAP_RK_SORT_FREE_SMS 24
#endif
#ifndef COVAP_RK_AHEAD  // random-k: steps drawn ahead (0, 1 or 2) on the side stream
#define COVAP_RK_AHEAD 1
#endif
static_assert(COVAP_RK_AHEAD >= 0 && COVAP_RK_AHEAD <= 2, "COVAP_RK_AHEAD");
constexpr int kRkBufs = COVAP_RK_AHEAD + 1;  // selection buffers in rotation

// Random-k selection of `step` into buffer b on the side stream: positions,
// sample bitmap (the previous selection's words cleared first), per-tile
// list offsets of the fused pass; ev_pos[b] marks completion.
void randomk_select_marks(covap_feedback* f, uint64_t step, int b) {
  CK(fb::launch_randomk_unmark(f->pos[b], f->k_total, f->bits[b], f->sms, f->side));
  fb::RandomkArgs a = randomk_args(f, step, f->pos[b]);
  a.bits = f->bits[b];
  CK(fb::launch_randomk_select(a, f->sms, f->side));
  const uint64_t W = 16 / f->esize;  // the fused pass's vector part ends at b16
  CK(fb::launch_randomk_tile_offsets(f->bits[b], f->rk_te, f->rk_ntiles, f->total / W * W,
                                     f->total, f->rk_cnt, f->toff[b], f->rk_tmp,
                                     f->rk_tmp_bytes, f->sms, f->side));
  CK(cudaEventRecord(f->ev_pos[b], f->side));
}

// The error-feedback step.  kept: dense kept gradient (NULL = not wanted);
// zero: buffer to zero-fill (the sparse filters' kept or the sync output);
// the sparse filters leave (index, value) pairs in list_idx / list_val and
// fp16 its halves in `half` when wire is set.
void ef_step(covap_feedback* f, const void* grad, void* kept, void* zero, bool wire,
             cudaStream_t st, bool kept_mean = false) {
  const int dt = f->dtype == COVAP_F64 ? 1 : 0;
  const double coeff = coeff_of(f);
  const uint32_t nt = static_cast<uint32_t>(f->numel.size());
  switch (f->filter.kind) {
    case COVAP_FILTER_FP16:
      // the TMA-bulk filter pass (covap_kernels.cu, op 5)
      CK(covapb::launch_filter_fp16(dt, grad, f->residual, kept, kept_mean ? 1 : 0,
                                    wire ? f->half : nullptr, f->d_sat, f->total, coeff,
                                    f->ef.enabled, st));
      break;
    case COVAP_FILTER_IDENTITY:
    case COVAP_FILTER_COVAP: {
      fb::DenseArgs a{};
      a.g = grad;
      a.r = f->residual;
      a.kept = kept;
      a.kept_mean = kept_mean ? 1 : 0;
      a.wire = wire ? f->half : nullptr;
      a.sat = f->d_sat;
      a.chunks = f->chunks;
      a.nchunks = f->nchunks;
      a.ef = f->ef.enabled;
      a.coeff = coeff;
      a.step = f->num_steps;
      a.interval = f->filter.interval;
      a.rule = f->filter.rule;
      CK(fb::launch_dense(dt, f->filter.kind, a, f->sms, st));
      break;
    }
    case COVAP_FILTER_TOPK: {
      // small layouts: programmatic dependent launch along the chain and the
      // 16-byte vector compensation loop (both measured, profiles/r2_f4.md)
      const bool pdl = f->total < fb::kTopkPdlMaxElems;
      CK(fb::launch_compensate(dt, grad, f->residual, zero, f->hist, f->chunks, f->nchunks,
                               f->ef.enabled, coeff, f->sms, st, pdl, pdl));
      fb::TopkArgs a{};
      a.pdl = pdl ? 1 : 0;
      a.r = f->residual;
      a.kept = kept;
      a.kept_mean = kept_mean ? 1 : 0;
      a.chunks = f->chunks;
      a.nchunks = f->nchunks;
      a.ntensors = nt;
      a.t_begin = f->d_begin;
      a.list_off = f->d_list_off;
      a.k = f->d_k;
      a.hist1 = f->hist;
      a.hist2 = f->hist2;
      a.thr = f->thr;
      a.need = f->need;
      a.thr2 = f->thr2;
      a.need2 = f->need2;
      a.sel_cnt = f->sel_cnt;
      a.cand_cnt = f->cand_cnt;
      a.cand2_cnt = f->cand2_cnt;
      a.cand_key = f->cand_key;
      a.cand_idx = f->cand_idx;
      a.cand2_key = f->cand2_key;
      a.cand2_idx = f->cand2_idx;
      a.list_idx = f->list_idx;
      a.list_val = f->list_val;
      CK(fb::launch_topk(dt, a, f->sms, st));
      break;
    }
    case COVAP_FILTER_RANDOMK: {
      // The sampled positions depend only on (seed, step, numels), never on
      // the gradient, so they are drawn on a side stream one step ahead: the
      // selection of step s + 1 (draws -> positions -> sample bitmap ->
      // per-tile list offsets) runs under step s's pass.  The step itself is
      // ONE streaming pass (covap_kernels.cu op 6) that patches the sampled
      // elements into its tiles: r = c - c, kept, the list in position order.
      // A step that was not drawn ahead (the first, or after set_step /
      // reset) draws its own first.  Under stream capture nothing is left
      // pending across steps.
      if (kept) need(kept == zero, "random-k: kept must be the zero-filled output");
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      CK(cudaStreamIsCapturing(st, &cap));
      const bool ahead = COVAP_RK_AHEAD && cap == cudaStreamCaptureStatusNone;
      const uint64_t s0 = f->num_steps;
      const int b0 = static_cast<int>(s0 % kRkBufs);
      CK(cudaEventRecord(f->ev_fork, st));
      CK(cudaStreamWaitEvent(f->side, f->ev_fork, 0));
      if (!ahead || f->pos_step[b0] != s0) {
        if (ahead) CK(cudaStreamWaitEvent(f->side, f->ev_used[b0], 0));
        randomk_select_marks(f, s0, b0);
        f->pos_step[b0] = ahead ? s0 : ~0ull;
      }
      CK(cudaStreamWaitEvent(st, f->ev_pos[b0], 0));
      CK(covapb::launch_filter_randomk(dt, grad, f->residual, zero, kept ? 1 : 0, kept_mean ? 1 : 0,
                                       f->bits[b0], f->toff[b0], f->list_idx, f->list_val,
                                       f->total, coeff, f->ef.enabled, st, f->rk_free));
      CK(cudaEventRecord(f->ev_used[b0], st));
      if (ahead) {  // steps s0 + 1 .. s0 + AHEAD, each into the buffers the pass
                    // AHEAD + 1 steps before it read
        for (uint64_t t = s0 + 1; t <= s0 + COVAP_RK_AHEAD; ++t) {
          const int bt = static_cast<int>(t % kRkBufs);
          if (f->pos_step[bt] == t) continue;
          CK(cudaStreamWaitEvent(f->side, f->ev_used[bt], 0));
          randomk_select_marks(f, t, bt);
          f->pos_step[bt] = t;
        }
      } else {  // join the side stream back into the capture
        CK(cudaEventRecord(f->ev_join, f->side));
        CK(cudaStreamWaitEvent(st, f->ev_join, 0));
      }
      break;
    }
    default:
      throw covap::InvalidInput("unknown filter kind");
  }
  ++f->num_steps;
}

// Wire payload of one rank: a = halves (fp16) or indices (top-k), b = values.
void wire_of(covap_feedback* f, void** a, uint64_t* ba, void** b, uint64_t* bb) {
  *a = nullptr;
  *b = nullptr;
  *ba = *bb = 0;
  switch (f->filter.kind) {
    case COVAP_FILTER_FP16:
      *a = f->half;
      *ba = f->total * 2;
      break;
    case COVAP_FILTER_TOPK:
      *a = f->list_idx;
      *ba = f->k_total * 4;
      *b = f->list_val;
      *bb = f->k_total * f->esize;
      break;
    case COVAP_FILTER_RANDOMK:
      *b = f->list_val;
      *bb = f->k_total * f->esize;
      break;
    default:
      throw covap::InvalidInput("the identity / covap filters have no sync wire (use covap_sync_step)");
  }
}

void combine(covap_feedback* f, const void* ra, const void* rb, int P, void* out,
             cudaStream_t st) {
  need(P >= 1, "P must be >= 1");
  const int dt = f->dtype == COVAP_F64 ? 1 : 0;
  const double inv = 1.0 / static_cast<double>(P);  // trainer.cpp:44
  switch (f->filter.kind) {
    case COVAP_FILTER_FP16:
      CK(fb::launch_fp16_mean(dt, static_cast<const uint16_t*>(ra), P, f->total, inv, out, f->sms,
                              st));
      break;
    case COVAP_FILTER_RANDOMK:
      CK(fb::launch_list_mean_aligned(dt, f->list_idx, rb, P, f->k_total, inv, out, f->sms, st));
      break;
    case COVAP_FILTER_TOPK: {
      if (P == 1) {
        CK(fb::launch_list_mean_aligned(dt, static_cast<const uint32_t*>(ra), rb, 1, f->k_total,
                                        inv, out, f->sms, st));
        break;
      }
      const auto* idx = static_cast<const uint32_t*>(ra);
      const auto* val = static_cast<const char*>(rb);
      for (int p = 0; p < P; ++p)  // rank order (trainer.cpp:41-43)
        CK(fb::launch_list_accumulate(dt, idx + static_cast<uint64_t>(p) * f->k_total,
                                      val + static_cast<uint64_t>(p) * f->k_total * f->esize,
                                      f->k_total, f->acc, f->sms, st));
      const uint64_t all = static_cast<uint64_t>(P) * f->k_total;
      CK(fb::launch_list_finish(dt, idx, all, f->acc, inv, out, 0, f->sms, st));
      CK(fb::launch_list_finish(dt, idx, all, f->acc, inv, out, 1, f->sms, st));
      break;
    }
    default:
      throw covap::InvalidInput("the identity / covap filters have no sync wire (use covap_sync_step)");
  }
}

void grow(void** p, uint64_t* cap, uint64_t bytes) {
  if (bytes <= *cap) return;
  if (*p) CK(cudaFree(*p));
  *p = nullptr;
  CK(cudaMalloc(p, bytes));
  *cap = bytes;
}

}  // namespace

extern "C" {

covap_status covap_sparsifier_k(uint64_t d, double k_fraction, uint64_t* k) {
  return guarded([&] {
    need(k != nullptr, "k must not be NULL");
    *k = sparsifier_k(d, k_fraction);
  });
}

covap_status covap_feedback_create(const uint64_t* numels, size_t n_tensors, int dtype,
                                   const covap_ef* schedule, const covap_filter* filter,
                                   int device, covap_feedback** out) {
  covap_feedback* f = nullptr;
  const covap_status st = guarded([&] {
    need(out != nullptr && filter != nullptr, "NULL argument");
    need(n_tensors > 0 && numels != nullptr, "need at least one tensor");
    need(dtype == COVAP_F32 || dtype == COVAP_F64, "dtype must be COVAP_F32 or COVAP_F64");
    need(filter->kind >= COVAP_FILTER_IDENTITY && filter->kind <= COVAP_FILTER_FP16,
         "unknown filter kind");
    if (filter->kind == COVAP_FILTER_COVAP) need(filter->interval >= 1, "interval must be >= 1");
    if (filter->kind == COVAP_FILTER_TOPK)
      need(n_tensors <= fb::kTopkMaxTensors, "top-k: at most 49152 tensors per state");
    if (schedule && schedule->enabled) need(schedule->ascend_steps >= 1, "ascend_steps must be >= 1");
    f = new covap_feedback;
    f->dtype = dtype;
    f->esize = dtype == COVAP_F64 ? 8 : 4;
    f->device = device;
    f->filter = *filter;
    if (schedule) f->ef = *schedule;
    f->numel.assign(numels, numels + n_tensors);
    for (uint64_t n : f->numel) {
      f->begin.push_back(f->total);
      f->total += n;
    }
    need(f->total < 0xffffffffull, "at most 2^32 - 1 elements");
    if (sparse(f)) {
      f->list_off.push_back(0);
      for (uint64_t n : f->numel) {
        f->k.push_back(sparsifier_k(n, filter->k_fraction));
        f->list_off.push_back(f->list_off.back() + f->k.back());
      }
      f->k_total = f->list_off.back();
    }
    DeviceGuard dg(device);
    CK(cudaDeviceGetAttribute(&f->sms, cudaDevAttrMultiProcessorCount, device));
    // Chunks never straddle tensors; a tensor's 16-byte-unaligned head and
    // tail get chunks of their own flagged scalar (pad = 1), so every other
    // chunk can be streamed with 16-byte vectors.
    std::vector<fb::Chunk> ch;
    const uint64_t W = 16 / f->esize;
    for (size_t t = 0; t < n_tensors; ++t) {
      const uint64_t b = f->begin[t], e = b + f->numel[t];
      const uint64_t ab = std::min(e, (b + W - 1) / W * W), ae = std::max(ab, e / W * W);
      const auto tt = static_cast<uint32_t>(t);
      if (ab > b) ch.push_back({b, ab, tt, 1});
      for (uint64_t x = ab; x < ae; x += fb::kChunk) ch.push_back({x, std::min(x + fb::kChunk, ae), tt, 0});
      if (e > ae) ch.push_back({ae, e, tt, 1});
    }
    f->nchunks = static_cast<uint32_t>(ch.size());
    f->residual = dalloc<void>(f, f->total * f->esize);
    CK(cudaMemset(f->residual, 0, std::max<uint64_t>(f->total, 1) * f->esize));
    f->chunks = dalloc<fb::Chunk>(f, ch.size() * sizeof(fb::Chunk));
    CK(cudaMemcpy(f->chunks, ch.data(), ch.size() * sizeof(fb::Chunk), cudaMemcpyHostToDevice));
    f->d_begin = dalloc<uint64_t>(f, n_tensors * 8);
    f->d_numel = dalloc<uint64_t>(f, n_tensors * 8);
    CK(cudaMemcpy(f->d_begin, f->begin.data(), n_tensors * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(f->d_numel, f->numel.data(), n_tensors * 8, cudaMemcpyHostToDevice));
    f->d_sat = dalloc<unsigned long long>(f, 8);
    CK(cudaMemset(f->d_sat, 0, 8));
    if (filter->kind == COVAP_FILTER_FP16) f->half = dalloc<uint16_t>(f, f->total * 2);
    if (sparse(f)) {
      f->d_list_off = dalloc<uint64_t>(f, (n_tensors + 1) * 8);
      CK(cudaMemcpy(f->d_list_off, f->list_off.data(), (n_tensors + 1) * 8,
                    cudaMemcpyHostToDevice));
      f->list_idx = dalloc<uint32_t>(f, f->k_total * 4);
      f->list_val = dalloc<void>(f, f->k_total * f->esize);
    }
    if (filter->kind == COVAP_FILTER_TOPK) {
      f->hist = dalloc<uint32_t>(f, n_tensors * fb::kBins * 4);
      CK(cudaMemset(f->hist, 0, n_tensors * fb::kBins * 4));
      std::vector<uint32_t> k32(f->k.begin(), f->k.end());
      f->d_k = dalloc<uint32_t>(f, n_tensors * 4);
      CK(cudaMemcpy(f->d_k, k32.data(), n_tensors * 4, cudaMemcpyHostToDevice));
      f->thr = dalloc<uint32_t>(f, n_tensors * 4);
      f->need = dalloc<uint32_t>(f, n_tensors * 4);
      f->sel_cnt = dalloc<uint32_t>(f, n_tensors * 4);
      f->cand_cnt = dalloc<uint32_t>(f, n_tensors * 4);
      f->cand_key = dalloc<void>(f, f->total * f->esize);
      f->cand_idx = dalloc<uint32_t>(f, f->total * 4);
      f->hist2 = dalloc<uint32_t>(f, n_tensors * fb::kDigits * 4);
      CK(cudaMemset(f->hist2, 0, n_tensors * fb::kDigits * 4));
      f->thr2 = dalloc<uint32_t>(f, n_tensors * 4);
      f->need2 = dalloc<uint32_t>(f, n_tensors * 4);
      f->cand2_cnt = dalloc<uint32_t>(f, n_tensors * 4);
      f->cand2_key = dalloc<void>(f, f->total * f->esize);
      f->cand2_idx = dalloc<uint32_t>(f, f->total * 4);
      f->acc = dalloc<void>(f, f->total * f->esize);
      CK(cudaMemset(f->acc, 0, std::max<uint64_t>(f->total, 1) * f->esize));
    }
    if (filter->kind == COVAP_FILTER_RANDOMK) {
      std::vector<uint32_t> owner(f->k_total);
      for (size_t t = 0; t < n_tensors; ++t)
        std::fill(owner.begin() + f->list_off[t], owner.begin() + f->list_off[t + 1],
                  static_cast<uint32_t>(t));
      f->tensor_of = dalloc<uint32_t>(f, f->k_total * 4);
      CK(cudaMemcpy(f->tensor_of, owner.data(), f->k_total * 4, cudaMemcpyHostToDevice));
      need(f->k_total < 0x7fffffffull, "random-k: at most 2^31 - 1 samples per state");
      f->j = dalloc<uint32_t>(f, f->k_total * 4);
      f->prv = dalloc<uint32_t>(f, f->k_total * 4);
      f->src = dalloc<uint32_t>(f, f->k_total * 4);
      f->key = dalloc<uint32_t>(f, f->k_total * 4);
      // up to 2^20 draws: per-position lists in a hash table at load <= 1/2
      // (<= 16 MB, L2-resident); more: a radix sort of the draws by target
      f->tbits = 10;
      while ((uint64_t(1) << f->tbits) < 2 * f->k_total) ++f->tbits;
      if (f->tbits > 21) f->tbits = 0;
      if (f->tbits) {
        f->table = dalloc<unsigned long long>(f, (uint64_t(1) << f->tbits) * 8);
        CK(cudaMemset(f->table, 0, (uint64_t(1) << f->tbits) * 8));
        f->slot = dalloc<uint32_t>(f, f->k_total * 4);
        f->nxt = dalloc<uint32_t>(f, f->k_total * 4);
      } else {
        f->key_sorted = dalloc<uint32_t>(f, f->k_total * 4);
        f->draw_sorted = dalloc<uint32_t>(f, f->k_total * 4);
        std::vector<uint32_t> iota(f->k_total);
        for (uint64_t e = 0; e < f->k_total; ++e) iota[e] = static_cast<uint32_t>(e);
        f->draw_iota = dalloc<uint32_t>(f, f->k_total * 4);
        CK(cudaMemcpy(f->draw_iota, iota.data(), f->k_total * 4, cudaMemcpyHostToDevice));
        f->sort_tmp_bytes = fb::randomk_sort_bytes(f->k_total);
        f->sort_tmp = dalloc<void>(f, f->sort_tmp_bytes);
      }
      f->reject = dalloc<int>(f, n_tensors * 4);
      CK(cudaMemset(f->reject, 0, n_tensors * 4));
      CK(cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&f->ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&f->ev_join, cudaEventDisableTiming));
      // Large selections sort their draws (cub onesweep), whose CTAs need
      // shared memory the streaming pass holds on every SM it runs on: the
      // pass leaves some SMs to the chain then (VGG-16 random-k 0.516 ->
      // 0.471 ms with 32, BERT-large 1.166 -> 1.134 with 16; the hash
      // variant co-runs without shared memory and gains nothing).
      f->rk_free = f->tbits ? 0 : COVAP_RK_SORT_FREE_SMS;
      CK(covapb::filter_tiles(f->dtype == COVAP_F64 ? 1 : 0, f->total, &f->rk_te, &f->rk_ntiles,
                              f->rk_free));
      f->rk_cnt = dalloc<uint32_t>(f, (f->rk_ntiles + 1) * 4);
      f->rk_tmp_bytes = fb::randomk_scan_bytes(f->rk_ntiles);
      f->rk_tmp = dalloc<void>(f, f->rk_tmp_bytes);
      for (int b = 0; b < kRkBufs; ++b) {
        f->pos[b] = dalloc<uint32_t>(f, f->k_total * 4);
        CK(cudaMemset(f->pos[b], 0, std::max<uint64_t>(f->k_total, 1) * 4));
        f->bits[b] = dalloc<uint32_t>(f, (f->total / 32 + 8) * 4);
        CK(cudaMemset(f->bits[b], 0, (f->total / 32 + 8) * 4));
        f->toff[b] = dalloc<uint32_t>(f, ((f->rk_ntiles + 1) / 4 * 4 + 8) * 4);
        CK(cudaMemset(f->toff[b], 0, ((f->rk_ntiles + 1) / 4 * 4 + 8) * 4));
        CK(cudaEventCreateWithFlags(&f->ev_pos[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&f->ev_used[b], cudaEventDisableTiming));
      }
    }
    CK(cudaDeviceSynchronize());
    *out = f;
  });
  if (st != COVAP_OK && f) {
    try {
      release(f);
    } catch (...) {
    }
  }
  return st;
}

void covap_feedback_destroy(covap_feedback* f) {
  try {
    release(f);
  } catch (...) {
  }
}

covap_status covap_feedback_residual(covap_feedback* f, void** p, uint64_t* n) {
  return guarded([&] {
    need(f && p, "NULL argument");
    *p = f->residual;
    if (n) *n = f->total;
  });
}

covap_status covap_feedback_get_step(const covap_feedback* f, uint64_t* s) {
  return guarded([&] {
    need(f && s, "NULL argument");
    *s = f->num_steps;
  });
}

covap_status covap_feedback_set_step(covap_feedback* f, uint64_t s) {
  return guarded([&] {
    need(f != nullptr, "NULL argument");
    f->num_steps = s;
  });
}

covap_status covap_feedback_reset(covap_feedback* f, void* stream) {
  return guarded([&] {
    need(f != nullptr, "NULL argument");
    DeviceGuard dg(f->device);
    CK(cudaMemsetAsync(f->residual, 0, f->total * f->esize, as_stream(stream)));
    f->num_steps = 0;
  });
}

covap_status covap_feedback_step(covap_feedback* f, const void* grad, void* kept, void* stream) {
  return guarded([&] {
    need(f && grad && kept, "NULL argument");
    need_aligned(grad, "grad");
    need_aligned(kept, "kept");
    DeviceGuard dg(f->device);
    ef_step(f, grad, kept, kept, false, as_stream(stream));
  });
}

covap_status covap_feedback_transmitted(const covap_feedback* f, uint64_t step, uint64_t* elems,
                                        uint64_t* bytes) {
  return guarded([&] {
    need(f != nullptr, "NULL argument");
    uint64_t e = 0, b = 0;
    switch (f->filter.kind) {
      case COVAP_FILTER_COVAP: {
        const auto keep = covapb::select(step, f->filter.interval, f->numel.size(), f->filter.rule);
        for (size_t t = 0; t < keep.size(); ++t)
          if (keep[t]) e += f->numel[t];
        b = e * 4;
        break;
      }
      case COVAP_FILTER_TOPK:
      case COVAP_FILTER_RANDOMK:
        e = f->k_total;
        b = e * 8;  // index + value pairs (trainer.cpp:398-400)
        break;
      case COVAP_FILTER_FP16:
        e = f->total;
        b = e * 2;
        break;
      default:
        e = f->total;
        b = e * 4;
    }
    if (elems) *elems = e;
    if (bytes) *bytes = b;
  });
}

covap_status covap_feedback_saturations(covap_feedback* f, uint64_t* count, void* stream) {
  return guarded([&] {
    need(f && count, "NULL argument");
    DeviceGuard dg(f->device);
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, f->d_sat, 8, cudaMemcpyDeviceToHost, as_stream(stream)));
    CK(cudaStreamSynchronize(as_stream(stream)));
    *count = v;
  });
}

covap_status covap_feedback_pack(covap_feedback* f, const void* grad, void* out, void* stream) {
  return guarded([&] {
    need(f && grad, "NULL argument");
    need(!sparse(f) || out != nullptr, "out must not be NULL for the sparse filters");
    need_aligned(grad, "grad");
    if (out) need_aligned(out, "out");
    need(f->filter.kind >= COVAP_FILTER_TOPK, "the identity / covap filters have no sync wire");
    DeviceGuard dg(f->device);
    ef_step(f, grad, nullptr, sparse(f) ? out : nullptr, true, as_stream(stream));
  });
}

covap_status covap_feedback_wire(covap_feedback* f, void** a, uint64_t* ba, void** b,
                                 uint64_t* bb) {
  return guarded([&] {
    need(f && a && ba && b && bb, "NULL argument");
    wire_of(f, a, ba, b, bb);
  });
}

covap_status covap_feedback_combine(covap_feedback* f, const void* ra, const void* rb, int P,
                                    void* out, void* stream) {
  return guarded([&] {
    need(f && out, "NULL argument");
    DeviceGuard dg(f->device);
    combine(f, ra, rb, P, out, as_stream(stream));
  });
}

covap_status covap_feedback_sync_step(covap_feedback* f, covap_comm* comm, const void* grad,
                                      void* out, void* stream) {
  return guarded([&] {
    need(f && grad && out, "NULL argument");
    need_aligned(grad, "grad");
    need_aligned(out, "out");
    need(f->filter.kind >= COVAP_FILTER_TOPK,
         "the identity / covap filters have no sync wire (use covap_sync_step)");
    DeviceGuard dg(f->device);
    const cudaStream_t st = as_stream(stream);
    const int P = world(comm);
    if (P == 1) {
      // One rank: the mean is (0 + kept) * 1, so the filter writes it straight
      // into out (zero-filled first for the sparsifiers) and no wire is built.
      ef_step(f, grad, out, sparse(f) ? out : nullptr, false, st, true);
      return;
    }
    ef_step(f, grad, nullptr, sparse(f) ? out : nullptr, true, st);
    void *a, *b;
    uint64_t ba, bb;
    wire_of(f, &a, &ba, &b, &bb);
    grow(&f->recv_a, &f->cap_a, ba * P);
    grow(&f->recv_b, &f->cap_b, bb * P);
    NK(ncclGroupStart());
    if (ba) NK(ncclAllGather(a, f->recv_a, ba, ncclUint8, comm->nccl, st));
    if (bb) NK(ncclAllGather(b, f->recv_b, bb, ncclUint8, comm->nccl, st));
    NK(ncclGroupEnd());
    combine(f, f->recv_a, f->recv_b, P, out, st);
  });
}

covap_status covap_topk_compress(int device, int dtype, const void* x, uint64_t d,
                                 double k_fraction, uint64_t* indices, void* values, uint64_t* k,
                                 void* stream) {
  covap_feedback* f = nullptr;
  const covap_filter flt{COVAP_FILTER_TOPK, 1, 0, k_fraction, 0};
  const covap_ef off{0, 0.0, 1, 0.0};
  covap_status st = guarded([&] { sparsifier_k(d, k_fraction); });
  if (st != COVAP_OK) return st;
  st = covap_feedback_create(&d, 1, dtype, &off, &flt, device, &f);
  if (st != COVAP_OK) return st;
  st = guarded([&] {
    need(x && indices && values && k, "NULL argument");
    DeviceGuard dg(device);
    const cudaStream_t s = as_stream(stream);
    ef_step(f, x, nullptr, nullptr, true, s);
    CK(fb::order_list(dtype == COVAP_F64 ? 1 : 0, fb::kTopk, f->list_idx, f->list_val, f->k_total,
                      indices, values, s));
    CK(cudaStreamSynchronize(s));
    *k = f->k_total;
  });
  covap_feedback_destroy(f);
  return st;
}

covap_status covap_randomk_compress(int device, int dtype, const void* x, uint64_t d,
                                    double k_fraction, uint64_t seed, uint64_t* indices,
                                    void* values, uint64_t* k, void* stream) {
  covap_feedback* f = nullptr;
  // randomk_compress draws from SplitMix64(seed) directly; the filter's
  // per-tensor seed is mix_seed(seed', step*0x10001 + t).  Drive the kernels
  // with that seed through a one-tensor state whose draws use `seed` as is.
  const covap_filter flt{COVAP_FILTER_RANDOMK, 1, 0, k_fraction, 0};
  const covap_ef off{0, 0.0, 1, 0.0};
  covap_status st = guarded([&] { sparsifier_k(d, k_fraction); });
  if (st != COVAP_OK) return st;
  st = covap_feedback_create(&d, 1, dtype, &off, &flt, device, &f);
  if (st != COVAP_OK) return st;
  st = guarded([&] {
    need(x && indices && values && k, "NULL argument");
    DeviceGuard dg(device);
    const cudaStream_t s = as_stream(stream);
    const int dt = dtype == COVAP_F64 ? 1 : 0;
    CK(fb::launch_compensate(dt, x, f->residual, nullptr, nullptr, f->chunks, f->nchunks, 0, 0.0,
                             f->sms, s));
    fb::RandomkArgs a = randomk_args(f, 0, f->pos[0]);
    a.raw_seed = 1;
    a.seed = seed;
    CK(fb::launch_randomk_select(a, f->sms, s));
    CK(fb::launch_randomk_gather(dt, f->pos[0], f->k_total, f->residual, nullptr, 0, f->list_idx,
                                 f->list_val, f->sms, s));
    CK(fb::order_list(dt, fb::kRandomk, f->list_idx, f->list_val, f->k_total, indices, values, s));
    CK(cudaStreamSynchronize(s));
    *k = f->k_total;
  });
  covap_feedback_destroy(f);
  return st;
}

covap_status covap_fp16_roundtrip(int device, int dtype, const void* x, uint64_t n, void* out,
                                  uint64_t* saturations, void* stream) {
  covap_feedback* f = nullptr;
  const covap_filter flt{COVAP_FILTER_FP16, 1, 0, 0.0, 0};
  const covap_ef off{0, 0.0, 1, 0.0};
  if (n == 0) {
    if (saturations) *saturations = 0;
    return COVAP_OK;
  }
  covap_status st = covap_feedback_create(&n, 1, dtype, &off, &flt, device, &f);
  if (st != COVAP_OK) return st;
  st = guarded([&] {
    need(x && out, "NULL argument");
    DeviceGuard dg(device);
    const cudaStream_t s = as_stream(stream);
    fb::DenseArgs a{};
    a.g = x;
    a.r = nullptr;
    a.kept = out;
    a.sat = f->d_sat;
    a.chunks = f->chunks;
    a.nchunks = f->nchunks;
    a.ef = 0;
    CK(fb::launch_dense(dtype == COVAP_F64 ? 1 : 0, COVAP_FILTER_FP16, a, f->sms, s));
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, f->d_sat, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (saturations) *saturations = v;
  });
  covap_feedback_destroy(f);
  return st;
}

}  // extern "C"

extern "C" {

covap_status covap_fp16_encode(int device, int dtype, const void* x, uint64_t n, uint16_t* bits,
                               uint64_t* saturations, void* stream) {
  if (n == 0) {
    if (saturations) *saturations = 0;
    return COVAP_OK;
  }
  covap_feedback* f = nullptr;
  const covap_filter flt{COVAP_FILTER_FP16, 1, 0, 0.0, 0};
  const covap_ef off{0, 0.0, 1, 0.0};
  covap_status st = covap_feedback_create(&n, 1, dtype, &off, &flt, device, &f);
  if (st != COVAP_OK) return st;
  st = guarded([&] {
    need(x && bits, "NULL argument");
    DeviceGuard dg(device);
    const cudaStream_t s = as_stream(stream);
    fb::DenseArgs a{};
    a.g = x;
    a.wire = bits;
    a.sat = f->d_sat;
    a.chunks = f->chunks;
    a.nchunks = f->nchunks;
    CK(fb::launch_dense(dtype == COVAP_F64 ? 1 : 0, COVAP_FILTER_FP16, a, f->sms, s));
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, f->d_sat, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (saturations) *saturations = v;
  });
  covap_feedback_destroy(f);
  return st;
}

covap_status covap_fp16_decode(int device, const uint16_t* bits, uint64_t n, float* out,
                               void* stream) {
  return guarded([&] {
    need(n == 0 || (bits && out), "NULL argument");
    DeviceGuard dg(device);
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CK(fb::launch_fp16_decode(bits, n, out, sms, as_stream(stream)));
  });
}

}  // extern "C"
