// covap_feedback.h — launchers for the baseline compressors under the generic
// error-feedback wrapper.  Internal; the boundary is
// include/covap_c.h (covap_feedback_*, covap_topk_compress, ...).
//
// Reference (paths under /root/reference/proj):
//   ErrorFeedback::step          compress.cpp:323-344
//   IdentityFilter / CovapFilter compress.cpp:241-264
//   TopkFilter / topk_compress   compress.cpp:119-133, 266-281
//   RandomkFilter / randomk      compress.cpp:135-155, 283-298
//   Fp16Filter / half bits       compress.cpp:157-236, 300-309
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace covapb {
namespace fb {

enum Kind { kIdentity = 0, kCovap = 1, kTopk = 2, kRandomk = 3, kFp16 = 4 };

constexpr int kBinBits = 12;  // top-k first-level histogram: top 12 bits of |x|
constexpr int kBins = 1 << kBinBits;
constexpr uint32_t kNone = 0xffffffffu;

// A slice of one tensor, at most kChunk elements; tensors are cut into
// chunks so a CTA's work never straddles two tensors.
struct Chunk {
  uint64_t begin;
  uint64_t end;
  uint32_t tensor;
  uint32_t pad;
};
constexpr uint64_t kChunk = 16384;

// Dense filters (identity, covap, fp16): c = g (+ coeff*r); kept = f(c);
// r = c - kept.  kept may be NULL; wire (fp16 only) receives the half bits;
// sat counts clamped values.
struct DenseArgs {
  const void* g;
  void* r;
  void* kept;
  int kept_mean;      // kept receives allreduce_mean's (0 + k) * 1 (one rank's sync output)
  uint16_t* wire;
  unsigned long long* sat;
  const Chunk* chunks;
  uint32_t nchunks;
  int ef;
  double coeff;
  uint64_t step;      // covap selection (compress.cpp:13-28)
  uint32_t interval;
  int rule;
};
cudaError_t launch_dense(int dtype, int kind, const DenseArgs& a, int sms, cudaStream_t s);

// Compensation pass of the sparsifiers: r = c; zero[i] = 0 when zero is not
// NULL; with hist, the per-tensor histogram of the top kBinBits of |c|.
// vec: 16-byte vector loop over the body chunks (small layouts).
cudaError_t launch_compensate(int dtype, const void* g, void* r, void* zero, uint32_t* hist,
                              const Chunk* chunks, uint32_t nchunks, int ef, double coeff,
                              int sms, cudaStream_t s, bool pdl = false, bool vec = false);

// Top-k after the compensation pass filled hist1: the k[t] largest |c| of
// every tensor (ties to the lower index) go to list_idx / list_val at
// list_off[t] (and kept, r = c - c).  Three levels: 4096-bin histogram,
// 2048-bin histogram of the threshold bin's candidates, exact radix select
// among the survivors.  Candidate arrays are indexed at the tensor's begin.
constexpr int kDigitBits = 11;
// The level-2 pass keeps a prefix over the tensors in shared memory.
constexpr uint64_t kTopkMaxTensors = 49152;
constexpr int kDigits = 1 << kDigitBits;
struct TopkArgs {
  void* r;
  void* kept;
  int kept_mean;      // as DenseArgs::kept_mean
  const Chunk* chunks;
  uint32_t nchunks;
  uint32_t ntensors;
  const uint64_t* t_begin;
  const uint64_t* list_off;
  const uint32_t* k;
  uint32_t* hist1;  // ntensors x kBins, zero between steps
  uint32_t* hist2;  // ntensors x kDigits, zero between steps
  uint32_t* thr;
  uint32_t* need;
  uint32_t* thr2;
  uint32_t* need2;
  uint32_t* sel_cnt;
  uint32_t* cand_cnt;
  uint32_t* cand2_cnt;
  void* cand_key;
  uint32_t* cand_idx;
  void* cand2_key;
  uint32_t* cand2_idx;
  uint32_t* list_idx;
  void* list_val;
  int pdl;  // programmatic dependent launch along the chain (small layouts)
};
// Layouts below this many elements run the top-k chain with programmatic
// dependent launch (its kernels are short enough for launch latency to show).
constexpr uint64_t kTopkPdlMaxElems = uint64_t(1) << 26;
cudaError_t launch_topk(int dtype, const TopkArgs& a, int sms, cudaStream_t s);

// Random-k: sample_without_replacement reproduced in parallel.  Entry e of
// the list belongs to tensor tensor_of[e], draw i = e - list_off[t].
struct RandomkArgs {
  const uint64_t* t_begin;
  const uint64_t* t_numel;
  const uint64_t* list_off;
  const uint32_t* tensor_of;  // per list entry
  uint32_t ntensors;
  uint64_t total;             // list entries
  uint64_t seed;
  uint64_t step;
  int raw_seed;               // 1: draw from SplitMix64(seed) itself (randomk_compress)
  uint32_t* j;                // draw targets (local)
  // sort variant (tbits = 0)
  uint32_t* key;              // draw targets (flat), the sort keys
  const uint32_t* draw_iota;  // 0, 1, ..., total - 1 (the sort values)
  uint32_t* key_sorted;
  uint32_t* draw_sorted;
  void* sort_tmp;
  size_t sort_tmp_bytes;
  uint64_t layout_n;          // elements in the layout (the sort key range)
  uint32_t* prv;
  uint32_t* src;
  // hash variant (tbits > 0): table of 2^tbits words, all 0 between
  // selections; per draw its slot and the next draw of its target's list
  unsigned long long* table;
  uint32_t tbits;
  uint32_t* slot;
  uint32_t* nxt;
  int* reject;                // per tensor
  uint32_t* pos;              // out: flat index S_e of every draw (data independent)
  uint32_t* bits;             // out (may be NULL): bit S_e of the sample bitmap set
};
// The selection alone (draws, rejection replay, swap-chain resolution) ->
// pos.  Depends only on (seed, step, numels), never on the gradient, so it
// may run ahead of the step that uses it.
cudaError_t launch_randomk_select(const RandomkArgs& a, int sms, cudaStream_t s);
size_t randomk_sort_bytes(uint64_t total);
// Sample bitmap bookkeeping for the fused random-k pass (covap_kernels.cu
// op 6): clear the words a previous selection set (its pos), and the list
// offset of every filter tile (exclusive scan of the per-tile sample counts;
// tile ntiles is the scalar tail).
cudaError_t launch_randomk_unmark(const uint32_t* pos, uint64_t total, uint32_t* bits, int sms,
                                  cudaStream_t s);
cudaError_t launch_randomk_tile_offsets(const uint32_t* bits, uint64_t te, uint64_t ntiles,
                                        uint64_t b16, uint64_t n, uint32_t* cnt, uint32_t* toff,
                                        void* tmp, size_t tmp_bytes, int sms, cudaStream_t s);
size_t randomk_scan_bytes(uint64_t ntiles);
// list[e] = (pos[e], c); kept[pos] = c; r[pos] = c - c.
cudaError_t launch_randomk_gather(int dtype, const uint32_t* pos, uint64_t total, void* r,
                                  void* kept, int kept_mean, uint32_t* list_idx, void* list_val,
                                  int sms, cudaStream_t s);

// Exchange side (the mean of the kept gradients over P ranks, trainer.cpp:402
// and 35-47): out was zero-filled by the compensation pass.
// fp16: out[i] = (0 + sum_p widen(recv[p*n + i])) * inv.
cudaError_t launch_fp16_mean(int dtype, const uint16_t* recv, int P, uint64_t n, double inv,
                             void* out, int sms, cudaStream_t s);
// Rank-aligned lists (random-k: same indices on every rank, same order):
// out[idx[e]] = (0 + sum_p vals[p*cnt + e]) * inv.
cudaError_t launch_list_mean_aligned(int dtype, const uint32_t* idx, const void* vals, int P,
                                     uint64_t cnt, double inv, void* out, int sms,
                                     cudaStream_t s);
// General lists (top-k): acc[idx] += val for rank p's list (call in rank order),
// then out[idx] = acc[idx] * inv over every rank's list, then acc[idx] = 0.
cudaError_t launch_list_accumulate(int dtype, const uint32_t* idx, const void* val, uint64_t cnt,
                                   void* acc, int sms, cudaStream_t s);
cudaError_t launch_list_finish(int dtype, const uint32_t* idx, uint64_t cnt, void* acc,
                               double inv, void* out, int clear, int sms, cudaStream_t s);

// float_from_half_bits over a vector (compress.cpp:207-224).
cudaError_t launch_fp16_decode(const uint16_t* bits, uint64_t n, float* out, int sms,
                               cudaStream_t s);

// Reference output order for the standalone compressors: top-k by (|x| desc,
// index asc), random-k by index asc.  idx are positions; writes 64-bit
// positions and values.
cudaError_t order_list(int dtype, int kind, const uint32_t* idx, const void* val, uint64_t cnt,
                       uint64_t* out_idx, void* out_val, cudaStream_t s);

}  // namespace fb
}  // namespace covapb
