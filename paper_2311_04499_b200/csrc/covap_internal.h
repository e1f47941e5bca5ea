// covap_internal.h — shared between the host planner / C-ABI (C++) and the
// sm_100a kernels (CUDA).  Not installed; the public boundary is
// include/covap_c.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace covapb {

// One maximal contiguous run of selected elements at one phase: flat
// [begin, end) goes to send[dst, dst + (end - begin)).  dst == begin (mod
// kSendAlign) so that 16-byte vectors of the gradient map onto 16-byte
// vectors of the send buffer.  Within a run, consecutive selected effective
// tensors are contiguous both in the flat layout and in the send buffer.
struct Run {
  uint64_t begin;
  uint64_t end;
  uint64_t dst;
};

constexpr uint64_t kSendAlign = 32;  // elements (128 B fp32, 256 B fp64)

// K1: c = g + coeff*r for flat [a, b); selected -> send, r = 0; else r = c
// and, when out != NULL, out = 0 (the zero fill of covap_decompress,
// compress.cpp:91, moved ahead of the allreduce so the unpack after it only
// touches the selected slots).  out may alias g.
cudaError_t launch_filter_pack(int dtype, const void* g, void* r, void* send, const Run* runs,
                               int nruns, uint64_t a, uint64_t b, double coeff, int ef,
                               cudaStream_t s, void* out = nullptr);
// K1F (one rank, fused K1 + K2): selected -> out = (0 + c) * inv, r = 0;
// unselected -> r = c, out = 0.  No send buffer: the allreduce over one rank
// is the identity.
cudaError_t launch_filter_unpack(int dtype, const void* g, void* r, void* out, const Run* runs,
                                 int nruns, uint64_t a, uint64_t b, double coeff, int ef,
                                 double inv, cudaStream_t s);
// K1F + SGD (one rank): selected -> params -= lr * ((0 + c) * inv), r = 0;
// unselected -> r = c, params untouched (trainer.cpp:408-409 fused).
cudaError_t launch_filter_sgd(int dtype, const void* g, void* r, void* params, const Run* runs,
                              int nruns, uint64_t a, uint64_t b, double coeff, int ef, double inv,
                              double lr, cudaStream_t s);
// The reference's Fp16Filter under error feedback (compress.cpp:300-309,
// 323-344) as a TMA-bulk filter pass over [0, n): c = g + coeff*r; h = half
// bits of c (with the reference's NaN / saturation / underflow rules); kept =
// widen(h) -> kept (as (0 + kept) when kept_mean), r = c - kept, h -> wire;
// kept and wire may be NULL; sat counts saturated values.  wire 16-byte aligned.
cudaError_t launch_filter_fp16(int dtype, const void* g, void* r, void* kept, int kept_mean,
                              uint16_t* wire, unsigned long long* sat, uint64_t n, double coeff,
                              int ef, cudaStream_t s);
// The random-k filter under error feedback as one TMA-bulk pass over [0, n)
// (compress.cpp:283-298, 323-344): c = g + coeff*r; sampled elements (bit e
// of bits[e / 32]) get r = c - c, out = keep ? kept value : 0 and the list
// entry (e, c) at toff[tile] + their rank in the tile (position order); the
// others get r = c, out = 0.  out may be NULL.  bits: n / 32 + 8 words;
// toff: filter_tiles()'s ntiles + 1 entries, padded to a multiple of 4 + 4.
// free_sms: SMs the pass leaves to work beside it (its grid is the rest).
cudaError_t launch_filter_randomk(int dtype, const void* g, void* r, void* out, int keep,
                                  int kept_mean, const uint32_t* bits, const uint32_t* toff,
                                  uint32_t* list_idx, void* list_val, uint64_t n, double coeff,
                                  int ef, cudaStream_t s, int free_sms = 0);
// Tile geometry of the filter passes over [0, n): tile te elements, ntiles
// vector tiles (elements from ntiles * te on are the scalar tail).  free_sms:
// as launch_filter_randomk's (the geometry depends on the grid).
cudaError_t filter_tiles(int dtype, uint64_t n, uint64_t* te, uint64_t* ntiles, int free_sms = 0);
// K2 + SGD: selected -> params -= lr * f(recv); unselected untouched.
cudaError_t launch_unpack_sgd(int dtype, const void* recv, void* params, const Run* runs,
                              int nruns, uint64_t a, uint64_t b, double inv, int mean, double lr,
                              cudaStream_t s);
// K2: out = in-run ? f(recv[dst + e - begin]) : 0 for flat [a, b), with
// f(x) = (0 + x) * inv when mean (allreduce_mean), x * inv otherwise.
// zfill = 0: unselected slots are not written (K1 already zeroed them), and
// the launch covers only the envelope of the selected runs in [a, b) —
// nothing at all when none is selected.
cudaError_t launch_unpack(int dtype, const void* recv, void* out, const Run* runs, int nruns,
                          uint64_t a, uint64_t b, double inv, int mean, cudaStream_t s,
                          int zfill = 1, const Run* host_runs = nullptr);
// allreduce_mean over P rows (P x n, worker-major) in worker order.
cudaError_t launch_mean_rows(int dtype, const void* rows, void* out, uint64_t P, uint64_t n,
                             cudaStream_t s, double inv = 0.0);
// K0: synthetic gradients.
cudaError_t launch_generate(int dtype, void* out, uint64_t n, uint64_t key, int kind,
                            uint64_t begin, cudaStream_t s);
// K3: spin emulator.
cudaError_t launch_spin(double us, int blocks, cudaStream_t s);
// SMs the calling thread's following K1 / K2 launches leave idle (0: none);
// returns the previous value.
int set_free_sms(int n);
struct ScopedFreeSms {
  int prev;
  explicit ScopedFreeSms(int n) : prev(set_free_sms(n)) {}
  ~ScopedFreeSms() { set_free_sms(prev); }
};
cudaError_t launch_busy(double us, double slice_us, cudaStream_t s);

uint64_t stream_key(uint64_t seed, uint64_t rank, uint64_t step);

// Peer (NVLink load/store) allreduce of the packed send buffers, rank-ordered
// (covap_peer.cu).  flags[p] is rank p's flag block: kMaxPeers uint64 per
// phase, 2 phases.
constexpr int kMaxPeers = 8;
struct PeerArgs {
  void* bufs[kMaxPeers];       // every rank's send buffer for this step
  uint64_t* flags[kMaxPeers];  // every rank's flag block
  unsigned* counter;           // this rank's grid-barrier counter
  int* err;                    // this rank's error flag (timeout)
  uint64_t epoch;              // monotonically increasing per collective
  uint64_t len;                // elements
  uint64_t timeout_ns;
  int P;
  int rank;
  // fused unpack (phase 2 writes the synchronised gradient directly, K2's
  // work: out[sel] = sum * inv read from the slice owner, out[unsel] = 0)
  int fused;
  void* out;
  const Run* runs;  // device pointer, this phase's run table
  int nruns;
  uint64_t n_out;   // device elements of out
  double inv;
  int zfill;        // fused: zero the unselected slots too (0: K1 already did)
  // NVLS: the multicast address of this launch's send buffers (NULL: none).
  // Phase 1 then reduces slice r in the switch (multimem.ld_reduce) and
  // stores the sum to every rank's buffer (multimem.st); phase 2 reads only
  // the local buffer.  The switch's summation order is not the rank order:
  // the |d| <= 1e-6 sum|x_w| tolerance applies, as for NCCL at P > 2.
  void* mc;
};
cudaError_t launch_peer_allreduce(int dtype, const PeerArgs& args, int max_ctas, cudaStream_t s);

// Peer memory from NCCL instead of CUDA IPC: `bytes` of ncclMemAlloc memory
// registered as a symmetric window on comm (collective over its ranks), every
// rank's address of it (the window's load/store-accessible peer pointers)
// and, with want_multimem, its multicast address through an NCCL device
// communicator with multimem on the NVLink team.  0 on success; else a
// description in *what.
struct NcclPeerMem;
int nccl_peer_mem_create(struct ncclComm* comm, int nranks, size_t bytes, int want_multimem,
                         NcclPeerMem** out, void** peers, void** mc, const char** what);
// Deregisters (comm != NULL: still alive) and frees.
void nccl_peer_mem_destroy(struct ncclComm* comm, NcclPeerMem* m);
// The window / device communicator only (comm going away first); the
// memory stays until nccl_peer_mem_destroy(NULL, m).
void nccl_peer_mem_release(struct ncclComm* comm, NcclPeerMem* m);

// The whole multi-rank step as ONE kernel per rank over peer memory
// (covap_peer.cu, peer_step_kernel): K1 packs the selected shards chunk by
// chunk and publishes each chunk; the chunk's owner (chunk % P) sums it over
// the P ranks in rank order as soon as every rank has published it and
// publishes the sum; every rank unpacks each reduced chunk straight from its
// owner into out (x 1/P) while the unselected range is filtered (r = c,
// out = 0).  Work items are taken from one in-order queue (pack, unselected
// tiles, reduce, unpack), so a CTA only ever waits for items already taken.
// Flag block (uint64 per rank): [0, 8) / [8, 16) the PeerArgs phases,
// [16, 24) step arrival, then chunk x published by rank q at
// 24 + 8 x + q, then the reduced flag of chunk x at 24 + 8 cmax + x.
constexpr uint64_t kPeerChunk = 32768;  // send elements per chunk
constexpr uint64_t kPeerTile = 32768;   // layout elements per unselected tile
constexpr uint64_t kPeerFlagBase = 3 * kMaxPeers;
inline uint64_t peer_flag_words(uint64_t cmax) { return kPeerFlagBase + cmax * (kMaxPeers + 1); }
struct PeerStepArgs {
  void* bufs[kMaxPeers];
  uint64_t* flags[kMaxPeers];
  unsigned* queue;        // this rank's [next item, finished CTAs]
  int* err;
  uint64_t epoch;         // this step
  uint64_t wait_epoch;    // every peer must have arrived at this epoch before my buffer is rewritten
  uint64_t len;           // send elements this step
  uint64_t cmax;          // chunk capacity of the flag block
  uint64_t timeout_ns;
  int P;
  int rank;
  const void* g;
  void* r;
  void* out;
  const Run* runs;
  int nruns;
  uint64_t n_out;
  double coeff;
  int ef;
  double inv;
};
cudaError_t launch_peer_step(int dtype, const PeerStepArgs& args, int max_ctas, cudaStream_t s);

}  // namespace covapb
