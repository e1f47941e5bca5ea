// covap_kernels.cu — the sm_100a kernels of the COVAP sync path.
//
//   K1  filter_pack    compress.cpp:59-81 (EF add, round-robin select, pack,
//                      residual write-back)
//   K1F filter_unpack  K1 + K2 fused for one rank: the allreduce over one
//                      rank is the identity (trainer.cpp:41-45 with P = 1),
//                      so c goes straight to its flat slot of the output
//   K2  unpack         compress.cpp:87-103 + trainer.cpp:41-45 (embed,
//                      sum-then-scale, zero fill)
//   K0  generate       synthetic gradients (rng.hpp:12-21 splitmix64 stream)
//   K3  spin           backward emulator for the overlap schedule
//
// K1/K1F/K2 are HBM-streaming passes (~0.2 flop/byte): no tensor cores.
// They are persistent TMA-bulk pipelines (design measured with
// scripts/kbench.cu on B200: 0.89-0.98 of the copy peak for K1's 2-read /
// 2-write shape vs 0.72-0.77 for a chunked LDG/STG version):
//   * one CTA per SM (160 KB smem) walks 16 KB tiles of the launch range in
//     interleaved order (tile = blockIdx + k * gridDim): all SMs stream
//     through neighbouring DRAM pages at any instant;
//   * thread 0 keeps kStages tiles of g and r (K2: kStagesK2 tiles of recv)
//     in flight with cp.async.bulk (global -> smem, mbarrier complete_tx);
//     results are staged in smem and written back with cp.async.bulk
//     (smem -> global); zero streams (residual reset of selected shards,
//     zero fill of unselected output) are plain 128-bit stores by all
//     threads, so the bulk-store queue only carries data;
//   * selection is positional: each tile binary-searches the phase's run
//     table (a few entries, L1-resident) and is "none selected" or "all
//     selected" (bulk path) or "mixed" (element path; only the tiles that
//     straddle a shard boundary);
//   * arithmetic uses __fmul_rn/__fadd_rn (__dmul_rn/__dadd_rn): nvcc can
//     never contract g + coeff*r into an FMA, so the multiply and the add
//     round separately exactly as compress.cpp:64 does on x86-64.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include <cub/cub.cuh>

#include "covap_half.cuh"
#include "covap_internal.h"

namespace covapb {
#ifdef COVAP_K2_TRACE
// Diagnostic build only: per-CTA K2 timeline (start, end ns; full / none /
// mixed tile counts; ns spent waiting on the load barrier).
__device__ unsigned long long g_k2_trace[1024 * 6];
#endif
namespace {

// Pipeline shape (defaults = the measured best on B200, see DESIGN.md §3;
// the macros exist so scripts/variants.sh can A/B them in one GPU session).
#ifndef COVAP_K1_STAGES
#define COVAP_K1_STAGES 2
#endif
#ifndef COVAP_K2_STAGES
#define COVAP_K2_STAGES 4
#endif
#ifndef COVAP_K1_TILE
#define COVAP_K1_TILE 24576
#endif
#ifndef COVAP_K2_TILE
#define COVAP_K2_TILE 32768
#endif
#ifndef COVAP_K1_MIN_WAVES  // small ranges: shrink tiles until every SM gets this many
#define COVAP_K1_MIN_WAVES 0
#endif
#ifndef COVAP_K2_MIN_WAVES
#define COVAP_K2_MIN_WAVES 0
#endif
#ifndef COVAP_FILTER_THREADS  // threads per CTA of the K1 / K1F / K1F+SGD passes
#define COVAP_FILTER_THREADS 256
#endif
#ifndef COVAP_FP16_THREADS  // threads per CTA of the fp16 filter pass (op 5)
#define COVAP_FP16_THREADS 1024
#endif
#ifndef COVAP_PDL  // programmatic dependent launch between consecutive sync kernels
#define COVAP_PDL 1
#endif
constexpr int kThreads = 256;
// K1/K1F: kStages slots of (g, r) tiles + 2 staging tiles + 1 zero tile;
// K1F+SGD adds a params tile per slot.
constexpr uint32_t kTileK1 = COVAP_K1_TILE;
constexpr int kStages = COVAP_K1_STAGES;
constexpr uint32_t kSmemK1 = (2 * kStages + 3) * kTileK1;
constexpr uint32_t kSmemK1Sgd = (3 * kStages + 3) * kTileK1;
// K1 fp16 (the reference's Fp16Filter under error feedback): per staging
// buffer a residual tile, a kept tile and the tile's fp16 wire halves.
constexpr uint32_t kStageFp16 = 2 * kTileK1 + kTileK1 / 2;
constexpr uint32_t kSmemK1Fp16 = 2 * kStages * kTileK1 + 2 * kStageFp16;
// K1 random-k (op 6): the K1F layout plus two out staging tiles (the sampled
// kept values on zeros) and, per slot, the tile's window of the sample
// bitmap and of the per-tile list offsets.
constexpr uint32_t kBmWords = kTileK1 / 4 / 32 + 8;  // bitmap window, 16-byte aligned ends
constexpr uint32_t kSlotRk = kBmWords * 4 + 16;
constexpr uint32_t kSmemK1Rk = (2 * kStages + 5) * kTileK1 + kStages * kSlotRk;
static_assert(kSmemK1Rk <= 227 * 1024, "op 6 shared memory");
// K2: kStagesK2 recv slots + 2 staging tiles + 1 zero tile; K2+SGD adds a
// params tile per slot.
constexpr uint32_t kTileK2 = COVAP_K2_TILE;
constexpr int kStagesK2 = COVAP_K2_STAGES;
constexpr uint32_t kSmemK2 = (kStagesK2 + 3) * kTileK2;
constexpr uint32_t kSmemK2Sel = (kStagesK2 + 2) * kTileK2;  // ring + 2 staging tiles
constexpr int kStagesK2Sgd = 2;
constexpr uint32_t kSmemK2Sgd = (2 * kStagesK2Sgd + 3) * kTileK2;

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// allreduce_mean's (0.0 + sum) * (1/P) (trainer.cpp:41-45) when mean — the
// leading +0 turns a -0 sum into +0 exactly as the reference does — else the
// plain embedding of covap_decompress (compress.cpp:100) times `inv`.
template <typename T>
__device__ __forceinline__ T scale_of(T x, T inv, int mean) {
  return mul_rn(mean ? add_rn(T(0), x) : x, inv);
}

// 16-byte vector of T and lane access.
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
};
template <>
struct Vec16<double> {
  using type = double2;
};
__device__ __forceinline__ float& lane(float4& v, int q) { return reinterpret_cast<float*>(&v)[q]; }
__device__ __forceinline__ float lane(const float4& v, int q) {
  return reinterpret_cast<const float*>(&v)[q];
}
__device__ __forceinline__ double& lane(double2& v, int q) { return reinterpret_cast<double*>(&v)[q]; }
__device__ __forceinline__ double lane(const double2& v, int q) {
  return reinterpret_cast<const double*>(&v)[q];
}

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "COVAP_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra COVAP_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// L2 evict-first policy on every bulk copy of the streaming passes: nothing a
// sync step reads or writes is reused within the step (16N bytes against a
// 126 MB L2), and marking it evict-first keeps the previous step's dirty
// lines from crowding the L2 in back-to-back steps: ResNet-50 K=4 sync step
// 1533-1547 -> 1557-1565 GB/s, K1F 0.938-0.947 -> 0.953-0.958 of the copy
// peak; VGG-16 / BERT-large unchanged (profiles/r2_design.md).
#ifndef COVAP_EVICT_FIRST
#define COVAP_EVICT_FIRST 1
#endif
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  if (COVAP_EVICT_FIRST) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(evict_first_policy())
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
  }
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  if (COVAP_EVICT_FIRST) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(evict_first_policy())
                 : "memory");
  } else {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
  }
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// Wait until at most N committed bulk groups still read shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// Wait until every committed bulk group has fully completed (writes visible).
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Programmatic dependent launch: let the next kernel in the stream be
// scheduled now (its CTAs take SMs as ours exit), and wait for the previous
// kernel's memory before touching global data.  No-ops without PDL.
__device__ __forceinline__ void pdl_launch_dependents() {
  if (COVAP_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
  if (COVAP_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ------------------------------------------------------------ selection

// Smallest j with runs[j].end > x (runs sorted, disjoint).
__device__ __forceinline__ int first_run_after(const Run* __restrict__ runs, int n, uint64_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (runs[mid].end > x)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

enum TileClass { kNone = 0, kFull = 1, kMixed = 2 };

struct TileSel {
  int cls;
  int j;        // first run ending after the tile start
  uint64_t rb;  // run begin / dst (kFull)
  uint64_t rd;
};

template <typename T>
__device__ __forceinline__ TileSel classify(const Run* __restrict__ runs, int n, uint64_t e0,
                                            uint64_t e1) {
  TileSel s;
  s.j = first_run_after(runs, n, e0);
  s.rb = s.rd = 0;
  if (s.j >= n || runs[s.j].begin >= e1) {
    s.cls = kNone;
  } else if (runs[s.j].begin <= e0 && e1 <= runs[s.j].end &&
             (runs[s.j].dst - runs[s.j].begin) % (16 / sizeof(T)) == 0) {
    // (the planner always aligns dst; caller-built tables may not, and a
    // misaligned run takes the element path)
    s.cls = kFull;
    s.rb = runs[s.j].begin;
    s.rd = runs[s.j].dst;
  } else {
    s.cls = kMixed;
  }
  return s;
}

// Selected run holding e (cursor j moves forward), or -1.
__device__ __forceinline__ int run_at(const Run* __restrict__ runs, int n, int& j, uint64_t e) {
  while (j < n && runs[j].end <= e) ++j;
  return (j < n && runs[j].begin <= e) ? j : -1;
}

// ------------------------------------------------------------ kernel args

template <typename T>
struct Args {
  const T* g;      // K1/K1F: fresh gradient
  T* r;            // K1/K1F: residual store (in/out)
  T* send;         // K1: packed send buffer
  T* out;          // K1F/K2: synchronised gradient; SGD variants: the parameters
  const T* recv;   // K2: allreduced send buffer
  const Run* runs;
  int nruns;
  uint64_t a, b;   // element range of the launch (device coordinates)
  T coeff;         // EF coefficient (K1/K1F)
  int ef;          // EF enabled: read r
  T inv;           // K1F/K2 scale (1/P)
  int mean;        // K2: allreduce_mean semantics
  T lr;            // SGD variants: learning rate
  uint64_t te;     // elements per tile of this launch (set by the launcher)
  int zfill;       // K2: zero-fill unselected slots (0: K1 did it); K1 (op 0): out != NULL zero-fills
  uint16_t* wire;  // fp16 (op 5): half bits of the kept values, or NULL
  unsigned long long* sat;  // fp16: saturation count (compress.cpp:185-190), or NULL
  // random-k (op 6): sample bitmap (bit e of word e / 32), per-tile list
  // offsets (samples before each tile; entry ntiles: before the tail), the
  // list; keep: out receives the sampled kept values (as (0 + c) when mean)
  const uint32_t* bits;
  const uint32_t* toff;
  uint32_t* list_idx;
  T* list_val;
  int keep;
};

// Operations of the element path / the filter kernel:
//   0 K1 pack, 1 K1F (one rank, out), 2 K2 unpack,
//   3 K1F + SGD (one rank, params -= lr * update), 4 K2 + SGD,
//   5 fp16 filter, 6 random-k filter (see filter_kernel).
// SGD restates trainer.cpp:408-409, params -= learning_rate * update, with
// the multiply and the subtraction rounded separately.  Unselected elements
// have update 0 and p - lr * 0 == p, so their parameters are not touched.
template <typename T>
__device__ __forceinline__ T sgd(T p, T lr, T u) {
  return sub_rn(p, mul_rn(lr, u));
}

// fp16 filter of one compensated value (compress.cpp:300-309, 339-341): wire
// bits h, kept value (half widened back), residual c - kept.
template <typename T>
__device__ __forceinline__ T fp16_keep(T c, uint16_t& h, unsigned& nsat) {
  bool s = false;
  h = half_bits(static_cast<float>(c), s);
  nsat += s ? 1u : 0u;
  return static_cast<T>(half_to_float(h));
}

template <typename T, int OP>
__device__ __forceinline__ void element(const Args<T>& A, int& j, uint64_t e, T gv, T rv) {
  if (OP == 5) {
    const T c = A.ef ? add_rn(gv, mul_rn(A.coeff, rv)) : gv;
    uint16_t h;
    unsigned ns = 0;
    const T k = fp16_keep(c, h, ns);
    A.r[e] = sub_rn(c, k);
    if (A.out) A.out[e] = A.mean ? add_rn(T(0), k) : k;
    if (A.wire) A.wire[e] = h;
    if (ns && A.sat) atomicAdd(A.sat, 1ull);
    return;
  }
  const int k = run_at(A.runs, A.nruns, j, e);
  if (OP == 2 || OP == 4) {
    if (k < 0) {
      if (OP == 2 && A.zfill) A.out[e] = T(0);
      return;
    }
    const T u = scale_of(A.recv[A.runs[k].dst + (e - A.runs[k].begin)], A.inv, A.mean);
    A.out[e] = OP == 2 ? u : sgd(A.out[e], A.lr, u);
    return;
  }
  const T c = A.ef ? add_rn(gv, mul_rn(A.coeff, rv)) : gv;
  if (k >= 0) {
    if (OP == 0)
      A.send[A.runs[k].dst + (e - A.runs[k].begin)] = c;
    else if (OP == 1)
      A.out[e] = scale_of(c, A.inv, 1);
    else
      A.out[e] = sgd(A.out[e], A.lr, scale_of(c, A.inv, 1));
    A.r[e] = T(0);
  } else {
    A.r[e] = c;
    if (OP == 1 || (OP == 0 && A.out)) A.out[e] = T(0);
  }
}

// Elements [a, a16) and [b16, b) that do not fill a 16-byte vector.
template <typename T, int OP>
__device__ void edges(const Args<T>& A, uint64_t a16, uint64_t b16) {
  constexpr bool reads_g = OP == 0 || OP == 1 || OP == 3 || OP == 5;
  for (uint64_t e = A.a + threadIdx.x; e < a16; e += blockDim.x) {
    int j = first_run_after(A.runs, A.nruns, e);
    element<T, OP>(A, j, e, reads_g ? A.g[e] : T(0), (reads_g && A.ef) ? A.r[e] : T(0));
  }
  for (uint64_t e = b16 + threadIdx.x; e < A.b; e += blockDim.x) {
    int j = first_run_after(A.runs, A.nruns, e);
    element<T, OP>(A, j, e, reads_g ? A.g[e] : T(0), (reads_g && A.ef) ? A.r[e] : T(0));
  }
}

// ------------------------------------------------------------ random-k (op 6)
//
// The random-k filter under error feedback in one streaming pass
// (compress.cpp:283-298, 323-344): every element gets r = c, out = 0 (the
// compensation pass), except the sampled ones, which get r = c - c, out = the
// kept value, and go to the wire list.  The sample positions are data
// independent and arrive as a bitmap plus per-tile list offsets
// (covap_feedback.cu, drawn a step ahead on a side stream), so the pass
// patches its smem tiles before their bulk stores: no gather afterwards, and
// the list comes out in position order (the same on every rank).

// Sequential elements [a, a16) and [b16, b) (fewer than 2 x 4), thread 0.
template <typename T>
__device__ void rk_edges(const Args<T>& A, uint64_t a, uint64_t a16, uint64_t b16, uint64_t b,
                         uint32_t tail_off) {
  uint32_t slot = tail_off;
  auto one = [&](uint64_t e) {
    const T gv = A.g[e];
    const T c = A.ef ? add_rn(gv, mul_rn(A.coeff, A.r[e])) : gv;
    if ((A.bits[e / 32] >> (e % 32)) & 1u) {
      A.r[e] = sub_rn(c, c);
      if (A.out) A.out[e] = A.keep ? (A.mean ? add_rn(T(0), c) : c) : T(0);
      A.list_idx[slot] = static_cast<uint32_t>(e);
      A.list_val[slot] = c;
      ++slot;
    } else {
      A.r[e] = c;
      if (A.out) A.out[e] = T(0);
    }
  };
  // the head precedes every tile, but op 6 launches start at 0 (no head)
  for (uint64_t e = a; e < a16; ++e) one(e);
  for (uint64_t e = b16; e < b; ++e) one(e);
}

// Patch tile [e0, e1) (staged compensated values st): sampled elements get
// st = c - c, ot = kept value, and their list slots.  ot holds zeros except
// where this tile writes it.  Block-wide; ends with the tile's writes done.
template <typename T, int NT>
__device__ __forceinline__ void rk_patch(const Args<T>& A, T* st, T* ot, const unsigned char* slot,
                                         uint64_t e0, uint64_t e1, uint64_t kg) {
  using Scan = cub::BlockScan<uint32_t, NT>;
  __shared__ typename Scan::TempStorage tmp;
  const uint32_t* bw = reinterpret_cast<const uint32_t*>(slot);
  const uint32_t base = reinterpret_cast<const uint32_t*>(slot + kBmWords * 4)[kg & 3];
  const uint64_t wa = e0 / 32, wb = (e1 - 1) / 32;
  const uint32_t wlo = static_cast<uint32_t>(wa) & ~3u;
  const uint32_t nw = static_cast<uint32_t>(wb - wa + 1);  // <= TE / 32 + 2 <= NT
  uint32_t w = 0;
  if (threadIdx.x < nw) {
    const uint64_t q = wa + threadIdx.x;
    w = bw[q - wlo];
    if (q * 32 < e0) w &= ~0u << (e0 - q * 32);
    if (q * 32 + 32 > e1) w &= (1u << (e1 - q * 32)) - 1u;  // e1 - 32q in [1, 31]
  }
  if (A.keep) {  // clear ot of the tile this staging buffer carried two tiles ago
    using V = typename Vec16<T>::type;
    constexpr uint32_t W = 16 / sizeof(T);
    V z;
#pragma unroll
    for (int q = 0; q < static_cast<int>(W); ++q) lane(z, q) = T(0);
    const uint32_t n = static_cast<uint32_t>(e1 - e0);
    for (uint32_t v = threadIdx.x; v < n / W; v += NT) reinterpret_cast<V*>(ot)[v] = z;
  }
  uint32_t rank = 0;
  Scan(tmp).ExclusiveSum(static_cast<uint32_t>(__popc(w)), rank);  // its barriers order the ot fill
  rank += base;
  for (; w; w &= w - 1) {
    const uint64_t e = (wa + threadIdx.x) * 32 + (__ffs(w) - 1);
    const uint32_t i = static_cast<uint32_t>(e - e0);
    const T c = st[i];
    st[i] = sub_rn(c, c);
    if (A.keep) ot[i] = A.mean ? add_rn(T(0), c) : c;
    A.list_idx[rank] = static_cast<uint32_t>(e);
    A.list_val[rank] = c;
    ++rank;
  }
}

// ------------------------------------------------------------ K1 / K1F / K1F+SGD
//
// Input ring: kStages slots of (g, r[, params]) tiles, refilled as soon as the
// tile has been consumed.  Results go to one of two staging tiles and leave
// with a bulk store; before a staging tile is rewritten, thread 0 waits until
// the bulk store issued two tiles earlier has read it.  Zero streams (r of
// selected tiles, out of unselected tiles in K1F) are bulk stores of a
// persistent zero tile.  K1F+SGD loads a params tile only for selected tiles.

template <int OP>
constexpr int k1_slot_tiles() {
  return OP == 3 ? 3 : 2;
}

template <int OP>
__host__ __device__ constexpr int filter_threads() {
  return OP == 5 ? COVAP_FP16_THREADS : COVAP_FILTER_THREADS;  // fp16: conversion-heavy, more warps
}

template <typename T, int OP>
__global__ void __launch_bounds__(filter_threads<OP>(), 1) filter_kernel(const Args<T> A) {
  constexpr int NT = filter_threads<OP>();
  static_assert(OP == 0 || OP == 1 || OP == 3 || OP == 5 || OP == 6,
                "filter_kernel ops: 0 pack, 1 K1F, 3 K1F+SGD, 5 fp16 filter, 6 random-k filter");
  constexpr uint32_t TE = kTileK1 / sizeof(T);  // elements per tile
  using V = typename Vec16<T>::type;
  constexpr uint32_t W = 16 / sizeof(T);
  extern __shared__ __align__(128) unsigned char smem[];
  T* gin = reinterpret_cast<T*>(smem);                  // kStages tiles (g)
  T* rin = gin + kStages * TE;                          // kStages tiles (r)
  T* pin = rin + kStages * TE;                          // kStages tiles (params, OP 3)
  T* stage = (OP == 3 ? pin + kStages * TE : pin);      // 2 staging tiles
  T* zero = stage + 2 * TE;                             // zero tile
  T* ostage = zero + TE;                                // op 6: 2 out staging tiles
  unsigned char* rkslot = reinterpret_cast<unsigned char*>(ostage + 2 * TE);  // op 6: kStages x kSlotRk
  __shared__ __align__(8) uint64_t bar[kStages];

  pdl_launch_dependents();
  const uint64_t a16 = (A.a + W - 1) / W * W;
  const uint64_t b16 = A.b / W * W;
  if (OP == 6 && a16 >= b16) {  // nothing vector-sized
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) rk_edges<T>(A, A.a, A.b, A.b, A.b, A.toff[0]);
    return;
  }
  if (a16 >= b16) {  // nothing vector-sized: element path only
    pdl_wait();
    if (blockIdx.x == 0) {
      for (uint64_t e = A.a + threadIdx.x; e < A.b; e += blockDim.x) {
        int j = first_run_after(A.runs, A.nruns, e);
        element<T, OP>(A, j, e, A.g[e], A.ef ? A.r[e] : T(0));
      }
    }
    return;
  }
  const uint64_t te = A.te;  // balanced tile (<= TE): every CTA gets the same tile count
  const uint64_t ntiles = (b16 - a16 + te - 1) / te;
  const uint64_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (OP != 5)
    for (uint32_t i = threadIdx.x; i < TE; i += NT) zero[i] = T(0);
  unsigned nsat = 0;  // fp16: saturated values of this thread
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) mbar_init(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  __syncthreads();
  pdl_wait();  // the previous kernel's writes (r, out, ...) are visible from here
  if (OP == 6) {
    if (blockIdx.x == 0 && threadIdx.x == 0) rk_edges<T>(A, A.a, a16, b16, A.b, A.toff[ntiles]);
  } else if (blockIdx.x == 0) {
    edges<T, OP>(A, a16, b16);
  }

  auto tile_lo = [&](uint64_t k) { return a16 + (blockIdx.x + k * gridDim.x) * te; };
  auto issue = [&](uint64_t k) {  // thread 0 only
    const int s = static_cast<int>(k % kStages);
    const uint64_t e0 = tile_lo(k), e1 = min(e0 + te, b16);
    const uint32_t bytes = static_cast<uint32_t>((e1 - e0) * sizeof(T));
    bool with_params = false;
    if (OP == 3) with_params = classify<T>(A.runs, A.nruns, e0, e1).cls == kFull;
    uint32_t rk_bytes = 0, wlo = 0, wbytes = 0;
    if (OP == 6) {  // the tile's bitmap words and its list offset, 16-byte windows
      wlo = static_cast<uint32_t>(e0 / 32) & ~3u;
      wbytes = (((static_cast<uint32_t>((e1 + 31) / 32) + 3u) & ~3u) - wlo) * 4u;
      rk_bytes = wbytes + 16;
    }
    mbar_arrive_tx(&bar[s], (A.ef ? 2 : 1) * bytes + (with_params ? bytes : 0) + rk_bytes);
    if (OP == 6) {
      const uint64_t kg = blockIdx.x + k * gridDim.x;
      bulk_load(rkslot + s * kSlotRk, A.bits + wlo, wbytes, &bar[s]);
      bulk_load(rkslot + s * kSlotRk + kBmWords * 4, A.toff + (kg & ~3ull), 16, &bar[s]);
    }
    bulk_load(gin + s * TE, A.g + e0, bytes, &bar[s]);
    if (A.ef) bulk_load(rin + s * TE, A.r + e0, bytes, &bar[s]);
    if (with_params) bulk_load(pin + s * TE, A.out + e0, bytes, &bar[s]);
  };
  if (threadIdx.x == 0)
    for (uint64_t k = 0; k < my && k < kStages; ++k) issue(k);

  for (uint64_t k = 0; k < my; ++k) {
    const int s = static_cast<int>(k % kStages);
    const uint64_t e0 = tile_lo(k), e1 = min(e0 + te, b16);
    const uint32_t n = static_cast<uint32_t>(e1 - e0);
    const TileSel sel = classify<T>(A.runs, A.nruns, e0, e1);
    T* st = stage + (k & 1) * TE;
    const T* gs = gin + s * TE;
    const T* rs = rin + s * TE;
    const T* ps = pin + s * TE;
    if (threadIdx.x == 0) bulk_wait_read<1>();  // staging tile (k & 1) free again
    mbar_wait(&bar[s], static_cast<uint32_t>((k / kStages) & 1));
    __syncthreads();
    if (OP == 5) {
      // fp16 filter: every element is kept as its half (no selection);
      // residual, kept and wire tiles leave with bulk stores.
      unsigned char* sb = smem + 2 * kStages * kTileK1 + (k & 1) * kStageFp16;
      T* sr = reinterpret_cast<T*>(sb);
      T* sk = reinterpret_cast<T*>(sb + kTileK1);
      uint16_t* sw = reinterpret_cast<uint16_t*>(sb + 2 * kTileK1);
      const V* gv = reinterpret_cast<const V*>(gs);
      const V* rv = reinterpret_cast<const V*>(rs);
      for (uint32_t v = threadIdx.x; v < n / W; v += NT) {
        V x = gv[v];
        if (A.ef) {
          const V y = rv[v];
#pragma unroll
          for (int q = 0; q < static_cast<int>(W); ++q)
            lane(x, q) = add_rn(lane(x, q), mul_rn(A.coeff, lane(y, q)));
        }
        V res, kv;
        uint16_t h[W];
#pragma unroll
        for (int q = 0; q < static_cast<int>(W); ++q) {
          const T kq = fp16_keep(lane(x, q), h[q], nsat);
          lane(res, q) = sub_rn(lane(x, q), kq);
          lane(kv, q) = A.mean ? add_rn(T(0), kq) : kq;
        }
        reinterpret_cast<V*>(sr)[v] = res;
        reinterpret_cast<V*>(sk)[v] = kv;
        if (W == 4)
          reinterpret_cast<uint2*>(sw)[v] =
              make_uint2(h[0] | (uint32_t(h[1 % W]) << 16), h[2 % W] | (uint32_t(h[3 % W]) << 16));
        else
          reinterpret_cast<uint32_t*>(sw)[v] = h[0] | (uint32_t(h[1 % W]) << 16);
      }
      fence_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t bytes = n * sizeof(T);
        bulk_store(A.r + e0, sr, bytes);
        if (A.out) bulk_store(A.out + e0, sk, bytes);
        if (A.wire) {  // 16-byte multiple by bulk store, the rest by thread 0
          const uint32_t wb = n * 2, wb16 = wb / 16 * 16;
          if (wb16) bulk_store(A.wire + e0, sw, wb16);
          for (uint32_t i = wb16 / 2; i < n; ++i) A.wire[e0 + i] = sw[i];
        }
        bulk_commit();
        if (k + kStages < my) issue(k + kStages);
      }
      continue;
    }
    if (sel.cls != kMixed) {
      // 16-byte vectors: a warp touches 512 contiguous bytes, no bank conflicts
      const bool full = sel.cls == kFull;
      const V* gv = reinterpret_cast<const V*>(gs);
      const V* rv = reinterpret_cast<const V*>(rs);
      const V* pv = reinterpret_cast<const V*>(ps);
      V* sv = reinterpret_cast<V*>(st);
      for (uint32_t v = threadIdx.x; v < n / W; v += NT) {
        V x = gv[v];
        if (A.ef) {
          const V y = rv[v];
#pragma unroll
          for (int q = 0; q < static_cast<int>(W); ++q)
            lane(x, q) = add_rn(lane(x, q), mul_rn(A.coeff, lane(y, q)));
        }
        if (OP != 0 && full) {
#pragma unroll
          for (int q = 0; q < static_cast<int>(W); ++q) lane(x, q) = scale_of(lane(x, q), A.inv, 1);
        }
        if (OP == 3 && full) {
          const V p = pv[v];
#pragma unroll
          for (int q = 0; q < static_cast<int>(W); ++q) lane(x, q) = sgd(lane(p, q), A.lr, lane(x, q));
        }
        sv[v] = x;
      }
    } else {
      // Tile straddling a shard boundary: segments wholly selected or wholly
      // unselected, each written by the block with 16-byte vectors between
      // scalar edges (the tile itself is 16-byte aligned; segments need not be).
      int j = sel.j;
      uint64_t pos = e0;
      while (pos < e1) {
        const bool in_run = j < A.nruns && A.runs[j].begin <= pos;
        const uint64_t end = in_run ? min(e1, A.runs[j].end)
                                    : (j < A.nruns ? min(e1, A.runs[j].begin) : e1);
        const uint64_t len = end - pos, i0 = pos - e0;
        const uint64_t head = (W - pos % W) % W < len ? (W - pos % W) % W : len;
        const uint64_t nv = (len - head) / W;
        // send slot of element pos + i is send_at[i] (OP 0); vectors need
        // dst == begin (mod W)
        T* send_at = (OP == 0 && in_run) ? A.send + A.runs[j].dst + (pos - A.runs[j].begin) : nullptr;
        const bool vec_ok = !(OP == 0 && in_run) || (A.runs[j].dst - A.runs[j].begin) % W == 0;
        auto one = [&](uint64_t i) {  // element pos + i
          const uint64_t e = pos + i;
          const T c = A.ef ? add_rn(gs[i0 + i], mul_rn(A.coeff, rs[i0 + i])) : gs[i0 + i];
          if (in_run) {
            if (OP == 0) send_at[i] = c;
            else if (OP == 1) A.out[e] = scale_of(c, A.inv, 1);
            else A.out[e] = sgd(A.out[e], A.lr, scale_of(c, A.inv, 1));
            A.r[e] = T(0);
          } else {
            A.r[e] = c;
            if (OP == 1 || (OP == 0 && A.out)) A.out[e] = T(0);
          }
        };
        const uint64_t body = vec_ok ? nv : 0;
        for (uint64_t i = threadIdx.x; i < head; i += NT) one(i);
        for (uint64_t i = head + body * W + threadIdx.x; i < len; i += NT) one(i);
        for (uint64_t v = threadIdx.x; v < body; v += NT) {
          const uint64_t i = head + v * W, e = pos + i;
          V x = *reinterpret_cast<const V*>(gs + i0 + i);
          if (A.ef) {
            const V y = *reinterpret_cast<const V*>(rs + i0 + i);
#pragma unroll
            for (int q = 0; q < static_cast<int>(W); ++q)
              lane(x, q) = add_rn(lane(x, q), mul_rn(A.coeff, lane(y, q)));
          }
          V z;
#pragma unroll
          for (int q = 0; q < static_cast<int>(W); ++q) lane(z, q) = T(0);
          if (in_run) {
            if (OP == 0) {
              *reinterpret_cast<V*>(send_at + i) = x;
            } else {
              V o = OP == 3 ? *reinterpret_cast<const V*>(A.out + e) : z;
#pragma unroll
              for (int q = 0; q < static_cast<int>(W); ++q)
                lane(o, q) = OP == 1 ? scale_of(lane(x, q), A.inv, 1)
                                     : sgd(lane(o, q), A.lr, scale_of(lane(x, q), A.inv, 1));
              *reinterpret_cast<V*>(A.out + e) = o;
            }
            *reinterpret_cast<V*>(A.r + e) = z;
          } else {
            *reinterpret_cast<V*>(A.r + e) = x;
            if (OP == 1 || (OP == 0 && A.out)) *reinterpret_cast<V*>(A.out + e) = z;
          }
        }
        if (in_run) ++j;
        pos = end;
      }
    }
    T* ot = ostage + (k & 1) * TE;
    if (OP == 6) rk_patch<T, NT>(A, st, ot, rkslot + s * kSlotRk, e0, e1, blockIdx.x + k * gridDim.x);
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = n * sizeof(T);
      if (sel.cls == kFull) {
        if (OP == 0)
          bulk_store(A.send + sel.rd + (e0 - sel.rb), st, bytes);
        else
          bulk_store(A.out + e0, st, bytes);  // K1F: out; K1F+SGD: params
        bulk_store(A.r + e0, zero, bytes);    // residual reset (compress.cpp:77)
      } else if (sel.cls == kNone) {
        bulk_store(A.r + e0, st, bytes);      // r = compensated (compress.cpp:79)
        if (OP == 1 || (OP == 0 && A.out)) bulk_store(A.out + e0, zero, bytes);  // compress.cpp:91
        if (OP == 6 && A.out) bulk_store(A.out + e0, A.keep ? ot : zero, bytes);
      }
      bulk_commit();  // one group per tile (possibly empty)
      if (k + kStages < my) issue(k + kStages);  // input slot s is consumed
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
  if (OP == 5 && A.sat) {
    for (int o = 16; o > 0; o >>= 1) nsat += __shfl_xor_sync(0xffffffffu, nsat, o);
    if ((threadIdx.x & 31) == 0 && nsat) atomicAdd(A.sat, static_cast<unsigned long long>(nsat));
  }
}

// ------------------------------------------------------------ K2 / K2+SGD
//
// Only "all selected" tiles need their recv slice: they go through a
// kStagesK2-slot input ring and two staging tiles as in K1.  "None selected"
// tiles are a bulk store of the zero tile (K2) or nothing at all (K2+SGD:
// their update is zero); "mixed" tiles take the element path.

template <typename T, bool SGD>
__global__ void __launch_bounds__(kThreads, 1) unpack_kernel(const Args<T> A) {
  constexpr uint32_t TE = kTileK2 / sizeof(T);
  constexpr int OP = SGD ? 4 : 2;
  using V = typename Vec16<T>::type;
  constexpr uint32_t W = 16 / sizeof(T);
  constexpr int kSlotTiles = SGD ? 2 : 1;  // recv [+ params]
  constexpr int NS = SGD ? kStagesK2Sgd : kStagesK2;
  extern __shared__ __align__(128) unsigned char smem[];
  T* in = reinterpret_cast<T*>(smem);                // NS x kSlotTiles tiles
  T* stage = in + NS * kSlotTiles * TE;              // 2 staging tiles
  T* zero = stage + 2 * TE;                          // zero tile
  __shared__ __align__(8) uint64_t bar[NS];

  pdl_launch_dependents();
#ifdef COVAP_K2_TRACE
  unsigned long long tr_t0, tr_wait = 0, tr_full = 0, tr_none = 0, tr_mixed = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_t0));
#endif
  const uint64_t a16 = (A.a + W - 1) / W * W;
  const uint64_t b16 = A.b / W * W;
  if (a16 >= b16) {
    pdl_wait();
    if (blockIdx.x == 0)
      for (uint64_t e = A.a + threadIdx.x; e < A.b; e += blockDim.x) {
        int j = first_run_after(A.runs, A.nruns, e);
        element<T, OP>(A, j, e, T(0), T(0));
      }
    return;
  }
  const uint64_t te = A.te;  // balanced tile (<= TE)
  const uint64_t ntiles = (b16 - a16 + te - 1) / te;
  const uint64_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (uint32_t i = threadIdx.x; i < TE; i += kThreads) zero[i] = T(0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  __syncthreads();
  pdl_wait();
  if (blockIdx.x == 0) edges<T, OP>(A, a16, b16);

  auto tile_lo = [&](uint64_t k) { return a16 + (blockIdx.x + k * gridDim.x) * te; };
  // Producer (thread 0): next tile to examine, next slot sequence number;
  // only "all selected" tiles take a slot.
  uint64_t kp = 0, qp = 0;
  auto produce_one = [&]() {
    while (kp < my) {
      const uint64_t e0 = tile_lo(kp), e1 = min(e0 + te, b16);
      const TileSel sel = classify<T>(A.runs, A.nruns, e0, e1);
      ++kp;
      if (sel.cls == kFull) {
        const int s = static_cast<int>(qp % NS);
        const uint32_t bytes = static_cast<uint32_t>((e1 - e0) * sizeof(T));
        mbar_arrive_tx(&bar[s], kSlotTiles * bytes);
        bulk_load(in + s * kSlotTiles * TE, A.recv + sel.rd + (e0 - sel.rb), bytes, &bar[s]);
        if (SGD) bulk_load(in + (s * kSlotTiles + 1) * TE, A.out + e0, bytes, &bar[s]);
        ++qp;
        return;
      }
    }
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < NS; ++i) produce_one();

  uint64_t qc = 0;  // consumer slot sequence number
  for (uint64_t k = 0; k < my; ++k) {
    const uint64_t e0 = tile_lo(k), e1 = min(e0 + te, b16);
    const uint32_t n = static_cast<uint32_t>(e1 - e0);
    const TileSel sel = classify<T>(A.runs, A.nruns, e0, e1);
    if (sel.cls == kNone) {  // zero fill (compress.cpp:91); SGD or K1-filled: nothing to do
      if (!SGD && A.zfill && threadIdx.x == 0) bulk_store(A.out + e0, zero, n * sizeof(T));
#ifdef COVAP_K2_TRACE
      ++tr_none;
#endif
      continue;
    }
    if (sel.cls == kMixed) {
#ifdef COVAP_K2_TRACE
      ++tr_mixed;
#endif
      // Tiles that straddle a shard boundary: walked as segments, each
      // wholly selected (out = scale(recv), straight from global) or wholly
      // unselected (zero fill / untouched); the block handles one segment at
      // a time with 16-byte vectors — recv and out line up modulo 16 bytes
      // whenever dst == begin (mod W), which the planner guarantees — and
      // batches its loads so a segment costs about one memory latency.
      // (A per-element path here made these few tiles the critical path:
      // ~5 us each, scripts/k2_trace.py.)
      int j = sel.j;
      uint64_t pos = e0;
      while (pos < e1) {
        const bool in_run = j < A.nruns && A.runs[j].begin <= pos;
        const uint64_t end = in_run ? min(e1, A.runs[j].end)
                                    : (j < A.nruns ? min(e1, A.runs[j].begin) : e1);
        if (in_run) {
          const T* src = A.recv + A.runs[j].dst + (pos - A.runs[j].begin);
          T* dst = A.out + pos;
          const uint64_t len = end - pos;
          const uint64_t mis = (reinterpret_cast<uintptr_t>(dst) / sizeof(T)) % W;
          const uint64_t head = (len < (W - mis) % W ? len : (W - mis) % W);
          const bool aligned = ((reinterpret_cast<uintptr_t>(src) / sizeof(T)) % W) == mis;
          const uint64_t nv = aligned ? (len - head) / W : 0;
          const uint64_t body_end = aligned ? head + nv * W : 0;
          // scalar head and tail (the whole segment when misaligned)
          auto scalar = [&](uint64_t i0, uint64_t i1) {
            for (uint64_t i = i0 + threadIdx.x; i < i1; i += kThreads) {
              const T u = scale_of(src[i], A.inv, A.mean);
              dst[i] = SGD ? sgd(dst[i], A.lr, u) : u;
            }
          };
          if (aligned) {
            scalar(0, head);
            scalar(body_end, len);
          } else {
            scalar(0, len);
          }
          const V* sv = reinterpret_cast<const V*>(src + head);
          V* dv = reinterpret_cast<V*>(dst + head);
          constexpr int kB = 4;  // vectors in flight per thread
          for (uint64_t v0 = 0; v0 < nv; v0 += kB * kThreads) {
            V x[kB];
#pragma unroll
            for (int q = 0; q < kB; ++q) {
              const uint64_t v = v0 + q * kThreads + threadIdx.x;
              if (v < nv) x[q] = sv[v];
            }
#pragma unroll
            for (int q = 0; q < kB; ++q) {
              const uint64_t v = v0 + q * kThreads + threadIdx.x;
              if (v >= nv) continue;
              V y = x[q];
#pragma unroll
              for (int w = 0; w < static_cast<int>(W); ++w) lane(y, w) = scale_of(lane(y, w), A.inv, A.mean);
              if (SGD) {
                const V p = dv[v];
#pragma unroll
                for (int w = 0; w < static_cast<int>(W); ++w) lane(y, w) = sgd(lane(p, w), A.lr, lane(y, w));
              }
              dv[v] = y;
            }
          }
          ++j;
        } else if (!SGD && A.zfill) {  // zero fill; tiles are 16-byte aligned, segments need not be
          T* dst = A.out + pos;
          const uint64_t len = end - pos;
          const uint64_t mis = (reinterpret_cast<uintptr_t>(dst) / sizeof(T)) % W;
          const uint64_t head = (len < (W - mis) % W ? len : (W - mis) % W);
          const uint64_t nv = (len - head) / W;
          for (uint64_t i = threadIdx.x; i < head; i += kThreads) dst[i] = T(0);
          for (uint64_t i = head + nv * W + threadIdx.x; i < len; i += kThreads) dst[i] = T(0);
          V z;
#pragma unroll
          for (int w = 0; w < static_cast<int>(W); ++w) lane(z, w) = T(0);
          V* dv = reinterpret_cast<V*>(dst + head);
          for (uint64_t v = threadIdx.x; v < nv; v += kThreads) dv[v] = z;
        }
        pos = end;
      }
      continue;
    }
    const int s = static_cast<int>(qc % NS);
    T* st = stage + (qc & 1) * TE;
#ifdef COVAP_K2_TRACE
    unsigned long long tw0, tw1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw0));
    ++tr_full;
#endif
    if (threadIdx.x == 0) bulk_wait_read<1>();
    mbar_wait(&bar[s], static_cast<uint32_t>((qc / NS) & 1));
    __syncthreads();
#ifdef COVAP_K2_TRACE
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw1));
    tr_wait += tw1 - tw0;
#endif
    const V* xv = reinterpret_cast<const V*>(in + s * kSlotTiles * TE);
    const V* pv = reinterpret_cast<const V*>(in + (s * kSlotTiles + 1) * TE);
    V* sv = reinterpret_cast<V*>(st);
    for (uint32_t v = threadIdx.x; v < n / W; v += kThreads) {
      V x = xv[v];
#pragma unroll
      for (int q = 0; q < static_cast<int>(W); ++q) lane(x, q) = scale_of(lane(x, q), A.inv, A.mean);
      if (SGD) {
        const V p = pv[v];
#pragma unroll
        for (int q = 0; q < static_cast<int>(W); ++q) lane(x, q) = sgd(lane(p, q), A.lr, lane(x, q));
      }
      sv[v] = x;
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(A.out + e0, st, n * sizeof(T));
      bulk_commit();
      produce_one();  // input slot s is consumed
    }
    ++qc;
  }
  if (threadIdx.x == 0) {
    bulk_commit();
    bulk_wait_all();
#ifdef COVAP_K2_TRACE
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x < 1024) {
      unsigned long long* o = g_k2_trace + blockIdx.x * 6;
      o[0] = tr_t0; o[1] = t1; o[2] = tr_full; o[3] = tr_none; o[4] = tr_mixed; o[5] = tr_wait;
    }
#endif
  }
}

// ------------------------------------------------------------ K2, selected slots only
//
// After a zero-filling K1 the unpack is a scaled gather of the allreduced
// send buffer back into the layout: out[begin_j + i] = (0 + recv[dst_j + i])
// * inv over the phase's runs.  It is tiled over the SEND space [o_lo, o_hi)
// — the packed selected shards, contiguous up to the < 32-element alignment
// gaps between runs — so every CTA streams the same number of bytes however
// the selected shards are scattered over the layout (tiling the layout
// instead left CTAs idle on unselected tiles: 0.45 of peak at BERT-large
// K=4).  A tile is bulk-loaded into a kStagesK2-slot ring, scaled into a
// staging tile and bulk-stored piece by piece (one piece per run it meets:
// dst == begin (mod kSendAlign), so a piece is 16-byte aligned in both
// spaces); scalar heads/tails only where a run or the [a, b) clip is not.

template <typename T>
struct SelArgs {
  const T* recv;
  T* out;
  const Run* runs;
  int nruns;
  uint64_t o_lo, o_hi;  // send-space range of the launch (o_lo 16-byte aligned)
  uint64_t a, b;        // layout clip (one bucket, or the whole arena)
  uint64_t te;          // elements per tile (balanced)
  T inv;
  int mean;
};

// Run holding send offset o, or the first run after it (runs ascend in dst).
__device__ __forceinline__ int run_by_dst(const Run* __restrict__ runs, int n, uint64_t o) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (runs[mid].dst + (runs[mid].end - runs[mid].begin) > o)
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 1) unpack_sel_kernel(const SelArgs<T> A) {
  constexpr uint32_t TE = kTileK2 / sizeof(T);
  constexpr uint64_t W = 16 / sizeof(T);
  using V = typename Vec16<T>::type;
  extern __shared__ __align__(128) unsigned char smem[];
  T* in = reinterpret_cast<T*>(smem);  // kStagesK2 tiles
  T* stage = in + kStagesK2 * TE;      // 2 staging tiles
  __shared__ __align__(8) uint64_t bar[kStagesK2];

  pdl_launch_dependents();
  const uint64_t te = A.te;
  const uint64_t ntiles = (A.o_hi - A.o_lo + te - 1) / te;
  const uint64_t my = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStagesK2; ++i) mbar_init(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  __syncthreads();
  pdl_wait();  // the allreduce (or K1) wrote recv

  auto tile_lo = [&](uint64_t k) { return A.o_lo + (blockIdx.x + k * gridDim.x) * te; };
  auto issue = [&](uint64_t k) {  // thread 0
    const int s = static_cast<int>(k % kStagesK2);
    const uint64_t o0 = tile_lo(k), o1 = min(o0 + te, A.o_hi);
    // whole 16-byte vectors only (a last tile ending mid-vector reads its
    // few tail elements from global memory below)
    const uint32_t bytes = static_cast<uint32_t>((o1 - o0) / W * W * sizeof(T));
    mbar_arrive_tx(&bar[s], bytes);
    if (bytes) bulk_load(in + s * TE, A.recv + o0, bytes, &bar[s]);
  };
  if (threadIdx.x == 0)
    for (uint64_t k = 0; k < my && k < kStagesK2; ++k) issue(k);

  for (uint64_t k = 0; k < my; ++k) {
    const int s = static_cast<int>(k % kStagesK2);
    const uint64_t o0 = tile_lo(k), o1 = min(o0 + te, A.o_hi);
    const uint32_t nv = static_cast<uint32_t>((o1 - o0) / W);
    T* st = stage + (k & 1) * TE;
    if (threadIdx.x == 0) bulk_wait_read<1>();  // staging tile (k & 1) free again
    mbar_wait(&bar[s], static_cast<uint32_t>((k / kStagesK2) & 1));
    __syncthreads();
    const V* xv = reinterpret_cast<const V*>(in + s * TE);
    V* sv = reinterpret_cast<V*>(st);
    for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
      V x = xv[v];
#pragma unroll
      for (int q = 0; q < static_cast<int>(W); ++q) lane(x, q) = scale_of(lane(x, q), A.inv, A.mean);
      sv[v] = x;
    }
    for (uint64_t i = nv * W + threadIdx.x; i < o1 - o0; i += kThreads)
      st[i] = scale_of(A.recv[o0 + i], A.inv, A.mean);
    fence_async_smem();
    __syncthreads();
    // the pieces of this tile: one per run it meets, clipped to [a, b)
    const int j0 = run_by_dst(A.runs, A.nruns, o0);
    for (int j = j0; j < A.nruns; ++j) {
      const Run R = A.runs[j];
      const uint64_t d1 = R.dst + (R.end - R.begin);
      if (R.dst >= o1) break;
      uint64_t ps = R.dst > o0 ? R.dst : o0, pe = d1 < o1 ? d1 : o1;  // send space
      // clip to the layout range [a, b)
      const uint64_t e_s = R.begin + (ps - R.dst);
      if (e_s < A.a) ps += A.a - e_s;
      if (R.begin + (pe - R.dst) > A.b) pe -= R.begin + (pe - R.dst) - A.b;
      if (ps >= pe) continue;
      const uint64_t e = R.begin + (ps - R.dst), n = pe - ps;
      // e == ps (mod W) for the planner's runs: head up to the next vector
      // boundary, bulk body, tail (a caller-built misaligned run: all scalar)
      const bool aligned = (R.dst - R.begin) % W == 0;
      const uint64_t head = !aligned ? n : (((W - e % W) % W) < n ? (W - e % W) % W : n);
      const uint64_t body = (n - head) / W * W;
      for (uint64_t i = threadIdx.x; i < head; i += kThreads) A.out[e + i] = st[ps - o0 + i];
      for (uint64_t i = head + body + threadIdx.x; i < n; i += kThreads)
        A.out[e + i] = st[ps - o0 + i];
      if (threadIdx.x == 0 && body)
        bulk_store(A.out + e + head, st + (ps - o0 + head), static_cast<uint32_t>(body * sizeof(T)));
    }
    if (threadIdx.x == 0) {
      bulk_commit();
      if (k + kStagesK2 < my) issue(k + kStagesK2);  // input slot s is consumed
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ---------------------------------------------------------------- mean of rows
// allreduce_mean for P in-process workers (trainer.cpp:41-45): out[i] =
// ((0 + x_0[i]) + x_1[i] + ... + x_{P-1}[i]) * inv, in worker order.
template <typename T>
__global__ void __launch_bounds__(kThreads)
    mean_rows_kernel(const T* __restrict__ rows, T* __restrict__ out, uint64_t P, uint64_t n, T inv) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    T acc = T(0);
    for (uint64_t w = 0; w < P; ++w) acc = add_rn(acc, rows[w * n + i]);
    out[i] = mul_rn(acc, inv);
  }
}

// ---------------------------------------------------------------- K0

__device__ __forceinline__ uint64_t splitmix_out(uint64_t z) {  // rng.hpp:17-20
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <typename T>
__device__ __forceinline__ T gen_value(uint64_t key, uint64_t i, int kind) {
  const uint64_t x = splitmix_out(key + (i + 1) * 0x9e3779b97f4a7c15ULL);
  if (kind == 0) {
    const int32_t s = static_cast<int32_t>((x & 0xffff) + ((x >> 16) & 0xffff) +
                                           ((x >> 32) & 0xffff) + (x >> 48)) -
                      131070;
    return mul_rn(static_cast<T>(s), static_cast<T>(1.0 / 32768.0));
  }
  return static_cast<T>(static_cast<int64_t>(x % 2001) - 1000);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    generate_kernel(T* __restrict__ out, uint64_t n, uint64_t key, int kind, uint64_t begin) {
  constexpr int W = 16 / sizeof(T);
  const uint64_t nvec = n / W;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec;
       v += stride) {
    T o[W];
#pragma unroll
    for (int k = 0; k < W; ++k) o[k] = gen_value<T>(key, begin + v * W + k, kind);
    if (W == 4)
      reinterpret_cast<float4*>(out)[v] = *reinterpret_cast<float4*>(o);
    else
      reinterpret_cast<double2*>(out)[v] = *reinterpret_cast<double2*>(o);
  }
  if (blockIdx.x == 0)
    for (uint64_t e = nvec * W + threadIdx.x; e < n; e += blockDim.x)
      out[e] = gen_value<T>(key, begin + e, kind);
}

// ---------------------------------------------------------------- K3

__global__ void spin_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// ---------------------------------------------------------------- launch

struct DeviceShape {
  int sms = 0;
  bool ready = false;
};

template <typename K>
cudaError_t opt_in(K kernel, uint32_t smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem));
}

// One-time per-device setup: SM count and the >48 KB dynamic-smem opt-in of
// every instantiation.
cudaError_t shape(DeviceShape** out) {
  static std::mutex mu;
  static DeviceShape shapes[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  DeviceShape& s = shapes[dev & 63];
  if (!s.ready) {
    if ((e = cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev))) return e;
    if ((e = opt_in(filter_kernel<float, 0>, kSmemK1)) || (e = opt_in(filter_kernel<float, 1>, kSmemK1)) ||
        (e = opt_in(filter_kernel<float, 3>, kSmemK1Sgd)) ||
        (e = opt_in(filter_kernel<double, 0>, kSmemK1)) ||
        (e = opt_in(filter_kernel<double, 1>, kSmemK1)) ||
        (e = opt_in(filter_kernel<double, 3>, kSmemK1Sgd)) ||
        (e = opt_in(filter_kernel<float, 5>, kSmemK1Fp16)) ||
        (e = opt_in(filter_kernel<double, 5>, kSmemK1Fp16)) ||
        (e = opt_in(filter_kernel<float, 6>, kSmemK1Rk)) ||
        (e = opt_in(filter_kernel<double, 6>, kSmemK1Rk)) ||
        (e = opt_in(unpack_kernel<float, false>, kSmemK2)) ||
        (e = opt_in(unpack_kernel<float, true>, kSmemK2Sgd)) ||
        (e = opt_in(unpack_kernel<double, false>, kSmemK2)) ||
        (e = opt_in(unpack_kernel<double, true>, kSmemK2Sgd)) ||
        (e = opt_in(unpack_sel_kernel<float>, kSmemK2Sel)) ||
        (e = opt_in(unpack_sel_kernel<double>, kSmemK2Sel)))
      return e;
    s.ready = true;
  }
  *out = &s;
  return cudaSuccess;
}

// Persistent grid: one CTA per SM (the smem footprint allows one), fewer
// when the range has fewer tiles than SMs.  The tile is then shrunk (in
// 16-byte vectors, never above the smem tile) so that the vector range splits
// into grid x m tiles: every CTA streams the same number of equal tiles and
// no CTA is left with one extra tile at the end (a ~3% tail at ResNet-50 size).
// Small ranges: at least min_tiles tiles (down to kMinTileBytes each), so a
// few-MB pass still spreads over every SM instead of giving a handful of
// CTAs one full-size tile each.
constexpr uint64_t kMinTileBytes = 4096;
// free_sms: SMs a pass leaves idle — the random-k pass, for the selection
// chain running beside it on a side stream; K1 / K2 of the overlapped
// multi-rank schedules (set_free_sms, this thread's launches), for the
// collective's kernels running beside them.
thread_local int t_free_sms = 0;
inline int grid_sms(int sms, int free_sms) {
  const int f = free_sms > t_free_sms ? free_sms : t_free_sms;
  return sms > f ? sms - f : 1;
}
template <typename T>
unsigned balance(uint64_t a, uint64_t b, int sms, uint32_t tile_bytes, uint64_t* te,
                 uint64_t min_tiles = 0) {
  constexpr uint64_t W = 16 / sizeof(T);
  const uint64_t a16 = (a + W - 1) / W * W, b16 = b / W * W;
  const uint64_t nvec = b16 > a16 ? (b16 - a16) / W : 0;
  const uint64_t max_vec = tile_bytes / 16;
  uint64_t tiles = std::max<uint64_t>(1, (nvec + max_vec - 1) / max_vec);
  if (tiles < min_tiles)
    tiles = std::max(tiles, std::min(min_tiles, nvec / (kMinTileBytes / 16)));
  const uint64_t grid = std::max<uint64_t>(1, std::min<uint64_t>(sms, tiles));
  const uint64_t m = (tiles + grid - 1) / grid;  // tiles per CTA
  const uint64_t vec = std::max<uint64_t>(1, (nvec + grid * m - 1) / (grid * m));
  *te = std::min(vec, max_vec) * W;
  return static_cast<unsigned>(grid);
}

template <typename T>
Args<T> make_args(const void* g, void* r, void* send, void* out, const void* recv,
                  const Run* runs, int nruns, uint64_t a, uint64_t b, double coeff, int ef,
                  double inv, int mean, double lr) {
  Args<T> A;
  A.g = static_cast<const T*>(g);
  A.r = static_cast<T*>(r);
  A.send = static_cast<T*>(send);
  A.out = static_cast<T*>(out);
  A.recv = static_cast<const T*>(recv);
  A.runs = runs;
  A.nruns = nruns;
  A.a = a;
  A.b = b;
  A.coeff = static_cast<T>(coeff);
  A.ef = ef;
  A.inv = static_cast<T>(inv);
  A.mean = mean;
  A.lr = static_cast<T>(lr);
  A.te = 0;  // set by balance()
  A.zfill = 1;
  A.wire = nullptr;
  A.sat = nullptr;
  A.bits = nullptr;
  A.toff = nullptr;
  A.list_idx = nullptr;
  A.list_val = nullptr;
  A.keep = 0;
  return A;
}

// Launch with the programmatic-stream-serialization attribute (PDL) so the
// kernel may start while the previous kernel in the stream drains.
template <typename T>
cudaError_t launch(void (*kernel)(const Args<T>), unsigned grid, unsigned smem, cudaStream_t s,
                   const Args<T>& args, unsigned threads = kThreads) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = COVAP_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// One of the streaming passes over [a, b): filter ops 0/1/3, unpack (2) or
// unpack + SGD (4), fp32 or fp64.
template <typename T>
cudaError_t pass(int op, const Args<T>& A, cudaStream_t s, int free_sms = 0) {
  if (A.b <= A.a) return cudaSuccess;
  DeviceShape* sh;
  cudaError_t e = shape(&sh);
  if (e) return e;
  const bool k1 = op == 0 || op == 1 || op == 3 || op == 5 || op == 6;
  Args<T> B = A;
  const uint64_t min_tiles = static_cast<uint64_t>(sh->sms) * (k1 ? COVAP_K1_MIN_WAVES : COVAP_K2_MIN_WAVES);
  const unsigned grid = balance<T>(A.a, A.b, grid_sms(sh->sms, free_sms),
                                   k1 ? kTileK1 : kTileK2, &B.te, min_tiles);
  if (op == 5) B.te = (B.te + 7) / 8 * 8;  // wire tiles: 16-byte multiples of halves
  switch (op) {
    case 5: return launch(filter_kernel<T, 5>, grid, kSmemK1Fp16, s, B, filter_threads<5>());
    case 6: return launch(filter_kernel<T, 6>, grid, kSmemK1Rk, s, B, filter_threads<6>());
    case 0: return launch(filter_kernel<T, 0>, grid, kSmemK1, s, B, filter_threads<0>());
    case 1: return launch(filter_kernel<T, 1>, grid, kSmemK1, s, B, filter_threads<1>());
    case 3: return launch(filter_kernel<T, 3>, grid, kSmemK1Sgd, s, B, filter_threads<3>());
    case 2: return launch(unpack_kernel<T, false>, grid, kSmemK2, s, B);
    default: return launch(unpack_kernel<T, true>, grid, kSmemK2Sgd, s, B);
  }
}

template <typename... X>
cudaError_t pass_dt(int dtype, int op, cudaStream_t s, X... x) {
  if (dtype == 0) return pass<float>(op, make_args<float>(x...), s);
  return pass<double>(op, make_args<double>(x...), s);
}

}  // namespace

cudaError_t launch_filter_pack(int dtype, const void* g, void* r, void* send, const Run* runs,
                               int nruns, uint64_t a, uint64_t b, double coeff, int ef,
                               cudaStream_t s, void* out) {
  return pass_dt(dtype, 0, s, g, r, send, out, nullptr, runs, nruns, a, b, coeff, ef, 1.0, 1, 0.0);
}

cudaError_t launch_filter_unpack(int dtype, const void* g, void* r, void* out, const Run* runs,
                                 int nruns, uint64_t a, uint64_t b, double coeff, int ef,
                                 double inv, cudaStream_t s) {
  return pass_dt(dtype, 1, s, g, r, nullptr, out, nullptr, runs, nruns, a, b, coeff, ef, inv, 1, 0.0);
}

cudaError_t launch_filter_sgd(int dtype, const void* g, void* r, void* params, const Run* runs,
                              int nruns, uint64_t a, uint64_t b, double coeff, int ef, double inv,
                              double lr, cudaStream_t s) {
  return pass_dt(dtype, 3, s, g, r, nullptr, params, nullptr, runs, nruns, a, b, coeff, ef, inv, 1,
                 lr);
}

cudaError_t launch_unpack(int dtype, const void* recv, void* out, const Run* runs, int nruns,
                          uint64_t a, uint64_t b, double inv, int mean, cudaStream_t s, int zfill,
                          const Run* host_runs) {
  if (!zfill) {
    // Only the selected slots: the send-space range of the runs that meet
    // [a, b) (host copy of the run table); nothing to launch if none does.
    if (nruns == 0 || b <= a) return cudaSuccess;  // nothing selected (an empty phase)
    if (host_runs == nullptr) return cudaErrorInvalidValue;
    uint64_t lo = UINT64_MAX, hi = 0;
    for (int j = 0; j < nruns; ++j) {
      const Run& R = host_runs[j];
      const uint64_t x0 = std::max(a, R.begin), x1 = std::min(b, R.end);
      if (x0 >= x1) continue;
      lo = std::min(lo, R.dst + (x0 - R.begin));
      hi = std::max(hi, R.dst + (x1 - R.begin));
    }
    if (hi <= lo) return cudaSuccess;
    DeviceShape* sh;
    cudaError_t e = shape(&sh);
    if (e) return e;
    auto go = [&](auto tag) {
      using T = decltype(tag);
      constexpr uint64_t W = 16 / sizeof(T);
      SelArgs<T> A;
      A.recv = static_cast<const T*>(recv);
      A.out = static_cast<T*>(out);
      A.runs = runs;
      A.nruns = nruns;
      A.o_lo = lo / W * W;  // the send buffer's runs start 16-byte aligned; keep tiles so
      A.o_hi = hi;
      A.a = a;
      A.b = b;
      A.inv = static_cast<T>(inv);
      A.mean = mean;
      const unsigned grid = balance<T>(A.o_lo, (A.o_hi + W - 1) / W * W, grid_sms(sh->sms, 0),
                                       kTileK2, &A.te,
                                       static_cast<uint64_t>(sh->sms) * COVAP_K2_MIN_WAVES);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kThreads);
      cfg.dynamicSmemBytes = kSmemK2Sel;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = COVAP_PDL ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const cudaError_t err = cudaLaunchKernelEx(&cfg, unpack_sel_kernel<T>, A);
      return err != cudaSuccess ? err : cudaGetLastError();
    };
    return dtype == 0 ? go(float(0)) : go(double(0));
  }
  auto go = [&](auto tag) {
    using T = decltype(tag);
    Args<T> A = make_args<T>(nullptr, nullptr, nullptr, out, recv, runs, nruns, a, b, 0.0, 0, inv,
                             mean, 0.0);
    A.zfill = zfill;
    return pass<T>(2, A, s);
  };
  return dtype == 0 ? go(float(0)) : go(double(0));
}

cudaError_t launch_unpack_sgd(int dtype, const void* recv, void* params, const Run* runs,
                              int nruns, uint64_t a, uint64_t b, double inv, int mean, double lr,
                              cudaStream_t s) {
  return pass_dt(dtype, 4, s, nullptr, nullptr, nullptr, params, recv, runs, nruns, a, b, 0.0, 0,
                 inv, mean, lr);
}

cudaError_t launch_filter_fp16(int dtype, const void* g, void* r, void* kept, int kept_mean,
                              uint16_t* wire, unsigned long long* sat, uint64_t n, double coeff,
                              int ef, cudaStream_t s) {
  auto go = [&](auto tag) {
    using T = decltype(tag);
    Args<T> A = make_args<T>(g, r, nullptr, kept, nullptr, nullptr, 0, 0, n, coeff, ef, 1.0,
                             kept_mean, 0.0);
    A.wire = wire;
    A.sat = sat;
    return pass<T>(5, A, s);
  };
  return dtype == 0 ? go(float(0)) : go(double(0));
}

cudaError_t filter_tiles(int dtype, uint64_t n, uint64_t* te, uint64_t* ntiles, int free_sms) {
  DeviceShape* sh;
  const cudaError_t e = shape(&sh);
  if (e) return e;
  const uint64_t W = dtype == 0 ? 4 : 2, b16 = n / W * W;
  uint64_t t = 0;
  if (dtype == 0)
    balance<float>(0, n, grid_sms(sh->sms, free_sms), kTileK1, &t,
                   static_cast<uint64_t>(sh->sms) * COVAP_K1_MIN_WAVES);
  else
    balance<double>(0, n, grid_sms(sh->sms, free_sms), kTileK1, &t,
                    static_cast<uint64_t>(sh->sms) * COVAP_K1_MIN_WAVES);
  *te = t;
  *ntiles = b16 == 0 ? 0 : (b16 + t - 1) / t;
  return cudaSuccess;
}

cudaError_t launch_filter_randomk(int dtype, const void* g, void* r, void* out, int keep,
                                  int kept_mean, const uint32_t* bits, const uint32_t* toff,
                                  uint32_t* list_idx, void* list_val, uint64_t n, double coeff,
                                  int ef, cudaStream_t s, int free_sms) {
  auto go = [&](auto tag) {
    using T = decltype(tag);
    Args<T> A = make_args<T>(g, r, nullptr, out, nullptr, nullptr, 0, 0, n, coeff, ef, 1.0,
                             kept_mean, 0.0);
    A.bits = bits;
    A.toff = toff;
    A.list_idx = list_idx;
    A.list_val = static_cast<T*>(list_val);
    A.keep = keep;
    return pass<T>(6, A, s, free_sms);
  };
  return dtype == 0 ? go(float(0)) : go(double(0));
}

int set_free_sms(int n) {
  const int prev = t_free_sms;
  t_free_sms = n > 0 ? n : 0;
  return prev;
}

cudaError_t launch_mean_rows(int dtype, const void* rows, void* out, uint64_t P, uint64_t n,
                             cudaStream_t s, double inv_override) {
  if (n == 0) return cudaSuccess;
  DeviceShape* sh;
  cudaError_t e = shape(&sh);
  if (e) return e;
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(
      1, std::min<uint64_t>(static_cast<uint64_t>(sh->sms) * 8, (n + kThreads - 1) / kThreads)));
  // inv_override: the scale of an already-summed single row (an NCCL sum of
  // P ranks is one row here, but still scales by 1/P)
  const double inv = inv_override > 0.0 ? inv_override : 1.0 / static_cast<double>(P);
  if (dtype == 0)
    mean_rows_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(rows),
                                                      static_cast<float*>(out), P, n,
                                                      static_cast<float>(inv));
  else
    mean_rows_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<const double*>(rows),
                                                       static_cast<double*>(out), P, n, inv);
  return cudaGetLastError();
}

cudaError_t launch_generate(int dtype, void* out, uint64_t n, uint64_t key, int kind,
                            uint64_t begin, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  DeviceShape* sh;
  cudaError_t e = shape(&sh);
  if (e) return e;
  const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(
      1, std::min<uint64_t>(static_cast<uint64_t>(sh->sms) * 8, (n / 4 + kThreads - 1) / kThreads)));
  if (dtype == 0)
    generate_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<float*>(out), n, key, kind, begin);
  else
    generate_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<double*>(out), n, key, kind, begin);
  return cudaGetLastError();
}

cudaError_t launch_spin(double us, int blocks, cudaStream_t s) {
  if (us <= 0) return cudaSuccess;
  spin_kernel<<<std::max(blocks, 1), 32, 0, s>>>(static_cast<uint64_t>(us * 1000.0));
  return cudaGetLastError();
}

// K3 (full-GPU form): a backward pass's kernels own the SMs while they run —
// one 1024-thread CTA per SM holding kBusySmem of shared memory, so no CTA of
// the filter / unpack kernels (172 / 229 KB) fits beside it; only small-
// footprint kernels (NCCL's) can co-reside.  The emulated backward of `us`
// is a sequence of such kernels of `slice_us` each, and side-stream work
// runs in the gaps between them, as it does between real backward kernels.
constexpr int kBusySmem = 160 * 1024;
__global__ void __launch_bounds__(1024) busy_kernel(uint64_t ns) {
  extern __shared__ unsigned char busy_smem[];
  if (threadIdx.x == 0) busy_smem[0] = 0;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

cudaError_t launch_busy(double us, double slice_us, cudaStream_t s) {
  if (us <= 0) return cudaSuccess;
  DeviceShape* sh;
  cudaError_t e = shape(&sh);
  if (e) return e;
  static bool attr = false;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(busy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kBusySmem)))
      return e;
    attr = true;
  }
  if (slice_us <= 0) slice_us = us;
  const int n = std::max(1, static_cast<int>(us / slice_us + 0.5));
  const uint64_t ns = static_cast<uint64_t>(us * 1000.0 / n);
  for (int i = 0; i < n; ++i) {
    busy_kernel<<<sh->sms, 1024, kBusySmem, s>>>(ns);
    if ((e = cudaGetLastError())) return e;
  }
  return cudaSuccess;
}

// Per-worker stream key: mix_seed(seed, 0x100 + rank) (trainer.cpp:126), then
// mixed with the step (rng.hpp:60-63 pattern).  Host side; same as oracle.
static uint64_t host_splitmix_out(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t host_mix_seed(uint64_t seed, uint64_t tag) {
  return host_splitmix_out((seed ^ (0x632be59bd9b4e019ULL + tag * 0x9e3779b97f4a7c15ULL)) +
                           0x9e3779b97f4a7c15ULL);
}
uint64_t stream_key(uint64_t seed, uint64_t rank, uint64_t step) {
  return host_mix_seed(host_mix_seed(seed, 0x100 + rank), step);
}

#ifdef COVAP_K2_TRACE
extern "C" int covap_debug_k2_trace(unsigned long long* host, int nblocks) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_k2_trace, sizeof(unsigned long long) * 6 *
                                                                     static_cast<size_t>(nblocks)));
}
#endif
}  // namespace covapb
