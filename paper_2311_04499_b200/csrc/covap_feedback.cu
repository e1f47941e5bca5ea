// covap_feedback.cu — sm_100a kernels for the baseline compressors under the
// generic error-feedback wrapper.
//
//   dense      identity / covap / fp16 filter in one pass: c = g + coeff*r,
//              kept = f(c), r = c - kept, fp16 wire bits    (compress.cpp:323-344)
//   compensate sparsifier pass 1: r = c, out = 0, per-tensor histogram of |c|
//   topk_*     exact top-k per tensor: threshold bin from the histogram, one
//              collect pass over c, radix select among the threshold-bin
//              candidates by (|c| desc, index asc)         (compress.cpp:119-133)
//   randomk_*  sample_without_replacement (compress.cpp:145-155) in parallel:
//              draws are counter-based splitmix64 outputs; the partial
//              Fisher-Yates swap chain is resolved with per-position lists
//   *_mean     the mean of the kept gradients over P ranks, in rank order
//              (trainer.cpp:35-47, 402): fp16 wire widened and summed; sparse
//              lists scattered into an accumulator
//
// Arithmetic follows the reference operation by operation with FMA
// contraction disabled (__fmul_rn / __fadd_rn / __fsub_rn), so the fp64
// instantiation is bit-exact against the reference and the fp32 one against
// the same sequence in single precision (the tests' fp32 restatement).
#include <cuda_fp16.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "covap_feedback.h"
#include "covap_half.cuh"

namespace covapb {
namespace fb {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;

// Programmatic dependent launch along the top-k chain (compensate ->
// threshold -> collect -> threshold -> filter2 -> final): each kernel waits
// for its predecessor's memory before touching global data and lets the next
// be scheduled once its own work is issued (letting it in at the start made
// the waiting CTAs crowd out the running ones: the step got 16 % slower), so
// the chain's launch latencies overlap.  No-ops without the attribute.
// Used only for small layouts (TopkArgs::pdl): ResNet-50 top-k 0.148 -> 0.140
// ms, but BERT-large 1.479 -> 1.525 ms, where the launches are already hidden.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_release() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
struct KeyOf;
// key: the |x| bit pattern (order == magnitude order); bits / value: the
// whole pattern with the sign, as the candidate lists store it so the later
// passes need not gather x again.
template <>
struct KeyOf<float> {
  using K = uint32_t;
  static constexpr int kBits = 31;
  static constexpr K kMask = 0x7fffffffu;
  static __device__ __forceinline__ K key(float x) { return __float_as_uint(x) & kMask; }
  static __device__ __forceinline__ K bits(float x) { return __float_as_uint(x); }
  static __device__ __forceinline__ float value(K b) { return __uint_as_float(b); }
};
template <>
struct KeyOf<double> {
  using K = uint64_t;
  static constexpr int kBits = 63;
  static constexpr K kMask = 0x7fffffffffffffffull;
  static __device__ __forceinline__ K key(double x) {
    return static_cast<uint64_t>(__double_as_longlong(x)) & kMask;
  }
  static __device__ __forceinline__ K bits(double x) {
    return static_cast<uint64_t>(__double_as_longlong(x));
  }
  static __device__ __forceinline__ double value(K b) {
    return __longlong_as_double(static_cast<long long>(b));
  }
};

template <typename T>
__device__ __forceinline__ uint32_t bin_of(T c) {
  return static_cast<uint32_t>(KeyOf<T>::key(c) >> (KeyOf<T>::kBits - kBinBits));
}

__device__ __forceinline__ uint64_t splitmix_out(uint64_t z) {  // rng.hpp:17-20
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t mix_seed(uint64_t seed, uint64_t tag) {  // rng.hpp:58-63
  return splitmix_out((seed ^ (0x632be59bd9b4e019ULL + tag * 0x9e3779b97f4a7c15ULL)) +
                      0x9e3779b97f4a7c15ULL);
}

// Warp-aggregated append: returns this lane's slot (valid when pred).
__device__ __forceinline__ uint32_t append_slot(bool pred, uint32_t* counter) {
  const unsigned mask = __ballot_sync(0xffffffffu, pred);
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (mask) {
    const int leader = __ffs(mask) - 1;
    if (lane == leader) base = atomicAdd(counter, static_cast<uint32_t>(__popc(mask)));
    base = __shfl_sync(0xffffffffu, base, leader);
  }
  return base + static_cast<uint32_t>(__popc(mask & ((1u << lane) - 1u)));
}

// The kept value as written to `kept`: itself, or — when kept is one rank's
// synchronised output — allreduce_mean's (0.0 + x) * (1/1) (trainer.cpp:41-45),
// which only turns -0 into +0.
template <typename T>
__device__ __forceinline__ T kept_value(T c, int mean) {
  return mean ? add_rn(T(0), c) : c;
}

template <typename T>
__device__ __forceinline__ T compensate(T g, T r, T coeff, int ef) {
  return ef ? add_rn(g, mul_rn(coeff, r)) : g;  // compress.cpp:332-336
}

// ---------------------------------------------------------------- dense

template <typename T, int KIND>
__global__ void __launch_bounds__(kThreads) dense_kernel(DenseArgs A) {
  const T* __restrict__ g = static_cast<const T*>(A.g);
  T* __restrict__ r = static_cast<T*>(A.r);
  T* __restrict__ kept = static_cast<T*>(A.kept);
  const T coeff = static_cast<T>(A.coeff);
  unsigned long long nsat = 0;
  for (uint32_t ci = blockIdx.x; ci < A.nchunks; ci += gridDim.x) {
    const Chunk ch = A.chunks[ci];
    bool sel = true;
    if (KIND == kCovap) {  // select_tensors (compress.cpp:13-28)
      const uint64_t phase = A.step % A.interval, rem = ch.tensor % A.interval;
      sel = A.rule ? ((rem + phase) % A.interval == 0) : (rem == phase);
    }
    // kept = f(c), residual = compensated - kept (compress.cpp:339-341)
    auto one = [&](T c, T& k, T& res, uint16_t& h) {
      if (KIND == kFp16) {
        bool s = false;
        h = half_bits(static_cast<float>(c), s);
        nsat += s ? 1 : 0;
        k = static_cast<T>(half_to_float(h));
      } else if (KIND == kCovap) {
        k = sel ? c : T(0);
      } else {
        k = c;
      }
      res = sub_rn(c, k);
    };
    if (ch.pad == 0) {
      // 16-byte-aligned body chunk: kVec vectors per thread in flight
      using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
      constexpr int W = 16 / static_cast<int>(sizeof(T));
      constexpr int kVec = 4;
      const uint32_t v1 = static_cast<uint32_t>(ch.end / W);
      const V* g4 = reinterpret_cast<const V*>(g);
      V* r4 = reinterpret_cast<V*>(r);
      V* k4 = reinterpret_cast<V*>(kept);
      for (uint32_t vb = static_cast<uint32_t>(ch.begin / W) + threadIdx.x; vb < v1;
           vb += kThreads * kVec) {
        V gv[kVec], rv[kVec];
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
          const uint32_t v = vb + u * kThreads;
          if (v < v1) {
            gv[u] = g4[v];
            rv[u] = A.ef ? r4[v] : V{};
          }
        }
#pragma unroll
        for (int u = 0; u < kVec; ++u) {
          const uint32_t v = vb + u * kThreads;
          if (v >= v1) continue;
          V kv, nr;
          uint16_t hv[W];
          const T* gs = reinterpret_cast<const T*>(&gv[u]);
          const T* rs = reinterpret_cast<const T*>(&rv[u]);
          T* ks = reinterpret_cast<T*>(&kv);
          T* ns = reinterpret_cast<T*>(&nr);
#pragma unroll
          for (int w = 0; w < W; ++w) one(compensate(gs[w], rs[w], coeff, A.ef), ks[w], ns[w], hv[w]);
          if (kept) {
#pragma unroll
            for (int w = 0; w < W; ++w) ks[w] = kept_value(ks[w], A.kept_mean);
            k4[v] = kv;
          }
          if (r) r4[v] = nr;
          if (KIND == kFp16 && A.wire) {
            if (W == 4)
              reinterpret_cast<uint2*>(A.wire)[v] =
                  make_uint2(hv[0] | (uint32_t(hv[1]) << 16), hv[2 % W] | (uint32_t(hv[3 % W]) << 16));
            else
              reinterpret_cast<uint32_t*>(A.wire)[v] = hv[0] | (uint32_t(hv[1 % W]) << 16);
          }
        }
      }
      continue;
    }
    for (uint64_t base = ch.begin; base < ch.end; base += kThreads) {
      const uint64_t i = base + threadIdx.x;
      if (i >= ch.end) continue;
      T k, res;
      uint16_t h = 0;
      one(compensate(g[i], A.ef ? r[i] : T(0), coeff, A.ef), k, res, h);
      if (kept) kept[i] = kept_value(k, A.kept_mean);
      if (r) r[i] = res;
      if (KIND == kFp16 && A.wire) A.wire[i] = h;
    }
  }
  if (KIND == kFp16 && A.sat) {
    for (int o = 16; o > 0; o >>= 1) nsat += __shfl_xor_sync(0xffffffffu, nsat, o);
    if ((threadIdx.x & 31) == 0 && nsat) atomicAdd(A.sat, nsat);
  }
}

// ---------------------------------------------------------- compensate

constexpr int kCompVec = 4;
#ifndef COVAP_COMP_PARTS  // compensation pass: work units per chunk
#define COVAP_COMP_PARTS 8
#endif
constexpr uint32_t kCompParts = COVAP_COMP_PARTS;

template <typename T, bool HIST>
__global__ void __launch_bounds__(kThreads)
    compensate_kernel(const T* __restrict__ g, T* __restrict__ r, T* __restrict__ zero,
                      uint32_t* __restrict__ ghist, const Chunk* __restrict__ chunks,
                      uint32_t nchunks, int ef, T coeff, int vec) {
  pdl_begin();
  __shared__ uint32_t hist[HIST ? kBins : 1];
  uint32_t cur = kNone;
  if (HIST) {
    for (int b = threadIdx.x; b < kBins; b += kThreads) hist[b] = 0;
    __syncthreads();
  }
  auto flush = [&]() {
    __syncthreads();
    uint32_t* dst = ghist + static_cast<uint64_t>(cur) * kBins;
    for (int b = threadIdx.x; b < kBins; b += kThreads) {
      const uint32_t v = hist[b];
      if (v) {
        atomicAdd(dst + b, v);
        hist[b] = 0;
      }
    }
    __syncthreads();
  };
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int W = 16 / static_cast<int>(sizeof(T));
  // Work units of kChunk / kCompParts elements, round-robin over the CTAs:
  // finer than chunks so the last wave leaves fewer SMs idle.
  constexpr uint32_t kParts = kCompParts;
  constexpr uint64_t kPlen = kChunk / kParts;
  for (uint32_t u = blockIdx.x; u < nchunks * kParts; u += gridDim.x) {
    Chunk ch = chunks[u / kParts];
    const uint64_t ub = ch.begin + (u % kParts) * kPlen;
    if (ub >= ch.end) continue;
    ch.begin = ub;
    ch.end = ch.end < ub + kPlen ? ch.end : ub + kPlen;
    if (HIST && ch.tensor != cur) {
      if (cur != kNone) flush();
      cur = ch.tensor;
    }
    if (vec && ch.pad == 0) {
      // body chunk (16-byte aligned ends): kCompVec vectors of g and r in
      // flight per thread.  Measured faster below 2^26 elements (ResNet-50
      // top-k 0.1215 -> 0.1159 ms), slower above (VGG-16 0.622 -> 0.630,
      // BERT-large 1.372 -> 1.412 ms, where the scalar loop already streams
      // at ~0.98 of the copy peak), profiles/r2_f4.md.
      const uint64_t vb = ch.begin / W, ve = ch.end / W;
      for (uint64_t base = vb; base < ve; base += kThreads * kCompVec) {
        V gv[kCompVec], rv[kCompVec];
#pragma unroll
        for (int q = 0; q < kCompVec; ++q) {
          const uint64_t i = base + q * kThreads + threadIdx.x;
          if (i < ve) {
            gv[q] = reinterpret_cast<const V*>(g)[i];
            rv[q] = ef ? reinterpret_cast<const V*>(r)[i] : V{};
          }
        }
#pragma unroll
        for (int q = 0; q < kCompVec; ++q) {
          const uint64_t i = base + q * kThreads + threadIdx.x;
          if (i >= ve) continue;
          V cv;
          const T* gs = reinterpret_cast<const T*>(&gv[q]);
          const T* rs = reinterpret_cast<const T*>(&rv[q]);
          T* cs = reinterpret_cast<T*>(&cv);
#pragma unroll
          for (int w = 0; w < W; ++w) {
            cs[w] = compensate(gs[w], rs[w], coeff, ef);
            if (HIST) atomicAdd(&hist[bin_of(cs[w])], 1u);
          }
          reinterpret_cast<V*>(r)[i] = cv;
          if (zero) reinterpret_cast<V*>(zero)[i] = V{};
        }
      }
      continue;
    }
    for (uint64_t base = ch.begin; base < ch.end; base += kThreads * kUnroll) {
      T gv[kUnroll], rv[kUnroll];
#pragma unroll
      for (int q = 0; q < kUnroll; ++q) {
        const uint64_t i = base + q * kThreads + threadIdx.x;
        if (i < ch.end) {
          gv[q] = g[i];
          rv[q] = ef ? r[i] : T(0);
        }
      }
#pragma unroll
      for (int q = 0; q < kUnroll; ++q) {
        const uint64_t i = base + q * kThreads + threadIdx.x;
        if (i >= ch.end) continue;
        const T c = compensate(gv[q], rv[q], coeff, ef);
        r[i] = c;
        if (zero) zero[i] = T(0);
        if (HIST) atomicAdd(&hist[bin_of(c)], 1u);
      }
    }
  }
  if (HIST && cur != kNone) flush();
  pdl_release();
}

// --------------------------------------------------------------- top-k

// Exact per-tensor top-k by (|c| desc, index asc) in three levels:
//   1. compensate: histogram of the top kBinBits of |c|; threshold: the bin
//      b1 holding the k-th largest and need1, the count still to take from it
//   2. collect: |c| above b1 -> list; in b1 -> candidates + histogram of the
//      next kDigitBits; threshold: digit d2 and need2; filter2: candidates
//      above d2 -> list, at d2 -> second-level candidates
//   3. final: exact radix select among the second-level candidates over (the
//      remaining key bits, ~index) — a handful of elements on real gradients.
// Appends reserve list slots once per CTA per tile (block scan + one atomic).

template <typename T>
constexpr int kShift2 = KeyOf<T>::kBits - kBinBits - kDigitBits;  // level-2 digit position

template <typename T>
__device__ __forceinline__ uint32_t digit2_of(typename KeyOf<T>::K key) {
  return static_cast<uint32_t>(key >> kShift2<T>) & (kDigits - 1);
}

// Block-wide: the bin where the count of elements in bins >= it first
// reaches need (thread j owns BINS/kThreads bins, highest first).  The
// crossing thread writes *s_bin / *s_need; ends with a barrier.
template <int BINS>
__device__ __forceinline__ void crossing(const uint32_t* h, uint32_t need, uint32_t* s_bin,
                                         uint32_t* s_need) {
  using Scan = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int kPer = BINS / kThreads;
  const int hi = BINS - kPer * threadIdx.x;
  uint32_t mine = 0;
  for (int b = hi - 1; b >= hi - kPer; --b) mine += h[b];
  uint32_t above = 0;
  Scan(tmp).ExclusiveSum(mine, above);
  if (above < need && need <= above + mine) {
    uint32_t acc = above;
    for (int b = hi - 1; b >= hi - kPer; --b) {
      if (acc + h[b] >= need) {
        *s_bin = static_cast<uint32_t>(b);
        *s_need = need - acc;
        break;
      }
      acc += h[b];
    }
  }
  __syncthreads();
}

// One CTA per tensor (levels 1 and 2): bin / need from the tensor's
// histogram, which is cleared for the next step; resets two counters.
template <int BINS>
__global__ void __launch_bounds__(kThreads)
    topk_threshold_kernel(uint32_t* hist, const uint32_t* need_in, uint32_t* bin_out,
                          uint32_t* need_out, uint32_t* reset0, uint32_t* reset1) {
  pdl_begin();
  __shared__ uint32_t s_bin, s_need;
  const uint32_t t = blockIdx.x;
  uint32_t* h = hist + static_cast<uint64_t>(t) * BINS;
  crossing<BINS>(h, need_in[t], &s_bin, &s_need);
  if (threadIdx.x == 0) {
    bin_out[t] = s_bin;
    need_out[t] = s_need;
    if (reset0) reset0[t] = 0;
    if (reset1) reset1[t] = 0;
  }
  for (int b = threadIdx.x; b < BINS; b += kThreads) h[b] = 0;
  pdl_release();
}

constexpr int kWarps = kThreads / 32;
#ifndef COVAP_COLLECT_CTAS  // collect CTAs per SM
#define COVAP_COLLECT_CTAS 4
#endif

// collect.  Per warp iteration (4 16-byte vectors per lane) a vector is a
// hit when its largest key reaches the candidate bin (one compare per
// vector: hits are ~1 % of elements); the warp then compacts its hit vectors into
// a per-warp shared FIFO (one warp scan per iteration) and handles them 32 at
// a time, one vector per lane: the per-hit work (classification, residual /
// kept stores, list appends, the level-2 histogram) runs lane-parallel with
// one list reservation per batch, instead of once per hit for the whole warp
// (round 2: a per-lane shared-memory ring claimed hit by hit, ResNet-50 45 ->
// 30 us, profiles/r2_f4.md).  Each CTA walks one contiguous run of chunks, so
// the FIFO and the level-2 histogram are flushed only where the tensor
// changes (round-robin chunks, or groups of 4 / 16, measured slower).
// 32-bit flat indices (the state checks N < 2^32); body chunks are 16-byte
// aligned (covap_feedback_create cuts every tensor's unaligned head and tail
// into chunks of their own, flagged scalar).
#ifndef COVAP_COLLECT_PARTS  // collect: work units per chunk
#define COVAP_COLLECT_PARTS 4
#endif
constexpr uint32_t kCollectParts = COVAP_COLLECT_PARTS;
constexpr uint32_t kFifo = 160;  // hit vectors per warp: 31 pending + 4 x 32 new fit

template <typename T>
__global__ void __launch_bounds__(kThreads, COVAP_COLLECT_CTAS) topk_collect_kernel(TopkArgs A) {
  pdl_begin();
  using K = typename KeyOf<T>::K;
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int W = 16 / static_cast<int>(sizeof(T));
  constexpr int kV = 4;  // vectors per lane per iteration
  __shared__ uint32_t hist2[kDigits];
  __shared__ V s_v[kWarps][kFifo];
  __shared__ uint32_t s_e[kWarps][kFifo];
  T* __restrict__ r = static_cast<T*>(A.r);
  T* __restrict__ kept = static_cast<T*>(A.kept);
  T* __restrict__ list_val = static_cast<T*>(A.list_val);
  K* __restrict__ cand_key = static_cast<K*>(A.cand_key);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  V* const fv = s_v[warp];
  uint32_t* const fe = s_e[warp];
  for (int b = threadIdx.x; b < kDigits; b += kThreads) hist2[b] = 0;
  __syncthreads();
  // the current tensor's parameters: bin > b1 taken (key >= k_take), bin ==
  // b1 candidate (key >= k_cand); list / candidate offsets
  uint32_t t = kNone;
  K k_cand = 0, k_take = 0;
  uint64_t lo = 0, cb = 0;
  // Lane-parallel hit handling: this lane's nw elements x[0..nw) at flat
  // indices e0 + w (nw = 0: idle lane); one reservation per list per call.
  auto handle = [&](const T* x, uint32_t e0, int nw) {
    uint32_t nt = 0, nc = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      if (w < nw) {
        const K key = KeyOf<T>::key(x[w]);
        nt += key >= k_take;
        nc += key >= k_cand && key < k_take;
      }
    }
    uint32_t pre = nt | (nc << 16);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
    pre -= nt | (nc << 16);  // exclusive
    uint32_t bt = 0, bc = 0;
    if (lane == 0) {
      if (tot & 0xffffu) bt = atomicAdd(A.sel_cnt + t, tot & 0xffffu);
      if (tot >> 16) bc = atomicAdd(A.cand_cnt + t, tot >> 16);
    }
    uint32_t st = __shfl_sync(0xffffffffu, bt, 0) + (pre & 0xffffu);
    uint32_t sc = __shfl_sync(0xffffffffu, bc, 0) + (pre >> 16);
#pragma unroll
    for (int w = 0; w < W; ++w) {
      if (w < nw) {
        const K key = KeyOf<T>::key(x[w]);
        const uint32_t i = e0 + w;
        if (key >= k_take) {
          if (kept) kept[i] = kept_value(x[w], A.kept_mean);
          r[i] = sub_rn(x[w], x[w]);
          A.list_idx[lo + st] = i;
          list_val[lo + st] = x[w];
          ++st;
        } else if (key >= k_cand) {
          A.cand_idx[cb + sc] = i;
          cand_key[cb + sc] = KeyOf<T>::bits(x[w]);  // with the sign: the value itself
          atomicAdd(&hist2[digit2_of<T>(key)], 1u);
          ++sc;
        }
      }
    }
  };
  uint32_t head = 0, pend = 0;  // FIFO [head, head + pend) mod kFifo, warp-uniform
  auto pop32 = [&](uint32_t m) {  // handle min(m, 32) queued vectors
    uint32_t q = head + lane;
    if (q >= kFifo) q -= kFifo;
    const bool act = static_cast<uint32_t>(lane) < m;
    const V v = act ? fv[q] : V{};
    const uint32_t e0 = act ? fe[q] : 0u;
    handle(reinterpret_cast<const T*>(&v), e0, act ? W : 0);
    const uint32_t n = m < 32 ? m : 32;
    head += n;
    if (head >= kFifo) head -= kFifo;
    pend -= n;
    __syncwarp();
  };
  auto end_tensor = [&]() {  // the FIFO's last entries, then the histogram
    if (pend) pop32(pend);
    __syncthreads();
    uint32_t* dst = A.hist2 + static_cast<uint64_t>(t) * kDigits;
    for (int b = threadIdx.x; b < kDigits; b += kThreads) {
      const uint32_t v = hist2[b];
      if (v) {
        atomicAdd(dst + b, v);
        hist2[b] = 0;
      }
    }
    __syncthreads();
  };
  // one contiguous run of work units (a chunk / kCollectParts each) per CTA
  constexpr uint32_t kParts = kCollectParts;
  constexpr uint64_t kPlen = kChunk / kParts;
  const uint32_t nu = A.nchunks * kParts;
  const uint32_t per = (nu + gridDim.x - 1) / gridDim.x;
  const uint32_t u_lo = min(nu, blockIdx.x * per), u_hi = min(nu, u_lo + per);
  constexpr uint32_t kSpan = 32 * kV * W;  // elements per warp iteration
  for (uint32_t u = u_lo; u < u_hi; ++u) {
    Chunk ch = A.chunks[u / kParts];
    const uint64_t ub = ch.begin + (u % kParts) * kPlen;
    if (ub >= ch.end) continue;
    ch.begin = ub;
    ch.end = ch.end < ub + kPlen ? ch.end : ub + kPlen;
    if (ch.tensor != t) {
      if (t != kNone) end_tensor();
      t = ch.tensor;
      const uint32_t b1 = A.thr[t];
      k_cand = static_cast<K>(b1) << (KeyOf<T>::kBits - kBinBits);
      k_take = static_cast<K>(b1 + 1) << (KeyOf<T>::kBits - kBinBits);
      lo = A.list_off[t];
      cb = A.t_begin[t];
    }
    const uint32_t cbeg = static_cast<uint32_t>(ch.begin), cend = static_cast<uint32_t>(ch.end);
    if (ch.pad == 0) {
      for (uint32_t base = cbeg + warp * kSpan; base < cend; base += kWarps * kSpan) {
        V x[kV];
#pragma unroll
        for (int j = 0; j < kV; ++j) {
          const uint32_t e0 = base + (j * 32 + lane) * W;
          x[j] = e0 < cend ? *reinterpret_cast<const V*>(r + e0) : V{};
        }
        uint32_t vm = 0;  // this lane's hit vectors
#pragma unroll
        for (int j = 0; j < kV; ++j) {
          const T* xs = reinterpret_cast<const T*>(&x[j]);
          K m = KeyOf<T>::key(xs[0]);
#pragma unroll
          for (int w = 1; w < W; ++w) m = max(m, KeyOf<T>::key(xs[w]));
          if (m >= k_cand && base + (j * 32 + lane) * W < cend) vm |= 1u << j;
        }
        const uint32_t cnt = __popc(vm);
        uint32_t pre = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, pre, o);
          if (lane >= o) pre += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, pre, 31);
        if (tot == 0) continue;
        uint32_t q = head + pend + pre - cnt;  // pend <= 31, tot <= 128: q < 2 kFifo
#pragma unroll
        for (int j = 0; j < kV; ++j) {
          if (vm >> j & 1u) {
            const uint32_t sl = q >= kFifo ? q - kFifo : q;
            fv[sl] = x[j];
            fe[sl] = base + (j * 32 + lane) * W;
            ++q;
          }
        }
        pend += tot;
        __syncwarp();
        while (pend >= 32) pop32(32);
      }
    } else {  // scalar chunk: one element per lane
      for (uint32_t base = cbeg + warp * 32; base < cend; base += kWarps * 32) {
        const uint32_t e = base + lane;
        T c = T(0);
        if (e < cend) c = r[e];
        handle(&c, e, e < cend ? 1 : 0);
      }
    }
  }
  // every CTA takes part in the barriers of end_tensor (chunk runs are per
  // CTA, so all its warps see the same tensors)
  if (t != kNone) end_tensor();
  pdl_release();
}

// Level-1 candidates above d2 are taken, those at d2 go on to the final
// selection.  The candidates of all tensors form one flat index space (the
// CTA scans cand_cnt into shared memory), so the work is balanced however
// unevenly the candidates fall and no tensor waits for another.  The pass is
// latency-bound (the candidate lists carry each value's bit pattern, so the
// pass reads no r; the appends and the scattered residual / kept stores remain), so every
// lane keeps kF2 candidates in flight and the grid fills the SMs.  Appends are
// warp-aggregated per tensor (one atomic per tensor present in the warp).
#ifndef COVAP_F2_INFLIGHT
#define COVAP_F2_INFLIGHT 4
#endif
constexpr int kF2 = COVAP_F2_INFLIGHT;

template <typename T>
__global__ void __launch_bounds__(kThreads) topk_filter2_kernel(TopkArgs A) {
  pdl_begin();
  using K = typename KeyOf<T>::K;
  using Scan = cub::BlockScan<uint32_t, kThreads>;
  extern __shared__ uint32_t s_pre[];  // ntensors + 1 (kTopkMaxTensors bounds it)
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t s_carry;
  T* __restrict__ r = static_cast<T*>(A.r);
  T* __restrict__ kept = static_cast<T*>(A.kept);
  T* __restrict__ list_val = static_cast<T*>(A.list_val);
  const K* __restrict__ ck = static_cast<const K*>(A.cand_key);
  K* __restrict__ ck2 = static_cast<K*>(A.cand2_key);
  const uint32_t nt = A.ntensors;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t b0 = 0; b0 < nt; b0 += kThreads) {  // exclusive prefix of cand_cnt
    const uint32_t t = b0 + threadIdx.x;
    const uint32_t v = t < nt ? A.cand_cnt[t] : 0u;
    uint32_t ex = 0, tot = 0;
    Scan(tmp).ExclusiveSum(v, ex, tot);
    if (t < nt) s_pre[t] = s_carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) s_pre[nt] = s_carry;
  __syncthreads();
  const uint32_t total = s_pre[nt];
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5), nw = gridDim.x * kWarps;
  for (uint32_t base = gw * 32 * kF2; base < total; base += nw * 32 * kF2) {
    uint32_t tq[kF2], iq[kF2];
    K kq[kF2];
    bool vq[kF2];
#pragma unroll
    for (int q = 0; q < kF2; ++q) {  // issue every lane's key / index loads first
      const uint32_t e = base + q * 32 + lane;
      vq[q] = e < total;
      uint32_t lo = 0, hi = nt;  // tensor t with s_pre[t] <= e < s_pre[t + 1]
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_pre[mid] <= e) lo = mid; else hi = mid;
      }
      tq[q] = lo;
      const uint64_t at = A.t_begin[lo] + (e - s_pre[lo]);
      kq[q] = vq[q] ? ck[at] : K(0);  // the candidate's whole bit pattern
      iq[q] = vq[q] ? A.cand_idx[at] : 0u;
    }
    T cq[kF2];
    bool tk[kF2], nx[kF2];
#pragma unroll
    for (int q = 0; q < kF2; ++q) {  // then the gathers of the taken values
      const uint32_t d = digit2_of<T>(kq[q] & KeyOf<T>::kMask), d2 = vq[q] ? A.thr2[tq[q]] : 0u;
      tk[q] = vq[q] && d > d2;
      nx[q] = vq[q] && d == d2;
      cq[q] = tk[q] ? KeyOf<T>::value(kq[q]) : T(0);  // no gather of r
    }
#pragma unroll
    for (int q = 0; q < kF2; ++q) {
      if (tk[q]) {
        if (kept) kept[iq[q]] = kept_value(cq[q], A.kept_mean);
        r[iq[q]] = sub_rn(cq[q], cq[q]);
      }
      // warp-aggregated appends, one round per tensor present in this slot
      unsigned pending = __ballot_sync(0xffffffffu, tk[q] || nx[q]);
      while (pending) {
        const uint32_t t = __shfl_sync(0xffffffffu, tq[q], __ffs(pending) - 1);
        const bool mine = tq[q] == t;
        const unsigned mt = __ballot_sync(0xffffffffu, mine && tk[q]);
        const unsigned mn = __ballot_sync(0xffffffffu, mine && nx[q]);
        pending &= ~(mt | mn);
        uint32_t bt = 0, bn = 0;
        if (lane == 0) {
          if (mt) bt = atomicAdd(A.sel_cnt + t, static_cast<uint32_t>(__popc(mt)));
          if (mn) bn = atomicAdd(A.cand2_cnt + t, static_cast<uint32_t>(__popc(mn)));
        }
        bt = __shfl_sync(0xffffffffu, bt, 0);
        bn = __shfl_sync(0xffffffffu, bn, 0);
        if (mine && tk[q]) {
          const uint64_t at = A.list_off[t] + bt + __popc(mt & lt);
          A.list_idx[at] = iq[q];
          list_val[at] = cq[q];
        }
        if (mine && nx[q]) {
          const uint64_t at = A.t_begin[t] + bn + __popc(mn & lt);
          A.cand2_idx[at] = iq[q];
          ck2[at] = kq[q];
        }
      }
    }
  }
  pdl_release();
}

// One CTA per tensor: the need2 best second-level candidates by composite
// (remaining key bits desc, index asc) — an exact radix select over
// (key low bits, ~index), then their emission.
template <typename T>
__global__ void __launch_bounds__(kThreads) topk_final_kernel(TopkArgs A) {
  pdl_begin();
  using K = typename KeyOf<T>::K;
  constexpr int kLow = kShift2<T>;  // key bits below the level-2 digit
  __shared__ uint32_t hist[kDigits];
  __shared__ uint32_t s_digit, s_need, s_count;
  T* __restrict__ r = static_cast<T*>(A.r);
  T* __restrict__ kept = static_cast<T*>(A.kept);
  T* __restrict__ list_val = static_cast<T*>(A.list_val);
  uint32_t* __restrict__ list_idx = A.list_idx;
  const uint32_t t = blockIdx.x;
  const uint32_t need0 = A.need2[t];
  uint32_t need = need0;
  const uint32_t m = A.cand2_cnt[t];
  if (need == 0) return;
  const uint64_t cb = A.t_begin[t];
  const K* ck = static_cast<const K*>(A.cand2_key) + cb;
  const uint32_t* cx = A.cand2_idx + cb;
  const K lowmask = (K(1) << kLow) - 1;
  uint64_t pa = 0;  // fixed prefix of the low key bits
  uint32_t pb = 0;  // fixed prefix of ~index
  // Few survivors (the usual case on real gradients): rank each one against
  // the others by the composite (low key bits, ~index) in one pass instead
  // of the multi-pass radix select.  Composites are distinct (the index is).
  __shared__ uint64_t s_a[kThreads];
  __shared__ uint32_t s_b[kThreads];
  __shared__ uint8_t s_take[kThreads];
  const bool fast = need < m && m <= static_cast<uint32_t>(kThreads);
  if (fast) {
    const uint32_t e = threadIdx.x;
    uint64_t a = 0;
    uint32_t b = 0;
    if (e < m) {
      a = static_cast<uint64_t>(ck[e] & lowmask);
      b = ~cx[e];
      s_a[e] = a;
      s_b[e] = b;
    }
    __syncthreads();
    if (e < m) {
      uint32_t rank = 0;
      for (uint32_t f = 0; f < m; ++f)
        rank += (s_a[f] > a || (s_a[f] == a && s_b[f] > b)) ? 1u : 0u;
      s_take[e] = rank < need ? 1 : 0;
    }
    __syncthreads();
  } else if (need < m) {
    // field 0: the low key bits, field 1: ~index (32 bits)
    for (int field = 0; field < 2; ++field) {
      int left = field == 0 ? kLow : 32;
      while (left > 0) {
        const int nb = left < kDigitBits ? left : kDigitBits;
        const int shift = left - nb;
        for (int b = threadIdx.x; b < kDigits; b += kThreads) hist[b] = 0;
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < m; e += kThreads) {
          const uint64_t a = static_cast<uint64_t>(ck[e] & lowmask);
          const uint32_t b = ~cx[e];
          uint32_t digit;
          bool match;
          if (field == 0) {
            match = (a >> left) == pa;
            digit = static_cast<uint32_t>(a >> shift) & ((1u << nb) - 1u);
          } else {
            match = a == pa && (left == 32 ? true : (b >> left) == pb);
            digit = (b >> shift) & ((1u << nb) - 1u);
          }
          if (match) atomicAdd(&hist[digit], 1u);
        }
        __syncthreads();
        crossing<kDigits>(hist, need, &s_digit, &s_need);
        const uint32_t d = s_digit;
        need = s_need;
        if (field == 0)
          pa = (pa << nb) | d;
        else
          pb = (nb == 32 ? 0u : (pb << nb)) | d;
        left = shift;
        __syncthreads();
      }
    }
  }
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  const uint64_t base = A.list_off[t] + A.sel_cnt[t];
  const bool all = need0 >= m;
  // warp-uniform trip count so append_slot's ballot sees every lane
  for (uint32_t e0 = 0; e0 < m; e0 += kThreads) {
    const uint32_t e = e0 + threadIdx.x;
    bool take = false;
    if (e < m) {
      const uint64_t a = static_cast<uint64_t>(ck[e] & lowmask);
      const uint32_t b = ~cx[e];
      take = all || (fast ? s_take[e] != 0 : (a > pa || (a == pa && b >= pb)));
    }
    const uint32_t slot = append_slot(take, &s_count);
    if (take) {
      const uint32_t i = cx[e];
      const T c = KeyOf<T>::value(ck[e]);  // the stored pattern is r[i]'s
      list_idx[base + slot] = i;
      list_val[base + slot] = c;
      if (kept) kept[i] = kept_value(c, A.kept_mean);
      r[i] = sub_rn(c, c);
    }
  }
  pdl_release();
}

// ------------------------------------------------------------- random-k

// RandomkFilter's per-tensor stream (compress.cpp:288) or, for the standalone
// randomk_compress, the caller's seed.
__device__ __forceinline__ uint64_t seed_of(const RandomkArgs& A, uint32_t t) {
  return A.raw_seed ? A.seed : mix_seed(A.seed, A.step * 0x10001ULL + t);
}

__device__ __forceinline__ uint32_t tensor_of_entry(const RandomkArgs& A, uint64_t e) {
  return A.tensor_of[e];
}

// Draw i of tensor t: j_i = i + next_below(d - i) assuming no rejection; a
// rejection (probability < n / 2^64 per draw) flags the tensor for the exact
// sequential replay below.
__global__ void randomk_draw_kernel(RandomkArgs A) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < A.total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = tensor_of_entry(A, e);
    const uint64_t i = e - A.list_off[t];
    const uint64_t n = A.t_numel[t] - i;
    const uint64_t seed = seed_of(A, t);
    const uint64_t x = splitmix_out(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
    // next_below's rejection bound (0 - n) % n (rng.hpp:29) is below n, so
    // only x < n can be rejected (probability n / 2^64)
    if (x < n && x < (0ULL - n) % n) A.reject[t] = 1;
    A.j[e] = static_cast<uint32_t>(i + x % n);
    A.key[e] = static_cast<uint32_t>(A.t_begin[t] + i + x % n);
  }
}

// Exact replay of next_below's rejection loop for flagged tensors (one thread
// per tensor; practically never taken).
__global__ void randomk_replay_kernel(RandomkArgs A) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= A.ntensors || !A.reject[t]) return;
  A.reject[t] = 0;
  const uint64_t d = A.t_numel[t], lo = A.list_off[t];
  const uint64_t k = A.list_off[t + 1] - lo;
  uint64_t state = seed_of(A, t);
  for (uint64_t i = 0; i < k; ++i) {
    const uint64_t n = d - i, threshold = (0ULL - n) % n;
    uint64_t x;
    do {
      state += 0x9e3779b97f4a7c15ULL;
      x = splitmix_out(state);
    } while (x < threshold);
    A.j[lo + i] = static_cast<uint32_t>(i + x % n);
    A.key[lo + i] = static_cast<uint32_t>(A.t_begin[t] + i + x % n);
  }
}

// Two ways to find, for every draw, the earlier draws with the same target
// (prv) and the last earlier draw that targeted its own position (src):
//   hash  (up to 2^20 draws): per-position linked lists whose heads live in
//         an open-addressed table of 2^tbits words (flat position + 1 : 32,
//         last draw + 1 : 32; 0 = empty), emptied again by the resolve pass.
//         ~2k words (4 MB at ResNet-50 size) stay in L2.
//   sort  (more draws, where the table would not stay in L2: BERT-large link
//         + chain 550 us): a radix sort of the draws by target, then one
//         coalesced pass over the runs of equal targets.
// Neither touches an N-sized array, so the selection that runs beside the
// compensation pass takes little of its DRAM bandwidth.
__device__ __forceinline__ uint32_t slot_of(uint32_t key, uint32_t tbits) {
  return static_cast<uint32_t>((static_cast<uint64_t>(key) * 0x9e3779b97f4a7c15ull) >> (64 - tbits));
}

__global__ void randomk_link_kernel(RandomkArgs A) {
  const uint32_t mask = (1u << A.tbits) - 1u;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < A.total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = tensor_of_entry(A, e);
    const uint32_t i = static_cast<uint32_t>(e - A.list_off[t]);
    const uint32_t key = static_cast<uint32_t>(A.t_begin[t] + A.j[e]) + 1u;
    const unsigned long long mine = (static_cast<unsigned long long>(key) << 32) | (i + 1u);
    uint32_t h = slot_of(key, A.tbits);
    uint32_t prev = kNone;
    for (;;) {
      const unsigned long long w = A.table[h];
      const uint32_t k = static_cast<uint32_t>(w >> 32);
      if (k != key && k != 0u) {
        h = (h + 1u) & mask;
        continue;
      }
      const unsigned long long got = atomicCAS(&A.table[h], w, mine);
      if (got == w) {
        prev = k == 0u ? kNone : static_cast<uint32_t>(w) - 1u;
        break;
      }
      // lost a race on this slot: look at it again
    }
    A.slot[e] = h;
    A.nxt[e] = prev;
  }
}

// last draw m < before whose target is position p (local), or kNone
__device__ __forceinline__ uint32_t last_before(const RandomkArgs& A, uint32_t t, uint32_t p,
                                                uint32_t before) {
  const uint64_t lo = A.list_off[t];
  const uint32_t key = static_cast<uint32_t>(A.t_begin[t] + p) + 1u;
  const uint32_t mask = (1u << A.tbits) - 1u;
  uint32_t h = slot_of(key, A.tbits);
  unsigned long long w;
  for (;;) {
    w = A.table[h];
    const uint32_t k = static_cast<uint32_t>(w >> 32);
    if (k == 0u) return kNone;
    if (k == key) break;
    h = (h + 1u) & mask;
  }
  uint32_t best = kNone;
  for (uint32_t m = static_cast<uint32_t>(w) - 1u; m != kNone; m = A.nxt[lo + m])
    if (m < before && (best == kNone || m > best)) best = m;
  return best;
}

__global__ void randomk_chain_hash_kernel(RandomkArgs A) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < A.total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = tensor_of_entry(A, e);
    const uint32_t i = static_cast<uint32_t>(e - A.list_off[t]);
    A.prv[e] = last_before(A, t, A.j[e], i);
    A.src[e] = last_before(A, t, i, i);
  }
}

// The draws sorted by flat target (stable, so draws in order within a
// target): the swap chains become neighbours.  prv[e] = the last earlier
// draw with the same target (the previous entry of its run); src[lo + p] =
// the last draw m < p whose target is position p itself (the last entry of
// p's run below p; only positions p < k are themselves draws).  src was
// filled with kNone before.  One coalesced pass instead of per-position
// linked lists: the k draws never touch an N-sized table, so the selection
// running beside the compensation pass costs it little DRAM bandwidth.
__global__ void randomk_chain_kernel(RandomkArgs A) {
  for (uint64_t s = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; s < A.total;
       s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t key = A.key_sorted[s], e = A.draw_sorted[s];
    const uint32_t t = tensor_of_entry(A, e);
    const uint64_t lo = A.list_off[t];
    const uint32_t m = static_cast<uint32_t>(e - lo);
    const bool run_prev = s > 0 && A.key_sorted[s - 1] == key;  // same target => same tensor
    A.prv[e] = run_prev ? static_cast<uint32_t>(A.draw_sorted[s - 1] - lo) : kNone;
    const uint64_t p = key - A.t_begin[t];
    if (p < A.list_off[t + 1] - lo && m < p) {
      const bool last = s + 1 == A.total || A.key_sorted[s + 1] != key ||
                        A.draw_sorted[s + 1] - lo >= p;
      if (last) A.src[lo + p] = m;
    }
  }
}

// Position i of the pool after the k swaps holds S_i = V(j_i, i), where
// V(p, i) is p unless an earlier draw m targeted p (then W(m)), and W(m), the
// content of position m when draw m starts, is m unless an earlier draw
// targeted position m (then W of that draw).  pos[i] = flat S_i.
__global__ void randomk_resolve_kernel(RandomkArgs A) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < A.total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = tensor_of_entry(A, e);
    const uint64_t lo = A.list_off[t];
    const uint32_t i = static_cast<uint32_t>(e - lo);
    const uint32_t j = A.j[e];
    uint32_t s;
    if (j == i || A.prv[e] != kNone) {
      uint32_t w = j == i ? i : A.prv[e];
      while (A.src[lo + w] != kNone) w = A.src[lo + w];
      s = w;
    } else {
      s = j;
    }
    A.pos[e] = static_cast<uint32_t>(A.t_begin[t] + s);
    if (A.bits) atomicOr(&A.bits[(A.t_begin[t] + s) / 32], 1u << ((A.t_begin[t] + s) % 32));
    if (A.tbits) A.table[A.slot[e]] = 0ull;  // the chain pass was the table's last reader
  }
}

// Empty the sample bitmap again: the words of the previous selection drawn
// into this buffer (its positions are still in pos).
__global__ void randomk_unmark_kernel(const uint32_t* __restrict__ pos, uint64_t total,
                                      uint32_t* __restrict__ bits) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    bits[pos[e] / 32] = 0u;
}

// Samples per filter tile (one warp per tile), for the list offsets of the
// fused pass — its tiles exactly: tile k < ntiles is [k te, min(k te + te,
// b16)), the 16-byte-vector part, and tile ntiles the scalar tail [b16, n)
// the pass handles element by element.
__global__ void randomk_tile_count_kernel(const uint32_t* __restrict__ bits, uint64_t te,
                                          uint64_t ntiles, uint64_t b16, uint64_t n,
                                          uint32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x / 32) + (threadIdx.x >> 5);
       k <= ntiles; k += nw) {
    const uint64_t e0 = k < ntiles ? k * te : b16, e1 = k < ntiles ? min(e0 + te, b16) : n;
    uint32_t c = 0;
    if (e1 > e0)
      for (uint64_t q = e0 / 32 + lane; q <= (e1 - 1) / 32; q += 32) {
        uint32_t w = bits[q];
        if (q * 32 < e0) w &= ~0u << (e0 - q * 32);
        if (q * 32 + 32 > e1) w &= (1u << (e1 - q * 32)) - 1u;
        c += __popc(w);
      }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[k] = c;
  }
}

// The data pass of the selection: kept[S] = c, r[S] = c - c, list = (S, c).
// Four draws in flight per thread (one dependent gather each).
template <typename T>
__global__ void randomk_gather_kernel(const uint32_t* __restrict__ pos, uint64_t total,
                                      T* __restrict__ r, T* __restrict__ kept, int kept_mean,
                                      uint32_t* __restrict__ list_idx, T* __restrict__ list_val) {
  constexpr int kQ = 4;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t e0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e0 < total;
       e0 += stride * kQ) {
    uint32_t f[kQ];
    T c[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const uint64_t e = e0 + q * stride;
      f[q] = e < total ? pos[e] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) c[q] = e0 + q * stride < total ? r[f[q]] : T(0);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
      const uint64_t e = e0 + q * stride;
      if (e >= total) continue;
      list_idx[e] = f[q];
      list_val[e] = c[q];
      if (kept) kept[f[q]] = kept_value(c[q], kept_mean);
      r[f[q]] = sub_rn(c[q], c[q]);
    }
  }
}


// ------------------------------------------------------------ exchange

__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(double* p, const double (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
}

template <typename T>
__global__ void fp16_mean_kernel(const uint16_t* __restrict__ recv, int P, uint64_t n, T inv,
                                 T* __restrict__ out) {
  // 8 halves (16 B) per thread per rank when the rows stay 16-byte aligned
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t tid = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nvec = (n % 8 == 0) ? n / 8 : 0;
  for (uint64_t v = tid; v < nvec; v += stride) {
    T acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = T(0);
    for (int p = 0; p < P; ++p) {
      const uint4 w = reinterpret_cast<const uint4*>(recv + static_cast<uint64_t>(p) * n)[v];
      const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint16_t h = static_cast<uint16_t>(u[q >> 1] >> (16 * (q & 1)));
        acc[q] = add_rn(acc[q], static_cast<T>(half_to_float(h)));
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = mul_rn(acc[q], inv);
    store8(out + v * 8, acc);
  }
  for (uint64_t i = nvec * 8 + tid; i < n; i += stride) {
    T a = T(0);
    for (int p = 0; p < P; ++p)
      a = add_rn(a, static_cast<T>(half_to_float(recv[static_cast<uint64_t>(p) * n + i])));
    out[i] = mul_rn(a, inv);
  }
}

template <typename T>
__global__ void list_mean_aligned_kernel(const uint32_t* __restrict__ idx,
                                         const T* __restrict__ vals, int P, uint64_t cnt, T inv,
                                         T* __restrict__ out) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    T acc = T(0);
    for (int p = 0; p < P; ++p) acc = add_rn(acc, vals[static_cast<uint64_t>(p) * cnt + e]);
    out[idx[e]] = mul_rn(acc, inv);
  }
}

template <typename T>
__global__ void list_accumulate_kernel(const uint32_t* __restrict__ idx, const T* __restrict__ val,
                                       uint64_t cnt, T* __restrict__ acc) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    acc[idx[e]] = add_rn(acc[idx[e]], val[e]);
}

template <typename T>
__global__ void list_finish_kernel(const uint32_t* __restrict__ idx, uint64_t cnt, T* acc, T inv,
                                   T* __restrict__ out, int clear) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (clear)
      acc[idx[e]] = T(0);
    else
      out[idx[e]] = mul_rn(acc[idx[e]], inv);
  }
}

__global__ void fp16_decode_kernel(const uint16_t* __restrict__ bits, uint64_t n,
                                   float* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = half_to_float(bits[i]);
}

// ------------------------------------------------------------- ordering

template <typename T>
__global__ void order_keys_kernel(const T* __restrict__ val, const uint64_t* __restrict__ p,
                                  uint64_t cnt, typename KeyOf<T>::K* __restrict__ key) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    key[e] = KeyOf<T>::key(val[p[e]]);
}

// out[e] = (idx_sorted[q[e]], val[p[q[e]]]), q = identity when NULL
template <typename T>
__global__ void order_emit_kernel(const uint32_t* __restrict__ idx_sorted,
                                  const uint64_t* __restrict__ p, const uint64_t* __restrict__ q,
                                  const T* __restrict__ val, uint64_t cnt,
                                  uint64_t* __restrict__ out_idx, T* __restrict__ out_val) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < cnt;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t f = q ? q[e] : e;
    out_idx[e] = idx_sorted[f];
    out_val[e] = val[p[f]];
  }
}

__global__ void iota_kernel(uint64_t* p, uint64_t n) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    p[e] = e;
}

// Reference output order (not on the sync path; the standalone compressors
// only): sort by index ascending, then for top-k stable-sort by |value|
// descending, which keeps equal magnitudes in index order (the tie rule of
// std::stable_sort in compress.cpp:123-126).  CUB radix sorts are stable.
template <typename T>
cudaError_t order_list_t(int kind, const uint32_t* idx, const T* val, uint64_t cnt,
                         uint64_t* out_idx, T* out_val, cudaStream_t s) {
  using K = typename KeyOf<T>::K;
  if (cnt == 0) return cudaSuccess;
  const uint64_t blocks = (cnt + kThreads - 1) / kThreads;
  const int grid = static_cast<int>(blocks < 1024 ? blocks : 1024);
  const int n = static_cast<int>(cnt);
  constexpr int kKeyBits = 8 * static_cast<int>(sizeof(K));
  uint32_t* i1 = nullptr;
  uint64_t *p0 = nullptr, *p1 = nullptr, *q0 = nullptr, *q1 = nullptr;
  K *k0 = nullptr, *k1 = nullptr;
  void* tmp = nullptr;
  size_t b1 = 0, b2 = 0;
  cudaError_t e = cudaSuccess;
  auto al = [&](void** ptr, size_t bytes) {
    if (e == cudaSuccess) e = cudaMallocAsync(ptr, bytes, s);
  };
  al(reinterpret_cast<void**>(&i1), cnt * 4);
  al(reinterpret_cast<void**>(&p0), cnt * 8);
  al(reinterpret_cast<void**>(&p1), cnt * 8);
  al(reinterpret_cast<void**>(&q0), cnt * 8);
  al(reinterpret_cast<void**>(&q1), cnt * 8);
  al(reinterpret_cast<void**>(&k0), cnt * sizeof(K));
  al(reinterpret_cast<void**>(&k1), cnt * sizeof(K));
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortPairs(nullptr, b1, idx, i1, p0, p1, n, 0, 32, s);
  if (e == cudaSuccess)
    e = cub::DeviceRadixSort::SortPairsDescending(nullptr, b2, k0, k1, q0, q1, n, 0, kKeyBits, s);
  al(&tmp, b1 > b2 ? b1 : b2);
  if (e == cudaSuccess) {
    iota_kernel<<<grid, kThreads, 0, s>>>(p0, cnt);
    e = cub::DeviceRadixSort::SortPairs(tmp, b1, idx, i1, p0, p1, n, 0, 32, s);
  }
  if (e == cudaSuccess && kind == kTopk) {
    order_keys_kernel<T><<<grid, kThreads, 0, s>>>(val, p1, cnt, k0);
    iota_kernel<<<grid, kThreads, 0, s>>>(q0, cnt);
    e = cub::DeviceRadixSort::SortPairsDescending(tmp, b2, k0, k1, q0, q1, n, 0, kKeyBits, s);
  }
  if (e == cudaSuccess)
    order_emit_kernel<T><<<grid, kThreads, 0, s>>>(i1, p1, kind == kTopk ? q1 : nullptr, val, cnt,
                                                   out_idx, out_val);
  for (void* ptr : {static_cast<void*>(i1), static_cast<void*>(p0), static_cast<void*>(p1),
                    static_cast<void*>(q0), static_cast<void*>(q1), static_cast<void*>(k0),
                    static_cast<void*>(k1), tmp})
    if (ptr) cudaFreeAsync(ptr, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e;
}

int grid_for(uint64_t work, int sms, int per_sm) {
  const uint64_t g = (work + kThreads - 1) / kThreads;
  const uint64_t cap = static_cast<uint64_t>(sms) * per_sm;
  return static_cast<int>(g < 1 ? 1 : (g < cap ? g : cap));
}

}  // namespace

// ------------------------------------------------------------ launchers

cudaError_t launch_dense(int dtype, int kind, const DenseArgs& a, int sms, cudaStream_t s) {
  const int grid = static_cast<int>(a.nchunks < static_cast<uint32_t>(sms * 4) ? a.nchunks : sms * 4);
  if (grid == 0) return cudaSuccess;
  if (dtype == 1) {
    switch (kind) {
      case kIdentity: dense_kernel<double, kIdentity><<<grid, kThreads, 0, s>>>(a); break;
      case kCovap: dense_kernel<double, kCovap><<<grid, kThreads, 0, s>>>(a); break;
      default: dense_kernel<double, kFp16><<<grid, kThreads, 0, s>>>(a); break;
    }
  } else {
    switch (kind) {
      case kIdentity: dense_kernel<float, kIdentity><<<grid, kThreads, 0, s>>>(a); break;
      case kCovap: dense_kernel<float, kCovap><<<grid, kThreads, 0, s>>>(a); break;
      default: dense_kernel<float, kFp16><<<grid, kThreads, 0, s>>>(a); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_compensate(int dtype, const void* g, void* r, void* zero, uint32_t* hist,
                              const Chunk* chunks, uint32_t nchunks, int ef, double coeff,
                              int sms, cudaStream_t s, bool pdl, bool vec) {
  const int grid = static_cast<int>(nchunks < static_cast<uint32_t>(sms * 4) ? nchunks : sms * 4);
  const int v = vec ? 1 : 0;
  if (grid == 0) return cudaSuccess;
  if (dtype == 1) {
    if (hist)
      return launch_pdl(pdl, compensate_kernel<double, true>, dim3(grid), dim3(kThreads), 0, s,
                        static_cast<const double*>(g), static_cast<double*>(r),
                        static_cast<double*>(zero), hist, chunks, nchunks, ef, coeff, v);
    else
      compensate_kernel<double, false><<<grid, kThreads, 0, s>>>(
          static_cast<const double*>(g), static_cast<double*>(r), static_cast<double*>(zero),
          hist, chunks, nchunks, ef, coeff, v);
  } else {
    const float c = static_cast<float>(coeff);
    if (hist)
      return launch_pdl(pdl, compensate_kernel<float, true>, dim3(grid), dim3(kThreads), 0, s,
                        static_cast<const float*>(g), static_cast<float*>(r),
                        static_cast<float*>(zero), hist, chunks, nchunks, ef, c, v);
    else
      compensate_kernel<float, false><<<grid, kThreads, 0, s>>>(
          static_cast<const float*>(g), static_cast<float*>(r), static_cast<float*>(zero), hist,
          chunks, nchunks, ef, c, v);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_topk_t(const TopkArgs& a, int sms, cudaStream_t s) {
  if (a.ntensors == 0) return cudaSuccess;
  const uint32_t cap = static_cast<uint32_t>(sms * COVAP_COLLECT_CTAS);
  const int grid = static_cast<int>(a.nchunks < cap ? a.nchunks : cap);
  cudaError_t e = launch_pdl(a.pdl != 0, topk_threshold_kernel<kBins>, dim3(a.ntensors), dim3(kThreads), 0, s,
                             a.hist1, a.k, a.thr, a.need, a.sel_cnt, a.cand_cnt);
  if (e == cudaSuccess && grid > 0)
    e = launch_pdl(a.pdl != 0, topk_collect_kernel<T>, dim3(grid), dim3(kThreads), 0, s, a);
  if (e == cudaSuccess)
    e = launch_pdl(a.pdl != 0, topk_threshold_kernel<kDigits>, dim3(a.ntensors), dim3(kThreads), 0, s, a.hist2,
                   a.need, a.thr2, a.need2, a.cand2_cnt, static_cast<uint32_t*>(nullptr));
  const uint32_t pre_bytes = (a.ntensors + 1) * 4;
  if (e == cudaSuccess && pre_bytes > 48 * 1024)
    e = cudaFuncSetAttribute(topk_filter2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(pre_bytes));
  if (e == cudaSuccess)
    e = launch_pdl(a.pdl != 0, topk_filter2_kernel<T>, dim3(sms * 4), dim3(kThreads), pre_bytes, s, a);
  if (e == cudaSuccess)
    e = launch_pdl(a.pdl != 0, topk_final_kernel<T>, dim3(a.ntensors), dim3(kThreads), 0, s, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_topk(int dtype, const TopkArgs& a, int sms, cudaStream_t s) {
  return dtype == 1 ? launch_topk_t<double>(a, sms, s) : launch_topk_t<float>(a, sms, s);
}

cudaError_t launch_randomk_select(const RandomkArgs& a, int sms, cudaStream_t s) {
  if (a.total == 0) return cudaSuccess;
  const int grid = grid_for(a.total, sms, 8);
  int bits = 1;  // key bits to sort: flat positions < 2^bits
  while (bits < 32 && (uint64_t(1) << bits) <= a.layout_n) ++bits;
  randomk_draw_kernel<<<grid, kThreads, 0, s>>>(a);
  randomk_replay_kernel<<<(a.ntensors + 63) / 64, 64, 0, s>>>(a);
  if (a.tbits) {
    randomk_link_kernel<<<grid, kThreads, 0, s>>>(a);
    randomk_chain_hash_kernel<<<grid, kThreads, 0, s>>>(a);
    randomk_resolve_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(a.src, 0xff, a.total * 4, s);  // kNone
  if (e == cudaSuccess) {
    size_t tmp = a.sort_tmp_bytes;
    e = cub::DeviceRadixSort::SortPairs(a.sort_tmp, tmp, a.key, a.key_sorted, a.draw_iota,
                                        a.draw_sorted, static_cast<int>(a.total), 0, bits, s);
  }
  if (e != cudaSuccess) return e;
  randomk_chain_kernel<<<grid, kThreads, 0, s>>>(a);
  randomk_resolve_kernel<<<grid, kThreads, 0, s>>>(a);
  return cudaGetLastError();
}

size_t randomk_sort_bytes(uint64_t total) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr),
                                  static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int>(total), 0, 32);
  return b;
}

cudaError_t launch_randomk_unmark(const uint32_t* pos, uint64_t total, uint32_t* bits, int sms,
                                  cudaStream_t s) {
  if (total == 0) return cudaSuccess;
  randomk_unmark_kernel<<<grid_for(total, sms, 8), kThreads, 0, s>>>(pos, total, bits);
  return cudaGetLastError();
}

cudaError_t launch_randomk_tile_offsets(const uint32_t* bits, uint64_t te, uint64_t ntiles,
                                        uint64_t b16, uint64_t n, uint32_t* cnt, uint32_t* toff,
                                        void* tmp, size_t tmp_bytes, int sms, cudaStream_t s) {
  const uint64_t warps = ntiles + 1;
  const int grid = static_cast<int>(std::min<uint64_t>((warps + kWarps - 1) / kWarps,
                                                       static_cast<uint64_t>(sms) * 8));
  randomk_tile_count_kernel<<<grid, kThreads, 0, s>>>(bits, te, ntiles, b16, n, cnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, toff, static_cast<int>(ntiles + 1), s);
}

size_t randomk_scan_bytes(uint64_t ntiles) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<const uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), static_cast<int>(ntiles + 1));
  return b;
}

cudaError_t launch_randomk_gather(int dtype, const uint32_t* pos, uint64_t total, void* r,
                                  void* kept, int kept_mean, uint32_t* list_idx, void* list_val,
                                  int sms, cudaStream_t s) {
  if (total == 0) return cudaSuccess;
  const int grid = grid_for((total + 3) / 4, sms, 8);
  if (dtype == 1)
    randomk_gather_kernel<double><<<grid, kThreads, 0, s>>>(
        pos, total, static_cast<double*>(r), static_cast<double*>(kept), kept_mean, list_idx,
        static_cast<double*>(list_val));
  else
    randomk_gather_kernel<float><<<grid, kThreads, 0, s>>>(
        pos, total, static_cast<float*>(r), static_cast<float*>(kept), kept_mean, list_idx,
        static_cast<float*>(list_val));
  return cudaGetLastError();
}

cudaError_t launch_fp16_mean(int dtype, const uint16_t* recv, int P, uint64_t n, double inv,
                             void* out, int sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = grid_for(n, sms, 8);
  if (dtype == 1)
    fp16_mean_kernel<double><<<grid, kThreads, 0, s>>>(recv, P, n, inv, static_cast<double*>(out));
  else
    fp16_mean_kernel<float><<<grid, kThreads, 0, s>>>(recv, P, n, static_cast<float>(inv),
                                                       static_cast<float*>(out));
  return cudaGetLastError();
}

cudaError_t launch_list_mean_aligned(int dtype, const uint32_t* idx, const void* vals, int P,
                                     uint64_t cnt, double inv, void* out, int sms,
                                     cudaStream_t s) {
  if (cnt == 0) return cudaSuccess;
  const int grid = grid_for(cnt, sms, 8);
  if (dtype == 1)
    list_mean_aligned_kernel<double><<<grid, kThreads, 0, s>>>(
        idx, static_cast<const double*>(vals), P, cnt, inv, static_cast<double*>(out));
  else
    list_mean_aligned_kernel<float><<<grid, kThreads, 0, s>>>(
        idx, static_cast<const float*>(vals), P, cnt, static_cast<float>(inv),
        static_cast<float*>(out));
  return cudaGetLastError();
}

cudaError_t launch_list_accumulate(int dtype, const uint32_t* idx, const void* val, uint64_t cnt,
                                   void* acc, int sms, cudaStream_t s) {
  if (cnt == 0) return cudaSuccess;
  const int grid = grid_for(cnt, sms, 8);
  if (dtype == 1)
    list_accumulate_kernel<double><<<grid, kThreads, 0, s>>>(
        idx, static_cast<const double*>(val), cnt, static_cast<double*>(acc));
  else
    list_accumulate_kernel<float><<<grid, kThreads, 0, s>>>(
        idx, static_cast<const float*>(val), cnt, static_cast<float*>(acc));
  return cudaGetLastError();
}

cudaError_t launch_list_finish(int dtype, const uint32_t* idx, uint64_t cnt, void* acc,
                               double inv, void* out, int clear, int sms, cudaStream_t s) {
  if (cnt == 0) return cudaSuccess;
  const int grid = grid_for(cnt, sms, 8);
  if (dtype == 1)
    list_finish_kernel<double><<<grid, kThreads, 0, s>>>(idx, cnt, static_cast<double*>(acc), inv,
                                                         static_cast<double*>(out), clear);
  else
    list_finish_kernel<float><<<grid, kThreads, 0, s>>>(idx, cnt, static_cast<float*>(acc),
                                                        static_cast<float>(inv),
                                                        static_cast<float*>(out), clear);
  return cudaGetLastError();
}

cudaError_t launch_fp16_decode(const uint16_t* bits, uint64_t n, float* out, int sms,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  fp16_decode_kernel<<<grid_for(n, sms, 8), kThreads, 0, s>>>(bits, n, out);
  return cudaGetLastError();
}

cudaError_t order_list(int dtype, int kind, const uint32_t* idx, const void* val, uint64_t cnt,
                       uint64_t* out_idx, void* out_val, cudaStream_t s) {
  if (dtype == 1)
    return order_list_t<double>(kind, idx, static_cast<const double*>(val), cnt, out_idx,
                                static_cast<double*>(out_val), s);
  return order_list_t<float>(kind, idx, static_cast<const float*>(val), cnt, out_idx,
                             static_cast<float*>(out_val), s);
}

}  // namespace fb
}  // namespace covapb
