// covap_peer.cu — C1 as a load/store collective over NVLink peer memory.
//
// The allreduce of the packed send buffers (trainer.cpp:41-43), written as
// one kernel per rank instead of an NCCL call:
//
//   phase 0  arrival: rank r publishes "step e is packed" into every peer's
//            flag block (st.release.sys over NVLink) and waits for all P;
//   phase 1  reduce-scatter: rank r owns slice r of the send buffer and sums
//            it over the P ranks IN RANK ORDER, ((0 + v_0) + v_1) + ... —
//            exactly allreduce_mean's order, so the result is bit-identical
//            to the reference for every P (NCCL's order is not) — writing the
//            sum over its own slice;
//   phase 2  all-gather: after a second flag exchange, rank r copies the
//            other ranks' reduced slices into its own buffer; K2 then unpacks
//            locally.
//
// Remote traffic per rank is 2(P-1)/P x 4S bytes, the ring/NCCL bus volume.
// Send buffers are double-buffered by collective-launch parity (steps with an
// empty selection launch nothing and do not count): a rank packs launch j+2
// into the buffer peers read at launch j only after the launch j+1 arrival,
// which every peer reaches only after finishing launch j — so no end-of-step
// barrier is needed.  Every spin-wait is bounded (%globaltimer): on timeout the
// kernel raises an error flag the host turns into COVAP_ERR_GENERIC instead of
// hanging the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <nccl.h>
#include <nccl_device.h>

#include "covap_internal.h"

namespace covapb {
namespace {

constexpr int kPeerThreads = 512;

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax(uint64_t a, uint64_t b) { return a > b ? a : b; }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
};
template <>
struct V16<double> {
  using type = double2;
};
__device__ __forceinline__ float4 vadd(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ double2 vadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
// (0 + sum) * inv: the sum already starts from +0 (phase 1), so this is
// allreduce_mean's scale step (trainer.cpp:44-45).
__device__ __forceinline__ float4 vscale(float4 a, float s) {
  return make_float4(__fmul_rn(a.x, s), __fmul_rn(a.y, s), __fmul_rn(a.z, s), __fmul_rn(a.w, s));
}
__device__ __forceinline__ double2 vscale(double2 a, double s) {
  return make_double2(__dmul_rn(a.x, s), __dmul_rn(a.y, s));
}
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename V>
__device__ __forceinline__ V vzero();
template <>
__device__ __forceinline__ float4 vzero<float4>() {
  return make_float4(0.f, 0.f, 0.f, 0.f);
}
template <>
__device__ __forceinline__ double2 vzero<double2>() {
  return make_double2(0.0, 0.0);
}

// NVLS: loads through a multicast address reduce the P ranks' copies in the
// NVSwitch; stores through it write every rank's copy.  The same memory is
// also accessed through its unicast address (K1's packing, the unpack), so a
// proxy fence orders the two views around the flag exchanges.
__device__ __forceinline__ void fence_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }
__device__ __forceinline__ float4 mm_ld_add(const float4* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ double2 mm_ld_add(const double2* p) {
  double2 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];"
               : "=d"(v.x)
               : "l"(reinterpret_cast<const double*>(p))
               : "memory");
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];"
               : "=d"(v.y)
               : "l"(reinterpret_cast<const double*>(p) + 1)
               : "memory");
  return v;
}
__device__ __forceinline__ float mm_ld_add(const float* p) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double mm_ld_add(const double* p) {
  double v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st(float4* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st(double2* p, double2 v) {
  asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(reinterpret_cast<double*>(p)),
               "d"(v.x)
               : "memory");
  asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(reinterpret_cast<double*>(p) + 1),
               "d"(v.y)
               : "memory");
}
__device__ __forceinline__ void mm_st(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void mm_st(double* p, double v) {
  asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Wait until flags[slot * 8 + q] >= epoch for every q < P (bounded).
__device__ __forceinline__ bool wait_all(const uint64_t* flags, int slot, int P, uint64_t epoch,
                                         uint64_t timeout_ns, int* err) {
  const uint64_t t0 = now_ns();
  for (int q = 0; q < P; ++q) {
    while (ld_acquire_sys(flags + slot * kMaxPeers + q) < epoch) {
      if (*reinterpret_cast<volatile int*>(err)) return false;
      if (now_ns() - t0 > timeout_ns) {
        atomicExch(err, 1);
        return false;
      }
    }
  }
  return true;
}

template <typename T>
__global__ void __launch_bounds__(kPeerThreads) peer_allreduce_kernel(const PeerArgs args) {
  using V = typename V16<T>::type;
  constexpr uint64_t W = 16 / sizeof(T);
  const int P = args.P, r = args.rank;
  T* const* bufs = reinterpret_cast<T* const*>(args.bufs);
  const uint64_t L = args.len;

  // ---- phase 0: every rank's buffer is packed --------------------------
  __shared__ int ok;
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();  // the packing kernel's writes, before the flag
      for (int p = 0; p < P; ++p) st_release_sys(args.flags[p] + 0 * kMaxPeers + r, args.epoch);
    }
    ok = wait_all(args.flags[r], 0, P, args.epoch, args.timeout_ns, args.err);
  }
  __syncthreads();
  if (!ok) return;

  // ---- phase 1: rank-ordered sum of my slice ---------------------------
  // Slice bounds in 16-byte vectors; the last slice takes the remainder.
  const uint64_t nvec = L / W;
  const uint64_t per = (nvec + P - 1) / P;
  const uint64_t v_lo = umin(nvec, per * r), v_hi = umin(nvec, per * (r + 1));
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kPeerThreads;
  // kAllB vectors per thread per round, so each rank's loads of a round are
  // in flight together (the loop is latency-bound otherwise)
  constexpr int kAllB = 4;
  if (args.mc) {  // NVLS: the switch sums slice r and stores it to every rank
    fence_alias();
    V* const mcv = static_cast<V*>(args.mc);
    for (uint64_t v0 = v_lo + blockIdx.x * kPeerThreads + threadIdx.x; v0 < v_hi;
         v0 += kAllB * stride) {
      V x[kAllB];
#pragma unroll
      for (int b = 0; b < kAllB; ++b)
        if (v0 + b * stride < v_hi) x[b] = mm_ld_add(mcv + v0 + b * stride);
#pragma unroll
      for (int b = 0; b < kAllB; ++b)
        if (v0 + b * stride < v_hi) mm_st(mcv + v0 + b * stride, x[b]);
    }
    if (r == P - 1 && blockIdx.x == 0)
      for (uint64_t e = nvec * W + threadIdx.x; e < L; e += kPeerThreads) {
        T* const mce = static_cast<T*>(args.mc);
        mm_st(mce + e, mm_ld_add(mce + e));
      }
  } else {
  for (uint64_t v0 = v_lo + blockIdx.x * kPeerThreads + threadIdx.x; v0 < v_hi;
       v0 += kAllB * stride) {
    V acc[kAllB];
#pragma unroll
    for (int b = 0; b < kAllB; ++b) acc[b] = vzero<V>();
    for (int p = 0; p < P; ++p) {
      V x[kAllB];
#pragma unroll
      for (int b = 0; b < kAllB; ++b) {
        const uint64_t v = v0 + b * stride;
        if (v < v_hi) x[b] = reinterpret_cast<const V*>(bufs[p])[v];
      }
#pragma unroll
      for (int b = 0; b < kAllB; ++b)
        if (v0 + b * stride < v_hi) acc[b] = vadd(acc[b], x[b]);
    }
#pragma unroll
    for (int b = 0; b < kAllB; ++b) {
      const uint64_t v = v0 + b * stride;
      if (v < v_hi) reinterpret_cast<V*>(bufs[r])[v] = acc[b];
    }
  }
  // the scalar tail (L not a multiple of W) belongs to the last rank
  if (r == P - 1 && blockIdx.x == 0)
    for (uint64_t e = nvec * W + threadIdx.x; e < L; e += kPeerThreads) {
      T acc = T(0);
      for (int p = 0; p < P; ++p) acc = add_rn(acc, bufs[p][e]);
      bufs[r][e] = acc;
    }
  }

  // ---- grid barrier, then phase-1 flag exchange ------------------------
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned done = atomicAdd(args.counter, 1u) + 1u;
    if (done == gridDim.x) {  // last CTA of this rank: my slice is reduced
      *args.counter = 0u;     // next launch (stream-ordered) starts from 0
      __threadfence_system();
      for (int p = 0; p < P; ++p) st_release_sys(args.flags[p] + 1 * kMaxPeers + r, args.epoch);
    }
    ok = wait_all(args.flags[r], 1, P, args.epoch, args.timeout_ns, args.err);
  }
  __syncthreads();
  if (!ok) return;
  if (args.mc) fence_alias();  // the switch's stores, read through the unicast view

  // ---- phase 2 (fused): unpack straight from the slice owners -----------
  if (args.fused) {
    T* out = static_cast<T*>(args.out);
    const T inv = static_cast<T>(args.inv);
    const Run* runs = args.runs;
    // the owner of send element o: its vector's slice; the scalar tail is
    // the last rank's (phase 1)
    auto owner = [&](uint64_t o) -> int {
      if (args.mc) return r;  // every rank holds every reduced slice
      const uint64_t v = o / W;
      return v >= nvec ? P - 1 : static_cast<int>(v / per);
    };
    auto zero_range = [&](uint64_t a, uint64_t b) {
      if (a >= b || !args.zfill) return;
      const uint64_t a16 = umin(b, (a + W - 1) / W * W), b16 = umax(a16, b / W * W);
      if (blockIdx.x == 0)
        for (uint64_t e = a + threadIdx.x; e < a16; e += kPeerThreads) out[e] = T(0);
      if (blockIdx.x == gridDim.x - 1)
        for (uint64_t e = b16 + threadIdx.x; e < b; e += kPeerThreads) out[e] = T(0);
      const V z = vzero<V>();
      for (uint64_t v = a16 / W + blockIdx.x * kPeerThreads + threadIdx.x; v < b16 / W; v += stride)
        reinterpret_cast<V*>(out)[v] = z;
    };
    uint64_t prev = 0;
    for (int j = 0; j < args.nruns; ++j) {
      const uint64_t rb = runs[j].begin, re = runs[j].end, rd = runs[j].dst;
      zero_range(prev, rb);
      prev = re;
      // dst == begin (mod 32): out vectors map onto send vectors
      const uint64_t a16 = umin(re, (rb + W - 1) / W * W), b16 = umax(a16, re / W * W);
      if (blockIdx.x == 0)
        for (uint64_t e = rb + threadIdx.x; e < a16; e += kPeerThreads) {
          const uint64_t o = rd + (e - rb);
          out[e] = mul_rn(bufs[owner(o)][o], inv);
        }
      if (blockIdx.x == gridDim.x - 1)
        for (uint64_t e = b16 + threadIdx.x; e < re; e += kPeerThreads) {
          const uint64_t o = rd + (e - rb);
          out[e] = mul_rn(bufs[owner(o)][o], inv);
        }
      constexpr int kUnB = 8;  // vectors in flight per thread
      for (uint64_t v0 = a16 / W + blockIdx.x * kPeerThreads + threadIdx.x; v0 < b16 / W;
           v0 += kUnB * stride) {
        V x[kUnB];
#pragma unroll
        for (int b = 0; b < kUnB; ++b) {
          const uint64_t v = v0 + b * stride;
          if (v < b16 / W) {
            const uint64_t o = rd + (v * W - rb);
            x[b] = *reinterpret_cast<const V*>(bufs[owner(o)] + o);
          }
        }
#pragma unroll
        for (int b = 0; b < kUnB; ++b) {
          const uint64_t v = v0 + b * stride;
          if (v < b16 / W) reinterpret_cast<V*>(out)[v] = vscale(x[b], inv);
        }
      }
    }
    zero_range(prev, args.n_out);
    return;
  }

  // ---- phase 2: gather the other ranks' reduced slices -----------------
  if (args.mc) return;  // the switch already stored them here
  for (int q = 1; q < P; ++q) {
    const int src = (r + q) % P;  // stagger the peers each rank reads first
    const uint64_t lo = umin(nvec, per * src), hi = umin(nvec, per * (src + 1));
    for (uint64_t v = lo + blockIdx.x * kPeerThreads + threadIdx.x; v < hi; v += stride)
      reinterpret_cast<V*>(bufs[r])[v] = reinterpret_cast<const V*>(bufs[src])[v];
    if (src == P - 1 && blockIdx.x == 0)
      for (uint64_t e = nvec * W + threadIdx.x; e < L; e += kPeerThreads) bufs[r][e] = bufs[src][e];
  }
}


// ------------------------------------------------------------------ whole step
//
// peer_step_kernel: K1 -> rank-ordered reduce -> unpack, one launch per rank
// (see covap_internal.h).  Every item is a 16-byte-vector pass between scalar
// edges; selected layout elements and their send slots share alignment
// (dst == begin mod kSendAlign).

constexpr int kStepThreads = 256;
#ifndef COVAP_PEER_BATCH  // 16-byte vectors each thread loads before storing (whole-step kernel)
#define COVAP_PEER_BATCH 8
#endif
#ifndef COVAP_PEER_MINB  // resident CTAs per SM the whole-step kernel is register-capped for
#define COVAP_PEER_MINB 1
#endif

__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) {
  return __ldcg(p);
}

// Spin (thread 0) until *f >= epoch; false on timeout or a peer's error.
__device__ __forceinline__ bool wait_flag(const uint64_t* f, uint64_t epoch, uint64_t timeout_ns,
                                          int* err) {
  const uint64_t t0 = now_ns();
  while (ld_acquire_sys(f) < epoch) {
    if (*reinterpret_cast<volatile int*>(err)) return false;
    if (now_ns() - t0 > timeout_ns) {
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}

// Publish (thread 0, after the block's stores): flags[p][idx] = epoch on every rank.
__device__ __forceinline__ void publish(const PeerStepArgs& A, uint64_t idx) {
  __threadfence_system();
  for (int p = 0; p < A.P; ++p) st_release_sys(A.flags[p] + idx, A.epoch);
}

// First run whose send range [dst, dst + len) ends after send offset o.
__device__ __forceinline__ int run_by_send(const Run* runs, int n, uint64_t o) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (runs[mid].dst + (runs[mid].end - runs[mid].begin) > o) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// Calls f(layout e, send o, count) for the selected pieces of send [o0, o1):
// (e, o) pairs with e == o (mod kSendAlign).
template <typename F>
__device__ __forceinline__ void for_send_pieces(const PeerStepArgs& A, uint64_t o0, uint64_t o1, F&& f) {
  for (int j = run_by_send(A.runs, A.nruns, o0); j < A.nruns; ++j) {
    const uint64_t d0 = A.runs[j].dst, d1 = d0 + (A.runs[j].end - A.runs[j].begin);
    if (d0 >= o1) break;
    const uint64_t a = d0 > o0 ? d0 : o0, b = d1 < o1 ? d1 : o1;
    if (a < b) f(A.runs[j].begin + (a - d0), a, b - a);
  }
}

// Block-wide pass over n elements starting at layout e / send o (same
// alignment mod W): scalar(i) for the unaligned head and tail; for the
// 16-byte vectors, load(i) then store(i, loaded) with kBatch vectors per
// thread loaded before any is stored, so each thread keeps several loads in
// flight (the pass is latency-bound otherwise: one CTA walks one chunk).
constexpr int kBatch = COVAP_PEER_BATCH;
template <typename T, typename S, typename Ld, typename St>
__device__ __forceinline__ void block_pass(uint64_t e, uint64_t n, S&& scalar, Ld&& load, St&& store) {
  constexpr uint64_t W = 16 / sizeof(T);
  const uint64_t head = ((W - e % W) % W) < n ? (W - e % W) % W : n;
  const uint64_t nv = (n - head) / W;
  for (uint64_t i = threadIdx.x; i < head; i += kStepThreads) scalar(i);
  for (uint64_t i = head + nv * W + threadIdx.x; i < n; i += kStepThreads) scalar(i);
  using X = decltype(load(uint64_t(0)));
  for (uint64_t v0 = 0; v0 < nv; v0 += kBatch * kStepThreads) {
    X x[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const uint64_t v = v0 + q * kStepThreads + threadIdx.x;
      if (v < nv) x[q] = load(head + v * W);
    }
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const uint64_t v = v0 + q * kStepThreads + threadIdx.x;
      if (v < nv) store(head + v * W, x[q]);
    }
  }
}

template <typename V>
struct Pair {
  V a, b;
};

template <typename T>
__global__ void __launch_bounds__(kStepThreads, COVAP_PEER_MINB) peer_step_kernel(const PeerStepArgs A) {
  using V = typename V16<T>::type;
  constexpr uint64_t W = 16 / sizeof(T);
  const int P = A.P, rank = A.rank;
  const T* __restrict__ g = static_cast<const T*>(A.g);
  T* __restrict__ r = static_cast<T*>(A.r);
  T* __restrict__ out = static_cast<T*>(A.out);
  T* mine = static_cast<T*>(A.bufs[rank]);
  const T coeff = static_cast<T>(A.coeff), inv = static_cast<T>(A.inv);
  const uint64_t rdy = kPeerFlagBase, red = kPeerFlagBase + A.cmax * kMaxPeers;
  __shared__ int s_ok;
  __shared__ unsigned s_item;

  // Arrival: my step has started (so my previous step, and every read of
  // the peers' buffers it made, is done).  My send buffer of this parity is
  // rewritten only after every peer arrived at the step after the one that
  // last read it.
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) publish(A, 2 * kMaxPeers + rank);
    bool ok = true;
    for (int q = 0; q < P && ok; ++q) {
      const uint64_t* f = A.flags[rank];
      const uint64_t t0 = now_ns();
      while (umax(ld_acquire_sys(f + 2 * kMaxPeers + q), ld_acquire_sys(f + q)) < A.wait_epoch) {
        if (*reinterpret_cast<volatile int*>(A.err) || now_ns() - t0 > A.timeout_ns) {
          atomicExch(A.err, 1);
          ok = false;
          break;
        }
      }
    }
    s_ok = ok;
  }
  __syncthreads();

  const uint64_t nchunks = (A.len + kPeerChunk - 1) / kPeerChunk;
  // unselected layout ranges: the gaps between runs, cut into tiles
  auto gap = [&](int k, uint64_t* b, uint64_t* e) {
    *b = k == 0 ? 0 : A.runs[k - 1].end;
    *e = k == A.nruns ? A.n_out : A.runs[k].begin;
  };
  uint64_t ntiles = 0;
  for (int k = 0; k <= A.nruns; ++k) {
    uint64_t b, e;
    gap(k, &b, &e);
    if (e > b) ntiles += (e - b + kPeerTile - 1) / kPeerTile;
  }
  const uint64_t nmine = nchunks > static_cast<uint64_t>(rank)
                             ? (nchunks - rank + P - 1) / P : 0;  // chunks I reduce
  const uint64_t total = nchunks + ntiles + nmine + nchunks;

  // thread 0 takes the next item while the block works on the current one
  unsigned next = 0;
  if (threadIdx.x == 0) next = atomicAdd(A.queue, 1u);
  while (s_ok) {
    if (threadIdx.x == 0) {
      s_item = next;
      if (next < total) next = atomicAdd(A.queue, 1u);
    }
    __syncthreads();
    const uint64_t item = s_item;
    __syncthreads();
    if (item >= total) break;
    if (item < nchunks) {
      // ---- pack chunk: c = g + coeff*r -> my send slot, r = 0 (compress.cpp:59-77)
      const uint64_t o0 = item * kPeerChunk, o1 = umin(A.len, o0 + kPeerChunk);
      for_send_pieces(A, o0, o1, [&](uint64_t e, uint64_t o, uint64_t n) {
        block_pass<T>(e, n,
            [&](uint64_t i) {
              const T c = A.ef ? add_rn(g[e + i], mul_rn(coeff, r[e + i])) : g[e + i];
              mine[o + i] = c;
              r[e + i] = T(0);
            },
            [&](uint64_t i) {
              Pair<V> x;
              x.a = *reinterpret_cast<const V*>(g + e + i);
              x.b = A.ef ? *reinterpret_cast<const V*>(r + e + i) : vzero<V>();
              return x;
            },
            [&](uint64_t i, Pair<V> x) {
              T* xs = reinterpret_cast<T*>(&x.a);
              const T* ys = reinterpret_cast<const T*>(&x.b);
              if (A.ef) {
#pragma unroll
                for (int w = 0; w < static_cast<int>(W); ++w) xs[w] = add_rn(xs[w], mul_rn(coeff, ys[w]));
              }
              *reinterpret_cast<V*>(mine + o + i) = x.a;
              *reinterpret_cast<V*>(r + e + i) = vzero<V>();
            });
      });
      __syncthreads();
      if (threadIdx.x == 0) publish(A, rdy + item * kMaxPeers + rank);
    } else if (item < nchunks + ntiles) {
      // ---- unselected tile: r = c (compress.cpp:79), out = 0 (compress.cpp:91)
      uint64_t u = item - nchunks, b = 0, e = 0;
      for (int k = 0; k <= A.nruns; ++k) {
        gap(k, &b, &e);
        const uint64_t t = e > b ? (e - b + kPeerTile - 1) / kPeerTile : 0;
        if (u < t) break;
        u -= t;
      }
      const uint64_t e0 = b + u * kPeerTile, n = umin(e, e0 + kPeerTile) - e0;
      block_pass<T>(e0, n,
          [&](uint64_t i) {
            r[e0 + i] = A.ef ? add_rn(g[e0 + i], mul_rn(coeff, r[e0 + i])) : g[e0 + i];
            out[e0 + i] = T(0);
          },
          [&](uint64_t i) {
            Pair<V> x;
            x.a = *reinterpret_cast<const V*>(g + e0 + i);
            x.b = A.ef ? *reinterpret_cast<const V*>(r + e0 + i) : vzero<V>();
            return x;
          },
          [&](uint64_t i, Pair<V> x) {
            T* xs = reinterpret_cast<T*>(&x.a);
            const T* ys = reinterpret_cast<const T*>(&x.b);
            if (A.ef) {
#pragma unroll
              for (int w = 0; w < static_cast<int>(W); ++w) xs[w] = add_rn(xs[w], mul_rn(coeff, ys[w]));
            }
            *reinterpret_cast<V*>(r + e0 + i) = x.a;
            *reinterpret_cast<V*>(out + e0 + i) = vzero<V>();
          });
    } else if (item < nchunks + ntiles + nmine) {
      // ---- reduce a chunk I own, in rank order (trainer.cpp:41-43)
      const uint64_t x = rank + (item - nchunks - ntiles) * P;
      if (threadIdx.x == 0) {
        bool ok = true;
        for (int q = 0; q < P && ok; ++q)
          ok = wait_flag(A.flags[rank] + rdy + x * kMaxPeers + q, A.epoch, A.timeout_ns, A.err);
        s_ok = ok;
      }
      __syncthreads();
      if (!s_ok) break;
      const uint64_t o0 = x * kPeerChunk, o1 = umin(A.len, o0 + kPeerChunk);
      block_pass<T>(o0, o1 - o0,
          [&](uint64_t i) {
            T acc = T(0);
            for (int q = 0; q < P; ++q) acc = add_rn(acc, ldcg(static_cast<const T*>(A.bufs[q]) + o0 + i));
            mine[o0 + i] = acc;
          },
          [&](uint64_t i) {
            V acc = vzero<V>();
            for (int q = 0; q < P; ++q)
              acc = vadd(acc, ldcg(reinterpret_cast<const V*>(static_cast<const T*>(A.bufs[q]) + o0 + i)));
            return acc;
          },
          [&](uint64_t i, V acc) { *reinterpret_cast<V*>(mine + o0 + i) = acc; });
      __syncthreads();
      if (threadIdx.x == 0) publish(A, red + x);
    } else {
      // ---- unpack a reduced chunk from its owner: out = sum * (1/P)
      const uint64_t x = item - nchunks - ntiles - nmine;
      const T* src = static_cast<const T*>(A.bufs[x % P]);
      if (threadIdx.x == 0) s_ok = wait_flag(A.flags[rank] + red + x, A.epoch, A.timeout_ns, A.err);
      __syncthreads();
      if (!s_ok) break;
      const uint64_t o0 = x * kPeerChunk, o1 = umin(A.len, o0 + kPeerChunk);
      for_send_pieces(A, o0, o1, [&](uint64_t e, uint64_t o, uint64_t n) {
        block_pass<T>(e, n,
            [&](uint64_t i) { out[e + i] = mul_rn(ldcg(src + o + i), inv); },
            [&](uint64_t i) { return ldcg(reinterpret_cast<const V*>(src + o + i)); },
            [&](uint64_t i, V x) { *reinterpret_cast<V*>(out + e + i) = vscale(x, inv); });
      });
    }
  }
  // the last CTA out resets the queue for the next (stream-ordered) launch
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(A.queue + 1, 1u) + 1u == gridDim.x) {
    A.queue[0] = 0u;
    A.queue[1] = 0u;
  }
}
}  // namespace

cudaError_t launch_peer_allreduce(int dtype, const PeerArgs& args, int max_ctas, cudaStream_t s) {
  if (args.len == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  // Every CTA spins at the barriers, so all must be resident: at most one
  // per SM (or the caller's cap), never more than the work needs.
  const uint64_t w = 16 / (dtype == 0 ? 4 : 8);
  const uint64_t vec_per_rank = (args.len / w + args.P - 1) / args.P;
  int grid = static_cast<int>(std::min<uint64_t>(
      sms, std::max<uint64_t>(1, (vec_per_rank + kPeerThreads - 1) / kPeerThreads)));
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  if (dtype == 0)
    peer_allreduce_kernel<float><<<grid, kPeerThreads, 0, s>>>(args);
  else
    peer_allreduce_kernel<double><<<grid, kPeerThreads, 0, s>>>(args);
  return cudaGetLastError();
}


cudaError_t launch_peer_step(int dtype, const PeerStepArgs& args, int max_ctas, cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev))) return e;
  // Work items come from an in-order queue, so no CTA waits for an item no
  // running CTA has taken: any grid is deadlock-free on its own GPU.  Ranks
  // sharing one GPU (tests) cap the grid so that they are co-resident.
  int grid = sms * COVAP_PEER_MINB;  // one wave: the queue hands out the work
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  if (dtype == 0)
    peer_step_kernel<float><<<grid, kStepThreads, 0, s>>>(args);
  else
    peer_step_kernel<double><<<grid, kStepThreads, 0, s>>>(args);
  return cudaGetLastError();
}



// ------------------------------------------------------- NCCL peer memory
//
// The peer collective's buffers as an NCCL symmetric window (NCCL 2.28's
// device API): NCCL maps every rank's allocation into every peer over NVLink
// (and, with multimem, binds them to one NVSwitch multicast object), so the
// kernels above get their peer / multicast addresses without CUDA IPC.

struct NcclPeerMem {
  void* base = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dc{};
  bool has_dc = false;
};

namespace {
__global__ void nccl_peer_ptrs_kernel(ncclWindow_t w, ncclDevComm dc, int has_dc, int P,
                                      void** out) {
  if (threadIdx.x != 0) return;
  for (int p = 0; p < P; ++p) out[p] = ncclGetPeerPointer(w, 0, p);
  out[P] = has_dc && dc.lsaMultimem.mcBasePtr ? ncclGetLsaMultimemPointer(w, 0, dc) : nullptr;
}
}  // namespace

void nccl_peer_mem_release(ncclComm* comm, NcclPeerMem* m) {
  if (!m || !comm) return;
  if (m->has_dc) ncclDevCommDestroy(comm, &m->dc);
  if (m->win) ncclCommWindowDeregister(comm, m->win);
  m->has_dc = false;
  m->win = nullptr;
}

void nccl_peer_mem_destroy(ncclComm* comm, NcclPeerMem* m) {
  if (!m) return;
  nccl_peer_mem_release(comm, m);
  if (m->base) ncclMemFree(m->base);
  delete m;
}

int nccl_peer_mem_create(ncclComm* comm, int nranks, size_t bytes, int want_multimem,
                         NcclPeerMem** out, void** peers, void** mc, const char** what) {
  NcclPeerMem* m = new NcclPeerMem;
  auto fail = [&](const char* msg) {
    *what = msg;
    nccl_peer_mem_destroy(comm, m);
    return 1;
  };
  if (ncclMemAlloc(&m->base, bytes) != ncclSuccess) return fail("ncclMemAlloc");
  if (cudaMemset(m->base, 0, bytes) != cudaSuccess) return fail("cudaMemset(peer window)");
  if (ncclCommWindowRegister(comm, m->base, bytes, &m->win, NCCL_WIN_COLL_SYMMETRIC) !=
      ncclSuccess)
    return fail("ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)");
  if (want_multimem) {
    ncclDevCommRequirements req{};
    req.lsaMultimem = true;
    if (ncclDevCommCreate(comm, &req, &m->dc) != ncclSuccess)
      return fail("ncclDevCommCreate(lsaMultimem): no NVSwitch multicast for this communicator");
    m->has_dc = true;
    if (m->dc.lsaSize != nranks) return fail("multimem needs every rank in one NVLink domain");
  }
  void** d_out = nullptr;
  if (cudaMalloc(reinterpret_cast<void**>(&d_out), (kMaxPeers + 1) * sizeof(void*)) != cudaSuccess)
    return fail("cudaMalloc");
  nccl_peer_ptrs_kernel<<<1, 32>>>(m->win, m->dc, m->has_dc ? 1 : 0, nranks, d_out);
  void* h[kMaxPeers + 1] = {};
  const cudaError_t e = cudaMemcpy(h, d_out, (nranks + 1) * sizeof(void*), cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  if (e != cudaSuccess) return fail("peer pointer query kernel");
  for (int p = 0; p < nranks; ++p) {
    if (!h[p]) return fail("a rank's window is not load/store-accessible (not on this NVLink domain)");
    peers[p] = h[p];
  }
  *mc = h[nranks];
  if (want_multimem && !*mc) return fail("the window has no multicast address");
  *out = m;
  return 0;
}

}  // namespace covapb
