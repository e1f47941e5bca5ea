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
// Send buffers are double-buffered by step parity: a rank packs step s+2 into
// the buffer peers read at step s only after the step s+1 arrival, which
// every peer reaches only after finishing step s — so no end-of-step barrier
// is needed.  Every spin-wait is bounded (%globaltimer): on timeout the
// kernel raises an error flag the host turns into COVAP_ERR_GENERIC instead of
// hanging the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

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
  for (uint64_t v = v_lo + blockIdx.x * kPeerThreads + threadIdx.x; v < v_hi; v += stride) {
    V acc = vzero<V>();
    for (int p = 0; p < P; ++p) acc = vadd(acc, reinterpret_cast<const V*>(bufs[p])[v]);
    reinterpret_cast<V*>(bufs[r])[v] = acc;
  }
  // the scalar tail (L not a multiple of W) belongs to the last rank
  if (r == P - 1 && blockIdx.x == 0)
    for (uint64_t e = nvec * W + threadIdx.x; e < L; e += kPeerThreads) {
      T acc = T(0);
      for (int p = 0; p < P; ++p) acc = add_rn(acc, bufs[p][e]);
      bufs[r][e] = acc;
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

  // ---- phase 2 (fused): unpack straight from the slice owners -----------
  if (args.fused) {
    T* out = static_cast<T*>(args.out);
    const T inv = static_cast<T>(args.inv);
    const Run* runs = args.runs;
    // the owner of send element o: its vector's slice; the scalar tail is
    // the last rank's (phase 1)
    auto owner = [&](uint64_t o) -> int {
      const uint64_t v = o / W;
      return v >= nvec ? P - 1 : static_cast<int>(v / per);
    };
    auto zero_range = [&](uint64_t a, uint64_t b) {
      if (a >= b) return;
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
      for (uint64_t v = a16 / W + blockIdx.x * kPeerThreads + threadIdx.x; v < b16 / W; v += stride) {
        const uint64_t o = rd + (v * W - rb);
        V x = *reinterpret_cast<const V*>(bufs[owner(o)] + o);
        reinterpret_cast<V*>(out)[v] = vscale(x, inv);
      }
    }
    zero_range(prev, args.n_out);
    return;
  }

  // ---- phase 2: gather the other ranks' reduced slices -----------------
  for (int q = 1; q < P; ++q) {
    const int src = (r + q) % P;  // stagger the peers each rank reads first
    const uint64_t lo = umin(nvec, per * src), hi = umin(nvec, per * (src + 1));
    for (uint64_t v = lo + blockIdx.x * kPeerThreads + threadIdx.x; v < hi; v += stride)
      reinterpret_cast<V*>(bufs[r])[v] = reinterpret_cast<const V*>(bufs[src])[v];
    if (src == P - 1 && blockIdx.x == 0)
      for (uint64_t e = nvec * W + threadIdx.x; e < L; e += kPeerThreads) bufs[r][e] = bufs[src][e];
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

}  // namespace covapb
