// covap_kernels.cu — the sm_100a kernels of the COVAP sync path.
//
//   K1 filter_pack   compress.cpp:59-81   (EF add, round-robin select, pack, residual write-back)
//   K2 unpack        compress.cpp:87-103 + trainer.cpp:41-45 (embed, sum-then-scale, zero fill)
//   K0 generate      synthetic gradients (rng.hpp:12-21 splitmix64 stream, counter-based)
//   K3 spin          backward emulator for the overlap schedule
//
// K1/K2 are HBM-streaming kernels (≈0.2 flop/byte): no tensor cores, no shared
// memory staging (no reuse).  Design:
//   * every CTA owns one contiguous, equal share of the 16-byte vectors of the
//     launch range (balanced to one vector, so no wave tail), walking it in
//     tiles of kThreads x kUnroll vectors; all kUnroll loads of a tile are
//     issued before any use (8 x 16 B in flight per thread for K1);
//   * loads are ld.global.cs (evict-first) 128-bit; stores st.global.cs;
//   * selection is positional: the phase's run table (a handful of entries)
//     is binary-searched once per CTA and walked forward per tile, so a tile
//     is "all selected", "none selected" (vector fast paths) or "mixed"
//     (per-element path, only at run boundaries);
//   * arithmetic uses __fmul_rn/__fadd_rn (__dmul_rn/__dadd_rn) so nvcc can
//     never contract g + coeff*r into an FMA: the multiply and the add round
//     separately exactly as compress.cpp:64 does on x86-64.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>

#include "covap_internal.h"

namespace covapb {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

template <typename T>
struct V16;
template <>
struct V16<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct V16<double> {
  using type = double2;
  static constexpr int n = 2;
};

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename V, typename T>
__device__ __forceinline__ T& lane(V& v, int k) {
  return reinterpret_cast<T*>(&v)[k];
}

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

// The selected-run index holding element e, or -1; j is a forward cursor.
__device__ __forceinline__ int run_of(const Run* __restrict__ runs, int n, int j, uint64_t e) {
  while (j < n && runs[j].end <= e) ++j;
  return (j < n && runs[j].begin <= e) ? j : -1;
}

// ---------------------------------------------------------------- K1

template <typename T>
__device__ __forceinline__ void filter_scalar(const T* __restrict__ g, T* __restrict__ r,
                                              T* __restrict__ send, const Run* __restrict__ runs,
                                              int nruns, uint64_t e, T coeff, int ef) {
  T c = g[e];
  if (ef) c = add_rn(c, mul_rn(coeff, r[e]));
  const int j = run_of(runs, nruns, first_run_after(runs, nruns, e), e);
  if (j >= 0) {
    send[runs[j].dst + (e - runs[j].begin)] = c;
    r[e] = T(0);
  } else {
    r[e] = c;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    filter_pack_kernel(const T* __restrict__ g, T* __restrict__ r, T* __restrict__ send,
                       const Run* __restrict__ runs, int nruns, uint64_t a, uint64_t b, T coeff,
                       int ef) {
  using V = typename V16<T>::type;
  constexpr int W = V16<T>::n;
  const uint64_t A = (a + W - 1) / W * W;
  uint64_t B;
  if (A >= b) {  // the whole range sits inside one vector: scalar only
    if (blockIdx.x == 0)
      for (uint64_t e = a + threadIdx.x; e < b; e += blockDim.x)
        filter_scalar(g, r, send, runs, nruns, e, coeff, ef);
    return;
  }
  B = b / W * W;
  if (blockIdx.x == 0) {  // unaligned head [a, A) and tail [B, b)
    if (threadIdx.x < A - a) filter_scalar(g, r, send, runs, nruns, a + threadIdx.x, coeff, ef);
    if (threadIdx.x < b - B) filter_scalar(g, r, send, runs, nruns, B + threadIdx.x, coeff, ef);
  }
  const uint64_t nvec = (B - A) / W;
  const uint64_t v0 = nvec * blockIdx.x / gridDim.x;
  const uint64_t v1 = nvec * (blockIdx.x + 1) / gridDim.x;
  if (v0 >= v1) return;
  const V* __restrict__ gv = reinterpret_cast<const V*>(g + A);
  V* __restrict__ rv = reinterpret_cast<V*>(r + A);

  int j = first_run_after(runs, nruns, A + v0 * W);
  constexpr uint64_t kTile = (uint64_t)kThreads * kUnroll;
  for (uint64_t t = v0; t < v1; t += kTile) {
    const uint64_t te0 = A + t * W;
    const uint64_t te1 = A + min(t + kTile, v1) * W;
    while (j < nruns && runs[j].end <= te0) ++j;
    uint64_t rb = 0, re = 0, rd = 0;
    if (j < nruns) {
      rb = runs[j].begin;
      re = runs[j].end;
      rd = runs[j].dst;
    }
    const bool none = (j >= nruns) || rb >= te1;
    const bool full = !none && rb <= te0 && te1 <= re;

    V x[kUnroll], y[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t v = t + (uint64_t)u * kThreads + threadIdx.x;
      if (v < v1) {
        x[u] = __ldcs(gv + v);
        if (ef) y[u] = __ldcs(rv + v);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t v = t + (uint64_t)u * kThreads + threadIdx.x;
      if (v >= v1) continue;
      V c = x[u];
      if (ef) {
#pragma unroll
        for (int k = 0; k < W; ++k)
          lane<V, T>(c, k) = add_rn(lane<V, T>(x[u], k), mul_rn(coeff, lane<V, T>(y[u], k)));
      }
      const uint64_t e = A + v * W;
      if (full) {
        __stcs(reinterpret_cast<V*>(send + rd + (e - rb)), c);
        V z;
#pragma unroll
        for (int k = 0; k < W; ++k) lane<V, T>(z, k) = T(0);
        __stcs(rv + v, z);
      } else if (none) {
        __stcs(rv + v, c);
      } else {
        int jj = j;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const uint64_t ee = e + k;
          while (jj < nruns && runs[jj].end <= ee) ++jj;
          if (jj < nruns && runs[jj].begin <= ee) {
            send[runs[jj].dst + (ee - runs[jj].begin)] = lane<V, T>(c, k);
            r[ee] = T(0);
          } else {
            r[ee] = lane<V, T>(c, k);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K2

// mean: allreduce_mean's (0.0 + sum) * (1/P) (trainer.cpp:41-45) -- the
// leading +0 turns a -0 sum into +0 exactly as the reference does; otherwise
// the plain embedding of covap_decompress (compress.cpp:100) times `inv`.
template <typename T>
__device__ __forceinline__ T scale_of(T x, T inv, int mean) {
  return mul_rn(mean ? add_rn(T(0), x) : x, inv);
}

template <typename T>
__device__ __forceinline__ void unpack_scalar(const T* __restrict__ recv, T* __restrict__ out,
                                              const Run* __restrict__ runs, int nruns, uint64_t e,
                                              T inv, int mean) {
  const int j = run_of(runs, nruns, first_run_after(runs, nruns, e), e);
  out[e] = (j >= 0) ? scale_of(recv[runs[j].dst + (e - runs[j].begin)], inv, mean) : T(0);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    unpack_kernel(const T* __restrict__ recv, T* __restrict__ out, const Run* __restrict__ runs,
                  int nruns, uint64_t a, uint64_t b, T inv, int mean) {
  using V = typename V16<T>::type;
  constexpr int W = V16<T>::n;
  const uint64_t A = (a + W - 1) / W * W;
  if (A >= b) {
    if (blockIdx.x == 0)
      for (uint64_t e = a + threadIdx.x; e < b; e += blockDim.x)
        unpack_scalar(recv, out, runs, nruns, e, inv, mean);
    return;
  }
  const uint64_t B = b / W * W;
  if (blockIdx.x == 0) {
    if (threadIdx.x < A - a) unpack_scalar(recv, out, runs, nruns, a + threadIdx.x, inv, mean);
    if (threadIdx.x < b - B) unpack_scalar(recv, out, runs, nruns, B + threadIdx.x, inv, mean);
  }
  const uint64_t nvec = (B - A) / W;
  const uint64_t v0 = nvec * blockIdx.x / gridDim.x;
  const uint64_t v1 = nvec * (blockIdx.x + 1) / gridDim.x;
  if (v0 >= v1) return;
  V* __restrict__ ov = reinterpret_cast<V*>(out + A);

  int j = first_run_after(runs, nruns, A + v0 * W);
  constexpr uint64_t kTile = (uint64_t)kThreads * kUnroll;
  for (uint64_t t = v0; t < v1; t += kTile) {
    const uint64_t te0 = A + t * W;
    const uint64_t te1 = A + min(t + kTile, v1) * W;
    while (j < nruns && runs[j].end <= te0) ++j;
    uint64_t rb = 0, re = 0, rd = 0;
    if (j < nruns) {
      rb = runs[j].begin;
      re = runs[j].end;
      rd = runs[j].dst;
    }
    const bool none = (j >= nruns) || rb >= te1;
    const bool full = !none && rb <= te0 && te1 <= re;
    if (none) {
      V z;
#pragma unroll
      for (int k = 0; k < W; ++k) lane<V, T>(z, k) = T(0);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t v = t + (uint64_t)u * kThreads + threadIdx.x;
        if (v < v1) __stcs(ov + v, z);
      }
    } else if (full) {
      V x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t v = t + (uint64_t)u * kThreads + threadIdx.x;
        if (v < v1) x[u] = __ldcs(reinterpret_cast<const V*>(recv + rd + (A + v * W - rb)));
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t v = t + (uint64_t)u * kThreads + threadIdx.x;
        if (v >= v1) continue;
        V o;
#pragma unroll
        for (int k = 0; k < W; ++k) lane<V, T>(o, k) = scale_of(lane<V, T>(x[u], k), inv, mean);
        __stcs(ov + v, o);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint64_t v = t + (uint64_t)u * kThreads + threadIdx.x;
        if (v >= v1) continue;
        const uint64_t e = A + v * W;
        int jj = j;
        V o;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const uint64_t ee = e + k;
          while (jj < nruns && runs[jj].end <= ee) ++jj;
          lane<V, T>(o, k) = (jj < nruns && runs[jj].begin <= ee)
                                 ? scale_of(recv[runs[jj].dst + (ee - runs[jj].begin)], inv, mean)
                                 : T(0);
        }
        __stcs(ov + v, o);
      }
    }
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
    const int32_t s = (int32_t)((x & 0xffff) + ((x >> 16) & 0xffff) + ((x >> 32) & 0xffff) +
                                (x >> 48)) -
                      131070;
    return mul_rn((T)s, (T)(1.0 / 32768.0));
  }
  return (T)((int64_t)(x % 2001) - 1000);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    generate_kernel(T* __restrict__ out, uint64_t n, uint64_t key, int kind, uint64_t begin) {
  using V = typename V16<T>::type;
  constexpr int W = V16<T>::n;
  const uint64_t nvec = n / W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    V o;
#pragma unroll
    for (int k = 0; k < W; ++k) lane<V, T>(o, k) = gen_value<T>(key, begin + v * W + k, kind);
    reinterpret_cast<V*>(out)[v] = o;
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
  int k1_f32 = 0, k1_f64 = 0, k2_f32 = 0, k2_f64 = 0;
};

DeviceShape& shape_for_current_device() {
  static std::mutex mu;
  static DeviceShape shapes[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  DeviceShape& s = shapes[dev & 63];
  if (s.sms == 0) {
    cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.k1_f32, filter_pack_kernel<float>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.k1_f64, filter_pack_kernel<double>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.k2_f32, unpack_kernel<float>, kThreads, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.k2_f64, unpack_kernel<double>, kThreads, 0);
  }
  return s;
}

// One resident wave (SMs x CTAs/SM), fewer when the range is small: each CTA
// then gets at least one full tile.
unsigned grid_for(uint64_t n_elems, int width, int sms, int per_sm) {
  const uint64_t nvec = n_elems / width;
  const uint64_t tiles = (nvec + (uint64_t)kThreads * kUnroll - 1) / ((uint64_t)kThreads * kUnroll);
  const uint64_t wave = (uint64_t)sms * (uint64_t)std::max(per_sm, 1);
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(wave, tiles));
}

}  // namespace

cudaError_t launch_filter_pack(int dtype, const void* g, void* r, void* send, const Run* runs,
                               int nruns, uint64_t a, uint64_t b, double coeff, int ef,
                               cudaStream_t s) {
  if (b <= a) return cudaSuccess;
  DeviceShape& sh = shape_for_current_device();
  if (dtype == 0) {
    const unsigned grid = grid_for(b - a, 4, sh.sms, sh.k1_f32);
    filter_pack_kernel<float><<<grid, kThreads, 0, s>>>(
        static_cast<const float*>(g), static_cast<float*>(r), static_cast<float*>(send), runs,
        nruns, a, b, (float)coeff, ef);
  } else {
    const unsigned grid = grid_for(b - a, 2, sh.sms, sh.k1_f64);
    filter_pack_kernel<double><<<grid, kThreads, 0, s>>>(
        static_cast<const double*>(g), static_cast<double*>(r), static_cast<double*>(send), runs,
        nruns, a, b, coeff, ef);
  }
  return cudaGetLastError();
}

cudaError_t launch_unpack(int dtype, const void* recv, void* out, const Run* runs, int nruns,
                          uint64_t a, uint64_t b, double inv, int mean, cudaStream_t s) {
  if (b <= a) return cudaSuccess;
  DeviceShape& sh = shape_for_current_device();
  if (dtype == 0) {
    const unsigned grid = grid_for(b - a, 4, sh.sms, sh.k2_f32);
    unpack_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(recv),
                                                   static_cast<float*>(out), runs, nruns, a, b,
                                                   (float)inv, mean);
  } else {
    const unsigned grid = grid_for(b - a, 2, sh.sms, sh.k2_f64);
    unpack_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<const double*>(recv),
                                                    static_cast<double*>(out), runs, nruns, a, b,
                                                    inv, mean);
  }
  return cudaGetLastError();
}

cudaError_t launch_generate(int dtype, void* out, uint64_t n, uint64_t key, int kind,
                            uint64_t begin, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  DeviceShape& sh = shape_for_current_device();
  const unsigned grid = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t)sh.sms * 8, (n / 4 + kThreads - 1) / kThreads));
  if (dtype == 0)
    generate_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<float*>(out), n, key, kind, begin);
  else
    generate_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<double*>(out), n, key, kind, begin);
  return cudaGetLastError();
}

cudaError_t launch_spin(double us, int blocks, cudaStream_t s) {
  if (us <= 0) return cudaSuccess;
  spin_kernel<<<std::max(blocks, 1), 32, 0, s>>>((uint64_t)(us * 1000.0));
  return cudaGetLastError();
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

}  // namespace covapb
