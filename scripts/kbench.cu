// kbench.cu — design-space microbenchmark for the K1/K2 streaming kernels
// (not product code).  Measures, at the ResNet-50 / BERT-large sizes, how the
// HBM throughput of a "read g, r; write send, r" pass (K1 shape) and a
// "read x; write y" pass (K2 shape, and a plain copy) depends on vector
// width, unroll depth, CTA shape, cache hints, work distribution, and a
// TMA-bulk (cp.async.bulk) pipeline.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o kbench kbench.cu
//   ./kbench [n_elems]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);    \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

enum Hint { kDefault = 0, kStream = 1, kNoAlloc = 2, kEvictLast = 3 };

template <int H>
__device__ __forceinline__ float4 ld(const float4* p) {
  if (H == kStream) return __ldcs(p);
  if (H == kNoAlloc) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
  }
  if (H == kEvictLast) {
    float4 r;
    asm volatile("ld.global.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
  }
  return *p;
}
template <int H>
__device__ __forceinline__ void st(float4* p, float4 v) {
  if (H == kStream)
    __stcs(p, v);
  else if (H == kNoAlloc)
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w));
  else
    *p = v;
}

// 256-bit vectors (sm_100: ld.global.v8.f32)
struct f8 {
  float v[8];
};
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                 "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ f8 ld8rw(const float* p) {
  f8 r;
  asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                 "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st8(float* p, const f8& x) {
  asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "f"(x.v[0]), "f"(x.v[1]), "f"(x.v[2]), "f"(x.v[3]), "f"(x.v[4]), "f"(x.v[5]),
               "f"(x.v[6]), "f"(x.v[7]));
}

// K1 shape, contiguous chunk per CTA (current product design).
template <int T, int U, int HL, int HS>
__global__ void __launch_bounds__(T) k1_chunk(const float4* g, float4* r, float4* s, uint64_t nv,
                                              float c) {
  const uint64_t v0 = nv * blockIdx.x / gridDim.x, v1 = nv * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t t = v0; t < v1; t += (uint64_t)T * U) {
    float4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) {
        x[u] = ld<HL>(g + v);
        y[u] = ld<HL == kNoAlloc ? kDefault : HL>(r + v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) {
        float4 o;
        o.x = __fadd_rn(x[u].x, __fmul_rn(c, y[u].x));
        o.y = __fadd_rn(x[u].y, __fmul_rn(c, y[u].y));
        o.z = __fadd_rn(x[u].z, __fmul_rn(c, y[u].z));
        o.w = __fadd_rn(x[u].w, __fmul_rn(c, y[u].w));
        st<HS>(s + v, o);
        st<HS>(r + v, make_float4(0, 0, 0, 0));
      }
    }
  }
}

// K1 shape, grid-stride interleaved.
template <int T, int U, int HL, int HS>
__global__ void __launch_bounds__(T) k1_stride(const float4* g, float4* r, float4* s, uint64_t nv,
                                               float c) {
  const uint64_t stride = (uint64_t)gridDim.x * T * U;
  for (uint64_t t = (uint64_t)blockIdx.x * T * U; t < nv; t += stride) {
    float4 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < nv) {
        x[u] = ld<HL>(g + v);
        y[u] = ld<HL == kNoAlloc ? kDefault : HL>(r + v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < nv) {
        float4 o;
        o.x = __fadd_rn(x[u].x, __fmul_rn(c, y[u].x));
        o.y = __fadd_rn(x[u].y, __fmul_rn(c, y[u].y));
        o.z = __fadd_rn(x[u].z, __fmul_rn(c, y[u].z));
        o.w = __fadd_rn(x[u].w, __fmul_rn(c, y[u].w));
        st<HS>(s + v, o);
        st<HS>(r + v, make_float4(0, 0, 0, 0));
      }
    }
  }
}

// K1 shape with 256-bit accesses, contiguous chunks.
template <int T, int U>
__global__ void __launch_bounds__(T) k1_v8(const float* g, float* r, float* s, uint64_t n8,
                                           float c) {
  const uint64_t v0 = n8 * blockIdx.x / gridDim.x, v1 = n8 * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t t = v0; t < v1; t += (uint64_t)T * U) {
    f8 x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) {
        x[u] = ld8(g + 8 * v);
        y[u] = ld8rw(r + 8 * v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) {
        f8 o, z;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          o.v[k] = __fadd_rn(x[u].v[k], __fmul_rn(c, y[u].v[k]));
          z.v[k] = 0.f;
        }
        st8(s + 8 * v, o);
        st8(r + 8 * v, z);
      }
    }
  }
}

// K2 / copy shape: read x, write y = x * c.
template <int T, int U, int HL, int HS>
__global__ void __launch_bounds__(T) k2_chunk(const float4* x, float4* y, uint64_t nv, float c) {
  const uint64_t v0 = nv * blockIdx.x / gridDim.x, v1 = nv * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t t = v0; t < v1; t += (uint64_t)T * U) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) a[u] = ld<HL>(x + v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) {
        float4 o = a[u];
        o.x = __fmul_rn(o.x, c);
        o.y = __fmul_rn(o.y, c);
        o.z = __fmul_rn(o.z, c);
        o.w = __fmul_rn(o.w, c);
        st<HS>(y + v, o);
      }
    }
  }
}

template <int T, int U>
__global__ void __launch_bounds__(T) k2_v8(const float* x, float* y, uint64_t n8, float c) {
  const uint64_t v0 = n8 * blockIdx.x / gridDim.x, v1 = n8 * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t t = v0; t < v1; t += (uint64_t)T * U) {
    f8 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) a[u] = ld8(x + 8 * v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < v1) {
        f8 o;
#pragma unroll
        for (int k = 0; k < 8; ++k) o.v[k] = __fmul_rn(a[u].v[k], c);
        st8(y + 8 * v, o);
      }
    }
  }
}

// ---- TMA bulk pipeline for the K1 shape --------------------------------
// Persistent CTAs; each CTA walks its contiguous chunk in tiles of TILE
// floats per array.  Thread 0 issues cp.async.bulk loads of g and r into an
// S-stage ring (mbarrier complete_tx); all threads compute; results are
// written to smem staging and bulk-stored (cp.async.bulk.global.shared).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" ::"r"(smem_u32(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int T, int TILE, int S, bool INTER>
__global__ void __launch_bounds__(T) k1_tma(const float* g, float* r, float* s, uint64_t ntiles,
                                            float c) {
  extern __shared__ __align__(128) float sm[];
  float* gin = sm;                   // S x TILE
  float* rin = sm + S * TILE;        // S x TILE
  float* sout = sm + 2 * S * TILE;   // 2 x TILE (double-buffered)
  float* rout = sm + 2 * S * TILE + 2 * TILE;
  __shared__ __align__(8) uint64_t bar[S];
  const uint64_t t0c = ntiles * blockIdx.x / gridDim.x, t1c = ntiles * (blockIdx.x + 1) / gridDim.x;
  const uint64_t my = INTER ? (ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0)
                            : t1c - t0c;
  auto tile_of = [&](uint64_t k) { return INTER ? blockIdx.x + k * gridDim.x : t0c + k; };
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < S && i < (int)my; ++i) {
      mbar_expect_tx(&bar[i], 2 * TILE * 4);
      bulk_g2s(gin + i * TILE, g + tile_of(i) * TILE, TILE * 4, &bar[i]);
      bulk_g2s(rin + i * TILE, r + tile_of(i) * TILE, TILE * 4, &bar[i]);
    }
  }
  for (uint64_t k = 0; k < my; ++k) {
    const int st_ = k % S;
    const uint32_t ph = (k / S) & 1;
    mbar_wait(&bar[st_], ph);
    const int ob = k & 1;
    // make sure the bulk store that used this output buffer two tiles ago has read it
    if (threadIdx.x == 0) bulk_wait_read<1>();
    __syncthreads();
    const float4* gi = reinterpret_cast<const float4*>(gin + st_ * TILE);
    const float4* ri = reinterpret_cast<const float4*>(rin + st_ * TILE);
    float4* so = reinterpret_cast<float4*>(sout + ob * TILE);
    float4* ro = reinterpret_cast<float4*>(rout + ob * TILE);
    for (int i = threadIdx.x; i < TILE / 4; i += T) {
      float4 x = gi[i], y = ri[i], o;
      o.x = __fadd_rn(x.x, __fmul_rn(c, y.x));
      o.y = __fadd_rn(x.y, __fmul_rn(c, y.y));
      o.z = __fadd_rn(x.z, __fmul_rn(c, y.z));
      o.w = __fadd_rn(x.w, __fmul_rn(c, y.w));
      so[i] = o;
      ro[i] = make_float4(0, 0, 0, 0);
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint64_t tile = tile_of(k);
      bulk_s2g(s + tile * TILE, sout + ob * TILE, TILE * 4);
      bulk_s2g(r + tile * TILE, rout + ob * TILE, TILE * 4);
      bulk_commit();
      // refill this stage with tile k + S
      if (k + S < my) {
        mbar_expect_tx(&bar[st_], 2 * TILE * 4);
        bulk_g2s(gin + st_ * TILE, g + tile_of(k + S) * TILE, TILE * 4, &bar[st_]);
        bulk_g2s(rin + st_ * TILE, r + tile_of(k + S) * TILE, TILE * 4, &bar[st_]);
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_read<0>();
}

template <int T, int TILE, int S, bool INTER>
__global__ void __launch_bounds__(T) k2_tma(const float* x, float* y, uint64_t ntiles, float c) {
  extern __shared__ __align__(128) float sm[];
  float* in = sm;
  float* out = sm + S * TILE;
  __shared__ __align__(8) uint64_t bar[S];
  const uint64_t t0c = ntiles * blockIdx.x / gridDim.x, t1c = ntiles * (blockIdx.x + 1) / gridDim.x;
  const uint64_t my = INTER ? (ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0)
                            : t1c - t0c;
  auto tile_of = [&](uint64_t k) { return INTER ? blockIdx.x + k * gridDim.x : t0c + k; };
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < S && i < (int)my; ++i) {
      mbar_expect_tx(&bar[i], TILE * 4);
      bulk_g2s(in + i * TILE, x + tile_of(i) * TILE, TILE * 4, &bar[i]);
    }
  for (uint64_t k = 0; k < my; ++k) {
    const int st_ = k % S;
    mbar_wait(&bar[st_], (k / S) & 1);
    const int ob = k & 1;
    if (threadIdx.x == 0) bulk_wait_read<1>();
    __syncthreads();
    const float4* xi = reinterpret_cast<const float4*>(in + st_ * TILE);
    float4* yo = reinterpret_cast<float4*>(out + ob * TILE);
    for (int i = threadIdx.x; i < TILE / 4; i += T) {
      float4 v = xi[i];
      v.x = __fmul_rn(v.x, c); v.y = __fmul_rn(v.y, c); v.z = __fmul_rn(v.z, c); v.w = __fmul_rn(v.w, c);
      yo[i] = v;
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(y + tile_of(k) * TILE, out + ob * TILE, TILE * 4);
      bulk_commit();
      if (k + S < my) {
        mbar_expect_tx(&bar[st_], TILE * 4);
        bulk_g2s(in + st_ * TILE, x + tile_of(k + S) * TILE, TILE * 4, &bar[st_]);
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_read<0>();
}

// K2 stride (interleaved) LDG variant
template <int T, int U, int HL, int HS>
__global__ void __launch_bounds__(T) k2_stride(const float4* x, float4* y, uint64_t nv, float c) {
  const uint64_t stride = (uint64_t)gridDim.x * T * U;
  for (uint64_t t = (uint64_t)blockIdx.x * T * U; t < nv; t += stride) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < nv) a[u] = ld<HL>(x + v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t v = t + u * T + threadIdx.x;
      if (v < nv) {
        float4 o = a[u];
        o.x = __fmul_rn(o.x, c); o.y = __fmul_rn(o.y, c); o.z = __fmul_rn(o.z, c); o.w = __fmul_rn(o.w, c);
        st<HS>(y + v, o);
      }
    }
  }
}

// ------------------------------------------------------------------ harness

struct Bufs {
  float *g, *r, *s, *flush;
  uint64_t n;
  size_t flush_n;
};

template <typename F>
float timeit(Bufs& b, F launch, int reps = 15) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<float> ts;
  for (int i = 0; i < reps + 3; ++i) {
    CK(cudaMemsetAsync(b.flush, i, b.flush_n * 4));
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (i >= 3) ts.push_back(ms);
  }
  CK(cudaGetLastError());
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

template <typename K>
int occ(K k, int T, size_t smem = 0) {
  int b = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, T, smem));
  return b;
}

int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 25557032ULL;
  n = n / 4096 * 4096;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  Bufs b;
  b.n = n;
  b.flush_n = (256u << 20) / 4;
  CK(cudaMalloc(&b.g, n * 4));
  CK(cudaMalloc(&b.r, n * 4));
  CK(cudaMalloc(&b.s, n * 4));
  CK(cudaMalloc(&b.flush, b.flush_n * 4));
  CK(cudaMemset(b.g, 0, n * 4));
  CK(cudaMemset(b.r, 0, n * 4));
  const double k1b = 16.0 * n, k2b = 8.0 * n;  // K1: 2 reads + 2 writes; K2: 1 + 1
  const uint64_t nv = n / 4;
  printf("n=%llu elems (%.1f MB/array), %d SMs\n", (unsigned long long)n, n * 4 / 1e6, sms);

#define RUN1(NAME, KER, T, U, HL, HS, OCCMUL)                                                    \
  {                                                                                            \
    auto kp = KER<T, U, HL, HS>;                                                               \
    int o = occ(kp, T);                                                                        \
    int grid = sms * o * OCCMUL;                                                               \
    float ms = timeit(b, [&] { kp<<<grid, T>>>((const float4*)b.g, (float4*)b.r, (float4*)b.s, \
                                               nv, 0.5f); });                                  \
    printf("K1 %-10s T=%4d U=%d HL=%d HS=%d occ=%d grid=%5d  %8.2f us  %7.1f GB/s\n", NAME, T, U, \
           HL, HS, o, grid, ms * 1e3, k1b / (ms * 1e-3) / 1e9);                                \
  }
  RUN1("chunk", k1_chunk, 256, 4, kStream, kStream, 1);
  RUN1("chunk", k1_chunk, 256, 4, kDefault, kDefault, 1);
  RUN1("chunk", k1_chunk, 256, 4, kNoAlloc, kNoAlloc, 1);
  RUN1("chunk", k1_chunk, 256, 4, kEvictLast, kStream, 1);
  RUN1("chunk", k1_chunk, 256, 2, kStream, kStream, 1);
  RUN1("chunk", k1_chunk, 256, 8, kStream, kStream, 1);
  RUN1("chunk", k1_chunk, 128, 4, kStream, kStream, 1);
  RUN1("chunk", k1_chunk, 512, 4, kStream, kStream, 1);
  RUN1("chunk", k1_chunk, 1024, 2, kStream, kStream, 1);
  RUN1("chunk", k1_chunk, 256, 4, kStream, kStream, 2);
  RUN1("chunk", k1_chunk, 256, 4, kNoAlloc, kDefault, 1);
  RUN1("stride", k1_stride, 256, 4, kStream, kStream, 1);
  RUN1("stride", k1_stride, 256, 4, kDefault, kDefault, 1);
  RUN1("stride", k1_stride, 256, 2, kStream, kStream, 1);
  RUN1("stride", k1_stride, 512, 2, kNoAlloc, kDefault, 1);
  {
    auto kp = k1_v8<256, 2>;
    int o = occ(kp, 256), grid = sms * o;
    float ms = timeit(b, [&] { kp<<<grid, 256>>>(b.g, b.r, b.s, n / 8, 0.5f); });
    printf("K1 v8         T=256 U=2 occ=%d grid=%5d  %8.2f us  %7.1f GB/s\n", o, grid, ms * 1e3,
           k1b / (ms * 1e-3) / 1e9);
  }
  {
    auto kp = k1_v8<256, 4>;
    int o = occ(kp, 256), grid = sms * o;
    float ms = timeit(b, [&] { kp<<<grid, 256>>>(b.g, b.r, b.s, n / 8, 0.5f); });
    printf("K1 v8         T=256 U=4 occ=%d grid=%5d  %8.2f us  %7.1f GB/s\n", o, grid, ms * 1e3,
           k1b / (ms * 1e-3) / 1e9);
  }
#define RUNTMA(T, TILE, S, CPS, INTER)                                                           \
  if ((2 * S * TILE + 4 * TILE) * 4 <= 227 * 1024) {                                           \
    auto kp = k1_tma<T, TILE, S, INTER>;                                                       \
    size_t smem = (2 * S * TILE + 4 * TILE) * 4;                                               \
    CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    int o = occ(kp, T, smem);                                                                  \
    int grid = sms * std::min(o, CPS);                                                         \
    uint64_t nt = n / TILE;                                                                    \
    float ms = timeit(b, [&] { kp<<<grid, T, smem>>>(b.g, b.r, b.s, nt, 0.5f); });            \
    printf("K1 tma T=%d TILE=%d S=%d I=%d smem=%zuKB occ=%d grid=%d  %8.2f us  %7.1f GB/s\n", T, \
           TILE, S, (int)INTER, smem / 1024, o, grid, ms * 1e3, k1b / (ms * 1e-3) / 1e9);      \
  }
  RUNTMA(256, 2048, 4, 8, false);
  RUNTMA(256, 4096, 3, 8, false);
  RUNTMA(256, 2048, 4, 8, true);
  RUNTMA(256, 4096, 3, 8, true);
  RUNTMA(256, 2048, 8, 8, true);
  RUNTMA(128, 1024, 6, 16, true);
  RUNTMA(256, 1024, 8, 16, true);
  RUNTMA(128, 2048, 4, 16, true);
  RUNTMA(512, 4096, 4, 8, true);

#define RUN2(NAME, T, U, HL, HS, OCCMUL)                                                        \
  {                                                                                            \
    auto kp = k2_chunk<T, U, HL, HS>;                                                          \
    int o = occ(kp, T);                                                                        \
    int grid = sms * o * OCCMUL;                                                               \
    float ms = timeit(b, [&] { kp<<<grid, T>>>((const float4*)b.s, (float4*)b.g, nv, 0.5f); }); \
    printf("K2 %-10s T=%4d U=%d HL=%d HS=%d occ=%d grid=%5d  %8.2f us  %7.1f GB/s\n", NAME, T, U, \
           HL, HS, o, grid, ms * 1e3, k2b / (ms * 1e-3) / 1e9);                                \
  }
  RUN2("chunk", 256, 4, kStream, kStream, 1);
  RUN2("chunk", 256, 4, kDefault, kDefault, 1);
  RUN2("chunk", 256, 8, kNoAlloc, kDefault, 1);
#define RUN2S(T, U, HL, HS, OCCMUL)                                                             \
  {                                                                                            \
    auto kp = k2_stride<T, U, HL, HS>;                                                         \
    int o = occ(kp, T);                                                                        \
    int grid = sms * o * OCCMUL;                                                               \
    float ms = timeit(b, [&] { kp<<<grid, T>>>((const float4*)b.s, (float4*)b.g, nv, 0.5f); }); \
    printf("K2 stride     T=%4d U=%d HL=%d HS=%d occ=%d grid=%5d  %8.2f us  %7.1f GB/s\n", T, U, \
           HL, HS, o, grid, ms * 1e3, k2b / (ms * 1e-3) / 1e9);                                \
  }
  RUN2S(256, 4, kDefault, kDefault, 1);
  RUN2S(256, 8, kDefault, kDefault, 1);
  RUN2S(256, 4, kNoAlloc, kDefault, 1);
  RUN2S(512, 4, kDefault, kDefault, 1);
#define RUN2TMA(T, TILE, S, CPS, INTER)                                                         \
  if ((S * TILE + 2 * TILE) * 4 <= 227 * 1024) {                                               \
    auto kp = k2_tma<T, TILE, S, INTER>;                                                       \
    size_t smem = (S * TILE + 2 * TILE) * 4;                                                   \
    CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    int o = occ(kp, T, smem);                                                                  \
    int grid = sms * std::min(o, CPS);                                                         \
    uint64_t nt = n / TILE;                                                                    \
    float ms = timeit(b, [&] { kp<<<grid, T, smem>>>(b.s, b.g, nt, 0.5f); });                 \
    printf("K2 tma T=%d TILE=%d S=%d I=%d smem=%zuKB occ=%d grid=%d  %8.2f us  %7.1f GB/s\n", T, \
           TILE, S, (int)INTER, smem / 1024, o, grid, ms * 1e3, k2b / (ms * 1e-3) / 1e9);      \
  }
  RUN2TMA(256, 4096, 4, 8, true);
  RUN2TMA(256, 4096, 6, 8, true);
  RUN2TMA(256, 2048, 8, 8, true);
  RUN2TMA(128, 2048, 4, 16, true);
  RUN2TMA(256, 8192, 4, 8, true);
  RUN2TMA(256, 4096, 4, 8, false);
  {
    auto kp = k2_v8<256, 4>;
    int o = occ(kp, 256), grid = sms * o;
    float ms = timeit(b, [&] { kp<<<grid, 256>>>(b.s, b.g, n / 8, 0.5f); });
    printf("K2 v8         T=256 U=4 occ=%d grid=%5d  %8.2f us  %7.1f GB/s\n", o, grid, ms * 1e3,
           k2b / (ms * 1e-3) / 1e9);
  }
  {
    float ms = timeit(b, [&] { cudaMemcpyAsync(b.g, b.s, n * 4, cudaMemcpyDeviceToDevice); });
    printf("K2 memcpyD2D                                      %8.2f us  %7.1f GB/s\n", ms * 1e3,
           k2b / (ms * 1e-3) / 1e9);
  }
  {
    float ms = timeit(b, [&] { cudaMemsetAsync(b.g, 0, n * 4); });
    printf("memset (write only, 4n B)                          %8.2f us  %7.1f GB/s\n", ms * 1e3,
           4.0 * n / (ms * 1e-3) / 1e9);
  }
  return 0;
}
