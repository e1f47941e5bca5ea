// zcopy_probe.cu — PCIe design probe for the host-buffer sync path (not
// product code).  Compares, for a ResNet-50-sized fp32 vector (102 MB):
//   ce_h2d / ce_d2h / ce_both   copy engines (cudaMemcpyAsync), both
//                               directions on two streams at once
//   zc_h2d                      kernel: LDG.128 from mapped pinned host memory
//                               -> STG to HBM
//   zc_d2h                      kernel: HBM -> STG.128 to mapped host memory
//   zc_both                     kernel: host -> host through the SMs (the
//                               shape of a fused K1F that reads g from and
//                               writes out to host buffers; r stays in HBM)
//   zc_both_r                   zc_both plus the HBM residual read/write
// for several grid sizes / unroll depths.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zcopy_probe zcopy_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

template <int U>
__global__ void copy_kernel(const float4* __restrict__ src, float4* __restrict__ dst, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nvec; base += stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x;
      if (i < nvec) v[u] = __ldcs(src + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x;
      if (i < nvec) __stcs(dst + i, v[u]);
    }
  }
}

// g (host) + c * r (HBM) -> out (host), r = c  (the K1F K=1 shape).
template <int U>
__global__ void k1f_host_kernel(const float4* __restrict__ g, float4* __restrict__ r,
                                float4* __restrict__ out, uint64_t nvec, float coeff) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nvec; base += stride) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x;
      if (i < nvec) {
        a[u] = __ldcs(g + i);
        b[u] = __ldcs(r + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x;
      if (i < nvec) {
        float4 c;
        c.x = __fadd_rn(a[u].x, __fmul_rn(coeff, b[u].x));
        c.y = __fadd_rn(a[u].y, __fmul_rn(coeff, b[u].y));
        c.z = __fadd_rn(a[u].z, __fmul_rn(coeff, b[u].z));
        c.w = __fadd_rn(a[u].w, __fmul_rn(coeff, b[u].w));
        __stcs(out + i, c);
        __stcs(r + i, make_float4(0.f, 0.f, 0.f, 0.f));
      }
    }
  }
}

static float time_it(cudaStream_t s, int reps, void (*f)(void*), void* ctx) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f(ctx);
  cudaDeviceSynchronize();
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) f(ctx);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / reps;
}

struct Ctx {
  float *h_in, *h_out, *d_a, *d_b, *d_r;
  uint64_t n;
  cudaStream_t s0, s1;
  int grid, mode, unroll;
};

template <int U>
static void launch_u(Ctx* c) {
  const uint64_t nvec = c->n / 4;
  switch (c->mode) {
    case 0: copy_kernel<U><<<c->grid, 256, 0, c->s0>>>((const float4*)c->h_in, (float4*)c->d_a, nvec); break;
    case 1: copy_kernel<U><<<c->grid, 256, 0, c->s0>>>((const float4*)c->d_b, (float4*)c->h_out, nvec); break;
    case 2: copy_kernel<U><<<c->grid, 256, 0, c->s0>>>((const float4*)c->h_in, (float4*)c->h_out, nvec); break;
    default:
      k1f_host_kernel<U><<<c->grid, 256, 0, c->s0>>>((const float4*)c->h_in, (float4*)c->d_r,
                                                     (float4*)c->h_out, nvec, 0.5f);
  }
}

static void run_kernel(void* p) {
  Ctx* c = (Ctx*)p;
  switch (c->unroll) {
    case 1: launch_u<1>(c); break;
    case 2: launch_u<2>(c); break;
    case 4: launch_u<4>(c); break;
    default: launch_u<8>(c); break;
  }
}

static void ce_h2d(void* p) {
  Ctx* c = (Ctx*)p;
  cudaMemcpyAsync(c->d_a, c->h_in, c->n * 4, cudaMemcpyHostToDevice, c->s0);
}
static void ce_d2h(void* p) {
  Ctx* c = (Ctx*)p;
  cudaMemcpyAsync(c->h_out, c->d_b, c->n * 4, cudaMemcpyDeviceToHost, c->s0);
}
static cudaEvent_t g_join;
static void ce_both(void* p) {
  Ctx* c = (Ctx*)p;
  cudaEventRecord(g_join, c->s0);
  cudaStreamWaitEvent(c->s1, g_join, 0);
  cudaMemcpyAsync(c->d_a, c->h_in, c->n * 4, cudaMemcpyHostToDevice, c->s0);
  cudaMemcpyAsync(c->h_out, c->d_b, c->n * 4, cudaMemcpyDeviceToHost, c->s1);
  cudaEventRecord(g_join, c->s1);
  cudaStreamWaitEvent(c->s0, g_join, 0);
}

int main(int argc, char** argv) {
  Ctx c;
  c.n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 25557032ull / 4 * 4;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaHostAlloc(&c.h_in, c.n * 4, cudaHostAllocDefault));
  CK(cudaHostAlloc(&c.h_out, c.n * 4, cudaHostAllocDefault));
  CK(cudaMalloc(&c.d_a, c.n * 4));
  CK(cudaMalloc(&c.d_b, c.n * 4));
  CK(cudaMalloc(&c.d_r, c.n * 4));
  for (uint64_t i = 0; i < c.n; ++i) c.h_in[i] = (float)(i % 1000);
  CK(cudaMemset(c.d_b, 0, c.n * 4));
  CK(cudaMemset(c.d_r, 0, c.n * 4));
  CK(cudaStreamCreateWithFlags(&c.s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&c.s1, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&g_join, cudaEventDisableTiming));
  const double mb = c.n * 4 / 1e6;
  printf("n=%llu (%.1f MB per direction), %d SMs\n", (unsigned long long)c.n, mb, sms);
  float t;
  t = time_it(c.s0, 10, ce_h2d, &c);
  printf("ce_h2d   %.3f ms  %.1f GB/s\n", t, mb / t);
  t = time_it(c.s0, 10, ce_d2h, &c);
  printf("ce_d2h   %.3f ms  %.1f GB/s\n", t, mb / t);
  t = time_it(c.s0, 10, ce_both, &c);
  printf("ce_both  %.3f ms  %.1f GB/s per direction\n", t, mb / t);
  const char* names[] = {"zc_h2d", "zc_d2h", "zc_both", "zc_k1f"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int mult : {1, 2, 4, 8}) {
      for (int u : {1, 2, 4, 8}) {
        c.mode = mode;
        c.grid = sms * mult;
        c.unroll = u;
        t = time_it(c.s0, 10, run_kernel, &c);
        CK(cudaGetLastError());
        printf("%-8s grid %4d unroll %d  %.3f ms  %.1f GB/s per direction\n", names[mode], c.grid, u, t,
               mb / t);
      }
    }
  }
  // hybrid: copy engines move a fraction f of both directions while a
  // zero-copy kernel on a third stream moves the rest (host -> host via SMs)
  {
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b, j1, j2;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventCreateWithFlags(&j1, cudaEventDisableTiming); cudaEventCreateWithFlags(&j2, cudaEventDisableTiming);
    for (double f : {1.0, 0.95, 0.9, 0.85, 0.8, 0.7}) {
      const uint64_t nce = (uint64_t)(c.n * f) / 1024 * 1024, nzc = c.n - nce;
      float best = 1e9;
      for (int rep = 0; rep < 8; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(a, c.s0);
        cudaStreamWaitEvent(c.s1, a, 0);
        cudaStreamWaitEvent(s2, a, 0);
        cudaMemcpyAsync(c.d_a, c.h_in, nce * 4, cudaMemcpyHostToDevice, c.s0);
        cudaMemcpyAsync(c.h_out, c.d_b, nce * 4, cudaMemcpyDeviceToHost, c.s1);
        if (nzc) copy_kernel<1><<<sms, 256, 0, s2>>>((const float4*)(c.h_in + nce), (float4*)(c.h_out + nce), nzc / 4);
        cudaEventRecord(j1, c.s1); cudaEventRecord(j2, s2);
        cudaStreamWaitEvent(c.s0, j1, 0); cudaStreamWaitEvent(c.s0, j2, 0);
        cudaEventRecord(b, c.s0);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("hybrid f=%.2f  %.3f ms  (%.1f GB/s per direction)\n", f, best, mb / best);
    }
  }
  // correctness of the zero-copy k1f path: out = g + 0.5 * 0 = g
  c.mode = 3; c.grid = sms; c.unroll = 4;
  CK(cudaMemset(c.d_r, 0, c.n * 4));
  run_kernel(&c);
  CK(cudaStreamSynchronize(c.s0));
  uint64_t bad = 0;
  for (uint64_t i = 0; i < c.n; ++i) bad += c.h_out[i] != c.h_in[i];
  printf("zc_k1f check: %llu mismatches\n", (unsigned long long)bad);
  return 0;
}
