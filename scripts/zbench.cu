// zbench.cu — write-only (zero fill) throughput probe (not product code).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <algorithm>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int T>
__global__ void __launch_bounds__(T) zero_stg(float4* p, uint64_t nv) {
  const float4 z = make_float4(0, 0, 0, 0);
  for (uint64_t v = blockIdx.x * (uint64_t)T + threadIdx.x; v < nv; v += (uint64_t)gridDim.x * T) p[v] = z;
}
template <int T>
__global__ void __launch_bounds__(T) zero_stg_tiles(float4* p, uint64_t nv, uint32_t tile_v) {
  // interleaved tiles of tile_v vectors, like K2's none tiles
  const float4 z = make_float4(0, 0, 0, 0);
  const uint64_t ntiles = (nv + tile_v - 1) / tile_v;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x)
    for (uint32_t i = threadIdx.x; i < tile_v && t * tile_v + i < nv; i += T) p[t * tile_v + i] = z;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void zero_bulk(float* p, uint64_t n, uint32_t tile_bytes) {
  extern __shared__ __align__(128) float zs[];
  for (uint32_t i = threadIdx.x; i < tile_bytes / 4; i += blockDim.x) zs[i] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t te = tile_bytes / 4, ntiles = (n + te - 1) / te;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const uint64_t e0 = t * te; const uint32_t b = (uint32_t)((min(e0 + te, n) - e0) * 4);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + e0), "r"(smem_u32(zs)), "r"(b) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 25557032ULL; n = n / 4096 * 4096;
  float* p; CK(cudaMalloc(&p, n * 4)); float* fl; CK(cudaMalloc(&fl, 256 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto t = [&](const char* name, auto f) {
    std::vector<float> v;
    for (int i = 0; i < 13; ++i) { cudaMemset(fl, i, 256 << 20); cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 3) v.push_back(ms); }
    std::sort(v.begin(), v.end()); float ms = v[v.size() / 2];
    printf("%-34s %8.2f us %8.1f GB/s\n", name, ms * 1e3, n * 4 / (ms * 1e-3) / 1e9);
  };
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  t("cudaMemsetAsync", [&] { cudaMemsetAsync(p, 0, n * 4); });
  t("stg 148x256", [&] { zero_stg<256><<<sms, 256>>>((float4*)p, n / 4); });
  t("stg 148x1024", [&] { zero_stg<1024><<<sms, 1024>>>((float4*)p, n / 4); });
  t("stg 1184x256", [&] { zero_stg<256><<<sms * 8, 256>>>((float4*)p, n / 4); });
  t("stg tiles32K 148x256", [&] { zero_stg_tiles<256><<<sms, 256>>>((float4*)p, n / 4, 2048); });
  t("stg tiles32K 592x256", [&] { zero_stg_tiles<256><<<sms * 4, 256>>>((float4*)p, n / 4, 2048); });
  cudaFuncSetAttribute(zero_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  t("bulk 32K 148", [&] { zero_bulk<<<sms, 128, 32768>>>(p, n, 32768); });
  t("bulk 64K 148", [&] { zero_bulk<<<sms, 128, 65536>>>(p, n, 65536); });
  t("bulk 16K 296", [&] { zero_bulk<<<sms * 2, 128, 16384>>>(p, n, 16384); });
  t("bulk 4K 592", [&] { zero_bulk<<<sms * 4, 128, 4096>>>(p, n, 4096); });
  CK(cudaGetLastError());
  return 0;
}
