// nvls_probe.cu — what the B200 box offers for an NVSwitch-multicast
// collective (probe, not product):
//   1. CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED;
//   2. a driver-API multicast object over this one device, memory bound to
//      it, and multimem.ld_reduce / multimem.st through the multicast VA;
//   3. a 1-rank NCCL communicator: ncclMemAlloc + symmetric window +
//      ncclDevCommCreate(lsaMultimem) and the window's LSA / multimem
//      pointers as a kernel sees them.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o nvls_probe
//        nvls_probe.cu -I$NCCL/include -L$NCCL/lib -l:libnccl.so.2 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CU(x)                                                             \
  do {                                                                    \
    CUresult e_ = (x);                                                    \
    if (e_ != CUDA_SUCCESS) {                                             \
      const char* s_ = nullptr;                                           \
      cuGetErrorString(e_, &s_);                                          \
      printf("  FAIL %s -> %d %s\n", #x, (int)e_, s_ ? s_ : "?");         \
      return 1;                                                           \
    }                                                                     \
  } while (0)
#define RT(x)                                                             \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) {                                              \
      printf("  FAIL %s -> %s\n", #x, cudaGetErrorString(e_));            \
      return 1;                                                           \
    }                                                                     \
  } while (0)
#define NC(x)                                                             \
  do {                                                                    \
    ncclResult_t e_ = (x);                                                \
    if (e_ != ncclSuccess) {                                              \
      printf("  FAIL %s -> %s (%s)\n", #x, ncclGetErrorString(e_),        \
             ncclGetLastError(nullptr));                                  \
      return 1;                                                           \
    }                                                                     \
  } while (0)

__global__ void mm_kernel(float* mc, float* mc_out, int n4) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float a, b, c, d;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
               : "l"(mc + 4 * i)
               : "memory");
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc_out + 4 * i),
               "f"(a * 2.f), "f"(b * 2.f), "f"(c * 2.f), "f"(d * 2.f)
               : "memory");
}

__global__ void ptr_kernel(ncclWindow_t w, ncclDevComm dc, void** out) {
  out[0] = ncclGetLocalPointer(w, 0);
  out[1] = ncclGetLsaPointer(w, 0, 0);
  out[2] = dc.lsaMultimem.mcBasePtr ? ncclGetLsaMultimemPointer(w, 0, dc) : nullptr;
}

static int driver_multicast_try(int dev, CUmemAllocationHandleType ht, const char* hname) {
  CUdevice d;
  CU(cuDeviceGet(&d, dev));
  const size_t n = 1 << 20;  // floats
  CUmulticastObjectProp mp{};
  mp.numDevices = 1;
  mp.size = n * 4;
  mp.handleTypes = ht;
  size_t gran = 0, gmin = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CU(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  mp.size = (mp.size + gmin - 1) / gmin * gmin;
  printf("[%s] multicast granularity recommended %zu minimum %zu, size %zu\n", hname, gran, gmin,
         mp.size);
  CUmemGenericAllocationHandle mh, ph;
  CU(cuMulticastCreate(&mh, &mp));
  CU(cuMulticastAddDevice(mh, d));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = ht;
  CU(cuMemCreate(&ph, mp.size, &ap, 0));
  CU(cuMulticastBindMem(mh, 0, ph, 0, mp.size, 0));
  CUdeviceptr uc, mcp;
  CU(cuMemAddressReserve(&uc, mp.size, gmin, 0, 0));
  CU(cuMemMap(uc, mp.size, 0, ph, 0));
  CU(cuMemAddressReserve(&mcp, mp.size, gmin, 0, 0));
  CU(cuMemMap(mcp, mp.size, 0, mh, 0));
  CUmemAccessDesc acc{};
  acc.location = ap.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(uc, mp.size, &acc, 1));
  CU(cuMemSetAccess(mcp, mp.size, &acc, 1));
  float* h = (float*)malloc(n * 4);
  for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 1000) * 0.5f;
  RT(cudaMemcpy((void*)uc, h, n * 4, cudaMemcpyHostToDevice));
  mm_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)mcp, (float*)mcp, (int)(n / 4));
  RT(cudaGetLastError());
  RT(cudaDeviceSynchronize());
  float* o = (float*)malloc(n * 4);
  RT(cudaMemcpy(o, (void*)uc, n * 4, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < n; ++i) bad += o[i] != h[i] * 2.f;
  printf("[%s] driver multicast 1 device: ld_reduce + st through the multicast VA: %s (%zu bad)\n",
         hname, bad ? "WRONG" : "ok", bad);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 20; ++it)
    mm_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)mcp, (float*)mcp, (int)(n / 4));
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("[%s] multimem ld_reduce+st 4 MB: %.2f us per launch\n", hname, ms * 1000 / 20);
  return 0;
}

static int driver_multicast(int dev) {
  CUdevice d;
  CU(cuDeviceGet(&d, dev));
  int mc = 0;
  CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
  int fab = 0;
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
  printf("multicast_supported=%d fabric_handles=%d\n", mc, fab);
  if (!mc) return 0;
  int rc = driver_multicast_try(dev, CU_MEM_HANDLE_TYPE_NONE, "none");
  rc |= driver_multicast_try(dev, CU_MEM_HANDLE_TYPE_FABRIC, "fabric");
  rc |= driver_multicast_try(dev, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, "posix_fd");
  return rc;
}

static int nccl_devcomm(int dev) {
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  ncclComm_t comm;
  NC(ncclCommInitRank(&comm, 1, id, 0));
  int ver = 0;
  ncclGetVersion(&ver);
  printf("nccl %d, 1-rank communicator up\n", ver);
  void* buf = nullptr;
  const size_t bytes = 64 << 20;
  NC(ncclMemAlloc(&buf, bytes));
  ncclWindow_t win;
  NC(ncclCommWindowRegister(comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC));
  for (int want_mm = 1; want_mm >= 0; --want_mm) {
    ncclDevCommRequirements req{};
    req.lsaMultimem = want_mm;
    req.lsaBarrierCount = 4;
    ncclDevComm dc;
    ncclResult_t r = ncclDevCommCreate(comm, &req, &dc);
    printf("ncclDevCommCreate(lsaMultimem=%d): %s %s\n", want_mm, ncclGetErrorString(r),
           r ? ncclGetLastError(comm) : "");
    if (r != ncclSuccess) continue;
    printf("  devcomm rank %d nRanks %d lsaSize %d lsaRank %d mcBase %p\n", dc.rank, dc.nRanks,
           dc.lsaSize, dc.lsaRank, dc.lsaMultimem.mcBasePtr);
    void** d_out;
    RT(cudaMalloc(&d_out, 3 * sizeof(void*)));
    ptr_kernel<<<1, 1>>>(win, dc, d_out);
    RT(cudaDeviceSynchronize());
    void* p[3];
    RT(cudaMemcpy(p, d_out, sizeof(p), cudaMemcpyDeviceToHost));
    printf("  buf %p local %p lsa[0] %p multimem %p\n", buf, p[0], p[1], p[2]);
    if (p[2]) {
      const size_t n = 1 << 20;
      float* h = (float*)malloc(n * 4);
      for (size_t i = 0; i < n; ++i) h[i] = (float)(i % 777) * 0.25f;
      RT(cudaMemcpy(buf, h, n * 4, cudaMemcpyHostToDevice));
      mm_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)p[2], (float*)p[2], (int)(n / 4));
      RT(cudaGetLastError());
      RT(cudaDeviceSynchronize());
      float* o = (float*)malloc(n * 4);
      RT(cudaMemcpy(o, buf, n * 4, cudaMemcpyDeviceToHost));
      size_t bad = 0;
      for (size_t i = 0; i < n; ++i) bad += o[i] != h[i] * 2.f;
      printf("  nccl lsa multimem ld_reduce + st: %s (%zu bad)\n", bad ? "WRONG" : "ok", bad);
    }
    cudaFree(d_out);
    NC(ncclDevCommDestroy(comm, &dc));
  }
  NC(ncclCommWindowDeregister(comm, win));
  NC(ncclMemFree(buf));
  NC(ncclCommDestroy(comm));
  return 0;
}

int main() {
  RT(cudaSetDevice(0));
  RT(cudaFree(0));
  CU(cuInit(0));
  int rc = driver_multicast(0);
  printf("driver probe rc=%d\n", rc);
  rc = nccl_devcomm(0);
  printf("nccl probe rc=%d\n", rc);
  return 0;
}
