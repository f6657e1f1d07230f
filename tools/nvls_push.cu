// NVLink SHARP multicast push probe (one process, N GPUs): can one survivor
// write the resolved state into every replacement's HBM at once through the
// NVSwitch, and at what rate?  Binds a cuMemCreate'd buffer of every device to
// one multicast object, maps the multicast address on device 0, and pushes a
// local source buffer with `multimem.st.global.v4.f32` from an SM kernel.
// Compares against a copy-engine peer copy (cudaMemcpyPeerAsync 0 -> 1).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/nvls_push.cu -o tools/nvls_push -lcuda
//   ./tools/nvls_push [ndev] [MiB]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char* s_ = nullptr;                                                        \
      cuGetErrorString(r_, &s_);                                                       \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_ ? s_ : "?");   \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)
#define CR(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__global__ void fill(uint32_t* p, uint64_t n, uint32_t seed) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = uint32_t(i * 2654435761u) ^ seed;
}
__global__ void checksum(const uint32_t* p, uint64_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    s += uint64_t(p[i]) * (i + 1);
  atomicAdd(out, s);
}
// push: 16 bytes per thread per iteration, multimem store to the multicast VA
__global__ void __launch_bounds__(512) push_multimem(const float4* __restrict__ src, uint64_t mc, uint64_t n16) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * blockDim.x) {
    const float4 v = __ldg(src + i);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 16 * i), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
  }
}
// plain SM stores to one peer (P2P mapping) for comparison
__global__ void __launch_bounds__(512) push_peer(const float4* __restrict__ src, float4* dst, uint64_t n16) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n16; i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = __ldg(src + i);
}

int main(int argc, char** argv) {
  int ndev = 0;
  CR(cudaGetDeviceCount(&ndev));
  const int n = argc > 1 ? std::atoi(argv[1]) : ndev;
  const uint64_t want = (argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4096ull) << 20;
  CK(cuInit(0));
  std::vector<CUdevice> dev(n);
  for (int d = 0; d < n; ++d) {
    CK(cuDeviceGet(&dev[d], d));
    int mcs = 0;
    CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[d]));
    if (!mcs) {
      std::printf("device %d: multicast not supported\n", d);
      return 1;
    }
    CR(cudaSetDevice(d));
    CR(cudaFree(nullptr));
  }
  CUmulticastObjectProp mp = {};
  mp.numDevices = n;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  mp.size = want;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const uint64_t size = (want + gran - 1) / gran * gran;
  mp.size = size;
  CUmemGenericAllocationHandle mc;
  CK(cuMulticastCreate(&mc, &mp));
  for (int d = 0; d < n; ++d) CK(cuMulticastAddDevice(mc, dev[d]));
  std::vector<CUmemGenericAllocationHandle> mem(n);
  std::vector<CUdeviceptr> ptr(n);
  for (int d = 0; d < n; ++d) {
    CR(cudaSetDevice(d));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t ag = 0;
    CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CK(cuMemCreate(&mem[d], size, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem[d], 0, size, 0));
    CK(cuMemAddressReserve(&ptr[d], size, gran, 0, 0));
    CK(cuMemMap(ptr[d], size, 0, mem[d], 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = d;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(ptr[d], size, &ad, 1));
    CR(cudaMemset(reinterpret_cast<void*>(ptr[d]), 0, size));
  }
  CR(cudaSetDevice(0));
  CUdeviceptr mcva = 0;
  CK(cuMemAddressReserve(&mcva, size, gran, 0, 0));
  CK(cuMemMap(mcva, size, 0, mc, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcva, size, &ad, 1));
  uint32_t* src = nullptr;
  CR(cudaMalloc(&src, size));
  fill<<<1184, 512>>>(src, size / 4, 77u);
  CR(cudaDeviceSynchronize());
  int sms = 0;
  CR(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CR(cudaEventCreate(&a));
  CR(cudaEventCreate(&b));
  for (int ctas : {sms, 2 * sms, 4 * sms}) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CR(cudaEventRecord(a));
      push_multimem<<<ctas, 512>>>(reinterpret_cast<const float4*>(src), mcva, size / 16);
      CR(cudaEventRecord(b));
      CR(cudaEventSynchronize(b));
      float ms = 0;
      CR(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    std::printf("multimem push n=%d ctas=%d: %.3f ms for %.2f GB -> %.1f GB/s per receiver\n", n, ctas, best,
                size / 1e9, size / (best * 1e-3) / 1e9);
  }
  CR(cudaGetLastError());
  // verify every device received the source
  unsigned long long* cs = nullptr;
  CR(cudaMallocManaged(&cs, sizeof(unsigned long long) * (n + 1)));
  for (int d = 0; d <= n; ++d) cs[d] = 0;
  CR(cudaSetDevice(0));
  checksum<<<1184, 512>>>(src, size / 4, cs + n);
  CR(cudaDeviceSynchronize());
  bool ok = true;
  for (int d = 0; d < n; ++d) {
    CR(cudaSetDevice(d));
    checksum<<<1184, 512>>>(reinterpret_cast<const uint32_t*>(ptr[d]), size / 4, cs + d);
    CR(cudaDeviceSynchronize());
    if (cs[d] != cs[n]) ok = false;
  }
  std::printf("multicast contents %s on all %d devices\n", ok ? "MATCH" : "DIFFER", n);
  // copy-engine and SM-store baselines 0 -> 1
  CR(cudaSetDevice(0));
  if (n > 1) {
    int can = 0;
    CR(cudaDeviceCanAccessPeer(&can, 0, 1));
    if (can) cudaDeviceEnablePeerAccess(1, 0);
    cudaGetLastError();
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CR(cudaEventRecord(a));
      CR(cudaMemcpyPeerAsync(reinterpret_cast<void*>(ptr[1]), 1, src, 0, size));
      CR(cudaEventRecord(b));
      CR(cudaEventSynchronize(b));
      float ms = 0;
      CR(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    std::printf("copy engine 0->1: %.3f ms -> %.1f GB/s\n", best, size / (best * 1e-3) / 1e9);
    // SM stores through the unicast mapping of device 1's buffer
    CUmemAccessDesc pd = {};
    pd.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    pd.location.id = 0;
    pd.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(ptr[1], size, &pd, 1));
    best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CR(cudaEventRecord(a));
      push_peer<<<2 * sms, 512>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(ptr[1]), size / 16);
      CR(cudaEventRecord(b));
      CR(cudaEventSynchronize(b));
      float ms = 0;
      CR(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    std::printf("SM stores 0->1: %.3f ms -> %.1f GB/s\n", best, size / (best * 1e-3) / 1e9);
  }
  return ok ? 0 : 2;
}
