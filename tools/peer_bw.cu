// NVLink write bandwidth GPU0 -> GPU1 by method (peer access enabled):
//   ce      cudaMemcpyPeerAsync (copy engines)
//   tma     kernel: global -> smem (TMA bulk) -> peer (cp.async.bulk smem->global)
//   st128   kernel: 128-bit loads, 128-bit stores straight to the peer
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/peer_bw.cu -o tools/peer_bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int SLOT, int STAGES>
__global__ void __launch_bounds__(128, 1) tma_push(const char* __restrict__ src, char* __restrict__ dst, size_t n) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar[STAGES];
  const size_t tiles = n / SLOT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t it = 0;
  for (size_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
    const int st = it % STAGES;
    unsigned char* buf = sm + st * SLOT;
    if (it >= STAGES) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(SLOT)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf)),
        "l"(src + t * SLOT), "r"(SLOT), "r"(smem_u32(&bar[st]))
        : "memory");
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
            smem_u32(&bar[st])),
        "r"((it / STAGES) & 1u)
        : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * SLOT),
                 "r"(smem_u32(buf)), "r"(SLOT)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void st128_push(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int main() {
  const size_t n = size_t(6) << 30;  // 6 GiB
  char *a, *b;
  cudaSetDevice(1);
  cudaMalloc(&b, n);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&a, n);
  cudaMemset(a, 1, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-28s %8.2f ms  %7.1f GB/s  (%s)\n", name, best, n / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  timeit("ce cudaMemcpyPeerAsync", [&] { cudaMemcpyPeerAsync(b, 1, a, 0, n); });
  cudaFuncSetAttribute(tma_push<8192, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 8192);
  cudaFuncSetAttribute(tma_push<32768, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  cudaFuncSetAttribute(tma_push<16384, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 16384);
  for (int g : {148, 296, 592})
    timeit((std::string("tma 8K x3 grid ") + std::to_string(g)).c_str(),
           [&] { tma_push<8192, 3><<<g, 128, 3 * 8192>>>(a, b, n); });
  for (int g : {148, 296})
    timeit((std::string("tma 32K x4 grid ") + std::to_string(g)).c_str(),
           [&] { tma_push<32768, 4><<<g, 128, 4 * 32768>>>(a, b, n); });
  timeit("tma 16K x6 grid 148", [&] { tma_push<16384, 6><<<148, 128, 6 * 16384>>>(a, b, n); });
  for (int g : {148 * 4, 148 * 8, 148 * 16})
    timeit((std::string("st128 grid ") + std::to_string(g)).c_str(),
           [&] { st128_push<<<g, 256>>>(reinterpret_cast<uint4*>(a), reinterpret_cast<uint4*>(b), n / 16); });
  return 0;
}
