// Raw tcgen05.mma issue rate, no data movement: cycles per instruction for
// cta_group::1 (M=128) and cta_group::2 (M=256 over a CTA pair) at N=128/256,
// operands SS from zeroed smem, whole GPU loaded (74 clusters of 2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_06173_b200/csrc \
//        tools/mma_rate.cu -o tools/mma_rate -lcuda
#include <cuda_bf16.h>

#include <cstdio>

#include "umma_gemm.cuh"

using namespace rwb::gemm;

__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG, int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_rate(int iters, long long* out, int rnd) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) {
    uint32_t w = 0;
    if (rnd) {  // two random bf16 in [-0.5, 0.5): real-data switching activity
      uint32_t h = uint32_t(i + blockIdx.x * 65536) * 2654435761u;
      h ^= h >> 15;
      h *= 2246822519u;
      h ^= h >> 13;
      const __nv_bfloat16 a = __float2bfloat16(float(h & 0xffff) / 65536.f - 0.5f);
      const __nv_bfloat16 b = __float2bfloat16(float(h >> 16) / 65536.f - 0.5f);
      w = uint32_t(*reinterpret_cast<const uint16_t*>(&a)) | (uint32_t(*reinterpret_cast<const uint16_t*>(&b)) << 16);
    }
    reinterpret_cast<uint32_t*>(smem)[i] = w;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                   "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  csync();
  tc_fence_after();
  const bool issuer = (CG == 1) || crank() == 0;
  if (warp == 0 && issuer) {
    constexpr uint32_t idesc = make_idesc(CG == 2 ? 256 : 128, N, K_MAJOR, K_MAJOR);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    long long t0 = clock64();
    if (lane == 0) {
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = make_desc(sa + k * 32, 16, 1024), bd = make_desc(sb + k * 32, 16, 1024);
          if constexpr (CG == 2) {
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
                "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
                : "memory");
          } else {
            tc_mma(tbase, ad, bd, idesc, 1u);
          }
        }
      }
      if constexpr (CG == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"(uint16_t(3))
            : "memory");
      else
        tc_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  } else if (warp == 0 && CG == 2) {
    mbar_wait(&bar, 0);  // the multicast commit arrives here too
  }
  tc_fence_before();
  __syncthreads();
  csync();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

template <int CG, int N>
void run(const char* name, int rnd) {
  const int iters = 20000, grid = 148;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  cudaMemset(d, 0, grid * sizeof(long long));
  auto k = mma_rate<CG, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  k<<<grid, 128, 66 * 1024>>>(100, d, rnd);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, 66 * 1024>>>(iters, d, rnd);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double n_instr = double(iters) * 4;
  const double flop = n_instr * 2.0 * (CG == 2 ? 256 : 128) * N * 16 * (CG == 2 ? grid / 2 : grid);
  printf("%-28s %s err=%d  cycles/instr(issuer)=%.1f  %.3f ms  %.1f TFLOP/s\n", name, rnd ? "random" : "zeros ", int(err), double(mx) / n_instr,
         ms, flop / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  for (int rnd = 0; rnd < 2; ++rnd) {
    run<1, 256>("cta_group::1 M128 N256", rnd);
    run<1, 128>("cta_group::1 M128 N128", rnd);
    run<2, 256>("cta_group::2 M256 N256", rnd);
    run<2, 128>("cta_group::2 M256 N128", rnd);
  }
  return 0;
}
