// CTA-pair (tcgen05 cta_group::2, M256 x N256 x K16) issue loop without data
// movement (random operands in a 4-stage ring of distinct 32 KB stages per
// CTA, as in umma_gemm2_kernel): the leader's MMA warp waits on a full
// barrier that a relay thread arrives once the multicast commit of the same
// stage S steps earlier has landed on the empty barriers.
//   mode 0: MMAs back to back (commit only at the end)
//   mode 1: relay through the LEADER's empty barrier only
//   mode 2: relay needs BOTH CTAs' empty barriers (peer relays to the leader's full barrier)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_06173_b200/csrc \
//        tools/mma_ring2.cu -o tools/mma_ring2 -lcuda
#include <cuda_bf16.h>

#include <cstdio>

#include "umma_gemm.cuh"

using namespace rwb::gemm;

template <int MODE, int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) ring2(int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t empty_bar[S], full_bar[S], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < S * 32768 / 4; i += blockDim.x) {
    uint32_t h = uint32_t(i + blockIdx.x * 65536) * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    const __nv_bfloat16 a = __float2bfloat16(float(h & 0xffff) / 65536.f - 0.5f);
    const __nv_bfloat16 b = __float2bfloat16(float(h >> 16) / 65536.f - 0.5f);
    reinterpret_cast<uint32_t*>(smem)[i] =
        uint32_t(*reinterpret_cast<const uint16_t*>(&a)) | (uint32_t(*reinterpret_cast<const uint16_t*>(&b)) << 16);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&empty_bar[i], 1);
      mbar_init(&full_bar[i], MODE == 2 ? 2 : 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  constexpr uint32_t idesc = make_idesc(256, 256, K_MAJOR, K_MAJOR);
  const uint32_t base = smem_u32(smem);
  if (warp == 0 && rank == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      const uint32_t ph = (i / S) & 1;
      if (MODE >= 1 && i >= S) {
        mbar_wait(&full_bar[s], ph ^ 1);
        tc_fence_after();
      }
      if (lane == 0) {
        const uint32_t sa = base + uint32_t(s) * 32768u, sb = sa + 16384u;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma2(tbase, make_desc(sa + k * 32, 16, 1024), make_desc(sb + k * 32, 16, 1024), idesc, 1u);
        if (MODE >= 1) tc_commit2_mc(&empty_bar[s]);
      }
      __syncwarp();
    }
    if (lane == 0) tc_commit2_mc(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x / 2] = t1 - t0;
  } else if (warp == 0 && rank == 1) {
    mbar_wait(&done, 0);  // the final multicast commit lands here too
  } else if (warp == 2 && MODE >= 1) {
    // relay: stage s free (commit landed here) -> the leader's full barrier for step i + S
    const uint32_t leader_full = mapa_rank0(smem_u32(&full_bar[0]));
    for (int i = 0; i + S < steps; ++i) {
      const int s = i % S;
      const uint32_t ph = (i / S) & 1;
      if (lane == 0 && (rank == 0 || MODE == 2)) {
        mbar_wait(&empty_bar[s], ph);
        if (rank == 0) mbar_arrive(&full_bar[s]);
        else mbar_arrive_cluster(leader_full + uint32_t(s) * 8u);
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

template <int MODE, int S>
void run() {
  const int steps = 20000, grid = 148;
  long long* d;
  cudaMalloc(&d, 74 * sizeof(long long));
  auto k = ring2<MODE, S>;
  const int sm = S * 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<grid, 128, sm>>>(100, d);
  cudaError_t err = cudaDeviceSynchronize();
  k<<<grid, 128, sm>>>(steps, d);
  err = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 74; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("pair mode %d  S=%d  cycles per M256 MMA %.1f  (%s)\n", MODE, S, double(mx) / (steps * 4.0),
         cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<0, 4>();
  run<1, 4>();
  run<1, 6>();
  run<2, 4>();
  run<2, 6>();
  return 0;
}
