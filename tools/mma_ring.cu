// tcgen05.mma issue loop variants (no data movement, random operands, whole
// GPU, cta_group::1 M128 N256 K16): what the GEMM main loop's per-k-block
// synchronisation costs on top of the raw 128 cycles per instruction.
//   mode 0: 4 MMAs per step, nothing else
//   mode 1: + tcgen05.commit to a ring barrier per step (nobody waits)
//   mode 2: + wait for the commit of step i-S before issuing step i (queue depth S steps)
//   mode 3: mode 2, the whole warp polls the barrier (as in the GEMM kernel)
//   mode 4: mode 3 + a second "producer" warp that relays each completion through a
//           second barrier (empty -> producer -> full -> MMA warp), as in the GEMM kernel
//   mode 5: mode 4 without tcgen05.fence::after_thread_sync
//   mode 6: mode 4 with a bare try_wait loop (no clock64 watchdog)
//   mode 7: mode 4, MMAs issued under elect.sync (no divergent lane-0 branch)
//   mode 8: mode 4, but one wait per two steps (a 128-deep K block per stage)
//   mode 9: mode 4 + four more warps polling a barrier that completes only at the end
//           (the GEMM's epilogue warps waiting for an accumulator)
//   mode 10: mode 9, the pollers back off with nanosleep between polls
//   mode 11: mode 4 + four warps reading the other TMEM accumulator (tcgen05.ld) nonstop
//   mode 12: mode 4 + four warps doing tanhf math nonstop (issue-slot competition)
//   mode 13: mode 4, each step's MMAs read the operands of its own ring stage
//            (4 x 48 KB of distinct smem, as in the GEMM) instead of one fixed stage
//   mode 14: mode 13, but the wait for step i+1 is issued after the first two MMAs of
//            step i (the barrier check overlaps queued MMAs instead of a drained queue)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2302_06173_b200/csrc \
//        tools/mma_ring.cu -o tools/mma_ring -lcuda
#include <cuda_bf16.h>

#include <cstdio>

#include "umma_gemm.cuh"

using namespace rwb::gemm;

template <int MODE, int S>
__global__ void __launch_bounds__(256, 1) ring(int steps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t empty_bar[S], full_bar[S], end_bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 4 * 49152 / 4; i += blockDim.x) {
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
      mbar_init(&full_bar[i], 1);
    }
    mbar_init(&end_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t idesc = make_idesc(128, 256, K_MAJOR, K_MAJOR);
  const uint32_t sa = smem_u32(smem), sb = sa + 16384;
  if (warp == 0 && MODE == 14) {
    const long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      const uint32_t so = uint32_t(s) * 49152u;
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
          tc_mma(tbase, make_desc(sa + so + k * 32, 16, 1024), make_desc(sb + so + k * 32, 16, 1024), idesc, 1u);
      }
      __syncwarp();
      const int i1 = i + 1;  // next step's stage must be ready before it is issued
      if (i1 >= S && i1 < steps) {
        mbar_wait(&full_bar[i1 % S], ((i1 / S) & 1) ^ 1);
        tc_fence_after();
      }
      if (lane == 0) {
#pragma unroll
        for (int k = 2; k < 4; ++k)
          tc_mma(tbase, make_desc(sa + so + k * 32, 16, 1024), make_desc(sb + so + k * 32, 16, 1024), idesc, 1u);
        tc_commit(&empty_bar[s]);
      }
      __syncwarp();
    }
    __shared__ uint64_t done14;
    if (lane == 0) {
      mbar_init(&done14, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      tc_commit(&done14);
    }
    __syncwarp();
    mbar_wait(&done14, 0);
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
    if (lane == 0) mbar_arrive(&end_bar);
  } else if (warp == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < steps; ++i) {
      const int s = i % S;
      const uint32_t ph = (i / S) & 1;
      if (MODE >= 2 && i >= S && (MODE != 8 || (i & 1) == 0)) {
        if (MODE == 6) {
          asm volatile(
              "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                  smem_u32(&full_bar[s])),
              "r"(ph ^ 1)
              : "memory");
        } else if (MODE >= 4) {
          mbar_wait(&full_bar[s], ph ^ 1);
        } else if (MODE == 3 || lane == 0) {
          mbar_wait(&empty_bar[s], ph ^ 1);
        }
        if (MODE != 5) tc_fence_after();
      }
      if (MODE == 8 && i >= S && (i & 1) == 1) {  // second half of a double step: no wait
      }
      uint32_t elected = lane == 0;
      if (MODE == 7) {
        asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(elected));
      }
      if (elected) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t so = MODE == 13 ? uint32_t(s) * 49152u : 0u;
          const uint64_t ad = make_desc(sa + so + k * 32, 16, 1024), bd = make_desc(sb + so + k * 32, 16, 1024);
          tc_mma(tbase, ad, bd, idesc, 1u);
        }
        if (MODE >= 1) tc_commit(&empty_bar[s]);
      }
      __syncwarp();
    }
    // wait until everything issued has completed: commit a final barrier
    __shared__ uint64_t done;
    if (lane == 0) {
      mbar_init(&done, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      tc_commit(&done);
    }
    __syncwarp();
    mbar_wait(&done, 0);
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
    if (lane == 0) mbar_arrive(&end_bar);
  } else if (warp == 1 && MODE >= 4) {
    // relay: completion of step i (empty) -> full for step i + S
    for (int i = 0; i + S < steps; ++i) {
      const int s = i % S;
      const uint32_t ph = (i / S) & 1;
      if (lane == 0) {
        mbar_wait(&empty_bar[s], ph);
        mbar_arrive(&full_bar[s]);
      }
      __syncwarp();
    }
  }
  else if (warp >= 4) {
    if (MODE == 11 || MODE == 12) {
      float accv = 0.f;
      uint32_t done = 0;
      int it = 0;
      while (!done) {
        if (MODE == 11) {
          float v[32];
          tmem_ld_32cols(tbase + (uint32_t((warp - 4) * 32) << 16) + 256u + uint32_t((it & 7) * 32), v);
#pragma unroll
          for (int j = 0; j < 32; ++j) accv += v[j];
        } else {
#pragma unroll 1
          for (int j = 0; j < 64; ++j) accv = tanhf(accv + 0.37f);
        }
        ++it;
        asm volatile(
            "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(&end_bar)), "r"(0u)
            : "memory");
      }
      if (accv == 12345.f) out[0] = 0;
    } else if (MODE == 9) {
      mbar_wait(&end_bar, 0);
    } else if (MODE == 10) {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(&end_bar)), "r"(0u)
            : "memory");
        if (!done) __nanosleep(2000);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

template <int MODE, int S>
void run() {
  const int steps = 20000, grid = 148;
  long long* d;
  cudaMalloc(&d, grid * sizeof(long long));
  auto k = ring<MODE, S>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 48 * 1024 + 1024);
  k<<<grid, 256, 4 * 48 * 1024 + 1024>>>(100, d);
  cudaError_t err = cudaDeviceSynchronize();
  k<<<grid, 256, 4 * 48 * 1024 + 1024>>>(steps, d);
  err = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mode %d  S=%2d  cycles/MMA %.1f  (%s)\n", MODE, S, double(mx) / (steps * 4.0), cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<0, 4>();
  run<1, 4>();
  run<2, 2>();
  run<2, 3>();
  run<2, 4>();
  run<2, 8>();
  run<3, 4>();
  run<3, 8>();
  run<4, 4>();
  run<4, 6>();
  run<4, 8>();
  run<5, 4>();
  run<6, 4>();
  run<7, 4>();
  run<8, 4>();
  run<9, 4>();
  run<10, 4>();
  run<11, 4>();
  run<12, 4>();
  run<13, 4>();
  run<14, 4>();
  return 0;
}
