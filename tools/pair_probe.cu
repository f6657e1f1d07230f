// Pipeline probe of the parked CTA-pair GEMM (umma_gemm2_kernel):
//   -DRWB_PAIR_EXPERIMENT=1  instrumented (wait cycles per role)
//   -DRWB_PAIR_EXPERIMENT=2  + no TMA after the first fill (MMA + sync only)
#include <cuda_bf16.h>

#include <cstdio>

#include "umma_gemm_host.h"

using namespace rwb::gemm;

int main() {
  const int M = 8192, N = 8192, K = 8192;
  __nv_bfloat16 *A, *B, *O;
  cudaMalloc(&A, size_t(M) * K * 2);
  cudaMalloc(&B, size_t(N) * K * 2);
  cudaMalloc(&O, size_t(M) * N * 2);
  cudaMemset(A, 0, size_t(M) * K * 2);
  cudaMemset(B, 0, size_t(N) * K * 2);
  EpiArgs ep{O, N, nullptr, nullptr, 0};
  for (int pair = 0; pair < 2; ++pair) {
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      long long z[148][4] = {};
      cudaMemcpyToSymbol(g_pair_dbg, z, sizeof(z));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      int e = pair ? launch2<256, K_MAJOR, K_MAJOR, EPI_BF16>(A, K, B, K, M, N, K, ep, 0)
                   : launch<256, K_MAJOR, K_MAJOR, EPI_BF16>(A, K, B, K, M, N, K, ep, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (e || err) printf("error %d %d\n", e, int(err));
      best = ms < best ? ms : best;
      if (pair && r == 3) {
        cudaMemcpyFromSymbol(z, g_pair_dbg, sizeof(z));
        double s[4] = {};
        int nl = 0;
        for (int i = 0; i < 148; i += 2) {
          ++nl;
          for (int j = 0; j < 3; ++j) s[j] += z[i][j];
        }
        for (int i = 0; i < 148; ++i) s[3] += z[i][3];
        const double n_instr = double(M) / 256 * N / 256 * K / 16 / 74;
        printf("leader avg: wait_full %.0f  wait_tempty %.0f  loop %.0f cycles; instr/leader %.0f -> %.1f cyc/instr; "
               "producer wait_empty avg %.0f\n",
               s[0] / nl, s[1] / nl, s[2] / nl, n_instr, s[2] / nl / n_instr, s[3] / 148);
      }
    }
    printf("%s %d^3: %.3f ms  %.1f TFLOP/s\n", pair ? "PAIR" : "single", M, best, 2.0 * M * N * K / (best * 1e-3) / 1e12);
  }
  return 0;
}
