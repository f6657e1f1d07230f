// Sustained-load pipeline probe of the replay GEMMs (random bf16 data, the
// replay's forward and dgrad shapes), single-CTA and CTA-pair kernels:
// TFLOP/s over ~2 s of back-to-back launches (the board settles at its power
// cap), then one instrumented launch: cycles per MMA instruction, the MMA
// warp's wait on full (data) / tempty (epilogue) barriers, and the SM clock
// implied by the loop cycles.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -DRWB_PAIR_EXPERIMENT=1 \
//        [-DRWB_GEMM_STAGES=4] [-DRWB_GEMM2_STAGES=6] -I paper_2302_06173_b200/csrc \
//        -o tools/gemm_probe tools/gemm_probe.cu -lcuda
#include <cuda_bf16.h>

#include <chrono>
#include <cstdio>

#include "umma_gemm_host.h"

using namespace rwb::gemm;
#ifndef RWB_PAIR_EXPERIMENT  // uninstrumented build: timing only
__device__ long long g_pair_dbg[148][4];
#endif

__global__ void fill(__nv_bfloat16* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = __float2bfloat16((float(h & 0xffff) / 65536.f - 0.5f) * scale);
  }
}

template <bool PAIR, int AM, int BMJ, int EPI, int MH = 1>
void probe(const char* name, int M, int N, int K, double secs) {
  __nv_bfloat16 *A, *B, *O, *Y;
  float* bias;
  cudaMalloc(&A, size_t(M) * K * 2);
  cudaMalloc(&B, size_t(N) * K * 2);
  cudaMalloc(&O, size_t(M) * N * 4);
  cudaMalloc(&Y, size_t(M) * N * 2);
  cudaMalloc(&bias, size_t(N) * 4);
  fill<<<1184, 256>>>(A, size_t(M) * K, 1, 1.f);
  fill<<<1184, 256>>>(B, size_t(N) * K, 2, 0.05f);
  fill<<<1184, 256>>>(Y, size_t(M) * N, 3, 1.f);
  cudaMemset(bias, 0, size_t(N) * 4);
  EpiArgs ep{O, N, bias, Y, N};
  const int64_t lda = AM == K_MAJOR ? K : M, ldb = BMJ == K_MAJOR ? K : N;
  auto run = [&] {
    return PAIR ? launch2<256, AM, BMJ, EPI, MH>(A, lda, B, ldb, M, N, K, ep, 0)
                : launch<256, AM, BMJ, EPI>(A, lda, B, ldb, M, N, K, ep, 0);
  };
  run();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // sustained
  int n = 0;
  auto t0 = std::chrono::steady_clock::now();
  cudaEventRecord(e0);
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < secs) {
    for (int i = 0; i < 20; ++i) run();
    n += 20;
    cudaDeviceSynchronize();  // keep the host near the queue head
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double tf = 2.0 * M * N * K * n / (ms * 1e-3) / 1e12;
  // one instrumented launch, still hot
  long long z[148][4] = {};
  cudaMemcpyToSymbol(g_pair_dbg, z, sizeof(z));
#ifdef RWB_PAIR_EXPERIMENT
  cudaMemcpyToSymbol(g_epi_dbg, z, sizeof(z));
#endif
  cudaEventRecord(e0);
  run();
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms1;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaMemcpyFromSymbol(z, g_pair_dbg, sizeof(z));
  long long ze[148][4] = {};
#ifdef RWB_PAIR_EXPERIMENT
  cudaMemcpyFromSymbol(ze, g_epi_dbg, sizeof(ze));
#endif
  double es[4] = {};
  for (int i = 0; i < 148; ++i)
    for (int j = 0; j < 4; ++j) es[j] += ze[i][j];
  double s[4] = {};
  int nl = 0;
  const int step = PAIR ? 2 : 1;
  for (int i = 0; i < 148; i += step) {
    ++nl;
    for (int j = 0; j < 3; ++j) s[j] += z[i][j];
  }
  for (int i = 0; i < 148; ++i) s[3] += z[i][3];
  const int pm = 256 * MH;
  const double tiles = PAIR ? double((M + pm - 1) / pm) * ((N + 255) / 256) : double((M + 127) / 128) * ((N + 255) / 256);
  const double instr = tiles * ((K + 63) / 64) * 4 * MH / nl;  // per-SM MMA instructions (pair: M256 each)
  const double loop = s[2] / nl;
  printf("%-6s %-28s sustained %7.1f TFLOP/s (%d launches, %.3f ms each) | last %.3f ms: %.1f cyc/MMA (ideal 128), "
         "wait_full %.1f%%, wait_tempty %.1f%%, producer wait_empty %.1f%%, SM clock ~%.0f MHz, %.3f TF/MHz %s\n",
         PAIR ? (MH == 2 ? "WIDE" : "PAIR") : "single", name, tf, n, ms / n, ms1, loop / instr, 100 * s[0] / nl / loop,
         100 * s[1] / nl / loop, 100 * s[3] / 148 / loop, loop / (ms1 * 1e3),
         2.0 * M * N * K / (ms1 * 1e-3) / 1e12 / (loop / (ms1 * 1e3)), err ? cudaGetErrorString(err) : "");
  if (es[0] > 0)
    printf("       epilogue (warp 4): %.0f cycles per CTA; waiting for buffers / input %.1f%%, TMEM loads %.1f%%, "
           "column sums %.1f%%\n",
           es[0] / 148, 100 * es[1] / es[0], 100 * es[2] / es[0], 100 * es[3] / es[0]);
  cudaFree(A);
  cudaFree(B);
  cudaFree(O);
  cudaFree(Y);
  cudaFree(bias);
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const double secs = argc > 1 ? atof(argv[1]) : 2.0;
  probe<true, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16, 2>("forward 16384x16384x4096", 16384, 16384, 4096, secs);
  probe<true, K_MAJOR, K_MAJOR, EPI_DTANH_BF16, 2>("dgrad 16384x16384x4096", 16384, 16384, 4096, secs);
  probe<true, MN_MAJOR, MN_MAJOR, EPI_F32_ACC, 2>("wgrad 4096x16384x16384", 4096, 16384, 16384, secs);
  if (argc > 2 && argv[2][0] == 'w') return 0;  // "wide": the MH = 2 kernels only
  probe<false, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16>("forward 16384x16384x4096", 16384, 16384, 4096, secs);
  probe<true, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16>("forward 16384x16384x4096", 16384, 16384, 4096, secs);
  probe<false, K_MAJOR, K_MAJOR, EPI_DTANH_BF16>("dgrad 16384x4096x16384", 16384, 4096, 16384, secs);
  probe<true, K_MAJOR, K_MAJOR, EPI_DTANH_BF16>("dgrad 16384x4096x16384", 16384, 4096, 16384, secs);
  probe<false, MN_MAJOR, MN_MAJOR, EPI_F32_ACC>("wgrad 4096x16384x16384", 4096, 16384, 16384, secs);
  probe<true, MN_MAJOR, MN_MAJOR, EPI_F32_ACC>("wgrad 4096x16384x16384", 4096, 16384, 16384, secs);
  probe<false, K_MAJOR, K_MAJOR, EPI_BF16>("plain KK 16384x16384x4096", 16384, 16384, 4096, secs);
  return 0;
}
