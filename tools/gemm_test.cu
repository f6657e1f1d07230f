// Standalone correctness + throughput harness for csrc/umma_gemm.cuh
// (tcgen05/TMEM/TMA bf16 GEMM).  Compares against a naive fp32-accumulate
// SIMT GEMM over the same bf16 operands, for all operand majors used by the
// replay (forward K/MN, dgrad K/K, wgrad MN/MN) and the fused epilogues.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_2302_06173_b200/csrc -o tools/gemm_test tools/gemm_test.cu
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "umma_gemm_host.h"

using namespace rwb::gemm;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <int BN, int AM, int BMJ, int EPI, bool PAIR>
int run_gemm(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K, const EpiArgs& ep,
             cudaStream_t s) {
  if constexpr (PAIR) return launch2<BN, AM, BMJ, EPI>(A, lda, B, ldb, M, N, K, ep, s);
  else return launch<BN, AM, BMJ, EPI>(A, lda, B, ldb, M, N, K, ep, s);
}

__global__ void fill_bf16(__nv_bfloat16* p, size_t n, uint32_t seed, float scale) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint32_t h = uint32_t(i) * 2654435761u ^ seed;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    p[i] = __float2bfloat16((float(h & 0xffff) / 65536.f - 0.5f) * scale);
  }
}

// C[m,n] = sum_k A(m,k) B(n,k); A(m,k) = amaj==0 ? A[m*lda+k] : A[k*lda+m]
__global__ void ref_gemm(const __nv_bfloat16* A, int64_t lda, int amaj, const __nv_bfloat16* B, int64_t ldb,
                         int bmaj, float* C, int M, int N, int K) {
  int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N || m >= M) return;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) {
    float a = __bfloat162float(amaj == 0 ? A[int64_t(m) * lda + k] : A[int64_t(k) * lda + m]);
    float b = __bfloat162float(bmaj == 0 ? B[int64_t(n) * ldb + k] : B[int64_t(k) * ldb + n]);
    acc = fmaf(a, b, acc);
  }
  C[int64_t(m) * N + n] = acc;
}

template <int BN, int AM, int BMJ, int EPI, bool PAIR = false>
bool check(const char* name, int M, int N, int K) {
  size_t na = size_t(M) * K, nb = size_t(N) * K;
  __nv_bfloat16 *A, *B, *Y, *O;
  float *C, *R, *bias;
  CK(cudaMalloc(&A, na * 2));
  CK(cudaMalloc(&B, nb * 2));
  CK(cudaMalloc(&C, size_t(M) * N * 4));
  CK(cudaMalloc(&R, size_t(M) * N * 4));
  CK(cudaMalloc(&O, size_t(M) * N * 2));
  CK(cudaMalloc(&Y, size_t(M) * N * 2));
  CK(cudaMalloc(&bias, size_t(N) * 4));
  fill_bf16<<<512, 256>>>(A, na, 1, 1.0f);
  fill_bf16<<<512, 256>>>(B, nb, 2, 1.0f);
  fill_bf16<<<512, 256>>>(Y, size_t(M) * N, 3, 1.8f);
  std::vector<float> hb(N);
  for (int i = 0; i < N; ++i) hb[i] = 0.01f * (i % 17) - 0.05f;
  CK(cudaMemcpy(bias, hb.data(), N * 4, cudaMemcpyHostToDevice));
  const int64_t lda = AM == K_MAJOR ? K : M, ldb = BMJ == K_MAJOR ? K : N;
  EpiArgs ep{};
  ep.ldo = N;
  ep.bias = bias;
  ep.y = Y;
  ep.ldy = N;
  if (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
    ep.out = C;
    CK(cudaMemset(C, 0, size_t(M) * N * 4));
  } else {
    ep.out = O;
  }
  int e = run_gemm<BN, AM, BMJ, EPI, PAIR>(A, lda, B, ldb, M, N, K, ep, 0);
  if (e) {
    printf("%s: launch error %d\n", name, e);
    return false;
  }
  if (EPI == EPI_F32_ACC) {  // second pass accumulates: result = 2 * C
    e = run_gemm<BN, AM, BMJ, EPI, PAIR>(A, lda, B, ldb, M, N, K, ep, 0);
  }
  CK(cudaDeviceSynchronize());
  dim3 g((N + 127) / 128, M);
  ref_gemm<<<g, 128>>>(A, lda, AM, B, ldb, BMJ, R, M, N, K);
  CK(cudaDeviceSynchronize());
  std::vector<float> hr(size_t(M) * N), hc(size_t(M) * N), hy(size_t(M) * N);
  std::vector<__nv_bfloat16> ho(size_t(M) * N), hyb(size_t(M) * N);
  CK(cudaMemcpy(hr.data(), R, hr.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hyb.data(), Y, hyb.size() * 2, cudaMemcpyDeviceToHost));
  if (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
    CK(cudaMemcpy(hc.data(), C, hc.size() * 4, cudaMemcpyDeviceToHost));
  } else {
    CK(cudaMemcpy(ho.data(), O, ho.size() * 2, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < ho.size(); ++i) hc[i] = __bfloat162float(ho[i]);
  }
  // the TMA-staged epilogue must equal the register epilogue bit for bit
  bool same = true;
  {
    tma_epi_override() = 0;
    if (EPI == EPI_F32 || EPI == EPI_F32_ACC) CK(cudaMemset(C, 0, size_t(M) * N * 4));
    run_gemm<BN, AM, BMJ, EPI, PAIR>(A, lda, B, ldb, M, N, K, ep, 0);
    if (EPI == EPI_F32_ACC) run_gemm<BN, AM, BMJ, EPI, PAIR>(A, lda, B, ldb, M, N, K, ep, 0);
    CK(cudaDeviceSynchronize());
    tma_epi_override() = -1;
    if (EPI == EPI_F32 || EPI == EPI_F32_ACC) {
      std::vector<float> h2(size_t(M) * N);
      CK(cudaMemcpy(h2.data(), C, h2.size() * 4, cudaMemcpyDeviceToHost));
      same = std::memcmp(h2.data(), hc.data(), h2.size() * 4) == 0;
    } else {
      std::vector<__nv_bfloat16> h2(size_t(M) * N);
      CK(cudaMemcpy(h2.data(), O, h2.size() * 2, cudaMemcpyDeviceToHost));
      same = std::memcmp(h2.data(), ho.data(), h2.size() * 2) == 0;
    }
  }
  double max_err = 0, max_ref = 0;
  for (size_t i = 0; i < hr.size(); ++i) {
    double ref = hr[i];
    const int n = int(i % N);
    if (EPI == EPI_BIAS_TANH_BF16) ref = std::tanh(ref + hb[n]);
    if (EPI == EPI_DTANH_BF16 || EPI == EPI_BOUNDARY_DTANH_BF16) {
      double y = __bfloat162float(hyb[i]);
      ref = ref * (1.0 - y * y);
    }
    if (EPI == EPI_F32_ACC) ref = 2 * ref;
    max_err = std::fmax(max_err, std::fabs(ref - hc[i]));
    max_ref = std::fmax(max_ref, std::fabs(ref));
  }
  // bf16 output: ~2^-8 relative; fp32 accumulation-order differences ~1e-6
  const double tol = (EPI == EPI_F32 || EPI == EPI_F32_ACC) ? 1e-4 * max_ref + 1e-3 : 1e-2 * max_ref + 1e-2;
  bool ok = max_err <= tol && std::isfinite(max_err) && same;
  printf("%-34s M=%5d N=%5d K=%5d  max|err|=%.3e  max|ref|=%.3e  %s%s\n", name, M, N, K, max_err, max_ref,
         ok ? "OK" : "FAIL", same ? "  (tma == register epilogue)" : "  (tma != register epilogue)");
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  cudaFree(R);
  cudaFree(O);
  cudaFree(Y);
  cudaFree(bias);
  return ok;
}

template <int BN, int AM, int BMJ, int EPI, bool PAIR = false>
void perf(const char* name, int M, int N, int K, int reps = 10) {
  __nv_bfloat16 *A, *B, *O;
  float* bias;
  CK(cudaMalloc(&A, size_t(M) * K * 2));
  CK(cudaMalloc(&B, size_t(N) * K * 2));
  CK(cudaMalloc(&O, size_t(M) * N * 4));
  CK(cudaMalloc(&bias, size_t(N) * 4));
  CK(cudaMemset(bias, 0, N * 4));
  fill_bf16<<<512, 256>>>(A, size_t(M) * K, 1, 1.0f);
  fill_bf16<<<512, 256>>>(B, size_t(N) * K, 2, 1.0f);
  const int64_t lda = AM == K_MAJOR ? K : M, ldb = BMJ == K_MAJOR ? K : N;
  EpiArgs ep{};
  ep.out = O;
  ep.ldo = N;
  ep.bias = bias;
  ep.y = reinterpret_cast<__nv_bfloat16*>(O);
  ep.ldy = N;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  run_gemm<BN, AM, BMJ, EPI, PAIR>(A, lda, B, ldb, M, N, K, ep, 0);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    run_gemm<BN, AM, BMJ, EPI, PAIR>(A, lda, B, ldb, M, N, K, ep, 0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  const double tf = 2.0 * M * N * K / (best * 1e-3) / 1e12;
  printf("PERF %-30s M=%5d N=%5d K=%5d  %.3f ms  %.1f TFLOP/s\n", name, M, N, K, best, tf);
  cudaFree(A);
  cudaFree(B);
  cudaFree(O);
  cudaFree(bias);
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  bool all = true;
  all &= check<256, K_MAJOR, K_MAJOR, EPI_F32>("KK f32 (dgrad layout)", 256, 512, 256);
  all &= check<256, K_MAJOR, MN_MAJOR, EPI_F32>("K/MN f32 (forward layout)", 256, 512, 256);
  all &= check<256, MN_MAJOR, MN_MAJOR, EPI_F32>("MN/MN f32 (wgrad layout)", 256, 512, 256);
  all &= check<256, MN_MAJOR, K_MAJOR, EPI_F32>("MN/K f32", 256, 512, 256);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_F32>("KK f32 ragged", 200, 300, 136);
  all &= check<256, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16>("forward bias+tanh bf16", 384, 768, 512);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_DTANH_BF16>("dgrad *(1-y^2) bf16", 384, 512, 768);
  all &= check<256, MN_MAJOR, MN_MAJOR, EPI_F32_ACC>("wgrad f32 accumulate", 512, 256, 1024);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_BF16>("KK bf16 big", 2048, 2048, 2048);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_BOUNDARY_DTANH_BF16>("boundary bf16(acc)*(1-y^2)", 384, 512, 768);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_DTANH_BF16>("dgrad dtanh ragged (TMA edge)", 200, 264, 136);
  all &= check<256, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16>("forward ragged (TMA edge)", 200, 264, 136);
  // (MN-major operands need M, N multiples of 8: a TMA row pitch is a multiple of 16 bytes)
  all &= check<256, MN_MAJOR, MN_MAJOR, EPI_F32_ACC>("wgrad acc ragged (TMA edge)", 208, 296, 136);
  // CTA-pair (cta_group::2) kernel
  all &= check<256, K_MAJOR, K_MAJOR, EPI_F32, true>("PAIR KK f32", 512, 512, 256);
  all &= check<256, K_MAJOR, MN_MAJOR, EPI_F32, true>("PAIR K/MN f32", 512, 512, 256);
  all &= check<256, MN_MAJOR, MN_MAJOR, EPI_F32, true>("PAIR MN/MN f32", 512, 512, 256);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_F32, true>("PAIR KK f32 ragged", 300, 300, 136);
  all &= check<256, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16, true>("PAIR forward bias+tanh", 512, 768, 512);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_DTANH_BF16, true>("PAIR dgrad dtanh", 512, 512, 768);
  all &= check<256, MN_MAJOR, MN_MAJOR, EPI_F32_ACC, true>("PAIR wgrad accumulate", 512, 256, 1024);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_BF16, true>("PAIR KK bf16 big", 2048, 2048, 2048);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_BOUNDARY_DTANH_BF16, true>("PAIR boundary", 512, 512, 768);
  all &= check<256, K_MAJOR, K_MAJOR, EPI_DTANH_BF16, true>("PAIR dgrad dtanh ragged", 200, 264, 136);
  all &= check<256, MN_MAJOR, MN_MAJOR, EPI_F32_ACC, true>("PAIR wgrad acc ragged", 208, 296, 136);
  printf("correctness: %s\n", all ? "ALL OK" : "FAILURES");
  if (argc > 1) {
    perf<256, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16>("forward 16384x16384x4096", 16384, 16384, 4096);
    perf<256, K_MAJOR, K_MAJOR, EPI_BF16>("dgrad 16384x4096x16384", 16384, 4096, 16384);
    perf<256, MN_MAJOR, MN_MAJOR, EPI_F32>("wgrad 4096x16384x16384", 4096, 16384, 16384);
    perf<256, K_MAJOR, K_MAJOR, EPI_BF16>("KK 8192^3", 8192, 8192, 8192);
    perf<256, K_MAJOR, MN_MAJOR, EPI_BIAS_TANH_BF16, true>("PAIR forward 16384x16384x4096", 16384, 16384, 4096);
    perf<256, K_MAJOR, K_MAJOR, EPI_BF16, true>("PAIR dgrad 16384x4096x16384", 16384, 4096, 16384);
    perf<256, MN_MAJOR, MN_MAJOR, EPI_F32, true>("PAIR wgrad 4096x16384x16384", 4096, 16384, 16384);
    perf<256, K_MAJOR, K_MAJOR, EPI_BF16, true>("PAIR KK 8192^3", 8192, 8192, 8192);
    perf<256, K_MAJOR, K_MAJOR, EPI_DTANH_BF16, true>("PAIR dgrad-dtanh 16384x16384x4096", 16384, 16384, 4096);
    perf<128, K_MAJOR, K_MAJOR, EPI_BF16, true>("PAIR BN128 KK 8192^3", 8192, 8192, 8192);
    perf<128, K_MAJOR, K_MAJOR, EPI_BF16, false>("BN128 KK 8192^3", 8192, 8192, 8192);
  }
  return all ? 0 : 1;
}
