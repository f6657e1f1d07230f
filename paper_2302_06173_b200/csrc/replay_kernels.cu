// Replay compute of one pipeline stage on the B200 (rows a16-a19 of SURVEY §8):
//   forward_stage  (model.cpp:77-92, affine_tanh :59-73)
//   backward_stage (model.cpp:94-156)
//   accumulate_grads / ordered_sum across micro-batches (model.cpp:158-172)
//   mse_loss gradient (model.cpp:174-188), synth inputs (:190-198)
//
// Precision: activations, weights and dz are bf16 GEMM operands; the tensor
// cores accumulate in fp32; parameter gradients are accumulated in fp32 in
// ascending micro-batch order (left to right, like ordered_sum).  Results
// are tolerance-matched to the fp64 reference and bit-reproducible run to
// run (fixed tiling, no atomics) — the replay-equals-ghost-run contract.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"
#include "umma_gemm_host.h"

namespace rwb {
namespace {

using bf16 = __nv_bfloat16;
constexpr int kBN = 256;
constexpr int kPairDefault = 2;  // the wide CTA-pair kernel (profiles/r02/engines3.log)

__device__ __forceinline__ bf16 dtanh1(bf16 g, bf16 y) {
  // dz = dL/dy * (1 - y^2)   (model.cpp:113-120)
  const float yv = __bfloat162float(y);
  return __float2bfloat16_rn(__fmul_rn(__bfloat162float(g), __fsub_rn(1.f, __fmul_rn(yv, yv))));
}
// 8 elements per thread per step (16-byte loads / store) when the pointers allow
__global__ void dtanh_first_kernel(const bf16* __restrict__ g, const bf16* __restrict__ y,
                                   bf16* __restrict__ dz, uint64_t n) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x, nt = uint64_t(gridDim.x) * blockDim.x;
  uint64_t done = 0;
  if (((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(dz)) & 15u) ==
      0) {
    const uint64_t n8 = n / 8;
    for (uint64_t i = tid; i < n8; i += nt) {
      const uint4 gv = __ldg(reinterpret_cast<const uint4*>(g) + i);
      const uint4 yv = __ldg(reinterpret_cast<const uint4*>(y) + i);
      const bf16* gp = reinterpret_cast<const bf16*>(&gv);
      const bf16* yp = reinterpret_cast<const bf16*>(&yv);
      uint4 o;
      bf16* op = reinterpret_cast<bf16*>(&o);
#pragma unroll
      for (int k = 0; k < 8; ++k) op[k] = dtanh1(gp[k], yp[k]);
      reinterpret_cast<uint4*>(dz)[i] = o;
    }
    done = n8 * 8;
  }
  for (uint64_t i = done + tid; i < n; i += nt) dz[i] = dtanh1(g[i], y[i]);
}

// db[c] (+)= sum_r dz[r, c]: fixed two-level order (row splits summed in order)
constexpr int kColSplit = 64;
// one thread per column pair (4-byte loads: 128 contiguous bytes per warp and
// row), rows of split s summed in order
__global__ void colsum_partial_kernel(const bf16* __restrict__ dz, int64_t rows, int64_t cols,
                                      float* __restrict__ part) {
  const int64_t c = 2 * (blockIdx.x * int64_t(blockDim.x) + threadIdx.x);
  const int s = blockIdx.y;
  if (c >= cols) return;
  const int64_t r0 = rows * s / kColSplit, r1 = rows * (s + 1) / kColSplit;
  float a0 = 0.f, a1 = 0.f;
  if (c + 1 < cols && (cols & 1) == 0) {
    for (int64_t r = r0; r < r1; ++r) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dz + r * cols + c));
      a0 = __fadd_rn(a0, f.x);
      a1 = __fadd_rn(a1, f.y);
    }
    part[int64_t(s) * cols + c] = a0;
    part[int64_t(s) * cols + c + 1] = a1;
  } else {
    for (int64_t r = r0; r < r1; ++r) {
      a0 = __fadd_rn(a0, __bfloat162float(dz[r * cols + c]));
      if (c + 1 < cols) a1 = __fadd_rn(a1, __bfloat162float(dz[r * cols + c + 1]));
    }
    part[int64_t(s) * cols + c] = a0;
    if (c + 1 < cols) part[int64_t(s) * cols + c + 1] = a1;
  }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int64_t nsplit, int64_t cols,
                                    float* __restrict__ db, int accumulate) {
  const int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  float acc = part[c];
  for (int64_t s = 1; s < nsplit; ++s) acc = __fadd_rn(acc, part[s * cols + c]);
  db[c] = accumulate ? __fadd_rn(db[c], acc) : acc;
}

// 8 elements per thread per step (two 16-byte loads, one 16-byte store) when
// both pointers allow it; the scalar loop covers the rest
__global__ void cast_f32_bf16_kernel(const float* __restrict__ in, bf16* __restrict__ out, uint64_t n) {
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x, nt = uint64_t(gridDim.x) * blockDim.x;
  uint64_t done = 0;
  if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15u) == 0) {
    const uint64_t n8 = n / 8;
    const float4* i4 = reinterpret_cast<const float4*>(in);
    uint4* o4 = reinterpret_cast<uint4*>(out);
    for (uint64_t i = tid; i < n8; i += nt) {
      const float4 a = __ldg(i4 + 2 * i), b = __ldg(i4 + 2 * i + 1);
      __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(a.z, a.w);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(b.x, b.y), h3 = __floats2bfloat162_rn(b.z, b.w);
      uint4 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&h0);
      pk.y = *reinterpret_cast<uint32_t*>(&h1);
      pk.z = *reinterpret_cast<uint32_t*>(&h2);
      pk.w = *reinterpret_cast<uint32_t*>(&h3);
      o4[i] = pk;
    }
    done = n8 * 8;
  }
  for (uint64_t i = done + tid; i < n; i += nt) out[i] = __float2bfloat16_rn(in[i]);
}

// mse_loss (model.cpp:174-188): grad = 2/(n*mbs) * (pred - target); the
// per-block partial loss sums are reduced in block order by a second pass.
__global__ void mse_grad_kernel(const bf16* __restrict__ pred, const float* __restrict__ target, uint64_t n,
                                float scale, bf16* __restrict__ grad, double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const float d = __fsub_rn(__bfloat162float(pred[i]), target[i]);
    grad[i] = __float2bfloat16_rn(__fmul_rn(scale, d));
    acc += double(d) * double(d);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void mse_final_kernel(const double* __restrict__ part, int nparts, uint64_t n, double* loss) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += part[i];
    *loss = s / double(n);
  }
}

int grid1d(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return int(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

}  // namespace

// SMs kept free of the GEMM grid while collectives run concurrently (a
// persistent grid with a static tile schedule waits for its last CTA, so a
// collective kernel holding one SM would stall the whole GEMM).
static int g_sm_reserve = 0;
int replay_set_sm_reserve(int n) {
  g_sm_reserve = n < 0 ? 0 : n;
  return 0;
}
static int gemm_cap() {
  if (g_sm_reserve == 0) return 0;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms - g_sm_reserve > 1 ? sms - g_sm_reserve : 1;
}

// GEMM engine: the single-CTA kernel (cta_group::1, M128) or the CTA-pair
// kernel (cta_group::2, M256: each SM stages half of the B tile, so L2->SM
// traffic per FLOP drops by a third).  RW_GEMM_PAIR=0/1 overrides the default.
// pair = 2: the wide CTA-pair kernel (256 rows per CTA, 512 per pair).
static int g_pair_override = -1;
static int pair_mode() {
  if (g_pair_override >= 0) return g_pair_override;
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RW_GEMM_PAIR");
    v = (e && *e) ? std::atoi(e) : kPairDefault;
  }
  return v;
}
int replay_set_gemm_engine(int epilogue, int pair) {
  gemm::tma_epi_override() = epilogue < 0 ? -1 : (epilogue != 0);
  g_pair_override = pair < 0 ? -1 : pair;
  return 0;
}
template <int AM, int BMJ, int EPI>
static int gemm_run(const void* A, int64_t lda, const void* B, int64_t ldb, int M, int N, int K,
                    const gemm::EpiArgs& ep, cudaStream_t st) {
  const int pm = pair_mode();
  if (pm == 2) return gemm::launch2<kBN, AM, BMJ, EPI, 2>(A, lda, B, ldb, M, N, K, ep, st, gemm_cap());
  if (pm == 1) return gemm::launch2<kBN, AM, BMJ, EPI>(A, lda, B, ldb, M, N, K, ep, st, gemm_cap());
  return gemm::launch<kBN, AM, BMJ, EPI>(A, lda, B, ldb, M, N, K, ep, st, gemm_cap());
}

int replay_forward_layer(const void* x, int64_t rows, int64_t in, int64_t out, const void* w, const float* b,
                         void* y, void* stream) {
  gemm::EpiArgs ep{};
  ep.out = y;
  ep.ldo = out;
  ep.bias = b;
  // Y[R,out] = X[R,in] . W[in,out]: A = X (K-major), B = W viewed [out,in] (MN-major)
  return gemm_run<gemm::K_MAJOR, gemm::MN_MAJOR, gemm::EPI_BIAS_TANH_BF16>(
      x, in, w, out, int(rows), int(out), int(in), ep, static_cast<cudaStream_t>(stream));
}

int replay_dgrad_layer(const void* dz, int64_t rows, int64_t in, int64_t out, const void* w,
                       const void* y_prev, void* dst, void* stream, float* colsum, int* fused) {
  gemm::EpiArgs ep{};
  ep.out = dst;
  ep.ldo = in;
  ep.y = static_cast<const bf16*>(y_prev);
  ep.ldy = in;
  auto st = static_cast<cudaStream_t>(stream);
  if (fused) *fused = 0;
  // dX[R,in] = dZ[R,out] . W[in,out]^T: A = dZ (K-major), B = W as [in,out] (K-major)
  if (y_prev) {
    if (colsum && gemm::tma_epi_enabled()) {
      ep.colsum = colsum;
      ep.ldc = in;
      const int e = gemm_run<gemm::K_MAJOR, gemm::K_MAJOR, gemm::EPI_DTANH_BF16>(dz, out, w, out, int(rows),
                                                                                 int(in), int(out), ep, st);
      if (e != static_cast<int>(cudaErrorNotSupported)) {
        if (fused && e == 0) *fused = 1;
        return e;
      }
      ep.colsum = nullptr;  // not a TMA operand: plain epilogue, the caller sums the columns
    }
    return gemm_run<gemm::K_MAJOR, gemm::K_MAJOR, gemm::EPI_DTANH_BF16>(dz, out, w, out, int(rows),
                                                                                 int(in), int(out), ep, st);
  }
  return gemm_run<gemm::K_MAJOR, gemm::K_MAJOR, gemm::EPI_BF16>(dz, out, w, out, int(rows), int(in),
                                                                         int(out), ep, st);
}

int replay_dgrad_boundary(const void* dz, int64_t rows, int64_t in, int64_t out, const void* w,
                          const void* y_prev_stage, void* dz_prev_stage, void* stream) {
  gemm::EpiArgs ep{};
  ep.out = dz_prev_stage;
  ep.ldo = in;
  ep.y = static_cast<const bf16*>(y_prev_stage);
  ep.ldy = in;
  return gemm_run<gemm::K_MAJOR, gemm::K_MAJOR, gemm::EPI_BOUNDARY_DTANH_BF16>(
      dz, out, w, out, int(rows), int(in), int(out), ep, static_cast<cudaStream_t>(stream));
}

int replay_wgrad_layer(const void* x, const void* dz, int64_t rows, int64_t in, int64_t out, float* dw,
                       int accumulate, void* stream) {
  gemm::EpiArgs ep{};
  ep.out = dw;
  ep.ldo = out;
  auto st = static_cast<cudaStream_t>(stream);
  // dW[in,out] = X[R,in]^T . dZ[R,out]: A(m=in,k=r) = X[r,m] (MN-major), B(n=out,k=r) = dZ[r,n] (MN-major)
  if (accumulate)
    return gemm_run<gemm::MN_MAJOR, gemm::MN_MAJOR, gemm::EPI_F32_ACC>(x, in, dz, out, int(in), int(out),
                                                                                int(rows), ep, st);
  return gemm_run<gemm::MN_MAJOR, gemm::MN_MAJOR, gemm::EPI_F32>(x, in, dz, out, int(in), int(out),
                                                                          int(rows), ep, st);
}

int replay_dtanh_first(const void* g, const void* y, void* dz, uint64_t n, void* stream) {
  dtanh_first_kernel<<<grid1d(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(g), static_cast<const bf16*>(y), static_cast<bf16*>(dz), n);
  return static_cast<int>(cudaGetLastError());
}

int replay_colsum(const void* dz, int64_t rows, int64_t cols, float* db, float* scratch, int accumulate,
                  void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  dim3 g(unsigned((cols + 255) / 256), kColSplit);  // 128 threads x 2 columns
  colsum_partial_kernel<<<g, 128, 0, st>>>(static_cast<const bf16*>(dz), rows, cols, scratch);
  colsum_final_kernel<<<unsigned((cols + 127) / 128), 128, 0, st>>>(scratch, kColSplit, cols, db, accumulate);
  return static_cast<int>(cudaGetLastError());
}

// Many partial rows (the fused db partials, ceil(rows/32) of them): 8 row
// lanes per column each sum a contiguous eighth in row order, then the eight
// sums are added in lane order -- a fixed order, more loads in flight.
__global__ void colsum_final8_kernel(const float* __restrict__ part, int64_t nsplit, int64_t cols,
                                     float* __restrict__ db, int accumulate) {
  __shared__ float sh[8][32];
  const int64_t c = blockIdx.x * int64_t(32) + threadIdx.x;
  const int j = threadIdx.y;
  const int64_t s0 = nsplit * j / 8, s1 = nsplit * (j + 1) / 8;
  float acc = 0.f;
  if (c < cols)
    for (int64_t s = s0; s < s1; ++s) acc = __fadd_rn(acc, part[s * cols + c]);
  sh[j][threadIdx.x] = acc;
  __syncthreads();
  if (j == 0 && c < cols) {
    float t = sh[0][threadIdx.x];
#pragma unroll
    for (int q = 1; q < 8; ++q) t = __fadd_rn(t, sh[q][threadIdx.x]);
    db[c] = accumulate ? __fadd_rn(db[c], t) : t;
  }
}

int replay_colsum_final(const float* part, int64_t nsplit, int64_t cols, float* db, int accumulate, void* stream) {
  colsum_final8_kernel<<<unsigned((cols + 31) / 32), dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(
      part, nsplit, cols, db, accumulate);
  return static_cast<int>(cudaGetLastError());
}

int replay_cast_bf16(const float* in, void* out, uint64_t n, void* stream) {
  cast_f32_bf16_kernel<<<grid1d(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(in, static_cast<bf16*>(out), n);
  return static_cast<int>(cudaGetLastError());
}

int replay_mse_grad(const void* pred, const float* target, uint64_t n, uint64_t micro_batches, void* grad,
                    double* loss, double* scratch, void* stream) {
  auto st = static_cast<cudaStream_t>(stream);
  const int blocks = 256;
  const float scale = static_cast<float>(2.0 / (double(n) * double(micro_batches)));
  mse_grad_kernel<<<blocks, 256, 0, st>>>(static_cast<const bf16*>(pred), target, n, scale,
                                          static_cast<bf16*>(grad), scratch);
  if (loss) mse_final_kernel<<<1, 32, 0, st>>>(scratch, blocks, n, loss);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace rwb
